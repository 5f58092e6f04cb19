# C3 pair-kernel DRAM traffic vs schedule: for each (row-block group, lane
# barrier spacing, L2 hint) one timed 400-slice probe and one ncu metric pass
# over a single 40-slice TTM launch.
cd ${GRAFT_REPO_ROOT:-.}
M=gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct
for cfg in "8 0 1" "8 4 1" "4 4 1" "6 4 1" "16 4 1" "8 4 2" "8 4 0" "4 0 1"; do
  set -- $cfg
  echo "== group $1 syncj $2 l2hint $3"
  XTSG_TTM_GROUP=$1 XTSG_TTM_SYNCJ=$2 XTSG_TTM_L2HINT=$3 timeout 300 python tools/c3_compress_probe.py 400
  XTSG_TTM_GROUP=$1 XTSG_TTM_SYNCJ=$2 XTSG_TTM_L2HINT=$3 timeout 300 ncu --metrics $M --clock-control none -k regex:ttm_pair --launch-skip 1 -c 1 --csv python tools/c3_compress_probe.py 80 2>/dev/null | grep -E '"(gpu__time|dram__bytes|sm__cycles|sm__pipe|lts__t)' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
