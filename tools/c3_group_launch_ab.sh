# C3: one TTM launch per row-block group with the group's U rows in a
# persisting L2 window (XTSG_TTM_GROUP_LAUNCH=G) vs the single launch
cd ${GRAFT_REPO_ROOT:-.}
M=gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for cfg in "0 8 8" "8 8 8" "16 16 8" "8 8 16" "16 16 16" "0 8 8"; do
  set -- $cfg
  echo "== group_launch $1 group $2 slab_gb $3"
  XTSG_TTM_GROUP_LAUNCH=$1 XTSG_TTM_GROUP=$2 XTSG_SLAB_GB=$3 timeout 300 python tools/c3_compress_probe.py 800
done
for cfg in "8 8" "16 16"; do
  set -- $cfg
  echo "== ncu group_launch $1 group $2"
  XTSG_TTM_GROUP_LAUNCH=$1 XTSG_TTM_GROUP=$2 timeout 300 ncu --metrics $M --clock-control none -k regex:ttm_pair --launch-skip 8 -c 2 --csv python tools/c3_compress_probe.py 80 2>/dev/null | grep -E '"(gpu__time|dram__bytes|sm__cycles|sm__pipe)' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
XTSG_TTM_GROUP_LAUNCH=8 timeout 300 python -m pytest tests/test_gpu_scale_parity.py -x -q -k "C3 or c3" 2>&1 | tail -2
