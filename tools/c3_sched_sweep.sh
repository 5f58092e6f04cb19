XTSG_TTM_SCHED=2 XTSG_TTM_SYNCJ=1 timeout 300 python -m pytest tests/test_gpu_plan.py -x -q 2>&1 | tail -1
for sj in 0 8 2 1; do for g in 8 12; do
echo "syncj $sj group $g"; XTSG_TTM_SCHED=2 XTSG_TTM_SYNCJ=$sj XTSG_TTM_L2HINT=0 XTSG_TTM_GROUP=$g timeout 300 python tools/c3_compress_probe.py 400
done; done
XTSG_TTM_SCHED=2 XTSG_TTM_SYNCJ=1 XTSG_TTM_L2HINT=0 XTSG_TTM_GROUP=8 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:ttm_pair -c 2 --csv --log-file gpurun_out/c3_syncj1.csv python tools/c3_compress_probe.py 80 > /dev/null 2>&1
