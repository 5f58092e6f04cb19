#!/bin/bash
# C4 sparse path on the GPU box: tests, timed runs (CSF / COO), optional ncu capture of the tile kernel.
# Every step has its own timeout; the whole script stays under ~15 min.
mkdir -p gpurun_out
timeout 240 python -u -m pytest tests/test_gpu_sparse_tc.py tests/test_gpu_sparse_factors.py tests/test_gpu_edges.py tests/test_gpu_fp16.py -x -v > gpurun_out/sp_test.log 2>&1; rc=$?; echo rc=$rc >> gpurun_out/sp_test.log
tail -5 gpurun_out/sp_test.log
[ $rc -ne 0 ] && exit 1
timeout 200 python tools/measure_configs.py c4 --csf --steps 5 --warmup 2 --out gpurun_out/c4_csf.jsonl > gpurun_out/c4.log 2>&1
if [ "$1" == "coo" ]; then
timeout 200 python tools/measure_configs.py c4 --presorted --steps 3 --warmup 1 --out gpurun_out/c4_presorted.jsonl >> gpurun_out/c4.log 2>&1
timeout 200 python tools/measure_configs.py c4 --steps 3 --warmup 1 --out gpurun_out/c4_coo.jsonl >> gpurun_out/c4.log 2>&1
fi
tail -3 gpurun_out/c4.log | cut -c1-300
if [ "$1" == "ncu" ]; then
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sparse_tc_kernel -c 1 -o gpurun_out/c4_tc python tools/measure_configs.py c4 --csf --steps 1 --warmup 0 > gpurun_out/c4_ncu.log 2>&1
tail -2 gpurun_out/c4_ncu.log
fi
