#!/bin/bash
# One GPU call's worth of ncu evidence (run under gpurun from the repo root):
#   launch list of the bench command, full captures of the dominant GEMM
#   launches, the fused attention kernels and the fused bdr+LayerNorm.
set -x
O=gpurun_out/prof
mkdir -p $O
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2600 --csv \
    --log-file $O/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/bench_under_ncu.log 2>&1
SHAPE=4096,8192,2048 ITERS=2 ncu --set full --import-source on --clock-control none -k regex:gemm_tc2 -s 1 -c 1 \
    -f -o $O/gemm_fc1 python tools/gemm_one.py > /dev/null 2>&1
ITERS=2 ncu --set full --import-source on --clock-control none -k regex:gemm_tc2 -s 2 -c 2 \
    -f -o $O/gemm_epi python tools/epi_one.py > /dev/null 2>&1
ITERS=1 REP=1 ncu --set full --import-source on --clock-control none -k regex:attn_ -c 3 \
    -f -o $O/attn python tools/attn_one.py > /dev/null 2>&1
ls -la $O
