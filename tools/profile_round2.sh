# Round-2 evidence in one GPU call (run under gpurun from the repo root):
#   bench line (default run, CPU baseline included), launch list of one bench step,
#   ncu --set full of the LayerNorm row kernels (C2 and C3-rank shapes), the attention
#   kernels (C2, mask-pass mode) and the dominant GEMMs; C3/C4 TMP=8 rank slices.
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 600 python bench.py > $O/bench.log 2>&1
timeout 300 python tools/rank_slice.py --config c3 --tp 8 > $O/c3_tp8.log 2>&1
timeout 300 python tools/rank_slice.py --config c4 --tp 8 > $O/c4_tp8.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
    --log-file $O/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/bench_under_ncu.log 2>&1
for sh in "4096 2048" "8192 4096"; do set -- $sh
  timeout 300 ncu --set full --clock-control none -k regex:lnp_ -c 4 -f -o $O/lnp_${1}x${2} python tools/lnp_one.py $1 $2 > /dev/null 2>&1
done
MODE=2 ITERS=1 REP=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:attn_ -c 4 -f -o $O/attn_c2 python tools/attn_one.py > /dev/null 2>&1
SHAPE=4096,8192,2048 ITERS=2 timeout 300 ncu --set full --clock-control none -k regex:gemm_tc2 -s 1 -c 1 -f -o $O/gemm_fc1 python tools/gemm_one.py > /dev/null 2>&1
ls -la $O
