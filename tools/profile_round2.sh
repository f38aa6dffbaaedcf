# Round-2 evidence in one GPU call (run under gpurun from the repo root):
#   bench line (default run, CPU baseline included), launch list of one bench step,
#   ncu --set full summaries (JSON; the .ncu-rep files are dropped to stay under the
#   64 MiB copy-back) of the LayerNorm row kernels (C2 and C3-rank shapes), the attention
#   kernels (C2 and a C3 rank) and the dominant GEMMs; C3/C4 TMP=8 rank slices.
O=gpurun_out/final; rm -rf $O; mkdir -p $O
S="python tools/ncu_kernel_summary.py"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 600 python bench.py > $O/bench.log 2>&1
timeout 300 python tools/rank_slice.py --config c3 --tp 8 > $O/c3_tp8.log 2>&1
timeout 300 python tools/rank_slice.py --config c4 --tp 8 > $O/c4_tp8.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
    --log-file $O/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras > $O/bench_under_ncu.log 2>&1
for sh in "4096 2048" "8192 4096"; do set -- $sh
  timeout 300 ncu --set full --clock-control none -k regex:lnp_ -c 4 -f -o $O/lnp python tools/lnp_one.py $1 $2 > /dev/null 2>&1
  $S $O/lnp.ncu-rep > $O/ncu_lnp_${1}x${2}.json 2>&1; rm -f $O/lnp.ncu-rep
done
MODE=2 ITERS=1 REP=1 timeout 300 ncu --set full --clock-control none -k regex:"attn_(fwd|dkdv)" -c 2 -f -o $O/a python tools/attn_one.py > /dev/null 2>&1
$S $O/a.ncu-rep > $O/ncu_attn_c2_cached.json 2>&1; rm -f $O/a.ncu-rep
MODE=0 ITERS=1 REP=1 OASES_ATTN_FWD2=0 timeout 300 ncu --set full --clock-control none -k regex:"attn_(fwd|dkdv)" -c 2 -f -o $O/a python tools/attn_one.py > /dev/null 2>&1
$S $O/a.ncu-rep > $O/ncu_attn_c2_philox.json 2>&1; rm -f $O/a.ncu-rep
MODE=2 ITERS=1 REP=1 N=4 HL=4 SEQ=2048 timeout 300 ncu --set full --clock-control none -k regex:"attn_(fwd|dkdv)" -c 2 -f -o $O/a python tools/attn_one.py > /dev/null 2>&1
$S $O/a.ncu-rep > $O/ncu_attn_c3rank_cached.json 2>&1; rm -f $O/a.ncu-rep
SHAPE=4096,8192,2048 ITERS=2 timeout 300 ncu --set full --clock-control none -k regex:gemm_tc2 -s 1 -c 1 -f -o $O/g python tools/gemm_one.py > /dev/null 2>&1
$S $O/g.ncu-rep > $O/ncu_gemm_fc1.json 2>&1; rm -f $O/g.ncu-rep
ITERS=2 timeout 300 ncu --set full --clock-control none -k regex:gemm_tc2 -s 2 -c 2 -f -o $O/g python tools/epi_one.py > /dev/null 2>&1
$S $O/g.ncu-rep > $O/ncu_gemm_epi.json 2>&1; rm -f $O/g.ncu-rep
CONFIG=c3 TP=8 LAYERS=2 STEPS=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/c3_tp8_launches.csv python tools/profile_slice.py > /dev/null 2>&1
du -sh $O; ls -la $O
