# LayerNorm kernel check: micro-bench (OASES_LNP=0 one-shot vs 1 persistent), GPU tests,
# C3 TMP=8 rank slice, bench, C2/C3 launch lists of one eager step (L=1)
O=gpurun_out/g2; mkdir -p $O; rm -f $O/ln_bench.log
for L in 0 1; do for sh in "8192 4096" "4096 2048"; do OASES_LNP=$L timeout 120 python tools/ln_bench.py $sh >> $O/ln_bench.log 2>&1; done; done
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo pytest $? >> $O/pytest.log
timeout 300 python tools/rank_slice.py --config c3 --tp 8 > $O/c3.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > $O/bench.log 2>&1
for C in c2:1 c3:8; do CONFIG=${C%:*} TP=${C#*:} LAYERS=1 STEPS=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/${C%:*}_launches.csv python tools/profile_slice.py > /dev/null 2>&1; done
