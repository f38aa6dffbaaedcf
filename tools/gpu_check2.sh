# tests + LN micro-bench + warm-L2 launch lists (ncu --cache-control none) + C3 slice + bench
O=gpurun_out/g6; mkdir -p $O; rm -f $O/*
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
for sh in "8192 4096" "4096 2048"; do timeout 120 python tools/ln_bench.py $sh 2>&1 | grep -v "^{" >> $O/ln.log; done
timeout 300 python tools/rank_slice.py --config c3 --tp 8 > $O/c3.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > $O/bench.log 2>&1
for C in c2:1 c3:8; do CONFIG=${C%:*} TP=${C#*:} LAYERS=2 STEPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file $O/${C%:*}_warm.csv python tools/profile_slice.py > /dev/null 2>&1; done
