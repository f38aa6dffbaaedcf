# quick round-2 check: C2/C3 launch lists of one eager step (L=1), C3 rank slice, bench
O=gpurun_out/q; mkdir -p $O
timeout 300 python tools/rank_slice.py --config c3 --tp 8 > $O/c3.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > $O/bench.log 2>&1
for C in c2:1 c3:8; do CONFIG=${C%:*} TP=${C#*:} LAYERS=1 STEPS=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/${C%:*}_launches.csv python tools/profile_slice.py > /dev/null 2>&1; done
