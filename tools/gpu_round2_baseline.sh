set -x
O=gpurun_out/g1; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo pytest $? >> $O/pytest.log
timeout 300 python bench.py > $O/bench.log 2>&1
timeout 300 python tools/rank_slice.py --config c3 --tp 8 > $O/c3.log 2>&1
CONFIG=c3 TP=8 LAYERS=1 STEPS=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/c3_launches.csv python tools/profile_slice.py > $O/c3_ncu.log 2>&1
CONFIG=c2 TP=1 LAYERS=1 STEPS=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/c2_launches.csv python tools/profile_slice.py > $O/c2_ncu.log 2>&1
