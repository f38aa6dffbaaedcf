O=gpurun_out/g2; mkdir -p $O
for L in 0 1; do for sh in "8192 4096" "4096 2048"; do OASES_LNP=$L timeout 120 python tools/ln_bench.py $sh >> $O/ln_bench.log 2>&1; done; done
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo pytest $? >> $O/pytest.log
timeout 300 python tools/rank_slice.py --config c3 --tp 8 > $O/c3.log 2>&1
OASES_LNP=0 timeout 300 python tools/rank_slice.py --config c3 --tp 8 > $O/c3_lnp0.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > $O/bench.log 2>&1
CONFIG=c3 TP=8 LAYERS=1 STEPS=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/c3_launches.csv python tools/profile_slice.py > $O/c3_ncu.log 2>&1
