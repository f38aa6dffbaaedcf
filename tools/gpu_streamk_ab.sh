# stream-K GEMM tail: correctness (GEMM + stack tests, hang-guarded) and step A/B
O=gpurun_out/sk; mkdir -p $O; rm -f $O/*
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q > $O/pytest_gemm.log 2>&1; echo rc $? >> $O/pytest_gemm.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
for M in 1 0 1 0; do OASES_STREAMK=$M timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 15 > $O/bench_sk$M.log 2>&1; python -c "
import json;d=json.loads(open('$O/bench_sk$M.log').read().strip().splitlines()[-1]);print('streamk=$M', d['value'],d['ms_per_step'],d['clocks']['sm_mhz'], d['roofline']['achieved'])" >> $O/ab.log; done
for M in 1 0; do OASES_STREAMK=$M timeout 300 python tools/rank_slice.py --config c3 --tp 8 >> $O/c3.log 2>&1; done
