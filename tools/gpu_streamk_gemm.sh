# stream-K (OASES_STREAMK=1) GEMM timing A/B + correctness of the SK path (hang-guarded)
O=gpurun_out/sk2; mkdir -p $O; rm -f $O/*
OASES_STREAMK=1 timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q -k "not grouped" > $O/pytest_gemm_sk.log 2>&1; echo rc $? >> $O/pytest_gemm_sk.log
for sh in 4096,2048,8192 4096,2048,2048 4096,6144,2048 4096,8192,2048; do for M in 0 1; do SHAPE=$sh OASES_STREAMK=$M timeout 120 python tools/gemm_time.py >> $O/t.log 2>&1; done; done
