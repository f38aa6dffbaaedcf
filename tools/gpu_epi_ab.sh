# A/B of the GEMM epilogue operand prefetch (liboases_old.so = previous build) + GEMM/stack tests
O=gpurun_out/epi; mkdir -p $O; rm -f $O/*
for i in 1 2; do
  OASES_LIB=$PWD/liboases_old.so timeout 120 python tools/epi_time.py >> $O/epi.log 2>&1
  timeout 120 python tools/epi_time.py >> $O/epi.log 2>&1
done
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_stack_gpu.py tests/test_attention_gpu.py -x -q > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 > $O/bench.log 2>&1
OASES_LIB=$PWD/liboases_old.so timeout 300 python bench.py --steps 10 --warmup 3 > $O/bench_old.log 2>&1
