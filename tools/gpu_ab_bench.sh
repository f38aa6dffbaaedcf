# bench A/B on one box: liboases_old.so (previous build) vs the in-tree build, alternating, + tests
O=gpurun_out/ab; mkdir -p $O; rm -f $O/*
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_stack_gpu.py tests/test_parity_baseline_gpu.py -x -q > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
for i in 1 2; do
  OASES_LIB=$PWD/liboases_old.so timeout 300 python bench.py --steps 10 --warmup 3 2>/dev/null | tail -1 > $O/old$i.json
  timeout 300 python bench.py --steps 10 --warmup 3 2>/dev/null | tail -1 > $O/new$i.json
done
