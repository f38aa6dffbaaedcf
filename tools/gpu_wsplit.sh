# per-sub-batch weight gradients (OASES_WGRAD_SPLIT=1): stack/parity/mixed tests, bench A/B on one box
O=gpurun_out/ws; mkdir -p $O; rm -f $O/*
OASES_WGRAD_SPLIT=1 timeout 900 python -m pytest tests/test_stack_gpu.py tests/test_parity_baseline_gpu.py tests/test_mixed_gpu.py -x -q > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
for i in 1 2; do
  OASES_WGRAD_SPLIT=0 timeout 300 python bench.py --steps 10 --warmup 3 2>/dev/null | tail -1 > $O/s0_$i.json
  OASES_WGRAD_SPLIT=1 timeout 300 python bench.py --steps 10 --warmup 3 2>/dev/null | tail -1 > $O/s1_$i.json
done
