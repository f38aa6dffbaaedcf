# side-stream attention mask pass: same-bits test, attention/stack tests, bench A/B on one box
O=gpurun_out/mside; mkdir -p $O; rm -f $O/*
timeout 900 python -m pytest tests/test_stack_gpu.py -x -q -k "side_stream or capped or deterministic" > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
timeout 600 python -m pytest tests/test_attention_gpu.py -x -q >> $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
for i in 1 2; do
  OASES_ATTN_MASK_SIDE=0 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 > $O/a$i.json
  OASES_ATTN_MASK_SIDE=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 > $O/b$i.json
done
