# attention mask pass A/B in the step + kernel timings + attention ncu (fwd2, dkdv, mask)
O=gpurun_out/g10; mkdir -p $O; rm -f $O/*
timeout 300 python -m pytest tests/test_attention_gpu.py tests/test_stack_gpu.py -x -q > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
MODE=2 timeout 120 python tools/attn_one.py > $O/attn_mode2.log 2>&1
for M in 1 0 1 0; do OASES_ATTN_MASK_PASS=$M timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 15 > $O/bench_mask$M.log 2>&1; python -c "
import json;d=json.loads(open('$O/bench_mask$M.log').read().strip().splitlines()[-1]);print('mask_pass=$M', d['value'],d['ms_per_step'],d['clocks']['sm_mhz'])" >> $O/ab.log; done
MODE=2 ITERS=1 REP=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:"attn_(fwd|dkdv|mask)" -s 3 -c 3 -f -o $O/attn_c2 python tools/attn_one.py > /dev/null 2>&1
