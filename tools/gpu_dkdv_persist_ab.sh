# persistent dK/dV kernel vs the one-shot grid (liboases_old.so): CTA timelines (trace builds), warm timing,
# attention tests, full GPU suite, bench A/B
O=gpurun_out/pers; mkdir -p $O; rm -f $O/*
OASES_LIB=$PWD/liboases_trace_old.so timeout 120 python tools/attn_cta_timeline.py > $O/cta_old_c2.log 2>&1
PERSISTENT=1 OASES_LIB=$PWD/liboases_trace_new.so timeout 120 python tools/attn_cta_timeline.py > $O/cta_new_c2.log 2>&1
for r in 1 2; do for L in old new; do
  if [ $L = old ]; then export OASES_LIB=$PWD/liboases_old.so; else unset OASES_LIB; fi
  echo "$L C2" >> $O/attn.log; MODE=2 timeout 120 python tools/attn_one.py 2>&1 | tail -1 >> $O/attn.log
  echo "$L C3" >> $O/attn.log; MODE=2 SEQ=2048 HL=4 N=4 timeout 120 python tools/attn_one.py 2>&1 | tail -1 >> $O/attn.log
  echo "$L C2 p0" >> $O/attn.log; P=0 timeout 120 python tools/attn_one.py 2>&1 | tail -1 >> $O/attn.log
done; done
unset OASES_LIB
timeout 600 python -m pytest tests/test_attention_gpu.py -x -q > $O/pytest_attn.log 2>&1; echo rc $? >> $O/pytest_attn.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
for i in 1 2; do for L in old new; do
  if [ $L = old ]; then export OASES_LIB=$PWD/liboases_old.so; else unset OASES_LIB; fi
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > $O/bench_${L}_$i.json
done; done
