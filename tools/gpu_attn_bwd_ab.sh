# dK/dV kernel A/B on one box: liboases_old.so (earlier build) vs the in-tree build; trace builds when present
O=gpurun_out/bwdab; mkdir -p $O; rm -f $O/*
for L in old new; do
  [ -f liboases_trace_$L.so ] && OASES_LIB=$PWD/liboases_trace_$L.so timeout 120 python tools/attn_bwd_trace.py > $O/trace_$L.log 2>&1
done
for r in 1 2; do for L in old new; do
  if [ $L = old ]; then export OASES_LIB=$PWD/liboases_old.so; else unset OASES_LIB; fi
  echo "$L C2" >> $O/attn.log; MODE=2 timeout 120 python tools/attn_one.py 2>&1 | tail -1 >> $O/attn.log
  echo "$L C3" >> $O/attn.log; MODE=2 SEQ=2048 HL=4 N=4 timeout 120 python tools/attn_one.py 2>&1 | tail -1 >> $O/attn.log
done; done
unset OASES_LIB
timeout 600 python -m pytest tests/test_attention_gpu.py -x -q > $O/pytest_attn.log 2>&1; echo rc $? >> $O/pytest_attn.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
for i in 1 2; do for L in old new; do
  if [ $L = old ]; then export OASES_LIB=$PWD/liboases_old.so; else unset OASES_LIB; fi
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 > $O/bench_${L}_$i.json
done; done
