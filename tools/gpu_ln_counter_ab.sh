# LayerNorm ring counters (no 64-bit division per item): liboases_old.so (HEAD) vs in-tree; bit identity, warm
# microbench at C2 / C3 shapes, in-step launch list, LN kernel tests, bench A/B
O=gpurun_out/lcnt; mkdir -p $O; rm -f $O/*
for L in old new; do
  if [ $L = old ]; then export OASES_LIB=$PWD/liboases_old.so; else unset OASES_LIB; fi
  echo "$L $(timeout 300 python tools/bitcheck.py 2 2>&1 | tail -1)" >> $O/bit.log
done
for L in old new old new; do
  if [ $L = old ]; then export OASES_LIB=$PWD/liboases_old.so; else unset OASES_LIB; fi
  echo "== $L C2" >> $O/ln.log; timeout 120 python tools/ln_bench.py 4096 2048 2>&1 | grep -v "^{" >> $O/ln.log
  echo "== $L C3" >> $O/ln.log; timeout 120 python tools/ln_bench.py 8192 4096 2>&1 | grep -v "^{" >> $O/ln.log
done
unset OASES_LIB
timeout 900 python -m pytest tests -m gpu -x -q -k "not target_width and not c2_full and not depth" > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
for i in 1 2; do for L in old new; do
  if [ $L = old ]; then export OASES_LIB=$PWD/liboases_old.so; else unset OASES_LIB; fi
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 > $O/bench_${L}_$i.json
done; done
