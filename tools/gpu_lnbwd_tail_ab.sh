# LayerNorm backward partial-plane tail: liboases_old.so vs in-tree; warm microbench (C2 sub-batch, C3 rank),
# ncu launch list of the in-step LN kernels, kernel tests, GPU suite, bench A/B
O=gpurun_out/ltail; mkdir -p $O; rm -f $O/*
for L in old new old new; do
  if [ $L = old ]; then export OASES_LIB=$PWD/liboases_old.so; else unset OASES_LIB; fi
  echo "== $L C2" >> $O/ln.log; timeout 120 python tools/ln_bench.py 4096 2048 >> $O/ln.log 2>&1
  echo "== $L C3" >> $O/ln.log; timeout 120 python tools/ln_bench.py 8192 4096 >> $O/ln.log 2>&1
done
for L in old new; do
  if [ $L = old ]; then export OASES_LIB=$PWD/liboases_old.so; else unset OASES_LIB; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lnp_ --csv --log-file $O/$L.csv python bench.py --steps 1 --warmup 3 --no-graph --no-extras --no-cpu-baseline > /dev/null 2>&1
done
unset OASES_LIB
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
for i in 1 2; do for L in old new; do
  if [ $L = old ]; then export OASES_LIB=$PWD/liboases_old.so; else unset OASES_LIB; fi
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 > $O/bench_${L}_$i.json
done; done
