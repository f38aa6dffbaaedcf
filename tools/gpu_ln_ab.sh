# LayerNorm microbench A/B (liboases_old.so vs in-tree) at C2 and C3-rank widths, then a bench A/B
O=gpurun_out/lnab; mkdir -p $O; rm -f $O/*
for sh in "4096 2048" "8192 4096"; do
  for L in old new old new; do
    if [ $L = old ]; then export OASES_LIB=$PWD/liboases_old.so; else unset OASES_LIB; fi
    echo "== $L $sh" >> $O/ln.log; timeout 300 python tools/ln_bench.py $sh 2>&1 | grep -v "^{" | head -3 >> $O/ln.log
  done
done
unset OASES_LIB
for i in 1 2; do
  OASES_LIB=$PWD/liboases_old.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 > $O/old$i.json
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 > $O/new$i.json
done
