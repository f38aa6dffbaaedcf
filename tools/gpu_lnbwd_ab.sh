# per-launch duration of the in-step LayerNorm backward, previous vs in-tree build (ncu launch list)
O=gpurun_out/lab; mkdir -p $O; rm -f $O/*
for L in old new; do
  if [ $L = old ]; then export OASES_LIB=$PWD/liboases_old.so; else unset OASES_LIB; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lnp_ --csv --log-file $O/$L.csv python bench.py --steps 1 --warmup 3 --no-graph > /dev/null 2>&1
done
