# bench A/B on one box: liboases_old.so (an earlier build) vs the in-tree build, alternating
O=gpurun_out/ab; mkdir -p $O; rm -f $O/*
for i in 1 2 3; do
  OASES_LIB=$PWD/liboases_old.so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 > $O/old$i.json
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 > $O/new$i.json
done
