# bench A/B of an env switch on one box: VAR=name A=value B=value (alternating, 2 x 2 runs)
O=gpurun_out/envab; mkdir -p $O; rm -f $O/*
for i in 1 2; do
  env $VAR=$A timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 > $O/a$i.json
  env $VAR=$B timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 > $O/b$i.json
done
