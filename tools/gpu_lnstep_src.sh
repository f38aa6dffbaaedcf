# source-level ncu of in-step LayerNorm kernels (C2 bench step): three consecutive lnp_fwd launches
O=gpurun_out/lstep; rm -rf $O; mkdir -p $O
for k in 40 41 42; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:lnp_fwd_kernel --launch-skip $k -c 1 -f -o $O/f$k python bench.py --steps 1 --warmup 3 --no-graph > /dev/null 2>&1
  ncu -i $O/f$k.ncu-rep --page source --csv --print-source sass > $O/f${k}_sass.csv 2>/dev/null
  ncu -i $O/f$k.ncu-rep --page details --csv > $O/f${k}_details.csv 2>/dev/null
done
rm -f $O/*.ncu-rep; ls -la $O
