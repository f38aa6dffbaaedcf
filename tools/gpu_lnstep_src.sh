# source-level ncu of the in-step LayerNorm backward (gout + keep bits) and BDR forward (C2 bench step)
O=gpurun_out/lstep; rm -rf $O; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lnp_bwd_kernel --launch-skip 40 -c 1 -f -o $O/bwd python bench.py --steps 1 --warmup 3 --no-graph > /dev/null 2>&1
ncu -i $O/bwd.ncu-rep --page source --csv --print-source sass > $O/bwd_sass.csv 2>/dev/null
ncu -i $O/bwd.ncu-rep --page details --csv > $O/bwd_details.csv 2>/dev/null
rm -f $O/*.ncu-rep; ls -la $O
