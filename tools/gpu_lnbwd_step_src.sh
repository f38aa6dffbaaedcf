# source-level ncu of an in-step LayerNorm backward (C2 bench step, eager)
O=gpurun_out/lbstep; rm -rf $O; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lnp_bwd_kernel --launch-skip 30 -c 1 -f -o $O/b python bench.py --steps 1 --warmup 3 --no-graph --no-extras --no-cpu-baseline > /dev/null 2>&1
ncu -i $O/b.ncu-rep --page source --csv --print-source sass > $O/b_sass.csv 2>/dev/null
ncu -i $O/b.ncu-rep --page details --csv > $O/b_details.csv 2>/dev/null
ncu -i $O/b.ncu-rep --page raw --csv > $O/b_raw.csv 2>/dev/null
rm -f $O/*.ncu-rep; ls -la $O
