# source-level ncu of the persistent LayerNorm backward at the C2 sub-batch (stall attribution)
O=gpurun_out/lsrc; rm -rf $O; mkdir -p $O
timeout 300 ncu --set full --import-source on --clock-control none -k regex:lnp_bwd -c 1 -f -o $O/bwd python tools/lnp_one.py 4096 2048 > /dev/null 2>&1
ncu -i $O/bwd.ncu-rep --page source --csv --print-source sass > $O/bwd_sass.csv 2>/dev/null
ncu -i $O/bwd.ncu-rep --page source --csv > $O/bwd_src.csv 2>/dev/null
ncu -i $O/bwd.ncu-rep --page raw --csv > $O/bwd_raw.csv 2>/dev/null
rm -f $O/bwd.ncu-rep; ls -la $O
