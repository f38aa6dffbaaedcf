# source-level ncu of the bias-dropout-residual + LayerNorm forward at the C2 sub-batch
O=gpurun_out/bsrc; rm -rf $O; mkdir -p $O
timeout 300 ncu --set full --import-source on --clock-control none -k regex:lnp_fwd --launch-skip 1 -c 1 -f -o $O/f python tools/lnp_one.py 4096 2048 > /dev/null 2>&1
ncu -i $O/f.ncu-rep --page source --csv --print-source sass > $O/sass.csv 2>/dev/null
ncu -i $O/f.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
rm -f $O/f.ncu-rep; ls -la $O
