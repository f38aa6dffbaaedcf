O=gpurun_out/g3; mkdir -p $O
timeout 300 ncu --set full --import-source on --clock-control none -k regex:lnp_ -c 4 -f -o $O/lnp_c3 python tools/lnp_one.py > $O/ncu.log 2>&1
