# ncu of the attention-backward dQ GEMM (gemm_tc_kernel, causal K-range) at the C2 sub-batch
O=gpurun_out/dq; rm -rf $O; mkdir -p $O
MODE=2 ITERS=1 REP=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -c 1 -f -o $O/q python tools/attn_one.py > /dev/null 2>&1
ncu -i $O/q.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i $O/q.ncu-rep --page source --csv --print-source sass > $O/sass.csv 2>/dev/null
ncu -i $O/q.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
rm -f $O/q.ncu-rep; ls -la $O
