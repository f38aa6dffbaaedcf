O=gpurun_out/g9; mkdir -p $O; rm -f $O/*
OASES_ATTN_FWD2=1 MODE=2 ITERS=1 REP=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:attn_fwd -c 1 -f -o $O/fwd2 python tools/attn_one.py > $O/ncu.log 2>&1
OASES_ATTN_FWD2=0 MODE=2 ITERS=1 REP=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:attn_fwd -c 1 -f -o $O/fwd1 python tools/attn_one.py >> $O/ncu.log 2>&1
