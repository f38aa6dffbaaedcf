O=gpurun_out/lnc; mkdir -p $O; rm -f $O/*
for sh in "4096 2048" "8192 4096" "8192 2048"; do timeout 300 python tools/ln_bench.py $sh >> $O/ln.log 2>&1; done
