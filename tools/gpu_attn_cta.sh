O=gpurun_out/acta; mkdir -p $O; rm -f $O/*
OASES_LIB=$PWD/liboases_trace.so timeout 120 python tools/attn_cta_timeline.py > $O/c2.log 2>&1
OASES_LIB=$PWD/liboases_trace.so N=4 HL=4 SEQ=2048 timeout 120 python tools/attn_cta_timeline.py > $O/c3.log 2>&1
