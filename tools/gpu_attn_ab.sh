# attention forward A/B at C2 and C3-rank shapes (mask pass mode) + attention/stack tests
O=gpurun_out/g8; mkdir -p $O; rm -f $O/*
for sh in "4 16 1024" "4 4 2048"; do set -- $sh; for F in 0 1; do echo "N=$1 HL=$2 SEQ=$3 FWD2=$F" >> $O/attn.log; OASES_ATTN_FWD2=$F MODE=2 N=$1 HL=$2 SEQ=$3 timeout 120 python tools/attn_one.py 2>&1 | tail -3 >> $O/attn.log; done; done
timeout 600 python -m pytest tests/test_attention_gpu.py tests/test_stack_gpu.py tests/test_mixed_gpu.py -x -q > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
