# fwd2 without the PV drain before S(j+1): bitwise vs the drained version and the
# one-tile kernel, repeat stability, timing A/B, attention tests
O=gpurun_out/pvw; mkdir -p $O; rm -f $O/*
for sh in "4 16 1024" "4 4 2048" "8 8 1024"; do set -- $sh
  for cfg in "FWD2=0 PVW=1" "FWD2=1 PVW=1" "FWD2=1 PVW=0"; do
    eval $cfg
    echo "N=$1 HL=$2 SEQ=$3 $cfg $(OASES_ATTN_FWD2=$FWD2 OASES_ATTN_PV_WAIT=$PVW N=$1 HL=$2 SEQ=$3 REPS=200 timeout 120 python tools/attn_repeat_check.py 2>&1 | tail -1)" >> $O/check.log
  done
  for PVW in 1 0 1 0; do echo "N=$1 HL=$2 SEQ=$3 PVW=$PVW" >> $O/attn.log; OASES_ATTN_PV_WAIT=$PVW MODE=2 N=$1 HL=$2 SEQ=$3 timeout 120 python tools/attn_one.py 2>&1 | tail -2 >> $O/attn.log; done
done
timeout 600 python -m pytest tests/test_attention_gpu.py -x -q > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
