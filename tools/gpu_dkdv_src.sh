# dK/dV kernel: ncu source page (stall reasons per line) + timing A/B against liboases_old.so
O=gpurun_out/dkdv; mkdir -p $O; rm -f $O/*
MODE=2 ITERS=1 REP=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:attn_dkdv -c 1 -f -o $O/dkdv python tools/attn_one.py > $O/ncu.log 2>&1
for r in 1 2; do for L in old new; do
  if [ $L = old ]; then export OASES_LIB=$PWD/liboases_old.so; else unset OASES_LIB; fi
  echo "$L C2" >> $O/attn.log; MODE=2 timeout 120 python tools/attn_one.py 2>&1 | tail -1 >> $O/attn.log
  echo "$L C3" >> $O/attn.log; MODE=2 SEQ=2048 HL=4 N=4 timeout 120 python tools/attn_one.py 2>&1 | tail -1 >> $O/attn.log
done; done
unset OASES_LIB
timeout 600 python -m pytest tests/test_attention_gpu.py -x -q > $O/pytest_attn.log 2>&1; echo rc $? >> $O/pytest_attn.log
