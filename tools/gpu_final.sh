# end-of-round evidence: bit-identity of the LN-backward change against the previous build,
# three default bench runs, then the round-2 profile set
O=gpurun_out/bit; mkdir -p $O; rm -f $O/*
for L in old new old new; do
  if [ $L = old ]; then export OASES_LIB=$PWD/liboases_old.so; else unset OASES_LIB; fi
  echo "$L $(timeout 300 python tools/bitcheck.py 2 2>&1 | tail -1)" >> $O/bit.log
done
unset OASES_LIB
bash tools/gpu_bench3.sh
bash tools/profile_round2.sh
