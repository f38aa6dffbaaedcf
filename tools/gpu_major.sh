# operand majorness at the wgrad shapes (f32 out not modelled: bf16 out)
O=gpurun_out/major; mkdir -p $O; rm -f $O/*
for sh in "2048,8192,8192" "8192,2048,8192" "6144,2048,8192" "4096,8192,2048"; do
  for mj in "0,0" "1,1" "0,1" "1,0"; do
    SHAPE=$sh MAJOR=$mj timeout 120 python tools/gemm_time.py >> $O/major.log 2>&1
  done
done
