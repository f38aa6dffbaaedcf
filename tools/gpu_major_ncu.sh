# ncu raw metrics of the CTA-pair GEMM with K-major vs MN-major operands (4096x8192x2048)
O=gpurun_out/mjn; rm -rf $O; mkdir -p $O
for mj in "0,0" "1,1"; do t=$(echo $mj | tr , _)
  SHAPE=4096,8192,2048 MAJOR=$mj ITERS=2 timeout 300 ncu --set full --clock-control none -k regex:gemm_tc2 -s 1 -c 1 -f -o $O/g$t python tools/gemm_one.py > /dev/null 2>&1
  ncu -i $O/g$t.ncu-rep --page raw --csv > $O/raw$t.csv 2>/dev/null
  ncu -i $O/g$t.ncu-rep --page details --csv > $O/det$t.csv 2>/dev/null
  rm -f $O/g$t.ncu-rep
done
