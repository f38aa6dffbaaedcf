O=gpurun_out/g4; mkdir -p $O; rm -f $O/*.log
for CL in 1 2 4 8; do for sh in "8192 4096" "4096 2048"; do echo "CL=$CL $sh" >> $O/ln.log; OASES_LNP_CLUSTER=$CL timeout 120 python tools/ln_bench.py $sh 2>&1 | grep -v "^{" >> $O/ln.log; done; done
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_stack_gpu.py -x -q > $O/pytest.log 2>&1; echo pytest $? >> $O/pytest.log
