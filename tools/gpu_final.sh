# end-of-round evidence: full GPU suite + smoke, three default bench runs, then the round-2 profile set
O=gpurun_out/fin2; mkdir -p $O; rm -f $O/*
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc $? >> $O/smoke.log
bash tools/gpu_bench3.sh
bash tools/profile_round2.sh
