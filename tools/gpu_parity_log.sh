# parity at BASELINE configs + mixed degrees, per-tensor errors logged (OASES_PARITY_LOG)
O=gpurun_out/parity; mkdir -p $O; rm -f $O/*
OASES_PARITY_LOG=$O/r02_parity.jsonl timeout 1500 python -m pytest tests/test_parity_baseline_gpu.py tests/test_mixed_gpu.py -q > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
