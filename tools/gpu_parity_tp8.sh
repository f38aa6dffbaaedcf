# parity at the C3 / C4 widths at TMP=8 (in-process ranks) with per-tensor errors logged
O=gpurun_out/ptp8; mkdir -p $O; rm -f $O/*
OASES_PARITY_LOG=$O/parity.jsonl timeout 1200 python -m pytest tests/test_parity_baseline_gpu.py -x -q -k target_width > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
