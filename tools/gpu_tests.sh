O=gpurun_out/g5; mkdir -p $O
timeout 600 python -m pytest tests/test_mixed_gpu.py -x -q > $O/mixed.log 2>&1; echo rc $? >> $O/mixed.log
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_mixed_gpu.py > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
