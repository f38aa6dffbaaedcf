O=gpurun_out/full; mkdir -p $O; rm -f $O/*
timeout 2400 python -m pytest tests/ -x -q -m gpu > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
