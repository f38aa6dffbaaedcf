# attention forward A/B (OASES_ATTN_FWD2=0 old kernel vs 1 ping-pong; MODE 0 Philox in-kernel vs 2 mask pass) + tests
O=gpurun_out/g7; mkdir -p $O; rm -f $O/*
for F in 0 1; do for M in 0 2; do echo "FWD2=$F MODE=$M" >> $O/attn.log; OASES_ATTN_FWD2=$F MODE=$M timeout 120 python tools/attn_one.py 2>&1 | tail -2 >> $O/attn.log; done; done
for F in 0 1; do echo "C3 FWD2=$F MODE=2" >> $O/attn.log; OASES_ATTN_FWD2=$F MODE=2 SEQ=2048 HL=4 N=4 timeout 120 python tools/attn_one.py 2>&1 | tail -2 >> $O/attn.log; done
timeout 600 python -m pytest tests/test_attention_gpu.py -x -q > $O/pytest_attn.log 2>&1; echo rc $? >> $O/pytest_attn.log
OASES_ATTN_FWD2=0 timeout 600 python -m pytest tests/test_attention_gpu.py -x -q > $O/pytest_attn_old.log 2>&1; echo rc $? >> $O/pytest_attn_old.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo rc $? >> $O/pytest.log
for F in 0 1; do OASES_ATTN_FWD2=$F timeout 300 python bench.py --no-cpu-baseline --steps 10 > $O/bench_fwd2_$F.log 2>&1; done
