# dense kernel: union k-th variants A/B (0 = bit-serial, 1 = lane ranks, 2 = lane ranks + segment loads issued
# together), dense parity tests with the default, then the default bench (developer tool)
O=gpurun_out/s4c; mkdir -p $O
timeout 900 python tools/dense_env_ab.py 1000000 2000 "BVSS_DENSE_UKTH=0" "BVSS_DENSE_UKTH=1" "" > $O/ab.log 2>&1; echo "rc=$?" >> $O/ab.log
timeout 1200 python -m pytest tests/test_gpu_dense.py tests/test_gpu_group.py tests/test_gpu_fullsize.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
