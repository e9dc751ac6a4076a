# K1 encoder A/B across builds: E0 = round start, E1 = bisection early exit, new = + W rows as 16-byte loads
O=gpurun_out/s3l; mkdir -p $O
timeout 900 python tools/enc_lib_ab.py $PWD/tools/old_lib/E0/libbvss.so $PWD/tools/old_lib/E1/libbvss.so new > $O/enc_lib_ab.log 2>&1
timeout 900 python tools/enc_lib_ab.py new $PWD/tools/old_lib/E1/libbvss.so $PWD/tools/old_lib/E0/libbvss.so >> $O/enc_lib_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_encoder.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
BVSS_LIB=$PWD/tools/old_lib/E1/libbvss.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k codes > $O/pytest_e1.log 2>&1; echo "rc=$?" >> $O/pytest_e1.log
