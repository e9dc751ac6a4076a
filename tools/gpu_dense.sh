#!/bin/bash
# dense-path bring-up: new GPU tests first (short timeouts), then the old suite
mkdir -p gpurun_out
export BVSS_DEBUG_SYNC=${BVSS_DEBUG_SYNC:-0}
timeout 600 python -m pytest tests/test_gpu_dense.py -x -q > gpurun_out/pytest_dense.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dense.log
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q > gpurun_out/pytest_scale.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_scale.log
