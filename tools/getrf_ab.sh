#!/bin/bash
# getrf: the square compile-time-shape kernel (getrf_sq.cu) vs the previous dispatch, then the LU tests
mkdir -p gpurun_out
{
echo "== PBGPU_GETRF_SQ=0"; PBGPU_GETRF_SQ=0 timeout 200 python tools/quick_all.py getrf
echo "== default"; timeout 200 python tools/quick_all.py getrf
for nu in 1 2 3; do echo "== PBGPU_GETRF_SQ_NU=$nu"; PBGPU_GETRF_SQ_NU=$nu timeout 200 python tools/quick_all.py getrf; done
} > gpurun_out/getrf_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_getrf.py tests/test_gpu_special.py tests/test_gpu_parity_full.py -x -q -k "getrf or cfg4" > gpurun_out/getrf_tests.txt 2>&1
tail -5 gpurun_out/getrf_tests.txt
