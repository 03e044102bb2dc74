#!/bin/bash
# tile engine: ragged cfg2 orders, the chain and potrf 256 (run before/after an engine change), then the tests that use it
mkdir -p gpurun_out
{
SIZES=68,100,128,132,160,196,256,260,320 timeout 300 python tools/quick_all.py gemm_nd
timeout 300 python tools/quick_all.py chain
timeout 200 python tools/quick_potrf.py 256
timeout 200 python tools/quick_all.py getrf
} > gpurun_out/engine_ab.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_chain.py tests/test_gpu_factor.py tests/test_gpu_getrf.py tests/test_gpu_round2.py -x -q > gpurun_out/engine_tests.txt 2>&1
tail -3 gpurun_out/engine_tests.txt
