#!/bin/bash
# chain: one stream vs the side-stream pool, then the chain tests
mkdir -p gpurun_out
{
for ns in 1 2 4; do echo "== PBGPU_CHAIN_STREAMS=$ns"; PBGPU_CHAIN_STREAMS=$ns timeout 300 python tools/quick_all.py chain; done
} > gpurun_out/chain_ab.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_chain.py tests/test_gpu_parity_full.py tests/test_gpu_round2.py -x -q -k "chain or cfg5 or riccati" > gpurun_out/chain_tests.txt 2>&1
tail -3 gpurun_out/chain_tests.txt
