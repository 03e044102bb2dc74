#!/bin/bash
# A/B of the potrf_cta variants on the trace tool (phase stamps + residual check)
mkdir -p gpurun_out
for n in "$@"; do
  for v in 1 2; do
    echo "=== n=$n variant $v"
    PBGPU_POTRF_V=$v timeout 120 ./tools/potrf_trace $n
  done
done > gpurun_out/trace_ab.txt 2>&1
