#!/bin/bash
# usage: tools/ncu_trace.sh <name> <n>   — ncu --set full of potrf_cta_kernel in the trace tool (tools/potrf_trace)
name=$1; n=$2
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:potrf_cta -s 1 -c 1 -f -o /tmp/$name ./tools/potrf_trace $n > gpurun_out/${name}_ncu.log 2>&1
ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>&1
ncu -i /tmp/$name.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${name}_source.csv 2>&1
