for nu in 1 2 3 5 7; do echo "NU=$nu"; PBGPU_GETRF_NU=$nu timeout 100 python tools/quick_all.py getrf; done > gpurun_out/sweep.log 2>&1
