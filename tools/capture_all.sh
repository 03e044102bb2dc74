# Round-end evidence capture (one gpurun call): launch lists and ncu --set full of the top kernels.
set -x
python bench.py --steps 2 --warmup 3 --no-series --no-cpu > gpurun_out/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-series --no-cpu > gpurun_out/bench_ncu.log 2>&1
bash tools/launch_list.sh chainC chain C 1
bash tools/launch_list.sh chainP chain P 1
bash tools/launch_list.sh getrf192 getrf 192 1
bash tools/launch_list.sh potrf256 potrf 256 1
bash tools/prof1.sh "potrf32 potrf_reg potrf 32 2" "potrf64 potrf_cta potrf 64 2" "potrf128 potrf_cta potrf 128 2" \
  "getrf24 getrf_reg getrf 24 2" "getrf48 getrf_cta getrf 48 2" "trsm256 trsm_rlt trsm 256 2" \
  "gemmnd4 gemm gemm_nd 4 2" "gemmnd48 gemm gemm_nd 48 2" "gemmnd96 gemm gemm_nd 96 2" "dgemm64 gemm gemm 64 3"
