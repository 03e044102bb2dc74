# Round-2 evidence after the engine work (one gpurun call): GPU tests, the full bench line, launch lists and
# ncu --set full captures of the kernels changed late in the round.
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.txt 2>&1
tail -3 gpurun_out/gputests.txt
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --steps 2 --warmup 3 --no-series --no-cpu > gpurun_out/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-series --no-cpu > gpurun_out/bench_ncu.log 2>&1
bash tools/prof1.sh "dgemm64 gemm_cm gemm 64 3" "sq48 getrf_sq getrf 48 3" "sq96 getrf_sq getrf 96 3" \
                    "cms16 gemm_cmsmall gemm 16 3" "potrf64 potrf_cta potrf 64 3" "potrf128 potrf_cta potrf 128 3" \
                    "eng128 gemm_tiles gemm_nd 128 3" "eng132 gemm_tiles gemm_nd 132 3" "trsm256 trsm_rlt_kernel trsm 256 3" > /dev/null 2>&1
bash tools/launch_list.sh chainC chain C 1
bash tools/launch_list.sh chainP chain P 1
bash tools/launch_list.sh getrf192 getrf 192 1
bash tools/launch_list.sh potrf256 potrf 256 1
python tools/launch_summary.py gpurun_out/bench_launches.csv > gpurun_out/bench_launches.txt 2>&1
for n in chainC chainP getrf192 potrf256; do python tools/launch_summary.py gpurun_out/${n}_launches.csv > gpurun_out/${n}_launches.txt 2>&1; done
for n in dgemm64 sq48 sq96 cms16 potrf64 potrf128 eng128 eng132 trsm256; do python tools/profile_summary.py gpurun_out/$n > gpurun_out/${n}_summary.json 2> gpurun_out/${n}_summary.err; done
python tools/cfg2_sweep.py > gpurun_out/cfg2_sweep.log 2>&1
rm -f gpurun_out/*_source.csv
