# Round-2 evidence capture (one gpurun call): full bench line, the headline's launch list,
# ncu --set full of the headline kernel, launch lists of the multi-kernel paths.
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --steps 2 --warmup 3 --no-series --no-cpu > gpurun_out/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-series --no-cpu > gpurun_out/bench_ncu.log 2>&1
bash tools/prof1.sh "dgemm64 gemm_cm gemm 64 3" > /dev/null 2>&1
bash tools/launch_list.sh chainC chain C 1
bash tools/launch_list.sh chainP chain P 1
bash tools/launch_list.sh getrf192 getrf 192 1
bash tools/launch_list.sh potrf256 potrf 256 1
python tools/launch_summary.py gpurun_out/bench_launches.csv > gpurun_out/bench_launches.txt 2>&1
for n in chainC chainP getrf192 potrf256; do python tools/launch_summary.py gpurun_out/${n}_launches.csv > gpurun_out/${n}_launches.txt 2>&1; done
