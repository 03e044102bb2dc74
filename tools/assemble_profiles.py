"""Copies one capture (tools/capture_r02c.sh, merged into gpurun_out/) into profiles/ under the
round-2 names and builds profiles/r02_ncu_kernels.json from the per-kernel ncu summaries, adding each
kernel's algorithmic bytes / flops per launch.  python tools/assemble_profiles.py"""
import json
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")

for src, dst in (("bench_full.json", "r02_bench.json"), ("bench_ref.json", "r02_bench_ref.json"),
                 ("bench_launches.txt", "r02_bench_launches.txt"), ("bench_launches.csv", "r02_launches.csv"),
                 ("chainC_launches.txt", "r02_chainC_launches.txt"), ("chainP_launches.txt", "r02_chainP_launches.txt"),
                 ("getrf192_launches.txt", "r02_getrf192_launches.txt"),
                 ("potrf256_launches.txt", "r02_potrf256_launches.txt"),
                 ("dgemm64_details.csv", "r02_dgemm64_ncu_details.csv"),
                 ("eng128_details.csv", "r02_engine128_ncu_details.csv"),
                 ("cfg2_all_sizes.json", "r02_cfg2_all_sizes.json")):
    if os.path.exists(os.path.join(G, src)):
        shutil.copyfile(os.path.join(G, src), os.path.join(P, dst))

# name in profiles <- (capture name, problems per launch, algorithmic bytes / problem, flops / problem)
K = {
    "dgemm64": ("dgemm64", 16384, 8 * 4 * 64 * 64, 2 * 64 ** 3),
    "getrf48_sq": ("sq48", 8192, 16 * 48 * 48 + 4 * 48, 48 ** 3 - 48 ** 3 // 3),
    "getrf96_sq": ("sq96", 8192, 16 * 96 * 96 + 4 * 96, 96 ** 3 - 96 ** 3 // 3),
    "dgemm16_cmsmall": ("cms16", 16384, 8 * 4 * 16 * 16, 2 * 16 ** 3),
    "potrf64": ("potrf64", 8192, 8 * 64 * 65, 64 ** 3 // 3),
    "potrf128": ("potrf128", 8192, 8 * 128 * 129, 128 ** 3 // 3),
    "engine_nt_pm128": ("eng128", (2 ** 31) // (32 * 128 * 128), 32 * 128 * 128, 2 * 128 ** 3),
    "engine_nt_pm132": ("eng132", (2 ** 31) // (32 * 132 * 132), 32 * 132 * 132, 2 * 132 ** 3),
    "trsm_rlt256": ("trsm256", 1024, 8 * (256 * 257 // 2 + 2 * 256 * 256), 256 ** 3),
}
out = {"_note": "ncu --set full --clock-control none, one launch each (tools/capture_r02c.sh), round 2 after the "
                "engine work: gemm_cm_kernel<8> (cfg1 16384 x 64^3), getrf_sq_kernel (cfg4 n = 48, 96; 8192 problems), "
                "gemm_cmsmall_kernel<2> (16384 x 16^3), potrf_cta_kernel (cfg3 n = 64, 128; 8192 problems), "
                "gemm_tiles_kernel (cfg2 NT panel-major s = 128 full tiles / s = 132 ragged tiles), trsm_rlt_kernel (X L^T = B, n = m = 256, 1024 problems); "
                "dram bytes are per launch"}
for name, (cap, nprob, by, fl) in K.items():
    f = os.path.join(G, cap + "_summary.json")
    if not os.path.exists(f):
        continue
    d = json.load(open(f))
    us = float(d["duration_us"])
    d["algorithmic_bytes"] = float(nprob * by)
    d["algorithmic_gbs"] = round(nprob * by / us / 1e3, 1)
    d["flops"] = float(nprob * fl)
    d["tflops"] = round(nprob * fl / us / 1e6, 2)
    out[name] = d
json.dump(out, open(os.path.join(P, "r02_ncu_kernels.json"), "w"), indent=1)
print("assembled", sorted(k for k in out if k != "_note"))
