"""Per-problem instruction counts of potrf_cta_kernel by source region (from a cuda,sass source CSV)."""
import csv, sys
path, batch = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 8192
rows = list(csv.reader(open(path)))
hdr = None; fname = None; agg = {}; stall = {}
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split('/')[-1]; continue
    if r[0] == "Line No":
        hdr = r; ii = hdr.index("Instructions Executed"); si = hdr.index("Warp Stall Sampling (All Samples)"); continue
    if hdr is None or r[0] in ("", "Function Name"): continue
    try:
        agg[(fname, int(r[0]))] = int(r[ii] or 0); stall[(fname, int(r[0]))] = int(r[si] or 0)
    except ValueError: pass
src = open('paper_1902_08115_b200/csrc/potrf_cta.cu').read().split('\n')
def find(pat):
    for i, l in enumerate(src):
        if pat in l: return i + 1
    raise KeyError(pat)
marks = [("header/helpers", 1), ("exact panel", find("__noinline__ int cta_factor_panel_exact")),
         ("panel fn", find("__device__ __forceinline__ int cta_factor_panel(")),
         ("update fn", find("__device__ __forceinline__ bool cta_update_block(")),
         ("kernel prologue", find("__global__ void __launch_bounds__")),
         ("staging", find("// ---- stage the lower triangle")),
         ("syrk prologue", find("if (P.pa && P.k_ab > 0) {")),
         ("role/sync", find("// Role rotation")),
         ("main loops", find("if (P.syrk_only) {")),
         ("writeback", find("// ---- write back")), ("launch", find("static cudaError_t cta_launch_t"))]
tot = sum(agg.values()); tots = sum(stall.values()) or 1
print(f"total warp-instr/problem {tot/batch:.0f}")
for i, (name, lo) in enumerate(marks):
    hi = marks[i + 1][1] - 1 if i + 1 < len(marks) else 10**9
    v = sum(x for (f, l), x in agg.items() if f == 'potrf_cta.cu' and lo <= l <= hi)
    st = sum(x for (f, l), x in stall.items() if f == 'potrf_cta.cu' and lo <= l <= hi)
    print(f"  {name:16s} {v/batch:8.0f}   stall {100*st/tots:5.1f}%")
for f in sorted({f for f, _ in agg if f != 'potrf_cta.cu'}):
    v = sum(x for (ff, l), x in agg.items() if ff == f); st = sum(x for (ff, l), x in stall.items() if ff == f)
    print(f"  [{f}] {v/batch:8.0f}   stall {100*st/tots:5.1f}%")
