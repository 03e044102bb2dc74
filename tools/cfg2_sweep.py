"""Config 2 over all 80 sizes (gemm_nd NT panel-major, s = 4..320 step 4, batch = 2^31 / (32 s^2)):
device time per launch (median of 3 after a warm-up) and fraction of the roofline
max(flops / DMMA peak, 32 s^2 B / HBM) per problem.  Writes gpurun_out/cfg2_all_sizes.json."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1902_08115_b200 as pb  # noqa: E402

PEAK, BW = 37.1e12, 6537.6e9
dev = torch.device("cuda:0")
st = torch.cuda.current_stream(dev)
R = pb.PanelRef
sizes = {}
for s in range(4, 324, 4):
    batch = (2 ** 31) // (32 * s * s)
    L = s * s
    A = torch.rand((batch, L), device=dev, dtype=torch.float64)
    B = torch.rand_like(A)
    C = torch.rand_like(A)
    D = torch.empty_like(A)
    fn = lambda: pb.gemm_nd_batched("n", "t", s, s, s, 1.0, R(A, s, s), L, R(B, s, s), L, 1.0, R(C, s, s), L,  # noqa
                                    R(D, s, s), L, batch, stream=st)
    fn()
    laps = []
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        laps.append(e0.elapsed_time(e1))
    ms = statistics.median(laps)
    roof_s = batch * max(2.0 * s ** 3 / PEAK, 32.0 * s * s / BW)
    sizes[str(s)] = {"ms": round(ms, 4), "batch": batch, "gflops": round(2.0 * s ** 3 * batch / ms / 1e6, 1),
                     "roofline_frac": round(roof_s * 1e3 / ms, 3)}
    del A, B, C, D
out = {"sizes": sizes,
       "note": "cfg2 all 80 sizes, device time per launch (median of 3), roofline = per problem "
               "max(flops/37.1 TF, 32 s^2 B / 6537.6 GB/s)"}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "cfg2_all_sizes.json"), "w"), indent=0)
fr = [v["roofline_frac"] for v in sizes.values()]
print(f"cfg2 sweep: min {min(fr):.3f} median {statistics.median(fr):.3f} max {max(fr):.3f}; below 0.5: "
      f"{[k for k, v in sizes.items() if v['roofline_frac'] < 0.5]}")
