"""A/B timing of library builds: python tools/ab_time.py <lib.so> [series ...]
Loads the given libpbgpu.so instead of the in-tree one and prints bench.py's series
(device times only, no CPU legs) for the chosen configs."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1902_08115_b200 as pb  # noqa: E402

pb.library_path = os.path.abspath(sys.argv[1])
pb.lib()
which = sys.argv[2:] or ["cfg3", "cfg4", "cfg5"]
dev = torch.device("cuda:0")
stream = torch.cuda.current_stream(dev)
bw, _ = bench.measured_peaks()
S = bench.Series(pb, dev, stream, pb.lib().pb_probe_dmma_tflops(), bw, 0.3, skip_cpu=True)
fns = {"cfg1": lambda: bench.series_dgemm(S),
       "cfg2": lambda: bench.series_gemm_nd(S, [4, 8, 16, 24, 32, 48, 64, 96, 128, 192, 256, 320]),
       "cfg2all": lambda: bench.series_gemm_nd(S, list(range(4, 321, 4))),
       "cfg3": lambda: bench.series_dpotrf(S), "cfg4": lambda: bench.series_dgetrf(S),
       "cfg5": lambda: bench.series_chain(S)}
for w in which:
    r = fns[w]()
    print(os.path.basename(sys.argv[1]), w, json.dumps({k: (v["ms"], v["roofline_frac"]) for k, v in r.items()}),
          flush=True)
