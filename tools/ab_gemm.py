"""A/B device timing of pb_dgemm_batched NN for library builds: python tools/ab_gemm.py <lib.so> ...
prints ms per launch for (s, batch, beta) cases (L2 flushed between launches, median of 5)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1902_08115_b200 as pb  # noqa: E402

dev = torch.device("cuda:0")
st = torch.cuda.current_stream(dev)
flush = torch.empty(64 * 2 ** 20, dtype=torch.float64, device=dev)
for lib in sys.argv[1:]:
    pb.library_path = os.path.abspath(lib)
    pb._lib = None
    pb.lib()
    out = []
    for (s, batch, beta) in ((64, 16384, 1.0), (64, 16384, 0.0), (32, 65536, 1.0), (48, 29127, 1.0)):
        A = torch.rand((batch, s, s), device=dev, dtype=torch.float64)
        B = torch.rand_like(A); C = torch.rand_like(A)
        laps = []
        for r in range(6):
            flush.fill_(r)
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            pb.dgemm_batched("n", "n", s, s, s, 1.0, A, s, s * s, B, s, s * s, beta, C, s, s * s, batch, stream=st)
            e1.record(st)
            torch.cuda.synchronize()
            if r:
                laps.append(e0.elapsed_time(e1))
        ms = statistics.median(laps)
        by = 8 * batch * s * s * (4 if beta else 3)
        out.append(f"s={s} beta={beta:g}: {ms:.4f} ms {by / ms / 1e6:.0f} GB/s")
        del A, B, C
    print(os.path.basename(lib), " | ".join(out), flush=True)
