"""Device timing of dtrsm_batched('r','l','t','n') (X L^T = B, the chain's solve), m = n, median of 5.
PBGPU_LIB=<other build> selects another library for A/B."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1902_08115_b200 as pb  # noqa: E402

if os.environ.get("PBGPU_LIB"):
    pb.library_path = os.path.abspath(os.environ["PBGPU_LIB"])
dev = torch.device("cuda:0")
st = torch.cuda.current_stream(dev)
out = []
for n in [int(x) for x in sys.argv[1:]] or (72, 96, 128, 160, 192, 224, 256):
    batch = max(256, (2 ** 30) // (16 * n * n))
    Lm = torch.tril(torch.rand((batch, n, n), device=dev, dtype=torch.float64)) + n * torch.eye(n, device=dev, dtype=torch.float64)
    Lc = Lm.transpose(1, 2).contiguous()
    B0 = torch.rand((batch, n, n), device=dev, dtype=torch.float64)
    B = B0.clone()
    info = torch.empty(batch, dtype=torch.int32, device=dev)
    laps = []
    for r in range(7):
        B.copy_(B0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        pb.dtrsm_batched('r', 'l', 't', 'n', n, n, 1.0, Lc, n, n * n, B, n, n * n, info, batch, stream=st)
        e1.record(st)
        torch.cuda.synchronize()
        if r >= 2:
            laps.append(e0.elapsed_time(e1))
    ms = statistics.median(laps)
    # residual of the first problem: X L^T = B0
    X = B[0].T  # column-major view -> (row, col)
    Lr = Lc[0].T
    res = (torch.linalg.norm(X @ Lr.T - B0[0].T) / torch.linalg.norm(B0[0])).item()
    out.append(f"n={n} {ms:.4f}ms {1.0 * n ** 3 * batch / ms / 1e9 / 37.1:.3f} res={res:.1e}")
print(" | ".join(out), flush=True)
