"""A/B timing of pb_syrk_potrf_nd_batched (panel-major, D = chol(C + A B^T)) at a few (n, k)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1902_08115_b200 as pb  # noqa: E402

pb.library_path = os.path.abspath(sys.argv[1])
pb.lib()
dev = torch.device("cuda:0")
st = torch.cuda.current_stream(dev)
R = pb.PanelRef
out = []
for (n, k, batch) in ((48, 32, 16384), (96, 64, 8192), (96, 96, 8192), (128, 64, 4096), (160, 160, 2048)):
    La, Lc = n * k, n * n
    A = torch.rand((batch, La), device=dev, dtype=torch.float64) - 0.5
    C0 = torch.zeros((batch, Lc), device=dev, dtype=torch.float64)
    i = torch.arange(n, device=dev)
    C0[:, (i // 4) * 4 * n + 4 * i + i % 4] = float(k + n)  # panel-major diagonal: S = C0 + A A^T is SPD
    D = torch.empty_like(C0)
    info = torch.empty(batch, dtype=torch.int32, device=dev)
    laps = []
    for r in range(4):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        pb.syrk_potrf_nd_batched(n, k, R(A, n, k), La, R(A, n, k), La, R(C0, n, n), Lc, R(D, n, n), Lc, info,
                                 batch, stream=st)
        e1.record(st)
        torch.cuda.synchronize()
        if r:
            laps.append(e0.elapsed_time(e1))
    assert int(info.abs().sum()) == 0
    out.append(f"n={n} k={k}: {statistics.median(laps):.4f} ms")
print(os.path.basename(sys.argv[1]), " | ".join(out))
