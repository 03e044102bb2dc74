"""Device timing of the tile engine's shapes (median of 7 launches after 3 warm-ups, inputs > L2):
column-major dgemm NN at n = 128, 256 (config-1 series) and gemm_nd NT panel-major at
s = 112, 128, 132, 192, 256, 320 (config 2), plus a lower dsyrk n = k = 256.
python tools/quick_engine.py            (PBGPU_ENGINE_STAGGER=<cycles> selects the consumer offset)"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1902_08115_b200 as pb  # noqa: E402

if os.environ.get("PBGPU_LIB"):  # A/B against another build
    pb.library_path = os.path.abspath(os.environ["PBGPU_LIB"])

dev = torch.device("cuda:0")
st = torch.cuda.current_stream(dev)
PEAK = 37.1e12


def med(fn):
    for _ in range(3):
        fn()
    laps = []
    for _ in range(7):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        laps.append(e0.elapsed_time(e1))
    return statistics.median(laps)


out = []
for n in (128, 256):
    batch = (2 ** 31) // (32 * n * n)
    A = torch.rand((batch, n, n), device=dev, dtype=torch.float64)
    B = torch.rand_like(A)
    C = torch.rand_like(A)
    ms = med(lambda: pb.dgemm_batched("n", "n", n, n, n, 1.0, A, n, n * n, B, n, n * n, 1.0, C, n, n * n, batch,
                                      stream=st))
    fl = 2.0 * n ** 3 * batch
    out.append(f"cm{n} {ms:.4f}ms {fl / ms / 1e9 / (PEAK / 1e12):.3f}")
    del A, B, C
R = pb.PanelRef
for s in (100, 104, 108, 112, 116, 124, 128, 132, 160, 192, 196, 256, 260, 320):
    batch = (2 ** 31) // (32 * s * s)
    L = s * s
    A = torch.rand((batch, L), device=dev, dtype=torch.float64)
    B = torch.rand_like(A)
    C = torch.rand_like(A)
    D = torch.empty_like(A)
    ms = med(lambda: pb.gemm_nd_batched("n", "t", s, s, s, 1.0, R(A, s, s), L, R(B, s, s), L, 1.0, R(C, s, s), L,
                                        R(D, s, s), L, batch, stream=st))
    fl = 2.0 * s ** 3 * batch
    out.append(f"pm{s} {ms:.4f}ms {fl / ms / 1e9 / (PEAK / 1e12):.3f}")
    del A, B, C, D
n = 256
batch = 2048
A = torch.rand((batch, n, n), device=dev, dtype=torch.float64)
C = torch.rand_like(A)
ms = med(lambda: pb.dsyrk_batched("l", "n", n, n, 1.0, A, n, n * n, 1.0, C, n, n * n, batch, stream=st))
out.append(f"syrk{n} {ms:.4f}ms {1.0 * n ** 3 * batch / ms / 1e9 / (PEAK / 1e12):.3f}")
print(f"stagger={os.environ.get('PBGPU_ENGINE_STAGGER', 'default')}: " + " | ".join(out), flush=True)
