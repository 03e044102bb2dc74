"""Column-major dgemm_nn at small orders (device-resident, CUDA events): the warp-per-problem kernel
(gemm_cmsmall.cu) vs the tile engine (PBGPU_GEMM_CMSMALL=0)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1902_08115_b200 as pb
dev = torch.device('cuda:0'); s = torch.cuda.current_stream()
BW, P = 6553.6e9, 37.1e12
for n in [int(x) for x in sys.argv[1:]] or [4, 8, 12, 16, 24, 28]:
    batch = min(4194304, (2 ** 31) // (32 * n * n))
    A = torch.rand((batch, n * n), device=dev, dtype=torch.float64)
    B = torch.rand_like(A); C = torch.rand_like(A)
    f = lambda: pb.dgemm_batched('n', 'n', n, n, n, 1.0, A, n, n * n, B, n, n * n, 1.0, C, n, n * n, batch, stream=s)
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(3): f()
    e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    fl = 2 * n**3 * batch; by = 32 * n * n * batch
    print(f"dgemm_nn cm n={n} batch={batch}: {ms:.4f} ms {fl/ms/1e9:.2f} TF {by/ms/1e6:.0f} GB/s roofline-frac {fl/(ms*1e-3)/min(P, BW*fl/by):.3f}")
    del A, B, C
