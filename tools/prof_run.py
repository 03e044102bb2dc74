"""Small driver for ncu captures: runs one routine at a config-sized batch a few times."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1902_08115_b200 as pb
what = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 64
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dev = torch.device("cuda:0")
if what == "gemm":
    batch = 16384
    A = torch.rand((batch, n, n), device=dev, dtype=torch.float64)
    B = torch.rand((batch, n, n), device=dev, dtype=torch.float64)
    C = torch.rand((batch, n, n), device=dev, dtype=torch.float64)
    for _ in range(reps):
        pb.dgemm_batched("n", "n", n, n, n, 1.0, A, n, n * n, B, n, n * n, 1.0, C, n, n * n, batch)
elif what == "potrf":
    batch = 8192
    Bm = torch.randn((batch, n, n), device=dev, dtype=torch.float64)
    A0 = Bm @ Bm.transpose(1, 2) + n * torch.eye(n, device=dev, dtype=torch.float64)
    A = A0.clone()
    info = torch.empty(batch, dtype=torch.int32, device=dev)
    for _ in range(reps):
        A.copy_(A0)
        pb.dpotrf_batched("l", n, A, n, n * n, info, batch)
elif what == "getrf":
    batch = 8192
    A0 = torch.rand((batch, n, n), device=dev, dtype=torch.float64)
    A = A0.clone()
    ipiv = torch.empty((batch, n), dtype=torch.int32, device=dev)
    info = torch.empty(batch, dtype=torch.int32, device=dev)
    for _ in range(reps):
        A.copy_(A0)
        pb.dgetrf_batched(n, n, A, n, n * n, ipiv, n, info, batch)
torch.cuda.synchronize()
print("done", what, n)
if what == "gemm_nd":
    batch = (2 ** 31) // (32 * n * n)
    L = n * n
    A = torch.rand((batch, L), device=dev, dtype=torch.float64)
    B = torch.rand_like(A); C = torch.rand_like(A); D = torch.empty_like(A)
    R = pb.PanelRef
    for _ in range(reps):
        pb.gemm_nd_batched("n", "t", n, n, n, 1.0, R(A, n, n), L, R(B, n, n), L, 1.0, R(C, n, n), L, R(D, n, n), L, batch)
    torch.cuda.synchronize()
    print("done gemm_nd", n)
if what == "trsm":
    batch = max(256, (2**30) // (16 * n * n))
    Lm = torch.tril(torch.rand((batch, n, n), device=dev, dtype=torch.float64)) + n * torch.eye(n, device=dev, dtype=torch.float64)
    Lc = Lm.transpose(1, 2).contiguous()
    B0 = torch.rand((batch, n, n), device=dev, dtype=torch.float64)
    tinfo = torch.empty(batch, dtype=torch.int32, device=dev)
    for _ in range(reps):
        pb.dtrsm_batched('r', 'l', 't', 'n', n, n, 1.0, Lc, n, n * n, B0, n, n * n, tinfo, batch)
    torch.cuda.synchronize()
    print("done trsm", n)
if what == "chain":
    import numpy as np
    layout = sys.argv[2] if len(sys.argv) > 2 else "C"
    rng = np.random.default_rng(5)
    batch = 32768
    ns = rng.integers(1, 65, batch) * 4
    offs = np.concatenate([[0], np.cumsum(ns.astype(np.int64) ** 2)[:-1]])
    total = int((ns.astype(np.int64) ** 2).sum())
    A = torch.rand(total, device=dev, dtype=torch.float64) * 2 - 1
    B = torch.rand(total, device=dev, dtype=torch.float64) * 2 - 1
    C = torch.zeros(total, device=dev, dtype=torch.float64)
    for nn_ in np.unique(ns):
        idx = np.nonzero(ns == nn_)[0]
        base = torch.from_numpy(offs[idx]).to(dev)
        ar = torch.arange(int(nn_), device=dev)
        diag = ar * (int(nn_) + 1) if layout == 'C' else (ar // 4) * 4 * int(nn_) + ar * 4 + ar % 4
        C[(base[:, None] + diag[None, :]).reshape(-1)] = float(nn_)
    dn = torch.from_numpy(ns.astype(np.int32)).to(dev); doff = torch.from_numpy(offs).to(dev)
    info = torch.empty(batch, dtype=torch.int32, device=dev)
    for _ in range(reps):
        pb.chain_vbatched(layout, dn, doff, A, C, B, info, batch, 256)
    torch.cuda.synchronize()
    print("done chain", layout)
