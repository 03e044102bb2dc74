"""Small driver for ncu captures: runs one routine at a config-sized batch a few times."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1902_08115_b200 as pb
what = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
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
