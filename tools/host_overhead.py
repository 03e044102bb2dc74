import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1902_08115_b200 as pb
dev = torch.device('cuda:0'); s = torch.cuda.current_stream()
n = 64
for batch in (1, 64, 8192):
    B = torch.randn((batch, n, n), device=dev, dtype=torch.float64)
    A0 = B @ B.transpose(1, 2) + n * torch.eye(n, device=dev, dtype=torch.float64)
    A = A0.clone(); info = torch.empty(batch, dtype=torch.int32, device=dev)
    for _ in range(3): pb.dpotrf_batched('l', n, A, n, n*n, info, batch, stream=s)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); R = 50
    for _ in range(R): pb.dpotrf_batched('l', n, A, n, n*n, info, batch, stream=s)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"batch={batch}: host {1e6*(t1-t0)/R:.1f} us/call, total {1e6*(t2-t0)/R:.1f} us/call")
