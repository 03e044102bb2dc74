import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1902_08115_b200 as pb
dev = torch.device('cuda:0'); s = torch.cuda.current_stream()
def timeit(fn, reps=3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize(); e0.record(s)
    for _ in range(reps): fn()
    e1.record(s); torch.cuda.synchronize(); return e0.elapsed_time(e1) / reps
for (m, n, ld, batch) in [(128, 128, 128, 1024), (128, 128, 256, 1024), (128, 128, 128, 4096)]:
    Lm = torch.tril(torch.rand((batch, ld, ld), device=dev, dtype=torch.float64)) + ld * torch.eye(ld, device=dev, dtype=torch.float64)
    Lc = Lm.transpose(1, 2).contiguous()
    B = torch.rand((batch, ld, ld), device=dev, dtype=torch.float64)
    info = torch.empty(batch, dtype=torch.int32, device=dev)
    f = lambda: pb.dtrsm_batched('r', 'l', 't', 'n', m, n, 1.0, Lc, ld, ld * ld, B, ld, ld * ld, info, batch, stream=s)
    ms = timeit(f)
    print(f"m={m} n={n} ld={ld} batch={batch}: {ms:.4f} ms {m*n*n*batch/ms/1e9:.2f} TF")
