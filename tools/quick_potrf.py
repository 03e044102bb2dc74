import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, statistics
import paper_1902_08115_b200 as pb
if os.environ.get('PBGPU_LIB'): pb.library_path = os.path.abspath(os.environ['PBGPU_LIB'])  # A/B against another build
dev = torch.device('cuda:0'); s = torch.cuda.current_stream()
ns = [int(x) for x in sys.argv[1:]] or [16, 32, 64, 128, 256]
for n in ns:
    batch = 8192
    R = 4 if n < 256 else 2
    B = torch.randn((batch, n, n), device=dev, dtype=torch.float64)
    A0 = B @ B.transpose(1, 2) + n * torch.eye(n, device=dev, dtype=torch.float64); del B
    As = [A0.clone() for _ in range(R)]; info = torch.empty(batch, dtype=torch.int32, device=dev)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); laps = []
    for rep in range(3):
        for A in As: A.copy_(A0)
        torch.cuda.synchronize(); e0.record(s)
        for A in As:  # back-to-back launches: host overhead hides behind the previous kernel
            pb.dpotrf_batched('l', n, A, n, n * n, info, batch, stream=s)
        e1.record(s); torch.cuda.synchronize()
        laps.append(e0.elapsed_time(e1) / R)
    ms = min(laps); fl = (n**3 // 3) * batch; by = 8 * n * (n + 1) * batch
    roof = min(37.1e12, 6553.6e9 * fl / by)
    print(f"potrf n={n}: {ms:.4f} ms  {fl/ms/1e9:.2f} TFLOP/s  {by/ms/1e6:.0f} GB/s  roofline-frac {fl/(ms*1e-3)/roof:.3f}  info0={int(info.abs().sum())==0}")
    del As, A0
