import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1902_08115_b200 as pb
dev = torch.device('cuda:0')
print('dmma probe TFLOP/s', pb.lib().pb_probe_dmma_tflops())
x = torch.empty(2**28, dtype=torch.float64, device=dev); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(5): y.copy_(x)
e1.record(); torch.cuda.synchronize(); print('copy GB/s', 5*2*x.numel()*8/e0.elapsed_time(e1)/1e6)
del x, y
for (m, batch) in [(64, 16384), (32, 65536), (128, 4096), (256, 1024)]:
    n = k = m
    A = torch.rand((batch, k, m), device=dev, dtype=torch.float64)
    B = torch.rand((batch, n, k), device=dev, dtype=torch.float64)
    C = torch.rand((batch, n, m), device=dev, dtype=torch.float64)
    s = torch.cuda.current_stream()
    for _ in range(3):
        pb.dgemm_batched('n','n',m,n,k,1.0,A,m,m*k,B,k,k*n,1.0,C,m,m*n,batch, stream=s)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    R = 10
    for _ in range(R):
        pb.dgemm_batched('n','n',m,n,k,1.0,A,m,m*k,B,k,k*n,1.0,C,m,m*n,batch, stream=s)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / R
    fl = 2.0*m*n*k*batch; by = 8.0*(m*k+k*n+2*m*n)*batch
    print(f'n={m} batch={batch}: {ms:.3f} ms  {fl/ms/1e9:.1f} TFLOP/s  {by/ms/1e6:.1f} GB/s')
