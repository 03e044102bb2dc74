"""Times every config's GPU path (device-resident inputs, CUDA events, back-to-back launches)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import numpy as np
import paper_1902_08115_b200 as pb
dev = torch.device('cuda:0'); s = torch.cuda.current_stream()
BW, P = 6553.6e9, 37.1e12


def timeit(fn, reps=3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    fn(); torch.cuda.synchronize(); e0.record(s)
    for _ in range(reps): fn()
    e1.record(s); torch.cuda.synchronize(); return e0.elapsed_time(e1) / reps


what = sys.argv[1:] or ['getrf', 'gemm_nd', 'chain']
if 'getrf' in what:
    for n in (24, 48, 96, 192):
        batch = 8192
        A0 = torch.rand((batch, n, n), device=dev, dtype=torch.float64) * 2 - 1
        As = [A0.clone() for _ in range(3)]
        ip = torch.empty((batch, n), dtype=torch.int32, device=dev); info = torch.empty(batch, dtype=torch.int32, device=dev)
        it = iter(range(100))
        def f():
            pb.dgetrf_batched(n, n, As[next(it) % 3], n, n * n, ip, n, info, batch, stream=s)
        ms = timeit(f)
        fl = (n**3 - n**3 // 3) * batch; by = (16 * n * n + 4 * n) * batch
        roof = min(P, BW * fl / by)
        print(f"getrf n={n}: {ms:.4f} ms {fl/ms/1e9:.2f} TF roofline-frac {fl/(ms*1e-3)/roof:.3f}")
if 'gemm_nd' in what:
    for sz in ([int(x) for x in os.environ.get("SIZES", "").split(",") if x] or (4, 8, 12, 16, 24, 32, 48, 64, 96, 128, 192, 256, 320)):
        batch = (2**31) // (32 * sz * sz)
        L = sz * sz
        A = torch.rand((batch, L), device=dev, dtype=torch.float64); B = torch.rand_like(A); C = torch.rand_like(A); D = torch.empty_like(A)
        R = pb.PanelRef
        f = lambda: pb.gemm_nd_batched('n', 't', sz, sz, sz, 1.0, R(A, sz, sz), L, R(B, sz, sz), L, 1.0, R(C, sz, sz), L, R(D, sz, sz), L, batch, stream=s)
        ms = timeit(f)
        fl = 2 * sz**3 * batch; by = 32 * sz * sz * batch
        roof = min(P, BW * fl / by)
        print(f"gemm_nd s={sz} batch={batch}: {ms:.4f} ms {fl/ms/1e9:.2f} TF roofline-frac {fl/(ms*1e-3)/roof:.3f}")
        del A, B, C, D
if 'chain' in what:
    rng = np.random.default_rng(5)
    batch = 32768
    ns = rng.integers(1, 65, batch) * 4
    offs = np.concatenate([[0], np.cumsum(ns.astype(np.int64) ** 2)[:-1]])
    total = int((ns.astype(np.int64) ** 2).sum())
    for layout in 'CP':
        A = torch.rand(total, device=dev, dtype=torch.float64) * 2 - 1
        B = torch.rand(total, device=dev, dtype=torch.float64) * 2 - 1
        C0 = torch.zeros(total, device=dev, dtype=torch.float64)
        for n in np.unique(ns):  # C0 = n I
            idx = np.nonzero(ns == n)[0]
            base = torch.from_numpy(offs[idx]).to(dev)
            ar = torch.arange(int(n), device=dev)
            diag = ar * (int(n) + 1) if layout == 'C' else (ar // 4) * 4 * int(n) + ar * 4 + ar % 4
            C0[(base[:, None] + diag[None, :]).reshape(-1)] = float(n)
        C = C0.clone()
        dn = torch.from_numpy(ns.astype(np.int32)).to(dev); doff = torch.from_numpy(offs).to(dev)
        info = torch.empty(batch, dtype=torch.int32, device=dev)
        def f():
            C.copy_(C0)
            pb.chain_vbatched(layout, dn, doff, A, C, B, info, batch, 256, stream=s)
        ms = timeit(f, 2)
        fl = float(sum(2 * int(n)**3 + int(n)**3 // 3 for n in ns))
        print(f"chain {layout}: {ms:.3f} ms (incl. C reset copy) {fl/ms/1e9:.2f} TF  info0={int(info.abs().sum())==0}")
if 'trsm' in what:
    for n in (32, 64, 128, 256):
        batch = max(256, (2**30) // (16 * n * n))
        Lm = torch.tril(torch.rand((batch, n, n), device=dev, dtype=torch.float64)) + n * torch.eye(n, device=dev, dtype=torch.float64)
        Lc = Lm.transpose(1, 2).contiguous()  # column-major storage of L
        B0 = torch.rand((batch, n, n), device=dev, dtype=torch.float64)
        Bs = [B0.clone() for _ in range(3)]
        it = iter(range(100))
        tinfo = torch.empty(batch, dtype=torch.int32, device=dev)
        f = lambda: pb.dtrsm_batched('r', 'l', 't', 'n', n, n, 1.0, Lc, n, n * n, Bs[next(it) % 3], n, n * n, tinfo, batch, stream=s)
        ms = timeit(f)
        fl = n ** 3 * batch; by = (8 * n * (n + 1) / 2 + 16 * n * n) * batch
        roof = min(P, BW * fl / by)
        print(f"trsm rltn n={n} batch={batch}: {ms:.4f} ms {fl/ms/1e9:.2f} TF roofline-frac {fl/(ms*1e-3)/roof:.3f}")
