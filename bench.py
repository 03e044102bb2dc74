#!/usr/bin/env python3
"""Benchmark: batched FP64 dgemm_nn (BASELINE.json config 1) on B200 through the pbgpu C ABI.

Step = one pass of the hot path over one batch: pb_dgemm_batched('n','n', 64,64,64,
alpha=1, beta=1, lda=ldb=ldc=64) over the 16384-problem config-1 batch.  With N GPUs
(torchrun, one process per GPU) the ONE host-generated batch is split by problem index
into N contiguous slices (`shard_of`), each rank runs its slice on its own
GPU and stream, and no collective touches the data path ("scaling": "strong").

  value  — FP64 GFLOP/s of the whole job: global batch flops / the slowest rank's device
           time (CUDA events on the launching stream, max over ranks), inputs in HBM;
  e2e    — the same metric through the public API with pinned HOST buffers: every step
           copies each rank's A, B, C slices host->device and C back (pbgpu stages and
           overlaps the copies);
  roofline — the dominant kernel (gemm_cm_kernel) against measured HBM bandwidth:
           algorithmic bytes 8*(mk + kn + 2mn) per problem;
  cpu_baseline — the reference's own CPU path (panelblas::dgemm compiled from
           /root/reference into oracle/_ref) on this host's cores, bounded sample;
  parity — the GPU's results on the cpu_baseline samples against the reference's results
           on the same inputs (max relative Frobenius error; pivot mismatches for dgetrf);
  series — every BASELINE config at N = 1, each entry with its roofline fraction, its own
           cpu_baseline and parity (cfg1 dgemm vs n, cfg2 gemm_nd s = 4..320, cfg3 dpotrf,
           cfg4 dgetrf, cfg5 chain cm/pm).

`--impl reference` runs only the reference CPU arm (rank 0) and prints its line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# torch's OpenMP pool must not spin-wait on the cores the CPU baseline times (a busy
# pool cost the in-process reference leg up to 1.7x); set before torch is imported
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")

M = N = K = 64
BATCH = 16384
FLOPS_PER_PROBLEM = 2 * M * N * K
BYTES_PER_PROBLEM = 8 * (M * K + K * N + 2 * M * N)
METRIC = "FP64 GFLOP/s (batched dgemm/dpotrf vs n) at 1/2/4/8 B200; % of FP64 roofline"
UNIT = "GFLOP/s"
CONFIG = {"workload": "cfg1: batched dgemm_nn column-major, m=n=k=64, lda=ldb=ldc=64, alpha=beta=1, "
                      "uniform[-1,1], one 16384-problem batch split by problem index over the GPUs",
          "global_batch": BATCH, "m": M, "n": N, "k": K,
          "l2": "inputs (2.1 GB in all; >= 268 MB per GPU at N = 8) exceed the 126 MB L2; no flush"}
NCU_SUMMARY = os.path.join(ROOT, "profiles", "r02_ncu_kernels.json")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ helpers
def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        import tempfile
        self.path = tempfile.mktemp(prefix="pbgpu_clocks_", suffix=".csv")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()
            with open(self.path) as f:
                self.lines = [ln.strip() for ln in f if ln.strip()]
            os.unlink(self.path)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        import torch
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return ws, rank, local


def max_over_ranks(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws: int):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cfg1_host_batch(lo: int, hi: int):
    """Problems [lo, hi) of the ONE seeded config-1 batch.  Block b of 256 problems draws from
    its own stream (PCG64 seeded [42, b]), so a rank generates exactly the blocks its slice
    touches and the bits of problem p never depend on the GPU count.  Returns (A, B, C) as
    (hi - lo, 64*64) float64 arrays."""
    import numpy as np
    cnt = hi - lo
    out = [np.empty((cnt, M * N)) for _ in range(3)]
    blk = 256
    for b in range(lo // blk, (hi + blk - 1) // blk):
        g = np.random.Generator(np.random.PCG64([42, b]))
        v = g.uniform(-1.0, 1.0, (3, blk, M * N))
        s0, s1 = max(lo, b * blk), min(hi, (b + 1) * blk)
        for i in range(3):
            out[i][s0 - lo:s1 - lo] = v[i][s0 - b * blk:s1 - b * blk]
    return out


# ------------------------------------------------------------------ CPU legs (oracle/_ref)
def cpu_lib():
    """The reference compiled from its own headers (oracle/_ref) where present, else the port."""
    from oracle import binding as ob
    if ob.have_ref():
        return ob.ref(), "reference"
    return ob.oracle(), "port"


def cpu_timed(make_run, reps=3):
    """Median wall time of `reps` runs after one warm-up; make_run() returns a callable over
    fresh copies of the sample's inputs (copies made outside the timed region) and the
    result of the last run stays in those copies."""
    laps = []
    last = None
    for r in range(reps + 1):
        run, state = make_run()
        t0 = time.perf_counter()
        run()
        dt = time.perf_counter() - t0
        if r:
            laps.append(dt)
        last = state
    return statistics.median(laps), last


def cpu_sample_size(per_problem_flops, batch, rate_gflops, target_s):
    s = int(target_s * rate_gflops * 1e9 / max(1, per_problem_flops))
    return max(1, min(batch, max(8, s)))


def cpu_entry(flops, sec, kind, threads, sample, batch):
    return {"value": round(flops / sec / 1e9, 3), "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{sample} of {batch} problems (the first), median of 3 after a warm-up, "
                      f"{threads} threads contiguous split, {sec:.3f} s per pass"}


def rel_rows(got, want):
    import numpy as np
    got = got.reshape(len(got), -1)
    want = want.reshape(len(want), -1)
    den = np.linalg.norm(want, axis=1)
    den[den == 0] = 1.0
    return np.linalg.norm(got - want, axis=1) / den


def cpu_reference_dgemm(A, B, C, batch, threads, reps):
    """Times the reference's own panelblas::dgemm loop over `batch` problems (C updated in place)."""
    lib, kind = cpu_lib()
    laps = []
    for _ in range(reps):
        t0 = time.perf_counter()
        lib.dgemm_batch(b"n", b"n", M, N, K, 1.0, A.ctypes.data, M, M * K, B.ctypes.data, K, K * N, 1.0,
                        C.ctypes.data, M, M * N, batch, threads)
        laps.append(time.perf_counter() - t0)
    sec = statistics.median(laps)
    return batch * FLOPS_PER_PROBLEM / sec / 1e9, kind, sec


def run_reference_arm(args, ws, rank):
    if rank != 0:
        return 0
    batch = BATCH
    A, B, C = cfg1_host_batch(0, batch)
    threads = host_threads()
    for _ in range(args.warmup):
        cpu_reference_dgemm(A, B, C, batch, threads, 1)
    secs = []
    kind = "port"
    for _ in range(args.steps):
        _, kind, s = cpu_reference_dgemm(A, B, C, batch, threads, 1)
        secs.append(s)
    total = sum(secs)
    value = args.steps * batch * FLOPS_PER_PROBLEM / total / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": CONFIG,
            "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": kind,
                             "sample": f"full cfg1 batch ({batch} problems) per step, "
                                       f"{threads} threads, contiguous split"},
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU timing helpers
def time_device(fn, steps, warmup, stream, ws):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    barrier(ws)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    return e0.elapsed_time(e1)


def _roof(flops, bytes_, peak_tf, bw):
    """FP64 roofline time (s) of one problem: max(flops / P, bytes / BW)."""
    return max(flops / (peak_tf * 1e12), bytes_ / (bw * 1e9))


def _median_ms(fn, stream, reps=3, setup=None):
    import torch
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    laps = []
    for r in range(reps + 1):
        if setup:
            setup()
        torch.cuda.synchronize()
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        if r:
            laps.append(e0.elapsed_time(e1))
    return statistics.median(laps)


def _time_copies(make_copy, launch, stream, footprint_bytes, l2_bytes=126 * 2 ** 20):
    """Device time of one launch when inputs come from HBM: R back-to-back launches on R
    distinct copies (R copies >= 2x L2), L2 flushed (a 512 MiB write) before the timed region;
    returns (ms per launch (median of 3), R, the first copy — which holds the result)."""
    import torch
    R = max(4, min(64, int(2 * l2_bytes // max(1, footprint_bytes)) + 1))
    copies = [make_copy() for _ in range(R)]
    scratch = torch.empty(64 * 2 ** 20, dtype=torch.float64, device=copies[0][0].device)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    laps = []
    for rep in range(4):
        for c in copies:
            c[1]()  # restore the pristine input
        scratch.fill_(float(rep))  # L2 flush
        torch.cuda.synchronize()
        e0.record(stream)
        for c in copies:
            launch(c[0])
        e1.record(stream)
        torch.cuda.synchronize()
        if rep:
            laps.append(e0.elapsed_time(e1) / R)
    first = copies[0][0]
    del copies, scratch
    return statistics.median(laps), R, first


class Series:
    """Shared state of the N = 1 series: CPU library, thread count, parity accumulator."""

    def __init__(self, pb, dev, stream, peak_tf, bw, cpu_target_s, skip_cpu=False):
        self.pb, self.dev, self.stream, self.peak, self.bw = pb, dev, stream, peak_tf, bw
        self.skip_cpu = skip_cpu
        self.lib, self.kind = cpu_lib()
        self.threads = host_threads()
        self.target = cpu_target_s
        self.parity: dict = {}

    def rate_probe(self, run_small, flops):
        sec, _ = cpu_timed(run_small, reps=1)
        return flops / max(sec, 1e-6) / 1e9

    def add_parity(self, cfg, key, err=None, pivots=None, tol=None):
        d = self.parity.setdefault(cfg, {"max_rel_frob_over_tol": 0.0, "problems_checked": 0})
        if err is not None:
            d["max_rel_frob_over_tol"] = max(d["max_rel_frob_over_tol"], float(err) / tol)
        if pivots is not None:
            d["pivot_mismatches"] = d.get("pivot_mismatches", 0) + int(pivots)
        d["problems_checked"] += int(key)


def series_dgemm(S: Series):
    """Config-1 shape at other n: dgemm_nn column-major, C += A B."""
    import numpy as np
    import torch
    pb, dev, stream = S.pb, S.dev, S.stream
    out = {}
    # 8 and 16: the small-n branch of the size switch (gemm_cmsmall.cu, a warp per problem)
    for n, batch in ((8, 1048576), (16, 262144), (32, 65536), (64, 16384), (128, 4096), (256, 1024)):
        g = torch.Generator(device=dev).manual_seed(n)
        A = torch.rand((batch, n, n), generator=g, device=dev, dtype=torch.float64) * 2 - 1
        B = torch.rand((batch, n, n), generator=g, device=dev, dtype=torch.float64) * 2 - 1
        C = torch.rand((batch, n, n), generator=g, device=dev, dtype=torch.float64) * 2 - 1
        fn = lambda: pb.dgemm_batched("n", "n", n, n, n, 1.0, A, n, n * n, B, n, n * n, 1.0, C, n, n * n,  # noqa
                                      batch, stream=stream)
        ms = time_device(fn, 5, 3, stream, 1) / 5
        fpp = 2 * n ** 3
        roof = batch * _roof(fpp, 32 * n * n, S.peak, S.bw)
        e = {"gflops": round(fpp * batch / ms / 1e6, 1), "ms": round(ms, 4), "batch": batch,
             "roofline_frac": round(roof * 1e3 / ms, 3)}
        if S.skip_cpu:
            out[str(n)] = e
            del A, B, C
            continue
        # CPU leg + parity on the first `smp` problems (fresh C for both sides)
        h = [x.cpu().numpy().reshape(batch, -1) for x in (A, B)]
        c0 = (torch.rand((min(batch, 4096), n * n), generator=g, device=dev, dtype=torch.float64) * 2 - 1)
        c0h = c0.cpu().numpy()

        def mk(cnt):
            def make():
                c = c0h[:cnt].copy()
                return (lambda: S.lib.dgemm_batch(b"n", b"n", n, n, n, 1.0, h[0].ctypes.data, n, n * n,
                                                  h[1].ctypes.data, n, n * n, 1.0, c.ctypes.data, n, n * n,
                                                  cnt, S.threads)), c
            return make
        rate = S.rate_probe(mk(min(64, len(c0h))), min(64, len(c0h)) * fpp)
        smp = cpu_sample_size(fpp, len(c0h), rate, S.target)
        sec, want = cpu_timed(mk(smp))
        e["cpu_baseline"] = cpu_entry(smp * fpp, sec, S.kind, S.threads, smp, batch)
        cg = c0[:smp].clone()
        assert pb.dgemm_batched("n", "n", n, n, n, 1.0, A, n, n * n, B, n, n * n, 1.0, cg, n, n * n, smp,
                                stream=stream).ok()
        err = float(rel_rows(cg.cpu().numpy(), want).max())
        e["parity"] = {"max_rel_frob": err, "problems": smp}
        S.add_parity("cfg1_dgemm_nn", smp, err, tol=1e-13 * n)
        out[str(n)] = e
        del A, B, C, c0, cg, h
        torch.cuda.empty_cache()
    return out


def series_gemm_nd(S: Series, sizes):
    """Config 2: gemm_nd NT on panel-major (ps = 4) operands, batch(s) = 2^31 / (32 s^2)."""
    import numpy as np
    import torch
    from oracle import binding as ob
    pb, dev, stream = S.pb, S.dev, S.stream
    out = {}
    for s_ in sizes:
        batch = (2 ** 31) // (32 * s_ * s_)
        L = s_ * s_
        g = torch.Generator(device=dev).manual_seed(2000 + s_)
        A = torch.rand((batch, L), generator=g, device=dev, dtype=torch.float64) * 2 - 1
        B = torch.rand((batch, L), generator=g, device=dev, dtype=torch.float64) * 2 - 1
        C = torch.rand((batch, L), generator=g, device=dev, dtype=torch.float64) * 2 - 1
        D = torch.empty_like(A)
        R = pb.PanelRef
        fn = lambda: pb.gemm_nd_batched("n", "t", s_, s_, s_, 1.0, R(A, s_, s_), L, R(B, s_, s_), L, 1.0,  # noqa
                                        R(C, s_, s_), L, R(D, s_, s_), L, batch, stream=stream)
        ms = _median_ms(fn, stream)
        fpp = 2 * s_ ** 3
        roof = batch * _roof(fpp, 32 * s_ * s_, S.peak, S.bw)
        e = {"gflops": round(fpp * batch / ms / 1e6, 1), "ms": round(ms, 4), "batch": batch,
             "roofline_frac": round(roof * 1e3 / ms, 3)}
        if S.skip_cpu:
            out[str(s_)] = e
            del A, B, C, D
            continue
        cap = min(batch, 65536)
        h = [x[:cap].cpu().numpy() for x in (A, B, C)]
        dm = lambda buf: ob.dmat(buf, s_, s_)  # noqa: E731

        def mk(cnt):
            def make():
                d = np.empty((cnt, L))
                return (lambda: S.lib.gemm_nd_batch(b"n", b"t", s_, s_, s_, 1.0, dm(h[0]), L, dm(h[1]), L, 1.0,
                                                    dm(h[2]), L, dm(d), L, cnt, S.threads)), d
            return make
        rate = S.rate_probe(mk(min(64, cap)), min(64, cap) * fpp)
        smp = cpu_sample_size(fpp, cap, rate, S.target)
        sec, want = cpu_timed(mk(smp))
        e["cpu_baseline"] = cpu_entry(smp * fpp, sec, S.kind, S.threads, smp, batch)
        err = float(rel_rows(D[:smp].cpu().numpy(), want).max())
        e["parity"] = {"max_rel_frob": err, "problems": smp}
        S.add_parity("cfg2_gemm_nd", smp, err, tol=1e-13 * s_)
        out[str(s_)] = e
        del A, B, C, D, h
        torch.cuda.empty_cache()
    return out


def series_dpotrf(S: Series):
    """dpotrf_l (config 3) at each n: inputs SPD = B B^T + n I, B ~ N(0,1); HBM-resident inputs."""
    import numpy as np
    import torch
    pb, dev, stream = S.pb, S.dev, S.stream
    out = {}
    g = torch.Generator(device=dev).manual_seed(3)
    for n in (16, 32, 64, 128, 256):
        batch = 8192
        Bm = torch.randn((batch, n, n), generator=g, device=dev, dtype=torch.float64)
        A0 = Bm @ Bm.transpose(1, 2) + n * torch.eye(n, device=dev, dtype=torch.float64)
        del Bm
        info = torch.empty(batch, dtype=torch.int32, device=dev)

        def make():
            A = A0.clone()
            return A, (lambda: A.copy_(A0))

        ms, R, res = _time_copies(make, lambda A: pb.dpotrf_batched("l", n, A, n, n * n, info, batch, stream=stream),
                                  stream, A0.numel() * 8)
        assert int(info.abs().sum()) == 0
        fpp = n * n * n // 3
        by = 8 * n * (n + 1) * batch
        roof = batch * _roof(fpp, 8 * n * (n + 1), S.peak, S.bw)
        e = {"gflops": round(fpp * batch / ms / 1e6, 1), "ms": round(ms, 4), "hbm_gbs": round(by / ms / 1e6, 1),
             "roofline_frac": round(roof * 1e3 / ms, 3), "launches_timed": R}
        if S.skip_cpu:
            out[str(n)] = e
            del A0, res
            continue
        h0 = A0.cpu().numpy().reshape(batch, -1)

        def mk(cnt):
            def make():
                a = h0[:cnt].copy()
                inf = np.zeros(cnt, np.int32)
                return (lambda: S.lib.dpotrf_batch(b"l", n, a.ctypes.data, n, n * n, inf.ctypes.data, cnt,
                                                   S.threads)), (a, inf)
            return make
        rate = S.rate_probe(mk(min(64, batch)), min(64, batch) * fpp)
        smp = cpu_sample_size(fpp, batch, rate, S.target)
        sec, (want, winfo) = cpu_timed(mk(smp))
        e["cpu_baseline"] = cpu_entry(smp * fpp, sec, S.kind, S.threads, smp, batch)
        lo = np.tril(np.ones((n, n), bool)).T.reshape(-1)
        got = res[:smp].cpu().numpy().reshape(smp, -1)
        err = float(rel_rows(got[:, lo], want[:, lo]).max())
        assert (winfo == 0).all()
        e["parity"] = {"max_rel_frob": err, "problems": smp}
        S.add_parity("cfg3_dpotrf", smp, err, tol=1e-13 * n)
        out[str(n)] = e
        del A0, res, h0
        torch.cuda.empty_cache()
    return out


def series_dgetrf(S: Series):
    """Config 4: dgetrf with partial pivoting, uniform[-1,1], batch 8192; HBM-resident inputs."""
    import numpy as np
    import torch
    pb, dev, stream = S.pb, S.dev, S.stream
    out = {}
    g = torch.Generator(device=dev).manual_seed(4)
    for n in (24, 48, 96, 192):
        batch = 8192
        A0 = torch.rand((batch, n, n), generator=g, device=dev, dtype=torch.float64) * 2 - 1
        ip = torch.empty((batch, n), dtype=torch.int32, device=dev)
        info = torch.empty(batch, dtype=torch.int32, device=dev)

        def make():
            A = A0.clone()
            return A, (lambda: A.copy_(A0))

        ms, R, res = _time_copies(make, lambda A: pb.dgetrf_batched(n, n, A, n, n * n, ip, n, info, batch,
                                                                     stream=stream), stream, A0.numel() * 8)
        fpp = n ** 3 - n ** 3 // 3
        roof = batch * _roof(fpp, 16 * n * n + 4 * n, S.peak, S.bw)
        e = {"gflops": round(fpp * batch / ms / 1e6, 1), "ms": round(ms, 4),
             "roofline_frac": round(roof * 1e3 / ms, 3), "launches_timed": R}
        if S.skip_cpu:
            out[str(n)] = e
            del A0, res
            continue
        h0 = A0.cpu().numpy().reshape(batch, -1)

        def mk(cnt):
            def make():
                a = h0[:cnt].copy()
                piv = np.zeros((cnt, n), np.int32)
                inf = np.zeros(cnt, np.int32)
                return (lambda: S.lib.dgetrf_batch(n, n, a.ctypes.data, n, n * n, piv.ctypes.data, n,
                                                   inf.ctypes.data, cnt, S.threads)), (a, piv)
            return make
        rate = S.rate_probe(mk(min(64, batch)), min(64, batch) * fpp)
        smp = cpu_sample_size(fpp, batch, rate, S.target)
        sec, (want, wpiv) = cpu_timed(mk(smp))
        e["cpu_baseline"] = cpu_entry(smp * fpp, sec, S.kind, S.threads, smp, batch)
        # the result copy was factored by the last timed launch; its pivots are in `ip`
        got = res[:smp].cpu().numpy().reshape(smp, -1)
        gp = ip[:smp].cpu().numpy()
        mism = int((~(gp == wpiv).all(axis=1)).sum())
        err = float(rel_rows(got, want).max())
        e["parity"] = {"pivot_mismatches": mism, "max_rel_frob_vs_reference_lu": err, "problems": smp}
        S.add_parity("cfg4_dgetrf", smp, err, pivots=mism, tol=1e-13 * n)
        out[str(n)] = e
        del A0, res, h0
        torch.cuda.empty_cache()
    return out


def series_chain(S: Series):
    """Config 5: 32768 problems, n = 4 U{1..64}: dsyrk_ln -> dpotrf_l -> dtrsm_rltn, cm and pm."""
    import numpy as np
    import torch
    pb, dev, stream = S.pb, S.dev, S.stream
    rng = np.random.default_rng(5)
    batch = 32768
    ns = (rng.integers(1, 65, batch) * 4).astype(np.int32)
    offs = np.concatenate([[0], np.cumsum(ns.astype(np.int64) ** 2)[:-1]]).astype(np.int64)
    total = int((ns.astype(np.int64) ** 2).sum())
    fl_p = np.array([2 * int(n) ** 3 + int(n) ** 3 // 3 for n in ns], dtype=np.float64)
    roof = float(sum(_roof(2 * int(n) ** 3 + int(n) ** 3 // 3, 8 * (3 * int(n) ** 2 + int(n) * (int(n) + 1)),
                           S.peak, S.bw) for n in ns))
    out = {}
    info = torch.empty(batch, dtype=torch.int32, device=dev)
    for layout in "CP":
        g = torch.Generator(device=dev).manual_seed(50 + (layout == "P"))
        A = torch.rand(total, generator=g, device=dev, dtype=torch.float64) * 2 - 1
        B0 = torch.rand(total, generator=g, device=dev, dtype=torch.float64) * 2 - 1
        C0 = torch.zeros(total, device=dev, dtype=torch.float64)
        for n in np.unique(ns):  # C0 = n I
            idx = np.nonzero(ns == n)[0]
            base = torch.from_numpy(offs[idx]).to(dev)
            ar = torch.arange(int(n), device=dev)
            diag = ar * (int(n) + 1) if layout == "C" else (ar // 4) * 4 * int(n) + ar * 4 + ar % 4
            C0[(base[:, None] + diag[None, :]).reshape(-1)] = float(n)
        C = C0.clone(); B = B0.clone()

        def setup():
            C.copy_(C0); B.copy_(B0)

        # n / offset passed as host arrays: the split by order is planned without a device round trip
        ms = _median_ms(lambda: pb.chain_vbatched(layout, ns, offs, A, C, B, info, batch, 256, stream=stream),
                        stream, reps=2, setup=setup)
        assert int(info.abs().sum()) == 0
        e = {"gflops": round(fl_p.sum() / ms / 1e6, 1), "ms": round(ms, 3), "roofline_frac": round(roof * 1e3 / ms, 3)}
        if S.skip_cpu:
            out["cm" if layout == "C" else "pm"] = e
            del A, B0, C0, C, B
            continue
        # CPU leg + parity: the first `smp` problems (a contiguous prefix of the buffers)
        cap = 4096
        end = int(offs[cap])
        h = [x[:end].cpu().numpy() for x in (A, C0, B0)]
        fn = S.lib.chain_cm_batch if layout == "C" else S.lib.chain_pm_batch
        cum = np.cumsum(fl_p[:cap])

        def mk(cnt):
            def make():
                e_ = int(offs[cnt]) if cnt < batch else total
                c, b = h[1][:e_].copy(), h[2][:e_].copy()
                inf = np.zeros(cnt, np.int32)
                return (lambda: fn(ns.ctypes.data, offs.ctypes.data, h[0].ctypes.data, c.ctypes.data,
                                   b.ctypes.data, inf.ctypes.data, cnt, S.threads)), (c, b, inf)
            return make
        rate = S.rate_probe(mk(64), float(cum[63]))
        smp = int(np.searchsorted(cum, S.target * rate * 1e9)) + 1
        smp = max(64, min(cap, smp))
        sec, (wc, wb, winf) = cpu_timed(mk(smp))
        e["cpu_baseline"] = cpu_entry(float(cum[smp - 1]), sec, S.kind, S.threads, smp, batch)
        assert (winf == 0).all()
        e_ = int(offs[smp])
        gc, gb = C[:e_].cpu().numpy(), B[:e_].cpu().numpy()
        worst = 0.0
        for p in range(smp):
            n, o = int(ns[p]), int(offs[p])
            for got, want in ((gc[o:o + n * n], wc[o:o + n * n]), (gb[o:o + n * n], wb[o:o + n * n])):
                den = np.linalg.norm(want)
                worst = max(worst, float(np.linalg.norm(got - want) / den) / (1e-13 * n))
        e["parity"] = {"max_rel_frob_over_tol": worst, "problems": smp}
        S.add_parity(f"cfg5_chain_{'cm' if layout == 'C' else 'pm'}", smp, worst, tol=1.0)
        out["cm" if layout == "C" else "pm"] = e
        del A, B0, C0, C, B, h
        torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------ GPU arm
def run_gpu_arm(args, ws, rank, local):
    import numpy as np
    import torch
    import paper_1902_08115_b200 as pb
    from paper_1902_08115_b200.shard import shard_of
    pb.lib()  # fail loudly when the CUDA library is missing (no CPU fallback)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    lo, hi = shard_of(BATCH, ws, rank)
    nb = hi - lo
    hA, hB, hC = (torch.from_numpy(x).pin_memory() for x in cfg1_host_batch(lo, hi))
    A, B, C = (x.to(dev) for x in (hA, hB, hC))

    def step():
        pb.dgemm_batched("n", "n", M, N, K, 1.0, A, M, M * K, B, K, K * N, 1.0, C, M, M * N, nb, stream=stream)

    with ClockSampler(local) as clk:
        # clock soak: keep the same workload running ~0.6 s so nvidia-smi (100 ms
        # period) samples the clocks under this load; then W warm-up + K timed steps
        t_end = time.perf_counter() + 0.6
        while time.perf_counter() < t_end:
            step()
            torch.cuda.synchronize()
        ms_local = time_device(step, args.steps, args.warmup, stream, ws)
    ms_total = max_over_ranks(ms_local, ws)
    ms_step = ms_total / args.steps
    value = BATCH * FLOPS_PER_PROBLEM / (ms_step * 1e-3) / 1e9

    # ---- end to end through the public API with pinned host buffers ----
    def e2e_step():
        r = pb.dgemm_batched("n", "n", M, N, K, 1.0, hA.data_ptr(), M, M * K, hB.data_ptr(), K, K * N, 1.0,
                             hC.data_ptr(), M, M * N, nb)
        assert r.ok()

    for _ in range(max(1, args.warmup)):
        e2e_step()
    barrier(ws)
    t0 = time.perf_counter()
    e2e_steps = max(1, min(args.steps, 10))
    for _ in range(e2e_steps):
        e2e_step()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps, ws)
    e2e_value = BATCH * FLOPS_PER_PROBLEM / e2e_s / 1e9
    h2d = 8 * BATCH * (M * K + K * N + M * N)
    d2h = 8 * BATCH * M * N

    line = None
    if rank == 0:
        bw, peak_kind = measured_peaks()
        ach = nb * BYTES_PER_PROBLEM / (ms_local / args.steps * 1e-3) / 1e9  # one launch per step
        traffic, ncu_src = None, None  # dram bytes read + write of this kernel per launch (ncu --set full)
        for tp in (NCU_SUMMARY, os.path.join(ROOT, "profiles", "r01_ncu_kernels.json")):
            if os.path.exists(tp):
                with open(tp) as f:
                    kd = json.load(f).get("dgemm64", {})
                if kd.get("dram_bytes_read") is not None and kd.get("dram_bytes_write") is not None:
                    traffic = (kd["dram_bytes_read"] + kd["dram_bytes_write"]) * nb / BATCH
                    ncu_src = os.path.relpath(tp, ROOT)
                    break
        dmma = pb.lib().pb_probe_dmma_tflops()
        line = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded uniform[-1,1] per problem, generated on the host)", "config": CONFIG,
                "parallelism": f"problem-index split over {ws} GPU(s): rank 0 owns [{lo}, {hi}) (no collective)",
                "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": bw, "unit": "GB/s",
                             "frac": round(ach / bw, 4), "traffic": traffic, "traffic_source": ncu_src,
                             "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
                             "kernel": "gemm_cm_kernel<8> (square packed NN branch of the size switch)",
                             "algorithmic_bytes_per_launch": nb * BYTES_PER_PROBLEM,
                             "fp64_roofline_gflops": round(ws * min(dmma * 1e3, bw * 4.0), 1),
                             "fp64_frac": round(value / ws / min(dmma * 1e3, bw * 4.0), 4),
                             "fp64_dmma_peak_tflops_measured": round(dmma, 2)},
                "e2e": {"value": round(e2e_value, 2), "unit": UNIT, "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h, "steps": e2e_steps},
                "gpu_launches": args.steps, "clocks": clk.summary()}
    # ---- CPU baseline + parity of the headline (rank 0, N = 1 only), bounded sample ----
    if rank == 0 and ws == 1 and not args.no_cpu:
        sample = min(nb, args.cpu_sample)
        a0, b0, c0 = cfg1_host_batch(0, sample)
        threads = host_threads()
        cpu_reference_dgemm(a0, b0, c0.copy(), sample, threads, 1)  # warm-up
        laps = []
        for _ in range(5):
            c = c0.copy()
            _, kind, sec = cpu_reference_dgemm(a0, b0, c, sample, threads, 1)
            laps.append(sec)
        sec = statistics.median(laps)
        line["cpu_baseline"] = {"value": round(sample * FLOPS_PER_PROBLEM / sec / 1e9, 3), "unit": UNIT,
                                "cores": threads, "kind": kind,
                                "sample": f"{sample} of the cfg1 problems, median of 5 passes after a warm-up "
                                          f"({sec:.3f} s each), {threads} threads contiguous split"}
        # parity: one fresh GPU pass over the same inputs vs the reference's result c
        cg = torch.from_numpy(c0).to(dev)
        assert pb.dgemm_batched("n", "n", M, N, K, 1.0, torch.from_numpy(a0).to(dev), M, M * K,
                                torch.from_numpy(b0).to(dev), K, K * N, 1.0, cg, M, M * N, sample).ok()
        err = float(rel_rows(cg.cpu().numpy(), c).max())
        line["parity"] = {"cfg1_headline": {"max_rel_frob": err, "tol": 1e-13 * K, "problems_checked": sample,
                                            "against": kind}}
    if rank == 0 and ws == 1 and not args.no_series:
        del A, B, C
        torch.cuda.empty_cache()
        bw, _ = measured_peaks()
        peak = pb.lib().pb_probe_dmma_tflops()
        S = Series(pb, dev, stream, peak, bw, args.cpu_target_s, skip_cpu=args.no_cpu)
        sizes = list(range(4, 321, 4)) if args.all_sizes else [4, 8, 16, 24, 32, 48, 64, 96, 128, 192, 256, 320]
        t0 = time.perf_counter()
        line["series"] = {"roofline": f"per problem max(flops / {peak:.2f} TFLOP/s measured DMMA, "
                                      f"algorithmic bytes / {bw} GB/s), summed over the batch",
                          "cpu": f"oracle/_ref (reference) on {S.threads} host threads" if S.kind == "reference"
                                 else f"oracle port on {S.threads} host threads",
                          }
        want = set(args.series.split(","))
        for key, tag, fn in (("cfg1_dgemm_nn_cm", "cfg1", lambda: series_dgemm(S)),
                             ("cfg2_gemm_nd_nt_pm", "cfg2", lambda: series_gemm_nd(S, sizes)),
                             ("cfg3_dpotrf_l", "cfg3", lambda: series_dpotrf(S)),
                             ("cfg4_dgetrf", "cfg4", lambda: series_dgetrf(S)),
                             ("cfg5_chain", "cfg5", lambda: series_chain(S))):
            if tag in want:
                line["series"][key] = fn()
        line.setdefault("parity", {}).update(S.parity)
        line["series"]["seconds"] = round(time.perf_counter() - t0, 1)
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="pbgpu", choices=["pbgpu", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=16384)
    ap.add_argument("--cpu-target-s", type=float, default=0.4, help="CPU seconds per series sample pass")
    ap.add_argument("--no-cpu", action="store_true", help="no CPU legs (and no parity block)")
    ap.add_argument("--no-series", action="store_true")
    ap.add_argument("--all-sizes", action="store_true", help="cfg2 series over all 80 sizes")
    ap.add_argument("--series", default="cfg1,cfg2,cfg3,cfg4,cfg5", help="which config series to run")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "pbgpu" else args.warmup
    ws, rank, local = dist_init()
    try:
        if args.impl == "reference":
            return run_reference_arm(args, ws, rank)
        return run_gpu_arm(args, ws, rank, local)
    finally:
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
