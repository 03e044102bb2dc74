"""Compact JSON summary of an ncu --set full capture exported as <name>_details.csv / <name>_raw.csv.

usage: python tools/profile_summary.py gpurun_out/<name> [algorithmic_bytes] [flops]  -> JSON on stdout
"""
import csv, json, sys

base = sys.argv[1]
alg_bytes = float(sys.argv[2]) if len(sys.argv) > 2 else None
flops = float(sys.argv[3]) if len(sys.argv) > 3 else None
rows = list(csv.reader(open(base + "_details.csv")))
hdr = rows[0]
ki, vi, ui = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
det = {}
for r in rows[1:]:
    if len(r) > vi and r[ki] not in det:
        det[r[ki]] = (r[vi], r[ui])
raw_rows = list(csv.reader(open(base + "_raw.csv")))
raw = dict(zip(raw_rows[0], raw_rows[2]))
units = dict(zip(raw_rows[0], raw_rows[1]))


def rawf(k):
    v = raw.get(k)
    try:
        return float(v.replace(",", ""))
    except Exception:
        return None


def to_bytes(k):
    v, u = rawf(k), units.get(k, "")
    if v is None:
        return None
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), rawf(k)) for k in raw
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and rawf(k)]
tot = sum(v for _, v in st) or 1
dur_ns = rawf("gpu__time_duration.sum")
dur_u = units.get("gpu__time_duration.sum", "ns")
dur_s = dur_ns * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}.get(dur_u, 1e-9)
rd, wr = to_bytes("dram__bytes_read.sum"), to_bytes("dram__bytes_write.sum")
out = {
    "kernel": rows[1][hdr.index("Kernel Name")],
    "duration_us": round(dur_s * 1e6, 2),
    "dram_bytes_read": rd, "dram_bytes_write": wr,
    "dram_gbs": round((rd + wr) / dur_s / 1e9, 1) if rd is not None and wr is not None else None,
    "fp64_pipe_pct": rawf("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
    "dmma_pipe_pct": rawf("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"),
    "ipc_active": det.get("Executed Ipc Active", ("", ""))[0],
    "issue_slots_busy_pct": det.get("Issue Slots Busy", ("", ""))[0],
    "warps_active_per_sm": det.get("Achieved Active Warps Per SM", ("", ""))[0],
    "registers": det.get("Registers Per Thread", ("", ""))[0],
    "smem_per_block": " ".join(det.get("Dynamic Shared Memory Per Block", ("", ""))),
    "instructions": det.get("Executed Instructions", ("", ""))[0],
    "top_stalls": {k: round(v / tot, 3) for k, v in sorted(st, key=lambda x: -x[1])[:6]},
}
if alg_bytes:
    out["algorithmic_bytes"] = alg_bytes
    out["algorithmic_gbs"] = round(alg_bytes / dur_s / 1e9, 1)
if flops:
    out["flops"] = flops
    out["tflops"] = round(flops / dur_s / 1e12, 2)
print(json.dumps(out, indent=1))
