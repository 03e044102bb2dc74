"""Aggregate an ncu `--page source --csv --print-source cuda,sass` dump per CUDA source line.

usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_lines.py x.csv [top]
prints: file:line, warp-instructions executed, stall samples, source text.
"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, agg = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ii = hdr.index("Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or r[0] in ("Function Name",):
        continue
    if r[0] != "":
        try:
            agg.append((int(r[ii] or 0), int(r[si] or 0), f"{fname}:{r[0]}", r[1].strip()[:90]))
        except ValueError:
            pass
tot_i = sum(a[0] for a in agg) or 1
tot_s = sum(a[1] for a in agg) or 1
print(f"total warp-instr {tot_i}  stall samples {tot_s}")
for a in sorted(agg, key=lambda a: -a[1])[:top]:
    print(f"{a[2]:28s} inst {a[0]:>10d} ({100*a[0]/tot_i:4.1f}%)  stall {a[1]:>6d} ({100*a[1]/tot_s:4.1f}%)  {a[3]}")


def reasons(path, lines):
    """per-line stall-reason breakdown for the given 'file:line' keys"""
    rows = list(csv.reader(open(path)))
    fname, hdr = None, None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "" or r[0] == "Function Name":
            continue
        key = f"{fname}:{r[0]}"
        if key in lines:
            out = []
            for i, h in enumerate(hdr):
                if h.startswith("stall_") and "Not Issued" not in h:
                    try:
                        v = int(r[i] or 0)
                    except ValueError:
                        continue
                    if v:
                        out.append((v, h[6:]))
            out.sort(reverse=True)
            print(key, " ".join(f"{h}={v}" for v, h in out[:6]))


if len(sys.argv) > 3:
    reasons(sys.argv[1], set(sys.argv[3].split(",")))
