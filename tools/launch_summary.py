"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel name."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; agg = collections.defaultdict(lambda: [0, 0.0]); tot = 0
for r in rows:
    if r and r[0] == "ID":
        hdr = r; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); continue
    if hdr and len(r) > vi:
        try: v = float(r[vi].replace(",", ""))
        except ValueError: continue
        k = r[ki][:80]; agg[k][0] += 1; agg[k][1] += v; tot += v
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{v/1e6:9.3f} ms {c:5d}x {100*v/tot:5.1f}%  {k}")
print("total", tot / 1e6, "ms")
