"""Prints the headline and the series of a bench.py JSON line (file argument, last line)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
s = d.pop("series", None) or {}
for k in ("value", "ms_per_step", "roofline", "e2e", "cpu_baseline", "parity", "clocks"):
    if k in d:
        print(k, json.dumps(d[k])[:600])
for cfg, v in s.items():
    if isinstance(v, dict):
        for n, e in v.items():
            print(f"{cfg:20s} {n:>4s} {e.get('ms')!s:>8} ms {e.get('gflops')!s:>9} GF/s frac {e.get('roofline_frac')!s:6}"
                  f" cpu {e.get('cpu_baseline', {}).get('value')!s:8} parity {e.get('parity')}")
    else:
        print(cfg, v)
