"""Kernel shares from an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, data = rows[0], rows[1:]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    try:
        v = float(r[iv])
    except ValueError:
        continue
    name = r[ik].split("(")[0].replace("void ", "").replace("dwdp::", "").replace("<unnamed>::", "")
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
out = [{"kernel": k, "launches": v[0], "total_ms": round(v[1] / 1e6, 3), "share": round(v[1] / tot, 4)}
       for k, v in sorted(agg.items(), key=lambda x: -x[1][1])]
if len(sys.argv) > 2:
    json.dump({"source": sys.argv[1], "kernel_share": out}, open(sys.argv[2], "w"), indent=1)
for o in out:
    print(f"{o['kernel']:45s} {o['launches']:4d} {o['total_ms']:9.2f} ms {o['share']:.3f}")
