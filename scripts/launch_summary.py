"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) into per-kernel shares."""
import csv, sys
from collections import defaultdict
path, out = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(path)) if len(r) > 5]
hdr = rows[0]; idx = {h: i for i, h in enumerate(hdr)}
agg = defaultdict(list)
for r in rows[1:]:
    if r[idx['Metric Name']] != 'gpu__time_duration.sum':
        continue
    name = r[idx['Kernel Name']].split('(')[0]
    agg[name].append(float(r[idx['Metric Value']].replace(',', '')))
tot = sum(sum(v) for v in agg.values())
lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)",
         f"# command: {' '.join(sys.argv[3:]) or 'bench.py'}", ""]
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"{k[:90]:90s} launches={len(v):4d} mean_ns={sum(v)/len(v):10.0f} share={sum(v)/tot*100:5.1f}%")
open(out, 'w').write("\n".join(lines) + "\n")
print("\n".join(lines))
