"""Per-launch kernel times from an ncu --csv gpu__time_duration log.
  python tools/launch_times.py gpurun_out/x.csv [substring ...]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]
pats = sys.argv[2:]
for r in rows[i + 1:]:
    d = dict(zip(h, r))
    if not pats or any(p in d["Kernel Name"] for p in pats):
        print(f"{d['Kernel Name'][:48]:48s} {d['Grid Size']:>14s} {d['Metric Value']:>14s} {d['Metric Unit']}")
