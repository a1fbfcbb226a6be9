"""Summarise an ncu --csv K6 capture (tools/k6_profile.py): per launch, ms, FP64 pipe %."""
import csv
import io
import sys

for f in sys.argv[1:]:
    lines = open(f).read().splitlines()
    hdr = [i for i, l in enumerate(lines) if l.startswith('"ID"')]
    print("==", f)
    if not hdr:
        print("\n".join(lines[-3:]))
        continue
    by = {}
    for r in csv.DictReader(io.StringIO("\n".join(lines[hdr[0]:]))):
        d = by.setdefault(r["ID"], {"k": r["Kernel Name"].split("(")[0], "g": r["Grid Size"]})
        d[r["Metric Name"]] = r["Metric Value"]
    tot = 0.0
    for i, d in by.items():
        ms = float(d["gpu__time_duration.sum"]) / 1e6
        tot += ms
        print(f"  {i} {d['k']:<32} grid {d['g']:<14} {ms:8.3f} ms  fp64 pipe "
              f"{d.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active')} %")
    print(f"  total {tot:.3f} ms")
