"""Extract the DRAM traffic of the dominant kernel from an `ncu --set full --csv --page raw`
capture and write it as JSON for bench.py's roofline.traffic:

    python profiles/traffic.py profiles/<capture>_raw.csv k_patch_apply_tma > profiles/k2_traffic.json

traffic = dram__bytes_read.sum + dram__bytes_write.sum of the first launch whose name
contains the given kernel substring (bytes per launch)."""
import csv
import json
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
want = sys.argv[2]
k = hdr.index("Kernel Name")
col = {n: hdr.index(n) for n in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}
for r in rows[2:]:
    if want in r[k]:
        val = {n: float(r[i].replace(",", "")) * UNITS.get(units[i], 1.0) for n, i in col.items()
               if n != "gpu__time_duration.sum"}
        print(json.dumps({"kernel": r[k].split("(")[0], "source": sys.argv[1],
                          "dram_read_bytes": val["dram__bytes_read.sum"],
                          "dram_write_bytes": val["dram__bytes_write.sum"],
                          "traffic_bytes_per_launch": val["dram__bytes_read.sum"] + val["dram__bytes_write.sum"],
                          "duration": f"{r[col['gpu__time_duration.sum']]} {units[col['gpu__time_duration.sum']]}"}))
        break
