"""Per-kernel achieved DRAM bandwidth from an ncu --csv launch list with
gpu__time_duration.sum, dram__bytes_read.sum and dram__bytes_write.sum:
the last launch of each kernel (steady state), GB/s and the fraction of the
measured HBM copy peak (MEASURED_PEAKS.json).
usage: python tools/hbm_table.py launches.csv > profiles/r1_all_kernels_hbm.txt"""
import collections
import csv
import io
import json
import os
import sys

txt = open(sys.argv[1]).read()
rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
per = collections.OrderedDict()
for r in rows:
    key = (r["ID"], r["Kernel Name"].split("(")[0].replace("<unnamed>::", "").replace("void ", ""))
    unit = r["Metric Unit"]
    v = float(r["Metric Value"].replace(",", ""))
    scale = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
    per.setdefault(key, {})[r["Metric Name"]] = v * scale
last = collections.OrderedDict()
count = collections.Counter()
for (i, name), m in per.items():
    last[name] = m
    count[name] += 1
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peaks = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))
peak = None
for k, v in peaks.items():
    if "hbm" in k.lower() and isinstance(v, (int, float)):
        peak = float(v)
        break
print(f"# per-kernel DRAM bandwidth, last launch of each kernel ({sys.argv[1]})")
print(f"# peak = {peak} GB/s (MEASURED_PEAKS.json HBM copy); ncu serialises launches and runs cold-cache")
print(f"{'kernel':34s} {'launches':>8s} {'us':>10s} {'MB read':>10s} {'MB write':>10s} {'GB/s':>8s} {'frac':>6s}")
for name, m in last.items():
    t = m.get("gpu__time_duration.sum", 0.0)
    rd, wr = m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0)
    gbs = (rd + wr) / t / 1e9 if t > 0 else 0.0
    frac = gbs / peak if peak else float("nan")
    print(f"{name:34s} {count[name]:8d} {t * 1e6:10.1f} {rd / 1e6:10.2f} {wr / 1e6:10.2f} {gbs:8.1f} {frac:6.3f}")
