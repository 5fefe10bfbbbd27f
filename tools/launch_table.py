"""Per-launch table from an ncu --csv log with gpu__time_duration + dram bytes (tools/gpu_stream.sh)."""
import csv, io, re, sys
txt = open(sys.argv[1]).read()
rows = list(csv.DictReader(io.StringIO(txt[txt.find('"ID"'):])))
agg = {}
for r in rows:
    n = re.sub(r"\(.*", "", r["Kernel Name"]).split("::")[-1]
    agg.setdefault((int(r["ID"]), n), {})[r["Metric Name"]] = (float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
T = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
for (i, n), m in sorted(agg.items()):
    t = m["gpu__time_duration.sum"]; t = t[0] * T[t[1]]
    d = sum(v[0] * B[v[1]] for k, v in m.items() if k.startswith("dram__bytes"))
    print(f"{i:>4} {n:26s} {t*1e6:10.1f} us  dram {d/1e6:10.1f} MB  {d/t/1e9:8.1f} GB/s")
