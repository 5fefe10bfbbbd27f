"""Summarise ncu outputs for profiles/: a launch list (gpu__time_duration per kernel, share of the
step) and the key metrics of a --set full capture.  Usage:
    python tools/ncu_summary.py launches <launches.csv> [steps]
    python tools/ncu_summary.py full <report.ncu-rep>
"""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    r"gpu__time_duration\.sum$", r"sm__cycles_elapsed\.avg\.per_second$",
    r"sm__pipe_tensor_cycles_active_realtime\.avg\.pct_of_peak_sustained_elapsed$",
    r"TriageCompute\.sm__pipe_tensor_cycles_active_realtime",
    r"dram__bytes_read\.sum$", r"dram__bytes_write\.sum$",
    r"dram__throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"gpu__dram_throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"lts__throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"l1tex__throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"sm__throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"launch__registers_per_thread$", r"launch__grid_size$", r"launch__block_size$",
    r"launch__shared_mem_per_block_dynamic$", r"sm__warps_active\.avg\.pct_of_peak_sustained_active$",
    r"smsp__inst_executed\.sum$",
]


def launches(path, steps=None):
    txt = open(path).read()
    start = txt.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    per = {}
    for r in rows:
        if r.get("Metric Name", "gpu__time_duration.sum") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).split("::")[-1]
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
        per.setdefault(name, []).append(v * scale)
    tot = sum(sum(v) for v in per.values())
    out = {k: {"launches": len(v), "mean_us": sum(v) / len(v), "share": sum(v) / tot} for k, v in per.items()}
    return out


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[hdr.index("Kernel Name")][:80]}
        for i, n in enumerate(hdr):
            if any(re.search(k, n) for k in KEYS):
                d[n] = f"{v[i]} {units[i]}".strip()
        res.append(d)
    return res


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if mode == "launches" else full(path), indent=1))
