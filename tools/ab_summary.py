import glob, json, sys
for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab_*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable", e); continue
    c = d["clocks"]; r = d["roofline"]
    pw = c.get("power_w") or 0
    mhz = c.get("sm_mhz") or 1965
    print(f"{f:28s} {d['value']:10.0f} p/s  K2 {r['achieved']:7.1f} TF/s  {mhz} MHz  {pw:.0f} W  "
          f"{pw / r['achieved'] if pw else 0:.3f} pJ/flop  per-clk {r['achieved']*1e12/(148*mhz*1e6)/8192:.3f}")
