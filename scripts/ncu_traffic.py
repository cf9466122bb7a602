"""Turn `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv` output for one DP
launch into profiles/traffic_<config>.json (read by bench.py for roofline.traffic).
Usage: python scripts/ncu_traffic.py <ncu.csv> <config> <Z> <N> <M>"""
import csv, json, os, sys

path, config, Z, N, M = sys.argv[1:6]
rows = [r for r in csv.reader(open(path)) if r]
hi = next(i for i, r in enumerate(rows) if "Metric Name" in r)
h = rows[hi]
kn, mn, mu, mv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
vals = {}
for r in rows[hi + 1:]:
    if "sdtw_dp" in r[kn] and r[mn].startswith("dram__bytes"):
        vals[r[mn]] = float(r[mv].replace(",", "")) * scale.get(r[mu], 1)
    if "sdtw_dp" in r[kn] and r[mn] == "gpu__time_duration.sum":
        vals["time_" + r[mu]] = float(r[mv].replace(",", ""))
out = {"config": config, "Z": int(Z), "N": int(N), "M": int(M), "precision": 32,
       "dram_bytes_read": vals.get("dram__bytes_read.sum"), "dram_bytes_write": vals.get("dram__bytes_write.sum"),
       "dram_bytes_per_launch": vals.get("dram__bytes_read.sum", 0) + vals.get("dram__bytes_write.sum", 0),
       "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (one DP launch of bench.py --config %s)" % config}
dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic_%s.json" % config)
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out))
