"""Sums an ncu --csv metric list (gpu__time_duration, dram__bytes_read/write) over
the captured launches: per-kernel table + totals, and writes a JSON summary.

    python tools/ncu_traffic.py launches.csv out.json "label"
"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
K = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    k = K.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")})
    k[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for k in K.values():
    a = agg[k["name"][:70]]
    a[0] += 1
    a[1] += k.get("gpu__time_duration.sum", 0) / 1e3
    a[2] += k.get("dram__bytes_read.sum", 0)
    a[3] += k.get("dram__bytes_write.sum", 0)
tot_us = sum(v[1] for v in agg.values())
tot_r = sum(v[2] for v in agg.values())
tot_w = sum(v[3] for v in agg.values())
print(f"{len(K)} launches, {tot_us:.1f} us (serialised, ncu), DRAM read {tot_r / 1e6:.1f} MB, write {tot_w / 1e6:.1f} MB")
for name, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v[1]:9.1f} us {v[0]:4d}x  r {v[2] / 1e6:8.1f} MB  w {v[3] / 1e6:8.1f} MB  {name}")
out = {"label": sys.argv[3] if len(sys.argv) > 3 else "", "launches": len(K), "ncu_serial_us": tot_us,
       "dram_bytes_read": tot_r, "dram_bytes_write": tot_w, "dram_bytes": tot_r + tot_w}
if len(sys.argv) > 4:  # UNet rows of the captured forward (bench.py matches its roofline traffic on it)
    out["rows"] = int(sys.argv[4])
    out["source"] = (f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none over one UNet "
                     f"forward (tools/prof_unet.py {out['rows']} 3, last forward), tools/gpu_profile_round.sh")
json.dump(out, open(sys.argv[2], "w"), indent=1)
