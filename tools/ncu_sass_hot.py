"""Top SASS instructions by warp-stall samples from an `ncu --page source --csv
--print-source sass` export, with the dominant stall reasons.

    python tools/ncu_sass_hot.py export.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = rows[2:]


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


tot = sum(num(r[idx["Warp Stall Sampling (All Samples)"]]) for r in data)
print(f"total samples {tot}")
order = sorted(range(len(data)), key=lambda i: -num(data[i][idx["Warp Stall Sampling (All Samples)"]]))
for i in order[:n]:
    r = data[i]
    s = num(r[idx["Warp Stall Sampling (All Samples)"]])
    top = sorted(((num(r[idx[h]]), h[6:]) for h in reasons), reverse=True)[:3]
    print(f"{i:5d} {s:6d} {100 * s / tot:5.1f}%  {r[1].strip()[:60]:60s} " + " ".join(f"{h}:{v}" for v, h in top if v))
