"""Per-(kernel, grid) totals of an ncu --metrics gpu__time_duration.sum --csv log:
tools/ncu_launches.py LOG [min_slots]  (batched launches only: a grid dimension >= min_slots)"""
import collections
import csv
import re
import sys


def summarize(path, min_slots=64):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, gi, vi, ui = (h.index(x) for x in ("Kernel Name", "Grid Size", "Metric Value", "Metric Unit"))
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        dims = [int(x) for x in re.findall(r"\d+", r[gi])]
        name = r[ki].split("(")[0].replace("void ", "").replace("rgbid_b200::", "")
        per_slot = name in ("k_solve", "k_covariance")  # grid.x = slots
        if (dims[0] if per_slot else max(dims[1:])) < min_slots:
            continue
        agg[(name, r[gi])][0] += 1
        agg[(name, r[gi])][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
    tot = sum(v[1] for v in agg.values())
    out = []
    for (k, g), (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"   {k:34s} {g:16s} {n:4d} {ms:9.3f} ms {ms / n * 1e3:9.1f} us/launch {ms / tot:6.3f}")
    return tot, out


if __name__ == "__main__":
    tot, out = summarize(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 64)
    print(f"total {tot:.3f} ms")
    print("\n".join(out))
