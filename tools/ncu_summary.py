"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per
(kernel, grid) — separates batched launches from single-pair ones."""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path, title=""):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, vi, ui, gi = (h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"),
                      h.index("Grid Size"))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("rgbid_b200::", "").replace("void ", "")
        a = agg[(name, r[gi])]
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    if title:
        print(title)
    print(f"{'kernel':34s} {'grid':16s} {'launches':>8s} {'total_ms':>10s} {'avg_us':>10s} {'share':>6s}")
    for (k, g), v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:34]:34s} {g:16s} {v[0]:8d} {v[1] / 1e3:10.3f} {v[1] / v[0]:10.1f} {v[1] / tot:6.3f}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
