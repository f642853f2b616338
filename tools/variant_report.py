"""Summarise gpurun_out/var_<v>.csv (ncu launch lists of k_tdist) per variant."""
import csv, sys
for v in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f"gpurun_out/var_{v}.csv")) if len(r) > 5]
    h = rows[0]
    t = [float(r[h.index("Metric Value")]) / 1e6 for r in rows[1:]]
    print(v, "total %.2f ms" % sum(t), " ".join("%.2f" % x for x in t))
