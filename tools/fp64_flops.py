"""Step-level FP64 work per kernel family from an ncu --csv metrics log of
tools/prof_run.py (bench workload): flops = 2 DFMA + DMUL + DADD (thread
instructions) + 512 per DMMA.884 warp instruction (8x8x4 FMAs).  Writes
profiles/r02_fp64_flops.json (bench.py's roofline.fp64_step reads it).
usage: tools/fp64_flops.py LOG N_ALIGNMENTS OUT_JSON"""
import collections
import csv
import json
import sys

FAM = [("warp_residuals", "warp (K1)"), ("tdist", "Student-t (K2b)"), ("gather", "sample gather (K2a)"),
       ("normal_eq", "normal equations (K3)"), ("bilateral", "bilateral"), ("prep_A", "prep_A"),
       ("solve", "solve (K4)"), ("covariance", "covariance")]


def family(name):
    for k, f in FAM:
        if k in name:
            return f
    return "other"


def main(log, n_align, out):
    rows = [r for r in csv.reader(open(log)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", "") or 0)
        names[r[ii]] = r[ki]
    fl = collections.Counter()
    for i, m in per.items():
        f = family(names[i])
        if f == "other":
            continue
        fl[f] += (2 * m.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 0)
                  + m.get("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", 0)
                  + m.get("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", 0)
                  + 512 * m.get("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", 0))
    res = {"flop_per_alignment": {f: v / n_align for f, v in sorted(fl.items())},
           "alignments": n_align,
           "source": "ncu --metrics dfma/dmul/dadd thread instructions + DMMA warp instructions of "
                     "tools/prof_run.py --pairs %d --levels 4 --iters 0 --variant mixed (bench workload)"
                     % n_align}
    json.dump(res, open(out, "w"), indent=1)
    tot = sum(res["flop_per_alignment"].values())
    for f, v in sorted(res["flop_per_alignment"].items(), key=lambda kv: -kv[1]):
        print(f"{f:26s} {v / 1e9:8.3f} GFLOP/alignment {v / tot:6.3f}")
    print(f"{'total':26s} {tot / 1e9:8.3f} GFLOP/alignment")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3])
