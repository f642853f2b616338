#!/bin/bash
# A/B of prebuilt library variants on one GPU (build/<v>/librgbid_b200.so; "cur" = the
# in-tree _lib): per-kernel ncu launch times of one 4-level batched align (512 pairs)
# and the bench step (device-resident, no e2e / CPU / extras), per variant.
# usage: tools/ab_variants.sh tag v1 v2 ...  -> gpurun_out/ab_<tag>_<v>.{csv,json}
tag=$1; shift
for v in "$@"; do
  if [ "$v" = cur ]; then lib=paper_1807_08271_b200/_lib/librgbid_b200.so; else lib=build/$v/librgbid_b200.so; fi
  RGBID_LIB=$lib python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu --no-extra \
    > gpurun_out/ab_${tag}_$v.json 2> gpurun_out/ab_${tag}_$v.err
  RGBID_GRAPH_SWITCH=0 RGBID_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ab_${tag}_$v.csv python tools/prof_run.py --pairs 512 --levels 4 --iters 2 \
    > gpurun_out/ab_${tag}_$v.log 2>&1
done
for v in "$@"; do
  python - "$tag" "$v" <<'PY'
import json, sys, csv, collections
tag, v = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/ab_{tag}_{v}.json").read().strip().splitlines()[-1])
    print(f"{v}: value {d['value']:.1f} align/s  ms/step {d['ms_per_step']:.1f}  ok {d['status']['ok']}")
except Exception as e:
    print(v, "bench failed", e)
rows = [r for r in csv.reader(open(f"gpurun_out/ab_{tag}_{v}.csv")) if len(r) > 10]
h = rows[0]
ki, gi, vi = h.index("Kernel Name"), h.index("Grid Size"), h.index("Metric Value")
ui = h.index("Metric Unit")
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[ki].startswith(("k_render", "void k_render")):  # the input synthesis
        continue
    k = (r[ki].split("(")[0][:40], r[gi])
    agg[k][0] += 1
    agg[k][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
print(f"   total {sum(ms for _, ms in agg.values()):.3f} ms")
for (k, g), (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"   {k:42s} {g:16s} {n:4d} {ms:9.3f} ms  {ms / n * 1e3:9.1f} us/launch")
PY
done
