#!/bin/bash
# ncu per-launch durations of the kernels matching $1 for each prebuilt variant under build/<v>/
# usage: tools/variant_times_k.sh REGEX v1 v2 ...   (results in gpurun_out/var_<v>.csv)
re=$1; shift
python tools/prof_run.py --pairs 512 --levels 4 --iters 2 > /dev/null || exit 1
for v in "$@"; do
  RGBID_LIB=build/$v/librgbid_b200.so ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"$re" --csv --log-file gpurun_out/var_$v.csv \
    python tools/prof_run.py --pairs 512 --levels 4 --iters 2 > gpurun_out/var_$v.log 2>&1
done
