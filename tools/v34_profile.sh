#!/bin/bash
# v34 evidence refresh: ncu --set full of the top kernels on the current build, and the bench launch list
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_warp_residuals|k_normal_eq_mma|k_tdist_big" -c 6 \
  -o gpurun_out/v34_top python tools/prof_run.py --pairs 512 --levels 4 --iters 1 > gpurun_out/v34_ncu_full.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v34_launches.csv \
  python bench.py --no-e2e --no-cpu --steps 1 --warmup 1 > gpurun_out/v34_launches.log 2>&1
