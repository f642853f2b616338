#!/bin/bash
# level-0 K1 and K3, ncu --set full on the current build (one 512-slot launch each)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_warp_residuals_l0|k_normal_eq_mma" -c 2 \
  -o gpurun_out/v35_l0 python tools/prof_run.py --pairs 512 --levels 1 --iters 1 > gpurun_out/v35_ncu_full.log 2>&1
