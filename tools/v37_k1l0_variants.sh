#!/bin/bash
# K1 level-0 occupancy variant (RGBID_K1L0_MINB=16: 2048 threads/SM at 32 registers) vs the default 12
for v in default k1l0_m16; do
  if [ $v = default ]; then L=paper_1807_08271_b200/_lib/librgbid_b200.so; else L=build/$v/librgbid_b200.so; fi
  RGBID_LIB=$L python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x > gpurun_out/v37_par_$v.log 2>&1
  RGBID_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_warp_residuals_l0 --csv \
    --log-file gpurun_out/v37_k1_$v.csv python tools/prof_run.py --pairs 512 --levels 1 --iters 3 > gpurun_out/v37_prof_$v.log 2>&1
done
bash tools/bench_variants.sh k1l0_m16
