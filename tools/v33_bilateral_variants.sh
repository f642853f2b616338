python -m pytest tests/test_golden.py -m gpu -q > gpurun_out/v33_golden_gpu.log 2>&1; echo exit=$? >> gpurun_out/v33_golden_gpu.log
for v in default bil_r4 bil_r1 bil_m6r4; do
  if [ $v = default ]; then L=paper_1807_08271_b200/_lib/librgbid_b200.so; else L=build/$v/librgbid_b200.so; fi
  RGBID_LIB=$L python -m pytest tests/test_gpu_parity.py -m gpu -q -k bilateral > gpurun_out/v33_par_$v.log 2>&1
  RGBID_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_bilateral --csv --log-file gpurun_out/v33_bil_$v.csv python tools/prof_run.py --pairs 512 --levels 1 --iters 1 > gpurun_out/v33_prof_$v.log 2>&1
done
bash tools/bench_variants.sh bil_r4 bil_m6r4
