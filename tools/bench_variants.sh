#!/bin/bash
# full bench (device-resident step only) for the default build and prebuilt variants
python bench.py --no-e2e --no-cpu --steps 2 --warmup 3 > gpurun_out/bv_default.json 2> /dev/null
for v in "$@"; do
  RGBID_LIB=build/$v/librgbid_b200.so python bench.py --no-e2e --no-cpu --steps 2 --warmup 3 \
    > gpurun_out/bv_$v.json 2> /dev/null
done
