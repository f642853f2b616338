#!/bin/bash
# single-pair latency (tools/latency.py, 4 levels) for prebuilt variants under build/<v>/
for v in "$@"; do
  echo "== $v"
  RGBID_LIB=build/$v/librgbid_b200.so timeout 300 python tools/latency.py 2>&1 | head -2
done
