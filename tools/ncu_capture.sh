#!/bin/bash
# One ncu --set full capture of the batched align (prof_run, one chunk of `pairs`
# slots, `levels` levels, 1 iteration), summarised on the box: per-kernel brief and
# per-source-line stall attribution of the named kernels; the .ncu-rep is kept only
# if small.  usage: tools/ncu_capture.sh tag "capture_regex" pairs levels kregex:mangled ...
tag=$1; regex=$2; pairs=$3; levels=$4; shift 4
out=gpurun_out/ncu_$tag
RGBID_GRAPH_SWITCH=0 RGBID_BATCH_SLOTS=$pairs ncu --set full --import-source on --clock-control none -k regex:"$regex" \
  -o $out python tools/prof_run.py --pairs $pairs --levels $levels --iters 1 > $out.log 2>&1
python tools/ncu_brief.py $out.ncu-rep > $out.brief.txt 2>&1
mkdir -p /tmp/cub_$tag && (cd /tmp/cub_$tag && cuobjdump -xelf all $GRAFT_REPO_ROOT/paper_1807_08271_b200/_lib/obj/align_kernels.cu.o > /dev/null)
cub=$(ls /tmp/cub_$tag/*.cubin | head -1)
for km in "$@"; do
  k=${km%:*}; m=${km##*:}
  python tools/ncu_src_stalls.py $out.ncu-rep "$k" $cub "$m" 45 > $out.src_$m.txt 2>&1
done
sz=$(stat -c %s $out.ncu-rep)
if [ "$sz" -gt 30000000 ]; then rm -f $out.ncu-rep; fi
