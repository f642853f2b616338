#!/bin/bash
# The round-end measurement set on one GPU: ncu FP64 flop count of the bench workload
# (-> profiles/r02_fp64_flops.json, read by bench.py), bench.py at 10 and 20 steps,
# and the ncu launch list of the bench step (switch nodes off: ncu cannot profile the
# kernel nodes of a graph with conditional nodes).  Outputs in gpurun_out/.
M=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum
RGBID_GRAPH_SWITCH=0 ncu --metrics $M --csv --log-file gpurun_out/fp64_metrics.csv python tools/prof_run.py --pairs 256 --levels 4 --iters 0 --variant mixed > gpurun_out/fp64_run.log 2>&1
python tools/fp64_flops.py gpurun_out/fp64_metrics.csv 256 profiles/r02_fp64_flops.json > gpurun_out/fp64_flops.txt 2>&1
cp profiles/r02_fp64_flops.json gpurun_out/r02_fp64_flops.json
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_final_s20.json 2> gpurun_out/bench_final_s20.err
RGBID_GRAPH_SWITCH=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extra > gpurun_out/launches_final.log 2>&1
