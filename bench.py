#!/usr/bin/env python
"""bench.py — frame-pair alignments/sec @640x480, 4-level (BASELINE.json config 5),
plus ms/frame latency.

Our arm (default):  `python bench.py --gpus N --steps K --warmup W` (torchrun for N>1,
one rank per GPU over NCCL).  Each rank holds its share of the 4096 independent
640x480 frame pairs resident in HBM (device-rendered, SURVEY §8d scene), and one
step aligns all of them (rgbid_align_batch: 4 levels, iterations {10,5,4,5} +
the filtered-Hessian covariance pass).  The only collective is the NCCL
all_gather of the fixed-size result records.  Timed with CUDA events on the
library stream, max over ranks.  Rank 0 prints one JSON line.

Reference arm: `python bench.py --impl reference ...` times the reference's own
CPU implementation (oracle/_ref: the unmodified reference sources compiled in
place) on the host cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frame-pair alignments/sec @640x480 4-lvl (1/2/4/8 GPU); ms/frame latency"
UNIT = "alignments/s"
W0, H0, F0 = 640, 480, 480.0
LEVELS, ITERS = 4, [10, 5, 4]  # level 3 defaults to 5 (src/alignment.cpp:373-374)
M_BYTES = W0 * H0 * 8  # one fp64 map
N0 = W0 * H0


def pairs_total(args, world):
    """weak scaling: --pairs per GPU; strong: --pairs split over the GPUs"""
    return args.pairs * world if args.scaling == "weak" else args.pairs


def workload_config(args, world):
    return {
        "workload": "config5: batched independent 640x480 frame-pair alignments, "
                    "4-level pyramid, iterations {10,5,4,5} + filtered-Hessian covariance",
        "pairs_total": pairs_total(args, world),
        "pairs_per_gpu": pairs_total(args, world) // world,
        "levels": LEVELS,
        "iterations": [10, 5, 4, 5],
        "variant": "noisy+occluder" if args.variant == 1 else "clean",
        "image": f"{W0}x{H0} fp64 (intensity + inverse depth), f={F0}",
        "parallelism": (f"{args.scaling} scaling over {world} GPU(s): each rank renders and aligns "
                        f"its own contiguous block of pair indices; NCCL all_gather of result "
                        f"records only"),
        "l2": "inputs (9.8 MB/pair, 40 GB per GPU) exceed the 126 MB L2; no flush needed",
    }


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--pairs", type=int, default=4096,
                   help="pairs per GPU (weak scaling) or in total (--scaling strong)")
    p.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                   help="weak: every GPU aligns its own --pairs independent pairs (the path "
                        "partitions into independent units, SURVEY 8e); strong: --pairs split")
    p.add_argument("--variant", type=int, default=1, help="0 clean, 1 noisy+occluder")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-sample", type=int, default=0, help="pairs in the CPU sample (0 = auto)")
    p.add_argument("--profile-json", default="", help="write per-kernel stats here")
    return p.parse_args()


def partition(pairs, world, rank, scaling="strong"):
    """Contiguous block of pair indices for this rank (no input scatter: each rank
    renders its own).  strong: `pairs` in total; weak: `pairs` per rank."""
    n_local = pairs if scaling == "weak" else pairs // world
    return rank * n_local, n_local


def result_records(results, n_local):
    """Fixed-size per-pair records (pose 12, status, iterations, cov_degenerate) for the gather."""
    import numpy as np
    rec = np.zeros((n_local, 16))
    for i, r in enumerate(results):
        rec[i, :9] = r.T_AB.R[:]
        rec[i, 9:12] = r.T_AB.t[:]
        rec[i, 12] = r.status
        rec[i, 13] = r.total_iterations
        rec[i, 14] = r.cov_degenerate
    return rec


def gather_records(rec, world, out, dist=None):
    """The only collective of the benchmark: all_gather of the result records."""
    import torch
    t = torch.from_numpy(rec).to(out.device)
    if world > 1:
        dist.all_gather_into_tensor(out, t)
    else:
        out.copy_(t)
    return out


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


# --------------------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms",
                 "200", "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- CPU reference


def host_pairs(n, variant, seed0=0):
    """The benchmark's pairs seed0..seed0+n-1 rendered on the host
    (rgbid_synth_pair_host: the same scene model and generator as the device
    rendering of the timed arm, host libm)."""
    from concurrent.futures import ThreadPoolExecutor
    import paper_1807_08271_b200 as rg
    K = rg.simple_intrinsics(W0, H0, F0)

    def one(i):
        fa, fb, _ = rg.synth_pair_host(K, seed0 + i, variant)
        return (fa.intensity, fa.inverse_depth, fb.intensity, fb.inverse_depth)

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        return K, list(ex.map(one, range(n)))


def cpu_reference_rate(pairs, K, cores):
    """oracle/_ref (reference sources compiled in place) when built, else the
    C restatement; independent pairs on `cores` host threads."""
    import paper_1807_08271_b200 as rg
    from oracle import oracle as O
    kind = "reference" if O.available("REF") else "port"
    orc = O.Oracle("REF" if kind == "reference" else "C")
    cfg = rg.AlignmentConfig(levels=LEVELS, iterations=ITERS).to_c()
    t0 = time.perf_counter()
    res = orc.align_many(pairs, K.to_c(), None, cfg, threads=cores)
    dt = time.perf_counter() - t0
    ok = sum(1 for r in res if r.status == 0)
    return len(pairs) / dt, dt, kind, ok


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    n = args.cpu_sample or max(8, cores)
    K, pairs = host_pairs(n, args.variant)
    vals = []
    kind = "reference"
    for step in range(args.warmup + args.steps):
        rate, dt, kind, ok = cpu_reference_rate(pairs, K, cores)
        if step >= args.warmup:
            vals.append((rate, dt))
    rate = statistics.median(v[0] for v in vals)
    ms = statistics.median(v[1] for v in vals) * 1000.0
    sample = (f"the benchmark's first {n} 640x480 pairs "
              f"({'noisy+occluder' if args.variant else 'clean'}), rendered on the host by the "
              f"same generator, per step; 4-level align + covariance on {cores} threads, one "
              f"pair per thread at a time")
    line = {
        "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- our arm


def algorithmic_bytes(results):
    """per alignment B = M[2 + 2*sum_{l>=1} 4^-l + sum_l it_l (3 + 2*4^-l) + 4];
    warp_residuals share: sum_l it_l (3 + 2*4^-l) M (+ the covariance pass 3M + 2M)."""
    tot, warp = 0.0, 0.0
    for r in results:
        if r.status != 0:
            continue
        its = {r.level_log[k].level: r.level_log[k].iterations for k in range(r.n_levels)}
        pyr = 2 + 2 * sum(4.0 ** -l for l in range(1, LEVELS))
        irls = sum(it * (3 + 2 * 4.0 ** -l) for l, it in its.items())
        tot += M_BYTES * (pyr + irls + 4)
        warp += M_BYTES * (irls + 5)
    return tot, warp


# ncu-measured per full-res pixel constants of the warp_residuals family
# (profiles/r01_k1_ncu_v14.txt): fp64 flop = dadd + dmul + 2 dfma per pixel warped
# (level 0 / covariance pass: 112; levels >= 1 add the in-tile downsample: ~122-124),
# and DRAM bytes per slot-iteration at level 0 (read + write / 512 slots).
K1_FLOP_PER_PX = {0: 112.0, 1: 121.4, 2: 123.8, 3: 124.5}
K1_TRAFFIC_L0 = (5.191611e9 + 2.551423e9) / 512


def warp_flops(results):
    """fp64 flops executed by the warp_residuals family: every iteration at every
    level warps all N0 full-res pixels (src/alignment.cpp:378-379), plus the
    covariance pass (level 0 kernel)."""
    tot = 0.0
    for r in results:
        if r.status != 0:
            continue
        for k in range(r.n_levels):
            lv = r.level_log[k]
            tot += lv.iterations * N0 * K1_FLOP_PER_PX.get(lv.level, K1_FLOP_PER_PX[3])
        tot += N0 * K1_FLOP_PER_PX[0]
    return tot


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1807_08271_b200 as rg
    from paper_1807_08271_b200 import abi

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = rg.Context(local)
    K = rg.simple_intrinsics(W0, H0, F0)
    cfg = rg.AlignmentConfig(levels=LEVELS, iterations=ITERS)
    base, n_local = partition(args.pairs, world, rank, args.scaling)

    # inputs resident in HBM: device-rendered pairs (pair seed = global index)
    A = [rg.DeviceFrame(W0, H0, ctx) for _ in range(n_local)]
    B = [rg.DeviceFrame(W0, H0, ctx) for _ in range(n_local)]
    for i in range(n_local):
        rg.synth_pair_device(A[i], B[i], K, base + i, args.variant)
    ctx.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream_ptr)
    gathered = torch.empty((world * n_local, 16), dtype=torch.float64, device="cuda")

    def gather(results):
        gather_records(result_records(results, n_local), world, gathered, dist)
        return results

    def step():
        for f in A:  # fresh inputs each step: pyramids are rebuilt like the reference does
            f.invalidate()
        return gather(rg.align_batch(A, B, K, config=cfg, ctx=ctx))

    for _ in range(args.warmup):
        results = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = ctx.kernel_launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        results = step()
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = ctx.kernel_launches - launches0
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = pairs_total(args, world) * args.steps / (ms_max / 1000.0)
    statuses = {int(r.status) for r in results}
    n_ok = sum(1 for r in results if r.status == 0)
    mean_iters = float(np.mean([r.total_iterations for r in results if r.status == 0] or [0]))

    # profiled step (graph-less, CUDA events around every launch) -> dominant kernel roofline
    ctx.set_profiling(True)
    ctx.reset_stats()
    presults = step()
    ctx.synchronize()
    kstats = ctx.kernel_stats()
    ctx.set_profiling(False)
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(peaks_path):
        peak, peak_src = float(json.load(open(peaks_path))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    tot_bytes, warp_bytes = algorithmic_bytes(presults)
    prof_total = sum(v[1] for v in kstats.values())
    fam = {}
    for k, v in kstats.items():
        f = k.split("_L")[0].replace("_cov", "")
        fam[f] = fam.get(f, 0.0) + v[1]
    dom = max(fam.items(), key=lambda kv: kv[1]) if fam else ("none", 0.0)
    dom = (dom[0], (0, dom[1]))
    warp_ms = sum(v[1] for k, v in kstats.items() if k.startswith("warp_residuals"))
    roofline = {
        "bound": "hbm", "kernel": "warp_residuals",
        "achieved": (warp_bytes / (warp_ms / 1e3)) / 1e9 if warp_ms else None,
        "peak": peak, "unit": "GB/s", "peak_source": peak_src,
        # ncu dram read+write per slot-iteration of the level-0 launch vs SURVEY 8(d)'s
        # algorithmic B_it(0) = 5M: no wasted re-reads
        "traffic": K1_TRAFFIC_L0, "traffic_algorithmic": 5 * M_BYTES,
        "traffic_unit": "bytes per slot-iteration at level 0 (profiles/r01_k1_ncu_v35.txt)",
        "frac": ((warp_bytes / (warp_ms / 1e3)) / 1e9) / peak if warp_ms else None,
        "kernel_share_of_step": warp_ms / prof_total if prof_total else None,
        "dominant_kernel": dom[0], "dominant_share": dom[1][1] / prof_total if prof_total else None,
        "pipeline_achieved_gbs": (tot_bytes / (ms_max / args.steps / 1e3)) / 1e9 * world
        if ms_max else None,
        "algorithmic_bytes_per_alignment": tot_bytes / max(1, sum(1 for r in presults if r.status == 0)),
        "note": "achieved = SURVEY 8(d) algorithmic bytes of the executed IRLS iterations / "
                "summed CUDA-event time of that kernel in a profiled (graph-less) step",
    }
    if args.profile_json and rank == 0:
        json.dump({"kernels": kstats, "bytes": {"total": tot_bytes, "warp": warp_bytes}},
                  open(args.profile_json, "w"), indent=1)

    # measured FP64 FMA peak: denominator of the FP64-issue-bound Student-t kernel
    fp64 = C.c_double(0.0)
    ctx.check(ctx.lib.rgbid_measure_fp64_peak(ctx.h, C.byref(fp64)), "fp64_peak")
    tdist_ms = sum(v[1] for k, v in kstats.items() if k.startswith("tdist"))
    roofline["fp64_peak_tflops_measured"] = fp64.value
    # the warp kernels are fp64-issue- and load-latency-bound rather than HBM-bound
    # (~2.8 TB/s and ~31% fp64 instruction issue per ncu): report both ceilings
    wfl = warp_flops(presults)
    if warp_ms and fp64.value > 0:
        ach = wfl / (warp_ms / 1e3) / 1e12
        roofline["fp64"] = {"kernel": "warp_residuals", "achieved": ach, "peak": fp64.value,
                            "unit": "TFLOP/s", "frac": ach / fp64.value,
                            "flop_per_px": K1_FLOP_PER_PX,
                            "note": "ncu-measured flop per full-res pixel x pixels warped in "
                                    "the profiled step / its CUDA-event time; peak = "
                                    "rgbid_measure_fp64_peak (dependent-free DFMA stream)"}
    roofline["tdist_share_of_step"] = tdist_ms / prof_total if prof_total else None

    # latency: one pair, device-resident, 4 levels; + one keyframe fusion
    lat = {}
    if rank == 0:
        for _ in range(3):
            rg.align(A[0], B[0], K, config=cfg, ctx=ctx)
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rg.align(A[0], B[0], K, config=cfg, ctx=ctx)
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        Cmap = torch.ones((H0, W0), dtype=torch.float64, device="cuda")
        arr = (C.c_void_p * 1)(B[0].h.value)
        P = (abi.Pose_t * 1)(rg.Pose().to_c())
        fs = []
        for k in range(13):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.check(ctx.lib.rgbid_integrate_frames(ctx.h, A[1].h, C.cast(Cmap.data_ptr(), abi.DP),
                                                     1, arr, P, C.byref(K.to_c()), 0.05),
                      "integrate_frames")
            e1.record(stream)
            e1.synchronize()
            if k >= 3:
                fs.append(e0.elapsed_time(e1))
        lat = {"align_ms": statistics.median(ts), "fusion_ms": statistics.median(fs),
               "frame_ms": statistics.median(ts) + statistics.median(fs),
               "what": "one 640x480 4-level align (device-resident pair, incl. covariance) + "
                       "one integrate_frame; CUDA events, median of 10"}

    # end-to-end through the C-ABI with HOST buffers (pinned), copies in the timed region
    e2e = None
    if not args.no_e2e:
        P = min(64, n_local)
        pool = torch.empty((P, 4, H0, W0), dtype=torch.float64, pin_memory=True)
        pn = pool.numpy()
        for i in range(P):
            fa, fb = A[i].download(), B[i].download()
            pn[i, 0], pn[i, 1], pn[i, 2], pn[i, 3] = fa.intensity, fa.inverse_depth, fb.intensity, \
                fb.inverse_depth
        ptrs = [[pn[i % P, k].ctypes.data_as(abi.DP) for i in range(n_local)] for k in range(4)]
        arrs = [(abi.DP * n_local)(*p) for p in ptrs]
        res = [(abi.AlignResult_t * n_local)() for _ in range(2)]
        cfg_c, K_c = cfg.to_c(), K.to_c()

        E2E_CHUNK = int(os.environ.get("RGBID_E2E_CHUNK", "512"))

        def e2e_step(k):
            # streaming form: step k's first uploads overlap step k-1's last chunks;
            # results alternate between two arrays (step k-1's finish during step k)
            ctx.check(ctx.lib.rgbid_align_batch_host_async(ctx.h, n_local, *arrs, W0, H0,
                                                           C.byref(K_c), None, C.byref(cfg_c),
                                                           E2E_CHUNK, res[k % 2]),
                      "align_batch_host_async")

        e2e_step(0)
        ctx.check(ctx.lib.rgbid_align_batch_host_wait(ctx.h), "align_batch_host_wait")
        ctx.reset_stats()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_steps = max(1, min(args.steps, 3))
        for k in range(e2e_steps):
            e2e_step(k)
        ctx.check(ctx.lib.rgbid_align_batch_host_wait(ctx.h), "align_batch_host_wait")
        e1.record(stream)
        torch.cuda.synchronize()
        assert all(r.status in (0, 1) for r in res[(e2e_steps - 1) % 2])
        h2d, d2h = ctx.transfer_bytes()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = {"value": pairs_total(args, world) * e2e_steps / (float(t.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": h2d // e2e_steps, "d2h_bytes_per_step": d2h // e2e_steps,
               "path": "rgbid_align_batch_host_async/_wait (C-ABI) from pinned host buffers, 2 lanes "
                       f"x chunks of {E2E_CHUNK}, consecutive steps streamed; "
                       f"host pool of {P} distinct pairs cycled"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the reference arm's measurement, in a clean process (this one holds a CUDA
        # context, torch threads and pinned pools that slow a host-thread sweep ~1.5x):
        # the benchmark's first n pairs from the same generator, rendered on the host
        cores = os.cpu_count() or 1
        n = args.cpu_sample or max(8, cores)
        env = {k: v for k, v in os.environ.items()
               if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE")}
        pr = subprocess.run([sys.executable, os.path.abspath(__file__), "--impl", "reference",
                             "--steps", "1", "--warmup", "1", "--cpu-sample", str(n),
                             "--variant", str(args.variant)],
                            env=env, capture_output=True, text=True, timeout=900)
        try:
            ref = json.loads(pr.stdout.strip().splitlines()[-1])
            cpu = dict(ref["cpu_baseline"])
            cpu["sample"] += " (bench.py --impl reference in a subprocess)"
        except (IndexError, KeyError, ValueError):
            cpu = {"value": None, "unit": UNIT, "cores": cores, "kind": "reference",
                   "sample": "reference subprocess failed: " + pr.stderr.strip()[-200:]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device-rendered textured slanted plane, SURVEY 8d)",
            "config": workload_config(args, world),
            "clocks": clk, "gpu_launches": launches, "e2e": e2e, "roofline": roofline,
            "cpu_baseline": cpu, "latency": lat,
            "status": {"ok": n_ok, "statuses": sorted(statuses), "mean_iterations": mean_iters},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
