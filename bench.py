#!/usr/bin/env python
"""Benchmark of the hot path: census cost volume + Dual MM (4 iterations) at the
KITTI shape 1242x375x128 (BASELINE.json configs[1]), one frame per GPU per step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step = census x2 + cost volume + `iters` Dual MM iterations (H and V
half-steps) + labelling + primal energy + dual bounds, on synthetic
warped-texture input resident in HBM.  Metric: cost-volume cell-iterations/s
= W*H*K*iters*frames / step time (whole job, all ranks).  One JSON line on rank 0.
Multi-GPU (torchrun): every rank solves its own frame (frame sharding, weak
scaling, no data-path collective); timing is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import datagen  # noqa: E402

# one JSON line on stdout: keep NCCL's banner off stdout unless the caller asks for it
os.environ.setdefault("NCCL_DEBUG", "WARN")

METRIC = "cost-volume cell-iterations/s (1242x375x128, 4 dual iterations)"


def metric_for(c):
    """BASELINE's metric on the config's shape (C2: exactly METRIC)."""
    if c["kind"] == "flow":
        return f"cost-volume cell-iterations/s ({c['W']}x{c['H']}, 2 x {c['K']} flow labels, {c['iters']} dual iterations)"
    return f"cost-volume cell-iterations/s ({c['W']}x{c['H']}x{c['K']}, {c['iters']} dual iterations)"
UNIT = "cell-iter/s"
W_REG, T_REG, FBITS = 3, 4, 4           # pairwise w, truncation T, fixed-point bits (DESIGN R2, R9)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def traffic_per_half_step(config):
    """dram__bytes_read.sum + dram__bytes_write.sum of one chain-DP half-step
    (its root + level + leaf launches, averaged over the H and V half-steps of
    one solve) from the committed ncu capture OF THIS CONFIG
    (profiles/ncu_traffic_<config>.json, written by profiles/summarize_ncu.py
    from the launch-list capture), or None when no capture of this config exists."""
    p = os.path.join(ROOT, "profiles", f"ncu_traffic_{config}.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        if d.get("config") == config:
            return d.get("hm_bytes_per_half_step")
    return None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def kp_of(K):
    """Label pitch of the stored cost volume (capi.cu kp_of: 32 x a power of two >= K)."""
    lpl = 1
    while 32 * lpl < K:
        lpl *= 2
    return 32 * lpl


def alg_bytes_compact(W, H, K, iters, frames=1):
    """SURVEY 8(d) algorithmic bytes of the chain-DP half-steps of one step, on
    the lossless compact basis (u16 label spans + one int32 offset per pixel
    and vector; each input read once, each output written once, messages on
    chip): H_1 = D (1) + f_ (2) B/cell + 4 B/pixel; H_t = D (1) + g_ (2) + f_ (2)
    B/cell + 8 B/pixel; V = f_ (2) + g_ (2) B/cell + 8 B/pixel, + 1 B/pixel of
    labels on the last V.  Cells = W*H*K (the padding to KP is not
    algorithmic; the V pass's D re-read is traffic, not algorithmic bytes)."""
    cells, px = W * H * K, W * H
    h1 = 3 * cells + 4 * px
    ht = 5 * cells + 8 * px
    v = 4 * cells + 8 * px
    return frames * (h1 + (iters - 1) * ht + iters * v + px)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_oracle_sample(left, right, K, iters, nthreads, rows=None):
    """Time the CPU oracle (as it stands) on a bounded sample; returns
    (cell-iter/s, seconds, description)."""
    import oracle
    oracle.build()
    if rows is not None:
        left, right = left[:rows], right[:rows]
    H, W = left.shape
    t0 = time.perf_counter()
    oracle.solve(left, right, 0, K, W_REG, T_REG, FBITS, iters, nthreads=nthreads)
    dt = time.perf_counter() - t0
    desc = (f"oracle (C, OpenMP over chains) census+cost+{iters} DMM iteration(s)+energy on "
            f"{W}x{H}x{K} ({'first %d rows of ' % rows if rows else ''}the step's frame), "
            f"{nthreads} threads")
    return W * H * K * iters / dt, dt, desc


def cpu_oracle_flow_sample(i1, i2, u_min, K, iters, nthreads, rows=None):
    """The flow discrete stage on the CPU oracle: census of both images, the
    decoupled costs, Dual MM on both layers; returns (cell-iter/s, s, desc)."""
    import oracle
    oracle.build()
    if rows is not None:
        i1, i2 = i1[:rows], i2[:rows]
    H, W = i1.shape
    t0 = time.perf_counter()
    f1, f2 = oracle.flow_costs(oracle.census(i1), oracle.census(i2), u_min, K, u_min, K)
    for D in (f1, f2):
        oracle.dmm(D, W_REG, W_REG, T_REG, FBITS, iters, nthreads=nthreads)
    dt = time.perf_counter() - t0
    desc = (f"oracle (C, OpenMP over chains) census+decoupled flow costs+{iters} DMM iterations on both "
            f"{W}x{H}x{K} layers ({'first %d rows of ' % rows if rows else ''}the pair), {nthreads} threads")
    return 2 * W * H * K * iters / dt, dt, desc


def run_reference(args):
    """--impl reference: the CPU oracle timed on the host cores, same config,
    metric and unit; each step runs the whole path (census, cost volume, all
    Dual MM iterations, energy) on the first `rows` rows of the frame, with
    `rows` chosen so the whole --warmup/--steps run takes about two minutes
    (the full frame whenever that fits).  Rank 0 only."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    c = datagen.CONFIGS[args.config]
    W, H, K, iters = c["W"], c["H"], c["K"], c["iters"]
    nth = os.cpu_count() or 1
    if c["kind"] == "flow":
        left, right, _, _ = datagen.flow_pair(W, H, -c["d_min"], seed=0)
        sample = lambda rows: cpu_oracle_flow_sample(left, right, c["d_min"], K, iters, nth, rows)  # noqa: E731
        cells_per_row = 2 * W * K
        what = f"optical flow {W}x{H}, {K}x{K} window decoupled into two {K}-label layers"
    else:
        left, right, _ = datagen.pair(c["kind"], W, H, K, seed=0)
        sample = lambda rows: cpu_oracle_sample(left, right, K, iters, nth, rows)  # noqa: E731
        cells_per_row = W * K
        what = f"stereo {W}x{H}, {K} disparities"
    _, t32, _ = sample(min(32, H))
    budget = 120.0
    rows = int(min(H, max(8, budget / (args.steps + args.warmup) / max(t32 / min(32, H), 1e-6))))
    for _ in range(args.warmup):
        sample(rows)
    times = []
    desc = ""
    for _ in range(args.steps):
        v, dt, desc = sample(rows)
        times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    value = cells_per_row * rows * iters / (ms / 1e3)
    line = {
        "impl": "reference", "metric": metric_for(c), "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {what}, census 5x5, {iters} dual iterations "
                               + ("(reference arm: the whole frame per step)" if rows == H else
                                  f"(reference arm: bounded sample of the first {rows} of {H} rows per step)"),
                   "W": W, "H": H, "K": K, "iters": iters, "sample_rows": rows, "same_config": rows == H},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nth, "kind": "oracle", "sample": desc,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)   # ~0.5 s timed: several nvidia-smi clock samples
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="C2", choices=("C1", "C2", "C3", "C4", "C5"),
                    help="C2 (default): one KITTI frame per GPU per step; C5: configs[4], 64 KITTI frames per "
                         "step sharded over the GPUs, each GPU solving its frames as one batch (throughput mode)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--pen", default=None,
                    help="NEXT-3 general penalty e1,e2,delta,c (units 2^-F, e.g. 8,16,2,80: eps=1/2, delta=2, C=5) "
                         "solved by the general int32 kernels")
    ap.add_argument("--edge-weights", action="store_true", help="NEXT-3 edge-aware pairwise weights")
    ap.add_argument("--minorant", choices=("hierarchical", "iterative"), default="hierarchical",
                    help="NEXT-4: chain minorant (iterative = Alg.4, max_pass 3, gamma 1/4)")
    ap.add_argument("--refine", action="store_true",
                    help="append the continuous refinement (NEXT-2: 5 warps x 40 PDHG iterations, P:497) to every "
                         "step (frames mode, one frame per GPU)")
    ap.add_argument("--mode", choices=("frames", "bands"), default="frames",
                    help="frames: one frame per GPU (weak scaling); bands: one frame sharded in row/column "
                         "bands with an all-to-all between half-steps (strong scaling)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    import paper_1601_06274_b200 as dmm

    world, rank, local = dist_env()
    # DMM_BENCH_SAME_GPU=1: a control-flow dry run of the multi-rank path on a
    # one-GPU box (every rank on cuda:0, gloo for the barrier / max-reduce of
    # the timings; frames mode has no data-path collective).  Never a
    # measurement: the ranks share one GPU.
    same_gpu = os.environ.get("DMM_BENCH_SAME_GPU") == "1" and world > 1
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    c = datagen.CONFIGS[args.config]
    W, H, K, iters = c["W"], c["H"], c["K"], c["iters"]
    if args.mode == "bands":
        return run_bands(args, c, world, rank, local, dev)
    if c["kind"] == "flow":
        return run_flow(args, c, world, rank, local, dev)
    total_frames = c.get("frames", world)          # C2: one frame per rank; C5: 64 frames per step
    nf = (total_frames + world - 1) // world
    distinct = [datagen.pair(c["kind"], W, H, K, seed=rank * nf + s) for s in range(min(nf, 8))]
    left, right = distinct[0][0], distinct[0][1]
    pen = tuple(int(v) for v in args.pen.split(",")) if args.pen else None
    ctx = dmm.Context(width=W, height=H, d_min=0, d_max=K - 1, w=W_REG, T=T_REG, frac_bits=FBITS,
                      max_iters=iters, batch=nf, device=dev, pen=pen, edge_weights=args.edge_weights,
                      minorant=args.minorant)
    Lh = np.stack([distinct[s % len(distinct)][0] for s in range(nf)])
    Rh = np.stack([distinct[s % len(distinct)][1] for s in range(nf)])
    lt = torch.from_numpy(Lh).to(dev)
    rt = torch.from_numpy(Rh).to(dev)
    stream = torch.cuda.current_stream(dev)
    us = [None] * nf

    def step():
        if nf == 1:
            ctx.cost_volume(lt[0], rt[0], stream=stream)
        else:
            ctx.cost_volume_frames(lt, rt, stream=stream)
        ctx.solve(iters, frame=0, nframes=nf, stream=stream)
        if args.refine:
            for f in range(nf):
                us[f] = ctx.refine(frame=f, stream=stream, energy=False)[0]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    # L2 (126 MB) is flushed between timed steps by overwriting a 256 MB buffer
    # outside the timed events; the step's own working set (~1.0 GB) exceeds L2.
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    ctx.set_profiling(False)     # the headline steps run exactly as a user's calls (no per-kernel events)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    launches0 = ctx.launch_count
    for i in range(args.steps):
        flush.fill_(i & 0xff)
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = ctx.launch_count - launches0
    clocks = sampler.stop()
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    e, b, hist = ctx.result()
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # per-kernel-class timings from a separate profiled pass (CUDA events
    # around every half-step on the launching stream, same L2 flush)
    prof_steps = max(1, min(args.steps, 50))
    ctx.read_profile()
    ctx.set_profiling(True)
    for i in range(prof_steps):
        flush.fill_(i & 0xff)
        step()
    torch.cuda.synchronize(dev)
    ctx.set_profiling(False)
    prof = ctx.read_profile()

    cells = W * H * K
    value = world * nf * cells * iters / (ms / 1e3)

    # roofline of the dominant kernel: the chain-DP half-step (root + level +
    # leaf launches, H and V); one "launch" = one half-step.  Achieved =
    # SURVEY 8(d) compact algorithmic bytes / the measured half-step time.
    hbm, peak_kind = peaks()
    ms_h, n_h = prof["hm_h"]
    ms_v, n_v = prof["hm_v"]
    alg_bytes_per_step = alg_bytes_compact(W, H, K, iters, nf)
    hm_ms_per_step = (ms_h + ms_v) / prof_steps
    achieved = alg_bytes_per_step / (hm_ms_per_step / 1e3) / 1e9
    tr = traffic_per_half_step(args.config)
    step_ms_prof = sum(v[0] for v in prof.values()) / prof_steps
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": tr, "kernel": "chain-DP half-step (root+level+leaf kernels), H and V",
                "basis": "SURVEY 8(d) compact: H_1 3, H_t 5, V 4 B/cell + int32 offsets 4/8/8 B/pixel "
                         "+ 1 B/pixel labels; achieved = bytes / CUDA-event half-step time",
                "peak_kind": peak_kind, "half_steps_per_step": 2 * iters * nf,
                "hm_ms_per_step": hm_ms_per_step, "profiled_steps": prof_steps,
                "kernel_family": ctx.kernel_family(),
                "alg_bytes_per_half_step": alg_bytes_per_step / (2 * iters * nf),
                "traffic_source": f"profiles/ncu_traffic_{args.config}.json" if tr else None,
                "share_of_step": hm_ms_per_step / step_ms_prof if step_ms_prof else None,
                "per_class_ms_per_step": {k: v[0] / prof_steps for k, v in prof.items()}}
    # the cost-volume pass (north star: "achieved HBM GB/s ... for the cost-volume
    # and DP passes"): census codes read (2 x 4 B/pixel) + D written (KP B/pixel)
    cv_ms = prof["cost_volume"][0] / prof_steps
    if cv_ms > 0:
        cv_bytes = nf * W * H * (8 + kp_of(K))
        roofline["cost_volume_pass"] = {"ms_per_step": cv_ms, "bytes_per_step": cv_bytes,
                                        "achieved": cv_bytes / (cv_ms / 1e3) / 1e9, "unit": "GB/s",
                                        "frac": cv_bytes / (cv_ms / 1e3) / 1e9 / hbm,
                                        "note": "popcount / byte-packing bound, not HBM (DESIGN.md cost_kernel)"}
    refine = None
    if args.refine:
        rms = prof["refine"][0] / prof_steps
        # per PDHG iteration and pixel (float64): reads u, u0, s1, s2, p_h, p_v, q_h, q_v and writes
        # u+, p_h+, p_v+, q_h+, q_v+ (13 doubles) -- the single-iteration sweep's bytes; the
        # temporally blocked kernel moves them once per 4 iterations, L2-resident
        rbytes = nf * W * H * 8 * 13 * 5 * 40
        refine = {"ms_per_step": rms, "warps": 5, "iters": 40, "achieved_gbs": rbytes / (rms / 1e3) / 1e9,
                  "bound": "fp64 issue (DESIGN.md refinement kernels)",
                  "note": "achieved = one-iteration-sweep bytes / time (exceeds HBM: 4 iterations per launch)"}

    # end to end through the public C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        lh = torch.from_numpy(Lh).pin_memory()
        rh = torch.from_numpy(Rh).pin_memory()
        lab = torch.empty((nf, H, W), dtype=torch.uint8).pin_memory()
        uh = torch.empty((nf, H, W), dtype=torch.float32).pin_memory()

        def host_step():
            if args.refine:      # H2D of the images, the device step, D2H of the refined float32 u
                lt.copy_(lh, non_blocking=True)
                rt.copy_(rh, non_blocking=True)
                step()
                for f in range(nf):
                    uh[f].copy_(us[f], non_blocking=True)
            elif nf == 1:
                ctx.run_host(lh[0], rh[0], iters, labels_out=lab[0], stream=stream)
            else:
                ctx.run_host_frames(lh, rh, iters, labels_out=lab, stream=stream)

        for _ in range(2):
            host_step()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        w0 = time.perf_counter()
        for _ in range(args.steps):
            host_step()
        t1.record(stream)
        torch.cuda.synchronize(dev)
        wall_ms = (time.perf_counter() - w0) * 1e3 / args.steps
        ems = max(t0.elapsed_time(t1) / args.steps, wall_ms)
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": world * nf * cells * iters / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": nf * 2 * W * H,
               "d2h_bytes_per_step": (nf * W * H * 4 if args.refine else
                                      nf * (W * H + 16) if nf > 1 else W * H + 8 + 16 * iters),
               "ms_per_step": ems}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nth = os.cpu_count() or 1
        v, dt, desc = cpu_oracle_sample(left, right, K, iters, nth)
        cpu = {"value": v, "unit": UNIT, "cores": nth, "kind": "oracle", "sample": desc, "seconds": dt,
               "cpu_model": cpu_model()}

    if rank == 0:
        line = {
            "metric": metric_for(c), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": f"{args.config}: stereo {W}x{H}, {K} disparities, census 5x5, "
                                   f"{iters} dual iterations, warped-texture pairs, "
                                   + ("1 frame per GPU" if nf == 1 else
                                      f"{total_frames} frames per step ({nf} per GPU, solved as one batch)"),
                       "W": W, "H": H, "K": K, "iters": iters, "w": W_REG, "T": T_REG, "frac_bits": FBITS,
                       "frames_per_gpu": nf,
                       "pairwise": ("general penalty e1,e2,delta,c=" + args.pen if args.pen else
                                    f"truncated linear w={W_REG}, T={T_REG}")
                                   + (", edge-aware weights" if args.edge_weights else ""),
                       "minorant": args.minorant,
                       "fps": world * nf / (ms / 1e3), "parallelism": f"frames x{world}",
                       "l2": "flushed between timed steps (256 MB write outside events); step working set ~1 GB"},
            "roofline": roofline,
            "refine": refine,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": launches,
            "result": {"energy": e / (1 << FBITS), "bound": b / (1 << FBITS)},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_flow(args, c, world, rank, local, dev):
    """configs[3] (C4), discrete stage of optical flow: census + the fused
    32x32-window decoupled-cost kernel (Eq. flow-decoupled-costs)
    + Dual MM on both K=32 layers (two frames of one context, same launches).
    One frame pair per GPU (weak scaling).  cells = W*H*(K1 + K2)."""
    import torch
    import torch.distributed as dist

    import paper_1601_06274_b200 as dmm
    W, H, K, iters, u_min = c["W"], c["H"], c["K"], c["iters"], c["d_min"]
    i1, i2, _, _ = datagen.flow_pair(W, H, -u_min, seed=rank)
    ctx = dmm.Context(width=W, height=H, d_min=u_min, d_max=u_min + K - 1, w=W_REG, T=T_REG, frac_bits=FBITS,
                      max_iters=iters, batch=2, device=dev)
    stream = torch.cuda.current_stream(dev)
    t1, t2 = torch.from_numpy(i1).to(dev), torch.from_numpy(i2).to(dev)

    out = {}

    def step():
        ctx.flow_cost_volume(t1, t2, u_min, stream=stream)
        ctx.solve(iters, frame=0, nframes=2, stream=stream)
        if args.refine:
            out["u"] = ctx.flow_refine(u_min, C=float(T_REG), stream=stream, energy=False)[:2]

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    launches0 = ctx.launch_count
    for i in range(args.steps):
        flush.fill_(i & 0xff)
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = ctx.launch_count - launches0
    clocks = sampler.stop()
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    prof_steps = max(1, min(args.steps, 50))
    ctx.read_profile()
    ctx.set_profiling(True)
    for i in range(prof_steps):
        flush.fill_(i & 0xff)
        step()
    torch.cuda.synchronize(dev)
    ctx.set_profiling(False)
    prof = ctx.read_profile()
    cells = W * H * 2 * K
    value = world * cells * iters / (ms / 1e3)
    hbm, peak_kind = peaks()
    hm_ms = (prof["hm_h"][0] + prof["hm_v"][0]) / prof_steps
    alg = alg_bytes_compact(W, H, K, iters, 2)
    flow_ms = prof["cost_volume"][0] / prof_steps
    roofline = {"bound": "hbm", "achieved": alg / (hm_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                "frac": alg / (hm_ms / 1e3) / 1e9 / hbm, "traffic": traffic_per_half_step("C4"),
                "kernel": "chain-DP half-step (root+level+leaf kernels), H and V, both flow layers",
                "basis": "SURVEY 8(d) compact bytes of the two K=32 layers",
                "peak_kind": peak_kind, "hm_ms_per_step": hm_ms, "profiled_steps": prof_steps,
                "flow_cost_kernel": {"ms": flow_ms, "hamming_per_s": W * H * K * K / (flow_ms / 1e3),
                                     "out_bytes_gbs": 2 * W * H * ctx.cost_volume_tensor(0).shape[2] /
                                     (flow_ms / 1e3) / 1e9},
                "per_class_ms_per_step": {k: v[0] / prof_steps for k, v in prof.items()}}
    refine = None
    if args.refine:
        rms = prof["refine"][0] / prof_steps
        # per PDHG iteration, pixel and component: the stereo iteration's 13 doubles
        rbytes = 2 * W * H * 8 * 13 * 5 * 40
        refine = {"ms_per_step": rms, "warps": 5, "iters": 40, "achieved_gbs": rbytes / (rms / 1e3) / 1e9,
                  "note": "flow refinement (Eq. 19-20), both components; state L2-resident; achieved is "
                          "algorithmic bytes / time"}
    # end to end through the public API with host buffers: H2D of both images,
    # flow costs, both layers' Dual MM (+ refinement), D2H of both labellings
    # (or of the refined float32 flow)
    h1 = torch.from_numpy(i1).pin_memory()
    h2 = torch.from_numpy(i2).pin_memory()
    lab = torch.empty((2, H, W), dtype=torch.float32 if args.refine else torch.uint8).pin_memory()

    def host_step():
        t1.copy_(h1, non_blocking=True)
        t2.copy_(h2, non_blocking=True)
        step()
        if args.refine:
            lab[0].copy_(out["u"][0], non_blocking=True)
            lab[1].copy_(out["u"][1], non_blocking=True)
        else:
            lab[0].copy_(ctx.labels(0, stream=stream), non_blocking=True)
            lab[1].copy_(ctx.labels(1, stream=stream), non_blocking=True)

    for _ in range(2):
        host_step()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    w0 = time.perf_counter()
    for _ in range(args.steps):
        host_step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ems = max(e0.elapsed_time(e1) / args.steps, (time.perf_counter() - w0) * 1e3 / args.steps)
    res = [ctx.result(f) for f in (0, 1)]
    if rank == 0:
        line = {
            "metric": metric_for(c), "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic",
            "config": {"workload": f"C4: optical flow {W}x{H}, {K}x{K} label window (u in [{u_min}, {u_min + K - 1}]^2), "
                                   f"decoupled into two {K}-label layers, {iters} dual iterations each"
                                   + (", continuous refinement 5 x 40" if args.refine else "") + ", 1 pair per GPU",
                       "W": W, "H": H, "K": K, "iters": iters, "fps": world / (ms / 1e3),
                       "parallelism": f"frames x{world}",
                       "l2": "flushed between timed steps (256 MB write outside events)"},
            "roofline": roofline, "refine": refine, "cpu_baseline": None,
            "e2e": {"value": world * cells * iters / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": 2 * W * H,
                    "d2h_bytes_per_step": 2 * W * H * lab.element_size(), "ms_per_step": ems},
            "clocks": clocks, "gpu_launches": launches,
            "result": {"energy": [r[0] / (1 << FBITS) for r in res], "bound": [r[1] / (1 << FBITS) for r in res]},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_bands(args, c, world, rank, local, dev):
    """One frame sharded in row bands (H) / column bands (V) over all ranks
    (SURVEY 8(e)): dmm_shard(ROWCOL) -- the library's own NCCL communicator
    does the all-to-all transposes between half-steps, the bound / energy
    all-reduce and the labelling all-gather.  Strong scaling."""
    import torch
    import torch.distributed as dist

    import paper_1601_06274_b200 as dmm
    from paper_1601_06274_b200 import sharding
    W, H, K, iters = c["W"], c["H"], c["K"], c["iters"]
    left, right, _ = datagen.pair(c["kind"], W, H, K, seed=0)       # the same frame on every rank
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29561")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    ctx = dmm.Context(width=W, height=H, d_min=0, d_max=K - 1, w=W_REG, T=T_REG, frac_bits=FBITS,
                      max_iters=iters, device=dev, shard_world=world)
    sharding.rowcol_setup(ctx)
    stream = torch.cuda.current_stream(dev)
    lt = torch.from_numpy(left).to(dev)
    rt = torch.from_numpy(right).to(dev)

    def step():
        ctx.cost_volume(lt, rt, stream=stream)
        ctx.solve(iters, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    dist.barrier()
    torch.cuda.synchronize(dev)
    launches0 = ctx.launch_count
    for i in range(args.steps):
        flush.fill_(i & 0xff)
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize(dev)
    dist.barrier()
    launches = ctx.launch_count - launches0
    clocks = sampler.stop()
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    energy, bound, hist = ctx.result()

    # profiled pass: this rank's half-step kernels (its row band for H, its
    # column band for V) -> roofline on the compact algorithmic bytes of its bands
    prof_steps = max(1, min(args.steps, 20))
    ctx.read_profile()
    ctx.set_profiling(True)
    for i in range(prof_steps):
        flush.fill_(i & 0xff)
        step()
    torch.cuda.synchronize(dev)
    ctx.set_profiling(False)
    prof = ctx.read_profile()
    r0, r1 = sharding.bands(H, world)[rank]
    c0, c1 = sharding.bands(W, world)[rank]
    hr, wc = r1 - r0, c1 - c0
    cells_h, cells_v, px_h, px_v = hr * W * K, H * wc * K, hr * W, H * wc
    alg = (3 * cells_h + 4 * px_h) + (iters - 1) * (5 * cells_h + 8 * px_h) + iters * (4 * cells_v + 8 * px_v) + px_v
    hm_ms = (prof["hm_h"][0] + prof["hm_v"][0]) / prof_steps
    hbm, peak_kind = peaks()
    achieved = alg / (hm_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": None, "kernel": "chain-DP half-step (root+level+leaf kernels), H and V, rank 0's bands",
                "basis": "SURVEY 8(d) compact bytes of this rank's row band (H) and column band (V)",
                "peak_kind": peak_kind, "hm_ms_per_step": hm_ms, "profiled_steps": prof_steps,
                "per_class_ms_per_step": {k: v[0] / prof_steps for k, v in prof.items()}}
    # expected NVLink bytes per half-step: every rank sends (world-1)/world of its band's records
    rec = 2 * (32 * (1 << max(0, (K - 1).bit_length() - 5))) + 16
    xfer = (hr * W - hr * wc) * rec

    # end to end with host buffers through the sharded context
    lh = torch.from_numpy(left).pin_memory()
    rh = torch.from_numpy(right).pin_memory()
    lab = torch.empty((H, W), dtype=torch.uint8).pin_memory()
    for _ in range(2):
        ctx.run_host(lh, rh, iters, labels_out=lab, stream=stream)
    torch.cuda.synchronize(dev)
    dist.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    w0 = time.perf_counter()
    for _ in range(args.steps):
        ctx.run_host(lh, rh, iters, labels_out=lab, stream=stream)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    ems = max(t0.elapsed_time(t1) / args.steps, (time.perf_counter() - w0) * 1e3 / args.steps)
    t = torch.tensor([ems], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ems = float(t.item())
    if rank == 0:
        cells = W * H * K
        line = {
            "metric": metric_for(c), "value": cells * iters / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": f"{args.config}: one {W}x{H}x{K} frame sharded in {world} row/column bands, "
                                   f"{iters} dual iterations, NCCL all-to-all transposes between half-steps "
                                   f"(dmm_shard ROWCOL)",
                       "W": W, "H": H, "K": K, "iters": iters, "fps": 1e3 / ms, "parallelism": f"bands x{world}",
                       "nvlink_bytes_per_half_step_per_rank": xfer,
                       "l2": "flushed between timed steps (256 MB write outside events)"},
            "roofline": roofline, "cpu_baseline": None,
            "e2e": {"value": cells * iters / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": 2 * W * H,
                    "d2h_bytes_per_step": W * H + 8 + 8, "ms_per_step": ems},
            "clocks": clocks, "gpu_launches": launches,
            "result": {"energy": energy / (1 << FBITS), "bound": bound / (1 << FBITS)},
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
