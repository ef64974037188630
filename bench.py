#!/usr/bin/env python3
"""bench.py -- FMM target evaluations per second on B200 (BASELINE.json metric).

A step = one pass of the whole hot path (fmm_build_tree + fmm_evaluate: keying,
radix sort, lists, P2M, M2M, M2L/L2L, L2P+P2P) over each tiling of the workload.
Default workload: config C4 of BASELINE.json (the 16.8M-point tiling comparison:
quadtree L9, septree L6, triangle-quadtree L9, N = M = 16,777,216 self-mode
points, p = 24, seed 3) -- the configuration the metric is quoted on.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4|C3|C5|C1|C2]
  python bench.py --impl reference ...     (the CPU oracle, bounded sample)

Multi-GPU (one process per GPU; `--gpus N` without a launcher starts N ranks
itself): every rank gets the full input (replicated), keys every point, takes a
work-balanced contiguous range of leaves, sorts only its own + halo leaves, runs
P2M / M2M over its own leaves and sums the multipole tree over the ranks with one
ncclAllReduce on the library's communicator (overlapped with the P2P pair
kernel), then evaluates its own targets; time = max over ranks;
value = all targets / time (strong scaling: the 16.8M-point problem is fixed).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import fmm_inputs as fi  # noqa: E402

METRIC = "FMM target evals/sec (FP64, 16M pts) at 1/2/4/8 B200; P2P/M2L % FP64 peak"
WORKLOADS = {
    "C4": ["C4q", "C4s", "C4t"],
    "C3": ["C3"],
    "C5": ["C5"],
    "C1": ["C1"],
    "C2": ["C2"],
    "C4q": ["C4q"],
    "C4s": ["C4s"],
    "C4t": ["C4t"],
}
# FP64 peak derived from the unit counts and clocks of the guides:
# 148 SMs x 64 FP64 FMA/clk/SM x 2 flop x 1.965 GHz
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
# SURVEY §8(d) algorithmic work per unit:
#  * P2P: F_pair FP64 flops per near-field interaction (ordered target-source pair), measured by
#    ncu on the one-pair-per-thread microbenchmark tools/fpair_micro.py: 39 flops of math
#    (|z|^2, log|z|^2, Arg z) + 2 DADD (y - x) + 2 DFMA (strength products) = 45
#    (profiles/r02/fp64_counts.json, re-measured after every change of the pair math: 50 in
#    round 1; the 1024-entry log table and the k/256 atan knots each removed a DFMA).  The symmetric self-mode kernel evaluates each unordered
#    pair once, so it executes fewer flops than this per interaction (reported beside it).
#  * M2L: the dense-operator count 8 (p+1)^2 flops per M2L op.
F_PAIR = 45.0
# FP64 flops k_p2p_pairs executes per interaction (ncu, sm__sass_thread_inst_executed_op_
# {dfma,dadd,dmul}_pred_on; profiles/r02/fp64_counts.json), for the executed-rate line
F_EXEC = {"C4q": 27.01, "C4s": 25.14, "C4t": 26.79, "C3": 44.48, "C5": 23.91}
# dram__bytes_read.sum + dram__bytes_write.sum of one k_p2p_pairs launch (ncu, profiles/r02/
# launch_dram_table_<cfg>_r02h.txt); C4 = mean over its three launches.  The self-mode writes are
# the per-(target, near slot) partial sums (m x nslot x 16 B, less the paired tasks' unwritten
# slots) that k_p2p_finish adds, the reads mostly the fills of their half-written 32-byte
# sectors; distinct targets (C3) write one slot per target.
P2P_DRAM_BYTES_PER_LAUNCH = {"C4q": 3.837e9, "C4s": 2.378e9, "C4t": 5.584e9, "C4": 3.933e9, "C3": 0.228e9,
                             "C5": 3.176e9}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- clocks sampler
class Clocks:
    def __init__(self):
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([s.strip() for s in line.split(",")])

    def stop(self, dev_index=0):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.samples if len(r) >= 8 and r[0] == str(dev_index)]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[4 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- inputs
def make_inputs(names):
    out = {}
    for nm in names:
        w = fi.get(nm)
        t0 = time.time()
        out[nm] = (w, fi.generate(w))
        log(f"[bench] generated {nm} ({w.note}) in {time.time() - t0:.1f}s")
    return out


def counters_for(tree):
    from paper_1204_3105_b200 import X

    return tree.export(X.COUNTERS)


# ---------------------------------------------------------------- GPU arm
def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_1204_3105_b200 as fmm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    comm = None
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # the library's own NCCL communicator (the multipole all-reduce inside fmm_evaluate):
        # rank 0's unique id reaches every rank through a torch.distributed broadcast
        uid = torch.zeros(fmm.native.COMM_ID_BYTES, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(fmm.Comm.unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        comm = fmm.Comm(bytes(uid.cpu().numpy().tobytes()), world, rank)
        log(f"[bench] rank {rank}/{world}: NCCL {fmm.nccl_version()} communicator ready")
    dev = torch.device("cuda", local)
    names = WORKLOADS[args.workload]
    inputs = make_inputs(names)
    stream = torch.cuda.current_stream(dev)

    def cfg_of(w, timing=False):
        return fmm.Config.make(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, w.self_mode,
                               rank=rank, nranks=world, timing=timing, comm=comm)

    # device-resident inputs and outputs
    dev_in, host_in, outs, host_out = {}, {}, {}, {}
    for nm, (w, d) in inputs.items():
        dev_in[nm] = (torch.from_numpy(d["src_xy"]).to(dev), torch.from_numpy(d["u"]).to(dev),
                      None if d["tgt_xy"] is None else torch.from_numpy(d["tgt_xy"]).to(dev))
        host_in[nm] = tuple(None if a is None else torch.from_numpy(a).pin_memory()
                            for a in (d["src_xy"], d["u"], d["tgt_xy"]))
        outs[nm] = torch.zeros(w.m, dtype=torch.complex128, device=dev)
        host_out[nm] = [torch.zeros(w.m, dtype=torch.complex128).pin_memory() for _ in range(2)]

    # e2e leg (the headline's end-to-end number): the same steps through the C ABI with pinned
    # HOST buffers, serial on the one timed stream like the device-resident value: every step
    # copies its inputs host -> device inside fmm_build_tree and Phi device -> host inside
    # fmm_evaluate.  The optional pipelined variant (--e2e-pipelined) alternates two streams
    # per tiling so that copies overlap kernels of other steps; it is reported separately.
    side = [{nm: torch.cuda.Stream(dev) for nm in names} for _ in range(2)]

    def one_step(timing=False, host=False, pipelined=False, fork=True, join=True, parity=0, kept=None):
        """one build + evaluate per tiling; every tree releases its device memory stream-ordered
        at the end of its own evaluation, so one tree's memory is live at a time (one stream).
        pipelined: one stream per tiling, forked from the timed stream at the step's start and
        joined at its end (when fork / join)."""
        launches = 0
        streams = side[parity] if pipelined else {nm: stream for nm in names}
        for nm in names:
            if fork and streams[nm] is not stream:
                streams[nm].wait_stream(stream)
        for nm, (w, d) in inputs.items():
            src, u, tgt = host_in[nm] if host else dev_in[nm]
            st = streams[nm]
            t = fmm.Tree(cfg_of(w, timing), src, u, tgt, stream=st)
            t.evaluate(host_out[nm][parity] if host else outs[nm], stream=st)
            launches += t.launch_count()
            if kept is not None:
                t.release()  # stream-ordered; the handle keeps its stage events
                kept.append((nm, t))
            else:
                t.close()
        for nm in names:
            if join and streams[nm] is not stream:
                stream.wait_stream(streams[nm])
        return launches

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # warm-up, then one checked tree per tiling (device status, counters, slab size)
    for i in range(args.warmup):
        one_step()
    barrier()
    counters, tree_bytes = {}, {}
    for nm, (w, d) in inputs.items():
        src, u, tgt = dev_in[nm]
        t = fmm.Tree(cfg_of(w), src, u, tgt, stream=stream)
        t.evaluate(outs[nm], stream=stream)
        t.check()
        counters[nm] = counters_for(t)
        tree_bytes[nm] = t.nbytes()
        t.close()
    # trees are released stream-ordered as each finishes, so one tree (plus its build scratch)
    # is live at a time whatever --steps is: grow the pool once to that size, so that no timed
    # step pays for first-touch allocation (the warm-up steps have usually done so already)
    torch.cuda.synchronize(dev)
    fmm.native.pool_reserve(int(1.5 * max(tree_bytes.values())) + (1 << 30))

    # ---- timed region: device-resident inputs, one stream
    clocks = Clocks()
    clocks.start()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    e0.record(stream)
    launches = 0
    kept = []  # released handles: their stage events are read after the timed region
    for s_ in range(args.steps):
        step_ev[s_].record(stream)
        launches += one_step(timing=True, kept=kept)
    step_ev[args.steps].record(stream)
    e1.record(stream)
    barrier()
    clk = clocks.stop(local)
    ms_total = e0.elapsed_time(e1)
    step_ms = [step_ev[i].elapsed_time(step_ev[i + 1]) for i in range(args.steps)]
    log(f"[bench] per-step ms: {[round(x, 2) for x in step_ms]}")
    build_ms, pair_ms, up_ms, down_ms, p2p_ms = ({nm: 0.0 for nm in names} for _ in range(5))
    for nm, t in kept:
        ms = t.stage_times()
        build_ms[nm] += ms[0] + ms[1]
        pair_ms[nm] += ms[2]
        up_ms[nm] += ms[3]
        down_ms[nm] += ms[4]
        p2p_ms[nm] += ms[5]
        t.close()
    kept.clear()
    ms_t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    total_targets = sum(inputs[nm][0].m for nm in names) * args.steps

    # ---- e2e: same metric through the C ABI with pinned host buffers (H2D + D2H inside)
    def e2e_run(mode):
        """serial: one stream; step: one stream per tiling forked and joined every step, so one
        tiling's copies overlap another tiling's kernels inside the step; cross: the streams
        alternate by step and join only at the end (copies also overlap the previous step)"""
        for _ in range(max(2, min(args.warmup, 3))):  # warm-up: every stream's pool blocks and pinned pages
            one_step(host=True, pipelined=mode != "serial")
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        marks = []
        f0.record(stream)
        for s_ in range(args.steps):
            if mode == "cross":  # a tiling's next copy waits only for its own previous step
                one_step(host=True, pipelined=True, fork=(s_ < 2), join=(s_ >= args.steps - 2), parity=s_ % 2)
            else:
                one_step(host=True, pipelined=mode == "step")
            if mode != "cross":  # per-step marks (diagnostic only: the reported time is f0 -> f1)
                marks.append(torch.cuda.Event(enable_timing=True))
                marks[-1].record(stream)
        f1.record(stream)
        barrier()
        if marks and rank == 0:
            prev, per = f0, []
            for m_ in marks:
                per.append(round(prev.elapsed_time(m_), 2))
                prev = m_
            log(f"[bench] e2e per-step ms ({mode}): {per}")
        t_ = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        return float(t_.item())

    e2e_mode = "step" if len(names) > 1 else "serial"
    e2e_ms = e2e_run(e2e_mode)
    e2e_pipe_ms = e2e_run("cross") if args.e2e_pipelined else None
    h2d = sum(w.n * 24 + (0 if w.self_mode else w.m * 16) for w, _ in inputs.values())
    d2h = sum(w.m * 16 for w, _ in inputs.values())

    if rank != 0:
        if world > 1:
            dist.barrier()
            comm.close()
            dist.destroy_process_group()
        return None

    # ---- roofline of the dominant kernel k_p2p_pairs (the near-field pair kernel), timed with
    # CUDA events on its stream around each launch inside the timed region: algorithmic flops =
    # near-field interactions x F_PAIR; the executed FP64 rate (ncu counts per
    # interaction x interactions / the same time) is reported beside it
    pairs = {nm: int(counters[nm][1]) for nm in names}
    pair_ms_avg = sum(pair_ms.values()) / args.steps
    flops = sum(pairs[nm] for nm in names) * F_PAIR
    ach = flops / (pair_ms_avg / 1e3) / 1e12 if pair_ms_avg > 0 else 0.0
    exec_fl = sum(pairs[nm] * F_EXEC[nm] for nm in names) if all(nm in F_EXEC for nm in names) else None
    roof = {"kernel": "k_p2p_pairs (P2P near field; L2P + final sum in k_p2p_finish)", "bound": "alu",
            "achieved": round(ach, 3), "peak": round(FP64_PEAK_TFLOPS, 2), "unit": "TFLOP/s",
            "frac": round(ach / FP64_PEAK_TFLOPS, 4), "traffic": P2P_DRAM_BYTES_PER_LAUNCH.get(args.workload),
            "peak_source": "FP64 FMA: 148 SM x 64 /clk x 2 x 1.965 GHz (DESIGN.md §7); DFMA microbenchmark "
                           "34.2 TF/s (profiles/r01/fp64_peak.log)",
            "f_pair_flops": F_PAIR,
            "interactions_per_s": sum(pairs.values()) / (pair_ms_avg / 1e3) if pair_ms_avg > 0 else 0.0,
            "executed_tflops": None if exec_fl is None or pair_ms_avg <= 0 else round(exec_fl / (pair_ms_avg / 1e3) / 1e12, 3),
            "kernel_ms_per_step": round(pair_ms_avg, 3)}
    # M2L (+ L2L) on the FP64 tensor cores: the downward stage time against 8 (p+1)^2 per op
    m2l_fl = sum(int(counters[nm][0]) * 8 * (inputs[nm][0].p + 1) ** 2 for nm in names)
    down_avg = sum(down_ms.values()) / args.steps
    m2l_ach = m2l_fl / (down_avg / 1e3) / 1e12 if down_avg > 0 else 0.0
    roof_m2l = {"kernel": "k_down_mma (M2L on DMMA m8n8k4 + L2L), all levels", "bound": "alu",
                "achieved": round(m2l_ach, 3), "peak": round(FP64_PEAK_TFLOPS, 2), "unit": "TFLOP/s",
                "frac": round(m2l_ach / FP64_PEAK_TFLOPS, 4), "flops_per_op": "8 (p+1)^2",
                "stage_ms_per_step": round(down_avg, 3)}

    per_tiling = {nm: {"build_ms": build_ms[nm] / args.steps, "upward_ms": up_ms[nm] / args.steps,
                       "downward_ms": down_ms[nm] / args.steps, "p2p_pairs_kernel_ms": pair_ms[nm] / args.steps,
                       "p2p_stage_ms": p2p_ms[nm] / args.steps, "p2p_interactions": pairs[nm],
                       "m2l_ops": int(counters[nm][0])} for nm in names}
    value = total_targets / (ms_max / 1e3)
    res = {
        "metric": METRIC, "value": value, "unit": "target evals/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic, seeded numpy PCG64 (fmm_inputs), shapes of BASELINE.json configs",
        "config": {"workload": args.workload + ": " + "; ".join(inputs[nm][0].note for nm in names),
                   "tilings": names, "step": "fmm_build_tree + fmm_evaluate per tiling",
                   "streams": "timed region: one stream, steps serial",
                   "memory": "each tree is released stream-ordered after its evaluation (one tree live at a time)",
                   "l2": "inputs larger than L2 (>= 400 MB per tiling)", "per_tiling": per_tiling},
        "roofline": roof,
        "roofline_m2l": roof_m2l,
        "e2e": {"value": total_targets / (e2e_ms / 1e3), "unit": "target evals/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / args.steps,
                "how": "every step: fmm_build_tree from pinned host inputs + fmm_evaluate into a pinned host "
                       "output per tiling (H2D / D2H copies inside the timed region), "
                       + ("one CUDA stream per tiling, forked from the timed stream at the start of each step "
                          "and joined at its end: one tiling's copies overlap another tiling's kernels inside "
                          "the step, nothing overlaps across steps" if e2e_mode == "step" else
                          "serial on the timed stream")},
        "gpu_launches": launches,
        "clocks": clk,
    }
    if e2e_pipe_ms is not None:
        res["e2e_pipelined"] = {"value": total_targets / (e2e_pipe_ms / 1e3), "unit": "target evals/s",
                                "how": "two CUDA streams per tiling alternating by step, joined only at the end: "
                                       "a step's copies also overlap the previous step's kernels"}
    if not args.no_cpu_baseline and world == 1:
        res["cpu_baseline"] = cpu_baseline(args, names, sample_targets=args.cpu_sample)
    if world > 1:
        dist.barrier()
        comm.close()
        dist.destroy_process_group()
    return res


# ---------------------------------------------------------------- oracle (CPU) arm
def oracle_time(w, d, sample_targets, seed=0):
    """Oracle as it stands on a bounded sample of the workload: full keying, sort and
    upward pass over all points, downward + L2P + P2P for `sample_targets` random
    targets; extrapolated to all M targets (per-target work is independent)."""
    import oracle

    cfg = oracle.config(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, w.self_mode)
    t0 = time.perf_counter()
    T = oracle.Tree(cfg, d["src_xy"], d["u"], d["tgt_xy"])
    T.upward()
    t1 = time.perf_counter()
    rng = np.random.default_rng(seed)
    ids = np.sort(rng.choice(w.m, size=min(sample_targets, w.m), replace=False))
    T.evaluate(ids)
    t2 = time.perf_counter()
    est = (t1 - t0) + (t2 - t1) * (w.m / len(ids))
    return est, t2 - t0, len(ids)


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(args, names, sample_targets):
    """the oracle as it stands on the box's host cores: at all cores (the reported value) and
    at one thread, each on a bounded sample (oracle_time)"""
    import oracle

    inputs = {nm: (fi.get(nm), fi.generate(fi.get(nm))) for nm in names}
    total = sum(w.m for w, _ in inputs.values())
    res = {}
    for label, threads, samp in (("all", os.cpu_count() or 1, sample_targets), ("one", 1, max(64, sample_targets // 4))):
        oracle.set_num_threads(threads)
        est, spent = 0.0, 0.0
        for nm, (w, d) in inputs.items():
            e, s_, _ = oracle_time(w, d, samp)
            est += e
            spent += s_
        res[label] = (total / est, oracle.num_threads(), samp, spent)
    oracle.set_num_threads(os.cpu_count() or 1)
    v, cores, samp, spent = res["all"]
    v1, _, samp1, spent1 = res["one"]
    return {"value": v, "unit": "target evals/s", "cores": cores, "kind": "oracle",
            "sample": f"full keying+sort+upward pass on every point of {', '.join(names)}, downward+L2P+P2P "
                      f"for {samp} random targets per tiling, extrapolated to all targets; "
                      f"{spent:.1f} s of CPU wall time",
            "extrapolated": True,
            "single_thread": {"value": v1, "unit": "target evals/s", "cores": 1,
                              "sample": f"same, {samp1} targets per tiling; {spent1:.1f} s of CPU wall time"},
            "cpu_model": cpu_model(), "nproc": os.cpu_count()}


def run_reference(args):
    """the tier's reference arm: the CPU oracle as it stands on the box's host cores.  A step
    is the bounded sample of oracle_time per tiling (full build + upward pass, downward + L2P
    + P2P for --cpu-sample targets); `ms_per_step` is the measured wall time of that sampled
    step, `value` the throughput extrapolated to every target (`extrapolated`: true)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import oracle

    oracle.set_num_threads(os.cpu_count() or 1)
    names = WORKLOADS[args.workload]
    inputs = {nm: (fi.get(nm), fi.generate(fi.get(nm))) for nm in names}
    # the oracle has no warm state worth discarding (no JIT, no caches across trees): warm-up
    # steps are skipped
    ests, walls = [], []
    for s in range(args.steps):
        est, wall = 0.0, 0.0
        for nm, (w, d) in inputs.items():
            e, sp, _ = oracle_time(w, d, args.cpu_sample, seed=s)
            est += e
            wall += sp
        ests.append(est)
        walls.append(wall)
    total = sum(w.m for w, _ in inputs.values())
    ms_extrap = 1e3 * sum(ests) / len(ests)
    value = total / (ms_extrap / 1e3)
    cores = oracle.num_threads()
    sample = (f"per step: full keying+sort+upward pass over every point, downward+L2P+P2P for {args.cpu_sample} "
              f"random targets per tiling ({args.cpu_sample * len(names)} targets per step); value extrapolated "
              f"to all {total} targets; {sum(walls):.1f} s CPU wall time total")
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "target evals/s",
            "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(walls) / len(walls), "ms_per_step_extrapolated": ms_extrap,
            "extrapolated": True, "sample_targets_per_step": args.cpu_sample * len(names),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic, seeded numpy PCG64 (fmm_inputs)",
            "config": {"workload": args.workload + ": " + "; ".join(inputs[nm][0].note for nm in names),
                       "tilings": names},
            "cpu_baseline": {"value": value, "unit": "target evals/s", "cores": cores, "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "target evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-pipelined", action="store_true",
                    help="also report e2e with two streams per tiling (copies overlap other steps' kernels)")
    ap.add_argument("--cpu-sample", type=int, default=2048)
    args = ap.parse_args()
    world = os.environ.get("WORLD_SIZE")
    if args.impl == "b200" and args.gpus > 1 and world is None:
        # --gpus N without a launcher: start N ranks (one process per GPU) on this node
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if args.impl == "b200" and world is not None and int(world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    res = run_reference(args) if args.impl == "reference" else run_gpu(args)
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
