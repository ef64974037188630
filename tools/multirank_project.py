"""Per-rank stage times of the multi-GPU path, measured on ONE GPU with the ranks run one after
another (no rank waits on another; the multipole all-reduce is played by a torch sum between
fmm_evaluate_begin and fmm_evaluate_end, outside the timed stages).  For each rank count R and
each tiling of the workload it records, per rank, the library's stage times (build: keys +
global counts + partition + local sort, lists + tasks; upward over own leaves; P2P pairs;
downward; near sums + L2P) and splits the build into its replicated part (work every rank
does on all points) and its partitioned part.

The projected R-GPU step is max over ranks of the sum over tilings of a rank's stage times,
plus the part of the all-reduce that the pair kernel does not hide (bytes / assumed NCCL
bus bandwidth, stated in the output).  This is a projection from single-GPU measurements, not
a multi-GPU measurement (the driver's SCALE run is that).

  python tools/multirank_project.py [--workload C4] [--ranks 1,2,4,8] [--reps 3] > out.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import fmm_inputs as fi  # noqa: E402

WORKLOADS = {"C4": ["C4q", "C4s", "C4t"], "C5": ["C5"], "C3": ["C3"], "C2": ["C2"], "C4q": ["C4q"], "C4s": ["C4s"],
             "C4t": ["C4t"]}


def dev_view(ptr, nbytes):
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": (nbytes // 8,), "typestr": "<f8", "data": (ptr, False), "version": 3}

    return torch.as_tensor(_Arr(), device="cuda")


def run_tiling(fmm, w, tensors, R):
    """one sequential pass of ranks 0..R-1; returns per-rank stage times (ms)"""
    import torch

    src, u, tgt, out = tensors
    stream = torch.cuda.current_stream()
    trees, evs = [], []
    for r in range(R):
        cfg = fmm.Config.make(w.tiling, w.depth, w.p, w.root_x, w.root_y, w.root_size, w.self_mode, rank=r,
                              nranks=R, timing=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t = fmm.Tree(cfg, src, u, tgt, stream=stream)
        t.evaluate_begin(stream=stream)
        e1.record(stream)
        trees.append(t)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    if R > 1:
        ptr0, nb = trees[0].multipole_buffer()
        total = torch.zeros(nb // 8, dtype=torch.float64, device="cuda")
        views = [dev_view(t.multipole_buffer()[0], nb) for t in trees]
        for v in views:
            total += v
        for v in views:
            v.copy_(total)
        torch.cuda.synchronize()
    ends = []
    for t in trees:
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        t.evaluate_end(out, stream=stream)
        f1.record(stream)
        ends.append((f0, f1))
    torch.cuda.synchronize()
    rows = []
    for r, t in enumerate(trees):
        ms = t.stage_times()
        bt = t.build_times()
        lo, hi = t.rank_range()
        rows.append({"rank": r, "leaf_lo": lo, "leaf_hi": hi, "keys_ms": bt[0], "select_ms": bt[1],
                     "sort_gather_ms": bt[2], "lists_tasks_ms": ms[1],
                     # downward = evaluate_end's own time minus its finish kernel (the library's
                     # ev7 -> ev5 span would include the other ranks' work and the test-side sum)
                     "upward_ms": ms[3], "pairs_ms": ms[2],
                     "downward_ms": ends[r][0].elapsed_time(ends[r][1]) - (ms[5] - ms[2]),
                     "finish_ms": ms[5] - ms[2],
                     "begin_wall_ms": evs[r][0].elapsed_time(evs[r][1]),
                     "end_wall_ms": ends[r][0].elapsed_time(ends[r][1])})
        t.close()
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--warm", type=int, default=1)
    ap.add_argument("--busbw-gbs", type=float, default=400.0,
                    help="assumed NCCL all-reduce bus bandwidth over NVLink 5 (GB/s) for the unhidden part")
    args = ap.parse_args()
    import torch

    import paper_1204_3105_b200 as fmm

    names = WORKLOADS[args.workload]
    inputs = {}
    for nm in names:
        w = fi.get(nm)
        d = fi.generate(w)
        tensors = (torch.from_numpy(d["src_xy"]).cuda(), torch.from_numpy(d["u"]).cuda(),
                   None if d["tgt_xy"] is None else torch.from_numpy(d["tgt_xy"]).cuda(),
                   torch.zeros(w.m, dtype=torch.complex128, device="cuda"))
        inputs[nm] = (w, tensors)
    # grow the library's stream-ordered pool once (the ranks' trees are all alive at the end of a
    # pass), so that no timed stage pays for mapping new pool memory
    free, _ = torch.cuda.mem_get_info()
    fmm.native.pool_reserve(int(0.6 * free))
    out = {"workload": args.workload, "tilings": names, "how": __doc__.strip().splitlines()[0], "ranks": {}}
    for R in [int(x) for x in args.ranks.split(",")]:
        per = {}
        for nm, (w, tensors) in inputs.items():
            for _ in range(args.warm):
                run_tiling(fmm, w, tensors, R)  # warm-up
            reps = [run_tiling(fmm, w, tensors, R) for _ in range(args.reps)]
            # per rank: the median over reps of each stage
            rows = []
            for r in range(R):
                row = {}
                for k in reps[0][r]:
                    vals = sorted(rep[r][k] for rep in reps)
                    row[k] = vals[len(vals) // 2]
                rows.append(row)
            per[nm] = rows
        # a rank's step = sum over tilings of its stages; projected step = max over ranks
        stage_keys = ["keys_ms", "select_ms", "sort_gather_ms", "lists_tasks_ms", "upward_ms", "pairs_ms",
                      "downward_ms", "finish_ms"]
        rank_tot = [sum(per[nm][r][k] for nm in names for k in stage_keys) for r in range(R)]
        mp_bytes = 0
        unhidden = 0.0
        for nm, (w, _) in inputs.items():
            B = 7 if w.tiling == "sept" else 4
            cells = sum(B ** l for l in range(w.depth + 1))
            nb = cells * (w.p + 1) * 16
            mp_bytes += nb
            if R > 1:
                ar_ms = 2.0 * (R - 1) / R * nb / (args.busbw_gbs * 1e9) * 1e3
                min_pairs = min(per[nm][r]["pairs_ms"] for r in range(R))
                unhidden += max(0.0, ar_ms - min_pairs)
        proj = max(rank_tot) + unhidden
        out["ranks"][R] = {"per_tiling": per, "rank_total_ms": rank_tot, "projected_step_ms": proj,
                           "allreduce_bytes_per_step": mp_bytes, "allreduce_unhidden_ms": unhidden,
                           "replicated_ms_per_rank": [sum(per[nm][r]["keys_ms"] + per[nm][r]["select_ms"]
                                                          for nm in names) for r in range(R)]}
        print(f"R={R}: rank totals {[round(x, 2) for x in rank_tot]} -> projected step {proj:.2f} ms",
              file=sys.stderr, flush=True)
    t1 = out["ranks"].get(1, {}).get("projected_step_ms")
    if t1:
        for R, v in out["ranks"].items():
            v["projected_efficiency"] = t1 / (R * v["projected_step_ms"])
    out["assumed_busbw_gbs"] = args.busbw_gbs
    print(json.dumps(out))


if __name__ == "__main__":
    main()
