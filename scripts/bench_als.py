"""Measurement of the f3 block ALS (R21) on one GPU: sweeps/s at a
BASELINE config (L2 flushed before every timed sweep, CUDA events around each sweep), the objective
reached against sWLR after the same number of iterations, and the fp64 oracle's time per sweep on
the host.  Prints one JSON line.

    python scripts/bench_als.py [--config 3] [--steps 50] [--warmup 3]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
import paper_1703_06303_b200 as w

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--oracle-sweeps", type=int, default=1)
args = ap.parse_args()
cfg = synth.CONFIGS[args.config]
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
A = torch.from_numpy(synth.make_A(cfg)).cuda()
W1n = synth.make_W1(cfg)
W1 = None if W1n is None else torch.from_numpy(W1n).cuda()
h = w.wlr_init(A, cfg.k, cfg.r, W1, w1=cfg.w_const or 1.0, stream=stream.cuda_stream)
w.wlr_als_iterate(h, args.warmup)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
torch.cuda.synchronize()
for i in range(args.steps):
    flush.fill_(float(i))
    ev[i][0].record(stream)
    w.wlr_als_iterate_async(h, 1)
    ev[i][1].record(stream)
torch.cuda.synchronize()
F = w.wlr_als_iterate(h, 0)
ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
n_it = args.warmup + args.steps
# sWLR after the same number of iterations (same inputs, GHS start)
h2 = w.wlr_init(A, cfg.k, cfg.r, W1, w1=cfg.w_const or 1.0, stream=stream.cuda_stream)
w.wlr_iterate(h2, n_it)
F_swlr = w.wlr_objective(h2)[0]
# fp64 oracle sweep time on the host (a bounded sample)
import oracle.block_als as ba
An = synth.make_A(cfg).astype(np.float64)
w1 = synth.dense_W1(cfg, W1n, cfg.m)
t0 = time.perf_counter()
ba.block_als(An, w1, cfg.k, cfg.r, args.oracle_sweeps)
t_or = (time.perf_counter() - t0) / max(args.oracle_sweeps, 1)
line = {"metric": "block-ALS sweeps/sec (SURVEY.md §8(f3))", "value": 1e3 / ms, "unit": "sweep/s",
        "ms_per_step": ms, "steps": args.steps, "warmup": args.warmup,
        "config": {"workload": f"BASELINE configs[{args.config - 1}] ({cfg.name}): m={cfg.m}, n={cfg.n}, k={cfg.k}, r={cfg.r}",
                   "l2": "flushed before every timed sweep (256 MB write)",
                   "timing": "CUDA events around one enqueued sweep (wlr_als_iterate with F = NULL)"},
        "F_after": {"iterations": n_it, "block_als": float(F[-1]), "swlr": float(F_swlr)},
        "oracle_fp64_seconds_per_sweep_incl_ghs_start": t_or,
        "gpu_launches_per_sweep": 9}
print(json.dumps(line), flush=True)
