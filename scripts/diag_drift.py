"""Drift of the device's running Grams G = X1^T X1, M = X1^T A2 from an fp64 recomputation from the
returned X1 (config 3 by default), with the tensor-core row pass on and off."""
import argparse, sys
sys.path.insert(0, ".")
import numpy as np
import torch
import synth
import paper_1703_06303_b200 as w

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--iters", type=int, nargs="+", default=[1, 2, 5, 20])
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
A = synth.make_A(cfg)
W1n = synth.make_W1(cfg)
At = torch.from_numpy(A).cuda()
Wt = None if W1n is None else torch.from_numpy(W1n).cuda()
A64 = A.astype(np.float64)
for tc in (True, False):
    h = w.wlr_init(At, cfg.k, cfg.r, Wt, w1=cfg.w_const or 1.0)
    got = w.wlr_row_path(h, tc)
    done = 0
    for it in a.iters:
        w.wlr_iterate(h, it - done)
        done = it
        X1 = w.wlr_result(h, b=False)["X1"].astype(np.float64)
        G = w.wlr_debug_state(h, "G").reshape(cfg.k, cfg.k)
        M = w.wlr_debug_state(h, "M").reshape(cfg.k, cfg.n - cfg.k)
        Gf = X1.T @ X1
        Mf = X1.T @ A64[:, cfg.k:]
        print(f"tc={got} p={it}: G drift {np.linalg.norm(G - Gf) / np.linalg.norm(Gf):.2e}  "
              f"M drift {np.linalg.norm(M - Mf) / np.linalg.norm(Mf):.2e}  F {w.wlr_objective(h)}", flush=True)
    w.wlr_destroy(h)
