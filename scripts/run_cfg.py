"""Run N sWLR iterations of a BASELINE config on cuda:0 (profiling driver)."""
import argparse, sys
sys.path.insert(0, ".")
import torch
import synth
import paper_1703_06303_b200 as w

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--H", type=int, default=0)
ap.add_argument("--W", type=int, default=0)
ap.add_argument("--no-graph", action="store_true")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
if a.H:
    cfg = synth.scaled(cfg, a.H, a.W)
A = torch.from_numpy(synth.make_A(cfg)).cuda()
W1n = synth.make_W1(cfg)
W1 = None if W1n is None else torch.from_numpy(W1n).cuda()
h = w.wlr_init(A, cfg.k, cfg.r, W1, w1=cfg.w_const or 1.0, use_graph=not a.no_graph)
w.wlr_iterate(h, a.iters)
print("F", w.wlr_objective(h))
