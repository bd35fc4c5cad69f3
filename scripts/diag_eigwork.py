"""Diagnostic: per-iteration eigen-solver work in K3a (S-products, outer Chebyshev passes,
residual ratio) over a run of config 3 -- to see whether a change alters convergence work."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import synth
import paper_1703_06303_b200 as w
cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
A = torch.from_numpy(synth.make_A(cfg)).cuda()
h = w.wlr_init(A, cfg.k, cfg.r, None, w1=cfg.w_const or 1.0)
prods = []
for it in range(60):
    w.wlr_iterate(h, 1)
    sc = w.wlr_debug_state(h, "scal")
    prods.append((int(sc[7]), sc[6], sc[4]))
print("S-products per iteration:", [p[0] for p in prods])
print("residual ratio (last 5):", ["%.1e" % p[1] for p in prods[-5:]], "rel step:", "%.2e" % prods[-1][2])
