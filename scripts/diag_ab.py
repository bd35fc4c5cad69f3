"""Diagnostic: A/B of two kernel paths (debug toggles, e.g. incrtc_on / incrtc_off) on the same problem -- agreement of
the iterates after N steps and per-kernel times (L2 flushed between iterations)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
import synth
import paper_1703_06303_b200 as w

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = synth.CONFIGS[ci]
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
A = torch.from_numpy(synth.make_A(cfg)).cuda()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
res = {}
for mode in (sys.argv[2] if len(sys.argv) > 2 else "incrtc_on", sys.argv[3] if len(sys.argv) > 3 else "incrtc_off"):
    h = w.wlr_init(A, cfg.k, cfg.r, None, w1=cfg.w_const, stream=stream.cuda_stream)
    on = w.wlr_debug_state(h, mode)
    w.wlr_iterate(h, 20)
    X1 = w.wlr_result(h)["X1"]
    F = w.wlr_objective(h)
    w.wlr_profile(h, enable=True, reset=True)
    for i in range(20):
        flush.fill_(float(i))
        w.wlr_iterate_async(h, 1)
    pr = w.wlr_profile(h, enable=False, reset=False)
    it = pr["iters"]
    res[mode] = (X1, F)
    print(mode, "active" if len(on) and on[0] else "inactive", "F", F,
          {k: round(v / it * 1e3, 1) for k, v in pr.items() if k not in ("launches", "iters")}, flush=True)
(X1a, Fa), (X1b, Fb) = list(res.values())
print("rel ||X1_tc - X1_cc|| =", float(np.linalg.norm(X1a - X1b) / np.linalg.norm(X1b)),
      " relF =", abs(Fa[0] - Fb[0]) / abs(Fb[0]))
