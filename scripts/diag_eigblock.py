"""K3a phase times and iteration rate vs eigen block width b (config 3)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
import synth
import paper_1703_06303_b200 as w
cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
A = torch.from_numpy(synth.make_A(cfg)).cuda()
W1n = synth.make_W1(cfg)
W1 = None if W1n is None else torch.from_numpy(W1n).cuda()
for b in (0, 3, 4, 6):
    h = w.wlr_init(A, cfg.k, cfg.r, W1, w1=cfg.w_const or 1.0, eig_block=b)
    w.wlr_iterate(h, 20)
    w.wlr_profile(h, enable=True, reset=True)
    w.wlr_iterate_async(h, 20)
    pr = w.wlr_profile(h, enable=False, reset=False)
    w.wlr_debug_state(h, "ktime_on")
    w.wlr_iterate_async(h, 1); torch.cuda.synchronize()
    kt = w.wlr_debug_state(h, "ktime")
    n = int(kt[0]); ts = kt[1:1 + n]
    outer = w.wlr_debug_state(h, "outer")
    F = w.wlr_objective(h)
    print(f"b={b or 'default'} K3a={pr['small_step']/pr['iters']*1e3:.1f}us deferred={pr['deferred']/pr['iters']*1e3:.1f}us "
          f"outer={outer} F={F[0]:.10f} rel={F[2]:.2e} phases=" + " ".join(f"{x:.1f}" for x in np.diff(ts) / 1e3), flush=True)
    w.wlr_destroy(h)
