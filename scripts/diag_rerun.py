"""Diagnostic: K3a phase times in the pipeline vs. rerun back to back (warm instruction cache).
ss_rerun relaunches the last critical half twice; the marks of the second launch are read."""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
import synth
import paper_1703_06303_b200 as w

def phases(kt, off=0):
    n = int(kt[off]); ts = kt[off + 1:off + 1 + n]
    return (ts[-1] - ts[0]) / 1e3, " ".join(f"{x:.1f}" for x in np.diff(ts) / 1e3)

for ci in (2, 3):
    cfg = synth.CONFIGS[ci]
    A = torch.from_numpy(synth.make_A(cfg)).cuda()
    W1n = synth.make_W1(cfg)
    W1 = None if W1n is None else torch.from_numpy(W1n).cuda()
    h = w.wlr_init(A, cfg.k, cfg.r, W1, w1=cfg.w_const or 1.0)
    w.wlr_iterate(h, 8)
    w.wlr_debug_state(h, "ktime_on")
    w.wlr_iterate_async(h, 1); torch.cuda.synchronize()
    tot, ph = phases(w.wlr_debug_state(h, "ktime"))
    print(f"cfg{ci} pipeline K3a {tot:.1f}us: {ph}")
    w.wlr_debug_state(h, "ss_rerun")
    tot, ph = phases(w.wlr_debug_state(h, "ktime"))
    print(f"cfg{ci} rerun    K3a {tot:.1f}us: {ph}")
