"""Diagnostic: K3 phase timestamps (globaltimer, CTA 0) for one steady-state iteration."""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
import synth
import paper_1703_06303_b200 as w

def run(ci, warm=8, H=None, Wd=None):
    cfg = synth.CONFIGS[ci]
    if H:
        cfg = synth.scaled(cfg, H, Wd)
    A = torch.from_numpy(synth.make_A(cfg)).cuda()
    W1n = synth.make_W1(cfg)
    W1 = None if W1n is None else torch.from_numpy(W1n).cuda()
    h = w.wlr_init(A, cfg.k, cfg.r, W1, w1=cfg.w_const or 1.0)
    w.wlr_iterate(h, warm)
    w.wlr_debug_state(h, "ktime_on")
    for rep in range(2):
        w.wlr_iterate(h, 1)
        kt = w.wlr_debug_state(h, "ktime")
        n = int(kt[0])
        ts = kt[1:1 + n]
        ck = kt[32:32 + n]
        d = np.diff(ts) / 1e3
        mhz = (ck[-1] - ck[0]) / (ts[-1] - ts[0]) * 1e3
        sc = w.wlr_debug_state(h, "scal")
        print(f"cfg{ci} m={cfg.m} nprod={int(sc[7])} total={(ts[-1]-ts[0])/1e3:.1f}us sm_clock={mhz:.0f}MHz phases(us)=" + " ".join(f"{x:.1f}" for x in d))

run(1)
run(2)
run(3)
run(4, H=120, Wd=160)
run(5, warm=3, H=90, Wd=160)

# i-cache hypothesis: relaunch the same small step back to back (second launch warm)
cfg = synth.CONFIGS[3]
A = torch.from_numpy(synth.make_A(cfg)).cuda()
h = w.wlr_init(A, cfg.k, cfg.r, None, w1=cfg.w_const)
w.wlr_iterate(h, 8)
w.wlr_debug_state(h, "ktime_on")
w.wlr_iterate(h, 1)
kt = w.wlr_debug_state(h, "ktime"); n = int(kt[0]); ts = kt[1:1+n]
print("after row pass: total %.1f us" % ((ts[-1]-ts[0])/1e3))
w.wlr_debug_state(h, "ss_rerun")
kt = w.wlr_debug_state(h, "ktime"); n = int(kt[0]); ts = kt[1:1+n]
print("back-to-back relaunch (2nd): total %.1f us; phases " % ((ts[-1]-ts[0])/1e3) + " ".join(f"{x:.1f}" for x in np.diff(ts)/1e3))
