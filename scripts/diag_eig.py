"""Diagnostic: eigensolver outer iterations and per-kernel times per iteration (GPU)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
import synth
import paper_1703_06303_b200 as w

def run(ci, iters=30, H=None, Wd=None, **kw):
  try:
    _run(ci, iters, H, Wd, **kw)
  except Exception as e:
    print('FAILED', ci, kw, e)

def _run(ci, iters=30, H=None, Wd=None, **kw):
    cfg = synth.CONFIGS[ci]
    if H:
        cfg = synth.scaled(cfg, H, Wd)
    A = torch.from_numpy(synth.make_A(cfg)).cuda()
    W1n = synth.make_W1(cfg)
    W1 = None if W1n is None else torch.from_numpy(W1n).cuda()
    h = w.wlr_init(A, cfg.k, cfg.r, W1, w1=cfg.w_const or 1.0, **kw)
    sc = w.wlr_debug_state(h, 'scal')
    print(f"cfg{ci} m={cfg.m} kw={kw} init outer={w.wlr_debug_state(h,'outer')[0]} res={sc[6]:.2e} nprod={sc[7]}")
    outs = []
    for p in range(iters):
        w.wlr_profile(h, enable=True, reset=True)
        w.wlr_iterate_async(h, 1)
        pr = w.wlr_profile(h, enable=False, reset=False)
        sc = w.wlr_debug_state(h, 'scal')
        outs.append((int(w.wlr_debug_state(h, 'outer')[0]), pr['small_step'], pr['row_pass'], pr['increments'], sc[6], int(sc[7])))
    tr = w.wlr_trace(h)
    for p, o in enumerate(outs):
        print(f"  p={p+1:3d} outer={o[0]:3d} nprod={o[5]:3d} res={o[4]:.1e} ss={o[1]*1e3:8.1f}us rp={o[2]*1e3:6.1f} inc={o[3]*1e3:6.1f}  rel={tr[p+1,2]:.3e}")

run(3, 25)
run(3, 10, eig_block=4)
run(2, 10)
run(1, 10)
run(4, 15, H=120, Wd=160)
run(5, 8, H=90, Wd=160)
