"""Quick GPU-vs-oracle diagnostic (prints per-state errors).  Test infrastructure."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from threadpoolctl import threadpool_limits
threadpool_limits(1)
import torch
import synth, oracle
from tests import gpu_util as gu
from tests import gram_route
import paper_1703_06303_b200 as w

which = [int(x) for x in sys.argv[1:]] or [1, 2]
for ci in which:
    cfg = synth.CONFIGS[ci]
    if ci >= 4:
        cfg = synth.scaled(cfg, 60, 80)
    A, W1 = gu.inputs(cfg)
    At = torch.from_numpy(A).cuda()
    Wt = None if W1 is None else torch.from_numpy(W1).cuda()
    t0 = time.time()
    h = w.wlr_init(At, cfg.k, cfg.r, Wt, w1=cfg.w_const or 1.0)
    torch.cuda.synchronize()
    print(f"cfg{ci} init {time.time()-t0:.3f}s", flush=True)
    A64 = A.astype(np.float64)
    st = gram_route.cd_gram(A64[:, :cfg.k], A64[:, cfg.k:], cfg.r)
    C = w.wlr_debug_state(h, "C").reshape(cfg.k, -1)
    lam = w.wlr_debug_state(h, "lam")
    V = w.wlr_debug_state(h, "V").reshape(-1, cfg.r - cfg.k)
    G = w.wlr_debug_state(h, "G").reshape(cfg.k, cfg.k)
    print("  G err", gu.rel(G, st["G"]), " C err", gu.rel(C, st["C"]), " lam", lam, st["lam"],
          " VV^T err", gu.rel(V @ V.T, st["V"] @ st["V"].T), "scal", w.wlr_debug_state(h, "scal"))
    iters = min(cfg.iters, 30)
    o = gu.run_oracle(cfg, A, W1, iters)
    done, conv = w.wlr_iterate(h, iters)
    tr = w.wlr_trace(h)
    for p in range(len(tr)):
        fo = o.trace[p]["F"]
        print(f"  p={p:3d} F={tr[p,0]:.10e} relF={abs(tr[p,0]-fo)/fo:.2e} step={tr[p,1]:.3e}/{o.trace[p].get('step',-1):.3e} rel={tr[p,2]:.3e}/{o.trace[p].get('rel',-1):.3e}")
    res = w.wlr_result(h, x2=True)
    print("  relX", gu.rel(gu.gpu_X(res), o.x), "scal", w.wlr_debug_state(h, "scal"))
    prof = None
