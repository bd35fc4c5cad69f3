"""Host wall-clock of wlr_init (device A, config 3) and of the first iterations, median of N
handles, for an env A/B (e.g. WLR_SHADOW=0 / 1 in separate processes)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch, synth
import paper_1703_06303_b200 as w
cfg = synth.CONFIGS[3]
A = torch.from_numpy(synth.make_A(cfg)).cuda()
ti, t1, t200 = [], [], []
for i in range(12):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = w.wlr_init(A, cfg.k, cfg.r, None, w1=cfg.w_const)
    torch.cuda.synchronize(); t1_ = time.perf_counter()
    w.wlr_iterate(h, 1)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    w.wlr_iterate(h, 200)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    w.wlr_destroy(h)
    if i >= 2:
        ti.append(t1_ - t0); t1.append(t2 - t1_); t200.append(t3 - t2)
print(f"init {np.median(ti)*1e3:.3f} ms  first iter {np.median(t1)*1e3:.3f} ms  200 iters {np.median(t200)*1e3:.3f} ms")
