"""Per-iteration eigen work of K3a at config 4 (full size): S-products (scal[7]) and the K3a time
of each iteration (CUDA events around single graph iterations, warm L2)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch, synth, paper_1703_06303_b200 as w
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = synth.CONFIGS[ci]
A = torch.from_numpy(synth.make_A(cfg)).cuda()
W1n = synth.make_W1(cfg)
W1 = None if W1n is None else torch.from_numpy(W1n).cuda()
h = w.wlr_init(A, cfg.k, cfg.r, W1, w1=cfg.w_const or 1.0)
torch.cuda.synchronize()
for it in range(1, 61):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); w.wlr_iterate_async(h, 1); e1.record(); torch.cuda.synchronize()
    sc = w.wlr_debug_state(h, "scal")
    print(f"it {it:3d}: {e0.elapsed_time(e1) * 1e3:8.1f} us  nprod {sc[7]:.0f}  res/theta {sc[6]:.2e}", flush=True)
