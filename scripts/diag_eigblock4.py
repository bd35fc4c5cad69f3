"""Config 4: iteration time and S-products per iteration against the eigen block width b (graph
iterations 21-40 after 20 warm-up iterations, warm L2)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch, synth, paper_1703_06303_b200 as w
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = synth.CONFIGS[ci]
A = torch.from_numpy(synth.make_A(cfg)).cuda()
W1 = torch.from_numpy(synth.make_W1(cfg)).cuda()
for b in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else "8,11,14,16,20")]:
    h = w.wlr_init(A, cfg.k, cfg.r, W1, eig_block=b)
    w.wlr_iterate(h, 20); torch.cuda.synchronize()
    ts, npr = [], []
    for it in range(20):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); w.wlr_iterate_async(h, 1); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3); npr.append(w.wlr_debug_state(h, "scal")[7])
    F = w.wlr_objective(h)[0]
    print(f"b={b:2d}: {np.mean(ts):7.1f} us/iter  S-products/iter {np.mean(npr):5.1f}  F_40 {F:.10e}", flush=True)
    w.wlr_destroy(h)
