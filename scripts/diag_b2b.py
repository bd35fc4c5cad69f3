"""Back-to-back iteration time (no L2 flush) and one e2e solve's phases at config 3."""
import sys, time
sys.path.insert(0, ".")
import torch, synth, paper_1703_06303_b200 as w
cfg = synth.CONFIGS[3]
A = torch.from_numpy(synth.make_A(cfg)).cuda()
h = w.wlr_init(A, cfg.k, cfg.r, None, w1=100.0)
w.wlr_iterate(h, 10); torch.cuda.synchronize()
for n in (1, 10, 200):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); w.wlr_iterate_async(h, n); e1.record(); torch.cuda.synchronize()
    print("b2b", n, "ms/iter", e0.elapsed_time(e1) / n, flush=True)
Ah = torch.from_numpy(synth.make_A(cfg)).pin_memory()
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    he = w.wlr_init(Ah, cfg.k, cfg.r, None, w1=100.0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    w.wlr_iterate_async(he, 200); torch.cuda.synchronize(); t2 = time.perf_counter()
    r = w.wlr_result(he); torch.cuda.synchronize(); t3 = time.perf_counter()
    w.wlr_destroy(he)
    print(f"e2e init {1e3*(t1-t0):.1f} ms, 200 it {1e3*(t2-t1):.1f} ms, result {1e3*(t3-t2):.1f} ms", flush=True)
