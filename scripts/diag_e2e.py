"""Diagnostic: where the end-to-end solve time goes (host wall clock, synchronised after each
part): wlr_init from pinned host A, the first 12 iterations (graph builds), the remaining ones,
and the result copy."""
import sys, time
sys.path.insert(0, ".")
import torch
import synth
import paper_1703_06303_b200 as w
cfg = synth.CONFIGS[3]
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
Ah = torch.from_numpy(synth.make_A(cfg)).pin_memory()
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = w.wlr_init(Ah, cfg.k, cfg.r, None, w1=cfg.w_const, stream=stream.cuda_stream)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    w.wlr_iterate_async(h, 12); torch.cuda.synchronize(); t2 = time.perf_counter()
    w.wlr_iterate_async(h, 188); torch.cuda.synchronize(); t3 = time.perf_counter()
    res = w.wlr_result(h, x2=False); torch.cuda.synchronize(); t4 = time.perf_counter()
    w.wlr_destroy(h); torch.cuda.synchronize(); t5 = time.perf_counter()
    print(f"rep {rep}: init {1e3*(t1-t0):.2f} ms | first 12 it {1e3*(t2-t1):.2f} ms | next 188 it {1e3*(t3-t2):.2f} ms "
          f"({1e3*(t3-t2)/188:.3f}/it) | result {1e3*(t4-t3):.2f} ms | destroy {1e3*(t5-t4):.2f} ms")
