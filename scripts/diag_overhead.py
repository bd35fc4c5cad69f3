"""Diagnostic: per-step time as bench.py measures it (events around one graph launch after an L2
flush) against back-to-back launches without a flush, to size the launch/graph overhead that
sits outside the kernels (compare with scripts/diag_timeline.py's kernel span)."""
import sys
sys.path.insert(0, ".")
import torch
import synth
import paper_1703_06303_b200 as w

cfg = synth.CONFIGS[3]
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
A = torch.from_numpy(synth.make_A(cfg)).cuda()
h = w.wlr_init(A, cfg.k, cfg.r, None, w1=cfg.w_const or 1.0, stream=stream.cuda_stream)
w.wlr_row_path(h, True)
w.wlr_incr_path(h, True)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
w.wlr_iterate_async(h, 10)
torch.cuda.synchronize()
E = lambda: torch.cuda.Event(enable_timing=True)
K = 50
# (1) bench style
ev = [(E(), E()) for _ in range(K)]
for i in range(K):
    flush.fill_(float(i))
    ev[i][0].record(stream)
    w.wlr_iterate_async(h, 1)
    ev[i][1].record(stream)
torch.cuda.synchronize()
t1 = sorted(a.elapsed_time(b) for a, b in ev)
print("bench-style (flush, 1 graph per timed region): median %.1f us" % (t1[K // 2] * 1e3))
# (2) same without the flush
ev = [(E(), E()) for _ in range(K)]
for i in range(K):
    ev[i][0].record(stream)
    w.wlr_iterate_async(h, 1)
    ev[i][1].record(stream)
torch.cuda.synchronize()
t2 = sorted(a.elapsed_time(b) for a, b in ev)
print("no flush, 1 graph per timed region: median %.1f us" % (t2[K // 2] * 1e3))
# (3) back to back, one timed region
a, b = E(), E()
a.record(stream)
w.wlr_iterate_async(h, K)
b.record(stream)
torch.cuda.synchronize()
print("no flush, %d back-to-back: %.1f us per iteration" % (K, a.elapsed_time(b) * 1e3 / K))
# (4) flush + a sync before each step (host waits: the graph launch is submitted to an idle GPU)
ev = [(E(), E()) for _ in range(K)]
for i in range(K):
    flush.fill_(float(i))
    torch.cuda.synchronize()
    ev[i][0].record(stream)
    w.wlr_iterate_async(h, 1)
    ev[i][1].record(stream)
torch.cuda.synchronize()
t4 = sorted(a.elapsed_time(b) for a, b in ev)
print("flush + host sync before the step: median %.1f us" % (t4[K // 2] * 1e3))
