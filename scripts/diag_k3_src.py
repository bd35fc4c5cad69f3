"""Run config 3 for a few graph iterations (for an ncu SourceCounters capture of the small-step
kernels: which SASS instructions execute per call, i.e. the code footprint fetched after an L2 flush)."""
import sys
sys.path.insert(0, ".")
import torch, synth, paper_1703_06303_b200 as w
cfg = synth.CONFIGS[3]
A = torch.from_numpy(synth.make_A(cfg)).cuda()
h = w.wlr_init(A, cfg.k, cfg.r, None, w1=100.0)
w.wlr_iterate(h, 30)
torch.cuda.synchronize()
print("ok")
