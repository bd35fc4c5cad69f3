"""Timeline of the tensor-core row pass: per-CTA globaltimer stamps (WLR_TC_DBG=16).  Usage: [config]"""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
import synth
import paper_1703_06303_b200 as w
cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
A = torch.from_numpy(synth.make_A(cfg)).cuda()
W1n = synth.make_W1(cfg)
W1 = None if W1n is None else torch.from_numpy(W1n).cuda()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
h = w.wlr_init(A, cfg.k, cfg.r, W1, w1=cfg.w_const or 1.0)
w.wlr_iterate(h, 5)
flush.fill_(1.0)
w.wlr_iterate_async(h, 1)
torch.cuda.synchronize()
tt = w.wlr_debug_state(h, "tctime").view(np.uint64).astype(np.int64)
t = tt[: tt.size // 2].reshape(-1, 8)
wc = tt[tt.size // 2:].reshape(-1, 8)
t0 = t[:, 0].min()
names = ["start", "first_full", "first_tma", "epi_wait", "accfull", "epi_done", "end"]
for i, nm in enumerate(names):
    v = (t[:, i] - t0) / 1e3
    print(f"{nm:11s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us")
wnames = ["prod wait rawfree", "mma wait lofull", "mma wait accfree", "conv wait full", "conv wait lofree",
          "epi wait accfull", "conv busy"]
for i, nm in enumerate(wnames):
    v = wc[:, i] / 1.965e3
    print(f"{nm:18s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us (cycles / 1965)")
end = (t[:, 6] - t0) / 1e3
order = np.argsort(end)[::-1][:8]
print("slowest CTAs (index: end us):", " ".join(f"{i}:{end[i]:.1f}" for i in order))
print("end by CTA block of 16:", " ".join(f"{end[i:i+16].mean():.1f}" for i in range(0, len(end), 16)))
