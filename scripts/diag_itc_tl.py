"""Timeline of the tensor-core increments: per-CTA globaltimer stamps (WLR_TC_DBG=32) after an
L2 flush + row pass, as in the bench step."""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
import synth
import paper_1703_06303_b200 as w
cfg = synth.CONFIGS[3]
A = torch.from_numpy(synth.make_A(cfg)).cuda()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
h = w.wlr_init(A, cfg.k, cfg.r, None, w1=cfg.w_const)
w.wlr_iterate(h, 8)
flush.fill_(1.0)
w.wlr_iterate_async(h, 1)
torch.cuda.synchronize()
tt = w.wlr_debug_state(h, "itctime").view(np.uint64).astype(np.int64).reshape(-1, 8)
tt = tt[tt[:, 0] > 0]
t0 = tt[:, 0].min()
for i, nm in enumerate(["start", "first_full", "conv_done", "acc_full", "end"]):
    v = (tt[:, i] - t0) / 1e3
    print(f"{nm:11s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us  (n={len(v)})")
