"""prop1 phase stamps (WLR_PROP_TS=1): per CTA %globaltimer at entry, before/after the dependency
wait, W' landed, Q rows done, partials done, G_A Y done; printed relative to the first CTA's entry
(min / median / max over the CTAs), warm and after an L2 flush."""
import os, sys
os.environ["WLR_PROP_TS"] = "1"
sys.path.insert(0, ".")
import numpy as np, torch, synth, paper_1703_06303_b200 as w
cfg = synth.CONFIGS[3]
A = torch.from_numpy(synth.make_A(cfg)).cuda()
h = w.wlr_init(A, cfg.k, cfg.r, None, w1=100.0)
w.wlr_iterate(h, 10); torch.cuda.synchronize()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
names = ["entry", "rows issued", "pdl_wait done", "G_A Y", "W' landed", "Q rows", "partials/end"]
for mode in ("warm", "flushed", "warm", "flushed"):
    if mode == "flushed":
        flush.fill_(1.0)
    torch.cuda.synchronize()
    w.wlr_iterate_async(h, 1)
    torch.cuda.synchronize()
    ts = w.wlr_debug_state(h, "proptime").view(np.uint64).astype(np.int64).reshape(-1, 8)[:, :7]
    ts = ts[ts[:, 0] > 0]                      # (the CTAs of the grid)
    t0 = ts[:, 0].min()
    rel = (ts - t0) / 1e3
    print(mode, " ".join(f"{nm}: {np.min(rel[:, i]):.1f}/{np.median(rel[:, i]):.1f}/{np.max(rel[:, i]):.1f}" for i, nm in enumerate(names)))
