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
names2 = ["entry", "pre-wait loads", "pdl_wait", "panel sums", "cluster gather", "W'X G terms", "end"]
names = ["entry", "rows issued", "pdl_wait done", "G_A Y", "W' landed", "Q rows", "partials/end"]
for mode in ("warm", "flushed", "warm", "flushed"):
    if mode == "flushed":
        flush.fill_(1.0)
    torch.cuda.synchronize()
    w.wlr_iterate_async(h, 1)
    torch.cuda.synchronize()
    allts = w.wlr_debug_state(h, "proptime").view(np.uint64).astype(np.int64).reshape(-1, 8)
    nb = min(cfg.n, torch.cuda.get_device_properties(0).multi_processor_count)
    ts = allts[:nb, :7]
    t0 = ts[:, 0].min()
    rel = (ts - t0) / 1e3
    print(mode, "prop1", " ".join(f"{nm}: {np.min(rel[:, i]):.1f}/{np.median(rel[:, i]):.1f}/{np.max(rel[:, i]):.1f}" for i, nm in enumerate(names)))
    t2 = allts[nb:nb + 3 * cfg.k, :7]
    r2 = (t2 - t0) / 1e3
    print(mode, "prop2", " ".join(f"{nm}: {np.min(np.where(t2[:, i] > 0, r2[:, i], 1e9)):.1f}/{np.median(r2[t2[:, i] > 0, i]):.1f}/{np.max(r2[:, i]):.1f}" for i, nm in enumerate(names2)))
