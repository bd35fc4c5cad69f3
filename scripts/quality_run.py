"""background quality on the synthetic scenes.  Solve on the GPU (GHS init,
eps = 1e-7), then the mean SSIM (metrics.mean_ssim, R19) of the recovered background
frames X2 = X1 C + B D (frames k..n-1, the ones carrying the moving foreground) against the
generator's clean background, next to the SSIM of the raw frames A2 (no processing)."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch
import metrics
import synth
import paper_1703_06303_b200 as w

for ci in [int(x) for x in sys.argv[1:]] or [2, 3]:
    cfg = synth.CONFIGS[ci]
    A = synth.make_A(cfg)
    bg = synth.make_background(cfg)
    h = w.wlr_init(torch.from_numpy(A).cuda(), cfg.k, cfg.r, None, w1=cfg.w_const, eps=1e-7)
    done, conv = w.wlr_iterate(h, 300)
    res = w.wlr_result(h, x2=True)
    X2 = res["X2"].astype(np.float64)
    s_est = metrics.mean_ssim(X2, bg[:, cfg.k:], cfg.H, cfg.W)
    s_raw = metrics.mean_ssim(A[:, cfg.k:].astype(np.float64), bg[:, cfg.k:], cfg.H, cfg.W)
    s_x1 = metrics.mean_ssim(res["X1"].astype(np.float64), bg[:, :cfg.k], cfg.H, cfg.W)
    print(json.dumps({"config": cfg.name, "m": cfg.m, "n": cfg.n, "k": cfg.k, "r": cfg.r, "iters": done,
                      "converged": conv, "mean_ssim_X2_vs_clean_bg": s_est,
                      "mean_ssim_raw_A2_vs_clean_bg": s_raw, "mean_ssim_X1_vs_clean_bg": s_x1}), flush=True)
