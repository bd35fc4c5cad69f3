"""Pins of the host-side background-quality metric (SPEC.md:415-423
examples and invariants), checked against a direct windowed evaluation written with loops."""
import numpy as np

import metrics
import synth


def _ssim_direct(x, y, win=11, sigma=1.5):
    """Wang et al. (2004) local SSIM with explicit loops over every valid window position."""
    w = metrics.gaussian_window(win, sigma)
    H, W = x.shape
    c1, c2 = (0.01) ** 2, (0.03) ** 2
    vals = []
    for i in range(H - win + 1):
        for j in range(W - win + 1):
            px, py = x[i:i + win, j:j + win], y[i:i + win, j:j + win]
            mx, my = (w * px).sum(), (w * py).sum()
            sxx = (w * (px - mx) ** 2).sum()
            syy = (w * (py - my) ** 2).sum()
            sxy = (w * (px - mx) * (py - my)).sum()
            vals.append(((2 * mx * my + c1) * (2 * sxy + c2)) / ((mx * mx + my * my + c1) * (sxx + syy + c2)))
    return float(np.mean(vals))


def test_ssim_matches_direct_window_loop():
    g = np.random.default_rng(3)
    x = g.uniform(0, 1, (17, 19))
    y = np.clip(x + 0.1 * g.standard_normal(x.shape), 0, 1)
    assert abs(metrics.ssim(x, y) - _ssim_direct(x, y)) < 1e-12


def test_ssim_identity_and_symmetry():
    g = np.random.default_rng(4)
    x = g.uniform(0, 1, (16, 16))
    y = g.uniform(0, 1, (16, 16))
    assert metrics.ssim(x, x) == 1.0
    assert abs(metrics.ssim(x, y) - metrics.ssim(y, x)) < 1e-15


def test_ssim_offset_decreasing_and_sign_flip():
    """a constant offset lowers SSIM monotonically in |c|; -truth of a
    mean-zero frame gives negative SSIM."""
    g = np.random.default_rng(5)
    t = 0.5 + 0.2 * g.standard_normal((12, 12))
    s = [metrics.ssim(t + c, t) for c in (0.0, 0.05, 0.1, 0.2, 0.4)]
    assert s[0] == 1.0 and all(a > b for a, b in zip(s, s[1:]))
    # sign flip of the structure around a common mean (local means of the checkerboard ~ 0):
    # the structure term is -1 and drives SSIM negative
    i, j = np.meshgrid(np.arange(12), np.arange(12), indexing="ij")
    d = 0.2 * (-1.0) ** (i + j)
    assert metrics.ssim(0.5 + d, 0.5 - d) < 0


def test_mean_ssim_of_clean_background_and_scene():
    cfg = synth.CONFIGS[2]
    bg = synth.make_background(cfg)
    assert bg.shape == (cfg.m, cfg.n)
    assert metrics.mean_ssim(bg, bg, cfg.H, cfg.W) == 1.0
    # the raw frames (foreground block + noise) are a worse background estimate than the truth
    A = synth.make_A(cfg).astype(np.float64)
    s = metrics.mean_ssim(A[:, cfg.k:], bg[:, cfg.k:], cfg.H, cfg.W)
    assert 0.0 < s < 1.0
