"""Host-side quality metric for the synthetic scenes:
mean SSIM of the recovered background frames against the generator's clean background.

The paper reports "Mean SSIM" (Fig. 3 caption, §4.3) without defining it; this is the
standard structural similarity of Wang, Bovik, Sheikh and Simoncelli (2004): Gaussian window
11 x 11 with sigma 1.5 (normalised), K1 = 0.01, K2 = 0.03, data range L = 1 (pixels in [0, 1]),
local statistics by 'valid' windowed filtering, SSIM map averaged over the frame, and the
mean over frames (reading R19).  Not part of the hot path; not used by the oracle.
"""
import numpy as np

K1, K2, L = 0.01, 0.03, 1.0


def gaussian_window(size: int = 11, sigma: float = 1.5) -> np.ndarray:
    ax = np.arange(size) - (size - 1) / 2.0
    g = np.exp(-0.5 * (ax / sigma) ** 2)
    w = np.outer(g, g)
    return w / w.sum()


def _filter_valid(img: np.ndarray, w: np.ndarray) -> np.ndarray:
    """'Valid' 2-D correlation of img with w (separable Gaussian, done as two 1-D passes)."""
    g = w.sum(axis=1)                       # the 1-D factor (w = outer(g, g) / sum)
    g = g / g.sum()
    n = g.size
    rows = np.lib.stride_tricks.sliding_window_view(img, n, axis=0) @ g
    return np.lib.stride_tricks.sliding_window_view(rows, n, axis=1) @ g


def ssim(x: np.ndarray, y: np.ndarray, window: int = 11, sigma: float = 1.5) -> float:
    """SSIM of two H x W frames (mean of the local SSIM map)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if x.shape != y.shape:
        raise ValueError("dims mismatch")
    w = gaussian_window(min(window, *x.shape) | 1, sigma)
    mx, my = _filter_valid(x, w), _filter_valid(y, w)
    sxx = _filter_valid(x * x, w) - mx * mx
    syy = _filter_valid(y * y, w) - my * my
    sxy = _filter_valid(x * y, w) - mx * my
    c1, c2 = (K1 * L) ** 2, (K2 * L) ** 2
    smap = ((2 * mx * my + c1) * (2 * sxy + c2)) / ((mx * mx + my * my + c1) * (sxx + syy + c2))
    return float(smap.mean())


def mean_ssim(est: np.ndarray, truth: np.ndarray, H: int, W: int) -> float:
    """Mean over columns (frames, pixels i = y W + x) of the per-frame SSIM."""
    est = np.asarray(est)
    truth = np.asarray(truth)
    if est.shape != truth.shape or est.shape[0] != H * W:
        raise ValueError("dims mismatch")
    return float(np.mean([ssim(est[:, j].reshape(H, W), truth[:, j].reshape(H, W))
                          for j in range(est.shape[1])]))
