"""Seeded synthetic inputs for the sWLR hot path (BASELINE.json ``configs``).

This module is shared by the tests, ``bench.py`` and ``__graft_entry__.smoke``.
It holds NONE of the method's arithmetic (no projection, no SVD, no row solve):
it only draws pixels and weights.  Both the CUDA path and the fp64 oracle
receive exactly the arrays produced here (for fp32 configs the arrays are rounded
to fp32 once, and the oracle sees those values upcast -- DESIGN.md reading R12).

Recipes.  PAPER.md §4.2
measures on the Stuttgart synthetic video; it is not in this container, so the
scene generator below stands in for it: columns are frames, rows are pixels
(i = y*W + x), a low-rank illumination-modulated background, a moving square
foreground block in frames k..n-1 (the A2 block), Gaussian sensor noise, and
optional salt-and-pepper corruption of A2.

Determinism: every array is a pure function of (config, seed).  Row chunks of
``CHUNK_ROWS`` pixels draw their noise from ``default_rng([seed, 1, chunk])`` so
any row range can be generated independently (row sharding) and the result does
not depend on how many ranks ask for it.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional, Tuple

import numpy as np

CHUNK_ROWS = 16384

# (a, b) cosine frequencies for background components 2..
_COS_FREQS = [(1, 0), (0, 1), (1, 1), (2, 0), (0, 2), (2, 1), (1, 2), (2, 2), (3, 0)]


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json config.  ``H*W == m`` for scene configs."""
    name: str
    m: int
    n: int
    k: int
    r: int
    dtype: str              # "f64" or "f32": storage / row-pass precision
    iters: int              # fixed iteration count of the config
    kind: str               # "lowrank" (config 1) or "scene"
    H: int = 0
    W: int = 0
    q: int = 0              # background rank
    block: int = 0          # foreground block side b
    sigma: float = 0.0      # noise std
    sp: float = 0.0         # salt-and-pepper fraction on A2
    w_const: Optional[float] = None     # uniform W1 value, or None
    w_logu: Optional[Tuple[float, float]] = None  # log-uniform W1 range
    seed: int = 0

    @property
    def np_dtype(self):
        return np.float64 if self.dtype == "f64" else np.float32

    @property
    def uniform_w(self) -> bool:
        return self.w_const is not None


CONFIGS = {
    # BJ configs[0]: tiny fp64, A = U V + N(0, 0.01^2), W1 = 50, 50 iterations, seed 0
    1: Config("tiny_fp64", 300, 40, 10, 12, "f64", 50, "lowrank", w_const=50.0, seed=0),
    # BJ configs[1]: 60x80 frames, n=100, k=20, r=22, rank-2 background, 10x10 block
    2: Config("small_fp32", 4800, 100, 20, 22, "f32", 100, "scene", H=60, W=80, q=2,
              block=10, sigma=0.02, sp=0.0, w_const=100.0, seed=0),
    # BJ configs[2]: QVGA 120x160, n=600, k=30, r=32, 20x20 blocks, 5% S&P in A2 (the metric)
    3: Config("qvga_fp32", 19200, 600, 30, 32, "f32", 200, "scene", H=120, W=160, q=2,
              block=20, sigma=0.02, sp=0.05, w_const=100.0, seed=0),
    # BJ configs[3]: 240x320, n=500, k=50, r=55, rank-5 bg, W1 log-uniform [1, 1e3]
    4: Config("nonuniform_fp32", 76800, 500, 50, 55, "f32", 100, "scene", H=240, W=320, q=5,
              block=20, sigma=0.02, sp=0.05, w_logu=(1.0, 1e3), seed=0),
    # BJ configs[4]: 720x1280, n=1000, k=100, r=110, rank-10 bg, 64x64 blocks, W1 log-U [10, 1e3]
    5: Config("large_fp32", 921600, 1000, 100, 110, "f32", 50, "scene", H=720, W=1280, q=10,
              block=64, sigma=0.02, sp=0.0, w_logu=(10.0, 1e3), seed=0),
}


def scaled(cfg: Config, H: int, W: int, name: Optional[str] = None) -> Config:
    """Same scene recipe on a smaller frame (parity-size stand-ins of configs 4/5)."""
    return dataclasses.replace(cfg, name=name or f"{cfg.name}_{H}x{W}", H=H, W=W, m=H * W)


# --------------------------------------------------------------------------- scene
def _scene_params(cfg: Config):
    """Small per-scene draws: illumination scales, block path and block values."""
    rng = np.random.default_rng([cfg.seed, 0])
    c = rng.uniform(0.9, 1.1, size=(cfg.q, cfg.n))            # per-frame illumination
    x0 = int(rng.integers(0, cfg.W - cfg.block + 1))
    y0 = int(rng.integers(0, cfg.H - cfg.block + 1))
    vels = np.array([-3, -2, -1, 1, 2, 3])
    vx = int(vels[rng.integers(0, 6)])
    vy = int(vels[rng.integers(0, 6)])
    vals = rng.uniform(0.0, 1.0, size=cfg.n)                   # block value per frame
    # bouncing trajectory of the top-left corner, one position per foreground frame
    xs = np.zeros(cfg.n, dtype=np.int64)
    ys = np.zeros(cfg.n, dtype=np.int64)
    x, y = x0, y0
    for j in range(cfg.k, cfg.n):
        xs[j], ys[j] = x, y
        x, vx = _bounce(x, vx, cfg.W - cfg.block)
        y, vy = _bounce(y, vy, cfg.H - cfg.block)
    return c, xs, ys, vals


def _bounce(p: int, v: int, hi: int):
    p2 = p + v
    if p2 < 0:
        p2, v = -p2, -v
    elif p2 > hi:
        p2, v = 2 * hi - p2, -v
    return min(max(p2, 0), hi), v


def _basis(cfg: Config, rows: np.ndarray) -> np.ndarray:
    """Background images phi_l evaluated at pixel rows (len(rows) x q)."""
    yy = rows // cfg.W
    xx = rows % cfg.W
    xh = xx / max(cfg.W - 1, 1)
    yh = yy / max(cfg.H - 1, 1)
    phi = np.empty((rows.size, cfg.q))
    phi[:, 0] = 0.3 + 0.4 * (0.6 * xh + 0.4 * yh)
    for l in range(1, cfg.q):
        a, b = _COS_FREQS[l - 1]
        phi[:, l] = 0.1 * np.cos(np.pi * a * xh) * np.cos(np.pi * b * yh)
    return phi


def _scene_rows(cfg: Config, r0: int, r1: int, params) -> np.ndarray:
    c, xs, ys, vals = params
    out = np.empty((r1 - r0, cfg.n), dtype=cfg.np_dtype)
    for c0 in range((r0 // CHUNK_ROWS) * CHUNK_ROWS, r1, CHUNK_ROWS):
        c1 = min(c0 + CHUNK_ROWS, cfg.m)
        rows = np.arange(c0, c1)
        blk = _basis(cfg, rows) @ c                                 # rank-q background
        db = np.arange(cfg.block)
        for j in range(cfg.k, cfg.n):                               # foreground frames k..n-1
            pix = ((ys[j] + db)[:, None] * cfg.W + (xs[j] + db)[None, :]).ravel()
            pix = pix[(pix >= c0) & (pix < c1)]
            blk[pix - c0, j] = vals[j]
        rng = np.random.default_rng([cfg.seed, 1, c0 // CHUNK_ROWS])
        blk += cfg.sigma * rng.standard_normal(blk.shape)
        np.clip(blk, 0.0, 1.0, out=blk)
        if cfg.sp > 0.0:                                            # salt & pepper, A2 only
            hit = rng.random((c1 - c0, cfg.n - cfg.k)) < cfg.sp
            salt = rng.random((c1 - c0, cfg.n - cfg.k)) < 0.5
            a2 = blk[:, cfg.k:]
            a2[hit] = salt[hit].astype(np.float64)
        lo, hi = max(r0, c0), min(r1, c1)
        out[lo - r0:hi - r0] = blk[lo - c0:hi - c0]
    return out


def _lowrank_rows(cfg: Config) -> np.ndarray:
    rng = np.random.default_rng(cfg.seed)
    U = rng.standard_normal((cfg.m, cfg.r))
    V = rng.standard_normal((cfg.r, cfg.n))
    noise = rng.standard_normal((cfg.m, cfg.n))
    return (U @ V + 0.01 * noise).astype(cfg.np_dtype)


def make_A(cfg: Config, r0: int = 0, r1: Optional[int] = None) -> np.ndarray:
    """Rows [r0, r1) of the m x n data matrix A = (A1 A2), C-contiguous, cfg dtype."""
    r1 = cfg.m if r1 is None else r1
    if cfg.kind == "lowrank":
        return np.ascontiguousarray(_lowrank_rows(cfg)[r0:r1])
    return _scene_rows(cfg, r0, r1, _scene_params(cfg))


def make_background(cfg: Config, r0: int = 0, r1: Optional[int] = None) -> np.ndarray:
    """Rows [r0, r1) of the clean background of a scene config: the rank-q illumination-
    modulated part of make_A before the foreground block, the noise, the clipping and the
    salt-and-pepper (the ground truth of SURVEY.md §8(f4) / SPEC.md's generate_scene)."""
    if cfg.kind == "lowrank":
        raise ValueError("the low-rank config has no background ground truth")
    r1 = cfg.m if r1 is None else r1
    c = _scene_params(cfg)[0]
    return (_basis(cfg, np.arange(r0, r1)) @ c).astype(np.float64)


def make_W1(cfg: Config, r0: int = 0, r1: Optional[int] = None) -> Optional[np.ndarray]:
    """Rows [r0, r1) of W1 (m x k, entries > 0), or None when W1 is uniform
    (then ``cfg.w_const`` is the scalar weight)."""
    r1 = cfg.m if r1 is None else r1
    if cfg.uniform_w:
        return None
    lo, hi = cfg.w_logu
    out = np.empty((r1 - r0, cfg.k), dtype=cfg.np_dtype)
    for c0 in range((r0 // CHUNK_ROWS) * CHUNK_ROWS, r1, CHUNK_ROWS):
        c1 = min(c0 + CHUNK_ROWS, cfg.m)
        rng = np.random.default_rng([cfg.seed + 1, 2, c0 // CHUNK_ROWS])
        w = np.exp(rng.uniform(math.log(lo), math.log(hi), size=(c1 - c0, cfg.k)))
        a, b = max(r0, c0), min(r1, c1)
        out[a - r0:b - r0] = w[a - c0:b - c0]
    return out


def dense_W1(cfg: Config, W1: Optional[np.ndarray], rows: int) -> np.ndarray:
    """W1 as an explicit rows x k float64 array (uniform configs expanded)."""
    if W1 is None:
        return np.full((rows, cfg.k), float(cfg.w_const))
    return W1.astype(np.float64)


def random_x1(m: int, k: int, seed: int, dtype=np.float64) -> np.ndarray:
    """Random-Gaussian X1_0 ("initialize X1 as a random matrix";
    SPEC.md:247 RandomGaussian), drawn on the host so both sides see the same bits."""
    rng = np.random.default_rng([seed, 3])
    return rng.standard_normal((m, k)).astype(dtype)


def shard_rows(m: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous pixel-row block [r0, r1) of ``rank`` among ``world`` (ceil split;
    the last shard may be shorter).  SURVEY.md §8(e)."""
    per = -(-m // world)
    r0 = min(rank * per, m)
    return r0, min(r0 + per, m)
