"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same
seeded inputs, same initialisation and same iteration count (BASELINE.json north_star
tolerances, see tests/gpu_util.py)."""
import dataclasses

import numpy as np
import pytest

import oracle
import synth
from tests import gpu_util as gu

pytestmark = pytest.mark.gpu


def test_config1_tiny_fp64_full_run():
    cfg = synth.CONFIGS[1]
    A, W1 = gu.inputs(cfg)
    g = gu.run_gpu(cfg, A, W1, cfg.iters)
    o = gu.run_oracle(cfg, A, W1, cfg.iters)
    gu.compare(cfg, g, o)


def test_config1_host_buffers_match_device_buffers():
    """wlr_init with HOST A (copied by the library) == device A (borrowed)."""
    cfg = synth.CONFIGS[1]
    A, W1 = gu.inputs(cfg)
    g_dev = gu.run_gpu(cfg, A, W1, 10, device=True)
    g_host = gu.run_gpu(cfg, A, W1, 10, device=False)
    np.testing.assert_array_equal(g_dev["X1"], g_host["X1"])
    np.testing.assert_array_equal(g_dev["trace"], g_host["trace"])


def test_config2_small_fp32_full_run():
    cfg = synth.CONFIGS[2]
    A, W1 = gu.inputs(cfg)
    g = gu.run_gpu(cfg, A, W1, cfg.iters)
    o = gu.run_oracle(cfg, A, W1, cfg.iters)
    gu.compare(cfg, g, o)


@pytest.mark.parametrize("tensor_cores", [True, False])
def test_config2_row_pass_paths(tensor_cores):
    """Uniform-weight fp32: the tcgen05 3xTF32 row pass (default) and the CUDA-core FP32 row
    pass each meet the parity bar; the tensor-core path is the one active by default."""
    cfg = synth.CONFIGS[2]
    A, W1 = gu.inputs(cfg)
    g = gu.run_gpu(cfg, A, W1, cfg.iters, tensor_cores=tensor_cores)
    assert g["tensor_cores"] == tensor_cores
    o = gu.run_oracle(cfg, A, W1, cfg.iters)
    gu.compare(cfg, g, o)


def test_row_pass_tensor_core_ragged_tail():
    """m not a multiple of the 64-row tensor-core tile, k = r - 1 < 32, n ragged vs the
    32-column chunk: tensor-core path against the oracle."""
    g0 = np.random.default_rng(5)
    m, n, k, r = 1000 + 37, 75, 13, 15
    A = (g0.standard_normal((m, 16)) @ g0.standard_normal((16, n)) + 0.02 * g0.standard_normal((m, n)))
    cfg = dataclasses.replace(synth.CONFIGS[2], m=m, n=n, k=k, r=r, w_const=30.0, iters=12)
    A = A.astype(np.float32)
    g = gu.run_gpu(cfg, A, None, cfg.iters)
    assert g["tensor_cores"]
    o = gu.run_oracle(cfg, A, None, cfg.iters)
    gu.compare(cfg, g, o)


def test_row_pass_tensor_core_one_tile_per_sm_plus_leftover_rows():
    """m just above one 128-row tile per SM (the config-3 regime: 150 tiles on 148 SMs): every
    CTA takes one tile on the tensor cores plus <= 4 leftover rows on the CUDA cores; the last
    CTA's leftover block is ragged."""
    import torch
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    g0 = np.random.default_rng(6)
    m, n, k, r = nsm * 128 + nsm + 37, 70, 13, 15
    A = (g0.standard_normal((m, 12)) @ g0.standard_normal((12, n)) + 0.02 * g0.standard_normal((m, n)))
    cfg = dataclasses.replace(synth.CONFIGS[2], m=m, n=n, k=k, r=r, w_const=30.0, iters=6)
    A = A.astype(np.float32)
    g = gu.run_gpu(cfg, A, None, cfg.iters)
    assert g["tensor_cores"]
    o = gu.run_oracle(cfg, A, None, cfg.iters)
    gu.compare(cfg, g, o)


def test_step0_is_ghs_on_gpu():
    """p = 0 is the Theorem 1 closed form on the GPU too (pin P1 path)."""
    cfg = synth.CONFIGS[2]
    A, W1 = gu.inputs(cfg)
    g = gu.run_gpu(cfg, A, W1, 0)
    o = gu.run_oracle(cfg, A, W1, 0)
    gu.compare(cfg, g, o)
    np.testing.assert_array_equal(g["X1"], A[:, : cfg.k])       # X1_0 = A1 exactly


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_ragged_odd_shapes(dtype):
    """n not a multiple of 4 (scalar load paths), k not a multiple of 4, m ragged vs the
    128-row tile, r - k = 1 (the paper's r = k + 1), non-uniform W1."""
    g0 = np.random.default_rng(21)
    m, n, k, r = 517, 37, 7, 8
    A = (g0.standard_normal((m, 9)) @ g0.standard_normal((9, n)) + 0.05 * g0.standard_normal((m, n)))
    W1 = g0.uniform(1.0, 30.0, size=(m, k))
    dt = np.float64 if dtype == "f64" else np.float32
    A, W1 = A.astype(dt), W1.astype(dt)
    cfg = synth.Config("ragged", m, n, k, r, dtype, 12, "lowrank", w_const=None, w_logu=(1, 30))
    g = gu.run_gpu(cfg, A, W1, 12)
    o = gu.run_oracle(cfg, A, W1, 12)
    gu.compare(cfg, g, o)


def test_paper_rank_setting_k15_r16_uniform():
    """k = 15, r = k + 1 (Basic sequence) on a small scene, uniform W1."""
    cfg = dataclasses.replace(synth.scaled(synth.CONFIGS[3], 48, 64), k=15, r=16, n=120, iters=20)
    A, W1 = gu.inputs(cfg)
    g = gu.run_gpu(cfg, A, W1, cfg.iters)
    o = gu.run_oracle(cfg, A, W1, cfg.iters)
    gu.compare(cfg, g, o)


def test_random_init_given_x1():
    """INIT_GIVEN with a host-drawn Gaussian X1_0 (PAPER.md:234 random initialisation)."""
    cfg = dataclasses.replace(synth.scaled(synth.CONFIGS[2], 30, 40), iters=15)
    A, W1 = gu.inputs(cfg)
    x0 = synth.random_x1(cfg.m, cfg.k, seed=5, dtype=np.float32)
    g = gu.run_gpu(cfg, A, W1, cfg.iters, init="given", x1_0=x0)
    o = gu.run_oracle(cfg, A, W1, cfg.iters, x1_0=x0.astype(np.float64))
    gu.compare(cfg, g, o)


def test_exactly_representable_gives_zero_objective():
    """rank(A) <= r with full-rank A1 => F -> 0; S = 0 degenerate eigenproblem."""
    g0 = np.random.default_rng(3)
    A = (g0.standard_normal((300, 6)) @ g0.standard_normal((6, 40))).astype(np.float64)
    cfg = synth.Config("rankr", 300, 40, 4, 6, "f64", 5, "lowrank", w_const=7.0)
    g = gu.run_gpu(cfg, A, None, 5)
    # F = f_w + ||A2||^2 - <M', C'> - sum(lambda) cancels O(||A2||^2) terms, so
    # "F -> 0" means F at the fp64 rounding floor, |F| <= ~45 eps ||A||^2
    assert abs(g["trace"][-1, 0]) <= 1e-14 * np.sum(A * A)


def test_errors_are_explicit():
    w = gu.need_gpu()
    import torch
    A = torch.rand(200, 30, dtype=torch.float32, device="cuda")
    with pytest.raises(w.WlrError) as e:
        w.wlr_init(A, 5, 5)                                  # r = k
    assert e.value.status == 1
    W1 = torch.ones(200, 5, dtype=torch.float32, device="cuda")
    W1[3, 2] = 0.0
    with pytest.raises(w.WlrError) as e:
        w.wlr_init(A, 5, 7, W1)                              # W1 > 0
    assert e.value.status == 1
    B = A.clone()
    B[7, 9] = float("nan")
    with pytest.raises(w.WlrError) as e:
        w.wlr_init(B, 5, 7)
    assert e.value.status == 5
    C = A.clone()
    C[:, 1] = C[:, 0]                                        # rank(A1) < k
    with pytest.raises(w.WlrError) as e:
        w.wlr_init(C, 5, 7)
    assert e.value.status == 2


def test_stopping_rule_eps():
    """eps > 0 stops on Error_p < eps or rel < eps like the oracle."""
    cfg = synth.CONFIGS[1]
    A, W1 = gu.inputs(cfg)
    eps = 1e-7
    w = gu.need_gpu()
    import torch
    h = w.wlr_init(torch.from_numpy(A).cuda(), cfg.k, cfg.r, None, w1=cfg.w_const, eps=eps)
    done, conv = w.wlr_iterate(h, 100)
    o = oracle.swlr(A, synth.dense_W1(cfg, W1, cfg.m), cfg.k, cfg.r, iters=100, eps=eps)
    assert conv and o.converged
    assert done == len(o.trace) - 1, (done, len(o.trace) - 1)


@pytest.mark.parametrize("ci,check_every", [(1, 1), (1, 8), (3, 8), (2, 3)])
def test_stopping_rule_on_device(ci, check_every):
    """eps > 0: the stopping rule (R3) is applied on the device -- the iterations
    launched after the first state that satisfies it do no work -- so the returned state is that
    state whatever the host's check period, and further wlr_iterate calls leave it unchanged."""
    import torch
    w = gu.need_gpu()
    cfg = synth.CONFIGS[ci]
    A, W1 = gu.inputs(cfg)
    eps = 1e-7
    h = w.wlr_init(torch.from_numpy(A).cuda(), cfg.k, cfg.r, None, w1=cfg.w_const, eps=eps,
                   check_every=check_every)
    done, conv = w.wlr_iterate(h, 100)
    o = oracle.swlr(A.astype(np.float64), synth.dense_W1(cfg, W1, cfg.m), cfg.k, cfg.r, iters=100, eps=eps)
    assert conv and o.converged
    assert done == len(o.trace) - 1, (done, len(o.trace) - 1)
    tr = w.wlr_trace(h)
    assert tr.shape[0] == done + 1
    F = w.wlr_objective(h)[0]
    X1 = w.wlr_result(h)["X1"].copy()
    more, conv2 = w.wlr_iterate(h, 10)
    assert more == 0 and conv2
    assert w.wlr_objective(h)[0] == F
    np.testing.assert_array_equal(w.wlr_result(h)["X1"], X1)
    assert abs(F - o.trace[-1]["F"]) <= gu.TOL_F[cfg.dtype] * abs(o.trace[-1]["F"])


@pytest.mark.parametrize("m,n,k,r", [
    (2049, 110, 40, 44),     # KPD 64
    (2517, 130, 70, 73),     # KPD 96, r - k = 3
    (3037, 150, 90, 94),     # KPD 96, ragged m
])
def test_nonuniform_tensor_core_increments(m, n, k, r):
    """Non-uniform fp32 W1 (log-uniform) at k = 40..90: the tcgen05 E-mode row pass
    (linear part, the per-row solver adds A1 . W1^2), the warp-per-row Cholesky and the tcgen05
    increments with a KPD = 64 / 96 wide Delta^T operand (4 x 4 register-block transpose) once the
    X1 step is small (the gate); against the fp64 oracle over 20 iterations."""
    w = gu.need_gpu()
    g0 = np.random.default_rng(3 + k)
    # rank r - 1 plus noise: the iteration settles within a few steps (relative X1 step ~3e-5), so the
    # gate (||Delta||^2 <= 1e-6 ||X1||^2) opens and most iterations run the tensor-core increments
    A = (g0.standard_normal((m, r - 1)) @ g0.standard_normal((r - 1, n)) + 0.1 * g0.standard_normal((m, n)))
    W1 = np.exp(g0.uniform(0.0, np.log(30.0), size=(m, k)))
    A, W1 = A.astype(np.float32), W1.astype(np.float32)
    cfg = synth.Config("nonuniform_tc", m, n, k, r, "f32", 20, "lowrank", w_const=None, w_logu=(1, 30))
    g = gu.run_gpu(cfg, A, W1, 20)
    gate = w.wlr_debug_state(g["handle"], "gate")
    assert g["tensor_cores"] and gate[0] == 1.0 and gate[2] == (64 if k <= 64 else 96)
    assert gate[1] == 1.0, "the tensor-core increments never engaged (X1 step never small)"
    o = gu.run_oracle(cfg, A.astype(np.float64), W1.astype(np.float64), 20)
    gu.compare(cfg, g, o)
