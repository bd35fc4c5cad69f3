"""World-size-2 host-side tests of the row-sharded (N > 1) path on CPU with the gloo backend
(DESIGN.md §7).  The library's data-path collective is one fp64 allreduce of
Gram partials that are additive over pixel rows (rows are independent given
(C_p, D_p)); these tests check the host logic around it: contiguous shards cover the rows,
every rank generates exactly its rows of the global scene, the summed per-shard partials equal
the single-process Grams, and bench.py's reference arm runs on rank 0 only under torchrun."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("m,world", [(300, 2), (300, 8), (19200, 8), (4800, 3), (7, 4)])
def test_shards_partition_rows(m, world):
    seen = []
    for r in range(world):
        r0, r1 = synth.shard_rows(m, world, r)
        assert 0 <= r0 <= r1 <= m
        seen.extend(range(r0, r1))
    assert seen == list(range(m))


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.scaled(synth.CONFIGS[4], 24, 32)            # non-uniform W1 recipe, m = 768
    r0, r1 = synth.shard_rows(cfg.m, world, rank)
    A = synth.make_A(cfg, r0, r1).astype(np.float64)
    W1 = synth.make_W1(cfg, r0, r1).astype(np.float64)
    full = synth.make_A(cfg)
    ok_rows = bool(np.array_equal(A, full[r0:r1].astype(np.float64)))
    ok_w = bool(np.array_equal(W1, synth.make_W1(cfg)[r0:r1].astype(np.float64)))
    # per-shard partial Grams at the GHS start (X1_0 = A1): [X1^T X1 | X1^T A2], A2^T A2, ||A2||^2
    x1, a2 = A[:, :cfg.k], A[:, cfg.k:]
    part = np.concatenate([(x1.T @ x1).ravel(), (x1.T @ a2).ravel(), (a2.T @ a2).ravel(),
                           [np.sum(a2 * a2)]])
    t = torch.from_numpy(part.copy())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)                # the library's exchange step (gloo here)
    # max-over-ranks timing reduction as bench.py does it
    tm = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    if rank == 0:
        Af = full.astype(np.float64)
        X1, A2 = Af[:, :cfg.k], Af[:, cfg.k:]
        ref = np.concatenate([(X1.T @ X1).ravel(), (X1.T @ A2).ravel(), (A2.T @ A2).ravel(),
                              [np.sum(A2 * A2)]])
        rel = float(np.max(np.abs(t.numpy() - ref)) / np.max(np.abs(ref)))
        np.save(out, np.array([rel, tm.item()]))
    flags = torch.tensor([int(ok_rows), int(ok_w)])
    dist.all_reduce(flags, op=dist.ReduceOp.MIN)
    if rank == 0:
        np.save(out + ".flags.npy", flags.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_partials_sum_to_global(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "res.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    rel, tmax = np.load(out)
    flags = np.load(out + ".flags.npy")
    assert flags.tolist() == [1, 1]          # each rank generated exactly its global rows
    assert rel < 1e-13                       # fp64 partial sums == single-process Grams
    assert tmax == 2.0                       # max over ranks


def test_bench_reference_arm_under_torchrun_two_ranks():
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
           "--warmup", "0", "--config", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                   # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle"
