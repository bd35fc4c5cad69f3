"""Write the oracle fixtures the full-size GPU parity tests compare against.

Calls only ``synth`` (seeded inputs) and ``oracle`` (fp64 Algorithm 1); nothing here touches the
CUDA path.  For each BASELINE.json config named on the command line it runs the oracle from the
GHS start (X1_0 = A1, R5) for the config's full iteration count (config 3: 200, config 4: 100,
config 5: 50) and stores

* the whole trace, one record per canonical state p = 0..N (R1, R11): F_p, F_mid, Error_p
  (``step``), rel_p = Error_p / ||X_p|| (R3), sigma_{r-k}, sigma_{r-k+1};
* X_N = (X1_N, X1_N C_N + D_N) on 1024 fixed sampled rows (plus rows 0 and m-1), as float32
  (the rounding, <= 6e-8 relative, is far below the 1e-4 parity bar);
* a fingerprint of the input (the fp64 sum of A and of W1, and A on 8 of the sampled rows), so
  a changed generator fails the test instead of comparing different problems.

Configs 3 and 4 (m < 1e5) run the literal oracle (``oracle.swlr``: QR + thin SVD); config 5 runs
``oracle.swlr_large`` (QR + eigh of the explicit P^T P, R22).

    python scripts/make_oracle_fixtures.py 3 4 --threads 3
    python scripts/make_oracle_fixtures.py 5 --threads 5
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

OUT = os.path.join(ROOT, "tests", "fixtures")
N_SAMPLE = 1024


def sample_rows(cfg):
    rng = np.random.default_rng([cfg.m, N_SAMPLE, 1703])
    rows = rng.choice(cfg.m, size=N_SAMPLE, replace=False)
    return np.unique(np.concatenate([rows, [0, cfg.m - 1]])).astype(np.int64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", type=int, nargs="+")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--iters", type=int, default=None, help="override (testing the script only)")
    args = ap.parse_args()
    from threadpoolctl import threadpool_limits

    import oracle
    import synth
    from oracle.swlr_large import swlr_large
    os.makedirs(OUT, exist_ok=True)
    for ci in args.configs:
        cfg = synth.CONFIGS[ci]
        iters = cfg.iters if args.iters is None else args.iters
        t0 = time.time()
        A = synth.make_A(cfg)
        W1 = synth.make_W1(cfg)
        tgen = time.time() - t0
        rows = sample_rows(cfg)
        log = open(os.path.join(OUT, f"oracle_cfg{ci}.log"), "w")

        def logrec(rec):
            log.write(json.dumps(rec) + f"  t={time.time() - t0:.1f}s\n")
            log.flush()
        t1 = time.time()
        if cfg.m >= 100_000:
            route = "swlr_large (QR + eigh(P^T P), R22)"
            with threadpool_limits(limits=1):
                res = swlr_large(A, W1, cfg.k, cfg.r, iters, w_const=cfg.w_const or 1.0,
                                 threads=args.threads, log=logrec)
            X = res.x_rows(rows)
            trace = res.trace
        else:
            route = "swlr (QR + thin SVD, literal)"
            with threadpool_limits(limits=args.threads):
                w1 = synth.dense_W1(cfg, W1, cfg.m)
                res = oracle.swlr(A.astype(np.float64), w1, cfg.k, cfg.r, iters=iters)
            X = res.x[rows]
            trace = res.trace
            for rec in trace:
                logrec(rec)
        trun = time.time() - t1
        keys = ["F", "F_mid", "step", "rel", "sig_t", "sig_t1"]
        tr = np.array([[rec.get(kk, np.nan) for kk in keys] for rec in trace])
        fp = dict(A_sum=float(np.sum(A, dtype=np.float64)),
                  W1_sum=None if W1 is None else float(np.sum(W1, dtype=np.float64)))
        np.savez_compressed(os.path.join(OUT, f"oracle_cfg{ci}.npz"), trace=tr,
                            trace_keys=np.array(keys), rows=rows, X_rows=X.astype(np.float32),
                            A_rows=A[rows[:8]].astype(np.float32))
        meta = dict(config=ci, name=cfg.name, m=cfg.m, n=cfg.n, k=cfg.k, r=cfg.r, iters=iters,
                    init="GHS (X1_0 = A1)", route=route, threads=args.threads,
                    seconds_generate=round(tgen, 1), seconds_oracle=round(trun, 1),
                    seconds_per_iteration=round(trun / max(iters, 1), 2),
                    host=platform.processor() or platform.machine(), fingerprint=fp,
                    written_by="scripts/make_oracle_fixtures.py (synth + oracle only)")
        with open(os.path.join(OUT, f"oracle_cfg{ci}.json"), "w") as f:
            json.dump(meta, f, indent=1)
        log.close()
        print(json.dumps(meta))


if __name__ == "__main__":
    main()
