"""the sWLR frames-vs-time sweep (analogue of PAPER.md Fig. 3(c), k = 15,
r = k + 1) on the QVGA scene (m = 19200 pixels, fp32, uniform W1 = 100),
n swept.  Per n: GHS init time, iterations/s of the fixed-count loop (device-resident A,
steps timed with CUDA events), and time-to-tolerance (eps = 1e-7, GHS init, max 300
iterations).  Same kernels as the bench; measurement only."""
import dataclasses
import json
import sys
import time

sys.path.insert(0, ".")
import torch
import synth
import paper_1703_06303_b200 as w

ns = [int(x) for x in sys.argv[1:]] or [32, 64, 128, 256, 400, 600, 800]
base = synth.CONFIGS[3]
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
rows = []
for n in ns:
    cfg = dataclasses.replace(base, name=f"qvga_k15_n{n}", n=n, k=15, r=16)
    A = torch.from_numpy(synth.make_A(cfg)).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = w.wlr_init(A, cfg.k, cfg.r, None, w1=cfg.w_const, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    t_init = (time.perf_counter() - t0) * 1e3
    w.wlr_iterate_async(h, 3)
    w.wlr_sync(h)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 50
    e0.record(stream)
    w.wlr_iterate_async(h, K)
    e1.record(stream)
    w.wlr_sync(h)
    ms_it = e0.elapsed_time(e1) / K
    w.wlr_destroy(h)
    # time to tolerance from GHS init (init excluded / included)
    h = w.wlr_init(A, cfg.k, cfg.r, None, w1=cfg.w_const, eps=1e-7, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    done, conv = w.wlr_iterate(h, 300)
    t_tol = (time.perf_counter() - t0) * 1e3
    F, step, rel = w.wlr_objective(h)
    w.wlr_destroy(h)
    row = {"n": n, "m": cfg.m, "k": cfg.k, "r": cfg.r, "init_ms": round(t_init, 3), "ms_per_iter": round(ms_it, 4),
           "iters_per_s": round(1e3 / ms_it, 1), "tol_eps": 1e-7, "tol_iters": done, "tol_converged": conv,
           "tol_ms": round(t_tol, 2), "tol_ms_incl_init": round(t_tol + t_init, 2), "F": F, "rel": rel}
    rows.append(row)
    print(json.dumps(row), flush=True)
# linear-growth check of SPEC.md:438: per-iteration time vs n within 2x of a linear fit through the largest n
big = rows[-1]
for r_ in rows:
    lin = big["ms_per_iter"] * r_["n"] / big["n"]
    r_["vs_linear"] = round(r_["ms_per_iter"] / lin, 2)
print("per-iteration time / linear-in-n model:", [(r_["n"], r_["vs_linear"]) for r_ in rows])
