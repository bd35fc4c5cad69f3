import sys, dataclasses, numpy as np
sys.path.insert(0, ".")
import torch, synth
from tests import gpu_util as gu
nsm = torch.cuda.get_device_properties(0).multi_processor_count
g0 = np.random.default_rng(6)
m, n, k, r = nsm * 128 + nsm + 37, 70, 13, 15
A = (g0.standard_normal((m, 12)) @ g0.standard_normal((12, n)) + 0.02 * g0.standard_normal((m, n))).astype(np.float32)
cfg = dataclasses.replace(synth.CONFIGS[2], m=m, n=n, k=k, r=r, w_const=30.0, iters=6)
for it in (1, 6):
    g = gu.run_gpu(cfg, A, None, it)
    o = gu.run_oracle(cfg, A, None, it)
    X = g["X1"].astype(np.float64); Xo = o.x1
    if Xo is None:
        print(o.keys()); break
    err = np.abs(X - Xo).max(axis=1) / np.abs(Xo).max()
    mm = nsm * 128
    print(f"iters {it}: max row err tiles {err[:mm].max():.3e}  extra rows {err[mm:].max():.3e}  worst extra row {mm + err[mm:].argmax()}")
