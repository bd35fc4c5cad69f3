"""Bitwise A/B of an environment switch (read at wlr_init): config N for K iterations in a
subprocess per setting; prints F, the step trace and a digest of X1 and C, V for each.
Usage: python scripts/diag_bitwise_env.py VAR val0 val1 [config] [iters]"""
import hashlib, json, os, subprocess, sys

if sys.argv[1] == "run":
    sys.path.insert(0, ".")
    import numpy as np, torch, synth
    import paper_1703_06303_b200 as w
    cfg = synth.CONFIGS[int(sys.argv[2])]
    A = torch.from_numpy(synth.make_A(cfg)).cuda()
    W1n = synth.make_W1(cfg)
    W1 = None if W1n is None else torch.from_numpy(W1n).cuda()
    h = w.wlr_init(A, cfg.k, cfg.r, W1, w1=cfg.w_const or 1.0)
    w.wlr_iterate(h, int(sys.argv[3]))
    tr = np.asarray(w.wlr_trace(h))
    r = w.wlr_result(h, x2=False)
    dig = hashlib.sha1(b"".join(np.ascontiguousarray(r[k]).tobytes() for k in ("X1", "C", "B", "D"))).hexdigest()
    print(json.dumps({"trace_digest": hashlib.sha1(tr.tobytes()).hexdigest(), "F": float(tr[-1][0]), "result_digest": dig}))
    sys.exit(0)
var, vals = sys.argv[1], sys.argv[2:4]
cfg = sys.argv[4] if len(sys.argv) > 4 else "3"
iters = sys.argv[5] if len(sys.argv) > 5 else "30"
out = {}
for v in vals:
    p = subprocess.run([sys.executable, __file__, "run", cfg, iters], env=dict(os.environ, **{var: v}), capture_output=True, text=True)
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    out[v] = json.loads(lines[-1]) if lines else {"error": p.stderr[-800:]}
    print(var, v, out[v])
print("bitwise identical:", out[vals[0]] == out[vals[1]])
