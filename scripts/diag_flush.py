"""Diagnostic: per-kernel times with and without an L2 flush between iterations (cfg 3)."""
import sys
sys.path.insert(0, ".")
import torch
import synth
import paper_1703_06303_b200 as w

cfg = synth.CONFIGS[3]
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
A = torch.from_numpy(synth.make_A(cfg)).cuda()
h = w.wlr_init(A, cfg.k, cfg.r, None, w1=cfg.w_const, stream=stream.cuda_stream)
w.wlr_iterate(h, 10)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for mode in ["noflush", "flush", "flush+sleep"]:
    w.wlr_profile(h, enable=True, reset=True)
    for i in range(20):
        if mode != "noflush":
            flush.fill_(float(i))
        if mode == "flush+sleep":
            torch.cuda._sleep(2000000)
        w.wlr_iterate_async(h, 1)
    pr = w.wlr_profile(h, enable=False, reset=False)
    it = pr["iters"]
    print(mode, {k: round(v / it * 1e3, 1) for k, v in pr.items() if k not in ("launches", "iters")})
