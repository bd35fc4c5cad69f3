"""Row-pass kernel time only (tensor-core path), for the WLR_TC_DBG experiments."""
import sys, os
sys.path.insert(0, ".")
import torch
import synth
import paper_1703_06303_b200 as w
cfg = synth.CONFIGS[3]
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
A = torch.from_numpy(synth.make_A(cfg)).cuda()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
h = w.wlr_init(A, cfg.k, cfg.r, None, w1=cfg.w_const, stream=stream.cuda_stream)
w.wlr_iterate_async(h, 5); torch.cuda.synchronize()
for fl in (False, True):
    w.wlr_profile(h, enable=True, reset=True)
    for i in range(20):
        if fl: flush.fill_(float(i))
        w.wlr_iterate_async(h, 1)
    pr = w.wlr_profile(h, enable=False, reset=False)
    print("dbg", os.environ.get("WLR_TC_DBG", "0"), "flush" if fl else "noflush", "row_pass %.1f us" % (pr["row_pass"] / pr["iters"] * 1e3))
