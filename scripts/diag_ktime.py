"""Diagnostic: K3 phase timestamps (globaltimer, CTA 0) for one steady-state iteration.
The timestamps of the last launched small-step half are recorded (the critical half K3a for
part=1; wlr_sync flushes the deferred half, so read before syncing)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
import synth
import paper_1703_06303_b200 as w

FLUSH = torch.empty(0)

def run(ci, warm=8, H=None, Wd=None, flush=False):
    cfg = synth.CONFIGS[ci]
    if H:
        cfg = synth.scaled(cfg, H, Wd)
    A = torch.from_numpy(synth.make_A(cfg)).cuda()
    W1n = synth.make_W1(cfg)
    W1 = None if W1n is None else torch.from_numpy(W1n).cuda()
    h = w.wlr_init(A, cfg.k, cfg.r, W1, w1=cfg.w_const or 1.0)
    w.wlr_iterate(h, warm)
    w.wlr_debug_state(h, "ktime_on")
    for rep in range(3):
        if flush:
            FLUSH.fill_(float(rep))
            torch.cuda.synchronize()
        w.wlr_iterate_async(h, 1)
        torch.cuda.synchronize()
        kt = w.wlr_debug_state(h, "ktime")   # [0:64] K3a(p), [64:128] K3b(p-1) (ran beside it)
        for name, off in (("K3a", 0), ("K3b", 64)):
            n = int(kt[off])
            ts = kt[off + 1:off + 1 + n]
            ck = kt[off + 32:off + 32 + n]
            if n < 2:
                continue
            d = np.diff(ts) / 1e3
            mhz = (ck[-1] - ck[0]) / max(ts[-1] - ts[0], 1) * 1e3
            print(f"cfg{ci}{'F' if flush else ''} {name} total={(ts[-1]-ts[0])/1e3:.1f}us clk={mhz:.0f}MHz phases(us)=" + " ".join(f"{x:.1f}" for x in d))
            xb = kt[128 + off: 128 + off + 32]
            xb = xb[xb > 0]
            if len(xb):
                print(f"   {name} exchange barrier releases (us from start): " +
                      " ".join(f"{(x - ts[0]) / 1e3:.1f}" for x in xb) +
                      " | marks: " + " ".join(f"{(x - ts[0]) / 1e3:.1f}" for x in ts))
        if name == "K3a" or True:
            pass
        print(f"   K3a: Jacobi {kt[240] / 1.9e3:.1f} us in {kt[241]:.0f} calls, filter products {kt[242] / 1.9e3:.1f} us, "
              f"S-products {kt[243]:.0f}, outer {kt[244]:.0f}  (cycles / 1.9 GHz); Jacobi warp alone {kt[245] / 1.9e3:.1f} us, "
              f"K^-1 warps {kt[246] / 1.9e3:.1f} us (last call)")
        if kt[167] > 0:
            print("   EXP NS#1 start %.1f end %.1f restore %.1f (us from K3a start)" % tuple((kt[i] - kt[1]) / 1e3 for i in (167, 168, 169)))
        t0a, t0b = kt[1], kt[65]
        if int(kt[64]) > 1:
            print(f"   K3b start - K3a start = {(t0b - t0a)/1e3:.1f}us")


for c in (sys.argv[1:] or ["1", "2", "3", "4"]):
    if c.startswith("F"):               # "F3": flush L2 (256 MB write) before each iteration, as bench.py does
        FLUSH = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
        run(int(c[1:]), flush=True)
        continue
    if c == "4":
        run(4, H=120, Wd=160)
    elif c in ("4f", "5f"):                 # full-size configs 4 / 5
        run(int(c[0]))
    else:
        run(int(c))
