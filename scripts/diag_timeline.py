"""Diagnostic: GPU timeline of a few bench steps (config 3, CUDA graph + PDL as in bench.py) from
the CUPTI kernel records of torch.profiler: start offset and duration of every kernel of the step,
and the gaps between them.  (Profiler timing, not a bench number.)"""
import json
import os
import sys
import tempfile

sys.path.insert(0, ".")
import torch
import synth
import paper_1703_06303_b200 as w

cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
NOFLUSH = "noflush" in sys.argv[2:]          # warm L2 (kernel durations without the cold-cache cost)
NOSYNC = "nosync" in sys.argv[2:]            # as bench.py: no host synchronisation between flush and step
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
A = torch.from_numpy(synth.make_A(cfg)).cuda()
W1n = synth.make_W1(cfg)
W1 = None if W1n is None else torch.from_numpy(W1n).cuda()
h = w.wlr_init(A, cfg.k, cfg.r, W1, w1=cfg.w_const or 1.0, stream=stream.cuda_stream)
w.wlr_row_path(h, True)
w.wlr_incr_path(h, True)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
w.wlr_iterate_async(h, 20)
torch.cuda.synchronize()
marks = []
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for i in range(6):
        if not NOFLUSH:
            flush.fill_(float(i))
        else:
            flush[:1].fill_(float(i))      # (a step marker kernel only)
        if not NOSYNC:
            torch.cuda.synchronize()
        w.wlr_iterate_async(h, 1)
        if not NOSYNC:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "trace.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
ks = [e for e in ev if e.get("cat") == "kernel"]
ks.sort(key=lambda e: e["ts"])
# split into steps at the fill kernels
steps, cur, fills = [], [], []
for e in ks:
    if "fill" in e["name"] or "elementwise" in e["name"].lower():
        if cur:
            steps.append(cur)
        cur = []
        fills.append(e)
        continue
    cur.append(e)
if cur:
    steps.append(cur)
for si, st in enumerate(steps[1:], 1):
    t0 = st[0]["ts"]
    end = max(e["ts"] + e["dur"] for e in st)
    fe = fills[si]["ts"] + fills[si]["dur"] if si < len(fills) else t0
    print(f"step {si}: span {end - t0:.1f} us (flush end -> first kernel {t0 - fe:.1f} us)")
    for e in st:
        nm = e["name"].replace("wlr::", "")[:48]
        print(f"   {e['ts'] - t0:7.1f} +{e['dur']:6.1f}  end {e['ts'] + e['dur'] - t0:7.1f}  stream {e['args'].get('stream')}  {nm}")
