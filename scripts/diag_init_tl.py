"""Diagnostic: CUPTI timeline (torch.profiler) of wlr_init from pinned host A and of wlr_result:
kernels and copies with their start offsets, to find the host-side gaps."""
import json, os, sys, tempfile
sys.path.insert(0, ".")
import torch
import synth
import paper_1703_06303_b200 as w
from torch.profiler import profile, ProfilerActivity
cfg = synth.CONFIGS[3]
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
Ah = torch.from_numpy(synth.make_A(cfg)).pin_memory()
h = w.wlr_init(Ah, cfg.k, cfg.r, None, w1=cfg.w_const, stream=stream.cuda_stream)
w.wlr_iterate(h, 3); w.wlr_result(h); w.wlr_destroy(h); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    h = w.wlr_init(Ah, cfg.k, cfg.r, None, w1=cfg.w_const, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    w.wlr_iterate(h, 2)
    torch.cuda.synchronize()
    res = w.wlr_result(h, x2=False)
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
gpu = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
gpu.sort(key=lambda e: e["ts"])
cpu = [e for e in ev if e.get("cat") == "cuda_runtime" and e.get("dur", 0) > 200]
t0 = min([e["ts"] for e in gpu] + [e["ts"] for e in cpu])
for e in gpu:
    print(f"GPU {e['ts'] - t0:9.1f} +{e['dur']:8.1f}  {e['name'][:70]}")
print("host runtime calls > 200 us:")
for e in sorted(cpu, key=lambda e: e["ts"]):
    print(f"CPU {e['ts'] - t0:9.1f} +{e['dur']:8.1f}  {e['name'][:70]}")
