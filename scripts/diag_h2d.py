"""Host->device bandwidth from pinned memory (46 MB, the config-3 A) with torch, and the library's
init phases (scripts/diag_e2e.py covers the solve)."""
import sys, time
sys.path.insert(0, ".")
import torch
x = torch.empty(19200 * 600, dtype=torch.float32).pin_memory()
y = torch.empty_like(x, device="cuda")
for rep in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    y.copy_(x, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"H2D 46 MB pinned: {1e3 * (t1 - t0):.3f} ms = {x.numel() * 4 / (t1 - t0) / 1e9:.1f} GB/s")
