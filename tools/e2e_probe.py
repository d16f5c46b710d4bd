"""PCIe probe for the e2e pipeline: pinned H2D / D2H bandwidth alone and
concurrent, and eg_compute_host on C3 for several chunk counts."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

n = 1 << 30
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
h2 = torch.empty(n, dtype=torch.float32).pin_memory()
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); a = time.perf_counter() - t
t = time.perf_counter(); h2.copy_(d2, non_blocking=True); torch.cuda.synchronize(); b = time.perf_counter() - t
t = time.perf_counter()
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); c = time.perf_counter() - t
print(f"H2D {4*n/a/1e9:.1f} GB/s  D2H {4*n/b/1e9:.1f} GB/s  both {8*n/c/1e9:.1f} GB/s ({c*1e3:.1f} ms)")
del d2, h2
import bench  # noqa: E402
import paper_2303_02724_b200 as eg  # noqa: E402
f, dims, _ = bench.make_input("C3", "cuda:0")
hf = f.cpu().pin_memory()
lab = torch.empty(f.numel(), dtype=torch.int32).pin_memory()
ctx = eg.Context(0)
for k in ["1", "16", "24", "32"]:
    os.environ["EG_E2E_CHUNKS"] = k
    ctx.compute_host(hf, dims=dims, labels_out=lab)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        ctx.compute_host(hf, dims=dims, labels_out=lab)
        ts.append(time.perf_counter() - t)
    print(f"chunks {k}: {min(ts)*1e3:.1f} ms  ({f.numel()/min(ts)/1e6:.0f} Mvert/s)  patched {ctx.stats()['n_exit_targets']}")
