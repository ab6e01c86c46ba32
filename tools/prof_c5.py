"""c5 shape on one GPU (N=1e8, D=128, K=4096 fp32): Gaussian blobs generated on
the device (same recipe as matrix.gaussian_mixture, torch RNG -- a perf run,
not a parity case), a few Lloyd steps through LloydEngine (graph replay)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2408_01391_b200 as P
from paper_2408_01391_b200 import _engine as E
from paper_2408_01391_b200.kmeans import LloydEngine

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
d, k = 128, 4096
ft = sys.argv[2] if len(sys.argv) > 2 else "off"
g = torch.Generator(device="cuda").manual_seed(0)
centers = torch.rand((k, d), generator=g, device="cuda", dtype=torch.float64) * 1.6
x = torch.empty((n, d), dtype=torch.float32, device="cuda")
ch = 1 << 22
for r0 in range(0, n, ch):
    r1 = min(n, r0 + ch)
    lab = torch.randint(0, k, (r1 - r0,), generator=g, device="cuda")
    x[r0:r1] = (centers[lab] + 0.25 * torch.randn((r1 - r0, d), generator=g, device="cuda",
                                                   dtype=torch.float64)).float()
idx = torch.randperm(n, generator=g, device="cuda")[:k]
c0 = x[idx].clone()
torch.cuda.synchronize()
t0 = time.perf_counter()
eng = LloydEngine(x, c0, k, np.float32, P.default_config(np.float32), ft,
                  P.Threshold.default_for(np.float32), 64, graph=True)
torch.cuda.synchronize()
print(f"engine init {time.perf_counter() - t0:.2f} s")
flops = 2.0 * n * d * k
for it in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    inertia, unch, moved = eng.step(it, eager=True)
    torch.cuda.synchronize()
    w = time.perf_counter() - t0
    fb = E.tc_fallback_rows()
    print(f"it {it}: {w * 1e3:.1f} ms ({1 / w:.2f} iter/s)  screen {E.tc_last_kernel_ms():.1f} ms "
          f"({flops / E.tc_last_kernel_ms() / 1e9:.0f} TF/s)  assign {eng.assign_ms:.1f} ms  "
          f"update {eng.update_ms:.1f} ms  fallback {fb}")
eng.close()
