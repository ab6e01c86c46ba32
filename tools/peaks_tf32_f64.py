"""Measured tensor-core denominators for the roofline: cuBLAS TF32 GEMM
(fp32 inputs, allow_tf32) and cuBLAS DGEMM, dense, on this GPU.  Best of 10
CUDA-event-timed launches after warm-up (burst) and the mean over ~3 s back
to back (sustained).  Writes profiles/peaks_tf32_f64.json."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def gemm_tflops(dtype, n, tf32):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps, t0 = 0, time.perf_counter()
    e0.record()
    while time.perf_counter() - t0 < 3.0:
        a @ b
        reps += 1
        if reps % 8 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    flops = 2.0 * n ** 3
    return flops / (best * 1e-3) / 1e12, flops * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12


torch.cuda.set_device(0)
tf_b, tf_s = gemm_tflops(torch.float32, 8192, True)
d_b, d_s = gemm_tflops(torch.float64, 8192, False)
out = {"tf32_tflops": tf_b, "tf32_tflops_sustained": tf_s, "f64_tflops": d_b,
       "f64_tflops_sustained": d_s, "gpu": torch.cuda.get_device_name(0),
       "how": "torch.matmul 8192^3 (2 n^3 flops): fp32 with allow_tf32 (cuBLAS TF32 tensor cores) and "
              "float64 (cuBLAS DGEMM); best of 10 CUDA-event-timed launches (burst), ~3 s back to back "
              "(sustained)"}
print(json.dumps(out))
if "--write" in sys.argv:
    with open(os.path.join(ROOT, "profiles", "peaks_tf32_f64.json"), "w") as fh:
        json.dump(out, fh, indent=1)
