"""Calibration runs for ncu's tensor-pipe utilisation metric: cuBLAS TF32
(fp32 + allow_tf32) and BF16 GEMMs at 8192^3, one launch each after warm-up.
Run under ncu with --metrics sm__pipe_tensor_cycles_active_realtime... to
relate the metric's percentage to achieved TF/s (the screen's 18-35 % is
read against what cuBLAS reaches on the same counter)."""
import torch

torch.cuda.set_device(0)
for dt, tf32 in ((torch.float32, True), (torch.bfloat16, False)):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(8192, 8192, device="cuda", dtype=dt)
    b = torch.randn(8192, 8192, device="cuda", dtype=dt)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    a @ b
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{dt} tf32={tf32}: {ms:.3f} ms = {2 * 8192 ** 3 / ms / 1e9:.0f} TF/s")
