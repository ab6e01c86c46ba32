"""cuBLAS DGEMM throughput on this GPU (calibrates the float64 roofline)."""
import torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    a @ b
torch.cuda.synchronize()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(5):
    st.record(); a @ b; en.record(); torch.cuda.synchronize()
    best = min(best, st.elapsed_time(en))
print(f"cuBLAS DGEMM {n}^3: {2 * n**3 / best / 1e9:.1f} TFLOP/s ({best:.2f} ms)")
x = torch.randn(2000000, 64, dtype=torch.float64, device="cuda")
c = torch.randn(256, 64, dtype=torch.float64, device="cuda")
for _ in range(3):
    x @ c.T
torch.cuda.synchronize()
st.record(); x @ c.T; en.record(); torch.cuda.synchronize()
ms = st.elapsed_time(en)
print(f"cuBLAS DGEMM c4 shape (2e6x64 @ 64x256): {2 * 2e6 * 64 * 256 / ms / 1e9:.1f} TFLOP/s ({ms:.2f} ms)")
