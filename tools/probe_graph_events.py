"""Can CUDA events recorded inside a captured graph time its phases?
Captures: ev0, matmul A, ev1, matmul B, ev2 -- replays, prints elapsed."""
import torch

torch.cuda.set_device(0)
a = torch.randn(4096, 4096, device="cuda")
b = torch.randn(8192, 8192, device="cuda")
evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    a @ a; b @ b
    torch.cuda.synchronize()
    try:
        g.capture_begin()
        evs[0].record()
        c = a @ a
        evs[1].record()
        d = b @ b
        evs[2].record()
        g.capture_end()
        ok = True
    except Exception as e:  # noqa
        print("capture failed:", e)
        ok = False
torch.cuda.synchronize()
if ok:
    for _ in range(3):
        g.replay()
        torch.cuda.synchronize()
        try:
            print("A %.3f ms  B %.3f ms" % (evs[0].elapsed_time(evs[1]), evs[1].elapsed_time(evs[2])))
        except Exception as e:  # noqa
            print("elapsed failed:", e)
