"""Write-only bandwidth ceiling for the advance output shape: fill 2 x 32 MiB
(scores f32 + next i32 for 8192 x 1024) per step, CUDA-graph replays,
CUDA events; compare with the measured copy peak."""
import json
import torch

dev = torch.device("cuda")
B, V = 8192, 1024
a = torch.empty(B * V, dtype=torch.float32, device=dev)
b = torch.empty(B * V, dtype=torch.int32, device=dev)
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]


def timed(fn, n=50):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / n)
    return best


bytes_ = 2 * B * V * 4
for name, fn in [("fill_ both", lambda: (a.fill_(1.0), b.fill_(3))),
                 ("zero_ both", lambda: (a.zero_(), b.zero_())),
                 ("one 64 MiB fill", lambda: torch.cat([a.view(-1)]).fill_(0) if False else a.view(torch.int32).fill_(7))]:
    ms = timed(fn)
    nb = bytes_ if "both" in name else B * V * 4
    print(name, f"{ms * 1e3:.2f} us", f"{nb / ms / 1e6:.0f} GB/s", f"{nb / ms / 1e6 / peak:.3f} of peak")
