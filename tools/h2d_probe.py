"""Host -> device copy rate of one AlexNet batch (128 x 3 x 224 x 224 fp32,
77 MB) from pinned memory, split over 1 / 2 / 4 / 8 streams, alone and
while a GEMM-heavy kernel stream runs (what train()'s input feed sees)."""
import torch

dev = torch.device("cuda", 0)
n = 128 * 3 * 224 * 224
h = torch.randn(n).pin_memory()
d = torch.empty(n, device=dev)
streams = [torch.cuda.Stream(dev) for _ in range(8)]


def run(ns, reps=10):
    chunks = [(i * n // ns, (i + 1) * n // ns) for i in range(ns)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        for s, (a, b) in zip(streams, chunks):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[a:b].copy_(h[a:b], non_blocking=True)
        for s in streams[:ns]:
            torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return ms, n * 4 / (ms / 1e3) / 1e9


for ns in (1, 2, 4, 8):
    ms, gbs = run(ns)
    print(f"h2d {ns} streams: {ms:.3f} ms  {gbs:.1f} GB/s", flush=True)
a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
busy = torch.cuda.Stream(dev)
with torch.cuda.stream(busy):
    for _ in range(200):
        a @ a
for ns in (1, 4):
    ms, gbs = run(ns)
    print(f"h2d {ns} streams under load: {ms:.3f} ms  {gbs:.1f} GB/s", flush=True)
torch.cuda.synchronize()
