"""Host<->device copy bandwidth on the box: one big pinned copy, chunked
copies on one / two streams, pageable copy, D2H."""
import time
import torch
torch.cuda.set_device(0)
GB = 1 << 30
n = 8 * GB // 8
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
big = t(lambda: d.copy_(h, non_blocking=True))
print(f"pinned H2D one copy 8 GiB: {8 * GB / big / 1e9:.1f} GB/s")
for chunk_mb in (64, 256, 1024):
    c = chunk_mb * (1 << 20) // 8
    def chunked():
        for o in range(0, n, c):
            d[o:o + c].copy_(h[o:o + c], non_blocking=True)
    dt = t(chunked)
    print(f"pinned H2D chunks {chunk_mb} MiB, 1 stream: {8 * GB / dt / 1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
c = 256 * (1 << 20) // 8
def two():
    for i, o in enumerate(range(0, n, c)):
        with torch.cuda.stream(s1 if i % 2 == 0 else s2):
            d[o:o + c].copy_(h[o:o + c], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
dt = t(two)
print(f"pinned H2D chunks 256 MiB, 2 streams: {8 * GB / dt / 1e9:.1f} GB/s")
dt = t(lambda: h.copy_(d, non_blocking=True))
print(f"pinned D2H one copy 8 GiB: {8 * GB / dt / 1e9:.1f} GB/s")
p = torch.empty(GB // 8, dtype=torch.float64)
p.fill_(1.0)
dt = t(lambda: d[:GB // 8].copy_(p))
print(f"pageable H2D 1 GiB: {GB / dt / 1e9:.1f} GB/s")
dt = t(lambda: p.copy_(d[:GB // 8]))
print(f"pageable D2H 1 GiB: {GB / dt / 1e9:.1f} GB/s")
