"""One-off: cuBLAS DGEMM (torch float64 matmul) and copy bandwidth on the box."""
import torch, time, json
d = torch.device("cuda:0")
res = {}
for nsz in (4096, 8192):
    a = torch.randn(nsz, nsz, dtype=torch.float64, device=d)
    b = torch.randn(nsz, nsz, dtype=torch.float64, device=d)
    for _ in range(2): torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[f"dgemm_{nsz}_tflops"] = 2 * nsz**3 / best / 1e9
# skinny shapes like the sketch: (m x n)(n x l)
for (m, n, l) in ((131072 // 4, 32768, 110), (4000, 3000, 50), (10000, 10000, 100)):
    a = torch.randn(m, n, dtype=torch.float64, device=d)
    x = torch.randn(n, l, dtype=torch.float64, device=d)
    y = torch.randn(m, l, dtype=torch.float64, device=d)
    for _ in range(2): a @ x; a.T @ y
    torch.cuda.synchronize()
    for name, f in (("NN", lambda: a @ x), ("TN", lambda: a.T @ y)):
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record(); e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        res[f"cublas_{name}_{m}x{n}x{l}_tflops"] = 2 * m * n * l / best / 1e9
    del a, x, y
x = torch.empty(1 << 30, dtype=torch.float64, device=d); y = torch.empty_like(x)
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); y.copy_(x); e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
res["copy_gbs"] = 2 * x.numel() * 8 / best / 1e6
print(json.dumps(res, indent=1))
