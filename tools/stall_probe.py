"""Find the occasional ~200 ms stalls of back-to-back C3 calls: torch.profiler
timeline of 6 corutv calls, largest idle gaps between device activities."""
import sys
import time
sys.path.insert(0, '.')
import torch
from torch.profiler import ProfilerActivity, profile
import bench
import paper_1906_04572_b200 as P
torch.cuda.set_device(0)
a = bench.gen_rows_device(torch, "c3", 0, 131072, torch.device("cuda", 0))
cfg = P.SketchConfig(ell=110, q_power=2)
P.corutv(a, cfg)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.corutv(a, cfg)
        torch.cuda.synchronize()
        print(f"call {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA" and e.device_time_total > 0],
            key=lambda e: e.time_range.start)
gaps = []
for x, y in zip(ev, ev[1:]):
    g = y.time_range.start - x.time_range.end
    gaps.append((g, x.name[:50], y.name[:50]))
gaps.sort(reverse=True)
for g, x, y in gaps[:12]:
    print(f"gap {g / 1e3:8.2f} ms after {x} before {y}")
cpu = sorted([e for e in prof.events() if e.device_type.name == "CPU"], key=lambda e: -e.cpu_time_total)
for e in cpu[:10]:
    print(f"cpu {e.cpu_time_total / 1e3:8.2f} ms {e.name[:60]}")
