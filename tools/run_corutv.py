"""Run one workload's CoR-UTV a few times (for ncu launch lists / timelines)."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1906_04572_b200 as P
import bench
wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
m, n, ell, q = bench.WORKLOADS[wl][:4]
torch.cuda.set_device(0)
a = bench.gen_rows_device(torch, wl, 0, m, torch.device("cuda", 0))
om = torch.from_numpy(P.gaussian_matrix(n, ell, 0)).cuda()
cfg = P.SketchConfig(ell=ell, q_power=q)
for _ in range(reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    P.corutv(a, cfg, omega=om)
    torch.cuda.synchronize(); print("%.3f ms" % ((time.perf_counter() - t0) * 1e3))
