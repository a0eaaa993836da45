"""C4 RPCA only (bench_rpca), for launch lists / timelines."""
import sys, json
sys.path.insert(0, '.')
import torch
import paper_1906_04572_b200 as P
import bench
torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
out = bench.bench_rpca(torch, P, torch.device("cuda", 0)) if n == 10000 else None
print(json.dumps(out))
