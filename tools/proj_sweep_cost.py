"""Marginal cost of one projection sweep at m = 16384 (diagnostic): time fastpfp_project with k
sweeps (sums pass + k sweeps, no finalize) for several k and fit time = a + b k."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1207_1114_b200 as F

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
g = torch.Generator(device="cuda").manual_seed(0)
Y0 = (torch.rand((m, m), device="cuda", generator=g) * 2.0 - 0.5).contiguous()
Y = torch.empty_like(Y0)
res = []
for k in (1, 2, 6, 11, 21):
    ts = []
    for rep in range(4):
        Y.copy_(Y0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        F.project(Y, 0.0, k, torch.cuda.current_stream().cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res.append((k, min(ts)))
    print(f"k={k:3d}  {min(ts):8.3f} ms", flush=True)
ks = np.array([r[0] for r in res], float); t = np.array([r[1] for r in res])
b, a = np.polyfit(ks, t, 1)
print(f"fit: {a:.3f} ms + {b:.4f} ms/sweep -> {8 * m * m / (b / 1e3) / 1e9:.0f} GB/s per sweep (8 m^2 bytes)")
