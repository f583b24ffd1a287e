import sys, os
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1207_1114_b200 as F
m = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A = torch.zeros(m, m, device="cuda")
s = F.Solver(m, m, 0)
s.set_option(F.OPT_PROJ_KERNEL, 1)
s.set_graphs(A, A)
s.iterate(0.5, 0.0, 0, 0, 2, 20, want_x=False)
s.set_option(F.OPT_PROFILE, 1)
s.reset_stats()
s.iterate(0.5, 0.0, 0, 0, 3, 20, want_x=False)
st = s.stats()
ms = st["proj_ms"] / st["proj_launches"]
byts = 4 * m * m + 8 * m * m * 20 + 28 * m * m
print(f"{os.environ.get('FASTPFP_LIB','default')}: m={m} proj launch {ms:.3f} ms -> {byts/ms/1e6:.0f} GB/s ; gemm {st['gemm_ms']/st['gemm_launches']:.2f} ms")
