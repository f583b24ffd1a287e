# c4: ncu of the new batched kernel vs the previous one (stall reasons), and the per-pair error vs the oracle
cat > /tmp/c4err.py <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, paper_1207_1114_b200 as F
from oracle import fastpfp as O
from paper_1207_1114_b200 import inputs
for fixed in (True, False):
    probs = inputs.config4(fixed=fixed, first=0, count=8)
    p0 = probs[0]
    s = F.BatchedSolver(len(probs), 128, 128, 0); s.set_graphs(*inputs.stack_pairs(probs))
    X, rep = s.iterate(p0.alpha, p0.lam, p0.eps1, p0.eps2, p0.max_iter1, p0.max_iter2)
    errs = [float(np.max(np.abs(X[k].astype(np.float64) - O.solve(p)[0]))) for k, p in enumerate(probs)]
    print("fixed" if fixed else "eps", "max|dX| per pair:", " ".join(f"{e:.2e}" for e in errs), "iters", list(rep.iterations[:8]))
PY
for v in "" varlib/var_ss_old/libfastpfp.so; do FASTPFP_LIB=$v python /tmp/c4err.py; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:small_solve_tc -c 1 -o gpurun_out/c4b_new -f python tools/ncu_driver.py c4 20 > gpurun_out/c4b_ncu_new.log 2>&1; echo "ncu new rc=$?"
FASTPFP_LIB=varlib/var_ss_old/libfastpfp.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:small_solve_tc -c 1 -o gpurun_out/c4b_old -f python tools/ncu_driver.py c4 20 > gpurun_out/c4b_ncu_old.log 2>&1; echo "ncu old rc=$?"
