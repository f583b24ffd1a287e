# c4: row-pair tile + shifted column frame + smem row transpose (new) vs the previous kernel (var_ss_old)
timeout 900 python -m pytest tests/test_gpu_batched.py -x -q > gpurun_out/c4a_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/c4a_tests.log
cat > /tmp/c4err.py <<'PY'
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
for v in "" varlib/var_ss_old/libfastpfp.so "" varlib/var_ss_old/libfastpfp.so; do
export FASTPFP_LIB=$v
timeout 300 python bench.py --workload c4 --steps 40 --warmup 3 --no-cpu-baseline --no-secondary 2>/dev/null > /tmp/c4.json
python -c "
import json,sys,os; d=json.loads([l for l in open('/tmp/c4.json') if l.startswith('{')][-1]); print(os.environ.get('FASTPFP_LIB') or 'main', 'c4', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
unset FASTPFP_LIB
FASTPFP_LIB=varlib/var_ssprof/libfastpfp.so timeout 300 python tools/ncu_driver.py c4 2 2>&1 | grep ss-prof | head -4
