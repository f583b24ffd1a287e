"""How far fp32-storage variants of Algorithm 1 drift from the fp64 oracle (diagnostic, CPU only):
oracle/twin32.py with every sweep's P1 correction in fp64 (the streaming kernel's arithmetic) and
with fp32 sweeps after the first one after each product (the on-chip kernel's), per outer iteration.

    python tools/twin_drift.py c2 c3 > profiles/r02_twin_drift.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import fastpfp as O  # noqa: E402
from oracle.twin32 import F64, Twin32  # noqa: E402
from paper_1207_1114_b200 import inputs  # noqa: E402

out = {}
for which in sys.argv[1:]:
    p = {"c1": inputs.config1, "c2": inputs.config2, "c3": inputs.config3}[which]()
    st = O.FastPFP(p.A, p.Ap, p.B, p.Bp, p.X0)
    tw = {k: Twin32(p.A, p.Ap, p.B, p.Bp, p.X0, sweep_arith=k) for k in ("f64", "f32")}
    rows = []
    for it in range(min(p.max_iter1, 10)):
        st.iterate(p.lam, p.alpha, 0.0, p.eps2, 1, p.max_iter2)
        row = {"iter": it}
        for k, t in tw.items():
            t.step(p.lam, p.alpha, p.eps2, p.max_iter2)
            row[k] = float(np.max(np.abs(t.X.astype(F64) - st.X)))
        rows.append(row)
        print(which, row, file=sys.stderr, flush=True)
    out[which] = {"max_abs_dX_vs_oracle_per_outer": rows,
                  "f64": "P1 correction in fp64 every sweep (streaming kernel)",
                  "f32": "fp64 first sweep after the product, fp32 later sweeps (on-chip kernel)"}
print(json.dumps(out, indent=1))
