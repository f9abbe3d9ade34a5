"""The `real` plan form (real blocks skip the products with their zero imaginary
parts, real inverses in real arithmetic) must not change a single bit: solves
config 2 (every 4th energy) and two golden problems with and without it and
compares diag G^r, diag G^< and the density with array_equal.

    python tools/real_check.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1305_1070_b200 import devices, negf  # noqa: E402

BASE = "symdiag_g,symdiag_p,sparse,hull,compact"


def solve(w, idx, forms):
    os.environ["NEGF_PLAN_FORMS"] = forms
    plan = negf.HscPlan(w.problem)
    info = plan.info()
    s = negf.HscGpuSolver(plan)
    s.set_residual_check(False)
    sr, sl = w.self_energies(idx)
    gr, gl = s.solve(w.energies[idx], w.weights[idx], sr, sl)
    return gr, gl, s.density(), 8 * info.exec_cmul / 1e9


for name, w, idx in [("config2", devices.config2(), np.arange(0, 256, 4)),
                     ("config1", devices.config1(), None)]:
    if idx is None:
        idx = np.arange(len(w.energies))
    a = solve(w, idx, BASE + ",real")
    b = solve(w, idx, BASE)
    same = [bool(np.array_equal(x, y)) for x, y in zip(a[:3], b[:3])]
    dmax = [float(np.max(np.abs(x - y))) for x, y in zip(a[:3], b[:3])]
    print(f"{name}: {len(idx)} energies, executed GFLOP/point {a[3]:.3f} (real form) vs {b[3]:.3f}; "
          f"bit-identical gr/gl/density: {same}, max |diff| {dmax}", flush=True)
