"""Margins of the full-grid config-2 parity test (tests/test_gpu_fullgrid.py) per
energy: err / bar for diag G^r and G^<, and the real-part residual of G^< over its
bar.  Needs oracle/_ref and a GPU.  NEGF_LIB selects a variant build.

    python tools/resid_margin.py
"""
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import refio  # noqa: E402
from paper_1305_1070_b200 import devices, negf  # noqa: E402
from tests.helpers import GOLDEN, per_energy_err, real_residual, workload_ref_problem  # noqa: E402

fx = np.load(os.path.join(GOLDEN, "cfg2_floor.npz"))
w = devices.config2()
idx = np.arange(len(w.energies))
rp, sr, sl = workload_ref_problem(w, idx)
s = negf.HscGpuSolver(negf.HscPlan(w.problem))
s.set_residual_check(False)
gr, gl = s.solve(w.energies, w.weights, sr, sl)
res = real_residual(gl)
rbar = np.maximum(1e-11, 2.0 * fx["resid_floor"])
q = res / rbar
top = np.argsort(-q)[:8]
print("lib", os.environ.get("NEGF_LIB", "default"))
print("residual/bar top:", [(int(k), float(f"{q[k]:.3g}"), float(f"{res[k]:.3g}")) for k in top], "n>0.5:", int((q > 0.5).sum()))
if "--ref" in sys.argv:
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "p.bin")
        refio.write_problem(rp, path)
        ref = refio.run_reference(path, os.path.join(tmp, "o.bin"), threads=os.cpu_count())
    er = per_energy_err(gr, ref.gr) / np.maximum(1e-10, 2.0 * fx["floor_r"])
    el = per_energy_err(gl, ref.gless) / np.maximum(1e-10, 2.0 * fx["floor_l"])
    print("err_r/bar top:", [(int(k), float(f"{er[k]:.3g}")) for k in np.argsort(-er)[:6]])
    print("err_l/bar top:", [(int(k), float(f"{el[k]:.3g}")) for k in np.argsort(-el)[:6]])
