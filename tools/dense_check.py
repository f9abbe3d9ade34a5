"""GPU vs the reference's dense oracle (dense_gr / dense_gless, oracle.cpp:27-65,
n <= 2500) and vs the reference's HSC on a small workload (test
infrastructure; prints per-energy errors).

    python tools/dense_check.py cfg3_12 0,100
"""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import refio  # noqa: E402
from paper_1305_1070_b200 import devices, negf  # noqa: E402
from tests.helpers import per_energy_err, workload_ref_problem  # noqa: E402

name = sys.argv[1]
idx = np.array([int(x) for x in sys.argv[2].split(",")])
w = {"cfg3_12": lambda: devices.config3(n_cells=12), "cfg1": devices.config1,
     "cfg2_100x25": lambda: devices.config2(nx=100, ny=25)}[name]()
rp, sr, sl = workload_ref_problem(w, idx)
s = negf.HscGpuSolver(negf.HscPlan(w.problem))
s.set_residual_check(False)
gr, gl = s.solve(w.energies[idx], w.weights[idx], sr, sl)
with tempfile.TemporaryDirectory() as tmp:
    refio.write_problem(rp, tmp + "/p.bin")
    d = refio.run_reference(tmp + "/p.bin", tmp + "/d.out", threads=len(idx), solver="dense")
    h = refio.run_reference(tmp + "/p.bin", tmp + "/h.out", threads=len(idx), solver="hsc")
for q, e in enumerate(idx):
    print(f"{name} E[{e}]: gpu-dense {per_energy_err(gr[q:q+1], d.gr[q:q+1])[0]:.2e} / "
          f"{per_energy_err(gl[q:q+1], d.gless[q:q+1])[0]:.2e}   ref-dense "
          f"{per_energy_err(h.gr[q:q+1], d.gr[q:q+1])[0]:.2e} / {per_energy_err(h.gless[q:q+1], d.gless[q:q+1])[0]:.2e}"
          f"   gpu-ref {per_energy_err(gr[q:q+1], h.gr[q:q+1])[0]:.2e} / {per_energy_err(gl[q:q+1], h.gless[q:q+1])[0]:.2e}")
