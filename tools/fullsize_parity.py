"""Full-size parity evidence: GPU vs the reference build (oracle/_ref) at a few
energies of config 2 / 4 / 5 (test infrastructure; writes nothing).

    python tools/fullsize_parity.py 5 0,700,1400,2047
    python tools/fullsize_parity.py 4 0 ref            # reference orientation (2557-dof root)
    python tools/fullsize_parity.py 4 341,683 complex  # E + i eta on the whole diagonal
"""
import sys, os, tempfile, time
sys.path.insert(0, '/root/repo')
import numpy as np
from oracle import refio
from paper_1305_1070_b200 import devices, negf
from tests.helpers import workload_ref_problem

cfg = int(sys.argv[1]); idx = np.array([int(x) for x in sys.argv[2].split(",")])
opts = sys.argv[3].split(",") if len(sys.argv) > 3 else []
ref_or, cplx = "ref" in opts, "complex" in opts  # reference orientation / E + i eta on the whole diagonal
w = (devices.config5() if cfg == 5 else devices.config4(ref_orientation=ref_or, complex_energy=cplx) if cfg == 4
     else devices.config3(complex_energy=cplx) if cfg == 3 else devices.config2(complex_energy=cplx))
p = w.problem
n = p.n
rp, sr, sl = workload_ref_problem(w, idx)
s = negf.HscGpuSolver(negf.HscPlan(p), max_energy_batch=len(idx)); s.set_residual_check(False)
t0 = time.time(); gr, gl = s.solve(w.energies[idx], w.weights[idx], sr, sl); tg = time.time() - t0
with tempfile.TemporaryDirectory() as tmp:
    path = os.path.join(tmp, "p.bin"); refio.write_problem(rp, path)
    t0 = time.time(); r = refio.run_reference(path, os.path.join(tmp, "o.bin"), threads=len(idx)); tr = time.time() - t0
print(f"cfg{cfg} n={n} energies {idx.tolist()}: GPU {tg:.1f}s, reference {tr:.1f}s on {len(idx)} threads, status {r.status} {r.message[:80]}")
for q, e in enumerate(idx):
    er = np.abs(gr[q] - r.gr[q]).max() / np.abs(r.gr[q]).max()
    el = np.abs(gl[q] - r.gless[q]).max() / np.abs(r.gless[q]).max()
    print(f"  E[{e}]={w.energies[e]:.5f}: rel err G^r {er:.2e}  G^< {el:.2e}")
    for tag, a, b in (("gpu", gr[q], gl[q]), ("ref", r.gr[q], r.gless[q])):
        ldos = -a.imag / np.pi
        print(f"     {tag}: max|G^r| {np.abs(a).max():.3e} min LDOS {ldos.min():.3e} max LDOS {ldos.max():.3e} "
              f"max|G^<| {np.abs(b).max():.3e} min Im G^< {b.imag.min():.3e} max |Re G^<|/|G^<| "
              f"{(np.abs(b.real) / np.maximum(np.abs(b), 1e-300)).max():.2e}")
