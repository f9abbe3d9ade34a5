"""Full-size parity evidence: GPU vs the reference build (oracle/_ref) at a few
energies of config 2 / 4 / 5 (test infrastructure; writes nothing).

    python tools/fullsize_parity.py 5 0,700,1400,2047
"""
import sys, os, tempfile, time
sys.path.insert(0, '/root/repo')
import numpy as np
from oracle import refio
from paper_1305_1070_b200 import devices, negf

cfg = int(sys.argv[1]); idx = np.array([int(x) for x in sys.argv[2].split(",")])
ref_or = len(sys.argv) > 3 and sys.argv[3] == "ref"
w = devices.config5() if cfg == 5 else devices.config4(ref_orientation=ref_or) if cfg == 4 else devices.config2()
p = w.problem
sr, sl = w.self_energies(idx)
ny = w.ny; w2 = ny * ny; n = p.n
L = np.asarray(p.atomic_groups[0], np.int32); R = np.asarray(p.atomic_groups[1], np.int32)
has_ph = len(p.sr_rows) > 2 * w2
ph = phl = None
if has_ph:
    inner = np.asarray(p.sr_rows[2 * w2:], np.int64)
    ph = np.zeros((len(idx), n), np.complex128); ph[:, inner] = sr[:, 2 * w2:]
    phl = np.zeros((len(idx), n), np.complex128); phl[:, inner] = sl[:, 2 * w2:]
rp = refio.RefProblem(n=n, h_rows=p.h_rows, h_cols=p.h_cols, h_vals=p.h_vals, layers=[np.asarray(l) for l in p.layers],
                      coords=p.coords, groups=[L, R], max_leaf=p.max_leaf, dofs_l=L, dofs_r=R,
                      has_ph=has_ph, has_ph_less=has_ph, energies=w.energies[idx], weights=w.weights[idx],
                      sig_l=sr[:, :w2].reshape(-1, ny, ny), sig_r=sr[:, w2:2 * w2].reshape(-1, ny, ny), ph=ph,
                      less_l=sl[:, :w2].reshape(-1, ny, ny), less_r=sl[:, w2:2 * w2].reshape(-1, ny, ny), ph_less=phl)
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
