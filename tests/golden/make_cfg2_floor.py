"""Per-energy conditioning floor of the reference on BASELINE config 2 (the
full 256-point grid of the 400 x 100 superlattice), for the full-grid GPU
parity test (tests/test_gpu_fullgrid.py).  Run here (oracle/_ref built):

    python tests/golden/make_cfg2_floor.py      -> tests/golden/cfg2_floor.npz

The floor of energy k is how far two correct FP64 evaluations of the
reference's own algorithm (hsc_fold + hsc_gless, oracle/_ref) drift apart
there: the maximum, over
  * the same algorithm with another matmul summation order (NEGF_SHIM_NAIVE=1:
    i-k-j loops instead of OpenBLAS ZGEMM), and
  * 24 runs on inputs perturbed by one unit in the last place (H and the
    contact self-energies, relative +-2^-52 per component, seeds 1-24; eight
    samples left the maximum of this noise underestimated: two correct GPU
    summation orders landed 0.92x and 1.02x of twice that maximum) --
    the rounding any FP64 producer of those inputs already carries,
of max_j |g_j - o_j| / max_j |o_j| against the unperturbed OpenBLAS run, for
diag G^r and diag G^< separately.  Also stored: the reference's own
max_j |Re G^<_jj| / |G^<_jj| per energy (electron_density's guard quantity)
of every run, and its maximum over the runs (resid_floor).
"""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import refio  # noqa: E402
from paper_1305_1070_b200 import devices  # noqa: E402
from tests.helpers import per_energy_err, real_residual, workload_ref_problem  # noqa: E402


def ulp_perturb(a: np.ndarray, rng) -> np.ndarray:
    s = rng.choice([-1.0, 1.0], size=a.shape) * 2.0 ** -52
    t = rng.choice([-1.0, 1.0], size=a.shape) * 2.0 ** -52
    return (a.real * (1 + s) + 1j * a.imag * (1 + t)).astype(np.complex128)


NSEEDS = 24


def main() -> None:
    w = devices.config2()
    idx = np.arange(len(w.energies))
    rp, _, _ = workload_ref_problem(w, idx)
    threads = os.cpu_count()
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "p.bin")
        refio.write_problem(rp, path)
        base = refio.run_reference(path, os.path.join(tmp, "b.out"), threads=threads)
        assert base.status == 0, base.message
        arms = []
        os.environ["NEGF_SHIM_NAIVE"] = "1"
        arms.append(("naive", refio.run_reference(path, os.path.join(tmp, "n.out"), threads=threads)))
        del os.environ["NEGF_SHIM_NAIVE"]
        for seed in range(1, NSEEDS + 1):
            rng = np.random.default_rng(seed)
            q = workload_ref_problem(w, idx)[0]
            q.h_vals = ulp_perturb(np.asarray(q.h_vals), rng)
            q.sig_l = ulp_perturb(q.sig_l, rng)
            q.sig_r = ulp_perturb(q.sig_r, rng)
            pp = os.path.join(tmp, f"p{seed}.bin")
            refio.write_problem(q, pp)
            arms.append((f"ulp{seed}", refio.run_reference(pp, os.path.join(tmp, f"u{seed}.out"), threads=threads)))
    out = {"energies": w.energies, "ref_resid": real_residual(base.gless)}
    fr = np.zeros(len(idx))
    fl = np.zeros(len(idx))
    rf = out["ref_resid"].copy()
    for name, r in arms:
        assert r.status == 0, (name, r.message)
        er, el = per_energy_err(r.gr, base.gr), per_energy_err(r.gless, base.gless)
        out[f"{name}_r"], out[f"{name}_l"] = er, el
        out[f"{name}_resid"] = real_residual(r.gless)
        fr, fl = np.maximum(fr, er), np.maximum(fl, el)
        rf = np.maximum(rf, out[f"{name}_resid"])
        print(f"{name}: G^r max {er.max():.2e} (#>1e-10 {(er > 1e-10).sum()}), G^< max {el.max():.2e}")
    out["floor_r"], out["floor_l"], out["resid_floor"] = fr, fl, rf
    np.savez(os.path.join(HERE, "cfg2_floor.npz"), **out)
    print(f"floor: #energies > 1e-10: G^r {(fr > 1e-10).sum()}, G^< {(fl > 1e-10).sum()}")


if __name__ == "__main__":
    main()
