"""Regenerates the committed golden fixtures from the REFERENCE itself.

Run here (where /root/reference exists and oracle/_ref is built):
    python tests/golden/make_golden.py

Every *.bin problem is written by the reference's own input builders
(make_synthetic_system, build_superlattice_hamiltonian/attach_contacts/...,
driven by oracle/ref_driver.cpp) and every *.out result by the reference's
own solvers (hsc_fold + hsc_gless, or the dense oracle) compiled from
/root/reference/proj/src.  The CLI goldens (cli_*.csv, tree.json) are the
reference's stored test artefacts from proj/cli_test_tmp, copied verbatim.
"""
from __future__ import annotations

import json
import os
import shutil
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import refio  # noqa: E402

REF_PROJ = "/root/reference/proj"

# (name, nx, ny, seed, fuzz, coupling, max_leaf, energies)  -- the first four
# are test_hsc.cpp:680-725's ND-vs-dense cases; the rest widen the shapes.
SYNTHETIC = [
    ("syn_4x6_s21_fuzz", 4, 6, 21, True, 1.3, 6, [0.7]),
    ("syn_5x5_s22_fuzz", 5, 5, 22, True, 1.3, 6, [0.7]),
    ("syn_6x4_s23_fuzz", 6, 4, 23, True, 1.3, 6, [0.7]),
    ("syn_5x6_s24", 5, 6, 24, False, 1.3, 6, [0.7]),
    ("syn_24x20_s5_fuzz", 24, 20, 5, True, 1.0, 16, [0.1, 0.4, 0.9]),
    ("syn_40x36_s6", 40, 36, 6, False, 1.0, 64, [0.0, 0.5]),
    ("syn_120x14_s7_fuzz", 120, 14, 7, True, 1.0, 64, [0.3]),
    # cmd_bench's HSC row (run.cpp:385-406): 4x4 synthetic at E = 0, seed 1
    ("syn_4x4_s1_bench", 4, 4, 1, False, 1.0, 64, [0.0]),
]

SUPERLATTICE_DIAG = {
    "device": {"kind": "superlattice", "nx": 3, "ny": 8, "dx_nm": 1.0, "dy_nm": 1.0, "m_eff": 1.0,
               "n_barriers": 2, "barrier_width_nm": 1.0, "well_width_nm": 1.0, "barrier_height_ev": 0.2,
               "left_flat_nm": 2.0, "right_flat_nm": 3.0, "fermi_energy_ev": 0.25},
    "solver": "hsc",
    "contact": {"model": "diagonal", "eta_ev": 1e-4, "eta_phonon_ev": 1e-3},
    "energy": {"points_ev": [0.18, 0.28]},
    "partition": {"max_leaf": 2},
}


def main() -> None:
    if not refio.ref_available():
        raise SystemExit("oracle/_ref/ref_driver missing: run make -C oracle")
    with tempfile.TemporaryDirectory() as tmp:
        for name, nx, ny, seed, fuzz, t, leaf, energies in SYNTHETIC:
            prob = os.path.join(HERE, name + ".bin")
            refio.dump_synthetic(nx, ny, seed, fuzz, t, leaf, energies, prob)
            refio.run_reference(prob, os.path.join(HERE, name + ".hsc.out"))
            if nx * ny <= 2500:
                refio.run_reference(prob, os.path.join(HERE, name + ".dense.out"), solver="dense")
        # The CLI fixture device (test_cli.cpp:83-97), diagonal contacts.
        cfg = os.path.join(tmp, "sl.json")
        with open(cfg, "w") as f:
            json.dump(SUPERLATTICE_DIAG, f)
        prob = os.path.join(HERE, "superlattice_3x8_diag.bin")
        refio.dump_device(cfg, prob)
        refio.run_reference(prob, os.path.join(HERE, "superlattice_3x8_diag.hsc.out"))
        # Same device with dense decimated leads (atomic contact groups).
        dense = json.loads(json.dumps(SUPERLATTICE_DIAG))
        dense["device"].update({"nx": 6, "ny": 20, "left_flat_nm": 6.0, "right_flat_nm": 11.0})
        dense["contact"] = {"model": "dense-lead", "eta_ev": 1e-4, "eta_phonon_ev": 1e-3}
        dense["energy"] = {"points_ev": [0.05, 0.18, 0.28]}
        dense["partition"] = {"max_leaf": 8}
        with open(cfg, "w") as f:
            json.dump(dense, f)
        prob = os.path.join(HERE, "superlattice_6x20_dense.bin")
        refio.dump_device(cfg, prob)
        refio.run_reference(prob, os.path.join(HERE, "superlattice_6x20_dense.hsc.out"))
        refio.run_reference(prob, os.path.join(HERE, "superlattice_6x20_dense.dense.out"), solver="dense")
        graphene = {"device": {"kind": "graphene", "nx": 8, "ny": 16, "onsite_ev": 0.0, "hopping_ev": -3.1,
                               "fermi_energy_ev": 0.0},
                    "contact": {"model": "dense-lead", "eta_ev": 1e-4}, "energy": {"points_ev": [0.5, 0.9]},
                    "partition": {"max_leaf": 8}}
        with open(cfg, "w") as f:
            json.dump(graphene, f)
        prob = os.path.join(HERE, "graphene_8x16_dense.bin")
        refio.dump_device(cfg, prob)
        refio.run_reference(prob, os.path.join(HERE, "graphene_8x16_dense.hsc.out"))
        refio.run_reference(prob, os.path.join(HERE, "graphene_8x16_dense.dense.out"), solver="dense")
    # Stored reference CLI artefacts (outputs of the reference's own test run).
    for sub, fn in [("solve_hsc", "density.csv"), ("solve_hsc", "ldos.csv"), ("solve_hsc", "line_density.csv"),
                    ("solve_dense", "density.csv"), ("partition", "tree.json"), ("bench", "bench.csv"),
                    ("bench_wall", "bench.csv")]:
        src = os.path.join(REF_PROJ, "cli_test_tmp", sub, fn)
        if os.path.exists(src):
            shutil.copy(src, os.path.join(HERE, f"cli_{sub}_{fn}"))


# Dense leads through the reference's surface_self_energy (device.cpp:195-251,
# ref_driver lead): (name, h00/h01 builder, eta, energies).  cnt80 is the
# config-3 (20,0) tube cell (E = 3.0 does not converge: ConvergenceError);
# em100 the config-2 2-D effective-mass lead; em120 exceeds the 112-wide
# shared-memory inverse (multi-CTA inverse path).
def _em_lead(w: int, t: float):
    import numpy as np
    h00 = np.diag(np.full(w, 4.0 * t)) - t * (np.eye(w, k=1) + np.eye(w, k=-1))
    return h00.astype(np.complex128), (-t * np.eye(w)).astype(np.complex128)


def _cnt_lead():
    import numpy as np
    from paper_1305_1070_b200 import devices
    h00, h01 = devices._cnt_cell(20, -2.7)
    return h00.astype(np.complex128), h01.astype(np.complex128)


T_EM = 0.0380998 / (0.067 * 0.5 * 0.5)
LEADS = [
    ("lead_cnt80", _cnt_lead, 1e-6, [-0.9, -0.3, 0.05, 0.4, 0.95, 3.0]),
    ("lead_em100", lambda: _em_lead(100, T_EM), 1e-6, [0.0, 0.13, 0.4]),
    ("lead_em120", lambda: _em_lead(120, T_EM), 1e-6, [0.05, 0.3]),
]


def make_leads() -> None:
    for name, build, eta, energies in LEADS:
        h00, h01 = build()
        path = os.path.join(HERE, name + ".bin")
        refio.write_lead(path, h00, h01, eta, energies)
        refio.run_lead(path, os.path.join(HERE, name + ".out"))


def make_rgf() -> None:
    """The reference's layered RGF (rgf_gr + rgf_gless, rgf.cpp:181-380) on
    every problem fixture's own layer map."""
    import glob
    for p in sorted(glob.glob(os.path.join(HERE, "*.bin"))):
        name = os.path.basename(p)[:-4]
        if name.startswith("lead_"):
            continue
        refio.run_reference(p, os.path.join(HERE, name + ".rgf.out"), solver="rgf")


if __name__ == "__main__":
    if sys.argv[1:] == ["leads"]:
        make_leads()
    elif sys.argv[1:] == ["rgf"]:
        make_rgf()
    else:
        main()
        make_leads()
        make_rgf()
