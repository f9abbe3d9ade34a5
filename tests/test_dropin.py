"""The drop-in at the reference's own call site: the reference's cmd_solve /
solve_all (run.cpp:218-327), built from its own sources with a new solver
kind "hsc-gpu" whose energy loop goes through the C ABI
(oracle/hsc_gpu_bridge.inc, oracle/Makefile -> oracle/_ref/ref_driver_gpu),
driven by a reference config file.  Its CSVs must match the reference's own
CLI artefacts (proj/cli_test_tmp/solve_hsc, tests/golden/cli_solve_hsc_*) and
the unmodified reference run of the same config."""
import json
import os
import subprocess

import numpy as np
import pytest

from tests.helpers import GOLDEN

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GPU_DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver_gpu")
REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")

# small_superlattice_json of the reference's CLI tests (test_cli.cpp:83-97).
CLI_CONFIG = {
    "device": {"kind": "superlattice", "nx": 3, "ny": 8, "dx_nm": 1.0, "dy_nm": 1.0, "m_eff": 1.0,
               "n_barriers": 2, "barrier_width_nm": 1.0, "well_width_nm": 1.0, "barrier_height_ev": 0.2,
               "left_flat_nm": 2.0, "right_flat_nm": 3.0, "fermi_energy_ev": 0.25},
    "contact": {"model": "diagonal", "eta_ev": 1e-4, "eta_phonon_ev": 1e-3},
    "energy": {"points_ev": [0.18, 0.28]},
    "partition": {"max_leaf": 2},
}


def _values(path):
    with open(path) as f:
        lines = f.read().strip().splitlines()
    return lines[0], [l.rsplit(",", 1)[0] for l in lines[1:]], np.array([float(l.rsplit(",", 1)[1]) for l in lines[1:]])


def _run(driver, cfg, out, tmp_path, name):
    c = dict(cfg, output={"dir": out})
    path = str(tmp_path / f"{name}.json")
    with open(path, "w") as f:
        json.dump(c, f)
    return subprocess.run([driver, "cli", "solve", path], capture_output=True, text=True, timeout=600)


def test_dropin_driver_builds_with_the_solver_kind():
    """CPU: the patched reference build exists and knows "hsc-gpu" (parse_solver,
    config.cpp:82-86) -- an unknown solver name is still a ConfigError (exit 2)."""
    if not os.path.exists(GPU_DRIVER):
        pytest.skip("oracle/_ref/ref_driver_gpu not built")
    import tempfile

    with tempfile.TemporaryDirectory() as tmp:
        import pathlib

        r = _run(GPU_DRIVER, dict(CLI_CONFIG, solver="hsc-cpu"), os.path.join(tmp, "o"), pathlib.Path(tmp), "bad")
        assert r.returncode == 2 and "solver" in r.stderr


@pytest.mark.gpu
def test_reference_cmd_solve_with_hsc_gpu_reproduces_cli_goldens(tmp_path, cuda_ok):
    if not os.path.exists(GPU_DRIVER):
        pytest.skip("oracle/_ref/ref_driver_gpu not built")
    out = str(tmp_path / "gpu")
    r = _run(GPU_DRIVER, dict(CLI_CONFIG, solver="hsc-gpu"), out, tmp_path, "gpu")
    assert r.returncode == 0, r.stderr
    for ours, ref in (("density.csv", "cli_solve_hsc_density.csv"), ("ldos.csv", "cli_solve_hsc_ldos.csv"),
                      ("line_density.csv", "cli_solve_hsc_line_density.csv")):
        ha, ka, va = _values(os.path.join(out, ours))
        hb, kb, vb = _values(os.path.join(GOLDEN, ref))
        assert ha == hb and ka == kb
        assert np.abs(va - vb).max() <= 1e-10 * np.abs(vb).max(), (ours, np.abs(va - vb).max())


@pytest.mark.gpu
@pytest.mark.parametrize("contact,leaf,energies", [("dense-lead", 8, [0.05, 0.18, 0.28]),
                                                   ("diagonal", 4, [0.1, 0.2, 0.3, 0.4])])
def test_reference_cmd_solve_hsc_gpu_vs_hsc(tmp_path, contact, leaf, energies, cuda_ok):
    """Same config through the unmodified reference ("hsc") and through the
    drop-in ("hsc-gpu"): wider device, dense decimated leads (atomic contact
    groups) or diagonal contacts, multi-threaded energy pool."""
    if not (os.path.exists(GPU_DRIVER) and os.path.exists(REF_DRIVER)):
        pytest.skip("oracle/_ref drivers not built")
    cfg = json.loads(json.dumps(CLI_CONFIG))
    cfg["device"].update({"nx": 6, "ny": 20, "left_flat_nm": 6.0, "right_flat_nm": 11.0})
    cfg["contact"] = {"model": contact, "eta_ev": 1e-4, "eta_phonon_ev": 1e-3}
    cfg["energy"] = {"points_ev": energies}
    cfg["partition"] = {"max_leaf": leaf}
    cfg["threads"] = 2
    a = _run(GPU_DRIVER, dict(cfg, solver="hsc-gpu"), str(tmp_path / "gpu"), tmp_path, "gpu")
    b = _run(REF_DRIVER, dict(cfg, solver="hsc"), str(tmp_path / "ref"), tmp_path, "ref")
    assert a.returncode == 0, a.stderr
    assert b.returncode == 0, b.stderr
    for f in ("density.csv", "ldos.csv", "line_density.csv"):
        ha, ka, va = _values(str(tmp_path / "gpu" / f))
        hb, kb, vb = _values(str(tmp_path / "ref" / f))
        assert ha == hb and ka == kb
        assert np.abs(va - vb).max() <= 1e-10 * np.abs(vb).max(), (f, np.abs(va - vb).max())
