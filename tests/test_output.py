"""Output path: cmd_solve's CSV artefacts with the
reference's format_double (run.cpp:276-326) and the binary shard writer.

Pins: every number string of the reference's stored CLI CSVs
(tests/golden/cli_*.csv) is reproduced bit-exactly by negf_format_double; the
CSV writer reproduces the reference's files line structure and values from
the GPU solve of the same device (GPU test)."""
from __future__ import annotations

import os

import numpy as np
import pytest

from paper_1305_1070_b200 import negf
from tests.helpers import GOLDEN, load_golden, rel_err

CSVS = ["cli_solve_hsc_density.csv", "cli_solve_hsc_ldos.csv", "cli_solve_hsc_line_density.csv",
        "cli_solve_dense_density.csv"]


def _lines(path):
    with open(path) as f:
        return f.read().splitlines()


@pytest.mark.parametrize("name", CSVS)
def test_format_double_reproduces_reference_strings(name):
    lines = _lines(os.path.join(GOLDEN, name))
    n = 0
    for line in lines[1:]:
        for tok in line.split(","):
            if any(c in tok for c in ".eE") or len(tok) > 3:
                assert negf.format_double(float(tok)) == tok
                n += 1
    assert n > 0


def test_format_double_edge_values():
    assert negf.format_double(3.0) == "3"
    assert negf.format_double(0.1) == "0.10000000000000001"
    for v in (-2.5e-300, 1e21, 0.0, 1.0 / 3.0, -7.25, 6.02214076e23, 2.0 ** -1074):
        assert negf.format_double(v) == "%.17g" % v  # to_chars(general, 17) == printf %.17g


def test_write_solve_csv_layout(tmp_path):
    """Headers, index columns and the line sums of line_density_y."""
    nx, ny, ne = 3, 4, 2
    rng = np.random.default_rng(3)
    dens = rng.random(nx * ny)
    gr = rng.random((ne, nx * ny)) + 1j * rng.random((ne, nx * ny))
    e = np.array([0.18, 0.28])
    out = str(tmp_path / "o" / "p")
    negf.write_solve_csv(out, nx, ny, e, dens, gr)
    d = _lines(os.path.join(out, "density.csv"))
    assert d[0] == "x_index,y_index,density" and len(d) == 1 + nx * ny
    assert d[1 + 1 * nx + 2] == "2,1," + negf.format_double(dens[1 * nx + 2])
    ld = _lines(os.path.join(out, "ldos.csv"))
    assert ld[0] == "x_index,y_index,energy_eV,ldos" and len(ld) == 1 + ne * nx * ny
    k, y, x = 1, 3, 0
    assert ld[1 + k * nx * ny + y * nx + x] == (f"{x},{y},{negf.format_double(e[k])},"
                                                 f"{negf.format_double(-gr[k, y * nx + x].imag / np.pi)}")
    ln = _lines(os.path.join(out, "line_density.csv"))
    s = 0.0
    for xx in range(nx):
        s += dens[2 * nx + xx]
    assert ln[0] == "y_index,density" and ln[3] == "2," + negf.format_double(s)
    negf.write_solve_csv(str(tmp_path / "q"), nx, ny, e, dens)  # no ldos
    assert not os.path.exists(tmp_path / "q" / "ldos.csv")


def test_write_solve_csv_errors(tmp_path):
    blocker = tmp_path / "file"
    blocker.write_text("x")
    with pytest.raises(negf.ConfigError):
        negf.write_solve_csv(str(blocker / "sub"), 2, 2, [0.1], np.zeros(4))


def test_shard_writer_host_round_trip(tmp_path):
    n = 37
    rng = np.random.default_rng(5)
    gr = rng.random((5, n)) + 1j * rng.random((5, n))
    gl = rng.random((5, n)) + 1j * rng.random((5, n))
    e = np.linspace(0.0, 0.4, 5)
    p = str(tmp_path / "s0.bin")
    with negf.ShardWriter(p, n, rank=1, world=4) as w:
        w.append(e[:3], 10, gr[:3], gl[:3])
        w.append(e[3:], 13, gr[3:], gl[3:])
    r = negf.read_shard(p)
    assert (r["rank"], r["world"], r["n_dofs"]) == (1, 4, n)
    assert np.array_equal(r["energy_index"], np.arange(10, 15))
    assert np.array_equal(r["energies"], e)
    assert np.array_equal(r["gr"], gr) and np.array_equal(r["gless"], gl)
    p2 = str(tmp_path / "s1.bin")
    with negf.ShardWriter(p2, n, gr=False) as w:
        w.append(e, 0, gless=gl)
    r2 = negf.read_shard(p2)
    assert "gr" not in r2 and np.array_equal(r2["gless"], gl)


def test_shard_writer_errors(tmp_path):
    with pytest.raises(negf.ConfigError):
        negf.ShardWriter(str(tmp_path / "missing" / "x.bin"), 4)
    with pytest.raises(negf.ContractViolation):
        negf.ShardWriter(str(tmp_path / "x.bin"), 4, gr=False, gless=False)
    w = negf.ShardWriter(str(tmp_path / "y.bin"), 4)
    with pytest.raises(negf.ContractViolation):
        w.append([0.1], 0, gr=np.zeros((1, 4), complex))  # gless required
    w.close()


# ---------------------------------------------------------------- GPU ----
@pytest.mark.gpu
def test_gpu_solve_to_reference_csvs(tmp_path, cuda_ok):
    """GPU solve of the CLI fixture device -> density/ldos/line_density CSVs
    matching the reference's own files line by line (values to 1e-10)."""
    rp, prob, hsc, _ = load_golden("superlattice_3x8_diag")
    plan = negf.HscPlan(prob)
    s = negf.HscGpuSolver(plan)
    sr, sl = rp.values(np.arange(len(rp.energies)))
    gr, gl = s.solve(rp.energies, rp.weights, sr, sl)
    dens = s.density() * 1.0  # density_scale = 1/(dx dy) = 1 nm^-2
    out = str(tmp_path / "solve")
    negf.write_solve_csv(out, 3, 8, rp.energies, dens, gr)
    for ours, ref in (("density.csv", "cli_solve_hsc_density.csv"), ("ldos.csv", "cli_solve_hsc_ldos.csv"),
                      ("line_density.csv", "cli_solve_hsc_line_density.csv")):
        a, b = _lines(os.path.join(out, ours)), _lines(os.path.join(GOLDEN, ref))
        assert len(a) == len(b) and a[0] == b[0]
        va = np.array([float(l.rsplit(",", 1)[1]) for l in a[1:]])
        vb = np.array([float(l.rsplit(",", 1)[1]) for l in b[1:]])
        assert [l.rsplit(",", 1)[0] for l in a[1:]] == [l.rsplit(",", 1)[0] for l in b[1:]]
        assert rel_err(va, vb) < 1e-10


@pytest.mark.gpu
def test_gpu_shard_writer_device_round_trip(tmp_path, cuda_ok):
    import torch

    n, ne = 1000, 4
    g = torch.randn(3, ne, n, dtype=torch.complex128, device="cuda")
    h = torch.randn(3, ne, n, dtype=torch.complex128, device="cuda")
    p = str(tmp_path / "dev.bin")
    with negf.ShardWriter(p, n) as w:
        for b in range(3):  # three appends through two pinned slots
            w.append_device(np.full(ne, 0.1 * b), b * ne, g[b], h[b])
        w.append(np.array([9.0]), 99, g[0, :1].cpu().numpy(), h[0, :1].cpu().numpy())
        torch.cuda.synchronize()
    r = negf.read_shard(p)
    assert np.array_equal(r["energy_index"], np.r_[np.arange(12), 99])
    assert np.array_equal(r["gr"][:12], g.reshape(12, n).cpu().numpy())
    assert np.array_equal(r["gless"][:12], h.reshape(12, n).cpu().numpy())
    assert np.array_equal(r["gr"][12], g[0, 0].cpu().numpy())
