"""The C++ host program on the C ABI alone (examples/negf_solve.cpp): the
reference's solve_all / cmd_solve routed to the B200 library, as a
maintainer would bind it.  It reads the reference's own
problem dumps and must reproduce the reference's outputs."""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

from paper_1305_1070_b200 import build, negf
from tests.helpers import GOLDEN, load_golden, rel_err

BIN = build.EXAMPLE_BIN


def _run(*args):
    return subprocess.run([BIN, *map(str, args)], capture_output=True, text=True, timeout=600)


def test_example_builds_and_maps_errors_like_the_cli(tmp_path):
    build.build_example()
    assert os.path.exists(BIN)
    r = _run()
    assert r.returncode == 1 and "usage" in r.stderr
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"not a problem")
    r = _run(bad, tmp_path / "out")
    assert r.returncode == 2 and "config error" in r.stderr  # ConfigError -> exit 2 (negf_main.cpp:65-77)


@pytest.mark.gpu
@pytest.mark.parametrize("name,nx,ny", [("superlattice_3x8_diag", 3, 8), ("superlattice_6x20_dense", 6, 20),
                                        ("graphene_8x16_dense", 0, 0), ("syn_24x20_s5_fuzz", 0, 0)])
def test_example_reproduces_reference(name, nx, ny, tmp_path, cuda_ok):
    build.build_example()
    rp, _, hsc, _ = load_golden(name)
    out = tmp_path / "o"
    args = [os.path.join(GOLDEN, name + ".bin"), out]
    if nx:
        args += ["--nx", nx, "--ny", ny]
    r = _run(*args)
    assert r.returncode == 0, r.stderr
    d = negf.read_shard(str(out / "diag.bin"))
    assert np.array_equal(d["energies"], rp.energies)
    for k in range(len(rp.energies)):
        assert rel_err(d["gr"][k], hsc.gr[k]) < 1e-10
        assert rel_err(d["gless"][k], hsc.gless[k]) < 1e-10
    if name == "superlattice_3x8_diag":  # the reference CLI's own fixture device
        for ours, ref in (("density.csv", "cli_solve_hsc_density.csv"), ("ldos.csv", "cli_solve_hsc_ldos.csv")):
            a = open(out / ours).read().splitlines()
            b = open(os.path.join(GOLDEN, ref)).read().splitlines()
            assert len(a) == len(b) and a[0] == b[0]
            va = np.array([float(x.rsplit(",", 1)[1]) for x in a[1:]])
            vb = np.array([float(x.rsplit(",", 1)[1]) for x in b[1:]])
            assert rel_err(va, vb) < 1e-10
