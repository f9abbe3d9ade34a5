"""GPU ledger bench mode: cmd_bench (run.cpp:361-419).

Pins: the synthetic-system restatement is bit-exact against the reference's
own dumps; the RGF and HSC reference-ledger counts equal the reference's on
every golden problem and the stored bench rows (cli_test_tmp/bench*)."""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import refio
from paper_1305_1070_b200 import devices, ledger_bench, negf
from tests.helpers import GOLDEN, golden_names, load_golden

SYN = [("syn_4x6_s21_fuzz", 4, 6, 21, True, 1.3), ("syn_5x5_s22_fuzz", 5, 5, 22, True, 1.3),
       ("syn_6x4_s23_fuzz", 6, 4, 23, True, 1.3), ("syn_5x6_s24", 5, 6, 24, False, 1.3),
       ("syn_24x20_s5_fuzz", 24, 20, 5, True, 1.0), ("syn_40x36_s6", 40, 36, 6, False, 1.0),
       ("syn_120x14_s7_fuzz", 120, 14, 7, True, 1.0), ("syn_4x4_s1_bench", 4, 4, 1, False, 1.0)]


@pytest.mark.parametrize("name,nx,ny,seed,fuzz,t", SYN)
def test_synthetic_system_bit_exact(name, nx, ny, seed, fuzz, t):
    rp = refio.read_problem(os.path.join(GOLDEN, name + ".bin"))
    s = devices.synthetic_system(nx, ny, seed, fuzz, t)
    assert np.array_equal(s["h_rows"], rp.h_rows) and np.array_equal(s["h_cols"], rp.h_cols)
    assert np.array_equal(s["h_vals"], rp.h_vals)
    assert np.array_equal(s["sig_l"], rp.sig_l[0]) and np.array_equal(s["sig_r"], rp.sig_r[0])
    dense = np.zeros((rp.n, rp.n), np.complex128)
    dense[s["sl_rows"], s["sl_cols"]] = s["sl_vals"]
    L, R = np.asarray(rp.dofs_l), np.asarray(rp.dofs_r)
    assert np.array_equal(dense[np.ix_(L, L)], rp.less_l[0])
    assert np.array_equal(dense[np.ix_(R, R)], rp.less_r[0])
    if rp.ph_less is not None:
        inner = np.setdiff1d(np.arange(rp.n), np.r_[L, R])
        assert np.array_equal(np.diag(dense)[inner], rp.ph_less[0][inner])


@pytest.mark.parametrize("name", golden_names())
def test_rgf_reference_ledger_exact(name):
    rp, prob, _, _ = load_golden(name)
    r = refio.read_result(os.path.join(GOLDEN, name + ".rgf.out"), rp.n)
    ne = len(rp.energies)
    assert ledger_bench.rgf_reference_ledger(prob, rp.layers) == (r.mul_ops // ne, r.inv_ops // ne)


def test_reference_bench_rows_counts():
    """rgf,4,4,1304,256 and hsc,4,4,8192,4096 (cli_test_tmp/bench_wall/bench.csv)."""
    with open(os.path.join(GOLDEN, "cli_bench_wall_bench.csv")) as f:
        rows = [l.strip().split(",") for l in f][1:]
    s = devices.synthetic_system(4, 4, 1, False, 1.0)
    for solver, nx, ny, mul, inv, _ in rows:
        assert (int(nx), int(ny)) == (4, 4)
        if solver == "rgf":
            got = ledger_bench.rgf_reference_ledger(s["problem"], s["layers"])
        else:
            i = negf.HscPlan(s["problem"]).info()
            got = (i.ref_fold_mul + i.ref_gless_mul, i.ref_fold_inv + i.ref_gless_inv)
        assert got == (int(mul), int(inv))


def test_skipped_rule(tmp_path):
    """rgf,64,2,skipped,skipped,skipped (cli_test_tmp/bench/bench.csv): the
    working-set estimate 16*8*Nx^2*Ny bytes above max_mem_mb skips a size."""
    rows = ledger_bench.bench_rows([(64, 2)], ["rgf"], max_mem_mb=0.5)
    ledger_bench.write_bench(str(tmp_path), rows)
    lines = open(tmp_path / "bench.csv").read().splitlines()
    ref = open(os.path.join(GOLDEN, "cli_bench_bench.csv")).read().splitlines()
    assert lines[0] == ref[0] and lines[1] == ref[2]


@pytest.mark.gpu
def test_gpu_ledger_bench_mode(tmp_path, cuda_ok):
    sizes = [(4, 4), (12, 10), (30, 8)]
    rows = ledger_bench.bench_rows(sizes, ["rgf", "hsc"], seed=1)
    ledger_bench.write_bench(str(tmp_path), rows)
    lines = open(tmp_path / "bench.csv").read().splitlines()
    assert lines[1].startswith("rgf,4,4,1304,256,") and lines[2].startswith("hsc,4,4,8192,4096,")
    for r in rows:
        s = devices.synthetic_system(r["nx"], r["ny"], 1)
        if r["solver"] == "rgf":
            assert (r["multiply_ops"], r["inverse_ops"]) == ledger_bench.rgf_reference_ledger(s["problem"], s["layers"])
        assert r["launches"] > 0 and r["exec_cmul"] > 0
    ex = open(tmp_path / "bench_executed.csv").read().splitlines()
    assert len(ex) == 1 + 2 * len(sizes)
