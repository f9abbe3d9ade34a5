"""CPU: the numpy restatement (oracle/hsc_numpy.py) pinned against the
reference's own outputs and stored artefacts.

* every golden problem: diag G^r / G^< of the restatement == the reference's
  hsc_fold + hsc_gless (tests/golden/*.hsc.out) and the dense oracle,
  and the FlopLedger counts are identical;
* the reference CLI artefacts proj/cli_test_tmp/solve_hsc/{density,ldos}.csv
  (copied to tests/golden/cli_*) are reproduced from the dumped device;
* closed forms of the two-leaf tree (test_hsc.cpp:126-243) and its exact
  ledger 99/78, 78, 482 (test_hsc.cpp:245-286);
* the stored bench row hsc,4,4,8192,4096 (cli_test_tmp/bench_wall/bench.csv).
"""
import csv
import os

import numpy as np
import pytest

from oracle import hsc_numpy as hn
from tests.helpers import GOLDEN, golden_names, load_golden, rel_err


@pytest.mark.parametrize("name", golden_names())
def test_restatement_matches_reference(name):
    rp, prob, hsc, dense = load_golden(name)
    tree = hn.Tree(hsc.parent, hsc.dofs, rp.n)
    sr, sl = rp.values(np.arange(len(rp.energies)))
    mul = inv = 0
    for e, E in enumerate(rp.energies):
        gr, gl, led = hn.solve_energy(tree, rp.n, rp.h_rows, rp.h_cols, rp.h_vals, prob.sr_rows, prob.sr_cols,
                                      sr[e], prob.sl_rows, prob.sl_cols, sl[e], E)
        assert rel_err(gr, hsc.gr[e]) <= 1e-12
        assert rel_err(gl, hsc.gless[e]) <= 1e-12
        if dense is not None:
            assert rel_err(gr, dense.gr[e]) <= 1e-9
            assert rel_err(gl, dense.gless[e]) <= 1e-9
        mul += led.mul
        inv += led.inv
    assert (mul, inv) == (hsc.mul_ops, hsc.inv_ops)


def _read_csv(path):
    with open(path) as f:
        rows = list(csv.reader(f))
    return rows[0], [[float(x) for x in r] for r in rows[1:]]


def test_cli_golden_csvs():
    """density.csv / ldos.csv of the reference's own test run (test_cli.cpp:83-97)."""
    rp, prob, hsc, _ = load_golden("superlattice_3x8_diag")
    tree = hn.Tree(hsc.parent, hsc.dofs, rp.n)
    sr, sl = rp.values(np.arange(len(rp.energies)))
    gls, grs = [], []
    for e, E in enumerate(rp.energies):
        gr, gl, _ = hn.solve_energy(tree, rp.n, rp.h_rows, rp.h_cols, rp.h_vals, prob.sr_rows, prob.sr_cols, sr[e],
                                    prob.sl_rows, prob.sl_cols, sl[e], E)
        grs.append(gr)
        gls.append(gl)
    dens = hn.electron_density(np.array(gls), rp.weights)  # density_scale = 1/(dx dy) = 1
    _, rows = _read_csv(os.path.join(GOLDEN, "cli_solve_hsc_density.csv"))
    nx = 3
    for x, y, v in rows:
        assert abs(dens[int(y) * nx + int(x)] - v) <= 1e-12 * max(abs(v), 1e-300) + 1e-16
    _, rows = _read_csv(os.path.join(GOLDEN, "cli_solve_hsc_ldos.csv"))
    for x, y, e, v in rows:
        k = int(np.argmin(np.abs(rp.energies - e)))
        assert abs(-grs[k][int(y) * nx + int(x)].imag / np.pi - v) <= 1e-12 * abs(v)


def _two_leaf(rng, nl=3, nr=4, ns=2):
    def rnd(r, c):
        return (rng.random((r, c)) - 0.5) + 1j * (rng.random((r, c)) - 0.5)

    def csym(n):
        r = rnd(n, n)
        return r + r.T + np.diag(4.0 - 1j * (0.5 + rng.random(n)))

    def skew(n):
        x = rnd(n, n)
        return x - x.conj().T

    a_ll, a_rr, a_ss = csym(nl), csym(nr), csym(ns)
    a_ls, a_rs = rnd(nl, ns), rnd(nr, ns)
    s_ll, s_rr, s_ss = skew(nl), skew(nr), skew(ns)
    return a_ll, a_rr, a_ss, a_ls, a_rs, s_ll, s_rr, s_ss


def two_leaf_inputs(seed=7, nl=3, nr=4, ns=2):
    rng = np.random.default_rng(seed)
    a_ll, a_rr, a_ss, a_ls, a_rs, s_ll, s_rr, s_ss = _two_leaf(rng, nl, nr, ns)
    n = nl + nr + ns
    A = np.zeros((n, n), complex)
    S = np.zeros((n, n), complex)
    L, R, Sp = slice(0, nl), slice(nl, nl + nr), slice(nl + nr, n)
    A[L, L], A[R, R], A[Sp, Sp] = a_ll, a_rr, a_ss
    A[L, Sp], A[Sp, L], A[R, Sp], A[Sp, R] = a_ls, a_ls.T, a_rs, a_rs.T
    S[L, L], S[R, R], S[Sp, Sp] = s_ll, s_rr, s_ss
    parent = [2, 2, -1]
    dofs = [list(range(nl)), list(range(nl, nl + nr)), list(range(nl + nr, n))]
    return A, S, parent, dofs, (a_ll, a_rr, a_ss, a_ls, a_rs, s_ll, s_rr, s_ss)


def closed_forms(parts):
    """test_hsc.cpp:152-176 restated."""
    a_ll, a_rr, a_ss, a_ls, a_rs, s_ll, s_rr, s_ss = parts
    inv = np.linalg.inv
    inv_l, inv_r = inv(a_ll), inv(a_rr)
    psi_l, psi_r = -inv_l @ a_ls, -inv_r @ a_rs
    g_ss = inv(a_ss + a_ls.T @ psi_l + a_rs.T @ psi_r)
    g_ls, g_rs = psi_l @ g_ss, psi_r @ g_ss
    g_ll, g_rr = inv_l + psi_l @ g_ls.T, inv_r + psi_r @ g_rs.T
    n_ss = s_ss @ g_ss.conj() + psi_l.T @ (s_ll @ g_ls.conj()) + psi_r.T @ (s_rr @ g_rs.conj())
    gl_ss = g_ss @ n_ss
    gl_ls = inv_l @ (s_ll @ g_ls.conj()) + psi_l @ gl_ss
    gl_rs = inv_r @ (s_rr @ g_rs.conj()) + psi_r @ gl_ss
    gl_ll = inv_l @ (s_ll @ g_ll.conj()) - psi_l @ gl_ls.conj().T
    gl_rr = inv_r @ (s_rr @ g_rr.conj()) - psi_r @ gl_rs.conj().T
    return (g_ll, g_rr, g_ss), (gl_ll, gl_rr, gl_ss)


def test_two_leaf_closed_forms_and_ledger():
    A, S, parent, dofs, parts = two_leaf_inputs()
    n = A.shape[0]
    tree = hn.Tree(parent, dofs, n)
    r, c = np.nonzero(A)
    blocks = hn.group_by_partition(tree, r, c, A[r, c])
    fold = hn.Ledger()
    psi, inv = hn.hsc_fold(tree, blocks, fold)
    assert (fold.inv, fold.mul) == (99, 78)  # test_hsc.cpp:268-269
    rs, cs = np.nonzero(S)
    view = hn.validate_sigma(tree, hn.group_by_partition(tree, rs, cs, S[rs, cs]))
    led = hn.Ledger()
    gd, pd = hn.hsc_gless(tree, psi, inv, view, led)
    assert led.mul == 482 and led.inv == 0  # test_hsc.cpp:279-283
    led_gr = hn.Ledger()
    hn.hsc_gless(tree, psi, inv, {}, led_gr)
    assert led_gr.mul == 78  # test_hsc.cpp:274
    g, gl = closed_forms(parts)
    for cl in range(3):
        assert np.abs(gd[cl] - g[cl]).max() <= 1e-11
        assert np.abs(pd[cl] - gl[cl]).max() <= 1e-11
        assert hn.skew_defect(pd[cl]) <= 1e-12


def test_bench_row_ledger():
    """hsc,4,4,8192,4096 (proj/cli_test_tmp/bench_wall/bench.csv:3)."""
    rp, prob, hsc, _ = load_golden("syn_4x4_s1_bench")
    assert (hsc.mul_ops, hsc.inv_ops) == (8192, 4096)
    tree = hn.Tree(hsc.parent, hsc.dofs, rp.n)
    sr, sl = rp.values([0])
    _, _, led = hn.solve_energy(tree, rp.n, rp.h_rows, rp.h_cols, rp.h_vals, prob.sr_rows, prob.sr_cols, sr[0],
                                prob.sl_rows, prob.sl_cols, sl[0], 0.0)
    assert (led.mul, led.inv) == (8192, 4096)
    with open(os.path.join(GOLDEN, "cli_bench_wall_bench.csv")) as f:
        assert "hsc,4,4,8192,4096," in f.read()


def test_singular_missing_block():
    """A missing diagonal block folds as zero -> SingularBlock (test_hsc.cpp:904-916)."""
    A, S, parent, dofs, _ = two_leaf_inputs(43, 2, 2, 2)
    A[0:2, 0:2] = 0
    tree = hn.Tree(parent, dofs, 6)
    r, c = np.nonzero(A)
    with pytest.raises(hn.SingularBlock):
        hn.hsc_fold(tree, hn.group_by_partition(tree, r, c, A[r, c]), hn.Ledger())


def test_sigma_validation():
    A, S, parent, dofs, _ = two_leaf_inputs(41, 2, 2, 2)
    tree = hn.Tree(parent, dofs, 6)
    bad = S.copy()
    bad[2:4, 2:4] = bad[2:4, 2:4] + bad[2:4, 2:4].conj().T + np.eye(2)  # Hermitian part
    rs, cs = np.nonzero(bad)
    with pytest.raises(hn.NonSkewHermitian):
        hn.validate_sigma(tree, hn.group_by_partition(tree, rs, cs, bad[rs, cs]))
    off = S.copy()
    off[0, 5] = 1.0
    rs, cs = np.nonzero(off)
    with pytest.raises(hn.ContractViolation):
        hn.validate_sigma(tree, hn.group_by_partition(tree, rs, cs, off[rs, cs]))
