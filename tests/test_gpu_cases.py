"""GPU: fixtures of the reference's own unit tests (test_hsc.cpp) restated,
error semantics, edge cases and host-side behaviour of the C ABI."""
import numpy as np
import pytest

from oracle import hsc_numpy as hn
from paper_1305_1070_b200 import negf
from tests.helpers import load_golden, rel_err
from tests.test_oracle import closed_forms, two_leaf_inputs

pytestmark = pytest.mark.gpu


def dense_problem(A, S, parent, dofs):
    """Explicit-tree problem with A = -H at E = 0 and Sigma^< given densely."""
    n = A.shape[0]
    r, c = np.nonzero(A)
    rs, cs = np.nonzero(S)
    prob = negf.Problem(n=n, h_rows=r, h_cols=c, h_vals=-A[r, c], sl_rows=rs, sl_cols=cs,
                        tree_parent=parent, tree_dofs=dofs)
    return prob, S[rs, cs]


def test_two_leaf_closed_forms(cuda_ok):
    A, S, parent, dofs, parts = two_leaf_inputs()
    prob, sl = dense_problem(A, S, parent, dofs)
    s = negf.HscGpuSolver(negf.HscPlan(prob))
    gr, gl = s.solve([0.0], [1.0], None, sl[None, :])
    g, glb = closed_forms(parts)
    want_gr = np.concatenate([np.diag(b) for b in g])
    want_gl = np.concatenate([np.diag(b) for b in glb])
    assert np.abs(gr[0] - want_gr).max() <= 1e-11
    assert np.abs(gl[0] - want_gl).max() <= 1e-11
    # dense oracle settles the signs independently (test_hsc.cpp:216-236)
    gd = np.linalg.inv(A)
    assert np.abs(gr[0] - np.diag(gd)).max() <= 1e-10
    assert np.abs(gl[0] - np.diag(gd @ S @ gd.conj().T)).max() <= 1e-10


def test_five_cluster_and_grandparent(cuda_ok):
    """Five-cluster layout 0,1 -> 2; 2,3 -> 4 (test_hsc.cpp:293-562) and the
    grandparent-only leaf (727-805), against the dense oracle."""
    rng = np.random.default_rng(31)
    for sizes, parent, pairs in (
        ([2, 3, 2, 2, 3], [2, 2, 4, 4, -1], [(0, 2), (0, 4), (1, 2), (1, 4), (2, 4), (3, 4)]),
        ([2, 2, 2], [1, 2, -1], [(0, 2), (1, 2)]),
    ):
        off = np.cumsum([0] + sizes)
        n = off[-1]
        A = np.zeros((n, n), complex)
        S = np.zeros((n, n), complex)
        for c, m in enumerate(sizes):
            r = rng.random((m, m)) - 0.5 + 1j * (rng.random((m, m)) - 0.5)
            A[off[c]:off[c + 1], off[c]:off[c + 1]] = r + r.T + np.diag(4.0 - 1j * (0.5 + rng.random(m)))
            x = rng.random((m, m)) - 0.5 + 1j * (rng.random((m, m)) - 0.5)
            S[off[c]:off[c + 1], off[c]:off[c + 1]] = x - x.conj().T
        for a, b in pairs:
            blk = rng.random((sizes[a], sizes[b])) - 0.5 + 1j * (rng.random((sizes[a], sizes[b])) - 0.5)
            A[off[a]:off[a + 1], off[b]:off[b + 1]] = blk
            A[off[b]:off[b + 1], off[a]:off[a + 1]] = blk.T
        dofs = [list(range(off[c], off[c + 1])) for c in range(len(sizes))]
        prob, sl = dense_problem(A, S, parent, dofs)
        gr, gl = negf.HscGpuSolver(negf.HscPlan(prob)).solve([0.0], [1.0], None, sl[None, :])
        gd = np.linalg.inv(A)
        assert np.abs(gr[0] - np.diag(gd)).max() <= 1e-11
        assert np.abs(gl[0] - np.diag(gd @ S @ gd.conj().T)).max() <= 1e-11


def singular_problem():
    """Leaf 0 has H_00 = 0.5 I and no other diagonal shift: A_00(E=0.5) = 0."""
    A, S, parent, dofs, _ = two_leaf_inputs(5, 2, 2, 2)
    H = -A.copy()
    H[0:2, 0:2] = 0.5 * np.eye(2)
    r, c = np.nonzero(H)
    rs, cs = np.nonzero(S)
    prob = negf.Problem(n=6, h_rows=r, h_cols=c, h_vals=H[r, c], sl_rows=rs, sl_cols=cs, tree_parent=parent,
                        tree_dofs=dofs)
    return prob, S[rs, cs]


def test_singular_block_lowest_energy_wins(cuda_ok):
    prob, sl = singular_problem()
    s = negf.HscGpuSolver(negf.HscPlan(prob))
    E = np.array([0.1, 0.5, 0.7, 0.5])
    with pytest.raises(negf.SingularBlock) as ei:
        s.solve(E, np.ones(4), None, np.tile(sl, (4, 1)), first_energy_index=10)
    assert ei.value.energy_index == 11
    assert ei.value.pivot_index == 0
    assert ei.value.cluster == 0
    # chunked into batches of one energy: same answer
    s1 = negf.HscGpuSolver(negf.HscPlan(prob), max_energy_batch=1)
    with pytest.raises(negf.SingularBlock) as ei:
        s1.solve(E, np.ones(4), None, np.tile(sl, (4, 1)), first_energy_index=10)
    assert ei.value.energy_index == 11


def test_non_skew_sigma_and_precedence(cuda_ok):
    prob, sl = singular_problem()
    s = negf.HscGpuSolver(negf.HscPlan(prob))
    bad = np.tile(sl, (3, 1))
    bad[0] = np.abs(bad[0])  # real positive entries: Hermitian, not skew
    with pytest.raises(negf.NonSkewHermitianInput) as ei:
        s.solve(np.array([0.1, 0.2, 0.3]), np.ones(3), None, bad)
    assert ei.value.energy_index == 0
    # energy 0: non-skew, energy 1 singular -> energy 0 wins (lowest index)
    with pytest.raises(negf.NonSkewHermitianInput):
        s.solve(np.array([0.1, 0.5, 0.3]), np.ones(3), None, bad)
    # same energy: the fold's SingularBlock comes first (run.cpp:164-169)
    with pytest.raises(negf.SingularBlock):
        s.solve(np.array([0.5, 0.2, 0.3]), np.ones(3), None, bad)


def test_chunking_density_and_nccl_single_rank(cuda_ok):
    rp, prob, hsc, _ = load_golden("syn_24x20_s5_fuzz")
    sr, sl = rp.values(np.arange(3))
    E = np.array([rp.energies[0], rp.energies[1], rp.energies[2], rp.energies[0], rp.energies[1]])
    W = np.array([0.1, 0.2, 0.3, 0.4, 0.5])
    SR, SL = sr[[0, 1, 2, 0, 1]], sl[[0, 1, 2, 0, 1]]
    big = negf.HscGpuSolver(negf.HscPlan(prob), max_energy_batch=8)
    small = negf.HscGpuSolver(negf.HscPlan(prob), max_energy_batch=2)
    g1, l1 = big.solve(E, W, SR, SL)
    g2, l2 = small.solve(E, W, SR, SL)
    assert np.array_equal(g1, g2) and np.array_equal(l1, l2)
    d = big.density()
    assert np.allclose(d, (W[:, None] * l1.imag).sum(0) / (2 * np.pi), rtol=1e-13, atol=0)
    # a second call accumulates; reset clears
    big.solve(E[:1], W[:1], SR[:1], SL[:1], want_diagonals=False)
    d2 = big.density(reset=True)
    assert np.allclose(d2, d + W[0] * l1[0].imag / (2 * np.pi), rtol=1e-13, atol=0)
    assert np.all(big.density() == 0)
    # one-rank NCCL communicator: the allreduce path is exercised, sum unchanged
    small.density(reset=True)
    small.solve(E, W, SR, SL, want_diagonals=False)
    before = small.density()
    small.nccl_init(negf.nccl_unique_id(), 1, 0)
    small.allreduce_density()
    assert np.array_equal(small.density(), before)


def test_empty_root_separator(cuda_ok):
    """Disconnected device: the artificial empty root (m = 0) flows through."""
    n = 8
    rng = np.random.default_rng(3)
    H = np.zeros((n, n), complex)
    for blk in (slice(0, 4), slice(4, 8)):
        r = rng.random((4, 4)) - 0.5
        H[blk, blk] = r + r.T + 3 * np.eye(4)
    coords = np.array([[0, 0], [1, 0], [2, 0], [3, 0], [20, 0], [21, 0], [22, 0], [23, 0]], float)
    r, c = np.nonzero(H)
    S = np.zeros((n, n), complex)
    S[0, 0], S[7, 7] = 0.3j, 0.2j
    prob = negf.Problem(n=n, h_rows=r, h_cols=c, h_vals=H[r, c], sr_rows=[0, 7], sr_cols=[0, 7],
                        sl_rows=[0, 7], sl_cols=[0, 7], coords=coords, max_leaf=4)
    plan = negf.HscPlan(prob)
    t = plan.tree()
    assert len(t.dofs[t.root]) == 0
    sr = np.array([[-0.05j, -0.07j]])
    gr, gl = negf.HscGpuSolver(plan).solve([0.3], [1.0], sr, np.array([[0.3j, 0.2j]]))
    A = 0.3 * np.eye(n) - H
    A[0, 0] += 0.05j
    A[7, 7] += 0.07j
    g = np.linalg.inv(A)
    assert rel_err(gr[0], np.diag(g)) <= 1e-12
    assert rel_err(gl[0], np.diag(g @ S @ g.conj().T)) <= 1e-12


def test_residual_guard_records(cuda_ok):
    rp, prob, hsc, _ = load_golden("superlattice_6x20_dense")
    sr, sl = rp.values(np.arange(len(rp.energies)))
    s = negf.HscGpuSolver(negf.HscPlan(prob))
    s.set_residual_check(False)
    s.solve(rp.energies, rp.weights, sr, sl)
    assert 0.0 <= s.max_real_residual < 1e-8


@pytest.mark.gpu
def test_density_accumulator_device_view(cuda_ok):
    """The solver's device density accumulator can be viewed zero-copy from
    torch (bench.py's fallback reduction over the torch process group)."""
    import torch

    rp, prob, _, _ = load_golden("syn_24x20_s5_fuzz")
    s = negf.HscGpuSolver(negf.HscPlan(prob))
    sr, sl = rp.values(np.arange(len(rp.energies)))
    s.solve(rp.energies, rp.weights, sr, sl)

    class View:
        def __init__(self, ptr, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}

    t = torch.as_tensor(View(s.density_ptr, rp.n), device="cuda")
    dens = s.density()
    assert np.allclose(t.cpu().numpy() / (2 * np.pi), dens, rtol=1e-15, atol=0)
    t.mul_(2.0)  # writes through to the accumulator
    torch.cuda.synchronize()
    assert np.allclose(s.density(), 2 * dens, rtol=1e-15, atol=0)


@pytest.mark.parametrize("m", [113, 700, 2048])
def test_large_block_inverse_any_size(m, cuda_ok):
    """The multi-CTA blocked Gauss-Jordan (rank-64 outer updates) on one
    cluster of m dofs, no size cap (inverse, dense.cpp:49-81 has none):
    diag G^r = diag(A^-1) and diag G^< = diag(A^-1 S A^-H) against numpy, for
    a random complex-symmetric A with row interchanges at most pivots; two
    energies (a batch of arenas), a 2x2 dense skew Sigma^< block."""
    rng = np.random.default_rng(m)
    B = (rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))) / np.sqrt(m)
    A = B + B.T
    S = np.zeros((m, m), complex)
    S[:2, :2] = [[1j, 0.3 + 0.2j], [-0.3 + 0.2j, 0.5j]]  # skew-Hermitian
    prob, sl = dense_problem(A, S, [-1], [list(range(m))])
    s = negf.HscGpuSolver(negf.HscPlan(prob))
    E = np.array([0.0, 0.25])
    gr, gl = s.solve(E, [1.0, 1.0], None, np.stack([sl, sl]))
    for q, e in enumerate(E):
        ginv = np.linalg.inv(A + e * np.eye(m))  # A(E) = E I - H with H = -A
        assert rel_err(gr[q], np.diag(ginv)) <= 1e-10
        want = np.einsum("ij,jk,ik->i", ginv, S, ginv.conj())
        assert rel_err(gl[q], want) <= 1e-10


def test_large_block_singular_pivot(cuda_ok):
    """A rank-deficient 300-dof block: SingularBlock with the pivot index of
    the reference's partial-pivoting rule |u_kk| <= 1e-13 max|a|."""
    m = 300
    rng = np.random.default_rng(3)
    U = rng.standard_normal((m, 150)) + 1j * rng.standard_normal((m, 150))
    A = U @ U.T  # complex symmetric, rank 150
    prob, sl = dense_problem(A, np.zeros((m, m), complex), [-1], [list(range(m))])
    s = negf.HscGpuSolver(negf.HscPlan(prob))
    with pytest.raises(negf.SingularBlock) as ei:
        s.solve([0.0], [1.0], None, None)
    assert ei.value.pivot_index == 150 and ei.value.energy_index == 0
