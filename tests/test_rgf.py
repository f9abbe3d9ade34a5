"""GPU layered RGF: rgf_gr + rgf_gless (rgf.cpp:181-380)
as a second, independent GPU path, checked against the reference's own RGF
outputs (tests/golden/*.rgf.out, make_golden.py rgf) and against the HSC path
(chain partition == RGF, test_hsc.cpp:648-678)."""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import refio
from paper_1305_1070_b200 import devices, negf
from tests.helpers import GOLDEN, golden_names, load_golden, rel_err

TOL = 1e-10


def _rgf_golden(name, n):
    return refio.read_result(os.path.join(GOLDEN, name + ".rgf.out"), n)


# ---------------------------------------------------------------- CPU ----
@pytest.mark.parametrize("name", golden_names())
def test_reference_rgf_equals_reference_hsc(name):
    """The pin of the cross-check itself: the reference's RGF and HSC agree."""
    rp, _, hsc, _ = load_golden(name)
    rgf = _rgf_golden(name, rp.n)
    assert rgf.status == 0 and hsc.status == 0
    assert rel_err(rgf.gr, hsc.gr) < 1e-12
    assert rel_err(rgf.gless, hsc.gless) < 1e-12


def _small_problem(layers_ok=True):
    rp, prob, _, _ = load_golden("syn_5x6_s24")
    return rp, prob


def test_rgf_plan_contract_errors():
    rp, prob = _small_problem()
    lay = [list(x) for x in rp.layers]
    plan = negf.RgfPlan(prob)
    info = plan.info()
    assert info.n_clusters == len(lay) and info.exec_cmul > 0
    with pytest.raises(negf.ContractViolation):
        plan.tree()
    with pytest.raises(negf.ContractViolation):  # not a cover
        negf.RgfPlan(prob, lay[:-1])
    with pytest.raises(negf.ContractViolation):  # overlapping
        negf.RgfPlan(prob, [lay[0] + [lay[1][0]]] + lay[1:])
    with pytest.raises(negf.PartitionViolation):  # layers 0 and 2 swapped: non-adjacent couplings
        negf.RgfPlan(prob, [lay[2], lay[1], lay[0]] + lay[3:])
    with pytest.raises(negf.ContractViolation):
        negf.RgfPlan(prob, [])


def test_rgf_plan_rejects_asymmetric_coupling_and_cross_layer_lesser():
    rp, prob = _small_problem()
    lay = [list(x) for x in rp.layers]
    a, b = lay[0][0], lay[1][0]
    bad = negf.Problem(n=prob.n, h_rows=np.r_[prob.h_rows, a], h_cols=np.r_[prob.h_cols, b],
                       h_vals=np.r_[prob.h_vals, 0.5], sr_rows=prob.sr_rows, sr_cols=prob.sr_cols,
                       sl_rows=prob.sl_rows, sl_cols=prob.sl_cols, coords=prob.coords, layers=prob.layers)
    with pytest.raises(negf.ContractViolation, match="transpose"):
        negf.RgfPlan(bad)
    bad2 = negf.Problem(n=prob.n, h_rows=prob.h_rows, h_cols=prob.h_cols, h_vals=prob.h_vals, sr_rows=prob.sr_rows,
                        sr_cols=prob.sr_cols, sl_rows=np.r_[prob.sl_rows, a], sl_cols=np.r_[prob.sl_cols, b],
                        coords=prob.coords, layers=prob.layers)
    with pytest.raises(negf.ContractViolation, match="block diagonal"):
        negf.RgfPlan(bad2)


# ---------------------------------------------------------------- GPU ----
@pytest.mark.gpu
@pytest.mark.parametrize("name", golden_names())
def test_gpu_rgf_matches_reference_rgf(name, cuda_ok):
    rp, prob, hsc, _ = load_golden(name)
    ref = _rgf_golden(name, rp.n)
    s = negf.HscGpuSolver(negf.RgfPlan(prob))
    sr, sl = rp.values(np.arange(len(rp.energies)))
    gr, gl = s.solve(rp.energies, rp.weights, sr, sl)
    assert s.last_launches > 0
    for k in range(len(rp.energies)):
        assert rel_err(gr[k], ref.gr[k]) < TOL, (name, k, rel_err(gr[k], ref.gr[k]))
        assert rel_err(gl[k], ref.gless[k]) < TOL, (name, k, rel_err(gl[k], ref.gless[k]))


@pytest.mark.gpu
def test_gpu_rgf_equals_gpu_hsc_config1(cuda_ok):
    wl = devices.config1()
    sr, sl = wl.self_energies([0])
    hs = negf.HscGpuSolver(negf.HscPlan(wl.problem))
    rs = negf.HscGpuSolver(negf.RgfPlan(wl.problem))
    g1, l1 = hs.solve(wl.energies, wl.weights, sr, sl)
    g2, l2 = rs.solve(wl.energies, wl.weights, sr, sl)
    assert rel_err(g2, g1) < TOL and rel_err(l2, l1) < TOL
    assert np.allclose(rs.density(), hs.density(), rtol=0, atol=1e-12 * np.abs(hs.density()).max())


@pytest.mark.gpu
def test_gpu_rgf_config2_slice_against_hsc(cuda_ok):
    """400 layers x 100 dofs, a few energies: the two GPU paths agree to the
    conditioning of this eta = 1e-6 workload (kappa(A) ~ 1e8, DESIGN.md §4;
    the reference's own two solvers differ by as much)."""
    wl = devices.config2(n_energies=256)
    idx = np.array([3, 77, 150, 240])
    sr, sl = wl.self_energies(idx)
    hs = negf.HscGpuSolver(negf.HscPlan(wl.problem), max_energy_batch=4)
    rs = negf.HscGpuSolver(negf.RgfPlan(wl.problem), max_energy_batch=4)
    hs.set_residual_check(False)
    rs.set_residual_check(False)
    g1, l1 = hs.solve(wl.energies[idx], wl.weights[idx], sr, sl)
    g2, l2 = rs.solve(wl.energies[idx], wl.weights[idx], sr, sl)
    for k in range(len(idx)):
        assert rel_err(g2[k], g1[k]) < 1e-6
        assert rel_err(l2[k], l1[k]) < 1e-6


@pytest.mark.gpu
def test_gpu_rgf_errors(cuda_ok):
    rp, prob, _, _ = load_golden("syn_5x6_s24")
    s = negf.HscGpuSolver(negf.RgfPlan(prob))
    sr, sl = rp.values(np.arange(len(rp.energies)))
    # a zero layer block: singular at the first energy, layer 0
    E = rp.energies.copy()
    zero = negf.Problem(n=prob.n, h_rows=prob.h_rows, h_cols=prob.h_cols, h_vals=np.zeros_like(prob.h_vals),
                        sr_rows=prob.sr_rows, sr_cols=prob.sr_cols, sl_rows=prob.sl_rows, sl_cols=prob.sl_cols,
                        coords=prob.coords, layers=prob.layers)
    z = negf.HscGpuSolver(negf.RgfPlan(zero))
    with pytest.raises(negf.SingularBlock) as ei:
        z.solve(np.zeros_like(E), rp.weights, np.zeros_like(sr), np.zeros_like(sl), first_energy_index=5)
    assert ei.value.energy_index == 5 and ei.value.cluster == 0
    if sl.shape[1]:
        bad = sl.copy()
        bad[:, 0] += 1.0  # Hermitian part on a diagonal entry
        with pytest.raises(negf.NonSkewHermitianInput):
            s.solve(E, rp.weights, sr, bad)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["syn_24x20_s5_fuzz", "superlattice_6x20_dense", "syn_5x6_s24"])
def test_gpu_chain_partition_equals_rgf(name, cuda_ok):
    """test_hsc.cpp:648-678 on the GPU: the HSC path on a chain partition (one
    cluster per layer, each layer's parent the next one) equals the layered
    RGF path to 1e-10."""
    rp, prob, _, _ = load_golden(name)
    L = [list(map(int, x)) for x in rp.layers]
    chain = negf.Problem(n=prob.n, h_rows=prob.h_rows, h_cols=prob.h_cols, h_vals=prob.h_vals,
                         sr_rows=prob.sr_rows, sr_cols=prob.sr_cols, sl_rows=prob.sl_rows, sl_cols=prob.sl_cols,
                         tree_parent=list(range(1, len(L))) + [-1], tree_dofs=L, layers=prob.layers)
    sr, sl = rp.values(np.arange(len(rp.energies)))
    g1, l1 = negf.HscGpuSolver(negf.HscPlan(chain)).solve(rp.energies, rp.weights, sr, sl)
    g2, l2 = negf.HscGpuSolver(negf.RgfPlan(prob)).solve(rp.energies, rp.weights, sr, sl)
    for k in range(len(rp.energies)):
        assert rel_err(g1[k], g2[k]) < TOL
        assert rel_err(l1[k], l2[k]) < TOL


@pytest.mark.gpu
def test_gpu_reruns_are_bitwise_identical(cuda_ok):
    """Byte-identical reruns (test_cli.cpp:396-411): no atomics on the data
    path, ordered accumulation -- two solves agree bit for bit, and so do two
    solver instances."""
    wl = devices.config1()
    sr, sl = wl.self_energies([0])
    a = negf.HscGpuSolver(negf.HscPlan(wl.problem))
    r1 = a.solve(wl.energies, wl.weights, sr, sl)
    d1 = a.density(reset=True)
    r2 = a.solve(wl.energies, wl.weights, sr, sl)
    d2 = a.density()
    b = negf.HscGpuSolver(negf.HscPlan(wl.problem))
    r3 = b.solve(wl.energies, wl.weights, sr, sl)
    for x, y in ((r1, r2), (r1, r3)):
        assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])
    assert np.array_equal(d1, d2)
