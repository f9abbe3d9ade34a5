"""Contact self-energies: the reference's
surface_self_energy (device.cpp:195-251) and lesser_self_energy
(device.cpp:322-366) on the GPU.

CPU tests pin the oracle restatement (oracle/lead_numpy.py) against the Sigma
blocks the reference itself wrote (tests/golden/lead_*.{bin,out}, the dense
leads inside *_dense.bin) and check the host-side contract errors; GPU tests
compare the batched kernels with the goldens / oracle (tolerance 1e-10
relative, the north_star bound) and the GPU self-energy pipeline with the
host generators of devices.py."""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import lead_numpy, refio
from paper_1305_1070_b200 import devices, negf
from tests.helpers import GOLDEN, dense_block, lead_names, rel_err

TOL = 1e-10
DEVICE_LEADS = [("superlattice_6x20_dense", 1e-4), ("graphene_8x16_dense", 1e-4)]


def _lead_fixture(name):
    w, eta, h00, h01, e = refio.read_lead(os.path.join(GOLDEN, name + ".bin"))
    codes, sig = refio.read_lead_out(os.path.join(GOLDEN, name + ".out"), w)
    return w, eta, h00, h01, e, codes, sig


def _device_leads(name):
    rp = refio.read_problem(os.path.join(GOLDEN, name + ".bin"))
    h = lambda r, c: dense_block(rp, r, c)  # noqa: E731
    left = lead_numpy.lead_blocks(h, rp.layers, "left")
    right = lead_numpy.lead_blocks(h, rp.layers, "right")
    return rp, left, right


# ---------------------------------------------------------------- CPU ----
@pytest.mark.parametrize("name", lead_names())
def test_oracle_lead_pinned_to_reference(name):
    w, eta, h00, h01, e, codes, sig = _lead_fixture(name)
    assert len(e) >= 2
    for k, en in enumerate(e):
        if codes[k] == 1:
            with pytest.raises(lead_numpy.ConvergenceError):
                lead_numpy.surface_self_energy(h00, h01, en, eta)
            continue
        assert codes[k] == 0
        s = lead_numpy.surface_self_energy(h00, h01, en, eta)
        assert rel_err(s, sig[k]) < 1e-12
        assert np.array_equal(s, s.T)


@pytest.mark.parametrize("name,eta", DEVICE_LEADS)
def test_oracle_lead_blocks_from_device_goldens(name, eta):
    """attach_contacts' block extraction + decimation reproduce the Sigma the
    reference stored in its own device dumps."""
    rp, (h00l, h01l), (h00r, h01r) = _device_leads(name)
    for k, en in enumerate(rp.energies):
        assert rel_err(lead_numpy.surface_self_energy(h00l, h01l, en, eta), rp.sig_l[k]) < 1e-12
        assert rel_err(lead_numpy.surface_self_energy(h00r, h01r, en, eta), rp.sig_r[k]) < 1e-12


def test_oracle_lesser_from_device_golden():
    """-f (S - S^H) at the dump's chemical potential (superlattice: mu = 0.25,
    300 K, the config's defaults)."""
    rp = refio.read_problem(os.path.join(GOLDEN, "superlattice_6x20_dense.bin"))
    kT = lead_numpy.K_BOLTZMANN_EV_PER_K * 300.0
    for k, en in enumerate(rp.energies):
        f = lead_numpy.fermi(en, 0.25, kT)
        assert rel_err(lead_numpy.lesser_block(rp.sig_l[k], f), rp.less_l[k]) < 1e-14
        assert rel_err(lead_numpy.lesser_block(rp.sig_r[k], f), rp.less_r[k]) < 1e-14


def test_lead_contract_errors_host_side():
    h = np.eye(4, dtype=np.complex128)
    with pytest.raises(negf.ConfigError):
        negf.SurfaceLead(h, h, 0.0)
    with pytest.raises(negf.ContractViolation):
        negf.SurfaceLead(h, np.eye(3), 1e-6)
    with pytest.raises(negf.ContractViolation):
        negf.SurfaceLead(np.ones((4, 3)), h, 1e-6)
    with pytest.raises(negf.ContractViolation):
        negf.SurfaceLead(h, h, 1e-6, criterion="nope")


def test_workload_contact_recipes():
    """Every BASELINE workload carries a GPU self-energy recipe whose pattern
    offsets agree with the host generator's layout."""
    for w in (devices.config1(), devices.config3(n_energies=4, n_cells=6),
              devices.config5(n_energies=4, nx=12, ny=10)):
        c = w.contacts
        assert c is not None and c["kind"] in ("modes", "sancho")
        sr, sl = w.self_energies([0])
        w2 = c["w"] ** 2
        for ld in c["leads"]:
            assert np.any(sr[0, ld["sr_off"]:ld["sr_off"] + w2] != 0)
            assert np.any(sl[0, ld["sl_off"]:ld["sl_off"] + w2] != 0)


# ---------------------------------------------------------------- GPU ----
@pytest.mark.gpu
@pytest.mark.parametrize("name", lead_names())
def test_gpu_lead_matches_reference_goldens(name, cuda_ok):
    w, eta, h00, h01, e, codes, sig = _lead_fixture(name)
    lead = negf.SurfaceLead(h00, h01, eta)
    ok = np.nonzero(codes == 0)[0]
    out = lead.sigma(e[ok])
    sweeps = lead.last_sweeps(len(ok))
    assert lead.last_launches > 0
    for q, k in enumerate(ok):
        assert rel_err(out[q], sig[k]) < TOL, (name, e[k], rel_err(out[q], sig[k]))
        assert np.array_equal(out[q], out[q].T)
        _, sw = lead_numpy.surface_self_energy(h00, h01, e[k], eta, return_sweeps=True)
        assert sweeps[q] == sw
    for k in np.nonzero(codes == 1)[0]:
        with pytest.raises(negf.ConvergenceError) as ei:
            lead.sigma(e[k:k + 1], first_energy_index=int(k))
        assert ei.value.energy_index == k


@pytest.mark.gpu
def test_gpu_lead_error_precedence_and_chunking(cuda_ok):
    """Lowest failing energy wins (run.cpp:258-262) across chunks; chunked
    and device-resident calls agree with one batch."""
    import torch

    w, eta, h00, h01, e, codes, sig = _lead_fixture("lead_cnt80")
    bad = int(np.nonzero(codes == 1)[0][0])
    lead = negf.SurfaceLead(h00, h01, eta, max_energy_batch=2)
    with pytest.raises(negf.ConvergenceError) as ei:
        lead.sigma(e, first_energy_index=100)
    assert ei.value.energy_index == 100 + bad
    ok = np.nonzero(codes == 0)[0]
    full = negf.SurfaceLead(h00, h01, eta).sigma(e[ok])
    chunked = lead.sigma(e[ok])
    assert np.array_equal(full, chunked)
    ld = w * w + 7
    dE = torch.from_numpy(e[ok].copy()).cuda()
    buf = torch.zeros(len(ok) * ld, dtype=torch.complex128, device="cuda")
    lead.sigma_device(dE, buf, ld=ld)
    got = buf.cpu().numpy()
    for q in range(len(ok)):
        assert np.array_equal(got[q * ld:q * ld + w * w].reshape(w, w), full[q])
        assert np.all(got[q * ld + w * w:(q + 1) * ld] == 0)


@pytest.mark.gpu
@pytest.mark.parametrize("name,eta", DEVICE_LEADS)
def test_gpu_lead_from_device_goldens(name, eta, cuda_ok):
    rp, (h00l, h01l), (h00r, h01r) = _device_leads(name)
    sl = negf.SurfaceLead(h00l, h01l, eta).sigma(rp.energies)
    sr = negf.SurfaceLead(h00r, h01r, eta).sigma(rp.energies)
    for k in range(len(rp.energies)):
        assert rel_err(sl[k], rp.sig_l[k]) < TOL
        assert rel_err(sr[k], rp.sig_r[k]) < TOL


@pytest.mark.gpu
def test_gpu_lead_decay_criterion_matches_host_sancho_rubio(cuda_ok):
    h00, h01 = devices._cnt_cell(20, -2.7)
    e = devices.uniform_grid(-1.0, 1.0, 512)[::53]
    for h in (h01.T.copy(), h01):
        lead = negf.SurfaceLead(h00, h, 1e-6, criterion="decay", tol=1e-12)
        got = lead.sigma(e)
        for k, en in enumerate(e):
            assert rel_err(got[k], devices.sancho_rubio(en, 1e-6, h00, h)) < TOL


@pytest.mark.gpu
@pytest.mark.parametrize("w", [100, 37])
def test_gpu_modes_sigma_matches_host(w, cuda_ok):
    import torch

    t = devices.HBAR2_OVER_2M0 / (0.067 * 0.25)
    phi, eps = devices._lead_modes(w, t)
    e = devices.uniform_grid(0.0, 0.4, 16)
    out = torch.empty((len(e), w, w), dtype=torch.complex128, device="cuda")
    negf.lead_modes_sigma_device(w, t, 1e-6, torch.from_numpy(e).cuda(), out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    for k, en in enumerate(e):
        ref = devices.analytic_lead_sigma(en, 1e-6, t, phi, eps)
        assert rel_err(got[k], ref) < 1e-12
        assert np.array_equal(got[k], got[k].T)


def _gpu_vs_host_self_energies(wl, idx):
    import torch

    gen = devices.GpuSelfEnergies(wl)
    e = torch.from_numpy(wl.energies[idx].copy()).cuda()
    sr, sl = gen(e)
    torch.cuda.synchronize()
    hr, hl = wl.self_energies(idx)
    return sr.cpu().numpy(), sl.cpu().numpy(), hr, hl


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["cfg1", "cfg3_short", "cfg5_small", "cfg2_complex_energy"])
def test_gpu_self_energies_match_host_generators(which, cuda_ok):
    if which == "cfg1":
        wl, idx = devices.config1(), np.array([0])
    elif which == "cfg3_short":
        wl, idx = devices.config3(n_energies=16, n_cells=8), np.arange(0, 16, 3)
    elif which == "cfg5_small":
        wl, idx = devices.config5(n_energies=12, nx=20, ny=14), np.arange(12)
    else:
        wl = devices.effective_mass_device("em_ce", 30, 12, 0.5, 0.067, np.zeros(360), np.linspace(0.01, 0.3, 6),
                                           1e-6, 0.1, 0.0, 0.025, complex_energy=True)
        idx = np.arange(6)
    sr, sl, hr, hl = _gpu_vs_host_self_energies(wl, idx)
    assert sr.shape == hr.shape and sl.shape == hl.shape
    for k in range(len(idx)):
        assert rel_err(sr[k], hr[k]) < 1e-12
        # Sigma^< = -f (S - S^H) cancels: measure on the scale of Sigma^r
        assert np.abs(sl[k] - hl[k]).max() <= 1e-12 * np.abs(hr[k]).max()


@pytest.mark.gpu
def test_gpu_solve_with_gpu_self_energies(cuda_ok):
    """Energies only on the host: GPU Sigma -> GPU HSC equals host Sigma -> GPU HSC."""
    import torch

    wl = devices.config5(n_energies=6, nx=24, ny=16)
    plan = negf.HscPlan(wl.problem)
    s = negf.HscGpuSolver(plan, max_energy_batch=6)
    E = torch.from_numpy(wl.energies.copy()).cuda()
    W = torch.from_numpy(wl.weights.copy()).cuda()
    sr, sl = devices.GpuSelfEnergies(wl)(E)
    torch.cuda.synchronize()  # the solver runs on its own stream
    gr = torch.empty((6, wl.n), dtype=torch.complex128, device="cuda")
    gl = torch.empty_like(gr)
    s.solve_device(E, W, sr, sl, out_gr=gr, out_gless=gl)
    hr, hl = wl.self_energies(np.arange(6))
    ref_gr, ref_gl = s.solve(wl.energies, wl.weights, hr, hl)
    assert rel_err(gr.cpu().numpy(), ref_gr) < 1e-10
    assert rel_err(gl.cpu().numpy(), ref_gl) < 1e-10
