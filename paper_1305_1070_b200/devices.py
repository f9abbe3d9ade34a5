"""Seeded synthetic devices for the BASELINE.json configurations.

Input generation only (outside the drop-in boundary): each builder returns a
``Workload`` whose ``problem`` goes to the C ABI unchanged and whose
``self_energies(idx)`` yields the per-energy Sigma^r / Sigma^< pattern values.

Conventions fixed here (the reference leaves them open):
* dof = x * Ny + y with x the transport coordinate (layers are columns x),
  coords = (x, y) by default: the top separator of config 4 is then the
  1024-dof column the BASELINE names;
* A(E) = E I - H - Sigma^r(E) with real E and eta only inside the lead
  self-energies -- the reference CLI convention (block.cpp:141-146,
  device.cpp:207) -- for every config by default (``complex_energy=False``).
  ``complex_energy=True`` adds -i*eta on every dof through the Sigma^r pattern
  (the reference's phonon-diagonal slot, with no Sigma^< counterpart), i.e.
  A = (E + i eta) I - H - Sigma, the BASELINE wording ("E + i eta"); at
  eta = 1e-6 it does not cure the ill-conditioned energies;
* ``ref_orientation`` (config 4) puts the within-layer index in coordinate 0
  as the reference builders do (device.cpp:120-121): nested dissection then
  merges a dense contact into the top separator (a 2557-dof root);
* random draws: std::mt19937_64(seed) + uniform01 (synthetic.hpp:18-20), onsite
  potential first in dof order, then any further draws;
* effective-mass leads: analytic semi-infinite uniform lead,
  Sigma = -t sum_m phi_m phi_m^T lambda_m, lambda_m = e^{i k_m a};
* the CNT lead: Sancho-Rubio decimation of the ideal tube (tolerance 1e-12);
* Sigma^< = -f (Sigma - Sigma^dagger) per contact (= i f Gamma), phonon
  Sigma^<_ph = -f_eq (s - conj s) (device.cpp:322-360); phonon self-energy is
  zero on the two boundary layers (device.cpp:313-318).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from .negf import Problem, trapezoid_weights
from .rng import MT19937_64

HBAR2_OVER_2M0 = 0.0380998  # eV nm^2 (device.hpp:20)


def fermi(e, mu, kT):
    x = (np.asarray(e, np.float64) - mu) / kT
    with np.errstate(over="ignore"):
        f = 1.0 / (1.0 + np.exp(np.clip(x, -700.0, 700.0)))
    f = np.where(x > 700.0, 0.0, np.where(x < -700.0, 1.0, f))
    return f


def uniform_grid(emin: float, emax: float, count: int) -> np.ndarray:
    """uniform_energy_grid (observables.cpp:34-49)."""
    if count == 1:
        return np.array([emin], np.float64)
    step = (emax - emin) / (count - 1)
    e = emin + step * np.arange(count, dtype=np.float64)
    e[-1] = emax
    return e


@dataclass
class Workload:
    name: str
    problem: Problem
    energies: np.ndarray
    weights: np.ndarray
    self_energies: Callable[[np.ndarray], tuple]
    nx: int
    ny: int
    description: str = ""
    contacts: dict | None = None  # GPU self-energy recipe (GpuSelfEnergies)

    @property
    def n(self) -> int:
        return self.problem.n


def _lead_modes(ny: int, t: float):
    y = np.arange(1, ny + 1)
    m = np.arange(1, ny + 1)
    phi = np.sqrt(2.0 / (ny + 1)) * np.sin(np.outer(y, m) * np.pi / (ny + 1))  # (y, m)
    eps = 4.0 * t - 2.0 * t * np.cos(m * np.pi / (ny + 1))
    return phi, eps


def analytic_lead_sigma(energy: float, eta: float, t: float, phi: np.ndarray, eps: np.ndarray) -> np.ndarray:
    """Retarded surface self-energy of a uniform semi-infinite 2D lead."""
    z = (eps - (energy + 1j * eta)) / (2.0 * t)
    s = np.sqrt(z * z - 1.0 + 0j)
    lam = z - s
    flip = np.abs(lam) > 1.0
    lam[flip] = (z + s)[flip]
    sig = (phi * (-t * lam)) @ phi.T
    return 0.5 * (sig + sig.T)  # exactly complex symmetric


def effective_mass_device(name: str, nx: int, ny: int, a_nm: float, m_eff: float, potential: np.ndarray,
                          energies: np.ndarray, eta: float, mu_l: float, mu_r: float, kT: float,
                          phonon_gamma: np.ndarray | None = None, max_leaf: int = 64,
                          description: str = "", complex_energy: bool = False,
                          ref_orientation: bool = False) -> Workload:
    t = HBAR2_OVER_2M0 / (m_eff * a_nm * a_nm)
    n = nx * ny
    idx = np.arange(n).reshape(nx, ny)  # dof = x*ny + y
    rows = [idx.ravel()]
    cols = [idx.ravel()]
    vals = [4.0 * t + potential.reshape(n)]
    for a, b in ((idx[:-1, :], idx[1:, :]), (idx[:, :-1], idx[:, 1:])):
        rows += [a.ravel(), b.ravel()]
        cols += [b.ravel(), a.ravel()]
        vals += [np.full(a.size, -t), np.full(a.size, -t)]
    h_rows = np.concatenate(rows).astype(np.int32)
    h_cols = np.concatenate(cols).astype(np.int32)
    h_vals = np.concatenate(vals).astype(np.complex128)
    coords = np.stack([np.repeat(np.arange(nx), ny), np.tile(np.arange(ny), nx)], 1).astype(np.float64)
    if ref_orientation:  # the reference builders' convention: within-layer index first (device.cpp:120-121)
        coords = coords[:, ::-1].copy()
    left, right = idx[0], idx[-1]
    lr, lc = np.meshgrid(left, left, indexing="ij")
    rr, rc = np.meshgrid(right, right, indexing="ij")
    sr_rows = [lr.ravel(), rr.ravel()]
    sr_cols = [lc.ravel(), rc.ravel()]
    interior = idx[1:-1].ravel()
    if phonon_gamma is not None:
        sr_rows.append(interior)
        sr_cols.append(interior)
    sl_rows = np.concatenate(sr_rows).astype(np.int32)
    sl_cols = np.concatenate(sr_cols).astype(np.int32)
    n_lesser = len(sl_rows)
    if complex_energy:  # -i eta on every dof: A = (E + i eta) I - H - Sigma
        sr_rows.append(np.arange(n))
        sr_cols.append(np.arange(n))
    sr_rows = np.concatenate(sr_rows).astype(np.int32)
    sr_cols = np.concatenate(sr_cols).astype(np.int32)
    prob = Problem(n=n, h_rows=h_rows, h_cols=h_cols, h_vals=h_vals, sr_rows=sr_rows, sr_cols=sr_cols,
                   sl_rows=sl_rows, sl_cols=sl_cols, coords=coords,
                   atomic_groups=[left.tolist(), right.tolist()], max_leaf=max_leaf,
                   layers=[idx[x].tolist() for x in range(nx)])
    phi, eps = _lead_modes(ny, t)
    w2 = ny * ny
    gam = None if phonon_gamma is None else np.asarray(phonon_gamma).reshape(n)[interior]
    mu_ph = 0.5 * (mu_l + mu_r)

    def self_energies(sel):
        sel = np.atleast_1d(np.asarray(sel))
        nnz = len(sr_rows)
        sr = np.zeros((len(sel), nnz), np.complex128)
        sl = np.zeros((len(sel), n_lesser), np.complex128)
        if complex_energy:
            sr[:, n_lesser:] = -1j * eta
        for q, k in enumerate(sel):
            e = float(energies[k])
            sig = analytic_lead_sigma(e, eta, t, phi, eps)  # same uniform lead on both sides
            sr[q, :w2] = sig.ravel()
            sr[q, w2:2 * w2] = sig.ravel()
            for side, mu in ((0, mu_l), (1, mu_r)):
                sl[q, side * w2:(side + 1) * w2] = (-fermi(e, mu, kT) * (sig - sig.conj().T)).ravel()
            if gam is not None:
                s = -1j * gam
                sr[q, 2 * w2:n_lesser] = s
                sl[q, 2 * w2:] = -fermi(e, mu_ph, kT) * (s - np.conj(s))
        return sr, sl

    contacts = dict(kind="modes", w=ny, t=t, eta=eta, kT=kT,
                    leads=[dict(sr_off=0, sl_off=0, mu=mu_l), dict(sr_off=w2, sl_off=w2, mu=mu_r)],
                    phonon=None if gam is None else dict(gamma=gam, sr_off=2 * w2, sl_off=2 * w2, mu=mu_ph),
                    sr_const=None if not complex_energy else (n_lesser, np.full(n, -1j * eta)))
    return Workload(name, prob, energies, trapezoid_weights(energies), self_energies, nx, ny, description,
                    contacts)


def config1() -> Workload:
    """Single-energy ballistic 2D effective-mass device, 64 x 32 (BASELINE configs[0])."""
    nx, ny = 64, 32
    v = 0.1 * MT19937_64(0).uniform01(nx * ny)
    return effective_mass_device("cfg1_em_64x32", nx, ny, 0.5, 0.067, v, np.array([0.05]), 1e-6, 0.1, 0.0,
                                 0.025, description="2D effective mass 64x32, V~U[0,0.1] seed 0, E=0.05")


def config2(n_energies: int = 256, ny: int = 100, complex_energy: bool = False, nx: int = 400) -> Workload:
    """Quantum-well superlattice 400 x 100, 256 energies in [0, 0.4] (configs[1]).
    Smaller ``nx`` / ``ny`` give the reduced superlattices of the dense-truth
    parity study (same barriers and energy grid; the disorder draws cover
    nx*ny)."""
    x = np.arange(nx)
    barrier = np.where((x // 10) % 2 == 1, 0.3, 0.0)  # 5 nm = 10 points, wells at the leads
    v = np.repeat(barrier, ny) + (MT19937_64(1).uniform01(nx * ny) - 0.5) * 0.01
    e = uniform_grid(0.0, 0.4, n_energies)
    return effective_mass_device(f"cfg2_superlattice_{nx}x{ny}", nx, ny, 0.5, 0.067, v, e, 1e-6, 0.1, 0.0, 0.025,
                                 description=f"superlattice {nx}x{ny}, 0.3 eV barriers/wells of 5 nm, "
                                             "+-5 meV disorder seed 1, 256 E in [0,0.4]",
                                 complex_energy=complex_energy)


def config4(n_energies: int = 1024, nx: int = 1024, ny: int = 1024, complex_energy: bool = False,
            ref_orientation: bool = False) -> Workload:
    """Wide 1024 x 1024 device, sum of 16 Gaussians (configs[3]).  With
    ref_orientation the coordinates follow the reference builders (transverse
    first): nested dissection then merges a dense contact into the top
    separator, a 2557-dof root block."""
    r = MT19937_64(3)
    cx = r.uniform01(16) * nx
    cy = r.uniform01(16) * ny
    X, Y = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    v = np.zeros((nx, ny))
    for i in range(16):
        v += 0.05 * np.exp(-((X - cx[i]) ** 2 + (Y - cy[i]) ** 2) / (2.0 * 20.0 ** 2))
    e = uniform_grid(0.0, 0.3, n_energies)
    return effective_mass_device(f"cfg4_em_{nx}x{ny}", nx, ny, 0.5, 0.067, v, e, 1e-6, 0.1, 0.0, 0.025,
                                 description="2D effective mass, 16 Gaussians 0.05 eV width 20a, seed 3"
                                             + (", reference coordinate orientation" if ref_orientation else ""),
                                 complex_energy=complex_energy, ref_orientation=ref_orientation)


def config5(n_energies: int = 2048, nx: int = 512, ny: int = 512) -> Workload:
    """512 x 512 + diagonal phonon self-energy (configs[4])."""
    r = MT19937_64(4)
    v = 0.1 * r.uniform01(nx * ny)
    gamma = 1e-3 + 4e-3 * r.uniform01(nx * ny)
    e = uniform_grid(0.0, 0.3, n_energies)
    return effective_mass_device(f"cfg5_em_{nx}x{ny}_phonon", nx, ny, 0.5, 0.067, v, e, 1e-6, 0.1, 0.0, 0.025,
                                 phonon_gamma=gamma,
                                 description="2D effective mass + phonon -i gamma, gamma~U[1,5] meV seed 4")


# ---------------------------------------------------------------------------
# Zigzag (20,0) carbon nanotube, config 3
# ---------------------------------------------------------------------------
def _cnt_cell(k_around: int, t: float):
    """Unit cell of a zigzag (k,0) tube: 4 atomic rings of k atoms; returns
    (H00, H01) with H01 the coupling from a cell to the next one."""
    m = 4 * k_around
    h00 = np.zeros((m, m))
    h01 = np.zeros((m, m))
    ring = lambda l, k: l * k_around + (k % k_around)  # noqa: E731
    for k in range(k_around):
        # ring0 - ring1: zigzag (k -> k, k-1); ring1 - ring2: straight;
        # ring2 - ring3: zigzag (k -> k, k+1); ring3 - next ring0: straight
        for a, b in ((ring(0, k), ring(1, k)), (ring(0, k), ring(1, k - 1)), (ring(1, k), ring(2, k)),
                     (ring(2, k), ring(3, k)), (ring(2, k), ring(3, k + 1))):
            h00[a, b] = h00[b, a] = t
        h01[ring(3, k), ring(0, k)] = t
    return h00, h01


def sancho_rubio(energy: float, eta: float, h00: np.ndarray, h01: np.ndarray, tol: float = 1e-12,
                 max_iter: int = 200) -> np.ndarray:
    """Surface Green's function by energy-doubling decimation; returns the
    retarded self-energy H01^T g_s H01 of the lead attached through h01
    (coupling device-edge-cell -> lead-cell = h01, real symmetric blocks)."""
    z = (energy + 1j * eta) * np.eye(len(h00))
    es = h00.astype(np.complex128)
    e = es.copy()
    alpha = h01.astype(np.complex128)
    beta = h01.T.astype(np.complex128)
    for _ in range(max_iter):
        g = np.linalg.inv(z - e)
        ag, bg = alpha @ g, beta @ g
        es = es + ag @ beta
        e = e + ag @ beta + bg @ alpha
        alpha = ag @ alpha
        beta = bg @ beta
        if np.abs(alpha).max() < tol and np.abs(beta).max() < tol:
            break
    else:
        raise RuntimeError("Sancho-Rubio decimation did not converge")
    gs = np.linalg.inv(z - es)
    sig = h01.T @ gs @ h01
    return 0.5 * (sig + sig.T)


def config3(n_energies: int = 512, n_cells: int = 600, complex_energy: bool = False) -> Workload:
    """Zigzag (20,0) CNT, single p_z, t = -2.7 eV, 600 cells x 80 atoms (configs[2])."""
    k_around, t = 20, -2.7
    cell = 4 * k_around
    h00, h01 = _cnt_cell(k_around, t)
    n = n_cells * cell
    onsite = 0.1 * (MT19937_64(2).uniform01(n) - 0.5)
    r00, c00 = np.nonzero(h00)
    r01, c01 = np.nonzero(h01)
    rows, cols, vals = [np.arange(n)], [np.arange(n)], [onsite]
    for c in range(n_cells):
        b = c * cell
        rows.append(b + r00); cols.append(b + c00); vals.append(h00[r00, c00])
        if c + 1 < n_cells:
            rows += [b + r01, b + cell + c01]
            cols += [b + cell + c01, b + r01]
            vals += [h01[r01, c01], h01[r01, c01]]
    h_rows = np.concatenate(rows).astype(np.int32)
    h_cols = np.concatenate(cols).astype(np.int32)
    h_vals = np.concatenate(vals).astype(np.complex128)
    axial = np.repeat(np.arange(n_cells * 4), k_around).astype(np.float64)
    around = np.tile(np.arange(k_around), n_cells * 4).astype(np.float64)
    coords = np.stack([axial, around], 1)
    left = np.arange(cell)
    right = np.arange(n - cell, n)
    lr, lc = np.meshgrid(left, left, indexing="ij")
    rr, rc = np.meshgrid(right, right, indexing="ij")
    sl_rows = np.concatenate([lr.ravel(), rr.ravel()]).astype(np.int32)
    sl_cols = np.concatenate([lc.ravel(), rc.ravel()]).astype(np.int32)
    extra = [np.arange(n)] if complex_energy else []
    sr_rows = np.concatenate([sl_rows] + extra).astype(np.int32)
    sr_cols = np.concatenate([sl_cols] + extra).astype(np.int32)
    prob = Problem(n=n, h_rows=h_rows, h_cols=h_cols, h_vals=h_vals, sr_rows=sr_rows, sr_cols=sr_cols,
                   sl_rows=sl_rows, sl_cols=sl_cols, coords=coords,
                   atomic_groups=[left.tolist(), right.tolist()], max_leaf=64,
                   layers=[list(range(c * cell, (c + 1) * cell)) for c in range(n_cells)])
    energies = uniform_grid(-1.0, 1.0, n_energies)
    mu_l, mu_r, kT, eta = 0.1, -0.1, 0.025, 1e-6
    w2 = cell * cell

    def self_energies(sel):
        sel = np.atleast_1d(np.asarray(sel))
        sr = np.zeros((len(sel), len(sr_rows)), np.complex128)
        sl = np.zeros((len(sel), 2 * w2), np.complex128)
        sr[:, 2 * w2:] = -1j * eta
        for q, k in enumerate(sel):
            e = float(energies[k])
            # left lead repeats the first cell: device cell 0 <- lead cell via h01^T
            sig_l = sancho_rubio(e, eta, h00, h01.T)
            sig_r = sancho_rubio(e, eta, h00, h01)
            sr[q, :w2], sr[q, w2:2 * w2] = sig_l.ravel(), sig_r.ravel()
            sl[q, :w2] = (-fermi(e, mu_l, kT) * (sig_l - sig_l.conj().T)).ravel()
            sl[q, w2:] = (-fermi(e, mu_r, kT) * (sig_r - sig_r.conj().T)).ravel()
        return sr, sl

    contacts = dict(kind="sancho", w=cell, eta=eta, kT=kT, tol=1e-12, h00=h00,
                    leads=[dict(h01=h01.T.copy(), sr_off=0, sl_off=0, mu=mu_l),
                           dict(h01=h01, sr_off=w2, sl_off=w2, mu=mu_r)],
                    phonon=None,
                    sr_const=None if not complex_energy else (2 * w2, np.full(n, -1j * eta)))
    return Workload("cfg3_cnt_20_0_600", prob, energies, trapezoid_weights(energies), self_energies,
                    n_cells * 4, k_around, "zigzag (20,0) CNT, 600 cells, onsite U[-0.05,0.05] seed 2", contacts)


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


# ---------------------------------------------------------------------------
# Self-energies on the GPU
# ---------------------------------------------------------------------------
class GpuSelfEnergies:
    """Builds a workload's Sigma^r / Sigma^< pattern values for device-resident
    energies on the GPU: the analytic mode sum (effective-mass leads) or the
    batched Sancho-Rubio decimation (config 3's tube), then the lesser
    self-energies and the phonon diagonal (lesser_self_energy,
    device.cpp:322-366) -- the device-side replacement of the per-energy host
    ``Workload.self_energies``.  Returns torch tensors laid out like the host
    arrays (rows = energies), ready for ``HscGpuSolver.solve_device``."""

    def __init__(self, workload: Workload, device: int = 0, max_energy_batch: int = 0):
        import torch

        from . import negf as _negf

        c = workload.contacts
        if c is None:
            raise ValueError(f"workload {workload.name} has no GPU self-energy recipe")
        self.c = c
        self.dev = torch.device("cuda", device)
        self.n_sr = len(workload.problem.sr_rows)
        self.n_sl = len(workload.problem.sl_rows)
        self.leads = []
        if c["kind"] == "sancho":
            for ld in c["leads"]:
                self.leads.append(_negf.SurfaceLead(c["h00"], ld["h01"], c["eta"], device=device,
                                                    max_energy_batch=max_energy_batch, criterion="decay",
                                                    tol=c["tol"]))
        ph = c.get("phonon")
        self.gamma = None if ph is None else torch.from_numpy(np.ascontiguousarray(ph["gamma"], np.float64)).to(
            self.dev)
        self.sr_const = None
        if c.get("sr_const") is not None:
            off, vals = c["sr_const"]
            self.sr_const = (off, torch.from_numpy(np.ascontiguousarray(vals)).to(self.dev))

    def __call__(self, energies, sigma_r=None, sigma_lesser=None):
        import torch

        from . import negf as _negf

        c = self.c
        ne = int(energies.numel())
        w = c["w"]
        if sigma_r is None:
            sigma_r = torch.zeros((ne, self.n_sr), dtype=torch.complex128, device=self.dev)
        if sigma_lesser is None:
            sigma_lesser = torch.zeros((ne, self.n_sl), dtype=torch.complex128, device=self.dev)
        stream = torch.cuda.current_stream(self.dev).cuda_stream
        blocks = []
        if c["kind"] == "modes":  # one uniform lead, the same block on both sides
            sig = torch.empty((ne, w, w), dtype=torch.complex128, device=self.dev)
            _negf.lead_modes_sigma_device(w, c["t"], c["eta"], energies, sig, stream=stream)
            blocks = [sig for _ in c["leads"]]
        else:
            torch.cuda.current_stream(self.dev).synchronize()
            for lead in self.leads:
                sig = torch.empty((ne, w, w), dtype=torch.complex128, device=self.dev)
                lead.sigma_device(energies, sig)
                blocks.append(sig)
        if self.sr_const is not None:
            off, vals = self.sr_const
            sigma_r[:, off:off + vals.numel()] = vals
        descs = [dict(w=w, sigma=b, sr_off=ld["sr_off"], sl_off=ld["sl_off"], mu=ld["mu"])
                 for b, ld in zip(blocks, c["leads"])]
        ph = c.get("phonon")
        _negf.contacts_fill_device(energies, c["kT"], descs, sigma_r, sigma_lesser,
                                   phonon_gamma=self.gamma,
                                   ph_sr_off=-1 if ph is None else ph["sr_off"],
                                   ph_sl_off=-1 if ph is None else ph["sl_off"],
                                   mu_phonon=0.0 if ph is None else ph["mu"], stream=stream)
        return sigma_r, sigma_lesser


# ---------------------------------------------------------------------------
# make_synthetic_system (synthetic.cpp:10-150): the reference's benchmark
# system (cmd_bench, run.cpp:361-419)
# ---------------------------------------------------------------------------
def synthetic_system(nx: int, ny: int, seed: int, fuzz: bool = False, coupling_t: float = 1.0,
                     max_leaf: int = 64, args_right_to_left: bool = True) -> dict:
    """Restatement of make_synthetic_system: dof = j*nx + i (layer j = row of
    the grid), coords (i, j), draws from mt19937_64(seed) in the reference's
    order.  ``args_right_to_left``: the evaluation order of the two draws
    inside one ``cplx(re, im)`` constructor call (unspecified in C++; GCC
    evaluates right to left) -- pinned against the reference's own dumps in
    tests/test_ledger_bench.py.  Returns H (COO, coo_normalize order), the
    contact blocks, the Sigma^< COO, layers, coords and a ``Problem``."""
    if nx < 1 or ny < 1:
        raise ValueError("synthetic grid dimensions must be positive")
    if coupling_t == 0.0:
        raise ValueError("synthetic coupling strength must be nonzero")
    rng = MT19937_64(seed)
    u = lambda: float(rng.uniform01(1)[0])  # noqa: E731

    def pair(f_re, f_im):
        if args_right_to_left:
            im = f_im()
            re = f_re()
        else:
            re = f_re()
            im = f_im()
        return complex(re, im)

    n = nx * ny
    t = coupling_t
    h = {}

    def add(r, c, v):
        h[(r, c)] = h.get((r, c), 0j) + v

    layers = [list(range(j * nx, (j + 1) * nx)) for j in range(ny)]
    coords = np.array([[d % nx, d // nx] for d in range(n)], np.float64)
    for d in range(n):
        re = 6.0 + u()
        im = -0.2 * u() if fuzz else 0.0
        add(d, d, complex(re, im))
    for j in range(ny):
        for i in range(nx - 1):
            d = j * nx + i
            v = pair(lambda: -(0.5 + u()), lambda: 0.3 * (u() - 0.5)) if fuzz else complex(-t, 0.0)
            add(d, d + 1, v)
            add(d + 1, d, v)
    for j in range(ny - 1):
        if not fuzz:
            for i in range(nx):
                d = j * nx + i
                add(d, d + nx, complex(-t, 0.0))
                add(d + nx, d, complex(-t, 0.0))
            continue
        kind = j % 3
        if kind == 0:
            v = complex(-(0.5 + u()), 0.0)
            for i in range(nx):
                d = j * nx + i
                add(d, d + nx, v)
                add(d + nx, d, v)
        else:
            for i in range(nx):
                v = pair(lambda: -(0.5 + u()), lambda: 0.2 * (u() - 0.5))
                d = j * nx + i
                add(d, d + nx, v)
                add(d + nx, d, v)
            if kind == 2 and nx >= 2:
                v = pair(lambda: -0.3 * u(), lambda: 0.1 * (u() - 0.5))
                d = j * nx
                add(d, d + nx + 1, v)
                add(d + nx + 1, d, v)
                w = pair(lambda: -0.3 * u(), lambda: 0.1 * (u() - 0.5))
                add(d + 1, d + nx, w)
                add(d + nx, d + 1, w)
    keys = sorted(h)
    h_rows = np.array([k[0] for k in keys], np.int32)
    h_cols = np.array([k[1] for k in keys], np.int32)
    h_vals = np.array([h[k] for k in keys], np.complex128)

    def draw_contact(m):
        r = np.zeros((m, m), np.complex128)
        for a in range(m):
            for b in range(m):
                r[a, b] = pair(lambda: 0.2 * (u() - 0.5), lambda: 0.2 * (u() - 0.5))
        s = r + r.T
        for a in range(m):
            s[a, a] -= complex(0.0, 0.5 + 0.25 * u())
        return s

    sig_l = draw_contact(nx)
    sig_r = draw_contact(nx) if ny > 1 else None
    less = {}

    def add_lesser(dofs):
        m = len(dofs)
        x = np.zeros((m, m), np.complex128)
        for a in range(m):
            for b in range(m):
                x[a, b] = pair(lambda: 0.3 * (u() - 0.5), lambda: 0.3 * (u() - 0.5))
        for a in range(m):
            for b in range(m):
                v = x[a, b] - np.conj(x[b, a])
                if v != 0:
                    less[(dofs[a], dofs[b])] = less.get((dofs[a], dofs[b]), 0j) + v

    add_lesser(layers[0])
    if ny > 1:
        add_lesser(layers[-1])
    if fuzz:
        for j in range(1, ny - 1):
            for d in layers[j]:
                less[(d, d)] = less.get((d, d), 0j) + complex(0.0, 0.1 + 0.2 * u())
    lk = sorted(less)
    sl_rows = np.array([k[0] for k in lk], np.int32)
    sl_cols = np.array([k[1] for k in lk], np.int32)
    sl_vals = np.array([less[k] for k in lk], np.complex128)
    # Sigma^r pattern: the dense contact blocks (assemble_system adds them whole)
    w = nx
    L = np.array(layers[0])
    sr_rows = [np.repeat(L, w)]
    sr_cols = [np.tile(L, w)]
    sr_vals = [sig_l.ravel()]
    if sig_r is not None:
        R = np.array(layers[-1])
        sr_rows.append(np.repeat(R, w))
        sr_cols.append(np.tile(R, w))
        sr_vals.append(sig_r.ravel())
    groups = [layers[0]] + ([layers[-1]] if ny > 1 else [])
    prob = Problem(n=n, h_rows=h_rows, h_cols=h_cols, h_vals=h_vals,
                   sr_rows=np.concatenate(sr_rows).astype(np.int32), sr_cols=np.concatenate(sr_cols).astype(np.int32),
                   sl_rows=sl_rows, sl_cols=sl_cols, coords=coords, atomic_groups=groups, max_leaf=max_leaf,
                   layers=layers)
    return dict(problem=prob, h_rows=h_rows, h_cols=h_cols, h_vals=h_vals, sig_l=sig_l, sig_r=sig_r,
                sl_rows=sl_rows, sl_cols=sl_cols, sl_vals=sl_vals, sr_vals=np.concatenate(sr_vals),
                layers=layers, coords=coords)
