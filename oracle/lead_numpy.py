"""TEST INFRASTRUCTURE ONLY (oracle/): numpy restatement of the reference's
contact self-energies, the CPU checker of the B200 lead kernels.

Follows:
  surface_self_energy   proj/src/device.cpp:195-251 (energy-doubling
                        decimation with the fixed-point residual test)
  attach_contacts       proj/src/device.cpp:262-304 (DenseLead blocks)
  fermi_function        proj/src/device.cpp:253-260
  lesser_self_energy    proj/src/device.cpp:322-366

Parity pin: tests/test_lead.py checks this restatement against the Sigma
blocks the reference itself wrote into tests/golden/*_dense.bin and
tests/golden/lead_*.bin (make_golden.py).  Never imported by the product path.
"""
from __future__ import annotations

import numpy as np

from .hsc_numpy import Ledger, SingularBlock, inverse

K_BOLTZMANN_EV_PER_K = 8.617333262e-5  # device.hpp:18


class ConvergenceError(RuntimeError):
    pass


def _z_minus(z: complex, m: np.ndarray) -> np.ndarray:
    r = -m.astype(np.complex128)
    r[np.diag_indices_from(r)] += z
    return r


def _inv(a: np.ndarray) -> np.ndarray:
    return inverse(a, Ledger())


def surface_self_energy(h00: np.ndarray, h01: np.ndarray, energy: float, eta: float,
                        return_sweeps: bool = False):
    """device.cpp:195-251.  Raises ValueError for bad shapes (ContractViolation),
    ValueError('eta') for eta <= 0 (ConfigError), ConvergenceError after 200
    sweeps, SingularBlock from the inverses."""
    n = h00.shape[0]
    if h00.shape != (n, n):
        raise ValueError("surface_self_energy: h00 must be square")
    if h01.shape != (n, n):
        raise ValueError("surface_self_energy: h01 must match h00's shape")
    if eta <= 0.0:
        raise ValueError("contact broadening eta must be positive")
    z = complex(energy, eta)
    h00 = h00.astype(np.complex128)
    h01 = h01.astype(np.complex128)
    h01ct = h01.conj().T
    es = h00.copy()
    e = h00.copy()
    alpha = h01ct.copy()
    beta = h01.copy()
    for sweep in range(200):
        g = _inv(_z_minus(z, es))
        rhs = _z_minus(z, h00) - (h01ct @ g) @ h01
        refined = _inv(rhs)
        diff = refined - g
        if np.sqrt(np.sum(diff.real ** 2 + diff.imag ** 2)) <= 1e-10:
            sigma = (h01ct @ refined) @ h01
            iu = np.triu_indices(n, 1)
            avg = 0.5 * (sigma[iu] + sigma.T[iu])
            sigma[iu] = avg
            sigma.T[iu] = avg
            return (sigma, sweep) if return_sweeps else sigma
        m = _inv(_z_minus(z, e))
        am = alpha @ m
        bm = beta @ m
        ab = am @ beta
        ba = bm @ alpha
        es = es + ab
        e = e + ab + ba
        alpha = am @ alpha
        beta = bm @ beta
    raise ConvergenceError("surface self-energy decimation did not reach a 1e-10 fixed-point "
                           "residual within 200 sweeps")


def lead_blocks(h_dense_rows, layers, side: str):
    """attach_contacts' lead blocks (device.cpp:284-303) from a dense-block
    accessor h_dense_rows(rows, cols) -> ndarray."""
    if side == "left":
        return h_dense_rows(layers[0], layers[0]), h_dense_rows(layers[0], layers[1])
    b_r = h_dense_rows(layers[-2], layers[-1])
    return h_dense_rows(layers[-1], layers[-1]), b_r.T.copy()


def fermi(energy: float, mu: float, kT: float) -> float:
    """fermi_function (device.cpp:253-260) with kT = kB * temperature."""
    x = (energy - mu) / kT
    if x > 700.0:
        return 0.0
    if x < -700.0:
        return 1.0
    return 1.0 / (1.0 + np.exp(x))


def lesser_block(sigma: np.ndarray, f: float) -> np.ndarray:
    """-f (S - S^dagger) entrywise (device.cpp:335-342)."""
    return -f * (sigma - sigma.conj().T)
