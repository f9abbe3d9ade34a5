"""Shared test helpers: golden fixtures -> product inputs, parity metrics."""
from __future__ import annotations

import glob
import os

import numpy as np

from oracle import refio
from paper_1305_1070_b200 import negf

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_names():
    """Problem fixtures (NEGFPRB1); lead_*.bin are lead fixtures (NEGFLED1)."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.bin"))
                  if not os.path.basename(p).startswith("lead_"))


def lead_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "lead_*.bin")))


def dense_block(rp, rows, cols) -> np.ndarray:
    """dense_block (device.cpp:27-43) of the problem's H over dof lists."""
    ri = {d: k for k, d in enumerate(rows)}
    ci = {d: k for k, d in enumerate(cols)}
    m = np.zeros((len(rows), len(cols)), np.complex128)
    for r, c, v in zip(rp.h_rows, rp.h_cols, rp.h_vals):
        if r in ri and c in ci:
            m[ri[r], ci[c]] += v
    return m


def load_golden(name: str):
    """(RefProblem, product Problem, reference hsc result, dense result or None)."""
    rp = refio.read_problem(os.path.join(GOLDEN, name + ".bin"))
    (srr, src, _), (slr, slc, _) = rp.patterns()
    prob = negf.Problem(n=rp.n, h_rows=rp.h_rows, h_cols=rp.h_cols, h_vals=rp.h_vals, sr_rows=srr, sr_cols=src,
                        sl_rows=slr, sl_cols=slc, coords=rp.coords, atomic_groups=rp.groups,
                        max_leaf=rp.max_leaf, layers=rp.layers)
    hsc = refio.read_result(os.path.join(GOLDEN, name + ".hsc.out"), rp.n)
    dpath = os.path.join(GOLDEN, name + ".dense.out")
    dense = refio.read_result(dpath, rp.n) if os.path.exists(dpath) else None
    return rp, prob, hsc, dense


def rel_err(x: np.ndarray, ref: np.ndarray) -> float:
    """max_j |x_j - o_j| / max_j |o_j| (SURVEY §8(d) parity metric)."""
    den = np.abs(ref).max()
    num = np.abs(x - ref).max()
    return float(num / den) if den > 0 else float(num)


def workload_ref_problem(w, idx):
    """The reference-side problem (NEGFPRB1) of a devices.Workload at energy
    indices idx: the same H, the same two dense contact blocks and phonon
    diagonal (the reference's ContactBlock / phonon vector, run.cpp:90-109),
    the same energies and trapezoid weights.  Returns (RefProblem, sr, sl)
    with sr / sl the product's pattern values for the same energies."""
    idx = np.atleast_1d(np.asarray(idx))
    p = w.problem
    sr, sl = w.self_energies(idx)
    n = p.n
    L = np.asarray(p.atomic_groups[0], np.int32)
    R = np.asarray(p.atomic_groups[1], np.int32)
    ny = len(L)  # contact width (both contacts are equally wide here)
    assert len(R) == ny
    w2 = ny * ny
    n_lesser = len(p.sl_rows)
    has_ph = n_lesser > 2 * w2
    ph = phl = None
    extra = len(p.sr_rows) - n_lesser  # complex_energy: -i eta on every dof
    if has_ph or extra:
        ph = np.zeros((len(idx), n), np.complex128)
        if has_ph:
            inner = np.asarray(p.sr_rows[2 * w2:n_lesser], np.int64)
            ph[:, inner] += sr[:, 2 * w2:n_lesser]
        if extra:
            ph[:, np.asarray(p.sr_rows[n_lesser:], np.int64)] += sr[:, n_lesser:]
    if has_ph:
        inner = np.asarray(p.sl_rows[2 * w2:], np.int64)
        phl = np.zeros((len(idx), n), np.complex128)
        phl[:, inner] = sl[:, 2 * w2:]
    rp = refio.RefProblem(n=n, h_rows=p.h_rows, h_cols=p.h_cols, h_vals=p.h_vals,
                          layers=[np.asarray(l) for l in p.layers], coords=p.coords, groups=[L, R],
                          max_leaf=p.max_leaf, dofs_l=L, dofs_r=R, has_ph=ph is not None, has_ph_less=phl is not None,
                          energies=w.energies[idx], weights=w.weights[idx],
                          sig_l=sr[:, :w2].reshape(-1, ny, ny), sig_r=sr[:, w2:2 * w2].reshape(-1, ny, ny), ph=ph,
                          less_l=sl[:, :w2].reshape(-1, ny, ny), less_r=sl[:, w2:2 * w2].reshape(-1, ny, ny),
                          ph_less=phl)
    return rp, sr, sl


def per_energy_err(x: np.ndarray, ref: np.ndarray) -> np.ndarray:
    """rel_err per row (energy)."""
    den = np.abs(ref).max(axis=1)
    return np.abs(x - ref).max(axis=1) / np.where(den > 0, den, 1.0)


def real_residual(gl: np.ndarray) -> np.ndarray:
    """max_j |Re G^<_jj| / |G^<_jj| per energy (electron_density's guard
    quantity, observables.cpp:79-84)."""
    a = np.abs(gl)
    return (np.abs(gl.real) / np.where(a > 0, a, 1.0)).max(axis=1)
