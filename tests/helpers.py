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
