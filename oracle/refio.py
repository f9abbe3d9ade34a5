"""TEST INFRASTRUCTURE ONLY (oracle/): binary problem/result exchange with the
reference build in oracle/_ref (see ref_driver.cpp for the formats) and the
conversion of a reference-style problem (contacts + phonon diagonal) into the
pattern form of the product's C ABI.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs use this.
"""
from __future__ import annotations

import os
import struct
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_BIN = os.path.join(HERE, "_ref", "ref_driver")

ERROR_NAMES = {1: "SingularBlock", 2: "NonSkewHermitianInput", 3: "ContractViolation", 7: "ConfigError",
               8: "PartitionViolation", 9: "ResidualTooLarge", 10: "Error"}


def ref_available() -> bool:
    return os.path.exists(REF_BIN)


@dataclass
class RefProblem:
    """A problem in the reference's own terms (NEGFPRB1)."""

    n: int
    h_rows: np.ndarray
    h_cols: np.ndarray
    h_vals: np.ndarray
    layers: list
    coords: np.ndarray | None
    groups: list
    max_leaf: int
    dofs_l: np.ndarray
    dofs_r: np.ndarray
    has_ph: bool
    has_ph_less: bool
    energies: np.ndarray
    weights: np.ndarray
    sig_l: np.ndarray      # (nE, wL, wL)
    sig_r: np.ndarray      # (nE, wR, wR)
    ph: np.ndarray | None  # (nE, n)
    less_l: np.ndarray
    less_r: np.ndarray
    ph_less: np.ndarray | None

    # -- conversion to the C-ABI pattern form -------------------------------
    def patterns(self):
        """Sigma^r and Sigma^< patterns: union over energies of the nonzero
        entries (the reference's producers drop exact zeros, device.cpp:344-356)."""
        n = self.n

        def pattern(blk_l, blk_r, diag):
            rows, cols, src = [], [], []
            for dofs, blk, tag in ((self.dofs_l, blk_l, 0), (self.dofs_r, blk_r, 1)):
                if len(dofs) == 0:
                    continue
                nz = np.any(blk != 0, axis=0)
                a, b = np.nonzero(nz)
                rows.append(dofs[a]); cols.append(dofs[b])
                src.append(np.stack([np.full(len(a), tag), a, b], 1))
            if diag is not None:
                d = np.nonzero(np.any(diag != 0, axis=0))[0]
                rows.append(d); cols.append(d)
                src.append(np.stack([np.full(len(d), 2), d, d], 1))
            if not rows:
                return np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros((0, 3), np.int64)
            return (np.concatenate(rows).astype(np.int32), np.concatenate(cols).astype(np.int32),
                    np.concatenate(src).astype(np.int64))

        self._sr = pattern(self.sig_l, self.sig_r, self.ph if self.has_ph else None)
        self._sl = pattern(self.less_l, self.less_r, self.ph_less if self.has_ph_less else None)
        return self._sr, self._sl

    def values(self, idx):
        """Per-energy pattern values (m, nnz) for energy indices idx."""
        idx = np.atleast_1d(np.asarray(idx))
        if not hasattr(self, "_sr"):
            self.patterns()

        def gather(pat, bl, br, dg):
            src = pat[2]
            out = np.zeros((len(idx), len(src)), np.complex128)
            for tag, blk in ((0, bl), (1, br)):
                sel = src[:, 0] == tag
                if sel.any():
                    out[:, sel] = blk[idx][:, src[sel, 1], src[sel, 2]]
            sel = src[:, 0] == 2
            if sel.any():
                out[:, sel] = dg[idx][:, src[sel, 1]]
            return out

        sr = gather(self._sr, self.sig_l, self.sig_r, self.ph)
        sl = gather(self._sl, self.less_l, self.less_r, self.ph_less)
        return sr, sl


def read_problem(path: str) -> RefProblem:
    with open(path, "rb") as f:
        buf = f.read()
    pos = 0

    def take(fmt):
        nonlocal pos
        v = struct.unpack_from(fmt, buf, pos)
        pos += struct.calcsize(fmt)
        return v

    def arr(dtype, count):
        nonlocal pos
        a = np.frombuffer(buf, dtype=dtype, count=count, offset=pos).copy()
        pos += a.nbytes
        return a

    assert buf[:8] == b"NEGFPRB1"
    pos = 8
    (n,) = take("<i")
    (nnz,) = take("<q")
    rows, cols, vals = arr(np.int32, nnz), arr(np.int32, nnz), arr(np.complex128, nnz)
    (nl,) = take("<i")
    layers = []
    for _ in range(nl):
        (c,) = take("<i")
        layers.append(arr(np.int32, c))
    (hc,) = take("<i")
    coords = arr(np.float64, 2 * n).reshape(n, 2) if hc else None
    (ng,) = take("<i")
    groups = []
    for _ in range(ng):
        (c,) = take("<i")
        groups.append(arr(np.int32, c))
    (max_leaf,) = take("<i")
    (c,) = take("<i")
    dl = arr(np.int32, c)
    (c,) = take("<i")
    dr = arr(np.int32, c)
    has_ph, has_ph_less = take("<ii")
    (ne,) = take("<i")
    energies, weights = arr(np.float64, ne), arr(np.float64, ne)
    wl, wr = len(dl), len(dr)
    sl, sr, ph, ll, lr, phl = [], [], [], [], [], []
    for _ in range(ne):
        sl.append(arr(np.complex128, wl * wl).reshape(wl, wl))
        sr.append(arr(np.complex128, wr * wr).reshape(wr, wr))
        if has_ph:
            ph.append(arr(np.complex128, n))
        ll.append(arr(np.complex128, wl * wl).reshape(wl, wl))
        lr.append(arr(np.complex128, wr * wr).reshape(wr, wr))
        if has_ph_less:
            phl.append(arr(np.complex128, n))
    return RefProblem(n, rows, cols, vals, layers, coords, groups, max_leaf, dl, dr, bool(has_ph), bool(has_ph_less),
                      energies, weights, np.array(sl).reshape(ne, wl, wl), np.array(sr).reshape(ne, wr, wr),
                      np.array(ph) if has_ph else None, np.array(ll).reshape(ne, wl, wl),
                      np.array(lr).reshape(ne, wr, wr), np.array(phl) if has_ph_less else None)


def write_problem(p: RefProblem, path: str) -> None:
    out = [b"NEGFPRB1", struct.pack("<i", p.n), struct.pack("<q", len(p.h_rows)),
           np.asarray(p.h_rows, np.int32).tobytes(), np.asarray(p.h_cols, np.int32).tobytes(),
           np.asarray(p.h_vals, np.complex128).tobytes(), struct.pack("<i", len(p.layers))]
    for l in p.layers:
        out += [struct.pack("<i", len(l)), np.asarray(l, np.int32).tobytes()]
    out.append(struct.pack("<i", 0 if p.coords is None else 1))
    if p.coords is not None:
        out.append(np.asarray(p.coords, np.float64).tobytes())
    out.append(struct.pack("<i", len(p.groups)))
    for g in p.groups:
        out += [struct.pack("<i", len(g)), np.asarray(g, np.int32).tobytes()]
    out.append(struct.pack("<i", p.max_leaf))
    for d in (p.dofs_l, p.dofs_r):
        out += [struct.pack("<i", len(d)), np.asarray(d, np.int32).tobytes()]
    out.append(struct.pack("<ii", int(p.has_ph), int(p.has_ph_less)))
    out += [struct.pack("<i", len(p.energies)), np.asarray(p.energies, np.float64).tobytes(),
            np.asarray(p.weights, np.float64).tobytes()]
    for e in range(len(p.energies)):
        out += [np.ascontiguousarray(p.sig_l[e], np.complex128).tobytes(),
                np.ascontiguousarray(p.sig_r[e], np.complex128).tobytes()]
        if p.has_ph:
            out.append(np.ascontiguousarray(p.ph[e], np.complex128).tobytes())
        out += [np.ascontiguousarray(p.less_l[e], np.complex128).tobytes(),
                np.ascontiguousarray(p.less_r[e], np.complex128).tobytes()]
        if p.has_ph_less:
            out.append(np.ascontiguousarray(p.ph_less[e], np.complex128).tobytes())
    with open(path, "wb") as f:
        for b in out:
            f.write(b)


@dataclass
class RefResult:
    status: int
    error_energy: int
    message: str
    parent: np.ndarray
    level: np.ndarray
    dofs: list
    mul_ops: int
    inv_ops: int
    wall_s: float
    tree_s: float
    threads: int
    energy_idx: np.ndarray
    gr: np.ndarray      # (m, n)
    gless: np.ndarray   # (m, n)


def read_result(path: str, n: int) -> RefResult:
    with open(path, "rb") as f:
        buf = f.read()
    assert buf[:8] == b"NEGFOUT1"
    pos = 8
    status, err_e = struct.unpack_from("<ii", buf, pos)
    pos += 8
    msg = buf[pos : pos + 512].split(b"\0", 1)[0].decode(errors="replace")
    pos += 512
    (nc,) = struct.unpack_from("<i", buf, pos)
    pos += 4
    parent, level, dofs = np.zeros(nc, np.int32), np.zeros(nc, np.int32), []
    for c in range(nc):
        parent[c], level[c], ln = struct.unpack_from("<iii", buf, pos)
        pos += 12
        dofs.append(np.frombuffer(buf, np.int32, ln, pos).copy())
        pos += 4 * ln
    mul, inv = struct.unpack_from("<qq", buf, pos)
    pos += 16
    wall, tree_s = struct.unpack_from("<dd", buf, pos)
    pos += 16
    threads, m = struct.unpack_from("<ii", buf, pos)
    pos += 8
    idx = np.frombuffer(buf, np.int32, m, pos).copy()
    pos += 4 * m
    gr = np.frombuffer(buf, np.complex128, m * n, pos).reshape(m, n).copy()
    pos += 16 * m * n
    gl = np.frombuffer(buf, np.complex128, m * n, pos).reshape(m, n).copy()
    return RefResult(status, err_e, msg, parent, level, dofs, mul, inv, wall, tree_s, threads, idx, gr, gl)


def run_reference(problem_path: str, out_path: str, threads: int = 1, solver: str = "hsc",
                  energies=None, timeout: float | None = None) -> RefResult:
    cmd = [REF_BIN, "solve", problem_path, out_path, "--threads", str(threads), "--solver", solver]
    if energies is not None:
        cmd += ["--energies", ",".join(str(int(e)) for e in energies)]
    subprocess.run(cmd, check=True, timeout=timeout)
    with open(problem_path, "rb") as f:
        f.seek(8)
        (n,) = struct.unpack("<i", f.read(4))
    return read_result(out_path, n)


def dump_synthetic(nx, ny, seed, fuzz, coupling, max_leaf, energies, path) -> None:
    subprocess.run([REF_BIN, "synthetic", str(nx), str(ny), str(seed), str(int(fuzz)), repr(float(coupling)),
                    str(max_leaf), path] + [repr(float(e)) for e in energies], check=True)


def dump_device(config_path: str, path: str) -> None:
    subprocess.run([REF_BIN, "device", config_path, path], check=True)


# -- dense leads (ref_driver lead: surface_self_energy, device.cpp:195-251) ----
def write_lead(path: str, h00: np.ndarray, h01: np.ndarray, eta: float, energies) -> None:
    w = h00.shape[0]
    e = np.asarray(energies, np.float64)
    with open(path, "wb") as f:
        f.write(b"NEGFLED1")
        f.write(struct.pack("<iid", w, len(e), float(eta)))
        f.write(np.ascontiguousarray(h00, np.complex128).tobytes())
        f.write(np.ascontiguousarray(h01, np.complex128).tobytes())
        f.write(e.tobytes())


def read_lead(path: str):
    """Returns (w, eta, h00, h01, energies) of a NEGFLED1 file."""
    with open(path, "rb") as f:
        buf = f.read()
    assert buf[:8] == b"NEGFLED1"
    w, ne, eta = struct.unpack_from("<iid", buf, 8)
    pos = 24
    h00 = np.frombuffer(buf, np.complex128, w * w, pos).reshape(w, w).copy()
    pos += 16 * w * w
    h01 = np.frombuffer(buf, np.complex128, w * w, pos).reshape(w, w).copy()
    pos += 16 * w * w
    e = np.frombuffer(buf, np.float64, ne, pos).copy()
    return w, eta, h00, h01, e


def read_lead_out(path: str, w: int):
    """Returns (codes[nE], sigma[nE, w, w]) of a NEGFLEO1 file."""
    with open(path, "rb") as f:
        buf = f.read()
    assert buf[:8] == b"NEGFLEO1"
    (ne,) = struct.unpack_from("<i", buf, 8)
    pos = 12
    codes = np.zeros(ne, np.int32)
    sig = np.zeros((ne, w, w), np.complex128)
    for k in range(ne):
        (codes[k],) = struct.unpack_from("<i", buf, pos)
        pos += 4
        sig[k] = np.frombuffer(buf, np.complex128, w * w, pos).reshape(w, w)
        pos += 16 * w * w
    return codes, sig


def run_lead(in_path: str, out_path: str, timeout: float | None = None):
    subprocess.run([REF_BIN, "lead", in_path, out_path], check=True, timeout=timeout)
    w = read_lead(in_path)[0]
    return read_lead_out(out_path, w)
