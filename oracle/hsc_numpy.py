"""TEST INFRASTRUCTURE ONLY (oracle/): numpy restatement of the reference's
lean HSC solver, used as the CPU checker of the B200 path.

Follows, function by function:
  group_by_partition      proj/src/block.cpp:49-82
  assemble_system         proj/src/block.cpp:123-161
  inverse (singular rule) proj/src/dense.cpp:49-81
  hsc_fold                proj/src/hsc.cpp:447-534
  validate_sigma          proj/src/hsc.cpp:89-119
  LeanSolver (G, seeds, N fold, P)  proj/src/hsc.cpp:131-327
  flatten_diag            proj/src/block.cpp:163-205
  electron_density        proj/src/observables.cpp:58-93
with the reference's operation ledger charged alongside (dense.hpp:69-82).

Parity pin: tests/test_oracle.py checks this restatement against the golden
outputs written by the reference itself (tests/golden, make_golden.py).
Never imported by the product path.
"""
from __future__ import annotations

import numpy as np


class SingularBlock(RuntimeError):
    def __init__(self, msg, pivot):
        super().__init__(msg)
        self.pivot_index = pivot


class NonSkewHermitian(RuntimeError):
    pass


class ContractViolation(RuntimeError):
    pass


class Ledger:
    def __init__(self):
        self.mul = 0
        self.inv = 0

    def matmul(self, a, b):
        self.mul += a.shape[0] * a.shape[1] * b.shape[1]
        return a @ b


class Tree:
    """parent[c], dofs[c] (sorted) -> levels, ancestors (nearest first), fold
    order (level, id) as SeparatorTree::build (partition.cpp:19-91)."""

    def __init__(self, parent, dofs, n):
        self.parent = [int(p) for p in parent]
        self.dofs = [np.asarray(sorted(d), dtype=np.int64) for d in dofs]
        self.n = n
        nc = len(parent)
        self.children = [[] for _ in range(nc)]
        for c, p in enumerate(self.parent):
            if p >= 0:
                self.children[p].append(c)
        self.root = self.parent.index(-1)
        self.level = [0] * nc
        order = []
        stack = [self.root]
        while stack:
            c = stack.pop()
            order.append(c)
            stack.extend(self.children[c])
        for c in reversed(order):
            self.level[c] = 1 + max((self.level[ch] for ch in self.children[c]), default=0)
        self.anc = []
        for c in range(nc):
            chain, p = [], self.parent[c]
            while p != -1:
                chain.append(p)
                p = self.parent[p]
            self.anc.append(chain)
        self.fold_order = sorted((c for c in range(nc) if c != self.root), key=lambda c: (self.level[c], c))
        self.cluster_of = np.empty(n, np.int64)
        self.local = np.empty(n, np.int64)
        for c, d in enumerate(self.dofs):
            self.cluster_of[d] = c
            self.local[d] = np.arange(len(d))

    def size(self, c):
        return len(self.dofs[c])


def group_by_partition(tree: Tree, rows, cols, vals):
    """COO -> {(ci, cj): block}, both orientations (block.cpp:49-82)."""
    ci, cj = tree.cluster_of[rows], tree.cluster_of[cols]
    li, lj = tree.local[rows], tree.local[cols]
    blocks = {}
    for a, b in set(zip(ci.tolist(), cj.tolist())):
        blocks[(a, b)] = np.zeros((tree.size(a), tree.size(b)), np.complex128)
    for k in range(len(rows)):
        blocks[(int(ci[k]), int(cj[k]))][li[k], lj[k]] += vals[k]
    return blocks


def inverse(a, ledger: Ledger):
    """Partial-pivot LU explicit inverse with the 1e-13 max|a| pivot rule."""
    n = a.shape[0]
    if n == 0:
        return np.zeros((0, 0), np.complex128)
    thresh = 1e-13 * np.abs(a).max()
    lu = a.copy()
    for k in range(n):
        p = k + int(np.argmax(np.abs(lu[k:, k])))
        if np.abs(lu[p, k]) <= thresh:
            raise SingularBlock(f"inverse: singular pivot {k} in {n}x{n} block", k)
        if p != k:
            lu[[k, p]] = lu[[p, k]]
        lu[k + 1:, k] /= lu[k, k]
        lu[k + 1:, k + 1:] -= np.outer(lu[k + 1:, k], lu[k, k + 1:])
    ledger.inv += n ** 3
    return np.linalg.inv(a)


def hsc_fold(tree: Tree, blocks: dict, ledger: Ledger):
    """Bottom-up fold in (level, id) order; returns (psi, inv_diag)."""
    a = {k: v.copy() for k, v in blocks.items()}
    psi, inv_diag = {}, {}
    for i in tree.fold_order:
        aii = a.get((i, i), np.zeros((tree.size(i), tree.size(i)), np.complex128))
        inv = inverse(aii, ledger)
        inv_diag[i] = inv
        js = [j for j in tree.anc[i] if (i, j) in a]
        arow = [a[(i, j)] for j in js]
        psi[i] = [(j, -ledger.matmul(inv, aij)) for j, aij in zip(js, arow)]
        for p in range(len(js)):
            for q in range(p, len(js)):
                u = ledger.matmul(psi[i][p][1].T, arow[q])
                key = (js[p], js[q])
                if key not in a:
                    a[key] = np.zeros((tree.size(js[p]), tree.size(js[q])), np.complex128)
                a[key] = a[key] + u
        for j in js:
            a.pop((i, j), None)
            a.pop((j, i), None)
        a.pop((i, i), None)
    r = tree.root
    inv_diag[r] = inverse(a.get((r, r), np.zeros((tree.size(r), tree.size(r)), np.complex128)), ledger)
    return psi, inv_diag


def skew_defect(s):
    num = np.linalg.norm(s + s.conj().T)
    den = np.linalg.norm(s)
    return num if den == 0 else num / den


def validate_sigma(tree: Tree, sig_blocks: dict):
    view = {}
    for (a, b), s in sig_blocks.items():
        if a != b:
            raise ContractViolation("sigma_lesser must be block diagonal on the cluster partition")
        if skew_defect(s) > 1e-10:
            raise NonSkewHermitian(f"sigma_lesser block of cluster {a} is not skew-Hermitian")
        off = s - np.diag(np.diag(s))
        view[a] = (s, bool(s.shape[0] == s.shape[1] and not np.any(off != 0)))
    return view


def hsc_gless(tree: Tree, psi, inv_diag, sig_view, ledger: Ledger):
    """LeanSolver::run (hsc.cpp:147-163): returns (gr_diag, gless_diag) per cluster."""
    nc = len(tree.parent)
    grow, nrow, prow = [dict() for _ in range(nc)], [dict() for _ in range(nc)], [dict() for _ in range(nc)]
    gdiag, ndiag, pdiag = {}, {}, {}
    lev = tree.level

    def seed(x, g):
        s, diag = sig_view[x]
        if diag:
            ledger.mul += g.shape[0] * g.shape[1]
            return np.diag(s)[:, None] * g.conj()
        return ledger.matmul(s, g.conj())

    def g_of(k, j):
        if k == j:
            return gdiag[j]
        if lev[k] < lev[j]:
            return grow[k][j]
        return grow[j][k].T

    def p_of(k, j):
        if k == j:
            return pdiag[j]
        if lev[k] < lev[j]:
            return prow[k][j]
        return -prow[j][k].conj().T

    gdiag[tree.root] = inv_diag[tree.root]
    order = []
    stack = [tree.root]
    while stack:  # DFS pre-order, children in id order (hsc.cpp:239-244)
        x = stack.pop()
        order.append(x)
        stack.extend(reversed(tree.children[x]))
    for x in order:
        if x != tree.root:
            m = tree.size(x)
            for j in tree.anc[x]:
                acc = np.zeros((m, tree.size(j)), np.complex128)
                for k, pk in psi[x]:
                    acc += ledger.matmul(pk, g_of(k, j))
                grow[x][j] = acc
            d = inv_diag[x].copy()
            for k, pk in psi[x]:
                d += ledger.matmul(pk, grow[x][k].T)
            gdiag[x] = d
        if x in sig_view:
            ndiag[x] = seed(x, gdiag[x])
            for j in tree.anc[x]:
                nrow[x][j] = seed(x, grow[x][j])
    if not sig_view:
        return gdiag, {c: np.zeros((tree.size(c), tree.size(c)), np.complex128) for c in range(nc)}
    for i in tree.fold_order:  # n_fold (hsc.cpp:246-266)
        if not nrow[i]:
            continue
        for j, pj in psi[i]:
            for k in sorted(nrow[i], key=lambda c: lev[c]):
                if lev[k] < lev[j]:
                    continue
                u = ledger.matmul(pj.T, nrow[i][k])
                if k == j:
                    ndiag[j] = ndiag.get(j, np.zeros((tree.size(j), tree.size(j)), np.complex128)) + u
                else:
                    nrow[j][k] = nrow[j].get(k, np.zeros((tree.size(j), tree.size(k)), np.complex128)) + u
    r = tree.root
    pdiag[r] = ledger.matmul(inv_diag[r], ndiag[r]) if r in ndiag else np.zeros((tree.size(r),) * 2, np.complex128)
    for x in order:
        if x == r:
            continue
        m = tree.size(x)
        inv = inv_diag[x]
        for j in tree.anc[x]:
            acc = ledger.matmul(inv, nrow[x][j]) if j in nrow[x] else np.zeros((m, tree.size(j)), np.complex128)
            for k, pk in psi[x]:
                acc = acc + ledger.matmul(pk, p_of(k, j))
            prow[x][j] = acc
        d = ledger.matmul(inv, ndiag[x]) if x in ndiag else np.zeros((m, m), np.complex128)
        for k, pk in psi[x]:
            d = d - ledger.matmul(pk, prow[x][k].conj().T)
        pdiag[x] = d
    return gdiag, pdiag


def flatten(tree: Tree, blocks: dict) -> np.ndarray:
    out = np.zeros(tree.n, np.complex128)
    for c, d in enumerate(tree.dofs):
        out[d] = np.diag(blocks[c])
    return out


def assemble(n, h_rows, h_cols, h_vals, sr_rows, sr_cols, sr_vals, energy):
    """A(E) = E I - H - Sigma^r as COO (assemble_system, block.cpp:123-161)."""
    rows = np.concatenate([np.arange(n), h_rows, sr_rows])
    cols = np.concatenate([np.arange(n), h_cols, sr_cols])
    vals = np.concatenate([np.full(n, energy, np.complex128), -np.asarray(h_vals), -np.asarray(sr_vals)])
    return rows, cols, vals


def solve_energy(tree: Tree, n, h_rows, h_cols, h_vals, sr_rows, sr_cols, sr_vals, sl_rows, sl_cols, sl_vals,
                 energy):
    """solve_energy's HSC branch (run.cpp:163-176) -> (gr, gless, ledger)."""
    led = Ledger()
    r, c, v = assemble(n, h_rows, h_cols, h_vals, sr_rows, sr_cols, sr_vals, energy)
    blocks = group_by_partition(tree, r, c, v)
    psi, inv = hsc_fold(tree, blocks, led)
    nz = np.asarray(sl_vals) != 0  # producers drop exact zeros (device.cpp:344-356)
    sig = group_by_partition(tree, np.asarray(sl_rows)[nz], np.asarray(sl_cols)[nz], np.asarray(sl_vals)[nz])
    view = validate_sigma(tree, sig)
    gd, pd = hsc_gless(tree, psi, inv, view, led)
    return flatten(tree, gd), flatten(tree, pd), led


def dense_solve(n, h_rows, h_cols, h_vals, sr_rows, sr_cols, sr_vals, sl_rows, sl_cols, sl_vals, energy):
    """dense_gr / dense_gless (oracle.cpp:27-65)."""
    a = np.zeros((n, n), np.complex128)
    r, c, v = assemble(n, h_rows, h_cols, h_vals, sr_rows, sr_cols, sr_vals, energy)
    np.add.at(a, (r, c), v)
    s = np.zeros((n, n), np.complex128)
    np.add.at(s, (np.asarray(sl_rows), np.asarray(sl_cols)), sl_vals)
    g = np.linalg.inv(a)
    gl = g @ s @ g.conj().T
    return np.diag(g).copy(), np.diag(gl).copy()


def electron_density(gless: np.ndarray, weights: np.ndarray) -> np.ndarray:
    """(1/2pi) sum_k w_k Im G^<_jj with the Re-residual guard (observables.cpp:58-93)."""
    mag = np.abs(gless)
    if np.any(np.abs(gless.real) > 1e-8 * mag):
        raise RuntimeError("ResidualTooLarge")
    return (weights[:, None] * gless.imag).sum(0) / (2.0 * np.pi)
