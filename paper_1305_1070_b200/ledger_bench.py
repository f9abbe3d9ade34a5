"""GPU ledger bench mode: the reference's ``cmd_bench``
(run.cpp:361-419) on the B200 path.

For each (Nx, Ny) and solver (hsc, rgf) it builds the reference's synthetic
system (``devices.synthetic_system`` = make_synthetic_system), solves it at
E = 0 on the GPU and writes ``bench.csv`` in the reference's exact format
(``solver,Nx,Ny,multiply_ops,inverse_ops,wall_seconds``; ``skipped`` rows by
the same working-set rule) with the *reference ledger* counts, so the SPEC
slopes reproduce; ``bench_executed.csv`` adds what the GPU
actually executed (needed-only complex MACs, inversion m^3) and its time.

Reference ledgers: HSC from the host plan (hsc_fold + hsc_gless charges,
validated against the reference on every golden problem); RGF restated here
from rgf.cpp:181-380 and the dense.cpp charges (matmul m*k*n, inverse n^3,
``scaled`` n^2 unless alpha = +-1, diagonal scalings n^2, skew_half_product
k*n(n+1)/2 [+ n(n+1)/2 for alpha != +-1]), per coupling kind
(classify_coupling, rgf.cpp:30-66).
"""
from __future__ import annotations

import argparse
import os
import time

import numpy as np

from . import devices, negf


def _couplings(problem: negf.Problem, layers):
    """A's upper coupling blocks A_{l,l+1} = -H_{l,l+1} (Sigma^r is layer-local
    for the synthetic system) and their classify_coupling kind."""
    lay = [np.asarray(x) for x in layers]
    pos = {}
    for l, dofs in enumerate(lay):
        for k, d in enumerate(dofs):
            pos[int(d)] = (l, k)
    blocks = [np.zeros((len(lay[l]), len(lay[l + 1])), np.complex128) for l in range(len(lay) - 1)]
    for r, c, v in zip(problem.h_rows, problem.h_cols, problem.h_vals):
        lr, ir = pos[int(r)]
        lc, ic = pos[int(c)]
        if lc == lr + 1:
            blocks[lr][ir, ic] += -v
    out = []
    for b in blocks:
        diag = b.shape[0] == b.shape[1] and np.count_nonzero(b - np.diag(np.diag(b))) == 0
        if diag:
            d = np.diag(b)
            if np.all(d == d[0]) and d.size > 0 and d[0] != 0:
                out.append(("scaled", d[0], b.shape))
            else:
                out.append(("diag", None, b.shape))
        else:
            out.append(("dense", None, b.shape))
    return out


def rgf_reference_ledger(problem: negf.Problem, layers) -> tuple[int, int]:
    """(multiply_ops, inverse_ops) of rgf_gr + rgf_gless (rgf.cpp:181-380)."""
    n = [len(x) for x in layers]
    cps = _couplings(problem, layers)
    L = len(n)
    mul = 0
    inv = 0
    pm1 = lambda a: a == 1 or a == -1  # noqa: E731  (scaled() is free for +-1)
    up = lambda m: m * (m + 1) // 2  # noqa: E731
    # rgf_gr forward
    for i in range(L):
        if i > 0:
            kind, a, _ = cps[i - 1]
            p = n[i - 1]
            if kind == "scaled":
                mul += 0 if pm1(a * a) else p * p
            elif kind == "diag":
                mul += 2 * p * p
            else:
                mul += p * p * n[i] + n[i] * p * n[i]
        inv += n[i] ** 3
    # rgf_gr backward
    for i in range(L - 2, -1, -1):
        kind, a, _ = cps[i]
        ni, nj = n[i], n[i + 1]
        if kind == "scaled":
            mul += nj * nj * ni + (0 if pm1(-a) else nj * ni)
            mul += ni * ni * ni + (0 if pm1(a) else ni * ni)
            mul += 0 if pm1(-a) else ni * nj
        elif kind == "diag":
            mul += ni * ni                      # diag_scale_left
            mul += nj * nj * ni                 # matmul(gd_next, btg)
            mul += ni * ni * ni                 # matmul(btg^T, goff)
            mul += ni * nj                      # diag_scale_right
        else:
            mul += nj * nj * ni + ni * nj * ni + ni * nj * ni
    # rgf_gless forward
    for i in range(L):
        if i > 0:
            kind, a, _ = cps[i - 1]
            p = n[i - 1]
            if kind == "scaled":
                mul += 0 if pm1(a * np.conj(a)) else p * p
            elif kind == "diag":
                mul += 2 * p * p
            else:
                mul += n[i] * p * p + n[i] * p * n[i]
        mul += n[i] ** 3 + up(n[i]) * n[i]
    # rgf_gless backward
    for i in range(L - 2, -1, -1):
        kind, a, _ = cps[i]
        ni, nj = n[i], n[i + 1]
        if kind == "scaled":
            al = a * np.conj(a)
            mul += ni * ni * ni + up(ni) * ni + (0 if pm1(al) else up(ni))
        elif kind == "diag":
            mul += ni * ni + ni * nj * nj + up(ni) * nj
        else:
            mul += ni * nj * nj + up(ni) * nj
        mul += ni * ni * ni
    return int(mul), int(inv)


def bench_rows(sizes, solvers=("rgf", "hsc"), seed: int = 1, coupling_t: float = 1.0, fuzz: bool = False,
               max_leaf: int = 64, max_mem_mb: float = 1024.0, record_wall: bool = True, device: int = 0):
    """One dict per (size, solver), in cmd_bench's loop order."""
    rows = []
    for nx, ny in sizes:
        if nx < 1 or ny < 1:
            raise negf.ConfigError("bench sizes must be positive")
        for solver in solvers:
            if 16.0 * 8.0 * nx * nx * ny > max_mem_mb * 1048576.0:
                rows.append(dict(solver=solver, nx=nx, ny=ny, skipped=True))
                continue
            s = devices.synthetic_system(nx, ny, seed, fuzz, coupling_t, max_leaf=max_leaf)
            prob = s["problem"]
            t0 = time.perf_counter()
            plan = negf.RgfPlan(prob, s["layers"]) if solver == "rgf" else negf.HscPlan(prob)
            gpu = negf.HscGpuSolver(plan, device=device, max_energy_batch=1)
            gpu.set_residual_check(False)
            t1 = time.perf_counter()
            gpu.solve(np.zeros(1), np.ones(1), s["sr_vals"][None, :], s["sl_vals"][None, :])
            t2 = time.perf_counter()
            info = plan.info()
            if solver == "rgf":
                mul, inv = rgf_reference_ledger(prob, s["layers"])
            else:
                mul, inv = info.ref_fold_mul + info.ref_gless_mul, info.ref_fold_inv + info.ref_gless_inv
            rows.append(dict(solver=solver, nx=nx, ny=ny, skipped=False, multiply_ops=mul, inverse_ops=inv,
                             wall_seconds=(t2 - t0) if record_wall else 0.0, solve_seconds=t2 - t1,
                             exec_cmul=info.exec_cmul - info.exec_inv_cmul, exec_inv_cmul=info.exec_inv_cmul,
                             launches=gpu.last_launches))
            del gpu, plan
    return rows


def write_bench(out_dir: str, rows) -> None:
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "bench.csv"), "w") as f:
        f.write("solver,Nx,Ny,multiply_ops,inverse_ops,wall_seconds\n")
        for r in rows:
            if r["skipped"]:
                f.write(f"{r['solver']},{r['nx']},{r['ny']},skipped,skipped,skipped\n")
            else:
                f.write(f"{r['solver']},{r['nx']},{r['ny']},{r['multiply_ops']},{r['inverse_ops']},"
                        f"{negf.format_double(r['wall_seconds'])}\n")
    with open(os.path.join(out_dir, "bench_executed.csv"), "w") as f:
        f.write("solver,Nx,Ny,exec_multiply_ops,exec_inverse_ops,gpu_solve_seconds,gpu_launches\n")
        for r in rows:
            if not r["skipped"]:
                f.write(f"{r['solver']},{r['nx']},{r['ny']},{int(r['exec_cmul'])},{int(r['exec_inv_cmul'])},"
                        f"{negf.format_double(r['solve_seconds'])},{r['launches']}\n")


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--sizes", default="4x4,8x8,16x16,32x32", help="NxxNy list")
    ap.add_argument("--solvers", default="rgf,hsc")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--coupling", type=float, default=1.0)
    ap.add_argument("--fuzz", action="store_true")
    ap.add_argument("--max-leaf", type=int, default=64)
    ap.add_argument("--max-mem-mb", type=float, default=1024.0)
    ap.add_argument("--out", default="bench_out")
    a = ap.parse_args()
    sizes = [tuple(int(v) for v in s.split("x")) for s in a.sizes.split(",")]
    rows = bench_rows(sizes, a.solvers.split(","), a.seed, a.coupling, a.fuzz, a.max_leaf, a.max_mem_mb)
    write_bench(a.out, rows)
    print(open(os.path.join(a.out, "bench.csv")).read(), end="")


if __name__ == "__main__":
    main()
