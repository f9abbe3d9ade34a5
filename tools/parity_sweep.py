"""Per-energy parity study (test infrastructure; writes an .npz summary).

GPU (product path, one plan per variant of the exact-arithmetic plan forms,
NEGF_PLAN_FORMS) vs the reference build oracle/_ref over a whole energy grid,
next to the reference's own floor: the same reference algorithm with a
different matmul order (NEGF_SHIM_NAIVE=1).  With --dense (n <= 2500,
oracle.hpp:14) every arm is also compared with the reference's dense oracle
(dense_gr / dense_gless, oracle.cpp:27-65) as the truth.

    python tools/parity_sweep.py --cfg 2 --out gpurun_out/par/c2.npz \
        --variants "base;plain;symdiag_g,symdiag_p,sparse,hull,woodbury"
"""
import argparse
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import refio  # noqa: E402
from paper_1305_1070_b200 import devices, negf  # noqa: E402
from tests.helpers import per_energy_err, real_residual, workload_ref_problem  # noqa: E402


def workload(args):
    if args.cfg == 2:
        return devices.config2(ny=args.ny, nx=args.nx, complex_energy=args.complex_energy)
    if args.cfg == 4:
        return devices.config4(complex_energy=args.complex_energy)
    if args.cfg == 5:
        return devices.config5()
    if args.cfg == 3:
        return devices.config3(n_cells=args.cells, complex_energy=args.complex_energy)
    return devices.config1()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--ny", type=int, default=100)
    ap.add_argument("--nx", type=int, default=400)
    ap.add_argument("--cells", type=int, default=600, help="config 3: unit cells of the tube")
    ap.add_argument("--complex-energy", action="store_true")
    ap.add_argument("--energies", default="", help="comma list of indices (default: whole grid)")
    ap.add_argument("--variants", default="base")
    ap.add_argument("--naive", action="store_true", help="also run the NEGF_SHIM_NAIVE reference")
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--out", required=True)
    ap.add_argument("--ref-cache", default="", help="npz of the reference arms' diagonals (read if present, "
                                                    "else written)")
    args = ap.parse_args()
    w = workload(args)
    idx = np.arange(len(w.energies)) if not args.energies else np.array([int(x) for x in args.energies.split(",")])
    rp, sr, sl = workload_ref_problem(w, idx)
    res = {"idx": idx, "energies": w.energies[idx]}

    class _R:  # cached reference arm
        def __init__(self, gr, gless):
            self.gr, self.gless = gr, gless

    cached = {}
    if args.ref_cache and os.path.exists(args.ref_cache):
        z = np.load(args.ref_cache)
        for name in ("ref", "naive", "dense"):
            if f"{name}_gr" in z.files:
                cached[name] = _R(z[f"{name}_gr"], z[f"{name}_gl"])
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "p.bin")
        refio.write_problem(rp, path)
        arms = [("ref", {}, "hsc")]
        if args.naive:
            arms.append(("naive", {"NEGF_SHIM_NAIVE": "1"}, "hsc"))
        if args.dense:
            arms.append(("dense", {}, "dense"))
        ref = {}
        for name, env, solver in arms:
            if name in cached:
                ref[name] = cached[name]
                res[f"{name}_resid"] = real_residual(ref[name].gless)
                res[f"{name}_ldos_min"] = (-ref[name].gr.imag).min(axis=1) / np.abs(ref[name].gr).max(axis=1)
                continue
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            t0 = time.time()
            r = refio.run_reference(path, os.path.join(tmp, name + ".out"), threads=args.threads, solver=solver)
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k)
                else:
                    os.environ[k] = v
            print(f"{name}: status {r.status} {r.message[:100]} {time.time() - t0:.1f}s", flush=True)
            ref[name] = r
            res[f"{name}_resid"] = real_residual(r.gless)
            res[f"{name}_ldos_min"] = (-r.gr.imag).min(axis=1) / np.abs(r.gr).max(axis=1)
        if args.ref_cache and not cached:
            np.savez(args.ref_cache, **{f"{k}_{a}": getattr(v, b) for k, v in ref.items()
                                        for a, b in (("gr", "gr"), ("gl", "gless"))})
        for name in ref:
            if name != "ref":
                res[f"{name}_vs_ref_r"] = per_energy_err(ref[name].gr, ref["ref"].gr)
                res[f"{name}_vs_ref_l"] = per_energy_err(ref[name].gless, ref["ref"].gless)
        if "dense" in ref:
            for name in ref:
                if name != "dense":
                    res[f"{name}_vs_dense_r"] = per_energy_err(ref[name].gr, ref["dense"].gr)
                    res[f"{name}_vs_dense_l"] = per_energy_err(ref[name].gless, ref["dense"].gless)
    for v in [x for x in args.variants.split(";") if x and x != "none"]:
        # a variant is the comma list of enabled plan forms (NEGF_PLAN_FORMS);
        # "base" = the product's default set, "none" = no rewrite form
        tag = v.replace(",", "+")
        if v == "base":
            os.environ.pop("NEGF_PLAN_FORMS", None)
        else:
            os.environ["NEGF_PLAN_FORMS"] = "" if v == "plain" else v
        plan = negf.HscPlan(w.problem)
        s = negf.HscGpuSolver(plan, max_energy_batch=args.batch or len(idx))
        s.set_residual_check(False)
        t0 = time.time()
        gr, gl = s.solve(w.energies[idx], w.weights[idx], sr, sl)
        dt = time.time() - t0
        res[f"{tag}_vs_ref_r"] = per_energy_err(gr, ref["ref"].gr)
        res[f"{tag}_vs_ref_l"] = per_energy_err(gl, ref["ref"].gless)
        res[f"{tag}_resid"] = real_residual(gl)
        res[f"{tag}_ldos_min"] = (-gr.imag).min(axis=1) / np.abs(gr).max(axis=1)
        if "dense" in ref:
            res[f"{tag}_vs_dense_r"] = per_energy_err(gr, ref["dense"].gr)
            res[f"{tag}_vs_dense_l"] = per_energy_err(gl, ref["dense"].gless)
        e = np.maximum(res[f"{tag}_vs_ref_r"], res[f"{tag}_vs_ref_l"])
        print(f"{tag}: {dt:.1f}s  max err vs ref {e.max():.2e} at {idx[e.argmax()]}, "
              f"#>1e-10 {int((e > 1e-10).sum())}, median {np.median(e):.1e}, max resid {res[tag + '_resid'].max():.2e}",
              flush=True)
        del s, plan
    os.environ.pop("NEGF_PLAN_FORMS", None)
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    np.savez(args.out, **res)
    if "naive" in ref:
        f = np.maximum(res["naive_vs_ref_r"], res["naive_vs_ref_l"])
        print(f"floor (naive vs ref): max {f.max():.2e} at {idx[f.argmax()]}, #>1e-10 {int((f > 1e-10).sum())}")


if __name__ == "__main__":
    main()
