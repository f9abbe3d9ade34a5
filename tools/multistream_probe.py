"""Probe: does splitting a rank's 256-energy step over S solver handles (each on
its own stream, 256/S energies) raise throughput by overlapping the latency-bound
inverse launches and launch tails of one slice with the GEMM launches of another?

    python tools/multistream_probe.py [--splits 1,2,4] [--steps 6]

Prints one line per split count (wall clock around a synchronised loop; a probe,
not a bench value).
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--splits", default="1,2,4")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--energies", type=int, default=256)
    args = ap.parse_args()
    import torch

    import bench
    from paper_1305_1070_b200 import negf

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    per = args.energies
    w = bench.make_workload(1, per)
    my = np.arange(per)
    plan = negf.HscPlan(w.problem)
    sr_h, sl_h = w.self_energies(my)
    E = torch.from_numpy(w.energies[my].copy()).to(dev)
    Wt = torch.from_numpy(w.weights[my].copy()).to(dev)
    SR = torch.from_numpy(sr_h).to(dev)
    SL = torch.from_numpy(sl_h).to(dev)
    for s in [int(x) for x in args.splits.split(",")]:
        n = per // s
        solvers = [negf.HscGpuSolver(plan, device=0, max_energy_batch=n) for _ in range(s)]
        for sv in solvers:
            sv.set_residual_check(False)

        def step():
            for i, sv in enumerate(solvers):
                sl = slice(i * n, (i + 1) * n)
                sv.solve_device(E[sl], Wt[sl], SR[sl], SL[sl], first_energy_index=i * n, sync=False)

        for _ in range(2):
            step()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize(dev)
        dt = (time.perf_counter() - t0) / args.steps
        for sv in solvers:
            sv.check()
        dens = sum(sv.density(reset=True) for sv in solvers)
        print(f"splits={s} energies/handle={n} ms/step={dt * 1e3:.2f} points/s={per / dt:.1f} "
              f"density_sum={float(dens.sum()):.12e}", flush=True)
        del solvers
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
