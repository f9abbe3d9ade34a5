"""Per-op CUDA-event profile of one config-2 batch (or a plan-only shape dump).

    python tools/op_profile.py plan            # CPU: op list with task shapes (no GPU)
    python tools/op_profile.py run [reps]      # GPU: per-op ms / TF/s, grouped and top ops

Kinds: 0 inverse, 1 gemm, 2 diag, 3 scale, 4 bigpanel, 5 bigperm, 6 skew, 7 combine,
8 spsi, 9 sschur, 10 leafdiag, 11 bigswap, 12 mgather.  Phases: 0 fold, 1 G, 2 seed, 3 N fold, 4 P, 6 big inverse.
"""
import collections
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402

NE = 256
KIND = {0: "inverse", 1: "gemm", 2: "diag", 3: "scale", 4: "bigpanel", 5: "bigperm", 6: "skew", 7: "combine",
        8: "spsi", 9: "sschur", 10: "leafdiag", 11: "bigswap", 12: "mgather"}
PEAK = 37.18


def shapes(plan, ops):
    tk = plan.gemm_tasks()
    tl = plan.gemm_tiles()
    out = []
    for i in range(len(ops["kind"])):
        k, b, c = int(ops["kind"][i]), int(ops["begin"][i]), int(ops["count"][i])
        if k == 1 and c > 0:
            t = np.unique(tl["task"][b:b + c])
            m, n, kk = tk["m"][t], tk["n"][t], tk["k"][t]
            out.append(f"tiles {c:5d} tasks {len(t):5d}  m {m.mean():6.1f} [{m.min()}-{m.max()}]  n {n.mean():6.1f} "
                       f"[{n.min()}-{n.max()}]  k {kk.mean():7.1f} [{kk.min()}-{kk.max()}]")
        else:
            out.append(f"count {c}")
    return out


def main():
    from paper_1305_1070_b200 import devices, negf
    mode = sys.argv[1] if len(sys.argv) > 1 else "plan"
    cfg = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    w = devices.config2(n_energies=NE if mode == "run" else 2) if cfg == 2 else None
    plan = negf.HscPlan(w.problem)
    ops = plan.ops()
    sh = shapes(plan, ops)
    if mode == "plan":
        for i in range(len(ops["kind"])):
            print(f"op {i:4d} {KIND[int(ops['kind'][i])]:9s} ph {ops['phase'][i]} lv {ops['level'][i]:2d} "
                  f"GF/E {8e-9 * ops['cmul'][i]:7.4f}  {sh[i]}")
        return
    import torch
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    solver = negf.HscGpuSolver(plan, device=0, max_energy_batch=NE)
    solver.set_residual_check(False)
    sr, sl = w.self_energies(np.arange(NE))
    dev = torch.device("cuda", 0)
    args = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (w.energies, w.weights, sr, sl)]
    for _ in range(2):
        solver.solve_device(*args)
    torch.cuda.synchronize()
    solver.profile(True)
    solver.profile_ops(reset=True)
    for _ in range(reps):
        solver.solve_device(*args)
    torch.cuda.synchronize()
    ms = solver.profile_ops(reset=True) / reps
    solver.profile(False)
    fl = 8.0 * ops["cmul"] * NE
    tot = ms.sum()
    print(f"total {tot:.2f} ms per {NE}-energy batch ({NE / tot * 1e3:.1f} points/s)")
    grp = collections.defaultdict(lambda: [0.0, 0.0, 0])
    for i in range(len(ms)):
        key = (KIND[int(ops["kind"][i])], int(ops["phase"][i]), min(int(ops["level"][i]), 99))
        g = grp[key]
        g[0] += ms[i]
        g[1] += fl[i]
        g[2] += 1
    print("\n== by (kind, phase, level)")
    for key, (m, f, c) in sorted(grp.items(), key=lambda kv: -kv[1][0]):
        tf = f / (m * 1e-3) / 1e12 if m > 0 else 0
        print(f"{key[0]:9s} ph {key[1]} lv {key[2]:2d}  ops {c:3d}  {m:8.3f} ms  {100 * m / tot:5.1f} %  "
              f"{tf:6.2f} TF/s ({tf / PEAK:5.1%})")
    print("\n== top 40 ops")
    for i in np.argsort(-ms)[:40]:
        tf = fl[i] / (ms[i] * 1e-3) / 1e12 if ms[i] > 0 else 0
        print(f"op {i:4d} {KIND[int(ops['kind'][i])]:9s} ph {ops['phase'][i]} lv {ops['level'][i]:2d} "
              f"{ms[i]:7.3f} ms {tf:6.2f} TF/s  {sh[i]}")


if __name__ == "__main__":
    main()
