"""Full-size throughput of BASELINE configs 4 / 5 on one B200 (not a bench
line: the bench workload is config 2).  One batch at the device's capacity,
device-resident energies, contact self-energies built on the GPU, timed with
CUDA events on the solver stream after a warm-up batch; per-kernel-kind and
per-level FP64 rates from the per-op events.

    python tools/fullsize_throughput.py 5      # or 4
"""
import json
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1305_1070_b200 import devices, negf  # noqa: E402

PEAK = 37.18  # measured DMMA TFLOP/s (profiles/fp64_peak_r01.txt)

cfg = int(sys.argv[1])
w = devices.config5() if cfg == 5 else devices.config4(ref_orientation=len(sys.argv) > 2 and sys.argv[2] == "ref")
t0 = time.time()
plan = negf.HscPlan(w.problem)
plan_s = time.time() - t0
info = plan.info()
solver = negf.HscGpuSolver(plan, device=0)
solver.set_residual_check(False)
B = solver.capacity
dev = torch.device("cuda", 0)
idx = np.linspace(0, len(w.energies) - 1, B).round().astype(np.int64)
E = torch.from_numpy(w.energies[idx].copy()).to(dev)
W = torch.from_numpy(w.weights[idx].copy()).to(dev)
gen = devices.GpuSelfEnergies(w, device=0, max_energy_batch=B)
stream = torch.cuda.ExternalStream(solver.stream_ptr, device=dev)
with torch.cuda.stream(stream):
    SR, SL = gen(E)
    solver.solve_device(E, W, SR, SL, sync=False)  # warm-up
    torch.cuda.synchronize(dev)
    solver.profile(True)
    solver.profile_read(reset=True)
    solver.profile_ops(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    SR, SL = gen(E, SR, SL)
    solver.solve_device(E, W, SR, SL, sync=False)
    e1.record(stream)
    torch.cuda.synchronize(dev)
ms = e0.elapsed_time(e1)
ks = solver.profile_read(reset=True)
op_ms = solver.profile_ops(reset=True)
solver.check()
ops = plan.ops()
by_level = {}
for cname, lo, hi in (("leaves", 1, 1), ("levels 2-4", 2, 4), ("levels >= 5", 5, 99)):
    sel = (ops["kind"] == 1) & (ops["level"] >= lo) & (ops["level"] <= hi)
    t = float(op_ms[sel].sum())
    if t > 0:
        by_level[f"gemm {cname}"] = round(8.0 * float(ops["cmul"][sel].sum()) * B / (t * 1e-3) / 1e12, 2)
inv = {}
for name, sel in (("inverse (single CTA)", ops["kind"] == 0), ("panel", ops["kind"] == 4), ("perm", ops["kind"] == 5),
                  ("bigswap", ops["kind"] == 11), ("inverse GEMM updates", (ops["kind"] == 1) & (ops["phase"] == 6))):
    t = float(op_ms[sel].sum())
    inv[name] = {"ms": round(t, 2), "launches": int(sel.sum()),
                 "tflops": round(8.0 * float(ops["cmul"][sel].sum()) * B / (t * 1e-3) / 1e12, 2) if t > 0 else None}
exec_gf = info.exec_flops / 1e9
out = dict(config=cfg, n_dofs=info.n_dofs, clusters=info.n_clusters, levels=info.levels,
           max_block=info.max_block, arena_mib_per_energy=info.arena_bytes_per_energy / 2**20, batch=B, ms=ms,
           points_per_s=B / (ms / 1e3), exec_gflop_per_point=exec_gf,
           ref_ledger_gflop_per_point=info.ref_ledger_flops / 1e9,
           step_tflops=exec_gf * B / ms, step_frac=exec_gf * B / ms / PEAK,
           gemm_tflops=8.0 * ks["gemm"]["cmul"] / (ks["gemm"]["ms"] * 1e-3) / 1e12,
           kernels_ms={k: round(v["ms"], 1) for k, v in ks.items()}, gemm_tflops_by_level=by_level,
           plan_s=plan_s, max_real_residual=solver.max_real_residual, inverse_ops=inv)
print(json.dumps(out))
