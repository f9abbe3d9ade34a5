#!/usr/bin/env python
"""Throughput of the B200 HSC path on BASELINE.json configs[1] (config 2:
400 x 100 quantum-well superlattice, 256 energy points per GPU per step).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU)

A step is one pass of the hot path over the rank's 256 energy points: A(E)
assembly, fold, G^r / N / G^< sweeps, per-dof diagonals and the weighted
density sum, plus (N > 1) the NCCL allreduce of the density.  Weak scaling:
every rank owns 256 points of an N*256-point grid on [0, 0.4] eV.
Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "energy points/sec (diag G^r+G^<) per GPU & 8×B200; FP64 tensor-peak fraction"
UNIT = "energy points/s"
FP64_PEAK_TFLOPS = 37.18  # DMMA m8n8k4 micro-benchmark on this pool's B200 (profiles/fp64_peak_r01.txt)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.lines: list[str] = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------
def make_workload(n_ranks: int, per_rank: int):
    from paper_1305_1070_b200 import devices

    # N*per_rank-point grid on [0, 0.4]; rank r owns the contiguous slice r.
    return devices.config2(n_energies=n_ranks * per_rank)


def bench_config(w, world: int, per_rank: int) -> dict:
    """The workload description both arms print (identical dicts, so the
    driver can match the reference arm's line with ours)."""
    return {"workload": w.name, "description": w.description, "n_dofs": w.n,
            "energy_grid": f"{world * per_rank} uniform points on [0, 0.4] eV, eta = 1e-6 (leads), "
                           f"rank r owns the contiguous slice of {per_rank}",
            "energies_per_gpu": per_rank,
            "l2": "inputs larger than L2: a step streams all per-energy arenas (tens of GiB) through HBM"}


def ref_problem_file(w, idx: np.ndarray, path: str) -> None:
    """The reference-arm / cpu_baseline input: the same arrays, in the
    reference's own terms (contacts + phonon diagonal)."""
    from oracle import refio

    sr, sl = w.self_energies(idx)
    p = w.problem
    ny = w.ny
    w2 = ny * ny
    rp = refio.RefProblem(
        n=p.n, h_rows=p.h_rows, h_cols=p.h_cols, h_vals=p.h_vals, layers=[np.asarray(l) for l in p.layers],
        coords=p.coords, groups=[np.asarray(g, np.int32) for g in p.atomic_groups], max_leaf=p.max_leaf,
        dofs_l=np.asarray(p.atomic_groups[0], np.int32), dofs_r=np.asarray(p.atomic_groups[1], np.int32),
        has_ph=False, has_ph_less=False, energies=w.energies[idx], weights=w.weights[idx],
        sig_l=sr[:, :w2].reshape(-1, ny, ny), sig_r=sr[:, w2:2 * w2].reshape(-1, ny, ny), ph=None,
        less_l=sl[:, :w2].reshape(-1, ny, ny), less_r=sl[:, w2:2 * w2].reshape(-1, ny, ny), ph_less=None)
    refio.write_problem(rp, path)


def run_reference_sample(w, n_energies: int, threads: int, tmpdir: str, offset: int = 0) -> dict:
    from oracle import refio

    idx = (offset + np.linspace(0, len(w.energies) - 1, n_energies).astype(int)) % len(w.energies)
    prob = os.path.join(tmpdir, f"ref_{n_energies}_{offset}.bin")
    if not os.path.exists(prob):
        ref_problem_file(w, idx, prob)
    res = refio.run_reference(prob, os.path.join(tmpdir, "ref.out"), threads=threads)
    if res.status != 0:
        raise RuntimeError(f"reference failed: {res.message}")
    return {"energies": n_energies, "wall_s": res.wall_s, "tree_s": res.tree_s, "threads": threads,
            "mul_ops": res.mul_ops, "inv_ops": res.inv_ops}


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU solver on all host cores
# ---------------------------------------------------------------------------
def bench_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    from oracle import refio

    if not refio.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_driver not built"}))
        return
    w = make_workload(world, args.energies)
    cores = host_cores()
    per_step = cores  # one energy point per core per step (bounded sample)
    with tempfile.TemporaryDirectory() as tmp:
        walls = []
        for s in range(args.warmup + args.steps):
            r = run_reference_sample(w, per_step, cores, tmp, offset=s)
            if s >= args.warmup:
                walls.append(r["wall_s"])
                log(f"[reference] step {s - args.warmup}: {per_step} energies in {r['wall_s']:.2f} s")
    ms = 1e3 * float(np.mean(walls))
    value = per_step / (ms / 1e3)
    sample = f"{per_step} energy points of config 2 per step ({cores} threads, 1 point per thread)"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic",
        "config": bench_config(w, world, args.energies),
        "step": {"energies_per_step": per_step,
                 "solver": "reference hsc_fold+hsc_gless (oracle/_ref, OpenBLAS-backed dense shim), "
                           "std::thread energy pool (solve_all, run.cpp:218-264)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def level_breakdown(ops, op_ms, energies_timed, steps):
    """FP64 rate of the GEMM and inverse ops by tree-level class (leaves /
    small separators / large separators), from per-op CUDA events."""
    classes = (("leaves (level 1)", 1, 1), ("separators, levels 2-4", 2, 4), ("separators, levels >= 5", 5, 99))
    out = {}
    inv_gemm = (ops["kind"] == 1) & (ops["phase"] == 6)  # GEMM updates inside multi-CTA inverses
    for kname, base in (("gemm", (ops["kind"] == 1) & ~inv_gemm),
                        ("inverse", np.isin(ops["kind"], (0, 4, 5, 11)) | inv_gemm)):
        for cname, lo, hi in classes:
            sel = base & (ops["level"] >= lo) & (ops["level"] <= hi)
            ms = float(op_ms[sel].sum())
            fl = 8.0 * float(ops["cmul"][sel].sum()) * energies_timed
            if ms > 0:
                out[f"{kname}: {cname}"] = {"ms_per_step": ms / steps, "tflops": fl / (ms * 1e-3) / 1e12,
                                             "frac": fl / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS}
    return out


def bench_fullsize(cfg: int, local_rank: int, reps: int = 2) -> dict:
    """One full-size BASELINE config beside the headline (config 4: 1024 x
    1024, 1024-wide top separators; config 5: 512 x 512 + phonon): a batch at
    the device's capacity, spread over the config's energy grid, device-
    resident energies, contact self-energies built on the GPU inside the
    timed region; one warm-up batch, then `reps` timed batches (CUDA events on
    the solver stream)."""
    import torch

    from paper_1305_1070_b200 import devices, negf

    dev = torch.device("cuda", local_rank)
    w = devices.config4() if cfg == 4 else devices.config5()
    t0 = time.perf_counter()
    plan = negf.HscPlan(w.problem)
    plan_s = time.perf_counter() - t0
    info = plan.info()
    solver = negf.HscGpuSolver(plan, device=local_rank)
    solver.set_residual_check(False)
    B = solver.capacity
    idx = np.linspace(0, len(w.energies) - 1, B).round().astype(np.int64)
    E = torch.from_numpy(w.energies[idx].copy()).to(dev)
    W = torch.from_numpy(w.weights[idx].copy()).to(dev)
    gen = devices.GpuSelfEnergies(w, device=local_rank, max_energy_batch=B)
    stream = torch.cuda.ExternalStream(solver.stream_ptr, device=dev)
    with torch.cuda.stream(stream):
        SR, SL = gen(E)
        solver.solve_device(E, W, SR, SL, sync=False)
        torch.cuda.synchronize(dev)
        solver.profile(True)
        solver.profile_read(reset=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            SR, SL = gen(E, SR, SL)
            solver.solve_device(E, W, SR, SL, sync=False)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / reps
    ks = solver.profile_read(reset=True)
    solver.profile(False)
    solver.check()
    gf = info.exec_flops / 1e9
    out = {"workload": w.name, "n_dofs": w.n, "clusters": info.n_clusters, "max_block": info.max_block,
           "value": B / (ms / 1e3), "unit": UNIT, "batch": B, "ms_per_batch": ms, "timed_batches": reps,
           "exec_gflop_per_energy": gf, "ref_ledger_gflop_per_energy": info.ref_ledger_flops / 1e9,
           "fp64_tflops_step": gf * B / ms, "fp64_peak_frac_step": gf * B / ms / FP64_PEAK_TFLOPS,
           "kernels_ms_per_batch": {k: round(v["ms"] / reps, 2) for k, v in ks.items()},
           "plan_seconds": plan_s, "max_real_residual": solver.max_real_residual}
    del solver, plan, gen, SR, SL
    torch.cuda.synchronize(dev)
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def bench_ours(args, rank: int, world: int, local_rank: int) -> None:
    import torch
    import torch.distributed as dist

    from paper_1305_1070_b200 import devices, negf

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    per_rank = args.energies
    w = make_workload(world, per_rank)
    my = np.arange(rank * per_rank, (rank + 1) * per_rank)
    t0 = time.perf_counter()
    plan = negf.HscPlan(w.problem)
    info = plan.info()
    plan_s = time.perf_counter() - t0
    solver = negf.HscGpuSolver(plan, device=local_rank, max_energy_batch=per_rank)
    # The reference's own solver leaves |Re G^<_jj| / |G^<_jj| up to ~5e-7 on
    # this eta = 1e-6 workload, and 0.53 at the breakdown energy (index 199,
    # DESIGN.md §4) -- its electron_density guard of 1e-8 would stop the
    # reference run too; record the residual instead of raising.
    solver.set_residual_check(False)
    if solver.capacity < per_rank:
        log(f"[bench] batch capacity {solver.capacity} < {per_rank}: solving in chunks")
    sr_h, sl_h = w.self_energies(my)
    E = torch.from_numpy(w.energies[my].copy()).to(dev)
    Wt = torch.from_numpy(w.weights[my].copy()).to(dev)
    SR = torch.from_numpy(sr_h).to(dev)
    SL = torch.from_numpy(sl_h).to(dev)
    stream = torch.cuda.ExternalStream(solver.stream_ptr, device=dev)
    # The one exchange: the density partials over the C ABI's own NCCL
    # communicator (rank-ordered all-gather + sum).  Decided collectively: if
    # any rank cannot bring it up, every rank reduces the same way over the
    # torch process group instead (still rank-ordered, still on the GPU).
    reduce_mode = "none"
    if world > 1:
        ok = 1
        uid = [None]
        if rank == 0:
            try:
                uid = [negf.nccl_unique_id()]
            except negf.NegfError:
                uid = [None]
        dist.broadcast_object_list(uid, src=0)
        try:
            if uid[0] is None:
                raise negf.NcclError("no NCCL unique id")
            solver.nccl_init(uid[0], world, rank)
        except negf.NegfError as exc:
            log(f"[bench] rank {rank}: C-ABI NCCL unavailable ({exc})")
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        reduce_mode = "negf-nccl" if int(flag.item()) == 1 else "torch"

    class _DensityView:  # zero-copy torch view of the solver's density accumulator
        def __init__(self, ptr, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}

    dens_dev = torch.as_tensor(_DensityView(solver.density_ptr, w.n), device=dev) if reduce_mode == "torch" else None

    def reduce_density():
        if reduce_mode == "negf-nccl":
            solver.allreduce_density()
        elif reduce_mode == "torch":
            with torch.cuda.stream(stream):
                parts = [torch.empty_like(dens_dev) for _ in range(world)]
                dist.all_gather(parts, dens_dev)
                s = parts[0].clone()
                for p in parts[1:]:
                    s += p
                dens_dev.copy_(s)

    def step():
        solver.solve_device(E, Wt, SR, SL, first_energy_index=int(my[0]), sync=False)
        if world > 1:
            reduce_density()

    for _ in range(args.warmup):
        step()
    solver.check()
    launches_per_step = solver.last_launches
    # ---- timed region (device events on the solver's stream, max over ranks)
    clocks = ClockSampler(local_rank)
    clocks.start()
    solver.profile(True)
    solver.profile_read(reset=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    kstats = solver.profile_read(reset=True)
    op_ms = solver.profile_ops(reset=True)
    solver.profile(False)
    by_level = level_breakdown(plan.ops(), op_ms, per_rank * args.steps, args.steps)
    clk = clocks.stop()
    solver.check()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * per_rank / (ms_max / 1e3)

    # ---- e2e: the public host-buffer call, H2D inputs + D2H diagonals inside
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    e_h, w_h = pin(w.energies[my].copy()), pin(w.weights[my].copy())
    sr_p, sl_p = pin(sr_h), pin(sl_h)
    gr_p = pin(np.empty((per_rank, w.n), np.complex128))
    gl_p = pin(np.empty((per_rank, w.n), np.complex128))
    dens = pin(np.empty(w.n, np.float64))

    def e2e_step():
        solver.solve(e_h, w_h, sr_p, sl_p, first_energy_index=int(my[0]), out_gr=gr_p, out_gless=gl_p)
        if world > 1:
            reduce_density()
        dens[:] = solver.density()

    e2e_step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    f1.record(stream)
    torch.cuda.synchronize(dev)
    ms_e2e = torch.tensor([f0.elapsed_time(f1) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_e2e, op=dist.ReduceOp.MAX)
    e2e_value = world * per_rank / (float(ms_e2e.item()) / 1e3)
    h2d = int(e_h.nbytes + w_h.nbytes + sr_p.nbytes + sl_p.nbytes)
    d2h = int(gr_p.nbytes + gl_p.nbytes + dens.nbytes)

    # ---- energies-only e2e: host energies/weights in, the contact
    # self-energies built on the GPU, diagonals +
    # density out -- the whole per-energy loop of solve_all on the device.
    gen = devices.GpuSelfEnergies(w, device=local_rank)
    E_d, W_d = torch.empty_like(E), torch.empty_like(Wt)
    SR_d, SL_d = torch.empty_like(SR), torch.empty_like(SL)
    gr_d = torch.empty((per_rank, w.n), dtype=torch.complex128, device=dev)
    gl_d = torch.empty_like(gr_d)
    # torch-owned pinned buffers (a tensor made from a numpy view of pinned
    # memory is not flagged pinned, and its copies would be synchronous)
    e_t = torch.from_numpy(e_h.copy()).pin_memory()
    w_t = torch.from_numpy(w_h.copy()).pin_memory()
    gr_t = torch.empty((per_rank, w.n), dtype=torch.complex128).pin_memory()
    gl_t = torch.empty((per_rank, w.n), dtype=torch.complex128).pin_memory()

    s2 = torch.cuda.Stream(dev)  # torch-owned: host<->device copies + self-energies

    def e2e_gpu_sigma_step():
        with torch.cuda.stream(s2):
            E_d.copy_(e_t, non_blocking=True)
            W_d.copy_(w_t, non_blocking=True)
            gen(E_d, SR_d, SL_d)
        stream.wait_stream(s2)
        solver.solve_device(E_d, W_d, SR_d, SL_d, first_energy_index=int(my[0]), out_gr=gr_d, out_gless=gl_d,
                            sync=False)
        if world > 1:
            reduce_density()
        s2.wait_stream(stream)
        with torch.cuda.stream(s2):
            gr_t.copy_(gr_d, non_blocking=True)
            gl_t.copy_(gl_d, non_blocking=True)
        dens[:] = solver.density()

    e2e_gpu_sigma_step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    g0 = torch.cuda.Event(enable_timing=True)
    g1 = torch.cuda.Event(enable_timing=True)
    g0.record(s2)
    for _ in range(args.steps):
        e2e_gpu_sigma_step()
    g1.record(s2)
    torch.cuda.synchronize(dev)
    ms_e2g = torch.tensor([g0.elapsed_time(g1) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_e2g, op=dist.ReduceOp.MAX)
    e2g_value = world * per_rank / (float(ms_e2g.item()) / 1e3)
    solver.check()

    # ---- the paper's comparison baseline on the same GPU: layered RGF
    # (rgf_gr + rgf_gless), same inputs, device-resident.
    max_resid = solver.max_real_residual
    rgf = None
    if not args.no_rgf:
        # the HSC arenas are no longer needed: give the RGF a full batch
        del gen, SR_d, SL_d, gr_d, gl_d
        del solver
        torch.cuda.synchronize(dev)
        torch.cuda.empty_cache()
        rplan = negf.RgfPlan(w.problem)
        rs = negf.HscGpuSolver(rplan, device=local_rank, max_energy_batch=per_rank)
        rs.set_residual_check(False)
        rstream = torch.cuda.ExternalStream(rs.stream_ptr, device=dev)
        rs.solve_device(E, Wt, SR, SL, first_energy_index=int(my[0]))
        torch.cuda.synchronize(dev)
        r0 = torch.cuda.Event(enable_timing=True)
        r1 = torch.cuda.Event(enable_timing=True)
        r0.record(rstream)
        rs.solve_device(E, Wt, SR, SL, first_energy_index=int(my[0]), sync=False)
        r1.record(rstream)
        torch.cuda.synchronize(dev)
        rs.check()
        rms = r0.elapsed_time(r1)
        rinfo = rplan.info()
        rgf = {"value": per_rank / (rms / 1e3), "unit": UNIT, "ms_per_step": rms,
               "exec_gflop_per_energy": rinfo.exec_cmul * 8 / 1e9,
               "fp64_tflops": rinfo.exec_cmul * 8 * per_rank / (rms / 1e3) / 1e12,
               "note": "layered RGF on the same GPU and inputs (one timed step, rank-local)"}
        del rs, rplan

    extra = {}
    if world == 1 and args.extra_configs:
        del E, Wt, SR, SL
        torch.cuda.empty_cache()
        for c in (int(x) for x in args.extra_configs.split(",")):
            try:
                extra[f"config{c}"] = bench_fullsize(c, local_rank)
                log(f"[bench] config {c}: {extra[f'config{c}']['value']:.2f} {UNIT}")
            except Exception as exc:  # reported, never fatal for the headline
                extra[f"config{c}"] = {"error": str(exc)}
    if rank != 0:
        return
    g = kstats["gemm"]
    gemm_tflops = 8.0 * g["cmul"] / (g["ms"] * 1e-3) / 1e12 if g["ms"] > 0 else 0.0
    step_tflops = 8.0 * info.exec_cmul * per_rank / (ms / 1e3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import refio

            if refio.ref_available():
                cores = host_cores()
                with tempfile.TemporaryDirectory() as tmp:
                    r = run_reference_sample(w, 6 * cores, cores, tmp)
                cpu = {"value": r["energies"] / r["wall_s"], "unit": UNIT, "cores": cores, "kind": "reference",
                       "sample": f"{r['energies']} evenly spaced energy points of config 2 on {cores} threads "
                                 f"(reference hsc_fold+hsc_gless, oracle/_ref), {r['wall_s']:.1f} s"}
        except Exception as exc:  # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": host_cores(), "kind": "reference",
                   "sample": f"failed: {exc}"}
    launches_timed = int(sum(v["launches"] for v in kstats.values()))
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic",
        "config": bench_config(w, world, per_rank),
        "parallelism": (f"energy-sharded x{world}, density reduced once per step "
                        f"({'C-ABI NCCL all-gather + rank-ordered sum' if reduce_mode == 'negf-nccl' else 'torch.distributed all-gather + rank-ordered sum'})")
                       if world > 1 else "single GPU",
        "plan": {"clusters": info.n_clusters, "levels": info.levels, "max_block": info.max_block,
                 "arena_mib_per_energy": info.arena_bytes_per_energy / 2**20,
                 "exec_gflop_per_energy": info.exec_flops / 1e9,
                 "needed_gflop_per_energy_8mkn": info.needed_flops / 1e9,
                 "real_clusters": info.n_real_clusters,
                 "ref_ledger_gflop_per_energy": info.ref_ledger_flops / 1e9,
                 "plan_seconds": plan_s, "max_real_residual": max_resid,
                 "fp64_tflops_step": step_tflops, "fp64_peak_frac_step": step_tflops / FP64_PEAK_TFLOPS,
                 "needed_8mkn_tflops_step": info.needed_flops * per_rank / (ms / 1e3) / 1e12,
                 "note": "exec = real FP64 flops the pipes execute: products with a real operand (blocks of "
                         "clusters the self-energies never reach have exactly zero imaginary parts) skip the "
                         "DMMAs of the zero part and count 1/2 (real x real, real inverses: 1/4); "
                         "needed_8mkn = the same needed-only work counted as complex throughout"},
        "roofline": {"bound": "tensor", "achieved": gemm_tflops, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": gemm_tflops / FP64_PEAK_TFLOPS, "traffic": traffic,
                     "kernel": "k_gemm (grouped complex GEMM, DMMA.8x8x4)",
                     "note": "achieved = executed real FP64 flops of k_gemm / its CUDA-event time; terms with a "
                             "real operand execute 2 (real x real: 1) of the 4 DMMAs of a complex product, so "
                             "most launches are bound by operand staging, not by the DMMA pipe",
                     "peak_source": "measured FP64 DMMA micro-benchmark (tools/fp64_peak.cu, profiles/fp64_peak_r01.txt); "
                                    "MEASURED_PEAKS.json has no FP64 figure",
                     "kernels": {k: {"ms_per_step": v["ms"] / args.steps,
                                     "tflops": (8.0 * v["cmul"] / (v["ms"] * 1e-3) / 1e12) if v["ms"] > 0 and v["cmul"] > 0 else None,
                                     "launches_per_step": v["launches"] / args.steps}
                                 for k, v in kstats.items()},
                     "by_level": by_level},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "e2e_gpu_sigma": {"value": e2g_value, "unit": UNIT, "h2d_bytes_per_step": int(e_h.nbytes + w_h.nbytes),
                          "d2h_bytes_per_step": d2h,
                          "note": "energies/weights in; contact self-energies built on the GPU "
                                  "(analytic lead modes + lesser fill) inside the timed region"},
        "rgf_gpu": rgf,
        "extra_configs": extra or None,
        "gpu_launches": launches_timed,
        "clocks": clk,
    }
    print(json.dumps(out))
    log(f"[bench] {value:.1f} {UNIT}  ({ms_max:.2f} ms/step, gemm {gemm_tflops:.2f} TF/s, step {step_tflops:.2f} TF/s, "
        f"e2e {e2e_value:.1f}, launches/step {launches_per_step})")


def relaunch(n: int) -> int:
    """`bench.py --gpus N` without a launcher: one rank per GPU through
    torch.distributed.run on 127.0.0.1 (the form the driver uses for N > 1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    log(f"[bench] launching {n} ranks: {' '.join(cmd)}")
    return subprocess.call(cmd)


def dry_run(args, rank: int, world: int) -> None:
    """Process-group plumbing of the N-rank run without a GPU: gloo barrier +
    max-over-ranks reduction of a per-rank number, rank 0 prints the line."""
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "max_over_ranks": float(t.item()),
                          "backend": "gloo" if world > 1 else "none"}))
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--energies", type=int, default=256, help="energy points per GPU per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-rgf", action="store_true", help="skip the GPU RGF comparison line")
    ap.add_argument("--extra-configs", default="4,5",
                    help="full-size BASELINE configs timed beside the headline at N=1 ('' = none)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher / process-group check only (gloo without CUDA): no solve")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        sys.exit(relaunch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        bench_reference(args, rank, world)
        return
    if args.dry_run:
        dry_run(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        bench_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
