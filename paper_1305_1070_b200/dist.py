"""Energy-sharded sweep over ranks: the B200 replacement of solve_all's
std::thread energy pool (proj/src/run.cpp:218-264) plus the single exchange
of the path, the allreduce of the energy-partial density.

One process per GPU.  Energy points are independent, so rank r owns a
contiguous slice of the grid; per-energy outputs stay rank-local and the
density partials are summed once (NCCL over NVLink through the C ABI when the
process group is NCCL, the process group's own all_reduce otherwise, e.g.
gloo in the CPU tests).  Errors follow run.cpp:258-262 across ranks: the
lowest failing energy index wins, on every rank.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import negf


def shard(n_energies: int, world: int, rank: int) -> np.ndarray:
    """Contiguous, balanced slice of energy indices owned by `rank`."""
    base, extra = divmod(n_energies, world)
    start = rank * base + min(rank, extra)
    return np.arange(start, start + base + (1 if rank < extra else 0))


@dataclass
class SweepResult:
    indices: np.ndarray          # global energy indices solved on this rank
    gr: np.ndarray | None        # (len(indices), n) diag G^r
    gless: np.ndarray | None     # (len(indices), n) diag G^<
    density: np.ndarray          # global (1/2pi) sum_k w_k Im G^<_jj


def _error_key(exc: Exception) -> int:
    idx = getattr(exc, "energy_index", -1)
    return idx if idx is not None and idx >= 0 else 2**62


def sweep(solver, energies, weights, self_energies, group=None, batch: int | None = None,
          keep_diagonals: bool = True, use_nccl: bool | None = None) -> SweepResult:
    """Solve this rank's shard of the grid and return the global density.

    solver        an ``negf.HscGpuSolver`` (or any object with its solve /
                  density / allreduce_density surface)
    self_energies callable: global indices -> (sigma_r, sigma_lesser) rows
    group         torch.distributed process group (None: single process)
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if group is not None or dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    idx = shard(len(energies), world, rank)
    step = batch or max(1, getattr(solver, "capacity", len(idx)) or len(idx))
    grs, gls = [], []
    err: Exception | None = None
    # The reference raises any solver error from solve_all before
    # electron_density checks a residual (run.cpp:258-291): solve with the
    # residual guard recording only, settle solver errors across ranks, then
    # apply the guard to the whole grid.
    guard = bool(getattr(solver, "residual_check", True))
    if hasattr(solver, "set_residual_check"):
        solver.set_residual_check(False)
    if hasattr(solver, "residual_violation"):
        solver.residual_violation(reset=True)
    try:
        for s0 in range(0, len(idx), step):
            sel = idx[s0:s0 + step]
            sr, sl = self_energies(sel)
            try:
                gr, gl = solver.solve(np.asarray(energies)[sel], np.asarray(weights)[sel], sr, sl,
                                      first_energy_index=int(sel[0]), want_diagonals=keep_diagonals)
            except negf.NegfError as exc:
                err = exc
                break
            if keep_diagonals:
                grs.append(gr)
                gls.append(gl)
    finally:
        if hasattr(solver, "set_residual_check"):
            solver.set_residual_check(guard)
    if world > 1:
        import torch

        key = torch.tensor([_error_key(err) if err is not None else 2**62], dtype=torch.int64)
        if dist.get_backend(group) == "nccl":
            key = key.cuda()
        dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)
        lowest = int(key.item())
        if lowest < 2**62:
            owner = [err if (err is not None and _error_key(err) == lowest) else None]
            gathered = [None] * world
            dist.all_gather_object(gathered, owner[0], group=group)
            first = next(e for e in gathered if e is not None)
            raise first
    elif err is not None:
        raise err
    if guard and hasattr(solver, "residual_violation"):
        v = solver.residual_violation(reset=True)
        key = (v[0] << 32 | v[1]) if v is not None else 2**62
        if world > 1:
            import torch

            t = torch.tensor([key], dtype=torch.int64)
            if dist.get_backend(group) == "nccl":
                t = t.cuda()
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
            key = int(t.item())
        if key < 2**62:
            e, d = key >> 32, key & 0xFFFFFFFF
            raise negf.ResidualTooLarge(
                f"energy point {e}: G^< diagonal entry has a real part beyond the skew-Hermitian tolerance "
                f"at dof {d}", e, d)
    if world > 1:
        nccl = use_nccl if use_nccl is not None else dist.get_backend(group) == "nccl"
        if nccl:
            solver.allreduce_density()          # ncclAllReduce inside the C ABI
            dens = solver.density()
        else:  # same semantics as the C ABI's ordered reduction
            dens = ordered_sum(solver.density() * (2.0 * np.pi), group) / (2.0 * np.pi)
    else:
        dens = solver.density()
    return SweepResult(idx, np.concatenate(grs) if grs else None, np.concatenate(gls) if gls else None, dens)


def ordered_sum(part: np.ndarray, group=None) -> np.ndarray:
    """All-gather the per-rank partials and sum them in rank order: the same
    result for any NCCL/gloo algorithm, bit-reproducible run to run (SURVEY
    §8(e)); the C ABI does the same on the device (negf_gpu_allreduce_density)."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.ascontiguousarray(part, np.float64))
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, t, group=group)
    out = parts[0].clone()
    for p in parts[1:]:
        out += p
    return out.numpy()


def init_nccl(solver, group=None) -> None:
    """Bootstraps the C ABI's NCCL communicator from the process group."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    uid = [negf.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0, group=group)
    solver.nccl_init(uid[0], world, rank)
