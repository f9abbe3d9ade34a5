"""CPU, world_size 2 over gloo: energy sharding, the density reduction and the
cross-rank error rule of the distributed sweep (dist.py), with the numpy
restatement standing in for the GPU solver (tests only)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hsc_numpy as hn
from paper_1305_1070_b200 import dist as pdist
from paper_1305_1070_b200 import negf
from tests.helpers import load_golden


class OracleSolver:
    """CPU stand-in with the HscGpuSolver surface (test infrastructure)."""

    def __init__(self, name, fail_at=None, resid_at=None):
        self.rp, self.prob, self.hsc, _ = load_golden(name)
        self.tree = hn.Tree(self.hsc.parent, self.hsc.dofs, self.rp.n)
        self.acc = np.zeros(self.rp.n)
        self.fail_at = fail_at or set()
        self.resid_at = resid_at or set()  # energies whose G^< gets a synthetic real part
        self.capacity = 2
        self.residual_check = True
        self._viol = None

    def set_residual_check(self, on):
        self.residual_check = bool(on)

    def residual_violation(self, reset=False):
        v = self._viol
        if reset:
            self._viol = None
        return v

    def solve(self, E, W, sr, sl, first_energy_index=0, want_diagonals=True):
        grs, gls = [], []
        for q, e in enumerate(E):
            gi = first_energy_index + q
            if gi in self.fail_at:
                raise negf.SingularBlock(f"energy point {gi}: synthetic failure", 0, gi, 0)
            p = self.prob
            gr, gl, _ = hn.solve_energy(self.tree, self.rp.n, p.h_rows, p.h_cols, p.h_vals, p.sr_rows, p.sr_cols,
                                        sr[q], p.sl_rows, p.sl_cols, sl[q], e)
            if gi in self.resid_at:
                gl = gl + 1e-3 * np.abs(gl)
            bad = np.nonzero(np.abs(gl.real) > 1e-8 * np.abs(gl))[0]
            if len(bad):
                v = (gi, int(bad[0]))
                self._viol = v if self._viol is None else min(self._viol, v)
                if self.residual_check:
                    raise negf.ResidualTooLarge(f"energy point {gi}: residual", gi, int(bad[0]))
            self.acc += W[q] * gl.imag
            grs.append(gr)
            gls.append(gl)
        return np.array(grs), np.array(gls)

    def density(self):
        return self.acc / (2.0 * np.pi)


def _grid():
    rp, _, _, _ = load_golden("syn_24x20_s5_fuzz")
    E = np.linspace(0.1, 0.9, 7)
    W = negf.trapezoid_weights(E)

    def se(sel):
        sr, sl = rp.values(np.zeros(len(sel), int))
        return sr, sl

    return E, W, se


def _worker(rank, world, port, fail_at, q, resid_at=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        E, W, se = _grid()
        solver = OracleSolver("syn_24x20_s5_fuzz", fail_at, resid_at)
        try:
            res = pdist.sweep(solver, E, W, se)
            q.put((rank, "ok", res.indices.tolist(), res.density))
        except negf.NegfError as exc:
            q.put((rank, "err", exc.energy_index, type(exc).__name__))
    finally:
        dist.destroy_process_group()


def _run(world, fail_at=None, resid_at=None):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fail_at, q, resid_at)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    return sorted(out, key=lambda x: x[0])


def test_shard_is_a_balanced_partition():
    for n in (1, 7, 256, 1024):
        for world in (1, 2, 3, 8):
            parts = [pdist.shard(n, world, r) for r in range(world)]
            allidx = np.concatenate(parts)
            assert np.array_equal(allidx, np.arange(n))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1


def test_two_ranks_match_single_process():
    E, W, se = _grid()
    ref = OracleSolver("syn_24x20_s5_fuzz")
    single = pdist.sweep(ref, E, W, se)
    out = _run(2)
    assert [o[1] for o in out] == ["ok", "ok"]
    assert out[0][2] + out[1][2] == list(range(len(E)))
    for o in out:
        assert np.allclose(o[3], single.density, rtol=1e-13, atol=1e-300)


def test_lowest_failing_energy_wins_across_ranks():
    out = _run(2, fail_at={5, 2})  # rank 0 owns 0..3, rank 1 owns 4..6
    assert [o[1] for o in out] == ["err", "err"]
    assert all(o[2] == 2 for o in out)


def test_density_reduction_is_rank_ordered_and_bitwise_reproducible():
    """The density partials are summed in rank order (all-gather + ordered
    sum, the same rule as the C ABI's ncclAllGather path): every rank holds
    bit-identical results equal to p0 + p1 + p2 computed in that order."""
    E, W, se = _grid()
    world = 3
    parts = []
    for r in range(world):
        s = OracleSolver("syn_24x20_s5_fuzz")
        idx = pdist.shard(len(E), world, r)
        sr, sl = se(idx)
        s.solve(E[idx], W[idx], sr, sl, first_energy_index=int(idx[0]))
        parts.append(s.density() * (2.0 * np.pi))
    expect = ((parts[0] + parts[1]) + parts[2]) / (2.0 * np.pi)
    out = _run(world)
    assert [o[1] for o in out] == ["ok"] * world
    for o in out:
        assert np.array_equal(o[3], expect)


def test_solver_error_beats_earlier_residual_across_ranks():
    """A residual violation at energy 1 (rank 0) must not hide a SingularBlock
    at energy 5 (rank 1): solve_all raises solver errors before
    electron_density checks residuals (run.cpp:258-291)."""
    out = _run(2, fail_at={5}, resid_at={1})
    assert [o[1] for o in out] == ["err", "err"]
    assert all(o[2] == 5 and o[3] == "SingularBlock" for o in out), out


def test_residual_guard_runs_after_the_whole_grid():
    out = _run(2, resid_at={5, 2})
    assert [o[1] for o in out] == ["err", "err"]
    assert all(o[2] == 2 and o[3] == "ResidualTooLarge" for o in out), out
