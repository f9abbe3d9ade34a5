"""Host-side API of the B200 HSC path, over the C ABI in include/negf_gpu.h.

Mirrors the reference's solver interface for this path (names, argument
meaning, error types):

* ``nested_dissection`` / ``SeparatorTree``  -- proj/include/negf/partition.hpp:19-87
* ``HscPlan``  -- build_tree + the structural analysis of hsc_fold/hsc_gless
  (proj/src/run.cpp:123-133, hsc.cpp), incl. the reference FlopLedger counts
* ``HscGpuSolver.solve`` -- solve_energy's HSC branch for a batch of energies
  (run.cpp:141-192): diag G^r, diag G^< per dof, plus the electron_density
  energy sum (observables.cpp:58-93)
* exceptions -- proj/include/negf/errors.hpp:15-74

There is no CPU fallback: if ``libnegf_b200.so`` is missing this module fails
to import, and without a GPU ``HscGpuSolver`` raises ``CudaError``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NEGF_LIB") or os.path.join(_HERE, "libnegf_b200.so")  # NEGF_LIB: variant builds


# ---------------------------------------------------------------------------
# errors (errors.hpp)
# ---------------------------------------------------------------------------
class NegfError(RuntimeError):
    """negf::Error"""


class ConfigError(NegfError):
    pass


class ContractViolation(NegfError):
    pass


class SingularBlock(NegfError):
    def __init__(self, msg: str, pivot_index: int, energy_index: int = -1, cluster: int = -1):
        super().__init__(msg)
        self.pivot_index = pivot_index
        self.energy_index = energy_index
        self.cluster = cluster

    def __reduce__(self):
        return (SingularBlock, (str(self), self.pivot_index, self.energy_index, self.cluster))


class PartitionViolation(NegfError):
    pass


class NonSkewHermitianInput(NegfError):
    def __init__(self, msg: str, energy_index: int = -1, cluster: int = -1):
        super().__init__(msg)
        self.energy_index = energy_index
        self.cluster = cluster

    def __reduce__(self):
        return (NonSkewHermitianInput, (str(self), self.energy_index, self.cluster))


class ResidualTooLarge(NegfError):
    def __init__(self, msg: str, energy_index: int = -1, dof: int = -1):
        super().__init__(msg)
        self.energy_index = energy_index
        self.dof = dof

    def __reduce__(self):
        return (ResidualTooLarge, (str(self), self.energy_index, self.dof))


class ConvergenceError(NegfError):
    def __init__(self, msg: str, energy_index: int = -1):
        super().__init__(msg)
        self.energy_index = energy_index

    def __reduce__(self):
        return (ConvergenceError, (str(self), self.energy_index))


class CudaError(NegfError):
    pass


class NcclError(NegfError):
    pass


class OutOfMemory(CudaError):
    pass


# ---------------------------------------------------------------------------
# C ABI
# ---------------------------------------------------------------------------
class _Status(C.Structure):
    _fields_ = [
        ("code", C.c_int),
        ("energy_index", C.c_int),
        ("cluster", C.c_int),
        ("pivot", C.c_int),
        ("dof", C.c_int),
        ("msg", C.c_char * 256),
    ]


class _Problem(C.Structure):
    _fields_ = [
        ("n_dofs", C.c_int),
        ("h_nnz", C.c_int64),
        ("h_rows", C.c_void_p),
        ("h_cols", C.c_void_p),
        ("h_vals", C.c_void_p),
        ("sr_nnz", C.c_int64),
        ("sr_rows", C.c_void_p),
        ("sr_cols", C.c_void_p),
        ("sl_nnz", C.c_int64),
        ("sl_rows", C.c_void_p),
        ("sl_cols", C.c_void_p),
        ("coords", C.c_void_p),
        ("n_groups", C.c_int),
        ("group_ptr", C.c_void_p),
        ("group_dofs", C.c_void_p),
        ("max_leaf", C.c_int),
        ("n_tree_clusters", C.c_int),
        ("tree_parent", C.c_void_p),
        ("tree_ptr", C.c_void_p),
        ("tree_dofs", C.c_void_p),
    ]


class _PlanInfo(C.Structure):
    _fields_ = [
        ("n_dofs", C.c_int),
        ("n_clusters", C.c_int),
        ("levels", C.c_int),
        ("root", C.c_int),
        ("max_block", C.c_int),
        ("arena_bytes_per_energy", C.c_int64),
        ("ref_fold_mul", C.c_int64),
        ("ref_fold_inv", C.c_int64),
        ("ref_gless_mul", C.c_int64),
        ("ref_gless_inv", C.c_int64),
        ("exec_cmul", C.c_double),
        ("exec_inv_cmul", C.c_double),
        ("n_ops", C.c_int),
        ("n_gemm_tasks", C.c_int),
        ("n_gemm_tiles", C.c_int),
        ("n_inv_tasks", C.c_int),
        ("needed_cmul", C.c_double),
        ("n_real_clusters", C.c_int),
        ("pad_", C.c_int),
    ]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -m paper_1305_1070_b200.build or __graft_entry__.build())"
        )
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64, st = C.c_void_p, C.c_int, C.c_int64, C.POINTER(_Status)
    sig = {
        "negf_plan_create": ([C.POINTER(_Problem), C.POINTER(vp), st], i32),
        "negf_plan_info_get": ([vp, C.POINTER(_PlanInfo)], i32),
        "negf_plan_tree": ([vp, vp, vp, vp, vp, vp], i32),
        "negf_plan_fill": ([vp, vp, vp], i32),
        "negf_plan_gemm_tasks": ([vp, vp, vp, vp, vp, vp], i32),
        "negf_plan_gemm_tiles": ([vp, vp, vp, vp, vp, vp], i32),
        "negf_plan_ops": ([vp, vp, vp, vp, vp, vp, vp], i32),
        "negf_plan_destroy": ([vp], None),
        "negf_rgf_plan_create": ([C.POINTER(_Problem), i32, vp, vp, C.POINTER(vp), st], i32),
        "negf_gpu_create": ([vp, i32, i32, C.POINTER(vp), st], i32),
        "negf_gpu_batch_capacity": ([vp], i32),
        "negf_gpu_solve_batch": ([vp, i32, vp, vp, vp, vp, i32, vp, vp, st], i32),
        "negf_gpu_solve_batch_device": ([vp, i32, vp, vp, vp, vp, i32, vp, vp, i32, st], i32),
        "negf_gpu_check": ([vp, st], i32),
        "negf_gpu_density": ([vp, vp, i32, st], i32),
        "negf_gpu_stream": ([vp], vp),
        "negf_gpu_density_device": ([vp], vp),
        "negf_gpu_last_launches": ([vp], i64),
        "negf_gpu_destroy": ([vp], None),
        "negf_nccl_unique_id": ([vp, st], i32),
        "negf_gpu_nccl_init": ([vp, vp, i32, i32, st], i32),
        "negf_gpu_allreduce_density": ([vp, st], i32),
        "negf_gpu_set_ordered_reduce": ([vp, i32], i32),
        "negf_gpu_profile": ([vp, i32], i32),
        "negf_gpu_set_residual_check": ([vp, i32], i32),
        "negf_gpu_max_real_residual": ([vp], C.c_double),
        "negf_gpu_residual_violation": ([vp, vp, vp, i32], i32),
        "negf_gpu_profile_read": ([vp, vp, i32], i32),
        "negf_gpu_profile_ops": ([vp, vp, i32], i32),
        "negf_lead_create": ([i32, i32, vp, vp, C.c_double, i32, C.c_double, i32, C.POINTER(vp), st], i32),
        "negf_lead_sigma": ([vp, i32, vp, i32, vp, st], i32),
        "negf_lead_sigma_device": ([vp, i32, vp, i32, vp, i64, st], i32),
        "negf_lead_last_sweeps": ([vp, vp], i32),
        "negf_lead_last_launches": ([vp], i64),
        "negf_lead_stream": ([vp], vp),
        "negf_lead_destroy": ([vp], None),
        "negf_lead_modes_sigma_device": ([i32, C.c_double, C.c_double, i32, vp, vp, i64, vp, st], i32),
        "negf_contacts_fill_device": ([i32, vp, C.c_double, i32, vp, i32, vp, i64, i64, C.c_double, vp, i64, vp,
                                       i64, vp, st], i32),
        "negf_format_double": ([C.c_double, C.c_char_p, i32], i32),
        "negf_write_solve_csv": ([C.c_char_p, i32, i32, i32, vp, vp, vp, st], i32),
        "negf_shard_writer_open": ([C.c_char_p, i32, i32, i32, i32, C.POINTER(vp), st], i32),
        "negf_shard_writer_append": ([vp, i32, i32, vp, vp, vp, st], i32),
        "negf_shard_writer_append_device": ([vp, i32, i32, vp, vp, vp, vp, st], i32),
        "negf_shard_writer_close": ([vp, st], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


class _Lib:
    """The C ABI library, mapped on first use: importing this module (for
    Problem / trapezoid_weights, e.g. by the input generators that the
    reference arm of bench.py shares) does not load libnegf_b200.so; the
    first ABI call does, and fails loudly if it is missing."""

    _real = None

    def __getattr__(self, name):
        if _Lib._real is None:
            _Lib._real = _load()
        return getattr(_Lib._real, name)


_lib = _Lib()
ABI_SYMBOLS = (
    "negf_rgf_plan_create negf_plan_create negf_plan_info_get negf_plan_tree negf_plan_fill negf_plan_gemm_tasks negf_plan_gemm_tiles negf_plan_ops negf_plan_destroy "
    "negf_gpu_create negf_gpu_batch_capacity negf_gpu_solve_batch negf_gpu_solve_batch_device "
    "negf_gpu_check negf_gpu_density negf_gpu_stream negf_gpu_density_device "
    "negf_gpu_last_launches negf_gpu_destroy negf_nccl_unique_id negf_gpu_nccl_init "
    "negf_gpu_allreduce_density negf_gpu_set_ordered_reduce negf_gpu_profile negf_gpu_profile_read negf_gpu_profile_ops negf_gpu_set_residual_check "
    "negf_gpu_max_real_residual negf_gpu_residual_violation negf_lead_create negf_lead_sigma negf_lead_sigma_device negf_lead_last_sweeps "
    "negf_lead_last_launches negf_lead_stream negf_lead_destroy negf_lead_modes_sigma_device "
    "negf_contacts_fill_device negf_format_double negf_write_solve_csv negf_shard_writer_open "
    "negf_shard_writer_append negf_shard_writer_append_device negf_shard_writer_close"
).split()

KSTAT_NAMES = ("gemm", "inverse", "diag", "scale", "assemble", "output")


class _KStat(C.Structure):
    _fields_ = [("ms", C.c_double), ("cmul", C.c_double), ("launches", C.c_int64)]


def _raise(st: _Status) -> None:
    code, msg = st.code, st.msg.decode(errors="replace")
    if code == 0:
        return
    if code == 1:
        raise SingularBlock(msg, st.pivot, st.energy_index, st.cluster)
    if code == 2:
        raise NonSkewHermitianInput(msg, st.energy_index, st.cluster)
    if code == 3:
        raise ContractViolation(msg)
    if code == 5:
        raise NcclError(msg)
    if code == 6:
        raise OutOfMemory(msg)
    if code == 7:
        raise ConfigError(msg)
    if code == 8:
        raise PartitionViolation(msg)
    if code == 9:
        raise ResidualTooLarge(msg, st.energy_index, st.dof)
    if code == 11:
        raise ConvergenceError(msg, st.energy_index)
    if code == 4:
        raise CudaError(msg)
    raise NegfError(msg)


def _ptr(a: np.ndarray | None) -> int | None:
    return None if a is None else a.ctypes.data


# ---------------------------------------------------------------------------
# problem description
# ---------------------------------------------------------------------------
@dataclass
class Problem:
    """Inputs of build_tree/solve_energy (run.cpp:123-192).

    A(E) = E I - H - Sigma^r(E); Sigma^r(E) and Sigma^<(E) have fixed patterns
    (sr_*/sl_*), their values come per energy from ``self_energies``.
    """

    n: int
    h_rows: np.ndarray
    h_cols: np.ndarray
    h_vals: np.ndarray
    sr_rows: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    sr_cols: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    sl_rows: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    sl_cols: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    coords: np.ndarray | None = None
    atomic_groups: Sequence[Sequence[int]] = ()
    max_leaf: int = 64
    tree_parent: Sequence[int] | None = None
    tree_dofs: Sequence[Sequence[int]] | None = None
    layers: Sequence[Sequence[int]] = ()

    def c_struct(self):
        keep = []

        def arr(x, dt):
            if x is None:
                return None
            a = np.ascontiguousarray(np.asarray(x), dtype=dt)
            keep.append(a)
            return a

        p = _Problem()
        p.n_dofs = int(self.n)
        hr, hc = arr(self.h_rows, np.int32), arr(self.h_cols, np.int32)
        hv = arr(self.h_vals, np.complex128)
        p.h_nnz, p.h_rows, p.h_cols, p.h_vals = len(hr), _ptr(hr), _ptr(hc), _ptr(hv)
        sr, sc = arr(self.sr_rows, np.int32), arr(self.sr_cols, np.int32)
        p.sr_nnz, p.sr_rows, p.sr_cols = len(sr), _ptr(sr), _ptr(sc)
        lr, lc = arr(self.sl_rows, np.int32), arr(self.sl_cols, np.int32)
        p.sl_nnz, p.sl_rows, p.sl_cols = len(lr), _ptr(lr), _ptr(lc)
        if self.coords is not None and np.asarray(self.coords).size != 2 * int(self.n):
            raise ContractViolation("nested_dissection: coordinate count mismatch")
        p.coords = _ptr(arr(self.coords, np.float64)) if self.coords is not None else None
        groups = [np.asarray(g, np.int32) for g in self.atomic_groups]
        gptr = arr(np.cumsum([0] + [len(g) for g in groups]), np.int32)
        gd = arr(np.concatenate(groups) if groups else np.zeros(0, np.int32), np.int32)
        p.n_groups, p.group_ptr, p.group_dofs = len(groups), _ptr(gptr), _ptr(gd)
        p.max_leaf = int(self.max_leaf)
        if self.tree_parent is not None:
            tp = arr(self.tree_parent, np.int32)
            td = [np.asarray(d, np.int32) for d in self.tree_dofs]
            tptr = arr(np.cumsum([0] + [len(d) for d in td]), np.int32)
            tdd = arr(np.concatenate(td) if td else np.zeros(0, np.int32), np.int32)
            p.n_tree_clusters, p.tree_parent, p.tree_ptr, p.tree_dofs = len(tp), _ptr(tp), _ptr(tptr), _ptr(tdd)
        return p, keep


@dataclass
class SeparatorTree:
    """partition.hpp:19-68 view of a plan's tree."""

    parent: np.ndarray
    level: np.ndarray
    dofs: list
    fold_order: np.ndarray

    @property
    def num_clusters(self) -> int:
        return len(self.parent)

    @property
    def root(self) -> int:
        return int(np.nonzero(self.parent == -1)[0][0])

    @property
    def levels(self) -> int:
        return int(self.level.max())

    def ancestors(self, c: int) -> list:
        out = []
        p = int(self.parent[c])
        while p != -1:
            out.append(p)
            p = int(self.parent[p])
        return out

    def to_dict(self) -> dict:
        return {
            "levels": self.levels,
            "num_dofs": int(sum(len(d) for d in self.dofs)),
            "clusters": [
                {"id": i, "level": int(self.level[i]), "parent": int(self.parent[i]), "dofs": [int(x) for x in self.dofs[i]]}
                for i in range(self.num_clusters)
            ],
        }


@dataclass
class PlanInfo:
    n_dofs: int
    n_clusters: int
    levels: int
    root: int
    max_block: int
    arena_bytes_per_energy: int
    ref_fold_mul: int
    ref_fold_inv: int
    ref_gless_mul: int
    ref_gless_inv: int
    exec_cmul: float
    exec_inv_cmul: float
    n_ops: int
    n_gemm_tasks: int
    n_gemm_tiles: int
    n_inv_tasks: int
    needed_cmul: float = 0.0
    n_real_clusters: int = 0

    @property
    def needed_flops(self) -> float:
        """The needed-only work per energy counted as complex throughout (8 m n k, 8 m^3)."""
        return 8.0 * self.needed_cmul

    @property
    def ref_ledger_flops(self) -> float:
        """Real FP64 flops per energy under the reference ledger (8 x cmul)."""
        return 8.0 * (self.ref_fold_mul + self.ref_fold_inv + self.ref_gless_mul + self.ref_gless_inv)

    @property
    def exec_flops(self) -> float:
        """Real FP64 flops per energy the GPU executes (needed-only)."""
        return 8.0 * self.exec_cmul


class HscPlan:
    """Host plan: tree + symbolic structure + schedule (built once)."""

    def __init__(self, problem: Problem):
        self.problem = problem
        p, keep = problem.c_struct()
        h = C.c_void_p()
        st = _Status()
        _lib.negf_plan_create(C.byref(p), C.byref(h), C.byref(st))
        del keep
        _raise(st)
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:  # None during interpreter teardown
            _lib.negf_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def info(self) -> PlanInfo:
        i = _PlanInfo()
        _lib.negf_plan_info_get(self._h, C.byref(i))
        return PlanInfo(*[getattr(i, f[0]) for f in _PlanInfo._fields_ if f[0] != "pad_"])

    def tree(self) -> SeparatorTree:
        info = self.info()
        nc, n = info.n_clusters, info.n_dofs
        parent = np.zeros(nc, np.int32)
        level = np.zeros(nc, np.int32)
        ptr = np.zeros(nc + 1, np.int32)
        dofs = np.zeros(n, np.int32)
        fo = np.zeros(max(nc - 1, 1), np.int32)
        _lib.negf_plan_tree(self._h, _ptr(parent), _ptr(level), _ptr(ptr), _ptr(dofs), _ptr(fo))
        return SeparatorTree(parent, level, [dofs[ptr[c] : ptr[c + 1]].copy() for c in range(nc)], fo[: nc - 1])

    def gemm_tasks(self) -> dict:
        """Per grouped-GEMM task: m, n, summed k, phase, level (schedule introspection)."""
        t = self.info().n_gemm_tasks
        out = {k: np.zeros(t, np.int64 if k == "k" else np.int32) for k in ("m", "n", "k", "phase", "level")}
        _lib.negf_plan_gemm_tasks(self._h, _ptr(out["m"]), _ptr(out["n"]), _ptr(out["k"]), _ptr(out["phase"]),
                                  _ptr(out["level"]))
        return out

    def gemm_tiles(self) -> dict:
        """CTA tiles of the grouped-GEMM launches: task, m0, n0, arrangement,
        mirrored (the tile also writes its transpose: symmetric tasks)."""
        t = self.info().n_gemm_tiles
        out = {k: np.zeros(t, np.int32) for k in ("task", "m0", "n0", "arr", "mirrored")}
        _lib.negf_plan_gemm_tiles(self._h, *(_ptr(out[k]) for k in ("task", "m0", "n0", "arr", "mirrored")))
        return out

    def ops(self) -> dict:
        """The replayed op list: kind, phase, level, begin, count, cmul per op."""
        t = self.info().n_ops
        out = {k: np.zeros(t, np.int32) for k in ("kind", "phase", "level", "begin", "count")}
        out["cmul"] = np.zeros(t, np.float64)
        _lib.negf_plan_ops(self._h, *(_ptr(out[k]) for k in ("kind", "phase", "level", "begin", "count", "cmul")))
        return out

    def fill_sets(self) -> list:
        nc = self.info().n_clusters
        ptr = np.zeros(nc + 1, np.int32)
        _lib.negf_plan_fill(self._h, _ptr(ptr), None)
        ids = np.zeros(max(int(ptr[-1]), 1), np.int32)
        _lib.negf_plan_fill(self._h, _ptr(ptr), _ptr(ids))
        return [ids[ptr[c] : ptr[c + 1]].tolist() for c in range(nc)]


class RgfPlan(HscPlan):
    """Layered recursive Green's function plan (rgf_gr + rgf_gless,
    rgf.cpp:181-380) over the problem's layers (or ``layers``): the
    independent second GPU path and the paper's comparison baseline.  Solved
    by the same ``HscGpuSolver``; errors as layered_from_coo (rgf.cpp:69-150):
    ContractViolation for a bad layer map, PartitionViolation for entries
    coupling non-adjacent layers."""

    def __init__(self, problem: Problem, layers=None):
        self.problem = problem
        layers = problem.layers if layers is None else layers
        if layers is None or len(layers) == 0:
            raise ContractViolation("layer map is empty")
        ptr = np.zeros(len(layers) + 1, np.int32)
        ptr[1:] = np.cumsum([len(x) for x in layers])
        dofs = np.ascontiguousarray(np.concatenate([np.asarray(x, np.int32) for x in layers]), np.int32)
        p, keep = problem.c_struct()
        h = C.c_void_p()
        st = _Status()
        _lib.negf_rgf_plan_create(C.byref(p), len(layers), _ptr(ptr), _ptr(dofs), C.byref(h), C.byref(st))
        del keep
        _raise(st)
        self._h = h

    def tree(self):
        raise ContractViolation("an RGF plan has layers, not a separator tree")

    def fill_sets(self):
        raise ContractViolation("an RGF plan has layers, not fill sets")


def nested_dissection(n: int, edges: np.ndarray, atomic_groups=(), max_leaf: int = 64, coords=None) -> SeparatorTree:
    """nested_dissection (partition.hpp:84-87) on an explicit edge list."""
    e = np.asarray(edges, np.int32).reshape(-1, 2)
    rows = np.concatenate([e[:, 0], e[:, 1]])
    cols = np.concatenate([e[:, 1], e[:, 0]])
    prob = Problem(n=n, h_rows=rows, h_cols=cols, h_vals=np.ones(len(rows), np.complex128),
                   coords=coords, atomic_groups=atomic_groups, max_leaf=max_leaf)
    return HscPlan(prob).tree()


class HscGpuSolver:
    """One GPU's arena + schedule (negf_gpu_create) and its batched solves."""

    def __init__(self, plan: HscPlan, device: int = 0, max_energy_batch: int = 0):
        self.plan = plan
        self.n = plan.info().n_dofs
        self.sr_nnz = len(plan.problem.sr_rows)
        self.sl_nnz = len(plan.problem.sl_rows)
        h = C.c_void_p()
        st = _Status()
        _lib.negf_gpu_create(plan.handle, int(device), int(max_energy_batch), C.byref(h), C.byref(st))
        _raise(st)
        self._h = h
        self.device = device

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.negf_gpu_destroy(h)
            self._h = None

    @property
    def capacity(self) -> int:
        return _lib.negf_gpu_batch_capacity(self._h)

    @property
    def last_launches(self) -> int:
        return int(_lib.negf_gpu_last_launches(self._h))

    def solve(self, energies, weights, sigma_r, sigma_lesser, first_energy_index: int = 0,
              want_diagonals: bool = True, out_gr=None, out_gless=None):
        """Host arrays in, host arrays out (diag G^r, diag G^< per dof)."""
        E = np.ascontiguousarray(energies, np.float64)
        W = np.ascontiguousarray(weights, np.float64)
        m = len(E)
        sr = np.ascontiguousarray(sigma_r, np.complex128).reshape(m, self.sr_nnz) if self.sr_nnz else None
        sl = np.ascontiguousarray(sigma_lesser, np.complex128).reshape(m, self.sl_nnz) if self.sl_nnz else None
        gr = gl = None
        if want_diagonals:
            gr = out_gr if out_gr is not None else np.empty((m, self.n), np.complex128)
            gl = out_gless if out_gless is not None else np.empty((m, self.n), np.complex128)
        st = _Status()
        _lib.negf_gpu_solve_batch(self._h, m, _ptr(E), _ptr(W), _ptr(sr), _ptr(sl), int(first_energy_index),
                                  _ptr(gr), _ptr(gl), C.byref(st))
        _raise(st)
        return gr, gl

    def solve_device(self, energies, weights, sigma_r, sigma_lesser, first_energy_index: int = 0,
                     out_gr=None, out_gless=None, sync: bool = True) -> None:
        """torch CUDA tensors in/out (inputs already resident in HBM)."""
        dp = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        st = _Status()
        _lib.negf_gpu_solve_batch_device(self._h, int(energies.numel()), dp(energies), dp(weights),
                                         dp(sigma_r), dp(sigma_lesser), int(first_energy_index),
                                         dp(out_gr), dp(out_gless), int(bool(sync)), C.byref(st))
        _raise(st)

    def check(self) -> None:
        st = _Status()
        _lib.negf_gpu_check(self._h, C.byref(st))
        _raise(st)

    def density(self, reset: bool = False) -> np.ndarray:
        """(1/2pi) sum_k w_k Im G^<_jj(E_k) over everything solved so far."""
        out = np.empty(self.n, np.float64)
        st = _Status()
        _lib.negf_gpu_density(self._h, _ptr(out), int(bool(reset)), C.byref(st))
        _raise(st)
        return out

    @property
    def stream_ptr(self) -> int:
        return int(_lib.negf_gpu_stream(self._h) or 0)

    @property
    def density_ptr(self) -> int:
        """Device address of the unscaled density accumulator (n float64)."""
        return int(_lib.negf_gpu_density_device(self._h) or 0)

    def set_residual_check(self, raise_error: bool) -> None:
        """True (default): ResidualTooLarge like electron_density; False: record only."""
        _lib.negf_gpu_set_residual_check(self._h, int(bool(raise_error)))
        self._residual_check = bool(raise_error)

    @property
    def residual_check(self) -> bool:
        return getattr(self, "_residual_check", True)

    def residual_violation(self, reset: bool = False):
        """(energy_index, dof) of the lowest entry with |Re G^<_jj| > 1e-8
        |G^<_jj| recorded since the last reset (whatever the check mode), or
        None -- electron_density's guard order (observables.cpp:79-84)."""
        e, d = C.c_int32(-1), C.c_int32(-1)
        hit = _lib.negf_gpu_residual_violation(self._h, C.byref(e), C.byref(d), int(bool(reset)))
        return (int(e.value), int(d.value)) if hit else None

    @property
    def max_real_residual(self) -> float:
        """Largest |Re G^<_jj| / |G^<_jj| seen (DensityMap::max_real_residual)."""
        return float(_lib.negf_gpu_max_real_residual(self._h))

    def profile(self, enable: bool = True) -> None:
        """Per-kernel CUDA-event timing of subsequent solves (on the solver's stream)."""
        _lib.negf_gpu_profile(self._h, int(bool(enable)))

    def profile_read(self, reset: bool = False) -> dict:
        arr = (_KStat * len(KSTAT_NAMES))()
        _lib.negf_gpu_profile_read(self._h, C.cast(arr, C.c_void_p), int(bool(reset)))
        return {k: {"ms": arr[i].ms, "cmul": arr[i].cmul, "launches": arr[i].launches}
                for i, k in enumerate(KSTAT_NAMES)}

    def profile_ops(self, reset: bool = False) -> np.ndarray:
        """Per plan op (HscPlan.ops order): summed CUDA-event ms of the profiled solves."""
        out = np.zeros(max(self.plan.info().n_ops, 1), np.float64)
        _lib.negf_gpu_profile_ops(self._h, _ptr(out), int(bool(reset)))
        return out[: self.plan.info().n_ops]

    def nccl_init(self, unique_id: bytes, nranks: int, rank: int) -> None:
        buf = C.create_string_buffer(bytes(unique_id), 128)
        st = _Status()
        _lib.negf_gpu_nccl_init(self._h, buf, int(nranks), int(rank), C.byref(st))
        _raise(st)

    def allreduce_density(self, ordered: bool = True) -> None:
        """Sum the density partials over the NCCL communicator's ranks;
        ``ordered`` (default): all-gather + rank-ordered sum, bit-reproducible
        for any rank count."""
        _lib.negf_gpu_set_ordered_reduce(self._h, int(bool(ordered)))
        st = _Status()
        _lib.negf_gpu_allreduce_density(self._h, C.byref(st))
        _raise(st)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = _Status()
    _lib.negf_nccl_unique_id(buf, C.byref(st))
    _raise(st)
    return buf.raw


def trapezoid_weights(energies) -> np.ndarray:
    """make_energy_grid (observables.cpp:14-32)."""
    e = np.asarray(energies, np.float64)
    if len(e) == 0:
        raise ConfigError("energy grid must not be empty")
    if np.any(np.diff(e) <= 0):
        raise ConfigError("energy grid must be strictly increasing")
    if len(e) == 1:
        return np.ones(1)
    w = np.empty_like(e)
    w[0] = 0.5 * (e[1] - e[0])
    w[1:-1] = 0.5 * (e[2:] - e[:-2])
    w[-1] = 0.5 * (e[-1] - e[-2])
    return w


# ---------------------------------------------------------------------------
# contact self-energies on the GPU (include/negf_gpu.h)
# ---------------------------------------------------------------------------
class _ContactDesc(C.Structure):
    _fields_ = [
        ("w", C.c_int),
        ("d_sigma", C.c_void_p),
        ("ld", C.c_int64),
        ("sr_off", C.c_int64),
        ("sl_off", C.c_int64),
        ("mu_ev", C.c_double),
    ]


class SurfaceLead:
    """surface_self_energy (device.cpp:195-251) on the GPU, batched over
    energies: one dense semi-infinite lead with onsite block ``h00`` and the
    coupling ``h01`` from a lead cell to the next one away from the device
    (attach_contacts, device.cpp:284-303, builds these from the device's
    boundary layers).  ``criterion="decay"`` switches to the Sancho-Rubio
    convention of ``devices.sancho_rubio`` (config 3's lead)."""

    CRITERIA = {"fixed-point": 0, "decay": 1}

    def __init__(self, h00: np.ndarray, h01: np.ndarray, eta: float, device: int = 0,
                 max_energy_batch: int = 0, criterion: str = "fixed-point", tol: float = 1e-12):
        h00 = np.ascontiguousarray(h00, np.complex128)
        h01 = np.ascontiguousarray(h01, np.complex128)
        w = h00.shape[0]
        if h00.shape != (w, w):
            raise ContractViolation("surface_self_energy: h00 must be square")
        if h01.shape != (w, w):
            raise ContractViolation("surface_self_energy: h01 must match h00's shape")
        self.w = w
        self._h = C.c_void_p()
        st = _Status()
        if criterion not in self.CRITERIA:
            raise ContractViolation(f"unknown lead criterion {criterion!r}")
        _lib.negf_lead_create(int(device), w, _ptr(h00), _ptr(h01), float(eta), self.CRITERIA[criterion],
                              float(tol), int(max_energy_batch), C.byref(self._h), C.byref(st))
        _raise(st)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.negf_lead_destroy(self._h)
            self._h = None

    def sigma(self, energies, first_energy_index: int = 0) -> np.ndarray:
        """Host energies -> Sigma^r blocks (nE, w, w)."""
        e = np.ascontiguousarray(np.atleast_1d(energies), np.float64)
        out = np.empty((len(e), self.w, self.w), np.complex128)
        st = _Status()
        _lib.negf_lead_sigma(self._h, len(e), _ptr(e), int(first_energy_index), _ptr(out), C.byref(st))
        _raise(st)
        return out

    def sigma_device(self, energies, out, ld: int | None = None, first_energy_index: int = 0) -> None:
        """torch CUDA tensors: energies (nE,) float64 -> out (complex128, energy k
        at element k*ld)."""
        ld = self.w * self.w if ld is None else int(ld)
        st = _Status()
        _lib.negf_lead_sigma_device(self._h, int(energies.numel()), energies.data_ptr(), int(first_energy_index),
                                    out.data_ptr(), ld, C.byref(st))
        _raise(st)

    def last_sweeps(self, n: int) -> np.ndarray:
        """Converging sweep index per energy of the last call."""
        out = np.zeros(n, np.int32)
        _lib.negf_lead_last_sweeps(self._h, _ptr(out))
        return out

    @property
    def last_launches(self) -> int:
        return int(_lib.negf_lead_last_launches(self._h))


def lead_modes_sigma_device(w: int, t: float, eta: float, energies, out, ld: int | None = None,
                            stream: int = 0) -> None:
    """Analytic transverse-mode Sigma^r of a uniform hard-wall 2-D lead
    (devices.analytic_lead_sigma) for torch CUDA energies -> out."""
    ld = w * w if ld is None else int(ld)
    st = _Status()
    _lib.negf_lead_modes_sigma_device(int(w), float(t), float(eta), int(energies.numel()), energies.data_ptr(),
                                      out.data_ptr(), ld, C.c_void_p(stream or None), C.byref(st))
    _raise(st)


def contacts_fill_device(energies, kT: float, contacts, sigma_r, sigma_lesser, phonon_gamma=None,
                         ph_sr_off: int = -1, ph_sl_off: int = -1, mu_phonon: float = 0.0, stream: int = 0) -> None:
    """lesser_self_energy (device.cpp:322-366) + pattern placement on the GPU.

    ``contacts``: sequence of dicts {w, sigma (torch complex tensor), ld,
    sr_off, sl_off, mu}; ``sigma_r``/``sigma_lesser``: (nE, nnz) complex128
    torch tensors (rows = energies)."""
    descs = (_ContactDesc * max(1, len(contacts)))()
    for k, c in enumerate(contacts):
        descs[k] = _ContactDesc(int(c["w"]), c["sigma"].data_ptr(), int(c.get("ld", c["w"] * c["w"])),
                                int(c.get("sr_off", -1)), int(c.get("sl_off", -1)), float(c["mu"]))
    n_ph = 0 if phonon_gamma is None else int(phonon_gamma.numel())
    st = _Status()
    _lib.negf_contacts_fill_device(int(energies.numel()), energies.data_ptr(), float(kT), len(contacts), descs, n_ph,
                                   None if phonon_gamma is None else phonon_gamma.data_ptr(), int(ph_sr_off),
                                   int(ph_sl_off), float(mu_phonon),
                                   None if sigma_r is None else sigma_r.data_ptr(),
                                   0 if sigma_r is None else int(sigma_r.shape[-1]),
                                   None if sigma_lesser is None else sigma_lesser.data_ptr(),
                                   0 if sigma_lesser is None else int(sigma_lesser.shape[-1]),
                                   C.c_void_p(stream or None), C.byref(st))
    _raise(st)


# ---------------------------------------------------------------------------
# output path (include/negf_gpu.h)
# ---------------------------------------------------------------------------
def format_double(v: float) -> str:
    """format_double (run.cpp:276-281): general format, 17 significant digits."""
    buf = C.create_string_buffer(64)
    n = _lib.negf_format_double(float(v), buf, 64)
    return buf.value[:n].decode()


def write_solve_csv(out_dir: str, nx: int, ny: int, energies, density, gr_diag=None) -> None:
    """cmd_solve's density.csv / ldos.csv / line_density.csv (run.cpp:284-326);
    ``density`` already scaled (density_scale), dof j = y*nx + x."""
    e = np.ascontiguousarray(energies, np.float64)
    d = np.ascontiguousarray(density, np.float64)
    g = None if gr_diag is None else np.ascontiguousarray(gr_diag, np.complex128)
    st = _Status()
    _lib.negf_write_solve_csv(out_dir.encode(), int(nx), int(ny), len(e), _ptr(e), _ptr(d), _ptr(g), C.byref(st))
    _raise(st)


class ShardWriter:
    """Binary per-shard writer of per-energy diag G^r / G^< (negf_shard_writer_*)."""

    def __init__(self, path: str, n_dofs: int, rank: int = 0, world: int = 1, gr: bool = True, gless: bool = True):
        self.n = n_dofs
        self.what = (1 if gr else 0) | (2 if gless else 0)
        self._h = C.c_void_p()
        st = _Status()
        _lib.negf_shard_writer_open(path.encode(), int(n_dofs), int(rank), int(world), self.what,
                                    C.byref(self._h), C.byref(st))
        _raise(st)

    def append(self, energies, first_energy_index: int, gr=None, gless=None) -> None:
        e = np.ascontiguousarray(energies, np.float64)
        g1 = None if gr is None else np.ascontiguousarray(gr, np.complex128)
        g2 = None if gless is None else np.ascontiguousarray(gless, np.complex128)
        st = _Status()
        _lib.negf_shard_writer_append(self._h, len(e), int(first_energy_index), _ptr(e), _ptr(g1), _ptr(g2),
                                      C.byref(st))
        _raise(st)

    def append_device(self, energies, first_energy_index: int, gr=None, gless=None, stream: int = 0) -> None:
        """``gr``/``gless``: torch CUDA complex128 tensors (nE, n); host energies."""
        e = np.ascontiguousarray(energies, np.float64)
        st = _Status()
        _lib.negf_shard_writer_append_device(self._h, len(e), int(first_energy_index), _ptr(e),
                                             None if gr is None else gr.data_ptr(),
                                             None if gless is None else gless.data_ptr(),
                                             C.c_void_p(stream or None), C.byref(st))
        _raise(st)

    def close(self) -> None:
        if self._h:
            st = _Status()
            _lib.negf_shard_writer_close(self._h, C.byref(st))
            self._h = None
            _raise(st)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                self.close()
            except NegfError:
                pass


def read_shard(path: str) -> dict:
    """Reads a NEGFSHD1 shard: energy_index[k], energy[k], gr[k, n], gless[k, n]."""
    import struct

    with open(path, "rb") as f:
        buf = f.read()
    if buf[:8] != b"NEGFSHD1":
        raise ContractViolation(f"{path}: not a shard file")
    ver, n, rank, world, what, _ = struct.unpack_from("<6i", buf, 8)
    (count,) = struct.unpack_from("<q", buf, 32)
    rec = 16 + (16 * n if what & 1 else 0) + (16 * n if what & 2 else 0)
    if len(buf) != 64 + rec * count:
        raise ContractViolation(f"{path}: truncated shard ({len(buf)} bytes for {count} records)")
    raw = np.frombuffer(buf, np.uint8, rec * count, 64).reshape(count, rec)
    out = {"n_dofs": n, "rank": rank, "world": world,
           "energy_index": raw[:, :4].copy().view(np.int32).ravel(),
           "energies": raw[:, 8:16].copy().view(np.float64).ravel()}
    at = 16
    if what & 1:
        out["gr"] = raw[:, at:at + 16 * n].copy().view(np.complex128)
        at += 16 * n
    if what & 2:
        out["gless"] = raw[:, at:at + 16 * n].copy().view(np.complex128)
    return out
