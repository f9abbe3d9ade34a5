"""CPU: the host plan behind the C ABI (tree, symbolic fold, ledger, errors)
and the C ABI surface itself.  No GPU needed: plan creation is host-only."""
import json
import os
import re

import numpy as np
import pytest

from paper_1305_1070_b200 import negf
from tests.helpers import GOLDEN, golden_names, load_golden

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name", golden_names())
def test_tree_and_ledger_match_reference(name):
    """Bit-exact nested dissection (partition.cpp:159-326) and the exact lean
    ledger of hsc_fold + hsc_gless (dense.hpp:69-82), per golden problem."""
    rp, prob, hsc, _ = load_golden(name)
    plan = negf.HscPlan(prob)
    t = plan.tree()
    assert t.num_clusters == len(hsc.parent)
    assert np.array_equal(t.parent, hsc.parent)
    assert np.array_equal(t.level, hsc.level)
    for a, b in zip(t.dofs, hsc.dofs):
        assert np.array_equal(a, b)
    i = plan.info()
    ne = len(rp.energies)
    assert (i.ref_fold_mul + i.ref_gless_mul) * ne == hsc.mul_ops
    assert (i.ref_fold_inv + i.ref_gless_inv) * ne == hsc.inv_ops
    assert i.exec_cmul <= i.ref_fold_mul + i.ref_fold_inv + i.ref_gless_mul  # needed-only never exceeds


def test_cli_partition_tree_json():
    """proj/cli_test_tmp/partition/tree.json: the 3x8 superlattice, max_leaf 2,
    diagonal contacts (no atomic groups), device coordinates."""
    rp, prob, _, _ = load_golden("superlattice_3x8_diag")
    want = json.load(open(os.path.join(GOLDEN, "cli_partition_tree.json")))
    got = negf.HscPlan(prob).tree().to_dict()
    assert got == want


def _chain_problem(edges, n, **kw):
    e = np.asarray(edges, np.int32).reshape(-1, 2)
    rows = np.concatenate([e[:, 0], e[:, 1], np.arange(n)])
    cols = np.concatenate([e[:, 1], e[:, 0], np.arange(n)])
    vals = np.concatenate([-np.ones(2 * len(e)), 4.0 * np.ones(n)]).astype(complex)
    return negf.Problem(n=n, h_rows=rows, h_cols=cols, h_vals=vals, **kw)


def test_nested_dissection_errors():
    edges = [(i, i + 1) for i in range(9)]
    with pytest.raises(negf.ConfigError):
        negf.HscPlan(_chain_problem(edges, 10, max_leaf=0))
    with pytest.raises(negf.ConfigError):
        negf.HscPlan(_chain_problem(edges, 10, atomic_groups=[[0, 1], [1, 2]]))
    with pytest.raises(negf.ConfigError):
        negf.HscPlan(_chain_problem(edges, 10, atomic_groups=[[0, 11]]))
    with pytest.raises(negf.ContractViolation):
        negf.HscPlan(_chain_problem(edges, 10, coords=np.zeros((3, 2))))


def test_explicit_tree_errors():
    edges = [(0, 2), (1, 2)]
    with pytest.raises(negf.ContractViolation):  # two roots
        negf.HscPlan(_chain_problem(edges, 3, tree_parent=[-1, -1, 0], tree_dofs=[[0], [1], [2]]))
    with pytest.raises(negf.ContractViolation):  # dof missing
        negf.HscPlan(_chain_problem(edges, 3, tree_parent=[1, -1], tree_dofs=[[0], [1]]))
    with pytest.raises(negf.PartitionViolation):  # sibling leaves coupled (rule 1)
        negf.HscPlan(_chain_problem([(0, 1)], 3, tree_parent=[2, 2, -1], tree_dofs=[[0], [1], [2]]))
    with pytest.raises(negf.ContractViolation):  # Sigma^< joining two clusters
        negf.HscPlan(_chain_problem(edges, 3, sl_rows=[0], sl_cols=[2], tree_parent=[2, 2, -1],
                                    tree_dofs=[[0], [1], [2]]))


def test_grandparent_only_psi_list():
    """A leaf coupled only to its grandparent folds straight past its parent:
    exactly one Psi entry (test_hsc.cpp:727-790)."""
    prob = _chain_problem([(0, 4), (1, 5), (2, 4), (3, 5)], 6, tree_parent=[1, 2, -1],
                          tree_dofs=[[0, 1], [2, 3], [4, 5]])
    fills = negf.HscPlan(prob).fill_sets()
    assert fills[0] == [2]
    assert fills[1] == [2]


def test_fill_is_transitive():
    """Schur fill (hsc.cpp:501-511): a leaf coupled to parent and grandparent
    makes the parent's S contain the grandparent."""
    prob = _chain_problem([(0, 1), (0, 2)], 3, tree_parent=[1, 2, -1], tree_dofs=[[0], [1], [2]])
    fills = negf.HscPlan(prob).fill_sets()
    assert fills == [[1, 2], [2], []]


def test_disconnected_graph_gets_empty_root():
    """Disconnected inputs: an artificial empty root separator (partition.hpp:73-75)."""
    coords = np.array([[0.0, 0.0], [1.0, 0.0], [10.0, 0.0], [11.0, 0.0]])
    prob = _chain_problem([(0, 1), (2, 3)], 4, max_leaf=2, coords=coords)
    t = negf.HscPlan(prob).tree()
    assert len(t.dofs[t.root]) == 0
    assert sorted(np.concatenate(t.dofs).tolist()) == [0, 1, 2, 3]


def test_abi_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "negf_gpu.h")).read()
    declared = set(re.findall(r"\b(negf_[a-z_0-9]+)\s*\(", header))
    assert declared, "no declarations found"
    lib = negf._lib
    for sym in sorted(declared):
        assert hasattr(lib, sym), sym
    assert declared <= set(negf.ABI_SYMBOLS) | {"negf_plan_info_get"}


def test_gpu_handle_fails_loudly_without_device():
    """No silent CPU fallback: without a GPU the device handle cannot be made."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    rp, prob, _, _ = load_golden("syn_5x6_s24")
    with pytest.raises(negf.CudaError):
        negf.HscGpuSolver(negf.HscPlan(prob))


def _check_tiles_cover_exactly(plan):
    tk = plan.gemm_tasks()
    tl = plan.gemm_tiles()
    tm = np.array([32, 16, 64, 16])  # arr 3: warp tiles (one warp per 16 x 16 block)
    tn = np.array([32, 64, 16, 16])
    cover = [np.zeros((int(m), int(n)), np.int32) for m, n in zip(tk["m"], tk["n"])]
    for t, m0, n0, a, mir in zip(tl["task"], tl["m0"], tl["n0"], tl["arr"], tl["mirrored"]):
        c = cover[t]
        c[m0 : m0 + tm[a], n0 : n0 + tn[a]] += 1  # numpy clips at the task edge
        if mir:  # a symmetric task's strictly-upper tile writes its transpose too
            assert c.shape[0] == c.shape[1] and n0 >= m0 + tm[a]
            c[n0 : n0 + tn[a], m0 : m0 + tm[a]] += 1
    for t, c in enumerate(cover):
        assert c.min() == 1 and c.max() == 1, f"task {t} ({c.shape}) covered {c.min()}..{c.max()} times"


@pytest.mark.parametrize("name", golden_names())
def test_gemm_tiles_cover_every_task_exactly_once(name):
    """Mixed 32x32 / 16x64 / 64x16 / warp 16x16 tiling: every output entry of every grouped
    GEMM task is computed by exactly one CTA tile (accumulating tasks would
    double-add otherwise)."""
    _, prob, _, _ = load_golden(name)
    _check_tiles_cover_exactly(negf.HscPlan(prob))


def test_gemm_tiles_cover_config2_exactly_once():
    from paper_1305_1070_b200 import devices

    _check_tiles_cover_exactly(negf.HscPlan(devices.config2(n_energies=2).problem))


def test_sparse_leaf_paths_are_exercised(monkeypatch):
    """The sparse-leaf ops (K_SPSI 8, K_SSCHUR 9) replace dense products only
    where the plan proves them exact; the golden problems the GPU parity tests
    run must cover each of them and the dense fallback (seeded / fuzzed
    leaves).  The Woodbury leaf diagonals (K_LEAFDIAG 10) are off by default
    (they lose accuracy at ill-conditioned energies) and, opted
    in with NEGF_PLAN_FORMS, cover every unseeded leaf of config 2."""
    from paper_1305_1070_b200 import devices

    seen = {8: 0, 9: 0, 10: 0}
    dense_leaf_fallback = False
    for name in golden_names():
        _, prob, _, _ = load_golden(name)
        o = negf.HscPlan(prob).ops()
        for k in seen:
            seen[k] += int(o["count"][o["kind"] == k].sum())
        dense_leaf_fallback |= bool((o["kind"] == 8).any() and not (o["kind"] == 10).any())
    assert seen[8] > 0 and seen[9] > 0 and seen[10] == 0, seen
    assert dense_leaf_fallback
    assert not (negf.HscPlan(devices.config2(n_energies=2).problem).ops()["kind"] == 10).any()
    monkeypatch.setenv("NEGF_PLAN_FORMS", WOODBURY_FORMS)
    plan = negf.HscPlan(devices.config2(n_energies=2).problem)
    o = plan.ops()
    t = plan.tree()
    leaves = int((np.asarray(t.level) == 1).sum())
    assert o["count"][o["kind"] == 10].tolist() == [leaves - 2, leaves - 2]  # all but the two contact leaves


WOODBURY_FORMS = "symdiag_g,symdiag_p,sparse,hull,woodbury"


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5, "4ref"])
def test_tree_matches_reference_at_baseline_size(cfg, tmp_path):
    """Bit-exact nested dissection at the BASELINE sizes (2k .. 1M dofs):
    the plan's tree against the reference's own build_tree + nested_dissection
    (run.cpp:123-133, partition.cpp:271-326; oracle/_ref ref_driver --solver
    tree), cluster for cluster: parent, level and the dof list."""
    from oracle import refio
    from paper_1305_1070_b200 import devices
    from tests.helpers import workload_ref_problem

    if not refio.ref_available():
        pytest.skip("oracle/_ref not built")
    # "4ref": config 4 in the reference builders' coordinate orientation (the
    # 2557-dof root block)
    w = devices.config4(ref_orientation=True) if cfg == "4ref" else devices.CONFIGS[cfg]()
    rp, _, _ = workload_ref_problem(w, [0])
    path = str(tmp_path / "p.bin")
    refio.write_problem(rp, path)
    r = refio.run_reference(path, str(tmp_path / "o.bin"), solver="tree")
    assert r.status == 0, r.message
    t = negf.HscPlan(w.problem).tree()
    assert t.num_clusters == len(r.parent)
    assert np.array_equal(t.parent, r.parent)
    assert np.array_equal(t.level, r.level)
    for a, b in zip(t.dofs, r.dofs):
        assert np.array_equal(a, b)
