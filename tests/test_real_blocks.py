"""The `real` plan form (plan.cpp mark_real_operands): clusters the retarded
self-energy never reaches -- directly or through a descendant's Schur fill --
are eliminated in real arithmetic.  CPU: which clusters qualify and how the
executed-work ledger counts them.  GPU: the outputs do not change by a bit."""
import os

import numpy as np
import pytest

from paper_1305_1070_b200 import devices, negf

BASE_FORMS = "symdiag_g,symdiag_p,sparse,hull,compact"


def _with_forms(forms, fn):
    old = os.environ.get("NEGF_PLAN_FORMS")
    os.environ["NEGF_PLAN_FORMS"] = forms
    try:
        return fn()
    finally:
        if old is None:
            del os.environ["NEGF_PLAN_FORMS"]
        else:
            os.environ["NEGF_PLAN_FORMS"] = old


def test_real_clusters_are_those_off_the_contact_paths():
    """Config 2 (real effective-mass H, dense contacts on the first and last
    layer): everything except the contact clusters and their ancestors."""
    w = devices.config2(n_energies=2)
    plan = negf.HscPlan(w.problem)
    info = plan.info()
    t = plan.tree()
    touched = np.zeros(info.n_dofs, bool)
    touched[np.asarray(w.problem.sr_rows)] = True
    touched[np.asarray(w.problem.sr_cols)] = True
    cplx = np.array([touched[d].any() for d in t.dofs])
    for c in np.nonzero(cplx)[0]:
        for a in t.ancestors(int(c)):
            cplx[a] = True
    assert info.n_real_clusters == int((~cplx).sum()) > 0.9 * info.n_clusters
    # executed work counts a real operand at 1/2, real x real and real inverses at 1/4
    assert 0.25 * info.needed_cmul < info.exec_cmul < 0.75 * info.needed_cmul
    off = _with_forms(BASE_FORMS, lambda: negf.HscPlan(w.problem).info())
    assert off.n_real_clusters == 0 and off.exec_cmul == off.needed_cmul == info.needed_cmul


def test_no_real_clusters_when_sigma_reaches_every_dof_or_h_is_complex():
    w = devices.config2(n_energies=2, ny=20, nx=40, complex_energy=True)  # -i eta on every dof through Sigma^r
    i = negf.HscPlan(w.problem).info()
    assert i.n_real_clusters == 0 and i.exec_cmul == i.needed_cmul
    w = devices.config2(n_energies=2, ny=20, nx=40)
    h = np.asarray(w.problem.h_vals).copy()
    k = int(np.nonzero(np.asarray(w.problem.h_rows) != np.asarray(w.problem.h_cols))[0][0])
    r, c = int(w.problem.h_rows[k]), int(w.problem.h_cols[k])
    rows, cols = np.asarray(w.problem.h_rows), np.asarray(w.problem.h_cols)
    h[(rows == r) & (cols == c)] += 1e-3j  # one Hermitian pair of complex hoppings
    h[(rows == c) & (cols == r)] -= 1e-3j
    w.problem.h_vals = h
    i = negf.HscPlan(w.problem).info()
    assert i.n_real_clusters == 0 and i.exec_cmul == i.needed_cmul


@pytest.mark.gpu
def test_real_form_is_bit_identical(cuda_ok):
    """Skipped products are exact zeros: diag G^r, diag G^< and the density of
    a 120 x 40 superlattice (16 energies) equal the complex evaluation's."""
    w = devices.config2(n_energies=16, ny=40, nx=120)
    idx = np.arange(len(w.energies))
    sr, sl = w.self_energies(idx)

    def solve():
        plan = negf.HscPlan(w.problem)
        s = negf.HscGpuSolver(plan)
        s.set_residual_check(False)
        gr, gl = s.solve(w.energies, w.weights, sr, sl)
        return gr, gl, s.density(), plan.info()

    a = solve()
    b = _with_forms(BASE_FORMS, solve)
    assert a[3].n_real_clusters > 0 and b[3].n_real_clusters == 0
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
