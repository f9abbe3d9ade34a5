"""GPU parity: the C-ABI path against the reference's own outputs (golden
fixtures written by the reference build, tests/golden/make_golden.py).

Bar (BASELINE.json north_star): diag G^r and diag G^< within 1e-10 relative
(max over entries, per energy) in FP64."""
import numpy as np
import pytest

from paper_1305_1070_b200 import negf
from tests.helpers import golden_names, load_golden, rel_err

TOL = 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("name", golden_names())
def test_golden_hsc_parity(name, cuda_ok):
    rp, prob, hsc, dense = load_golden(name)
    plan = negf.HscPlan(prob)
    solver = negf.HscGpuSolver(plan)
    sr, sl = rp.values(np.arange(len(rp.energies)))
    gr, gl = solver.solve(rp.energies, rp.weights, sr, sl)
    assert solver.last_launches > 0
    for e in range(len(rp.energies)):
        assert rel_err(gr[e], hsc.gr[e]) <= TOL, (name, e, "G^r", rel_err(gr[e], hsc.gr[e]))
        assert rel_err(gl[e], hsc.gless[e]) <= TOL, (name, e, "G^<", rel_err(gl[e], hsc.gless[e]))
        if dense is not None:
            assert rel_err(gr[e], dense.gr[e]) <= 1e-9
            assert rel_err(gl[e], dense.gless[e]) <= 1e-9
    # density = (1/2pi) sum_k w_k Im G^<  (observables.cpp:71-91)
    want = (rp.weights[:, None] * hsc.gless.imag).sum(0) / (2 * np.pi)
    got = solver.density()
    assert np.abs(got - want).max() <= 1e-10 * max(np.abs(want).max(), 1e-300)
