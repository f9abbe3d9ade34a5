"""Where does the Woodbury leaf diagonal (K_LEAFDIAG, opt-in form) lose
accuracy?  GPU with and without the form on the 12-cell CNT at chosen
energies, against the dense truth; per leaf: max error of diag G^r of each
path and the leaf's shape (test infrastructure)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1305_1070_b200 import devices, negf  # noqa: E402

w = devices.config3(n_cells=12)
p = w.problem
n = p.n
idx = np.array([int(x) for x in sys.argv[1].split(",")])
sr, sl = w.self_energies(idx)
res = {}
for tag, forms in (("plain", None), ("wood", "symdiag_g,symdiag_p,sparse,hull,woodbury")):
    if forms:
        os.environ["NEGF_PLAN_FORMS"] = forms
    else:
        os.environ.pop("NEGF_PLAN_FORMS", None)
    plan = negf.HscPlan(p)
    s = negf.HscGpuSolver(plan)
    s.set_residual_check(False)
    res[tag] = s.solve(w.energies[idx], w.weights[idx], sr, sl)
    if forms:
        ops = plan.ops()
        t = plan.tree()
        fill = plan.fill_sets()
os.environ.pop("NEGF_PLAN_FORMS", None)
for q, k in enumerate(idx):
    A = np.zeros((n, n), complex)
    np.add.at(A, (p.h_rows, p.h_cols), -p.h_vals)
    A[np.arange(n), np.arange(n)] += w.energies[k]
    np.add.at(A, (p.sr_rows, p.sr_cols), -sr[q])
    G = np.linalg.inv(A)
    d = np.diag(G)
    sc = np.abs(d).max()
    print(f"E[{k}] = {w.energies[k]:.4f}: plain {np.abs(res['plain'][0][q] - d).max() / sc:.2e}  "
          f"wood {np.abs(res['wood'][0][q] - d).max() / sc:.2e}")
    rows = []
    for x in range(t.num_clusters):
        if t.level[x] != 1:
            continue
        dx = np.asarray(t.dofs[x])
        ew = np.abs(res["wood"][0][q][dx] - d[dx]).max() / sc
        ep = np.abs(res["plain"][0][q][dx] - d[dx]).max() / sc
        rows.append((ew, ep, x, len(dx), len(fill[x])))
    rows.sort(reverse=True)
    for ew, ep, x, m, ns in rows[:6]:
        print(f"   leaf {x}: m={m} |S|={ns} S={fill[x]} levels={[int(t.level[j]) for j in fill[x]]}  "
              f"wood {ew:.2e} plain {ep:.2e}")
