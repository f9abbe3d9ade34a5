"""Map an ncu launch list of one config-2 batch onto the plan's ops.

    python tools/launch_map.py ops  out.json          # plan op list (GEMM rows per warp arrangement)
    python tools/launch_map.py batch [repeats]        # one 256-point batch (run under ncu)
    python tools/launch_map.py map launches.csv ops.json   # per (phase, level) GEMM time and TF/s
    python tools/launch_map.py traffic dram.csv ops.json   # k_gemm DRAM bytes vs algorithmic bytes
    python tools/launch_map.py shares launches.csv         # kernel shares of any ncu launch list

traffic: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_gemm
         --clock-control none --csv --log-file dram.csv python tools/launch_map.py batch

ncu: ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file L.csv \\
         python tools/launch_map.py batch
"""
import collections
import csv
import json
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402

NE = 256


def op_list(path):
    from paper_1305_1070_b200 import devices, negf
    w = devices.config2(n_energies=2)
    plan = negf.HscPlan(w.problem)
    ops, tl, tk = plan.ops(), plan.gemm_tiles(), plan.gemm_tasks()
    tms, tns = np.array([32, 16, 64, 16]), np.array([32, 64, 16, 16])
    rows = []
    for i in range(len(ops["kind"])):
        k, b, c = int(ops["kind"][i]), int(ops["begin"][i]), int(ops["count"][i])
        base = dict(op=i, kind=k, phase=int(ops["phase"][i]), level=int(ops["level"][i]), cmul=float(ops["cmul"][i]))
        if k != 1:
            rows.append(dict(base, count=c))
            continue
        arrs = tl["arr"][b:b + c]
        for a in dict.fromkeys(arrs.tolist()):  # launch order = plan order
            sel = np.arange(b, b + c)[arrs == a]
            t = tl["task"][sel]
            lm = np.minimum(tms[a], tk["m"][t] - tl["m0"][sel])
            ln = np.minimum(tns[a], tk["n"][t] - tl["n0"][sel])
            ut = np.unique(t)  # algorithmic bytes: every operand read once, C read + written once
            ab = float((16.0 * (tk["m"][ut] * tk["k"][ut] + tk["k"][ut] * tk["n"][ut]
                                + 2.0 * tk["m"][ut] * tk["n"][ut])).sum())
            rows.append(dict(base, arr=int(a), tiles=int(len(sel)), flops=float((8.0 * lm * ln * tk["k"][t]).sum()),
                             alg_bytes=ab))
    json.dump(rows, open(path, "w"))


def batch(repeats):
    import torch
    from paper_1305_1070_b200 import devices, negf
    w = devices.config2(n_energies=NE)
    solver = negf.HscGpuSolver(negf.HscPlan(w.problem), device=0, max_energy_batch=NE)
    solver.set_residual_check(False)
    sr, sl = w.self_energies(np.arange(NE))
    dev = torch.device("cuda", 0)
    args = [torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (w.energies, w.weights, sr, sl)]
    for _ in range(repeats):
        solver.solve_device(*args)
    torch.cuda.synchronize()


def map_launches(csv_path, ops_path):
    lines = [ln for ln in open(csv_path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h, rows = rows[0], rows[1:]
    i_n, i_v = h.index("Kernel Name"), h.index("Metric Value")
    launches = [(r[i_n], float(r[i_v]) / 1e6) for r in rows]
    gl = [x for x in launches if "k_gemm" in x[0]]
    g = [o for o in json.load(open(ops_path)) if o["kind"] == 1]
    assert len(gl) == len(g), (len(gl), len(g))
    tot, gt = sum(t for _, t in launches), sum(t for _, t in gl)
    print(f"# {len(launches)} launches, {tot:.2f} ms; k_gemm {len(gl)} launches, {gt:.2f} ms ({100 * gt / tot:.1f} %)")
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    for (_, t), o in zip(gl, g):
        agg[(o["phase"], o["level"])][0] += t
        agg[(o["phase"], o["level"])][1] += o["flops"] * NE
    print("# phase level    ms   TF/s(8mkn)  share-of-gemm")
    for k in sorted(agg):
        t, f = agg[k]
        print(f"  {k[0]:5d} {k[1]:5d} {t:7.2f} {f / t / 1e9:8.2f} {100 * t / gt:7.1f} %")
    byname = collections.defaultdict(lambda: [0, 0.0])
    for name, t in launches:
        key = name.split("(")[0].replace("(anonymous namespace)::", "").replace("negfb::", "")
        byname[key][0] += 1
        byname[key][1] += t
    print("# kernel, launches, total ms, share")
    for k, (n, t) in sorted(byname.items(), key=lambda x: -x[1][1]):
        print(f"  {k[-44:]:44s} {n:4d} {t:9.2f} ms {100 * t / tot:5.1f} %")


def traffic(csv_path, ops_path):
    """Per k_gemm launch: DRAM bytes (ncu) against the algorithmic bytes of its
    tasks (operands and C once per energy; a task split over two arrangement
    launches counts in both)."""
    lines = [ln for ln in open(csv_path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h, rows = rows[0], rows[1:]
    i_id, i_m, i_v = h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
    per = collections.defaultdict(dict)
    for r in rows:
        per[int(r[i_id])][r[i_m]] = float(r[i_v].replace(",", ""))
    ls = [per[k] for k in sorted(per)]
    g = [o for o in json.load(open(ops_path)) if o["kind"] == 1]
    assert len(ls) == len(g), (len(ls), len(g))
    tot_d = tot_a = tot_t = 0.0
    out = []
    for m, o in zip(ls, g):
        d = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        t = m["gpu__time_duration.sum"] * 1e-9
        a = o["alg_bytes"] * NE
        tot_d, tot_a, tot_t = tot_d + d, tot_a + a, tot_t + t
        out.append((t, d, a, o))
    print(f"# k_gemm: {len(out)} launches {tot_t * 1e3:.2f} ms, DRAM {tot_d / 1e9:.2f} GB, algorithmic "
          f"{tot_a / 1e9:.2f} GB ({tot_d / tot_a:.2f}x)")
    print("# top launches: ms, DRAM GB, algorithmic GB, ratio, phase, level, arr")
    for t, d, a, o in sorted(out, key=lambda x: -x[0])[:12]:
        print(f"  {t * 1e3:7.3f} {d / 1e9:7.2f} {a / 1e9:7.2f} {d / a:6.2f}  ph {o['phase']} lv {o['level']} arr {o['arr']}")


def shares(csv_path):
    """Kernel shares of an ncu launch list (any command, e.g. bench.py)."""
    lines = [ln for ln in open(csv_path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h, rows = rows[0], rows[1:]
    i_n, i_v = h.index("Kernel Name"), h.index("Metric Value")
    byname = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows:
        t = float(r[i_v].replace(",", "")) / 1e6
        key = r[i_n].split("(")[0].replace("(anonymous namespace)::", "").replace("negfb::", "")
        byname[key][0] += 1
        byname[key][1] += t
        tot += t
    print(f"# {len(rows)} launches, {tot:.2f} ms (ncu per-launch times: serialised, cold caches)")
    print("# kernel, launches, total ms, share")
    for k, (n, t) in sorted(byname.items(), key=lambda x: -x[1][1]):
        print(f"  {k[-52:]:52s} {n:5d} {t:9.2f} ms {100 * t / tot:5.1f} %")


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "shares":
        shares(sys.argv[2])
        sys.exit(0)
    if cmd == "ops":
        op_list(sys.argv[2])
    elif cmd == "batch":
        batch(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    elif cmd == "traffic":
        traffic(sys.argv[2], sys.argv[3])
    else:
        map_launches(sys.argv[2], sys.argv[3])
