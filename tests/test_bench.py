"""bench.py plumbing on CPU: the N-rank launcher (gloo) and the reference
arm's isolation from the product library."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


def test_gpus_flag_launches_n_ranks():
    """`bench.py --gpus 2` without torchrun re-executes itself under
    torch.distributed.run with one rank per GPU; rank 0 prints the line."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = _last_json(r.stdout)
    assert line["n_gpus"] == 2 and line["backend"] == "gloo"
    assert line["max_over_ranks"] == 2.0  # max over ranks of (rank + 1)


def test_reference_arm_does_not_map_product_library(tmp_path):
    """The reference arm shares only the input generator with our arm: making
    the workload and the reference's problem file must not load
    libnegf_b200.so (the product's C ABI library is mapped lazily)."""
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "import bench\n"
        "w = bench.make_workload(1, 256)\n"
        "bench.ref_problem_file(w, np.arange(2), %r)\n"
        "maps = open('/proc/self/maps').read()\n"
        "print('MAPPED' if 'libnegf_b200' in maps else 'CLEAN')\n"
    ) % (ROOT, str(tmp_path / "p.bin"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().splitlines()[-1] == "CLEAN"
