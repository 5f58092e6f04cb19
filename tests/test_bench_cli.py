"""bench.py's multi-rank plumbing on CPU: `--gpus 2` outside torchrun
re-launches itself with two ranks (gloo here), splits the mode-3 slabs,
reduces once and prints one JSON line from rank 0 (the driver's
`bench.py --gpus N` must reach the multi-rank path)."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_bench_gpus2_spawns_two_ranks_on_cpu():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--cpu-smoke", "--steps", "2",
                        "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout          # rank 0 only
    d = json.loads(lines[0])
    assert d["impl"] == "cpu-smoke" and d["n_gpus"] == 2 and d["steps"] == 2
    assert d["config"]["parallelism"] == "mode-3 slabs x2"
    assert d["check_max_rel_err"] <= 1e-12


def test_bench_reference_arm_other_ranks_exit_quietly():
    # under torchrun only rank 0 of the reference arm runs and prints
    import os
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2"],
                       capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert r.returncode == 0 and not r.stdout.strip()
