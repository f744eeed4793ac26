"""bench.py's launcher contract on CPU: `--gpus N` self-launches N ranks through
torch.distributed.run (rank 0 alone runs the reference arm and prints one JSON line), the
reference arm runs the full workload it names (no scaling) on every host core."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_self_launches_two_ranks():
    p = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--impl", "reference",
                        "--extent", "64", "--steps", "2", "--warmup", "1"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["config"]["n"] == 64
    assert d["steps"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["cores"] == (os.cpu_count() or 1)
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_workload_grids():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.workload_config(1024) == 205 and bench.workload_degree(1024) == 5
    assert bench.workload_config(2048) == 683 and bench.workload_degree(2048) == 3
