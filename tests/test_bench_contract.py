"""bench.py's launch contract on the host (no GPU needed): a GPU count that does not
match the process group fails loudly instead of silently benchmarking a different
configuration (`--gpus 2` on one process), and both arms describe the same
workload with the same config dict."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_gpu_count_mismatch_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--no-cpu-baseline"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0
    assert "needs 2 ranks" in (r.stderr + r.stdout)


@pytest.mark.parametrize("world", [1, 2, 8])
def test_workload_and_config_match_between_arms(world):
    import argparse

    import bench
    args = argparse.Namespace(workload=None, graph_steps=64)
    name, label, make = bench.workload_for(args, world)
    assert name == ("cfg4" if world == 1 else "cfg5_16m")
    assert ("1,000,000 el" in label) if world == 1 else ("16,003,008 el" in label)

    class P:  # the config dict needs only the sizes
        num_elements, num_nodes = 123, 45
    a = bench.bench_config(name, label, P, world, 64)
    b = bench.bench_config(name, label, P, world, 64)
    assert a == b and a["parallelism"] == ("single" if world == 1 else f"rcb{world}")
