"""bench.py's launch contract: `--gpus N` runs N ranks and reports n_gpus = N.

The CPU test drives the reference arm (no GPU needed; rank 0 prints, the
other ranks exit 0); the GPU test drives our arm with N = 2 ranks sharing
the one GPU of the box over gloo (a functional check of the multi-rank path,
never a timing configuration).
"""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None, timeout=600):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], cwd=REPO,
                       env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_two_ranks_one_line():
    import oracle
    if oracle.reference_package() is None:
        pytest.skip("oracle/_ref not built")
    line = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
                 "--ref-frames", "1"])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["global_batch"] == 2 * line["config"]["frames_per_gpu_per_step"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_bench_config_is_shared_by_both_arms():
    sys.path.insert(0, REPO)
    import bench
    assert bench.bench_config(256, 1) == bench.bench_config(256, 1)
    assert bench.bench_config(256, 4)["global_batch"] == 1024


@pytest.mark.gpu
def test_bench_gpus_2_launches_two_ranks():
    line = _run(["--gpus", "2", "--steps", "2", "--warmup", "3", "--batch", "8", "--no-cpu"],
                {"SPX_BENCH_BACKEND": "gloo"})
    assert line["n_gpus"] == 2
    assert line["config"]["global_batch"] == 16
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["gpu_launches"] > 0


@pytest.mark.gpu
def test_bench_c5_row_strips_two_ranks():
    # C5 (16384^2) as two row strips, ranks sharing the GPU over gloo
    line = _run(["--workload", "c5", "--gpus", "2", "--steps", "1", "--warmup", "3", "--no-cpu"],
                {"SPX_BENCH_BACKEND": "gloo"}, timeout=900)
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["value"] > 0 and line["e2e"]["value"] > 0
