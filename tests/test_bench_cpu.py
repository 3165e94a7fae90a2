"""bench.py contract checks that need no GPU: the reference arm (the CPU oracle
timed as it stands) prints one JSON line with the contract's keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_reference(*extra):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--cpu-sample-n", "16", *extra],
                         capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_reference()
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == "trotter_steps_per_s" and d["n_gpus"] == 1
    assert d["value"] > 0 and d["unit"] == "steps/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["n"] == 30


def test_reference_arm_multi_gpu_units():
    """--gpus 4 (rank 0 of a torchrun job): n = 32, whole-job shard-steps/s."""
    one = run_reference()
    four = run_reference("--gpus", "4")
    assert four["config"]["n"] == 32 and four["n_gpus"] == 4
    assert four["unit"].startswith("shard-steps/s")
    # 4 shards of 2^30 amplitudes per step at 4x the per-step cost: same order as N = 1
    assert 0.2 < four["value"] / one["value"] < 5.0
