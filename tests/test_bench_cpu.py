"""bench.py contract checks that need no GPU: the reference arm (the CPU oracle
timed as it stands) prints one JSON line with the contract's keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_reference(*extra):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", *extra],
                         capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0])


def test_reference_arm_line():
    """At a small n (--qubits 16, the checked-in instance); the default is the
    bench's n = 30 (one oracle step ~11 s on 16 cores, too long for the CPU suite)."""
    d = run_reference("--qubits", "16")
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == "trotter_steps_per_s" and d["n_gpus"] == 1
    assert d["value"] > 0 and d["unit"] == "steps/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["n"] == 16
    assert len(d["cpu_baseline"]["step_s"]) == 2 and d["cpu_baseline"]["cpu"]
    # one oracle step of the schedule per bench step: ms_per_step is their mean
    assert abs(d["ms_per_step"] / 1e3 - sum(d["cpu_baseline"]["step_s"]) / 2) < 1e-9


def test_reference_arm_multi_gpu_units():
    """--gpus 4 (rank 0 of a torchrun job): whole-job shard-steps/s, i.e. the
    state's Trotter steps/s times 2^(n - 30) shards of 2^30 amplitudes."""
    four = run_reference("--gpus", "4", "--qubits", "18")
    assert four["config"]["n"] == 18 and four["n_gpus"] == 4
    assert four["unit"].startswith("shard-steps/s")
    assert abs(four["value"] - 2.0 ** (18 - 30) / (four["ms_per_step"] / 1e3)) < 1e-9 * four["value"]
