"""The bench's reference arm (the CPU oracle, the task's tier framing) runs on
a GPU-less host and prints one JSON line with the contract's keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_json_line_survives_stdout_noise():
    """The GPU arm routes fd 1 to stderr (NCCL prints its version line to
    stdout at communicator setup) and writes its one JSON line to the saved
    stdout: Python prints, C-level writes and child processes all land on
    stderr, the JSON line alone on stdout."""
    code = ("import os, bench; bench.quiet_stdout(); print('python noise'); os.write(1, b'fd noise\\n'); "
            "os.system('echo child noise'); bench.emit({'metric': 'm', 'value': 1.0}); print('late noise')")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.splitlines() == ['{"metric": "m", "value": 1.0}']
    for noise in ("python noise", "fd noise", "child noise", "late noise"):
        assert noise in r.stderr
