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
    # the contract: the reference arm runs on OUR arm's config, key for key;
    # what a bounded step really runs is stated beside it
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.gpu_config(d["config"]["mode"], 1)
    assert d["sample_run"]["copy_bytes_per_tenant"] < d["config"]["copy_bytes"]


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


def test_bench_gpus_2_dry_run_spawns_two_ranks():
    """`bench.py --gpus 2` with no WORLD_SIZE launches two
    ranks itself (torch.distributed.run, 127.0.0.1).  The dry run goes through
    the bench's rank plumbing on CPU (gloo; one virtual arena per rank: the
    partition manager and the launcher's validation of every C2 / C5 item, no
    kernels) and must print exactly one JSON line, from rank 0, with n_gpus 2,
    the max-over-ranks makespan and the stats summed over both ranks (C5:
    3 x 671,089 x launches x 2 violations)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run", "--c5-launches", "20"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"] is True
    assert d["makespan_ms_max"] == 11.0                         # rank 1's 11 ms: max over ranks
    assert d["items_validated_per_rank"] == 24                  # 16 C2 + 8 C5 items
    c5 = d["multi_tenant_c5"]
    assert c5["violations_expected"] == 3 * 671089 * 20 * 2
    assert c5["violations_allreduced"] == c5["violations_expected"] and c5["violations_exact"]
    assert d["stats_allreduced"]["launches"] == 2 * 8 * 20


def test_bench_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "1", "--dry-run"], cwd=ROOT, capture_output=True,
                       text=True, timeout=120, env=env)
    assert r.returncode != 0
    assert "WORLD_SIZE=2" in r.stderr and r.stdout.strip() == ""
