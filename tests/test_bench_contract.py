"""bench.py contract on the CPU: the reference arm (the oracle, the one leg bench.py may
run without a GPU) prints one JSON line with the contract's keys, and the ranks other
than 0 exit without work."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env=None, *args):
    env = dict(os.environ)
    env.update(extra_env or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "C1",
                        "--steps", "1", "--warmup", "3", "--ref-seconds", "0.3", *args],
                       capture_output=True, text=True, env=env, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr
    return r.stdout.strip()


def test_reference_arm_json_line():
    out = _run()
    lines = [l for l in out.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == "literal-evals/sec" and d["value"] > 0
    assert d["config"]["workload"] == "C1" and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and "sample" in cb
    assert cb["single_core"]["value"] > 0
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_quietly():
    out = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, "--gpus", "2")
    assert out == ""


def test_batch_sharding_and_lanes_rules():
    """Host rules of the bench: weak scaling keeps the per-GPU batch (C2: 4096 per GPU),
    C5's global batch of 65536 is sharded (strong); the lanes the engine forms (galois.h
    galois_engine_set_lanes: ceil(b_loc / lanes) rounded up to 1024 members)."""
    sys.path.insert(0, ROOT)
    import bench
    assert bench.batch_of("C2", 1) == (4096, 4096, "weak")
    assert bench.batch_of("C2", 8) == (32768, 4096, "weak")
    assert bench.batch_of("C5", 1) == (65536, 65536, "strong")
    assert bench.batch_of("C5", 8) == (65536, 8192, "strong")
    assert bench.default_lanes(4096) == 4 and bench.default_lanes(1024) == 1
    assert bench.default_lanes(16384) == 2 and bench.default_lanes(65536) == 2
    assert bench.effective_lanes(4096, 4, 1) == 4
    assert bench.effective_lanes(3000, 4, 1) == 3          # 1024 + 1024 + 952
    assert bench.effective_lanes(16384, 4, 1) == 4
    assert bench.effective_lanes(2100, 2, 1) == 2          # 2048 + 52
    assert bench.effective_lanes(4096, 4, 8) == 1          # no lanes with an NCCL communicator
    assert bench.effective_lanes(1024, 4, 1) == 1
    assert bench.effective_lanes(8192, 1, 1) == 1
