"""bench.py's driver contract on the CPU: --gpus N spawns N ranks itself,
a world size that disagrees with --gpus is refused, and the reference arm
prints the GPU arm's config (the driver compares the two lines)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _run(args, env=None, timeout=240):
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(env or {})
    return subprocess.run([sys.executable, BENCH] + args, capture_output=True, text=True, timeout=timeout, env=e,
                          cwd=ROOT)


def _last_json(out: str) -> dict:
    return json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])


def test_gpus_flag_spawns_that_many_ranks():
    p = _run(["--gpus", "2", "--launch-probe"])
    assert p.returncode == 0, p.stderr[-2000:]
    d = _last_json(p.stdout)
    assert d["n_gpus"] == 2 and d["gpus_flag"] == 2
    assert sorted(r["rank"] for r in d["ranks"]) == [0, 1]
    assert sorted(r["local_rank"] for r in d["ranks"]) == [0, 1]
    assert len({r["pid"] for r in d["ranks"]}) == 2


def test_single_gpu_runs_in_process():
    p = _run(["--launch-probe"])
    assert p.returncode == 0
    d = _last_json(p.stdout)
    assert d["n_gpus"] == 1 and len(d["ranks"]) == 1


def test_world_size_must_match_gpus_flag():
    p = _run(["--gpus", "2", "--launch-probe"], env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert p.returncode == 2
    assert "world size 1 != --gpus 2" in p.stdout


def test_reference_arm_prints_the_gpu_arm_config():
    sys.path.insert(0, ROOT)
    import bench
    p = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"], timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    d = _last_json(p.stdout)
    ns = type("A", (), {"tokens": 8192, "zero1": False})()
    assert d["impl"] == "reference" and d["config"] == bench.layer_config(ns, 1)
    assert d["unit"] == "TFLOP/s" and d["higher_is_better"] is True and d["metric"] == bench.METRIC
    assert d["cpu_baseline"]["kind"] == "port" and "tokens=1024" in d["cpu_baseline"]["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
