"""bench.py's launch contract on a CPU-only box (no GPU needed): --gpus N
is honoured -- re-launch under torch.distributed.run, loud failure when the
GPUs are not there or WORLD_SIZE disagrees -- and the reference arm runs on
rank 0 only under N ranks."""

import json
import os
import subprocess
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _run(args, env=None, timeout=300):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, env=e, capture_output=True, text=True,
                          timeout=timeout)


def test_gpus_more_than_visible_fails_loudly():
    import torch
    n = torch.cuda.device_count()
    p = _run(["--gpus", str(max(2, n + 1)), "--steps", "1", "--warmup", "0"])
    assert p.returncode != 0
    assert "requested but only" in p.stderr


def test_world_size_mismatch_fails():
    p = _run(["--gpus", "1", "--impl", "reference", "--steps", "1", "--warmup", "0"],
             env={"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert p.returncode != 0 and "WORLD_SIZE=2" in p.stderr


def test_reference_arm_under_two_ranks():
    """--gpus 2 without torchrun: re-launched as 2 ranks; rank 0 prints the
    one JSON line, rank 1 exits 0 without work."""
    p = _run(["--gpus", "2", "--impl", "reference", "--steps", "1", "--warmup", "0"], timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["config"]["workload"].startswith("1920x1080")
