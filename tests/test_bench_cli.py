"""bench.py's contract pieces that need no GPU: the reference arm's JSON line
(the CPU oracle on a bounded sample, all host threads) and the launcher's
refusal to run N ranks on fewer than N GPUs."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=300):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, env=env, cwd=ROOT)


def test_reference_arm_json_line():
    r = _run("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["n_gpus"] == 1 and line["steps"] == 1 and line["warmup"] == 3
    assert line["unit"] == "Mkeys/s" and line["higher_is_better"] is True and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == (os.cpu_count() or 1) and cb["value"] == line["value"]
    assert "2^22" in line["config"]["reference_sample"] and "nproc" in cb["host"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_launcher_refuses_more_ranks_than_gpus():
    import torch
    if torch.cuda.device_count() >= 2:
        return  # (a multi-GPU host: the launcher would run)
    r = _run("--gpus", "2", "--steps", "1")
    assert r.returncode == 2
    assert "one rank per GPU" in r.stderr
