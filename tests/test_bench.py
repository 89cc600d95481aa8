"""CPU: bench.py's launcher contract — `--gpus N` re-launches itself under
torch.distributed.run (N ranks over gloo here) and rank 0 prints one JSON
line with n_gpus == N; a WORLD_SIZE that disagrees with --gpus fails loudly.
Exercised through the reference arm (the only arm without a GPU)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          timeout=600, env=e, cwd=ROOT)


def test_gpus_two_relaunches_two_ranks():
    r = _run(["--gpus", "2", "--impl", "reference", "--config", "si8", "--steps", "1", "--warmup", "0"])
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == 2 and line["impl"] == "reference"
    assert line["cpu_baseline"]["kind"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["extrapolated"]["fixed_pieces_measured_once_s"] >= 0


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "2", "--impl", "reference", "--config", "si8", "--steps", "1", "--warmup", "0"],
             env={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE" in (r.stdout + r.stderr)
