"""bench.py's multi-GPU launcher (CPU): `--gpus N` without a torchrun environment starts N ranks
through torch.distributed.run on 127.0.0.1; a WORLD_SIZE that disagrees with --gpus is refused."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _env():
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT", "LOCAL_WORLD_SIZE"):
        env.pop(k, None)
    return env


def test_launcher_starts_n_ranks():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "3", "--probe"], env=_env(),
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1, 2]
    assert all(d["world_size"] == 3 for d in lines)
    assert len({d["pid"] for d in lines}) == 3  # one process per rank


def test_launcher_refuses_mismatch():
    env = _env()
    env.update(WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--probe"], env=env,
                         capture_output=True, text=True, timeout=120)
    assert out.returncode == 2 and "refusing" in out.stderr


def test_single_gpu_runs_in_process():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--probe"], env=_env(), capture_output=True,
                         text=True, timeout=120)
    assert out.returncode == 0
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["world_size"] == 1 and d["rank"] == 0
