"""bench.py's launch contract on CPU (no GPU needed): `--gpus N` without a launcher re-execs
under torch.distributed.run only when N devices exist (else exit 2 with a message), and a
launcher whose WORLD_SIZE disagrees with --gpus is refused (exit 2) -- VERDICT r01 item 1."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env_extra):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "ICL_BENCH_ONE_GPU")}
    env.update(env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], env=env, capture_output=True,
                          text=True, timeout=300)


def test_world_size_mismatch_is_refused():
    r = run(["--gpus", "4"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr


def test_more_gpus_than_devices_is_refused():
    torch = pytest.importorskip("torch")
    if torch.cuda.device_count() >= 8:
        pytest.skip("this host has 8 GPUs")
    r = run(["--gpus", "8"], {})
    assert r.returncode == 2 and "CUDA device" in r.stderr
