"""CPU: bench.py's multi-GPU launcher.  ``--gpus N`` without a torchrun
environment starts N ranks itself (torch.distributed.run on 127.0.0.1) and
rank 0 reports the real world size; here the ranks only rendezvous over gloo
(KMB200_BENCH_SELFTEST=1), which is what the launcher is responsible for."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

BENCH = os.path.join(ROOT, "bench.py")


def _run(args, extra_env=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["KMB200_BENCH_SELFTEST"] = "1"
    env.update(extra_env or {})
    out = subprocess.run([sys.executable, BENCH] + args, capture_output=True, text=True, timeout=300, env=env)
    return out


@pytest.mark.parametrize("impl", ["ours", "reference"])
def test_launcher_spawns_n_ranks(impl):
    out = _run(["--gpus", "2", "--impl", impl, "--steps", "1", "--warmup", "3"])
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 only
    assert lines[0]["n_gpus"] == 2 and lines[0]["ranks_seen"] == 2 and lines[0]["impl"] == impl


def test_world_size_mismatch_fails_loudly():
    out = _run(["--gpus", "4"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


def test_too_few_gpus_fails_loudly():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK",
                                                             "KMB200_BENCH_SELFTEST")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    out = subprocess.run([sys.executable, BENCH, "--gpus", "2"], capture_output=True, text=True, timeout=300,
                         env=env)
    assert out.returncode != 0 and "visible GPUs" in out.stderr
