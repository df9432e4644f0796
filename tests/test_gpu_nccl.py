"""GPU: the NCCL path of the slab stepper, launched like bench.py's multi-GPU run
(torchrun, one process per GPU, 127.0.0.1 rendezvous).  With one visible GPU the
world size is 1 (the all-to-all is a self-exchange); on a multi-GPU box set
KMB_SLAB_WORLD to the GPU count."""

import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n,steps,exchange", [(64, 3, "nccl"), (256, 2, "nccl"), (64, 3, "peer"), (256, 2, "peer"),
                                              (64, 3, "gpe"), (128, 2, "gpe"), (64, 3, "tdpot"), (128, 2, "tdpot")])
def test_slab_stepper_over_nccl(n, steps, exchange):
    import torch

    world = int(os.environ.get("KMB_SLAB_WORLD", str(min(torch.cuda.device_count(), 8))))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tools", "slab_check.py"), str(n), str(steps), exchange]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "max_rel_l2" in r.stdout
