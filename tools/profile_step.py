"""Short workload for ncu captures: a few exact 256^3 complex128 steps (3 mumode launches each)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2103_01691_b200 import _device as dv  # noqa: E402
from paper_2103_01691_b200 import dist  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
u, cache = bench.build_inputs()
dev = torch.device("cuda", 0)
runner = dist.LocalStepper(dv.to_device(u, np.complex128, dev), cache.device_exps((np.complex128,) * 3, dev))
for _ in range(steps):
    runner.step()
torch.cuda.synchronize()
print("ok", steps)
