"""Run under torchrun (any world size): the NCCL slab stepper against a single-GPU
reference computed on rank 0.  Exits non-zero on a parity failure.

    torchrun --nproc-per-node P --master-addr 127.0.0.1 --master-port 29511 tools/slab_check.py [n] [steps] [nccl|peer|gpe|tdpot]

nccl / peer: exact steps (SlabStepper / PeerSlabStepper) against LocalStepper;
gpe: SlabGpeStepper.run (config 5) against gpe_strang_run on one GPU;
tdpot: SlabTdpotStepper.run (config 4) against tdpot_strang_step on one GPU.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as tdist  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from paper_2103_01691_b200 import _device as dv, dist  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    exchange = sys.argv[3] if len(sys.argv) > 3 else "nccl"
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ngpu = torch.cuda.device_count()
    dev = torch.device("cuda", local % ngpu)
    torch.cuda.set_device(dev)
    tdist.init_process_group("nccl", device_id=dev)
    rank, world = tdist.get_rank(), tdist.get_world_size()
    if exchange == "gpe":
        from paper_2103_01691_b200.problems import weighted_vortex_state

        grids, lin_op, weights = km.gpe_setup(n)
        u = weighted_vortex_state(grids, weights)
        cache = km.prepare(lin_op, 0.1)
        st = dist.SlabGpeStepper.from_global(u, cache, weights, 0.1, dev)
        st.run(steps)
        want = km.gpe_strang_run(cache, weights, u, 0.1, steps)
    elif exchange == "tdpot":
        from paper_2103_01691_b200.hermite import physical_propagator
        from paper_2103_01691_b200.problems import schrodinger_initial_state

        b = km.hermite_basis(n)
        tau = 0.02
        p = physical_propagator(b, tau)
        cache = km.PropagatorCache(tau, (p, p, p))
        u = schrodinger_initial_state((b.nodes,) * 3)
        st = dist.SlabTdpotStepper.from_global(u, cache, b.nodes, dev)
        st.run(0.0, tau, steps)
        want = u
        for s_ in range(steps):
            want = km.tdpot_strang_step(cache, b.nodes, want, s_ * tau, tau)
    else:
        rng = np.random.default_rng(0)
        u = np.asfortranarray(rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3))
        d2 = km.heat_factors(n, 2).factors[0]
        cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
        cls = dist.PeerSlabStepper if exchange == "peer" else dist.SlabStepper
        st = cls.from_global(u, cache, dev)
        for _ in range(steps):
            st.step()
        ref = dist.LocalStepper(dv.to_device(u, np.complex128, dev), cache.device_exps((np.complex128,) * 3, dev))
        for _ in range(steps):
            ref.step()
        want = dv.to_host(ref.state)
    torch.cuda.synchronize()
    mine = dv.to_host(st.local_state())
    want_slab = st.plan.slab_a(want, rank) if st.layout == "A" else st.plan.slab_b(want, rank)
    err = float(np.linalg.norm((mine - want_slab).ravel()) / np.linalg.norm(want_slab.ravel()))
    errs = torch.tensor([err], device=dev)
    tdist.all_reduce(errs, op=tdist.ReduceOp.MAX)
    if rank == 0:
        print(f"slab_check exchange={exchange} world={world} n={n} steps={steps} layout={st.layout} "
              f"max_rel_l2={errs.item():.3e}")
    tdist.destroy_process_group()
    sys.exit(0 if errs.item() <= 1e-12 else 1)


if __name__ == "__main__":
    main()
