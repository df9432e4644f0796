"""Rank 0 of the P-rank slab step (256^3 c128) on one GPU: serial vs two-half schedule.

    python tools/overlap_probe.py [n]

For P = 2, 4, 8 and both schedules (dist.SlabPlan.schedule), rank 0's products run
exactly as in a P-GPU job (same shapes, blocked layouts, derived E3 forms).  Three
numbers per case:

* compute: the products alone (no exchange), ms per step;
* emulated: each all-to-all replaced by a device-to-device copy of the same bytes
  on a side stream, ordered exactly as the NCCL calls are (side stream waits for
  the products that fill the half; the post products wait for the copy) — shows
  how much of the transfer the schedule hides when the transfer takes as long as
  an HBM copy;
* model: compute + the exposed part of an exchange at NVLink speed (the measured
  770 GB/s peer bandwidth), from the per-group times: serial exposes
  all of it; the two-half schedule hides half 0 under the half-1 products and
  half 1 under the first post group (half 0's share of the post products).

One GPU stands in for rank 0 only; no kernel waits on another rank's work.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from paper_2103_01691_b200 import dist  # noqa: E402

DEV = torch.device("cuda", 0)
PEAK = 37.14e12
NVLINK = 770e9  # B/s per direction, measured peer bandwidth


class CopyExchange:
    """Stand-in for NcclExchange: a D2D copy of the same bytes on a side stream."""

    def __init__(self):
        self.side = torch.cuda.Stream(DEV)

    def exchange_async(self, recv, send):
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(DEV))
        self.side.wait_event(ev)
        with torch.cuda.stream(self.side):
            recv.copy_(send)
            done = torch.cuda.Event()
            done.record(self.side)

        class W:
            def wait(self_inner):
                torch.cuda.current_stream(DEV).wait_event(done)
        return W()


def time_steps(st, reps=20, warm=4):
    for _ in range(warm):
        st.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        st.step()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def group_times(st, reps=20):
    """Mean ms of each pre / post group for the even and the odd step (no exchange)."""
    out = {}
    for layout in ("A", "B"):
        pre, post, size = st.plan.schedule(layout, st.overlap)
        st.layout = layout
        ts = []
        for groups in (pre, post):
            row = []
            for g in groups:
                if not g:
                    row.append(0.0)
                    continue
                st._exec(g)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    st._exec(g)
                e1.record()
                e1.synchronize()
                row.append(e0.elapsed_time(e1) / reps)
            ts.append(row)
        out[layout] = (ts, size)
    st.layout = "A"
    return out


def model(gt, overlap, es=16):
    """Per-step ms (average of even and odd) with the exchange at NVLink speed."""
    tot = 0.0
    for layout in ("A", "B"):
        (pre, post), size = gt[layout]
        x = size * es * (1 - 1 / P) / NVLINK * 1e3  # ms per exchange half (or whole, serial)
        comp = sum(pre) + sum(post)
        if not overlap:
            tot += comp + x
            continue
        # half 0 moves during the half-1 pre products; half 1 during post group 0
        exposed = max(0.0, x - pre[1]) + max(0.0, x - post[0])
        tot += comp + exposed
    return tot / 2


n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
rng = np.random.default_rng(0)
u = np.asfortranarray(rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3))
d2 = km.heat_factors(n, 2).factors[0]
cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
flop = 8 * 3 * n**4
for P in (2, 4, 8):
    for overlap in (False, True):
        g = dist.VirtualSlabGroup(u, cache, DEV, P, overlap=overlap)
        r0 = g.ranks[0]
        if overlap and not r0.overlap:
            print(f"P={P}: two-half schedule not applicable")
            continue
        r0.comm = None
        ms_comp = time_steps(r0)
        gt = group_times(r0)
        r0.comm = CopyExchange()
        ms_emul = time_steps(r0)
        r0.comm = None
        ms_model = model(gt, overlap)
        name = "two-half" if overlap else "serial"
        print(f"P={P} {name:8s}: compute {ms_comp:.3f} ms/step ({flop / P / (ms_comp * 1e-3) / PEAK:.3f} of peak), "
              f"emulated exchange {ms_emul:.3f}, NVLink model {ms_model:.3f} "
              f"-> {flop / P / (ms_model * 1e-3) / PEAK:.3f} of peak; groups even {gt['A'][0]} odd {gt['B'][0]}",
              flush=True)
        del g, r0
        torch.cuda.empty_cache()
