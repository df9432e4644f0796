"""Small-state step timing (config 1 and neighbours): eager vs graph, per-launch device time.

Usage: python tools/small_probe.py [--ncu]  (with --ncu: 10 eager steps only, for the launch list)
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2103_01691_b200 as km  # noqa: E402
from paper_2103_01691_b200 import _device as dv, dist  # noqa: E402

DEV = torch.device("cuda", 0)


def stepper(n):
    rng = np.random.default_rng(0)
    u = np.asfortranarray(rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3))
    d2 = km.heat_factors(n, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    return dist.LocalStepper(dv.to_device(u, np.complex128, DEV), cache.device_exps((np.complex128,) * 3, DEV))


def graph_ms(st, steps=10, reps=50, paired=False):
    for _ in range(3):
        st.step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            if paired:
                st.run(steps)
            else:
                for _ in range(steps):
                    st.step()
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


if __name__ == "__main__":
    if "--ncu" in sys.argv:
        st = stepper(64)
        for _ in range(10):
            st.step()
        torch.cuda.synchronize()
        sys.exit(0)
    from paper_2103_01691_b200 import _native

    lib = _native.lib()
    for n in (32, 48, 64, 96, 128):
        res = {}
        for name, pol in (("fused planes", _native.POLICY_AUTO), ("per product", _native.POLICY_NO_PLANE_FUSION)):
            _native.check(lib.km_set_kernel_policy(pol))
            st = stepper(n)
            ms = graph_ms(st)
            flop = 8 * 3 * n**4 * 10
            per_launch = [round(x * 1e3, 2) for x in st.time_launches(50)]
            st2 = stepper(n)
            for _ in range(10):
                st2.step()
            res[name] = dv.to_host(st2.a)
            print(f"n={n} {name}: 10 steps {ms*1e3:.1f} us ({ms*100:.2f} us/step), {flop/ms/1e9:.2f} TFLOP/s; "
                  f"eager per-launch us {per_launch}", flush=True)
        a, b = res["fused planes"], res["per product"]
        print(f"   fused vs per-product after 10 steps: rel l2 {np.linalg.norm(a - b) / np.linalg.norm(b):.2e}")
        st = stepper(n)
        if st.paired_ok():
            ms = graph_ms(st, paired=True)
            st2 = stepper(n)
            st2.run(10)
            c = dv.to_host(st2.a)
            print(f"n={n} paired steps (km_steps_paired, {st.launches_for(10)} launches): 10 steps {ms*1e3:.1f} us "
                  f"({ms*100:.2f} us/step), {8 * 3 * n**4 * 10 / ms / 1e9:.2f} TFLOP/s; vs per-product rel l2 "
                  f"{np.linalg.norm(c - b) / np.linalg.norm(b):.2e}", flush=True)
    _native.check(lib.km_set_kernel_policy(_native.POLICY_AUTO))
