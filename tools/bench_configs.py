"""Measure every BASELINE.json config on one B200 against the CPU reference algorithm.

    python tools/bench_configs.py [--cpu-budget S] [--out profiles/rNN_configs.json]

Each config: device time (CUDA events, device-resident state, warmed up),
achieved TFLOP/s at the SURVEY §8(d) flop convention, parity against the CPU
oracle on the same inputs, and the oracle's own time on the host cores
(bounded sample).  The headline config (256^3 exact step) is bench.py's job.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from oracle import kronmode_oracle as orc  # noqa: E402
from paper_2103_01691_b200 import _device as dv  # noqa: E402
from paper_2103_01691_b200 import dist  # noqa: E402
from paper_2103_01691_b200.hermite import physical_propagator  # noqa: E402
from paper_2103_01691_b200.problems import schrodinger_initial_state, weighted_vortex_state  # noqa: E402

DEV = torch.device("cuda", 0)


def dev_time(fn, reps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def cpu_time(fn, budget, max_reps=5):
    fn()  # warm-up
    ts = []
    t_end = time.perf_counter() + budget
    while len(ts) < max_reps:
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end:
            break
    return min(ts) * 1e3, len(ts)


def crand(rng, shape):
    return np.asfortranarray(rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


def schrod(n, tau=0.01):
    d2 = km.heat_factors(n, 2).factors[0]
    return km.prepare(km.KroneckerOp((1j * d2,) * 3), tau)


def config1(budget):
    n, steps = 64, 10
    u = crand(np.random.default_rng(0), (n,) * 3)
    cache = schrod(n)
    st = dist.LocalStepper(dv.to_device(u, np.complex128, DEV), cache.device_exps((np.complex128,) * 3, DEV))

    def ten():
        for _ in range(steps):
            st.step()

    ms = dev_time(ten, 20)
    # graph-captured variant: the 30 launches replayed as one graph
    st2 = dist.LocalStepper(dv.to_device(u, np.complex128, DEV), cache.device_exps((np.complex128,) * 3, DEV))
    for _ in range(3):
        st2.step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(steps):
                st2.step()
    torch.cuda.synchronize()
    ms_graph = dev_time(g.replay, 50)
    # LocalStepper.run(10): km_steps_paired, two steps per three fused launches, in a graph
    st3 = dist.LocalStepper(dv.to_device(u, np.complex128, DEV), cache.device_exps((np.complex128,) * 3, DEV))
    st3.run(2)
    torch.cuda.synchronize()
    g3 = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g3, stream=s):
            st3.run(steps)
    torch.cuda.synchronize()
    ms_paired = dev_time(g3.replay, 50)
    st4 = dist.LocalStepper(dv.to_device(u, np.complex128, DEV), cache.device_exps((np.complex128,) * 3, DEV))
    st4.run(steps)
    got = u
    for _ in range(steps):
        got = km.step(cache, got)
    want = u
    for _ in range(steps):
        want = orc.step(cache.exps, want)
    cpu_ms, k = cpu_time(lambda: [orc.step(cache.exps, u) for _ in range(steps)], budget)
    flop = 8 * 3 * n**4 * steps
    best = min(ms, ms_graph, ms_paired)
    return {"config": "1: 3D Schrodinger free 64^3 c128, 10 steps", "gpu_ms": ms, "gpu_ms_graph": ms_graph,
            "gpu_ms_paired_graph": ms_paired, "tflops": flop / (best * 1e-3) / 1e12, "cpu_ms": cpu_ms,
            "cpu_reps": k, "speedup": cpu_ms / best, "parity_rel_l2": orc.rel_l2(got, want),
            "parity_rel_l2_paired": orc.rel_l2(dv.to_host(st4.a), want)}


def config2(budget):
    n = 1024
    op = km.pipeflow_factors(n)
    cache = km.prepare(op, 4.0 / 8)
    rho, z = np.linspace(0.1, 5.0, n), np.linspace(0.0, 8.0, n)
    c0 = np.asfortranarray(np.exp(-8.0 * (rho - 2.55) ** 2)[:, None] * np.exp(-8.0 * (z - 1.5) ** 2)[None, :])
    st = dist.LocalStepper(dv.to_device(c0, np.float64, DEV), cache.device_exps((np.float64,) * 2, DEV))
    ms = dev_time(st.step, 50)
    cpu_ms, k = cpu_time(lambda: orc.step(cache.exps, c0), budget, 20)
    flop = 2 * 2 * n**3
    return {"config": "2: 2D pipe flow 1024^2 f64, one exact step", "gpu_ms": ms,
            "tflops": flop / (ms * 1e-3) / 1e12, "cpu_ms": cpu_ms, "cpu_reps": k, "speedup": cpu_ms / ms,
            "parity_rel_l2": orc.rel_l2(km.step(cache, c0), orc.step(cache.exps, c0))}


def config3(budget, k=256):
    b = km.hermite_basis(k)
    bases = (b,) * 3
    psi0 = schrodinger_initial_state((b.nodes,) * 3)
    op = km.KroneckerOp(tuple(km.hamiltonian_factor(b, v) for v in
                              (lambda x: np.cos(2 * np.pi * x), lambda x: 0.5 * x * x, lambda x: 0.5 * x * x)))
    cache = km.prepare(op, 1.0)
    p_dev = dv.to_device(psi0, np.complex128, DEV)

    def hkp():
        c = km.forward_transform(bases, p_dev)
        c = km.step(cache, c)
        return km.inverse_transform(bases, c)

    ms = dev_time(hkp, 10)
    got = dv.to_host(hkp())
    fwd_o = lambda: orc.forward_transform([b.phi] * 3, [b.mod_weights] * 3, psi0)  # noqa: E731

    def hkp_cpu():
        c = fwd_o()
        c = orc.step(cache.exps, c)
        return orc.inverse_transform([b.phi.T] * 3, c)

    want = hkp_cpu()
    cpu_ms, kk = cpu_time(hkp_cpu, budget, 3)
    flop = 4 * 3 * k**4 * 2 + 8 * 3 * k**4
    return {"config": "3: HKP 256^3 c128 forward + exact step + inverse", "gpu_ms": ms,
            "tflops": flop / (ms * 1e-3) / 1e12, "cpu_ms": cpu_ms, "cpu_reps": kk, "speedup": cpu_ms / ms,
            "parity_rel_l2": orc.rel_l2(got, want)}


def config4(budget, k=256):
    b = km.hermite_basis(k)
    tau = 0.02
    p = physical_propagator(b, tau)
    cache = km.PropagatorCache(tau, (p, p, p))
    psi = schrodinger_initial_state((b.nodes,) * 3)
    p_dev = dv.to_device(psi, np.complex128, DEV)
    ms = dev_time(lambda: km.tdpot_strang_step(cache, b.nodes, p_dev, 0.3, tau), 10)
    got = km.tdpot_strang_step(cache, b.nodes, psi, 0.3, tau)
    want = orc.tdpot_strang_step(cache.exps, b.nodes, psi, 0.3, tau)
    cpu_ms, kk = cpu_time(lambda: orc.tdpot_strang_step(cache.exps, b.nodes, psi, 0.3, tau), budget, 3)
    # the 8-rank slab schedule of the TD-potential step (SlabTdpotStepper: per-step fold of E3 on
    # every rank, fused pack/unpack, one exchange per step) run as 8 virtual ranks on this GPU;
    # per-rank time = the group's time / 8 (every rank's kernels run back to back here)
    grp = dist.VirtualSlabGroup(psi, cache, DEV, 8, kind="tdpot", x_nodes=b.nodes)
    tt = [0.0]

    def vstep():
        grp.step(t=tt[0], tau=tau)
        tt[0] += tau

    ms_virtual8 = dev_time(vstep, 5, warm=1)
    grp2 = dist.VirtualSlabGroup(psi, cache, DEV, 8, kind="tdpot", x_nodes=b.nodes)
    for s_ in range(3):
        grp2.step(t=0.3 + s_ * tau, tau=tau)
    v8 = grp2.gather()
    w8 = psi
    for s_ in range(3):
        w8 = orc.tdpot_strang_step(cache.exps, b.nodes, w8, 0.3 + s_ * tau, tau)
    flop = 8 * 3 * k**4
    return {"config": "4: TD-potential Strang 256^3 c128 (1 GPU; 8-rank schedule as virtual ranks)",
            "gpu_ms": ms, "tflops": flop / (ms * 1e-3) / 1e12, "cpu_ms": cpu_ms, "cpu_reps": kk,
            "speedup": cpu_ms / ms, "parity_rel_l2": orc.rel_l2(got, want),
            "virtual8_group_step_ms": ms_virtual8, "virtual8_per_rank_ms": ms_virtual8 / 8,
            "virtual8_parity_rel_l2_3_steps": orc.rel_l2(v8, w8)}


def config5(budget, n=512):
    grids, lin_op, weights = km.gpe_setup(n)
    psi = weighted_vortex_state(grids, weights)
    tau = 0.1
    cache = km.prepare(lin_op, tau)
    p_dev = dv.to_device(psi, np.complex128, DEV)
    ms = dev_time(lambda: km.gpe_strang_step(cache, weights, p_dev, tau), 5)
    got = km.gpe_strang_step(cache, weights, psi, tau)
    want = orc.gpe_strang_step(cache.exps, weights, psi, tau)
    cpu_ms, kk = cpu_time(lambda: orc.gpe_strang_step(cache.exps, weights, psi, tau), budget, 1)
    c64 = km.PropagatorCache(tau, tuple(e.astype(np.complex64) for e in cache.exps))
    p64 = dv.to_device(psi.astype(np.complex64), np.complex64, DEV)
    ms64 = dev_time(lambda: km.gpe_strang_step(c64, weights, p64, tau), 5)
    ms_run = dev_time(lambda: km.gpe_strang_run(cache, weights, p_dev, tau, 4), 2, warm=1) / 4
    # the P-rank slab schedule (SlabGpeStepper) as P virtual ranks on this GPU: per-rank time
    # = group time / P; parity of 2 steps against the single-GPU fused run
    virtual = {}
    for P in (2, 4, 8):
        grp = dist.VirtualSlabGroup(psi, cache, DEV, P, kind="gpe", weights=weights, tau=tau)
        kk_ = [0]

        def vstep():
            grp.step(k=kk_[0] % 2, steps=2)
            kk_[0] += 1

        gms = dev_time(vstep, 2, warm=2)
        grp2 = dist.VirtualSlabGroup(psi, cache, DEV, P, kind="gpe", weights=weights, tau=tau)
        for k_ in range(2):
            grp2.step(k=k_, steps=2)
        ref2 = km.gpe_strang_run(cache, weights, p_dev, tau, 2)
        virtual[P] = {"group_step_ms": gms, "per_rank_ms": gms / P,
                      "parity_vs_single_gpu_2_steps": orc.rel_l2(grp2.gather(), dv.to_host(ref2))}
        del grp, grp2
    flop = 8 * 3 * n**4
    return {"config": "5: GPE 512^3 Strang step c128 (c64 input follows the reference's promotion to c128)",
            "gpu_ms": ms, "gpu_ms_c64_input": ms64, "gpu_ms_per_step_fused_run": ms_run,
            "virtual_ranks": virtual,
            "tflops": flop / (ms * 1e-3) / 1e12, "cpu_ms": cpu_ms,
            "cpu_reps": kk, "speedup": cpu_ms / ms, "parity_rel_l2": orc.rel_l2(got, want)}


def config_magnus(budget, k=256, steps=4):
    """Extra: HKMP Magnus midpoint steps, host vs device exponentials."""
    from paper_2103_01691_b200.problems import hkmp_factors, schrodinger_initial_state

    b = km.hermite_basis(k)
    psi0 = schrodinger_initial_state((b.nodes,) * 3)
    c0 = dv.to_device(km.forward_transform((b,) * 3, psi0), np.complex128, DEV)
    tau = 1.0 / 32

    def run(device_expm):
        u = c0
        for s in range(steps):
            u = km.magnus_midpoint_step(lambda t: hkmp_factors(b, t), u, s * tau, tau, device_expm=device_expm)
        return u

    import time as _t

    for flag in (False, True, False, True):
        run(flag)
    torch.cuda.synchronize()

    def timed(flag):  # best of 3 chained runs of `steps` steps (wall clock: exponentials + products)
        best, res = None, None
        for _ in range(3):
            t0 = _t.perf_counter()
            res = run(flag)
            torch.cuda.synchronize()
            ms = (_t.perf_counter() - t0) * 1e3 / steps
            best = ms if best is None else min(best, ms)
        return best, res

    ms_host, host = timed(False)
    ms_dev, devr = timed(True)
    c0h = dv.to_host(c0)

    def cpu_run():
        from paper_2103_01691_b200.linalg import matexp

        u = c0h
        for s in range(steps):
            op = hkmp_factors(b, (s + 0.5) * tau)
            u = orc.step([matexp(tau * a) for a in op.factors], u)
        return u

    cpu_ms, kk = cpu_time(cpu_run, budget, 2)
    return {"config": f"extra: HKMP Magnus midpoint step k={k} c128 (wall clock per step incl. exponentials)",
            "gpu_ms_host_expm": ms_host, "gpu_ms_device_expm": ms_dev, "cpu_ms": cpu_ms / steps, "cpu_reps": kk,
            "speedup_device_expm": cpu_ms / steps / ms_dev,
            "parity_rel_l2_device_vs_host_expm": orc.rel_l2(dv.to_host(devr), dv.to_host(host))}


def config_c64(budget, n=256):
    """Extra: the complex64 exact step (tcgen05 3xTF32 kernels) vs the reference's own complex64 path."""
    u = crand(np.random.default_rng(0), (n,) * 3).astype(np.complex64)
    c128 = schrod(n)
    cache = km.PropagatorCache(0.01, tuple(e.astype(np.complex64) for e in c128.exps))
    t = dv.to_device(u, np.complex64, DEV)
    ms = dev_time(lambda: km.step(cache, t), 20)
    got = km.step(cache, u)
    want = orc.step(cache.exps, u)
    want128 = orc.step(c128.exps, u.astype(np.complex128))
    cpu_ms, kk = cpu_time(lambda: orc.step(cache.exps, u), budget, 3)
    flop = 8 * 3 * n**4
    return {"config": "extra: 3D Schrodinger 256^3 complex64 exact step (tcgen05 kind::tf32, 3xTF32)", "gpu_ms": ms,
            "tflops": flop / (ms * 1e-3) / 1e12, "cpu_ms": cpu_ms, "cpu_reps": kk, "speedup": cpu_ms / ms,
            "parity_rel_l2_vs_reference_c64": orc.rel_l2(got, want),
            "rel_l2_vs_c128": orc.rel_l2(got, want128), "reference_c64_rel_l2_vs_c128": orc.rel_l2(want, want128)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default="12345ms")
    args = ap.parse_args()
    cores = os.cpu_count() or 1
    from threadpoolctl import threadpool_info

    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), model)
    except OSError:
        pass
    res = {"cores": cores, "cpu_model": model,
           "blas": [f"{i.get('internal_api')} {i.get('version')} x{i.get('num_threads')}" for i in threadpool_info()],
           "configs": []}
    print(json.dumps({"cores": cores, "cpu_model": model, "blas": res["blas"]}), flush=True)
    fns = {"1": config1, "2": config2, "3": config3, "4": config4, "5": config5, "m": config_magnus, "s": config_c64}
    with threadpool_limits(limits=cores):
        for key in args.only:
            t0 = time.time()
            r = fns[key](args.cpu_budget)
            r["wall_s"] = time.time() - t0
            print(json.dumps(r), flush=True)
            res["configs"].append(r)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
