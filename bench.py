"""Benchmark of the north-star workload: the 3D complex128 μ-mode exponential step at n=256^3.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = one exact propagator step ``u <- u x_1 E_1 x_2 E_2 x_3 E_3`` of a
256^3 complex128 tensor (E_mu = expm(0.01 i D2), D2 the periodic p=2 second
difference on [0, 2π)), i.e. 103.08 GFLOP at 8 flop per
complex multiply-add.  Prints ONE JSON line (rank 0).

* value      — steps/s of the whole job, device-resident inputs, CUDA events
               around exactly K steps, max over ranks.
* e2e        — the same metric through the public drop-in call
               ``km.step(cache, u_host)`` with a pinned host array in and a host
               array out (H2D + D2H inside the timed region).
* roofline   — the dominant kernel (mumode_tma_kernel, DMMA) achieved TFLOP/s vs
               the measured FP64 tensor-core peak (profiles/fp64_peak.json).
* cpu_baseline — the reference algorithm (oracle/ numpy restatement, same
               numpy.matmul calls as tensor.py:124-139) on the host cores.

The state (268 MB) exceeds the 126 MB L2, so no flush is needed between steps.
Multi-GPU (N>1): the 256^3 state is split into slabs along direction 3
(strong scaling); see paper_2103_01691_b200/dist.py.  Launched either by the
driver's torchrun or, for ``--gpus N`` without a torchrun environment, by
bench.py itself (one rank per GPU on 127.0.0.1); ``n_gpus`` is the world size
the ranks actually formed, in both arms.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N = 256
TAU = 0.01
FLOP_PER_STEP = 8 * 3 * N**4  # 8 flop per complex MAC, 3 directions, N^3 * n MACs each
METRIC = "3D μ-mode step/s & GFLOP/s (complex128, n=256³) at 1/2/4/8 B200 vs CPU ref"
WORKLOAD = {
    "workload": "schrodinger3d_free_step_c128_n256",
    "n": N,
    "tau": TAU,
    "factors": "E_mu = expm(i*tau*D2), D2 periodic 2nd-order on [0,2pi) (host scipy)",
    "state_bytes": 16 * N**3,
    "l2": "state 268 MB > 126 MB L2; no flush needed",
    "flop_per_step": FLOP_PER_STEP,
}
PROFILES = os.path.join(ROOT, "profiles")


def build_inputs():
    import paper_2103_01691_b200 as km

    rng = np.random.default_rng(0)
    u = np.asfortranarray(rng.standard_normal((N,) * 3) + 1j * rng.standard_normal((N,) * 3))
    d2 = km.heat_factors(N, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), TAU)
    return u, cache


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.15)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, flag in zip(names, parts[4:8]):
                if flag.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def fp64_peak():
    path = os.path.join(PROFILES, "fp64_peak.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["dmma_tflops_sustained"]), p.get("source", path)
    except (OSError, KeyError, ValueError):
        return 37.1, "fallback: DMMA.8x8x4 microbenchmark burst (tools/fp64_peak.cu), not committed"


def traffic_from_profile():
    path = os.path.join(PROFILES, "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def cpu_model():
    """The host CPU's model name (lscpu's "Model name", from /proc/cpuinfo)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_reference(u, cache, budget_s, max_steps):
    """The reference algorithm (oracle numpy restatement) on all host threads."""
    from threadpoolctl import threadpool_info, threadpool_limits

    from oracle import kronmode_oracle as orc

    cores = os.cpu_count() or 1
    with threadpool_limits(limits=cores):
        blas = [f"{i.get('internal_api')} {i.get('version')} x{i.get('num_threads')}" for i in threadpool_info()]
        orc.step(cache.exps, u)  # warm-up
        times = []
        v = u
        t_start = time.perf_counter()
        while len(times) < max_steps:
            t0 = time.perf_counter()
            v = orc.step(cache.exps, v)
            times.append(time.perf_counter() - t0)
            if time.perf_counter() - t_start > budget_s:
                break
    sps = len(times) / sum(times)
    return {
        "value": sps,
        "unit": "steps/s",
        "cores": cores,
        "cpu_model": cpu_model(),
        "kind": "port",
        "sample": f"{len(times)} full 256^3 c128 steps after 1 warm-up, numpy.matmul ({'; '.join(blas)})",
        "gflops": sps * FLOP_PER_STEP / 1e9,
        "ms_per_step": 1e3 / sps,
    }


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    u, cache = build_inputs()
    steps = max(1, args.steps)
    # bounded: at most ~120 s of CPU work whatever K is
    cb = cpu_reference(u, cache, budget_s=120.0, max_steps=steps)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": cb["value"],
        "unit": "steps/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": args.warmup,
        "ms_per_step": cb["ms_per_step"],
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "complex128",
        "data": "synthetic (seeded normal complex tensor)",
        "config": dict(WORKLOAD),
        "parallelism": "CPU reference (host cores of rank 0)",
        "gflops": cb["gflops"],
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def e2e_slabs(runner, u_host, rank, world, dev, args):
    """End-to-end at N > 1: every rank copies its input slab from pinned host memory, the ranks run
    one distributed step (exchange included), and every rank copies its result slab back.
    Not exercised with more than one GPU in round 1 (gpurun provides one).
    Time = max over ranks of the host wall clock; bytes = the rank's slab each way."""
    import torch
    import torch.distributed as tdist

    plan = runner.plan
    slab = np.asfortranarray(plan.slab_a(u_host, rank))
    h_in = torch.empty(plan.local, dtype=torch.complex128, pin_memory=True)
    h_in.numpy()[...] = slab.reshape(-1, order="F")
    h_out = torch.empty(plan.local, dtype=torch.complex128, pin_memory=True)

    def one():
        # fresh input each call, in the slab layout the schedule is in (A and B slabs have the same
        # size; the layouts keep alternating, which the peer exchange's buffer parity relies on)
        runner.a.copy_(h_in, non_blocking=True)
        runner.step()
        h_out.copy_(runner.a, non_blocking=True)
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        one()
    steps = max(3, min(args.steps, 30))
    tdist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    el = time.perf_counter() - t0
    t = torch.tensor([el], device=dev, dtype=torch.float64)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    el = float(t.item())
    nbytes = int(h_in.numel() * h_in.element_size())
    return {"value": steps / el, "unit": "steps/s", "h2d_bytes_per_step": nbytes * world,
            "d2h_bytes_per_step": nbytes * world, "steps": steps,
            "call": "dist.SlabStepper: per-rank pinned slab -> device, one distributed step, slab -> pinned host"}


def config_sweep(dev):
    """Every BASELINE.json configuration on this GPU, device-resident: ms per unit, TFLOP/s at the
    8-flop-per-complex-MAC convention (4 for real x complex, 2 for real x real) and the fraction of
    the measured DMMA peak.  Parity of each one at its BASELINE size is the -m gpu tests'
    (tests/test_gpu_configs.py); the CPU reference times are tools/bench_configs.py's."""
    import torch

    import paper_2103_01691_b200 as km
    from paper_2103_01691_b200 import _device as dv
    from paper_2103_01691_b200 import dist
    from paper_2103_01691_b200.hermite import physical_propagator
    from paper_2103_01691_b200.problems import schrodinger_initial_state, ti_potentials, weighted_vortex_state

    peak, _ = fp64_peak()

    def dev_ms(fn, reps, warm=3):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / reps

    def entry(name, ms, flop, unit):
        tf = flop / (ms * 1e-3) / 1e12
        return {"config": name, "ms": ms, "unit": unit, "tflops": tf, "frac_of_dmma_peak": tf / peak}

    rng = np.random.default_rng(0)
    out = []
    # 1: 64^3 c128, 10 exact steps as one LocalStepper.run (km_steps_paired: two steps per three
    # fused launches) captured in a CUDA graph
    n = 64
    d2 = km.heat_factors(n, 2).factors[0]
    c1 = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    u1 = np.asfortranarray(rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3))
    st = dist.LocalStepper(dv.to_device(u1, np.complex128, dev), c1.device_exps((np.complex128,) * 3, dev))
    for _ in range(3):
        st.step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            st.run(10)
    torch.cuda.synchronize()
    out.append(entry(f"1: Schrodinger free 64^3 c128, 10 steps (CUDA graph, {st.launches_for(10)} launches)",
                     dev_ms(g.replay, 50), 10 * 8 * 3 * n**4, "ms per 10 steps"))
    del g, st
    # 2: pipe flow 1024^2 f64, one exact step
    n = 1024
    c2 = km.prepare(km.pipeflow_factors(n), 4.0 / 8)
    rho, z = np.linspace(0.1, 5.0, n), np.linspace(0.0, 8.0, n)
    u2 = np.asfortranarray(np.exp(-8.0 * (rho - 2.55) ** 2)[:, None] * np.exp(-8.0 * (z - 1.5) ** 2)[None, :])
    st = dist.LocalStepper(dv.to_device(u2, np.float64, dev), c2.device_exps((np.float64,) * 2, dev))
    out.append(entry("2: pipe flow 1024^2 f64, one step", dev_ms(st.step, 50), 2 * 2 * n**3, "ms per step"))
    del st
    # 3: HKP 256^3: forward transform + exact step + inverse transform
    k = 256
    b = km.hermite_basis(k)
    op = km.KroneckerOp(tuple(km.hamiltonian_factor(b, v) for v in ti_potentials()))
    c3 = km.prepare(op, 1.0)
    p3 = dv.to_device(schrodinger_initial_state((b.nodes,) * 3), np.complex128, dev)
    hkp = lambda: km.inverse_transform((b,) * 3, km.step(c3, km.forward_transform((b,) * 3, p3)))  # noqa: E731
    out.append(entry("3: HKP 256^3 c128 forward + step + inverse", dev_ms(hkp, 10), 4 * 3 * k**4 * 2 + 8 * 3 * k**4,
                     "ms per solve"))
    # 4: TD-potential Strang step 256^3 (E3 folded per step)
    tau = 0.02
    pp = physical_propagator(b, tau)
    c4 = km.PropagatorCache(tau, (pp, pp, pp))
    out.append(entry("4: TD-potential Strang 256^3 c128, one step",
                     dev_ms(lambda: km.tdpot_strang_step(c4, b.nodes, p3, 0.3, tau), 10), 8 * 3 * k**4, "ms per step"))
    del p3
    torch.cuda.empty_cache()
    # 5: GPE Strang step 512^3 c128 (and per step of a fused run)
    n = 512
    grids, lin_op, weights = km.gpe_setup(n)
    c5 = km.prepare(lin_op, 0.1)
    p5 = dv.to_device(weighted_vortex_state(grids, weights), np.complex128, dev)
    out.append(entry("5: GPE Strang 512^3 c128, one step", dev_ms(lambda: km.gpe_strang_step(c5, weights, p5, 0.1), 3,
                                                                   warm=1), 8 * 3 * n**4, "ms per step"))
    del p5
    torch.cuda.empty_cache()
    return out


def run_ours(args):
    import torch

    import paper_2103_01691_b200 as km
    from paper_2103_01691_b200 import _device as dv
    from paper_2103_01691_b200 import dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as tdist

        tdist.init_process_group("nccl", device_id=dev)

    u_host, cache = build_inputs()
    stream = torch.cuda.current_stream(dev)
    slab = world > 1 or args.slab  # --slab: the multi-GPU code path on one rank (torchrun world 1)
    if slab and world == 1:
        import torch.distributed as tdist

        tdist.init_process_group("nccl", device_id=dev)

    if not slab:
        state = dv.to_device(u_host, np.complex128, dev)
        mats = cache.device_exps((np.complex128,) * 3, dev)
        runner = dist.LocalStepper(state, mats)
    else:
        cls = dist.PeerSlabStepper if args.exchange == "peer" else dist.SlabStepper
        runner = cls.from_global(u_host, cache, dev)

    for _ in range(max(args.warmup, 3)):
        runner.step()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as tdist

            tdist.barrier()
        torch.cuda.synchronize()

    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        start.record(stream)
        for _ in range(args.steps):
            runner.step()
        stop.record(stream)
        barrier()
    ms = start.elapsed_time(stop)
    if world > 1:
        import torch.distributed as tdist

        t = torch.tensor([ms], device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = 1e3 / ms_per_step  # whole job: one global 256^3 step per step

    # per-launch roofline of the dominant kernel (single GPU timing of one step's launches)
    roof = None
    if rank == 0:
        per_mode = runner.time_launches(reps=10) if not slab else None
        peak, peak_src = fp64_peak()
        if slab:  # per-GPU share of the step's flops over the whole step (exchange included)
            achieved = FLOP_PER_STEP / world / (ms_per_step * 1e-3) / 1e12
            roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": None,
                    "kernel": "per-rank step: 3 x mumode_tma_kernel on the slab + exchange",
                    "algorithmic_per_launch": f"{FLOP_PER_STEP // world} flop per rank per step",
                    "peak_source": peak_src}
        if per_mode:
            flop_launch = 8 * N**4
            avg_ms = sum(per_mode) / len(per_mode)
            achieved = flop_launch / (avg_ms * 1e-3) / 1e12
            roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": traffic_from_profile(),
                    "kernel": "mumode_tma_kernel (TMA + mbarrier ring, DMMA.8x8x4, complex128)",
                    "algorithmic_per_launch": f"{flop_launch} flop (8 * 256^4)",
                    "launch_ms": per_mode, "peak_source": peak_src}

    # e2e through the public drop-in call with host buffers
    e2e = None
    if not slab:
        pinned = torch.empty((N, N, N), dtype=torch.complex128, pin_memory=True)
        pinned_np = pinned.numpy()
        pinned_np[...] = u_host.transpose(2, 1, 0)  # C-order buffer ...
        host_in = pinned_np.transpose(2, 1, 0)      # ... viewed column-major, same memory
        assert host_in.flags.f_contiguous
        e2e_steps = max(3, min(args.steps, 30))
        for _ in range(max(args.warmup, 3)):  # warm-up: device allocator, pinned result pool, module loading
            out = km.step(cache, host_in)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            out = km.step(cache, host_in)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        e2e = {"value": e2e_steps / el, "unit": "steps/s", "h2d_bytes_per_step": int(host_in.nbytes),
               "d2h_bytes_per_step": int(out.nbytes), "steps": e2e_steps,
               "call": "paper_2103_01691_b200.step(cache, numpy F-array in pinned memory) -> numpy"}
        # the same call with an ordinary (pageable) numpy input, as a typical caller passes it
        # (reported beside the headline e2e, not instead of it)
        pageable = np.asfortranarray(u_host.copy())
        for _ in range(2):
            out = km.step(cache, pageable)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            out = km.step(cache, pageable)
        torch.cuda.synchronize()
        e2e["pageable_input"] = {"value": e2e_steps / (time.perf_counter() - t0), "unit": "steps/s",
                                 "steps": e2e_steps}
    else:
        try:
            e2e = e2e_slabs(runner, u_host, rank, world, dev, args)
        except Exception as exc:  # an e2e failure must not lose the device-timed line
            e2e = {"value": None, "unit": "steps/s", "error": f"{type(exc).__name__}: {exc}"}

    if rank == 0:
        cb = cpu_reference(u_host, cache, budget_s=20.0, max_steps=50) if not args.no_cpu else None
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "steps/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": max(args.warmup, 3),
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "complex128",
            "data": "synthetic (seeded normal complex tensor, host-built expm factors)",
            "config": dict(WORKLOAD),
            "parallelism": ("single GPU" if not slab else
                            f"slab{world} along direction 3, {args.exchange} exchange"),
            "gflops": value * FLOP_PER_STEP / 1e9,
            "roofline": roof,
            "cpu_baseline": cb,
            "e2e": e2e,
            "clocks": clocks.summary(),
            "gpu_launches": runner.launches_per_step * args.steps,
        }
        if not slab and not args.no_configs:
            try:
                line["configs"] = config_sweep(dev)
            except Exception as exc:  # the sweep must not lose the headline line
                line["configs"] = {"error": f"{type(exc).__name__}: {exc}"}
    if slab:
        import torch.distributed as tdist

        # every rank is done before the communicators go (their teardown lines come first),
        # so rank 0's JSON line is the last thing it prints
        tdist.barrier()
        tdist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def launch_ranks(args, argv):
    """``--gpus N`` (N > 1) without a torchrun environment: start the N ranks ourselves.

    Runs ``python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1``
    on this same script and arguments (one process per GPU, rank = local GPU), after
    checking that N GPUs are visible, and returns its exit code; rank 0 prints the JSON
    line.  ``KMB200_BENCH_SELFTEST=1`` skips the GPU check (the CPU launcher test).
    """
    selftest = os.environ.get("KMB200_BENCH_SELFTEST") == "1"
    if not selftest:
        import torch

        have = torch.cuda.device_count() if torch.cuda.is_available() else 0
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}", file=sys.stderr)
            return 2
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + argv
    return subprocess.run(cmd).returncode


def selftest_rank(args):
    """KMB200_BENCH_SELFTEST=1 under the launcher: gloo rendezvous only, rank 0 reports the world."""
    import torch
    import torch.distributed as tdist

    tdist.init_process_group("gloo")
    t = torch.tensor([1.0])
    tdist.all_reduce(t)
    if tdist.get_rank() == 0:
        print(json.dumps({"impl": args.impl, "n_gpus": tdist.get_world_size(), "ranks_seen": int(t.item()),
                          "selftest": True}), flush=True)
    tdist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-configs", action="store_true", help="skip the BASELINE config sweep (N = 1)")
    ap.add_argument("--slab", action="store_true", help="run the multi-GPU slab path even on one rank (testing)")
    ap.add_argument("--exchange", choices=["nccl", "peer"], default="nccl",
                    help="multi-GPU all-to-all: NCCL, or fused into the products via NVLink peer stores")
    argv = sys.argv[1:]
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args, argv))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if os.environ.get("KMB200_BENCH_SELFTEST") == "1":
        selftest_rank(args)
        return
    if world > 1 and args.impl == "ours":
        # communicator lines (nranks) for the driver's check; INIT only, so the JSON line stays last
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
