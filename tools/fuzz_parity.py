"""Randomised parity sweep of the public API against the CPU oracle (a longer version of
tests/test_gpu_random_shapes.py): random d, extents (ragged, tiny, TMA-sized), dtype mixes,
directions, factor row counts, None slots and kernel policies, for a wall-clock budget.

    python tools/fuzz_parity.py [seconds] [seed]

Prints one line per failure and a summary (cases per route, worst error per dtype).
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from oracle import kronmode_oracle as orc  # noqa: E402
from paper_2103_01691_b200 import _device as dv, _native, dist  # noqa: E402

DEV = torch.device("cuda", 0)
TOL = {np.dtype(np.complex128): 1e-12, np.dtype(np.float64): 1e-12, np.dtype(np.complex64): 1e-5,
       np.dtype(np.float32): 1e-5}
POLICIES = [_native.POLICY_AUTO, _native.POLICY_AUTO, _native.POLICY_NO_STREAMK, _native.POLICY_NO_TMA,
            _native.POLICY_NO_PLANE_FUSION]


def rand(rng, shape, dt):
    a = rng.standard_normal(shape)
    if np.dtype(dt).kind == "c":
        a = a + 1j * rng.standard_normal(shape)
    return np.asfortranarray(a.astype(dt))


def extent(rng):
    r = rng.random()
    if r < 0.25:
        return int(rng.integers(1, 12))
    if r < 0.55:
        return int(rng.choice([32, 48, 64, 128, 256]))
    return int(rng.integers(12, 300))


def diagnose(u, mats, device_in, tol):
    """Replay a failing tucker product by product (oracle intermediates as inputs) under every
    policy, and print which product and policy go wrong."""
    lib = _native.lib()
    cur = u
    for mu, mat in enumerate(mats, start=1):
        if mat is None:
            continue
        want = orc.mu_mode_product(cur, mat, mu)
        shape = cur.shape
        nl, nr = int(np.prod(shape[:mu - 1])), int(np.prod(shape[mu:]))
        for pol in (_native.POLICY_AUTO, _native.POLICY_NO_STREAMK, _native.POLICY_NO_TMA):
            _native.check(lib.km_set_kernel_policy(pol))
            x = dv.to_device(cur, cur.dtype, DEV) if device_in else cur
            got = km.mu_mode_product(x, mat, mu)
            got = dv.to_host(got) if isinstance(got, torch.Tensor) else got
            e = orc.rel_l2(got, want)
            if not e <= tol:
                bad = np.argwhere(np.abs(got - want) > 1e-6 * np.abs(want).max())
                print(f"   product mu={mu} (m={mat.shape[0]}, nl={nl}, nmu={shape[mu - 1]}, nr={nr}, "
                      f"u {cur.dtype}, L {mat.dtype}) policy={pol}: err {e:.3e}, bad entries {len(bad)} "
                      f"first {bad[:3].tolist()}", flush=True)
        _native.check(lib.km_set_kernel_policy(_native.POLICY_AUTO))
        cur = want


def main(budget=600.0, seed=0):
    rng = np.random.default_rng(seed)
    lib = _native.lib()
    worst, counts, fails = {}, {}, 0
    t_end = time.time() + budget
    n = 0
    while time.time() < t_end:
        n += 1
        pol = int(rng.choice(POLICIES))
        _native.check(lib.km_set_kernel_policy(pol))
        kind = rng.random()
        try:
            if kind < 0.1:  # paired steps on a small cube
                dims = tuple(int(rng.choice([32, 48, 64])) for _ in range(3))
                steps = int(rng.integers(1, 6))
                mats = [rand(rng, (m, m), np.complex128) / m for m in dims]
                u = rand(rng, dims, np.complex128)
                st = dist.LocalStepper(dv.to_device(u, np.complex128, DEV),
                                       [dv.matrix_to_device(m, np.complex128, DEV) for m in mats])
                st.run(steps)
                want = u
                for _ in range(steps):
                    want = orc.tucker(want, mats)
                got, route, dt = dv.to_host(st.a), "steps_paired", np.dtype(np.complex128)
            else:
                d = int(rng.integers(2, 4))
                while True:
                    dims = tuple(extent(rng) for _ in range(d))
                    if np.prod(dims) <= (1 << 24):
                        break
                udt = rng.choice([np.complex128, np.float64, np.complex64, np.float32])
                mdt = rng.choice([np.complex128, np.float64]) if np.dtype(udt).itemsize * (
                    1 if np.dtype(udt).kind == "c" else 2) >= 16 else rng.choice([np.complex64, np.float32])
                u = rand(rng, dims, udt)
                device_in = rng.random() < 0.7
                if kind < 0.55:  # one product
                    mu = int(rng.integers(1, d + 1))
                    m = max(1, int(rng.integers(1, dims[mu - 1] + 40)))
                    mat = rand(rng, (m, dims[mu - 1]), mdt) / np.sqrt(dims[mu - 1])
                    x = dv.to_device(u, udt, DEV) if device_in else u
                    got = km.mu_mode_product(x, mat, mu)
                    want = orc.mu_mode_product(u, mat, mu)
                    route = f"product d{d} mu{mu}"
                else:  # tucker with None slots
                    mats = []
                    for k in range(d):
                        if rng.random() < 0.2:
                            mats.append(None)
                        else:
                            m = max(1, int(rng.integers(max(1, dims[k] // 2), dims[k] + 20)))
                            mats.append(rand(rng, (m, dims[k]), mdt) / np.sqrt(dims[k]))
                    x = dv.to_device(u, udt, DEV) if device_in else u
                    got = km.tucker(x, mats)
                    want = orc.tucker(u, mats)
                    route = f"tucker d{d}"
                got = dv.to_host(got) if isinstance(got, torch.Tensor) else got
                dt = np.result_type(np.dtype(udt), np.dtype(mdt))
            err = orc.rel_l2(got, want)
            key = str(dt)
            worst[key] = max(worst.get(key, 0.0), err)
            counts[route.split()[0]] = counts.get(route.split()[0], 0) + 1
            if not (err <= TOL[np.dtype(dt)]):
                fails += 1
                print(f"FAIL #{n}: {route} dims={dims} dtype={dt} policy={pol} err={err:.3e} "
                      f"device_in={device_in if kind >= 0.1 else True}", flush=True)
                if kind >= 0.55:
                    _native.check(lib.km_set_kernel_policy(pol))
                    again = [orc.rel_l2((lambda g: dv.to_host(g) if isinstance(g, torch.Tensor) else g)(
                        km.tucker(dv.to_device(u, udt, DEV) if device_in else u, mats)), want) for _ in range(3)]
                    print(f"   same call again: {['%.1e' % e for e in again]}", flush=True)
                    diagnose(u, mats, device_in, TOL[np.dtype(dt)])
        except Exception as exc:  # noqa: BLE001
            fails += 1
            print(f"ERROR #{n}: {type(exc).__name__}: {exc}", flush=True)
    _native.check(lib.km_set_kernel_policy(_native.POLICY_AUTO))
    print(f"cases {n}, failures {fails}; per route {counts}; worst rel l2 per dtype "
          f"{ {k: f'{v:.2e}' for k, v in worst.items()} }", flush=True)


if __name__ == "__main__":
    main(float(sys.argv[1]) if len(sys.argv) > 1 else 600.0, int(sys.argv[2]) if len(sys.argv) > 2 else 0)
