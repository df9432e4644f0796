"""Repeat one product / Tucker call many times against a fixed oracle result, to catch
intermittent (timing-dependent) errors, per input route (numpy -> host pipeline, device
tensor -> km_tucker) and kernel policy.

    python tools/race_probe.py [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from oracle import kronmode_oracle as orc  # noqa: E402
from paper_2103_01691_b200 import _device as dv, _native  # noqa: E402

DEV = torch.device("cuda", 0)


def case(dims, dt, mu=None, seed=0):
    rng = np.random.default_rng(seed)
    u = np.asfortranarray(rng.standard_normal(dims).astype(dt))
    if mu is None:
        mats = [np.asarray(rng.standard_normal((int(rng.integers(n // 2, n + 20)), n)) / np.sqrt(n), dtype=dt)
                for n in dims]
        return u, mats, orc.tucker(u, mats)
    n = dims[mu - 1]
    mat = np.asarray(rng.standard_normal((n, n)) / np.sqrt(n), dtype=dt)
    return u, (mu, mat), orc.mu_mode_product(u, mat, mu)


def per_product(reps=200, dims=(216, 213, 263), dt=np.float64, seed=0):
    """The failing Tucker of main(), one product at a time on device inputs (the oracle's
    intermediate as the input), under each policy: which product is intermittent."""
    lib = _native.lib()
    u, mats, _ = case(dims, dt, None, seed)
    cur = u
    for mu, mat in enumerate(mats, start=1):
        want = orc.mu_mode_product(cur, mat, mu)
        x = dv.to_device(cur, dt, DEV)
        dm = dv.matrix_to_device(mat, dt, DEV)
        for pol in (_native.POLICY_AUTO, _native.POLICY_NO_STREAMK, _native.POLICY_NO_TMA):
            _native.check(lib.km_set_kernel_policy(pol))
            bad = 0
            for _ in range(reps):
                got = dv.to_host(km.mu_mode_product(x, dm, mu))
                if not orc.rel_l2(got, want) <= 1e-12:
                    bad += 1
            print(f"  product mu={mu} shape {cur.shape} m={mat.shape[0]} policy={pol}: {bad}/{reps} bad", flush=True)
        cur = want
    _native.check(lib.km_set_kernel_policy(_native.POLICY_AUTO))


def f32_products(reps=200):
    """float32 direction-1 products with rectangular factors (the fuzz's other failure)."""
    lib = _native.lib()
    rng = np.random.default_rng(5)
    for dims in ((256, 128, 256), (200, 150, 300), (256, 256, 128)):
        u = np.asfortranarray(rng.standard_normal(dims).astype(np.float32))
        for m in (dims[0], int(dims[0] * 0.7) + 3, dims[0] + 17):
            mat = (rng.standard_normal((m, dims[0])) / np.sqrt(dims[0])).astype(np.float32)
            want = orc.mu_mode_product(u, mat, 1)
            for route in ("numpy", "device"):
                x = u if route == "numpy" else dv.to_device(u, np.float32, DEV)
                for pol in (_native.POLICY_AUTO, _native.POLICY_NO_STREAMK):
                    _native.check(lib.km_set_kernel_policy(pol))
                    bad, worst = 0, 0.0
                    for _ in range(reps):
                        got = km.mu_mode_product(x, mat, 1)
                        got = dv.to_host(got) if isinstance(got, torch.Tensor) else got
                        e = orc.rel_l2(got, want)
                        worst = max(worst, e)
                        bad += not e <= 1e-5
                    print(f"f32 mu=1 {dims} m={m} {route} policy={pol}: {bad}/{reps} bad, worst {worst:.2e}",
                          flush=True)
    _native.check(lib.km_set_kernel_policy(_native.POLICY_AUTO))


def main(reps=300):
    lib = _native.lib()
    cases = [((216, 213, 263), np.float64, None), ((256, 225, 128), np.float64, None),
             ((256, 243, 238), np.float64, None), ((256, 128, 256), np.float32, 1),
             ((256, 225, 128), np.complex128, None)]
    for dims, dt, mu in cases:
        u, arg, want = case(dims, dt, mu)
        tol = 1e-12 if np.dtype(dt) in (np.dtype(np.float64), np.dtype(np.complex128)) else 1e-5
        for route in ("numpy", "device"):
            for pol in (_native.POLICY_AUTO, _native.POLICY_NO_STREAMK):
                _native.check(lib.km_set_kernel_policy(pol))
                x = u if route == "numpy" else dv.to_device(u, dt, DEV)
                bad, worst = 0, 0.0
                for r in range(reps):
                    got = km.tucker(x, arg) if mu is None else km.mu_mode_product(x, arg[1], arg[0])
                    got = dv.to_host(got) if isinstance(got, torch.Tensor) else got
                    e = orc.rel_l2(got, want)
                    worst = max(worst, e)
                    if not e <= tol:
                        bad += 1
                        if bad <= 3:
                            diff = np.abs(got - want) > 1e-6 * np.abs(want).max()
                            idx = np.argwhere(diff)
                            print(f"   rep {r}: err {e:.2e}, {len(idx)} bad entries, index ranges "
                                  f"{idx.min(axis=0).tolist()}..{idx.max(axis=0).tolist()}", flush=True)
                print(f"{dims} {np.dtype(dt)} {'tucker' if mu is None else f'mu={mu}'} {route} policy={pol}: "
                      f"{bad}/{reps} bad, worst {worst:.2e}", flush=True)
    _native.check(lib.km_set_kernel_policy(_native.POLICY_AUTO))


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "per-product":
        per_product(int(sys.argv[1]))
    elif len(sys.argv) > 2 and sys.argv[2] == "f32":
        f32_products(int(sys.argv[1]))
    else:
        main(int(sys.argv[1]) if len(sys.argv) > 1 else 300)
