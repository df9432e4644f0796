"""Small cases of every kernel family, for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [family ...]

Families (each checked against the CPU oracle, so a run also proves the kernels
still compute the right numbers under the tool):
  tma      persistent TMA + mbarrier DMMA kernel, whole tiles (complex and real factor,
           directions 1 and 3, fused GPE epilogue)
  streamk  the same kernel with the stream-K tail (bound stream workspace)
  cpasync  cp.async DMMA kernel (small tiles, f32/f64/mixed)
  tc32     tcgen05 CTA-pair kernel (K' <= 512), HALVES (K' <= 1024) and the chunked kernel
  peer     km_mumode_peer / km_mumode_split through P=2 virtual slab ranks (both exchanges)
  misc     pointwise phases, km_norm, km_diag_phase_fold
  plane    the fused first-two-products launch (mumode_plane12_kernel), also after a GPE
           pre-pass, and float32 x float32 fiber pairs on the tcgen05 kernel
Sizes are the smallest that still select each kernel (tile-count and K rules in
inst_tma_c128.cu / inst_tc32_c64.cu).
"""

from __future__ import annotations

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01691_b200 as km  # noqa: E402
from oracle import kronmode_oracle as orc  # noqa: E402
from paper_2103_01691_b200 import _device as dv  # noqa: E402
from paper_2103_01691_b200 import _native, dist  # noqa: E402

DEV = torch.device("cuda", 0)


def crand(rng, shape, dtype=np.complex128):
    return np.asfortranarray((rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(dtype))


def check(name, got, want, tol):
    err = orc.rel_l2(got, want)
    status = "ok" if err <= tol else "FAIL"
    print(f"{name}: rel_l2 {err:.2e} {status}", flush=True)
    if err > tol:
        raise SystemExit(f"{name} parity {err:.3e} > {tol}")


def product(u, mat, mu):
    return dv.to_host(km.mu_mode_product(dv.to_device(u, u.dtype, DEV), mat, mu))


def fam_tma(rng, policy=_native.POLICY_NO_STREAMK):
    lib = _native.lib()
    _native.check(lib.km_set_kernel_policy(policy))
    try:
        shape = (128, 128, 256)  # direction 3: 128 x 4 = 512 tiles of 128 x 64, K = 256
        u = crand(rng, shape)
        e = crand(rng, (256, 256))
        check("tma dir3 c128xc128", product(u, e, 3), orc.mu_mode_product(u, e, 3), 1e-12)
        ur = crand(rng, (256, 128, 128))
        phi = np.ascontiguousarray(rng.standard_normal((256, 256)))
        check("tma dir1 c128xf64", product(ur, phi, 1), orc.mu_mode_product(ur, phi, 1), 1e-12)
        # GPE step: the closing phase fused into the direction-3 epilogue
        n = 128
        grids, lin_op, weights = km.gpe_setup(n)
        from paper_2103_01691_b200.problems import weighted_vortex_state

        psi = weighted_vortex_state(grids, weights)
        cache = km.prepare(lin_op, 0.1)
        got = km.gpe_strang_step(cache, weights, dv.to_device(psi, np.complex128, DEV), 0.1)
        check("tma fused GPE", dv.to_host(got), orc.gpe_strang_step(cache.exps, weights, psi, 0.1), 1e-12)
    finally:
        _native.check(lib.km_set_kernel_policy(_native.POLICY_AUTO))


def fam_streamk(rng):
    fam_tma(rng, _native.POLICY_AUTO)


def fam_cpasync(rng):
    for dt, tol in ((np.complex128, 1e-12), (np.float64, 1e-12), (np.complex64, 1e-5), (np.float32, 1e-5)):
        u = crand(rng, (24, 40, 12), dt) if np.iscomplexobj(np.zeros(1, dt)) else \
            np.asfortranarray(rng.standard_normal((24, 40, 12)).astype(dt))
        for mu, n in ((1, 24), (2, 40), (3, 12)):
            mat = rng.standard_normal((n + 8, n)).astype(np.float64 if dt in (np.complex128, np.float64)
                                                        else np.float32)
            check(f"cp.async {np.dtype(dt).name} dir{mu}", product(u, mat, mu), orc.mu_mode_product(u, mat, mu), tol)


def fam_tc32(rng):
    u = crand(rng, (128, 128, 64), np.complex64)
    e = crand(rng, (128, 128), np.complex64) / np.sqrt(128)
    check("tc32 pair dir2", product(u, e, 2), orc.mu_mode_product(u, e, 2), 1e-5)
    uh = crand(rng, (384, 64, 16), np.complex64)  # direction 1: K' = 768 (HALVES)
    eh = crand(rng, (384, 384), np.complex64) / np.sqrt(384)
    check("tc32 halves dir1", product(uh, eh, 1), orc.mu_mode_product(uh, eh, 1), 1e-5)
    uc = crand(rng, (640, 32, 8), np.complex64)  # direction 1: K' = 1280 (chunked)
    ec = crand(rng, (640, 640), np.complex64) / np.sqrt(640)
    check("tc32 chunked dir1", product(uc, ec, 1), orc.mu_mode_product(uc, ec, 1), 1e-5)


def fam_peer(rng):
    n = 64
    u = crand(rng, (n,) * 3)
    d2 = km.heat_factors(n, 2).factors[0]
    cache = km.prepare(km.KroneckerOp((1j * d2,) * 3), 0.01)
    want = orc.step(cache.exps, orc.step(cache.exps, u))
    for exchange in ("nccl", "peer"):
        grp = dist.VirtualSlabGroup(u, cache, DEV, 2, exchange=exchange)
        grp.step()
        grp.step()
        check(f"slab P=2 {exchange}", grp.gather(), want, 1e-12)


def fam_misc(rng):
    shape = (48, 40, 36)
    u = crand(rng, shape)
    ws = [rng.random(n) + 0.5 for n in shape]
    from paper_2103_01691_b200.problems import _gpe_op
    from paper_2103_01691_b200.tensor import inner_weight_product

    w_dev = [dv.cached_vector(w, np.float64, DEV) for w in ws]
    inner = dv.cached_vector(inner_weight_product(ws, shape), np.float64, DEV)
    op = _gpe_op(shape, w_dev, 0.05, inner)
    t = dv.to_device(u, np.complex128, DEV)
    out = torch.empty_like(t)
    import ctypes

    _native.check(_native.lib().km_pointwise(t.data_ptr(), out.data_ptr(), _native.KM_C128, t.numel(),
                                             ctypes.byref(op), dv.stream_ptr(DEV)))
    check("pointwise GPE phase", dv.to_host(out), orc.nonlinear_half(u, orc.weight_product(ws, shape), 0.05), 1e-14)
    for kind in ("max", "two", "weighted_two"):
        w = ws if kind == "weighted_two" else None
        got = km.norm(t, kind, w)
        if kind == "max":
            want = np.abs(u).max()
        elif kind == "two":
            want = np.linalg.norm(u.ravel())
        else:
            want = np.sqrt(np.sum(orc.weight_product(ws, shape) * np.abs(u) ** 2))
        check(f"norm {kind}", np.array([got]), np.array([want]), 1e-13)
    from paper_2103_01691_b200.hermite import physical_propagator
    from paper_2103_01691_b200.problems import schrodinger_initial_state

    b = km.hermite_basis(32)
    p = physical_propagator(b, 0.02)
    cache = km.PropagatorCache(0.02, (p, p, p))
    psi = schrodinger_initial_state((b.nodes,) * 3)
    got = km.tdpot_strang_step(cache, b.nodes, dv.to_device(psi, np.complex128, DEV), 0.1, 0.02)
    check("diag fold + step", dv.to_host(got), orc.tdpot_strang_step(cache.exps, b.nodes, psi, 0.1, 0.02), 1e-12)


def fam_plane(rng):
    for shape in ((64, 64, 8), (48, 32, 5), (32, 64, 3)):
        u = crand(rng, shape)
        mats = [crand(rng, (n, n)) / n for n in shape]
        t = dv.to_device(u, np.complex128, DEV)
        got = km.tucker(t, [dv.matrix_to_device(m, np.complex128, DEV) for m in mats])
        check(f"plane fusion {shape}", dv.to_host(got), orc.tucker(u, mats), 1e-12)
    shape = (64, 64, 6)
    factors = [-0.5j * (lambda h: h + h.conj().T)(crand(rng, (n, n))) / n for n in shape]
    cache = km.prepare(km.KroneckerOp(tuple(factors)), 0.1)
    ws = [rng.random(n) + 0.5 for n in shape]
    psi = crand(rng, shape) * 0.3
    got = km.gpe_strang_step(cache, ws, dv.to_device(psi, np.complex128, DEV), 0.1)
    check("plane fusion after the GPE pre-pass", dv.to_host(got), orc.gpe_strang_step(cache.exps, ws, psi, 0.1), 1e-12)
    # two steps in three fused launches (plane, pencil, plane), 32- and 16-fiber pencil blocks
    from paper_2103_01691_b200 import dist

    for shape in ((64, 64, 64), (48, 48, 48)):
        factors = [-0.5j * (lambda h: h + h.conj().T)(crand(rng, (n, n))) / n for n in shape]
        cache = km.prepare(km.KroneckerOp(tuple(factors)), 0.1)
        u = crand(rng, shape)
        st = dist.LocalStepper(dv.to_device(u, np.complex128, DEV), cache.device_exps((np.complex128,) * 3, DEV))
        st.run(3)
        check(f"paired steps {shape}", dv.to_host(st.a),
              orc.step(cache.exps, orc.step(cache.exps, orc.step(cache.exps, u))), 1e-12)
    # float32 fiber pairs on the tcgen05 kernel (large-state route)
    shape = (256, 256, 128)
    u = np.asfortranarray(rng.standard_normal(shape).astype(np.float32))
    mats = [(rng.standard_normal((n, n)) / np.sqrt(n)).astype(np.float32) for n in shape]
    got = km.tucker(dv.to_device(u, np.float32, DEV), mats)
    check("float32 fiber pairs", dv.to_host(got), orc.tucker(u.astype(np.float64), [m.astype(np.float64) for m in mats]),
          1e-5)


FAMILIES = {"tma": fam_tma, "streamk": fam_streamk, "cpasync": fam_cpasync, "tc32": fam_tc32, "peer": fam_peer,
            "misc": fam_misc, "plane": fam_plane}


def main():
    names = sys.argv[1:] or list(FAMILIES)
    rng = np.random.default_rng(0)
    for name in names:
        t0 = time.time()
        FAMILIES[name](rng)
        torch.cuda.synchronize()
        print(f"[{name}] done in {time.time() - t0:.1f} s", flush=True)
    print("sanitize cases: all ok", flush=True)


if __name__ == "__main__":
    main()
