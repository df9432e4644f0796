"""Generate the golden vectors in tests/golden/*.npz from the REFERENCE itself.

Run in the dev container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array stored here is an input to, or an output of, a reference
(kronmode 0.1.0) function, named by that function.  The fixtures travel with
the repo; no test reads /root/reference at run time.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("KRONMODE_REF", "/root/reference/pkg/src"))

from kronmode import fd, hermite, kron, problems, tensor  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def crand(rng, shape, dtype=np.complex128):
    a = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    return np.asfortranarray(a.astype(dtype))


def rrand(rng, shape, dtype=np.float64):
    return np.asfortranarray(rng.standard_normal(shape).astype(dtype))


def mumode_cases():
    rng = np.random.default_rng(20261018)
    out = {}
    cases = [
        ("c128_3d_m1", crand(rng, (7, 5, 6)), crand(rng, (4, 7)), 1),
        ("c128_3d_m2", crand(rng, (7, 5, 6)), crand(rng, (9, 5)), 2),
        ("c128_3d_m3", crand(rng, (7, 5, 6)), crand(rng, (6, 6)), 3),
        ("c128_sq_m1", crand(rng, (33, 17, 9)), crand(rng, (33, 33)), 1),
        ("c128_sq_m2", crand(rng, (33, 17, 9)), crand(rng, (17, 17)), 2),
        ("c128_sq_m3", crand(rng, (33, 17, 9)), crand(rng, (9, 9)), 3),
        ("f64_2d_m1", rrand(rng, (5, 6)), rrand(rng, (5, 5)), 1),
        ("f64_2d_m2", rrand(rng, (5, 6)), rrand(rng, (3, 6)), 2),
        ("c64_3d_m2", crand(rng, (8, 8, 8), np.complex64), crand(rng, (8, 8), np.complex64), 2),
        ("f32_2d_m1", rrand(rng, (5, 6), np.float32), rrand(rng, (5, 5), np.float32), 1),
        ("real_u_cplx_L", rrand(rng, (3, 4)), crand(rng, (4, 4)), 2),
        ("cplx_u_real_L", crand(rng, (6, 4, 3)), rrand(rng, (6, 6)), 1),
        ("c128_4d_m3", crand(rng, (2, 3, 4, 5)), crand(rng, (4, 4)), 3),
        ("c128_1d", crand(rng, (9,)), crand(rng, (9, 9)), 1),
        ("c128_ext1", crand(rng, (1, 7, 1)), crand(rng, (2, 1)), 1),
    ]
    for name, u, mat, mu in cases:
        out[f"{name}__u"] = u
        out[f"{name}__mat"] = mat
        out[f"{name}__mu"] = np.array(mu)
        out[f"{name}__out"] = tensor.mu_mode_product(u, mat, mu)
    # tucker with a skipped slot, and the identity case
    u = crand(rng, (6, 5, 4))
    mats = [crand(rng, (6, 6)), None, crand(rng, (3, 4))]
    out["tucker_none__u"] = u
    out["tucker_none__m0"] = mats[0]
    out["tucker_none__m2"] = mats[2]
    out["tucker_none__out"] = tensor.tucker(u, mats)
    return out


def step_cases():
    out = {}
    # the headline construction at n=16
    n = 16
    rng = np.random.default_rng(0)
    u = np.asfortranarray(rng.standard_normal((n,) * 3) + 1j * rng.standard_normal((n,) * 3))
    d2 = fd.heat_factors(n, 2).factors[0]
    cache = kron.prepare(kron.KroneckerOp((1j * d2,) * 3), 0.01)
    out["schrod16__u"] = u
    out["schrod16__d2"] = d2
    for i, e in enumerate(cache.exps):
        out[f"schrod16__e{i}"] = e
    out["schrod16__out"] = kron.step(cache, u)
    v = u
    for _ in range(10):
        v = kron.step(cache, v)
    out["schrod16__out10"] = v
    # heat step (real)
    hop = fd.heat_factors(n, 2)
    hcache = kron.prepare(hop, 0.1)
    x = 2 * np.pi * np.arange(n) / n
    c = np.cos(x)
    u0 = np.asfortranarray(c[:, None, None] + c[None, :, None] + c[None, None, :])
    out["heat16__u"] = u0
    out["heat16__e0"] = hcache.exps[0]
    out["heat16__out"] = kron.step(hcache, u0)
    out["heat16__error"] = np.array(problems.heat3d_run(16).error)
    out["heat200__error"] = np.array(1.0)  # filled by the closed form in the test
    return out


def hermite_cases():
    out = {}
    k = 12
    b = hermite.hermite_basis(k)
    bases = (b,) * 3
    rng = np.random.default_rng(5)
    vals = crand(rng, (k, k, k))
    out["herm12__nodes"] = b.nodes
    out["herm12__w"] = b.mod_weights
    out["herm12__phi"] = b.phi
    out["herm12__values"] = vals
    out["herm12__forward"] = hermite.forward_transform(bases, vals)
    out["herm12__inverse"] = hermite.inverse_transform(bases, out["herm12__forward"])
    pts = [np.linspace(-2, 2, 7), np.linspace(-1, 3, 5), np.array([0.0, 0.5])]
    out["herm12__pts0"], out["herm12__pts1"], out["herm12__pts2"] = pts
    out["herm12__inverse_pts"] = hermite.inverse_transform(bases, out["herm12__forward"], eval_points=pts)
    for kk in (16, 64):
        bb = hermite.hermite_basis(kk)
        out[f"basis{kk}__nodes"] = bb.nodes
        out[f"basis{kk}__w"] = bb.mod_weights
        out[f"basis{kk}__phi"] = bb.phi
    # HKP: forward, step with ti potentials, inverse (problems.py:314-342 structure)
    kb = hermite.hermite_basis(10)
    psi0 = problems.schrodinger_initial_state((kb.nodes,) * 3)
    op = kron.KroneckerOp(tuple(hermite.hamiltonian_factor(kb, v) for v in problems.ti_potentials()))
    cache = kron.prepare(op, 1.0)
    c0 = hermite.forward_transform((kb,) * 3, psi0)
    ct = kron.step(cache, c0)
    out["hkp10__psi0"] = psi0
    for i, e in enumerate(cache.exps):
        out[f"hkp10__e{i}"] = e
    out["hkp10__c0"] = c0
    out["hkp10__ct"] = ct
    out["hkp10__values"] = hermite.inverse_transform((kb,) * 3, ct)
    # Magnus (problems.py:397-420) at k=8
    basis, c0m, cm = problems.hkmp_solve(8, T=0.5, steps=4)
    out["hkmp8__c0"] = c0m
    out["hkmp8__out"] = cm
    return out


def gpe_cases():
    out = {}
    n = 16
    grids, lin_op, weights = problems.gpe_setup(n)
    psi = problems.vortex_pair_state(grids)
    for ax, w in enumerate(weights):
        psi = psi * np.sqrt(w).reshape((1,) * ax + (n,) + (1,) * (2 - ax))
    psi = np.asfortranarray(psi)
    tau = 0.1
    cache = kron.prepare(lin_op, tau)
    out["gpe16__psi0"] = psi
    for i in range(3):
        out[f"gpe16__w{i}"] = weights[i]
        out[f"gpe16__e{i}"] = cache.exps[i]
        out[f"gpe16__a{i}"] = lin_op.factors[i]
        out[f"gpe16__x{i}"] = grids[i].points
    p1 = problems.gpe_strang_step(cache, weights, psi, tau)
    out["gpe16__out1"] = p1
    p = p1
    for _ in range(4):
        p = problems.gpe_strang_step(cache, weights, p, tau)
    out["gpe16__out5"] = p
    # single-precision state goes through the same call
    cache64 = kron.PropagatorCache(tau, tuple(e.astype(np.complex64) for e in cache.exps))
    out["gpe16c64__out1"] = problems.gpe_strang_step(cache64, weights, psi.astype(np.complex64), tau)
    return out


def builder_cases():
    out = {}
    for p in (2, 4):
        out[f"heat_d2_n16_p{p}"] = fd.heat_factors(16, p).factors[0]
    out["heat_d2_n16_pinf"] = fd.heat_factors(16, np.inf).factors[0]
    pf = fd.pipeflow_factors(16)
    out["pipe16__a0"], out["pipe16__a1"] = pf.factors
    return out


def main():
    for name, fn in [("mumode", mumode_cases), ("step", step_cases), ("hermite", hermite_cases),
                     ("gpe", gpe_cases), ("builders", builder_cases)]:
        data = fn()
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **data)
        print(f"{path}: {len(data)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
