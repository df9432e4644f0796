"""GPU: seeded random shapes against the oracle — every dtype mix, every direction,
ragged extents (not multiples of any tile), rectangular factors, size-1 directions,
d = 1..4, with and without the accumulate epilogue.  The kernel choice is
size dependent, so sweeping shapes sweeps the launch rules (cp.async tile sizes, the
TMA eligibility, stream-K) as well as the edge handling of each kernel."""

import numpy as np
import pytest

import paper_2103_01691_b200 as km
from oracle import kronmode_oracle as orc
from paper_2103_01691_b200 import _device as dv
from paper_2103_01691_b200 import _native

pytestmark = pytest.mark.gpu

TOL = {np.dtype(np.complex128): 1e-12, np.dtype(np.float64): 1e-12,
       np.dtype(np.complex64): 1e-5, np.dtype(np.float32): 1e-5}
PAIRS = [(np.complex128, np.complex128), (np.complex128, np.float64), (np.float64, np.complex128),
         (np.float64, np.float64), (np.complex64, np.complex64), (np.complex64, np.float32),
         (np.float32, np.complex64), (np.float32, np.float32)]


def _rand(rng, shape, dt):
    x = rng.standard_normal(shape)
    if np.dtype(dt).kind == "c":
        x = x + 1j * rng.standard_normal(shape)
    return np.asfortranarray(x.astype(dt))


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    d = int(rng.integers(1, 5))
    hi = {1: 3000, 2: 300, 3: 70, 4: 24}[d]
    shape = tuple(int(rng.integers(1, hi)) for _ in range(d))
    mu = int(rng.integers(1, d + 1))
    m = int(rng.integers(1, 2 * shape[mu - 1] + 2))
    udt, ldt = PAIRS[seed % len(PAIRS)]
    return rng, shape, mu, m, udt, ldt


@pytest.mark.parametrize("seed", range(48))
def test_random_mu_mode_product(seed):
    rng, shape, mu, m, udt, ldt = _case(seed)
    u = _rand(rng, shape, udt)
    mat = (_rand(rng, (m, shape[mu - 1]), ldt) / np.sqrt(shape[mu - 1])).astype(ldt)  # keep the factor's dtype
    got = km.mu_mode_product(u, mat, mu)
    want = orc.mu_mode_product(u, mat, mu)
    assert got.shape == want.shape and got.dtype == want.dtype
    assert orc.rel_l2(got, want) <= TOL[want.dtype], (shape, mu, m, udt, ldt)


@pytest.mark.parametrize("seed", range(16))
def test_random_accumulate_into_output(seed):
    """km_mumode_split(accumulate = 1) on random plain layouts: out = out0 + u x_mu L."""
    import torch

    rng, shape, mu, m, udt, ldt = _case(seed)
    cdt = np.result_type(udt, ldt)
    u = _rand(rng, shape, udt)
    mat = (_rand(rng, (m, shape[mu - 1]), ldt) / np.sqrt(shape[mu - 1])).astype(ldt)
    out_shape = shape[:mu - 1] + (m,) + shape[mu:]
    out0 = _rand(rng, out_shape, cdt)
    dev = torch.device("cuda", 0)
    ut = dv.to_device(u, udt, dev)
    lt = torch.from_numpy(np.ascontiguousarray(mat)).to(dev)
    ot = dv.to_device(out0, cdt, dev)
    nl = int(np.prod(shape[:mu - 1], dtype=np.int64))
    nr = int(np.prod(shape[mu:], dtype=np.int64))
    n = shape[mu - 1]
    _native.check(_native.lib().km_mumode_split(
        ut.data_ptr(), dv.code(udt), lt.data_ptr(), dv.code(ldt), ot.data_ptr(), m, nl, n, nr, n, 0, m, 0, 1, None,
        dv.stream_ptr(dev)))
    want = out0 + orc.mu_mode_product(u, mat, mu)
    assert orc.rel_l2(dv.to_host(ot), want) <= TOL[np.dtype(cdt)], (shape, mu, m, udt, ldt)
