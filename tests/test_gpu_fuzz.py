"""A bounded run of the randomised parity sweep (tools/fuzz_parity.py): random shapes (ragged,
tiny, TMA-sized), dtype mixes, directions, None slots, kernel policies and paired small steps,
every case against the CPU oracle.  ~45 s on a B200; the long runs are in profiles/r02p_fuzz.log."""

import io
import os
import sys
from contextlib import redirect_stdout

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_randomised_parity_sweep():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import fuzz_parity

    buf = io.StringIO()
    with redirect_stdout(buf):
        fuzz_parity.main(budget=45.0, seed=2026)
    out = buf.getvalue()
    summary = out.strip().splitlines()[-1]
    assert "failures 0" in summary, out[-4000:]
