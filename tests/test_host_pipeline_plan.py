"""CPU: the host pipeline's slab plans (_pipeline._chunks, _input_slabs) tile the
last direction exactly, in order, and shrink at the end as DESIGN.md §2.6 says."""

import pytest

from paper_2103_01691_b200 import _pipeline


def covers(slabs, n):
    start = 0
    for s, size in slabs:
        assert s == start and size >= 1
        start += size
    assert start == n


@pytest.mark.parametrize("n", [1, 2, 7, 20, 64, 100, 128, 256, 257, 512, 1000, 1024])
@pytest.mark.parametrize("parts", [1, 2, 4, 8, 16])
def test_plans_cover_the_extent(n, parts):
    covers(_pipeline._chunks(n, parts), n)
    covers(_pipeline._input_slabs(n, parts), n)
    assert len(_pipeline._input_slabs(n, parts)) <= max(1, min(parts, n))


def test_input_slabs_shrink_geometrically_at_the_end():
    slabs = _pipeline._input_slabs(256, 8)
    assert [size for _, size in slabs[-4:]] == [32, 16, 8, 4]
    assert all(size >= 32 for _, size in slabs[:-4])
    # small extents keep the uniform split
    assert _pipeline._input_slabs(64, 8) == _pipeline._chunks(64, 8)
