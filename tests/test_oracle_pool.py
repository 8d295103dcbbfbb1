"""Pins for the allocator / migration oracle (oracle/pool.py)."""
import numpy as np
import pytest

from oracle import pool as opool


def test_lowest_free_first_and_all_or_nothing():
    p = opool.PagePool(8)
    assert p.alloc(3) == [0, 1, 2]
    assert p.alloc(2) == [3, 4]
    p.release([1, 3])
    assert p.alloc(3) == [1, 3, 5]
    with pytest.raises(opool.NoPages):
        p.alloc(3)                       # only 6, 7 free
    assert p.num_free() == 2             # unchanged by the failed alloc
    assert p.alloc(2) == [6, 7]
    assert p.alloc(0) == []


def test_double_free_rejected_without_side_effects():
    p = opool.PagePool(4)
    p.alloc(2)
    with pytest.raises(opool.InvalidFree):
        p.release([0, 0])
    with pytest.raises(opool.InvalidFree):
        p.release([1, 2])               # page 2 is free
    assert p.num_free() == 2
    p.release([0, 1])
    assert p.num_free() == 4


def test_no_page_owned_twice_random():
    rng = np.random.default_rng(0)
    p = opool.PagePool(64)
    owned = {}
    for step in range(2000):
        if owned and rng.random() < 0.45:
            rid = list(owned)[int(rng.integers(len(owned)))]
            p.release(owned.pop(rid))
        else:
            n = int(rng.integers(0, 12))
            try:
                owned[step] = p.alloc(n)
            except opool.NoPages:
                pass
        allp = sum(owned.values(), [])
        assert len(allp) == len(set(allp))
        assert p.num_free() == 64 - len(allp)


def test_migrate_copies_pages():
    rng = np.random.default_rng(1)
    src_k = rng.standard_normal((10, 2, 16, 4))
    src_v = rng.standard_normal((10, 2, 16, 4))
    dst_k = np.zeros((6, 2, 16, 4))
    dst_v = np.zeros((6, 2, 16, 4))
    pool = opool.PagePool(6)
    pool.alloc(1)                        # page 0 busy
    dst = opool.migrate(src_k, src_v, [7, 2, 9], dst_k, dst_v, pool)
    assert dst == [1, 2, 3]
    for s, d in zip([7, 2, 9], dst):
        assert np.array_equal(dst_k[d], src_k[s]) and np.array_equal(dst_v[d], src_v[s])
    with pytest.raises(opool.NoPages):
        opool.migrate(src_k, src_v, [0, 1, 3], dst_k, dst_v, pool)
    assert pool.num_free() == 2
