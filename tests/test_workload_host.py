"""Host-side workload generation: chunked databases and per-rank row ranges."""

import numpy as np
import pytest

from paper_2512_02281_b200.workload import gen_rows_chunked, gen_vectors_chunked


def test_rows_chunked_equals_slices_of_the_whole():
    whole = gen_vectors_chunked(1000, 8, 5, chunk=64)
    for lo, hi in [(0, 1000), (13, 500), (64, 128), (999, 1000), (100, 100), (5, 63), (0, 1)]:
        assert np.array_equal(gen_rows_chunked(lo, hi, 8, 5, chunk=64), whole[lo:hi]), (lo, hi)
    # the same rows whatever the total size drawn after them (chunk prefix property)
    assert np.array_equal(gen_vectors_chunked(700, 8, 5, chunk=64), whole[:700])


def test_rows_chunked_shards_tile_the_database():
    from paper_2512_02281_b200.sharded import shard_bounds

    whole = gen_vectors_chunked(3001, 4, 9, chunk=128)
    parts = [gen_rows_chunked(*shard_bounds(3001, 7, r), 4, 9, chunk=128) for r in range(7)]
    assert np.array_equal(np.concatenate(parts), whole)


def test_rows_chunked_rejects_bad_ranges():
    with pytest.raises(ValueError):
        gen_rows_chunked(5, 3, 4, 1)
    with pytest.raises(ValueError):
        gen_rows_chunked(-1, 3, 4, 1)
