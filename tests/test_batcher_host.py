"""RetrievalBatcher.submit validation (host only, no device): a bad submission
raises at submit time and never reaches a batch."""

import numpy as np
import pytest

from paper_2512_02281_b200.batcher import RetrievalBatcher


class _Index:
    dim, nlist = 4, 32


def test_submit_rejects_bad_requests_and_keeps_explicit_values():
    b = RetrievalBatcher(_Index())
    with pytest.raises(ValueError):
        b.submit(np.array([0.0, np.nan, 0.0, 0.0]))
    with pytest.raises(ValueError):
        b.submit(np.zeros(3))
    with pytest.raises(ValueError):
        b.submit(np.zeros(4), k=0)  # an explicit 0 is an error, not "use the default"
    with pytest.raises(ValueError):
        b.submit(np.zeros(4), nprobe=0)
    with pytest.raises(ValueError):
        b.submit(np.zeros(4), nprobe=33)
    assert b.pending == 0
    b.submit(np.zeros(4), stage="prefill", nprobe=8)
    b.submit(np.zeros(4), k=3)
    assert [(p.k, p.nprobe) for p in b._queue] == [(100, 8), (3, 16)]
