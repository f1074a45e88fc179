"""Host logic of the engine drop-in (no device): packer, parents, expand, merge, stop, finalize."""

import numpy as np
import pytest

from paper_2512_02281_b200.ann_graph import NeighborGraph
from paper_2512_02281_b200.engine import (
    CONVERGED,
    DUMMY,
    FINISHED,
    CandidateEntry,
    EngineConfig,
    SearchRequestState,
    build_task_array,
    check_early_stop,
    expand,
    finalize,
    scatter_merge,
    seed_entry_ids,
    select_parents,
)


def state_of(entries, rid=0, extends=0):
    st = SearchRequestState(request_id=rid, query=np.zeros(1), k=1)
    for i, d, x in entries:
        st.top_m.append(CandidateEntry(id=i, dist=d, expanded=x))
        st.visited.add(i)
    st.extends_done = extends
    return st


def test_seed_ids():  # engine.py:136-143
    assert seed_entry_ids(100, 4) == [0, 25, 50, 75]
    assert seed_entry_ids(100, 1) == [0]
    assert seed_entry_ids(3, 8) == [0, 1, 2]


def test_task_array_padding_and_split():  # engine.py:208-226, acceptance C3 accounting
    assert build_task_array({}, 8) == [] and build_task_array({0: []}, 8) == []
    b = build_task_array({0: [1, 2, 3, 4, 5]}, 8)
    assert len(b) == 1 and b[0].real_count == 5
    assert [t.owner for t in b[0].tasks[5:]] == [DUMMY] * 3 and [t.candidate for t in b[0].tasks[5:]] == [0] * 3
    b = build_task_array({0: list(range(9)), 1: list(range(8))}, 8)
    assert [x.real_count for x in b] == [8, 8, 1] and all(len(x.tasks) == 8 for x in b)
    b = build_task_array({3: [30], 1: [10], 2: [20]}, 8)
    assert [t.owner for t in b[0].tasks[:3]] == [1, 2, 3]


def test_parents_and_expand():
    st = state_of([(5, 0.1, True), (7, 0.2, False)])
    assert select_parents(st, 2) == [7]
    assert select_parents(state_of([(5, 0.1, True)]), 2) == []
    g = NeighborGraph(degree=2, adjacency=np.array([[1, 2], [0, 2], [0, 1]], dtype=np.uint32))
    st = state_of([(1, 1.0, False), (2, 4.0, False)])
    assert expand(st, g, [1, 2]) == [0]  # shared neighbor emitted once
    st = state_of([(1, 1.0, False)])
    with pytest.raises(RuntimeError):
        expand(st, g, [2])


def test_merge_and_stop_and_finalize():
    st = state_of([(1, 0.1, False), (2, 0.5, False)])
    rep = scatter_merge(st, [(3, 0.3)], m=2)
    assert rep.changed and rep.inserted_count == 1 and [(e.id, e.dist) for e in st.top_m] == [(1, 0.1), (3, 0.3)]
    assert not scatter_merge(st, [(4, 0.9)], m=2).changed
    with pytest.raises(RuntimeError):
        scatter_merge(st, [(1, 0.1)], m=4)
    cfg = EngineConfig(m=4, p=1, entry_count=1, batch_capacity=4, stop_streak=2, max_extends=50)
    st = state_of([(1, 0.1, False)])
    check_early_stop(st, cfg, changed=False)
    assert st.no_change_streak == 1 and st.status != CONVERGED
    assert check_early_stop(st, cfg, changed=False) == CONVERGED
    st = state_of([(1, 0.1, True), (2, 0.5, True)])
    st.status = CONVERGED
    assert [n.id for n in finalize(st, 2)] == [1, 2] and st.status == FINISHED
    with pytest.raises(RuntimeError):
        finalize(st, 1)


def test_config_validation():
    with pytest.raises(ValueError):
        EngineConfig(m=2, p=3)
    with pytest.raises(ValueError):
        EngineConfig(batch_capacity=0)


def test_ivf_file_roundtrip_and_errors(tmp_path):
    """IVF index file (ivf.py write_ivf / read_ivf): exact round trip, corrupt files rejected."""
    import numpy as np
    import pytest

    from paper_2512_02281_b200.ivf import read_ivf, write_ivf

    rng = np.random.default_rng(0)
    cen = rng.standard_normal((7, 5)).astype(np.float32)
    asg = rng.integers(0, 7, 100).astype(np.int32)
    p = tmp_path / "x.ivf"
    write_ivf(str(p), cen, asg)
    c2, a2 = read_ivf(str(p))
    assert np.array_equal(c2, cen) and np.array_equal(a2, asg)
    raw = p.read_bytes()
    (tmp_path / "short.ivf").write_bytes(raw[:-4])
    with pytest.raises(ValueError):
        read_ivf(str(tmp_path / "short.ivf"))
    (tmp_path / "magic.ivf").write_bytes(b"XXXXXXXX" + raw[8:])
    with pytest.raises(ValueError):
        read_ivf(str(tmp_path / "magic.ivf"))
    with pytest.raises(ValueError):
        write_ivf(str(tmp_path / "bad.ivf"), cen, np.array([0, 9], np.int32))
