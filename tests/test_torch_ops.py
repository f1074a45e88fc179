"""torch front end (torch.library ops over the C-ABI): registration and shape
inference on the CPU, results on the GPU equal the Python API's."""

import numpy as np
import pytest
import torch


def test_ops_registered_and_fake_shapes():
    from paper_2512_02281_b200 import torch_ops  # noqa: F401
    from torch._subclasses.fake_tensor import FakeTensorMode

    for name in ("ivf_search", "knn", "merge_topk"):
        assert hasattr(torch.ops.trinity, name)
    with FakeTensorMode():
        q = torch.empty((5, 8), dtype=torch.float64)
        ids, d = torch.ops.trinity.ivf_search(0, q, torch.ones(5, dtype=torch.int32),
                                              torch.ones(5, dtype=torch.int32), 7)
        assert ids.shape == (5, 7) and ids.dtype == torch.int64 and d.dtype == torch.float64
        oi, od = torch.ops.trinity.merge_topk(torch.empty((3, 5, 4), dtype=torch.float64),
                                              torch.empty((3, 5, 4), dtype=torch.int64), 6)
        assert oi.shape == (5, 6) and od.shape == (5, 6)


@pytest.mark.gpu
def test_ops_match_python_api():
    from oracle import trinity_oracle as orc
    from paper_2512_02281_b200 import torch_ops  # noqa: F401
    from paper_2512_02281_b200.ann_graph import VectorStore
    from paper_2512_02281_b200.ivf import IVFFlatIndex
    from paper_2512_02281_b200.workload import gen_matrix

    data = gen_matrix(10_000, 24, 71)
    store = VectorStore(data=data)
    idx = IVFFlatIndex.train(store, nlist=32, iters=3, seed=1)
    qs = gen_matrix(12, 24, 72).astype(np.float64)
    q = torch.from_numpy(qs).cuda()
    k = torch.tensor([10, 3] * 6, dtype=torch.int32)
    npb = torch.tensor([4, 16] * 6, dtype=torch.int32)
    ids, d = torch.ops.trinity.ivf_search(idx.handle.value, q, k, npb, 10)
    ri, rd = idx.search(qs, k.numpy(), npb.numpy())
    assert np.array_equal(ids.cpu().numpy(), ri) and np.array_equal(d.cpu().numpy(), rd)
    bi, bd = torch.ops.trinity.knn(store.device().handle.value, q, torch.full((12,), 5, dtype=torch.int32), 5)
    for i in range(12):
        oi, od = orc.exact_knn(data, qs[i], 5)
        assert np.array_equal(bi[i].cpu().numpy(), oi) and np.array_equal(bd[i].cpu().numpy(), od)
    mi, md = torch.ops.trinity.merge_topk(d.view(2, 6, 10), ids.view(2, 6, 10), 10)
    assert mi.shape == (6, 10)
