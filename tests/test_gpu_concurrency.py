"""A Capt is safe for any number of concurrent readers (ref tree.py:67-71):
host threads issuing host-buffer queries (CAPT_HOST_IO, the two-stream
chunked pipeline above 4 M spheres) and device queries on their own streams
against one tree at the same time get exactly the single-threaded results,
including a first_bad report that belongs to their own batch."""

import threading

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2406_02807_b200")
from paper_2406_02807_b200 import workloads as W  # noqa: E402
from paper_2406_02807_b200.query import _host_inputs, _host_query  # noqa: E402


def test_concurrent_host_io_queries():
    cloud = W.cfg1_cloud()
    tree = P.construct(P.PointCloud(cloud), P.BuildParams(0.02, 0.08))
    ref = O.construct(cloud, 0.02, 0.08)
    n = (4 << 20) + (1 << 20)  # > one 4 M-sphere pipeline chunk
    batches = []
    for t in range(4):
        c, r = W.cfg1_queries(cloud, n_groups=n // 8, seed=500 + t)
        if t == 3:  # one batch with an out-of-band radius late in the batch
            r = r.copy()
            r[n - 12345] = np.float32(0.5)
        batches.append((c, r))
    exp = [O.collides_groups(ref, c, r, 8) for c, r in batches[:3]]
    results = [None] * 4
    errors = []

    def run(t):
        try:
            c, r = batches[t]
            cc, rr, f64 = _host_inputs(tree, c, r)
            for _ in range(3):
                bits, _, bad = _host_query(tree, cc, rr, f64, 8, None, True, t == 3)
            results[t] = (bits, bad)
        except Exception as exc:  # noqa: BLE001
            errors.append(exc)

    th = [threading.Thread(target=run, args=(t,)) for t in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for t in range(3):
        assert results[t][1] == -1
        assert np.array_equal(results[t][0], exp[t]), t
    assert results[3][0] is None and results[3][1] == n - 12345


def test_concurrent_device_queries_on_streams():
    torch = pytest.importorskip("torch")
    cloud = W.cfg3_cloud(n=32768, n_comp=8, seed=9)
    tree = P.construct(P.PointCloud(cloud), P.BuildParams(0.01, 0.1))
    ref = O.construct(cloud, 0.01, 0.1)
    data = [W.cfg3_queries(1 << 21, seed=900 + t) for t in range(4)]
    exp = [O.collides_many(ref, c, r) for c, r in data]
    outs = [None] * 4
    errors = []

    def run(t):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                cd = torch.from_numpy(data[t][0]).cuda()
                rd = torch.from_numpy(data[t][1]).cuda()
                for _ in range(5):
                    w = P.query_bits(tree, cd, rd, 1, stream=s.cuda_stream)
                s.synchronize()
                outs[t] = w.cpu().numpy()
        except Exception as exc:  # noqa: BLE001
            errors.append(exc)

    th = [threading.Thread(target=run, args=(t,)) for t in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    from oracle.parity import unpack_words
    for t in range(4):
        assert np.array_equal(unpack_words(outs[t], len(exp[t])), exp[t]), t
