"""Multi-process host logic of the N>1 path with world_size 2 over gloo (CPU):
sharding, the byte broadcast used for tree replication, and the final
counter all-reduce -- checked against the oracle on the whole batch."""

import os
import socket

import numpy as np
import pytest

from paper_2406_02807_b200.dist import shard_range


def test_shard_range_covers_and_aligns():
    for n in (0, 1, 31, 32, 33, 1000, 4096 * 8 + 5):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, world, r, align=32) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            for a, b in spans[:-1]:
                assert a % 32 == 0 and b % 32 == 0 or b == n
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2406_02807_b200 import workloads as W
    from paper_2406_02807_b200.dist import broadcast_bytes, reduce_counters

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # "tree replica": rank 0 serialises, every rank receives identical bytes
        cloud = W.cfg1_cloud(2048, seed=4)
        if rank == 0:
            t = O.construct(cloud, 0.02, 0.08)
            blob = np.concatenate([t["tests"].view(np.uint8), t["aff_lo"].ravel().view(np.uint8),
                                   t["aff_hi"].ravel().view(np.uint8),
                                   t["offsets"].view(np.uint8), t["aff_values"].view(np.uint8)])
            buf = torch.from_numpy(blob.copy())
        else:
            buf = None
        buf = broadcast_bytes(buf, src=0)
        n = 2048
        raw = buf.numpy()
        sizes = [4 * (n - 1), 12 * n, 12 * n, 8 * (n + 1)]
        cut = np.cumsum([0] + sizes)
        offsets = raw[cut[3]:cut[4]].view(np.int64)
        tree = dict(k=3, n=n, n_points=n, r_min=0.02, r_max=0.08,
                    tests=raw[cut[0]:cut[1]].view(np.float32),
                    aff_lo=raw[cut[1]:cut[2]].view(np.float32).reshape(n, 3),
                    aff_hi=raw[cut[2]:cut[3]].view(np.float32).reshape(n, 3),
                    offsets=offsets, aff_values=raw[cut[4]:].view(np.float32))
        # weak scaling: each rank its own seeded batch; counters all-reduced
        c, r = W.cfg1_queries(cloud, n_groups=4096, seed=101 + 1000 * rank)
        g, cnt = O.collides_groups(tree, c, r, 8, return_counters=True)
        counters = torch.tensor([cnt[0], 0, cnt[2], 0, cnt[1], 0], dtype=torch.int64)
        reduce_counters(counters)
        q.put((rank, counters.tolist(), int(g.sum())))
    finally:
        dist.destroy_process_group()


def test_two_rank_broadcast_and_counter_reduce():
    import torch.multiprocessing as mp

    from oracle import oracle as O
    from paper_2406_02807_b200 import workloads as W

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # both ranks see the same global sums, equal to the single-process oracle
    assert res[0][1] == res[1][1]
    cloud = W.cfg1_cloud(2048, seed=4)
    tree = O.construct(cloud, 0.02, 0.08)
    tot = np.zeros(3, np.int64)
    for rank in range(2):
        c, r = W.cfg1_queries(cloud, n_groups=4096, seed=101 + 1000 * rank)
        tot += np.array(O.collides_groups(tree, c, r, 8, return_counters=True)[1])
    assert res[0][1][0] == tot[0] and res[0][1][4] == tot[1] and res[0][1][2] == tot[2]
    assert res[0][2] + res[1][2] == tot[0]
