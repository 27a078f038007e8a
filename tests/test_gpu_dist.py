"""The N > 1 product path with world_size 2 over gloo, both ranks on cuda:0
(no kernel waits on another rank; the exchanges are host-side gloo
collectives): rank 0 builds the tree on the device, its position-independent
slab is broadcast as bytes, rank 1 adopts the received slab as its replica
(Capt.from_slab(adopt=True), no second copy), each rank queries its
dist.shard_range share of ONE global batch (strong scaling) through the
product path, the counters are summed with reduce_counters, and the
gathered verdict words equal the oracle's for the whole batch
(query.py:184-219, 126-167)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, L, q):
    import torch
    import torch.distributed as dist

    import paper_2406_02807_b200 as P
    from paper_2406_02807_b200 import workloads as W
    from paper_2406_02807_b200.dist import broadcast_bytes, reduce_counters, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        cloud = W.cfg1_cloud()
        if rank == 0:
            tree = P.construct(P.PointCloud(cloud), P.BuildParams(0.02, 0.08), device=0)
            blob = tree.slab_tensor().cpu()
        else:
            tree, blob = None, None
        blob = broadcast_bytes(blob, src=0)  # gloo: CPU bytes
        if rank != 0:
            tree = P.Capt.from_slab(blob.cuda(), adopt=True)
        c, r = W.cfg1_queries(cloud, n_groups=1 << 17, seed=77)  # the global batch
        if L == 1:
            c, r = c[: (1 << 19)], r[: (1 << 19)]
        g0, g1 = shard_range(len(r) // L, world, rank, align=32)
        cd = torch.from_numpy(c[g0 * L: g1 * L]).cuda()
        rd = torch.from_numpy(r[g0 * L: g1 * L]).cuda()
        words = P.query_bits(tree, cd, rd, L)
        counters = torch.zeros(6, dtype=torch.int64, device="cuda")
        P.query_bits(tree, cd, rd, L, counters=counters)
        tot = reduce_counters(counters.cpu())
        q.put((rank, g0, g1, words.cpu().numpy().tobytes(), tot.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("L", [8, 1])
def test_two_ranks_product_path(L):
    import torch.multiprocessing as mp

    from oracle import oracle as O
    from oracle.parity import unpack_words
    from paper_2406_02807_b200 import workloads as W

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(rk, 2, port, L, q)) for rk in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cloud = W.cfg1_cloud()
    ref = O.construct(cloud, 0.02, 0.08)
    c, r = W.cfg1_queries(cloud, n_groups=1 << 17, seed=77)
    if L == 1:
        c, r = c[: (1 << 19)], r[: (1 << 19)]
    units = len(r) // L
    assert res[0][1] == 0 and res[0][2] == res[1][1] and res[1][2] == units
    got = np.concatenate([unpack_words(np.frombuffer(w, np.uint32), b - a)
                          for _, a, b, w, _ in res])
    if L == 1:
        exp, cnt = O.collides_many(ref, c, r, return_counters=True)
        assert res[0][4][1] == cnt[1]  # boundary spheres, summed over ranks
        assert res[0][4][2] == cnt[2]  # counted tests
    else:
        exp, cnt = O.collides_groups(ref, c, r, L, return_counters=True)
        assert res[0][4][2] == cnt[2] and res[0][4][4] == cnt[1]
    assert np.array_equal(got, exp)
    assert res[0][4] == res[1][4] and res[0][4][0] == int(exp.sum())
