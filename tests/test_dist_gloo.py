"""World-size-2 gloo test of the multi-rank batch path (CPU only): shards are
disjoint and cover the batch, every rank gets the full result equal to the
serial oracle, and the max-over-ranks reduce returns the slowest rank's time."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1603_09337_b200.dist import shard_range


def test_shard_range_partitions():
    for n in range(0, 23):
        for world in range(1, 6):
            covered = []
            for r in range(world):
                a, b = shard_range(n, r, world)
                assert 0 <= a <= b <= n
                covered.extend(range(a, b))
            assert covered == list(range(n))
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import oracle as O
    from paper_1603_09337_b200 import workloads as W
    from paper_1603_09337_b200.dist import hasf_sharded, max_over_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(5)
    imgs = np.stack([W.random_image(rng, 24, 40, 0.5) for _ in range(5)])   # uneven: 3 + 2
    out = hasf_sharded(imgs, 2, fn=lambda x, r, adj: O.hasf_batch(x, r, adj.fg, threads=1))
    t = max_over_ranks(10.0 + rank)
    q.put((rank, out, t))
    dist.destroy_process_group()


def test_two_rank_gloo_batch():
    import oracle as O
    from paper_1603_09337_b200 import workloads as W
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(5)
    imgs = np.stack([W.random_image(rng, 24, 40, 0.5) for _ in range(5)])
    want = O.hasf_batch(imgs, 2, 8, threads=1)
    for rank, out, t in res:
        assert np.array_equal(out, want), rank
        assert t == 11.0


def test_pack_rows_is_p4_layout():
    import torch
    from paper_1603_09337_b200.dist import pack_rows, unpack_rows
    rng = np.random.default_rng(9)
    for w in (1, 7, 8, 13, 40):
        a = (rng.random((3, 4, w)) < 0.5).astype(np.uint8)
        p = pack_rows(torch.from_numpy(a))
        assert np.array_equal(p.numpy(), np.packbits(a, axis=2))
        assert np.array_equal(unpack_rows(p, w).numpy(), a)
