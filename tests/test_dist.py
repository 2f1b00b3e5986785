"""Multi-rank host logic on CPU (gloo, world size 2): image sharding and the
final detection gather -- the only collective of the path."""

import os
import socket

import numpy as np
import pytest

from paper_1707_03268_b200 import _lib
from paper_1707_03268_b200.dist import gather_detections, shard


def test_shard_is_a_balanced_partition():
    for n in (1, 7, 64, 65):
        for world in (1, 2, 3, 8):
            blocks = [list(shard(n, world, r)) for r in range(world)]
            assert sum(blocks, []) == list(range(n))
            sizes = [len(b) for b in blocks]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = list(shard(5, world, rank))
    recs = np.zeros(len(mine) * (rank + 1), dtype=_lib.DETECTION)
    for i, r in enumerate(recs):
        recs[i]["image"] = mine[i % len(mine)]
        recs[i]["rank_tag" if False else "level"] = rank
        recs[i]["score"] = rank * 100 + i
        recs[i]["parts"][:] = np.arange(16) + rank
    out = gather_detections(recs)
    q.put((rank, out.tobytes()))
    dist.destroy_process_group()


def test_gather_detections_world2_gloo():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = np.frombuffer(res[0], dtype=_lib.DETECTION)
    b = np.frombuffer(res[1], dtype=_lib.DETECTION)
    assert np.array_equal(a, b)
    # rank 0 owns images 0..2 (3 records), rank 1 owns 3..4 (2 images x 2 = 4 records)
    assert len(a) == 3 + 4
    assert list(a["level"]) == [0, 0, 0, 1, 1, 1, 1]
    assert list(a["score"][3:]) == [100, 101, 102, 103]
    assert np.all(a["parts"][3:] == np.arange(16) + 1)
