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


def test_bench_self_launches_two_ranks_stub_gloo():
    """``bench.py --gpus 2`` without torchrun re-launches itself with two
    ranks (torch.distributed.run on 127.0.0.1); with the stub scorer the
    ranks run gloo on CPU through the same harness: image sharding,
    barrier + max-over-ranks timing, the detection gather and ONE JSON line
    from rank 0 accounting for all 64 images."""
    import hashlib
    import json
    import subprocess
    import sys

    from conftest import REPO

    sys.path.insert(0, REPO)
    import bench

    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--stub",
                        "--steps", "2", "--warmup", "3"], capture_output=True, text=True,
                       timeout=240, cwd=REPO)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["steps"] == 2 and out["warmup"] == 3
    assert out["config"]["images"] == 64
    union = np.concatenate([bench.stub_detections(i) for i in range(64)])
    union = np.sort(union, order=["image", "level", "component", "ry", "rx"])
    g = out["e2e"]["gathered"]
    assert g["detections"] == len(union) == out["e2e"]["detections_per_step"]
    assert g["images"] == 64
    assert g["sha16"] == hashlib.sha256(union.tobytes()).hexdigest()[:16]
    assert out["value"] > 0 and out["e2e"]["value"] > 0
