"""Image-level data parallelism.

Each rank (one process per GPU) owns a contiguous block of whole images and
their pyramids; the data path has no collective.  The only exchange is the
final detection gather: an all_gather of per-rank record counts, then of
the fixed-size records padded to the largest count, over NCCL (gloo on CPU
for the tests).
"""

import numpy as np

from ._lib import DETECTION

__all__ = ["shard", "gather_detections"]


def shard(n_items, world, rank):
    """Contiguous balanced block of ``range(n_items)`` owned by ``rank``."""
    base, extra = divmod(int(n_items), int(world))
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def gather_detections(records, group=None, device=None):
    """All ranks receive every rank's detection records (structured array of
    ``DETECTION``), concatenated in rank order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = torch.device("cpu") if device is None else torch.device(device)
    recs = np.ascontiguousarray(records, dtype=DETECTION)
    count = torch.tensor([len(recs)], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(count) for _ in range(world)]
    dist.all_gather(counts, count, group=group)
    counts = [int(c.item()) for c in counts]
    width = max(max(counts), 1) * DETECTION.itemsize
    buf = torch.zeros(width, dtype=torch.uint8, device=dev)
    raw = recs.view(np.uint8).reshape(-1)
    if raw.size:
        buf[: raw.size] = torch.from_numpy(raw.copy()).to(dev)
    bufs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf, group=group)
    out = [b[: c * DETECTION.itemsize].cpu().numpy().view(DETECTION) for b, c in zip(bufs, counts)]
    return np.concatenate(out) if out else np.zeros(0, dtype=DETECTION)
