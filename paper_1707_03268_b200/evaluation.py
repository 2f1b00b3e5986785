"""Detection emission downstream of the GPU detectors.

Drop-ins for ``cpdetect.evaluation`` (evaluation.py:47-162): greedy NMS on
root boxes, truth matching and the ROC sweep, with the reference's names,
arguments, tie-breaks and exact IoU arithmetic.  Detection itself (K1-K4 and
the GPU tau-compaction) runs on the device through :func:`detect` /
:func:`dense_detect`; NMS and matching are host-side list operations over
the compacted detections, as the survey allows ("host or GPU NMS").
``nms_records`` applies the same suppression to the batched detection
records of :class:`PyramidScorer` (per image and level, per-component root
extents).
"""

from dataclasses import dataclass

import numpy as np

from .detection import dense_detect, detect
from .errors import ValidationError

__all__ = ["RocPoint", "nms", "nms_records", "match_detections", "roc_eval"]


@dataclass(frozen=True)
class RocPoint:
    """Operating point at threshold ``tau`` (evaluation.py:18-29)."""

    tau: float
    misdetection_rate: float
    false_positives_per_scene: float
    false_positives_per_window: float


def _strongest_first(detections):
    # (-score, level, root): the reference's deterministic order (evaluation.py:53-56)
    return sorted(detections, key=lambda d: (-d.score, d.hypothesis.level, d.hypothesis.root))


def _greedy_keep(y0, x0, hh, ww, iou_threshold):
    """Greedy suppression over boxes already in strongest-first order; returns
    the kept indices.  IoU = integer intersection / integer union in float64,
    0 for an empty union (evaluation.py:36-44)."""
    y1, x1 = y0 + hh, x0 + ww
    area = hh * ww
    kept = []
    for i in range(y0.size):
        if kept:
            k = np.asarray(kept)
            iy = np.maximum(0, np.minimum(y1[i], y1[k]) - np.maximum(y0[i], y0[k]))
            ix = np.maximum(0, np.minimum(x1[i], x1[k]) - np.maximum(x0[i], x0[k]))
            inter = iy * ix
            union = area[i] + area[k] - inter
            iou = np.where(union != 0, inter / np.where(union != 0, union, 1), 0.0)
            if np.any(iou >= iou_threshold):
                continue
        kept.append(i)
    return kept


def nms(detections, root_dims, iou_threshold=0.5):
    """Greedy overlap suppression on root boxes, strongest first; only
    detections on the same level compete (evaluation.py:47-68).  Returns the
    kept detections sorted by (level, root)."""
    ordered = _strongest_first(detections)
    kept = []
    by_level = {}
    for d in ordered:
        by_level.setdefault(d.hypothesis.level, []).append(d)
    h, w = int(root_dims[0]), int(root_dims[1])
    for lvl, ds in by_level.items():
        y0 = np.array([d.hypothesis.root[0] for d in ds], dtype=np.int64)
        x0 = np.array([d.hypothesis.root[1] for d in ds], dtype=np.int64)
        hh = np.full(y0.size, h, dtype=np.int64)
        ww = np.full(y0.size, w, dtype=np.int64)
        kept.extend(ds[i] for i in _greedy_keep(y0, x0, hh, ww, iou_threshold))
    kept.sort(key=lambda d: (d.hypothesis.level, d.hypothesis.root))
    return kept


def nms_records(records, root_dims, iou_threshold=0.5):
    """NMS over :data:`DETECTION` records of the batched scorer: records of the
    same (image, level) compete, each with its component's root extent
    ``root_dims[component]``; same strongest-first order (score descending,
    then level, ry, rx).  Returns the kept records sorted by
    (image, level, ry, rx)."""
    if len(records) == 0:
        return records
    dims = np.asarray(root_dims, dtype=np.int64).reshape(-1, 2)
    order = np.lexsort((records["rx"], records["ry"], records["level"], -records["score"]))
    recs = records[order]
    keep = []
    seg = recs["image"].astype(np.int64) * 65536 + recs["level"]
    for s in np.unique(seg):
        idx = np.flatnonzero(seg == s)
        r = recs[idx]
        comp = r["component"]
        kept = _greedy_keep(r["ry"].astype(np.int64), r["rx"].astype(np.int64),
                            dims[comp, 0], dims[comp, 1], iou_threshold)
        keep.extend(idx[kept])
    out = recs[np.asarray(keep, dtype=np.int64)]
    return out[np.lexsort((out["rx"], out["ry"], out["level"], out["image"]))]


def match_detections(detections, truths, radius=1):
    """Greedy matching of detections to truths on the same level within
    Chebyshev ``radius``, strongest first; returns (matched, false
    positives) (evaluation.py:71-99)."""
    claimed = [False] * len(truths)
    fps = 0
    for d in _strongest_first(detections):
        dy, dx = d.hypothesis.root
        hit = next((i for i, (lvl, t) in enumerate(truths)
                    if not claimed[i] and lvl == d.hypothesis.level
                    and max(abs(t.root[0] - dy), abs(t.root[1] - dx)) <= radius), None)
        if hit is None:
            fps += 1
        else:
            claimed[hit] = True
    return sum(claimed), fps


def roc_eval(model, scenes, taus, match_radius=1, pruning=False, nms_iou=0.5,
             part_prune_mode="kill"):
    """Threshold sweep over scenes (evaluation.py:102-162): detect once per
    scene at the lowest threshold on the GPU, NMS once, then sweep."""
    taus = sorted(float(t) for t in taus)
    if not taus:
        raise ValidationError("tau grid must not be empty")
    if hasattr(model, "root_cp"):
        root_dims = tuple(model.root_cp.dims)

        def runner(pyr, tau):
            return detect(model, pyr, tau, pruning=pruning, part_prune_mode=part_prune_mode)
    elif hasattr(model, "root"):
        root_dims = np.asarray(model.root).shape

        def runner(pyr, tau):
            return dense_detect(model, pyr, tau)
    else:
        raise ValidationError(f"unsupported model type {type(model).__name__}")
    per_scene, truths_total, windows = [], 0, 0
    for scene in scenes:
        dets, stats = runner(scene.pyramid, taus[0])
        per_scene.append((nms(dets, root_dims, nms_iou), scene.planted))
        truths_total += len(scene.planted)
        windows += stats.positions_examined
    n_scenes = max(1, len(per_scene))
    points = []
    for tau in taus:
        matched = fps = 0
        for kept, truths in per_scene:
            got, fp = match_detections([d for d in kept if d.score >= tau], truths, match_radius)
            matched += got
            fps += fp
        points.append(RocPoint(
            tau=tau,
            misdetection_rate=1.0 - matched / truths_total if truths_total else 0.0,
            false_positives_per_scene=fps / n_scenes,
            false_positives_per_window=fps / windows if windows else 0.0))
    return points
