"""Drop-in scoring / placement / detection on the B200 (K1-K4).

Mirrors ``cpdetect.detection`` for the pruning-off hot path
(``detection.py:128-616``): same names, arguments, return types, error
classes and messages.  The GPU computes response maps in FP32 and placement
and assembly in FP64 with the reference's exact expression order, so for a
given response map the placed values and argmaxes are bit-identical to
``_placement_grid``.

``detect(..., pruning=True)`` (Algorithm 1, convolution shortening) is the
next tier and raises NotImplementedError here.
"""

import time

import numpy as np

from .correlation import cp_core
from .engine import AssemblyDef, FilterDef, PartDef, Plan, unpack_positions
from .errors import ValidationError, check_feature_map
from .geometry import cp_multiplications, full_multiplications, hypothesis_rect
from .types import Detection, DetectStats, Hypothesis

__all__ = [
    "deformation_penalty",
    "best_part_placement",
    "_placement_grid",
    "detect",
    "dense_detect",
    "score_hypothesis",
    "cp_score_hypothesis",
    "validate",
    "require_valid",
]


def deformation_penalty(deformation, dy, dx):
    """c_dx*dx + c_dy*dy + c_dxx*dx^2 + c_dyy*dy^2 (detection.py:128-131)."""
    cdx, cdy, cdxx, cdyy = deformation
    return cdx * dx + cdy * dy + cdxx * dx * dx + cdyy * dy * dy


def validate(model):
    """Model invariants as a list of violations (model.py:171-201)."""
    out = []
    root = np.asarray(model.root)
    if not np.isfinite(root).all():
        out.append("root: filter contains non-finite values")
    ch = root.shape[2]
    for i, part in enumerate(model.parts):
        name = f"parts[{i}]"
        f = np.asarray(part.filter)
        if not np.isfinite(f).all():
            out.append(f"{name}: filter contains non-finite values")
        if f.shape[2] != ch:
            out.append(f"{name}: filter channel extent {f.shape[2]} differs "
                       f"from root filter channel extent {ch}")
        _, _, cdxx, cdyy = part.deformation
        if cdxx < 0:
            out.append(f"{name}.deformation.c_dxx: must be >= 0, got {cdxx}")
        if cdyy < 0:
            out.append(f"{name}.deformation.c_dyy: must be >= 0, got {cdyy}")
        if part.search_radius < 1:
            out.append(f"{name}.search_radius: must be >= 1, got {part.search_radius}")
    return out


def require_valid(model):
    v = validate(model)
    if v:
        raise ValidationError("invalid model: " + "; ".join(v))


def _as_map(score_map):
    s = score_map.scores if hasattr(score_map, "scores") else np.asarray(score_map)
    s = np.asarray(s, dtype=np.float64)
    if s.ndim != 2 or min(s.shape) < 1:
        raise ValidationError(f"score map must be 2-D and non-empty, got {s.shape}")
    return s


def _place(score_map, anchor, deformation, radius, rect):
    """Windowed placement of one part map over a root rectangle (K3/K4)."""
    hp, wp = score_map.shape
    plan = Plan(1, [(hp, wp)], np.ones((1, 1), np.float32),
                [FilterDef(np.ones((1, 1, 1), np.float32))],
                assemblies=[AssemblyDef(None, tuple(int(v) for v in rect),
                                        (PartDef(0, 0, tuple(anchor), tuple(deformation),
                                                 int(radius), 1),))],
                outputs=("positions", "placed"))
    plan.load_levels(0, [score_map.astype(np.float32)[:, :, None]])
    plan.run()
    out = plan.assembly_outputs(0, 0)
    placed = out["placed"][0].cpu().numpy()
    py, px = unpack_positions(out["positions"][0].cpu().numpy())
    return placed, py, px


def best_part_placement(part, score_map, root_pos):
    """Penalty-adjusted window argmax for one root (detection.py:180-207)."""
    s = _as_map(score_map)
    ry, rx = int(root_pos[0]), int(root_pos[1])
    placed, py, px = _place(s, part.anchor, part.deformation, part.search_radius, (ry, ry, rx, rx))
    if not np.isfinite(placed[0, 0]):
        raise ValidationError(f"search window around {root_pos} is empty after clipping")
    return (int(py[0, 0]), int(px[0, 0])), float(placed[0, 0])


def _placement_grid(final_map, part, rect):
    """Vectorised placement over a root rectangle (detection.py:320-373)."""
    s = _as_map(final_map)
    return _place(s, part.anchor, part.deformation, part.search_radius, rect)


def _require_pyramid(pyramid, channels):
    # detection.py:376-383
    out = []
    for idx, level in enumerate(pyramid):
        try:
            out.append(check_feature_map(level, channels=channels))
        except ValidationError as exc:
            raise ValidationError(f"pyramid level {idx}: {exc}") from exc
    return out


def _detect_plan(levels, C, filters, root_f, part_fs, parts, bias):
    """Plan scoring every level: root map + windowed parts on the reference rect."""
    asms, rects = [], []
    for k, lv in enumerate(levels):
        rect = hypothesis_rect(lv.shape, filters[root_f].core.shape, parts)
        rects.append(rect)
        if rect is None:
            continue
        pd = tuple(PartDef(k, f, tuple(p.anchor), tuple(p.deformation), int(p.search_radius), 1)
                   for f, p in zip(part_fs, parts))
        asms.append(AssemblyDef((k, root_f), rect, pd, float(bias), level_tag=k))
    return asms, rects


def _collect(plan, asms, tau, model_id, detections):
    for ai, a in enumerate(asms):
        out = plan.assembly_outputs(0, ai)
        tot = out["totals"].cpu().numpy()
        iy, ix = np.nonzero(tot >= tau)
        if iy.size == 0:
            continue
        py, px = unpack_positions(out["positions"][:, iy, ix].cpu().numpy()) if a.parts else (None, None)
        ry0, _, rx0, _ = a.rect
        for n in range(iy.size):
            parts = tuple((int(py[p, n]), int(px[p, n])) for p in range(len(a.parts)))
            score = float(tot[iy[n], ix[n]])
            hyp = Hypothesis(level=a.level_tag, root=(ry0 + int(iy[n]), rx0 + int(ix[n])),
                             parts=parts, score=score)
            detections.append(Detection(hyp, model_id=model_id, score=score, tau=tau))


def _run_detect(levels, C, filters, root_f, part_fs, parts, bias, tau, model_id, stats):
    asms, rects = _detect_plan(levels, C, filters, root_f, part_fs, parts, bias)
    detections = []
    for rect in rects:
        if rect is not None:
            stats.positions_examined += (rect[1] - rect[0] + 1) * (rect[3] - rect[2] + 1)
    if asms:
        L = levels[0].shape[2]
        plan = Plan(L, [lv.shape[:2] for lv in levels], C, filters, assemblies=asms,
                    outputs=("totals", "positions"))
        for k, lv in enumerate(levels):
            plan.x_view(0, k).copy_(_t().from_numpy(lv.astype(np.float32)))
        plan.run()
        _collect(plan, asms, tau, model_id, detections)
    detections.sort(key=lambda d: (d.hypothesis.level, d.hypothesis.root))
    return detections, rects


def _t():
    import torch

    return torch


def detect(dec, pyramid, tau, pruning=False, part_prune_mode="kill", model_id="model",
           collect_maps=False):
    """Decomposed detector, pruning off (detection.py:386-542)."""
    if part_prune_mode not in ("kill", "lenient"):
        raise ValidationError(f"unknown part_prune_mode {part_prune_mode!r}")
    if pruning and not dec.calibrated:
        raise ValidationError("pruning requires calibrated thresholds")
    if pruning:
        raise NotImplementedError("pruned detection (Algorithm 1) is the next tier of the "
                                  "B200 path; call with pruning=False")
    levels = _require_pyramid(pyramid, dec.channels)
    start = time.perf_counter()
    stats = DetectStats()
    # per-filter CP: each filter projects onto its own c columns
    cps = [dec.root_cp] + [p.cp for p in dec.parts]
    C = np.concatenate([np.asarray(cp.factors_c, dtype=np.float32) for cp in cps], axis=1)
    filters, off = [], 0
    for cp in cps:
        filters.append(FilterDef(cp_core(cp), chan_off=off))
        off += cp.rank
    dets, rects = _run_detect(levels, C, filters, 0, list(range(1, len(cps))), dec.parts,
                              dec.bias, tau, model_id, stats)
    for lv, rect in zip(levels, rects):
        if rect is None:
            continue
        for cp in cps:
            stats.multiplications += cp_multiplications(lv.shape, cp.dims, cp.rank)
    if collect_maps:
        stats.prune_maps = [{"rect": r} for r in rects]
    stats.wall_time = time.perf_counter() - start
    return dets, stats


def dense_detect(model, pyramid, tau, model_id="model"):
    """Dense-filter detector (detection.py:570-616): basis = identity."""
    require_valid(model)
    levels = _require_pyramid(pyramid, model.channels)
    start = time.perf_counter()
    stats = DetectStats()
    L = model.channels
    flts = [np.asarray(model.root)] + [np.asarray(p.filter) for p in model.parts]
    filters = [FilterDef(f.astype(np.float32)) for f in flts]
    dets, rects = _run_detect(levels, np.eye(L, dtype=np.float32), filters, 0,
                              list(range(1, len(flts))), model.parts, model.bias, tau, model_id,
                              stats)
    for lv, rect in zip(levels, rects):
        if rect is None:
            continue
        for f in flts:
            stats.multiplications += full_multiplications(lv.shape, f.shape)
    stats.wall_time = time.perf_counter() - start
    return dets, stats


def _maps_at(level, C, filters):
    H, W, L = level.shape
    plan = Plan(L, [(H, W)], C, filters, apps=[(0, f) for f in range(len(filters))], outputs=())
    plan.load_levels(0, [level.astype(np.float32)])
    plan.run(stages=("project", "correlate"))
    return [plan.map(0, 0, f).double().cpu().numpy() for f in range(len(filters))]


def _check_pos(level, dims, pos):
    H, W = level.shape[:2]
    y, x = pos
    if not (0 <= y <= H - dims[0] and 0 <= x <= W - dims[1]):
        raise ValidationError(f"position {tuple(pos)} out of support for filter {tuple(dims)}")


def score_hypothesis(model, level, hypothesis):
    """Dense score of a fixed hypothesis (detection.py:144-161)."""
    require_valid(model)
    level = check_feature_map(level, channels=model.channels)
    if len(hypothesis.parts) != len(model.parts):
        raise ValidationError(f"hypothesis has {len(hypothesis.parts)} part positions, model "
                              f"has {len(model.parts)} parts")
    flts = [np.asarray(model.root)] + [np.asarray(p.filter) for p in model.parts]
    for f, pos in zip(flts, (hypothesis.root,) + tuple(hypothesis.parts)):
        _check_pos(level, f.shape, pos)
    maps = _maps_at(level, np.eye(level.shape[2], dtype=np.float32),
                    [FilterDef(f.astype(np.float32)) for f in flts])
    ry, rx = hypothesis.root
    score = float(maps[0][ry, rx])
    for part, m, pos in zip(model.parts, maps[1:], hypothesis.parts):
        dy, dx = pos[0] - ry - part.anchor[0], pos[1] - rx - part.anchor[1]
        score += float(m[pos[0], pos[1]])
        score -= deformation_penalty(part.deformation, dy, dx)
    return score + model.bias


def cp_score_hypothesis(dec, level, hypothesis):
    """Full-rank CP score of a fixed hypothesis (detection.py:164-177)."""
    level = check_feature_map(level, channels=dec.channels)
    cps = [dec.root_cp] + [p.cp for p in dec.parts]
    C = np.concatenate([np.asarray(cp.factors_c, dtype=np.float32) for cp in cps], axis=1)
    filters, off = [], 0
    for cp in cps:
        filters.append(FilterDef(cp_core(cp), chan_off=off))
        off += cp.rank
    maps = _maps_at(level, C, filters)
    ry, rx = hypothesis.root
    score = float(maps[0][ry, rx])
    for part, m, pos in zip(dec.parts, maps[1:], hypothesis.parts):
        dy, dx = pos[0] - ry - part.anchor[0], pos[1] - rx - part.anchor[1]
        score += float(m[pos[0], pos[1]])
        score -= deformation_penalty(part.deformation, dy, dx)
    return score + dec.bias
