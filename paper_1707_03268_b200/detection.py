"""Drop-in scoring / placement / detection on the B200 (K1-K4).

Mirrors ``cpdetect.detection`` for the pruning-off hot path
(``detection.py:128-616``): same names, arguments, return types, error
classes and messages.  The GPU computes response maps in FP32 and placement
and assembly in FP64 with the reference's exact expression order, so for a
given response map the placed values and argmaxes are bit-identical to
``_placement_grid``.

``detect(..., pruning=True)`` (Algorithm 1, convolution shortening) runs its
rank-prefix maps (K2), the per-rank root / part-window checks
(``dpm_prune_ranks``), placement and assembly on the GPU; which hypotheses
are alive when each part is checked, the lenient-mode sums and the
reference's work counters are composed on the host from the returned ranks.
``calibrate_thresholds`` reads its per-rank floors from the GPU's own prefix
maps, so a model calibrated here never prunes its own positives.
"""

import time

import numpy as np

from .correlation import cp_core
from .engine import AssemblyDef, FilterDef, PartDef, Plan, unpack_positions
from .errors import ValidationError, check_feature_map
from .geometry import cp_multiplications, full_multiplications, hypothesis_rect
from .plancache import lease
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
    "calibrate_thresholds",
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
        # every filter on every scored level: a rank-prefix family is computed
        # whole (one pass over the ranks) even when only its last map is read
        apps = [(a.level_tag, f) for a in asms for f in range(len(filters))]
        plan = Plan(L, [lv.shape[:2] for lv in levels], C, filters, apps=apps, assemblies=asms,
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
    levels = _require_pyramid(pyramid, dec.channels)
    if pruning:
        return _detect_pruned(dec, levels, tau, part_prune_mode, model_id, collect_maps)
    start = time.perf_counter()
    stats = DetectStats()
    # per-filter CP: each filter projects onto its own c columns; its
    # response is the last rank prefix (cp_partial_stack(...)[-1], as the
    # reference's detect and the pruned path read it)
    cps = [dec.root_cp] + [p.cp for p in dec.parts]
    C, filters, pref = _prefix_filters(cps)
    dets, rects = _run_detect(levels, C, filters, pref[0][-1], [pr[-1] for pr in pref[1:]],
                              dec.parts, dec.bias, tau, model_id, stats)
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
    with lease(L, [(H, W)], C, filters, [(0, f) for f in range(len(filters))]) as plan:
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
    C, filters, pref = _prefix_filters(cps)
    allmaps = _maps_at(level, C, filters)
    maps = [allmaps[pr[-1]] for pr in pref]  # cp_partial_stack(...)[-1] (detection.py:164-177)
    ry, rx = hypothesis.root
    score = float(maps[0][ry, rx])
    for part, m, pos in zip(dec.parts, maps[1:], hypothesis.parts):
        dy, dx = pos[0] - ry - part.anchor[0], pos[1] - rx - part.anchor[1]
        score += float(m[pos[0], pos[1]])
        score -= deformation_penalty(part.deformation, dy, dx)
    return score + dec.bias


# ------------------------------------------------- pruned detection (Alg. 1)

def _prefix_filters(cps):
    """Every rank prefix of every CP filter over its own basis columns:
    prefix k keeps ranks < k (the cp_partial_stack order, bit-identical
    prefixes), all of a filter's prefixes from one rank-prefix K2 pass.
    Returns (C, filters, pref) with pref[i] the filter indices of CP i's
    prefixes 1..R_i."""
    C = np.concatenate([np.asarray(cp.factors_c, dtype=np.float32) for cp in cps], axis=1)
    filters, pref, off = [], [], 0
    for cp in cps:
        idx = []
        core = cp_core(cp)  # one family: the rank-prefix kernel writes all R maps in one pass
        for k in range(cp.rank):
            filters.append(FilterDef(core, chan_off=off, prefix=k + 1))
            idx.append(len(filters) - 1)
        pref.append(idx)
        off += cp.rank
    return C, filters, pref


def _dilate_any(mask, radius):
    """Box dilation onto a grid extended by ``radius`` on every side
    (detection.py:302-317): cell (Y, X) is set when a mask cell lies in the
    (2r+1)^2 box centred at mask coordinate (Y - r, X - r)."""
    from numpy.lib.stride_tricks import sliding_window_view

    width = 2 * radius + 1
    return sliding_window_view(np.pad(mask, 2 * radius), (width, width)).any(axis=(-2, -1))


def _covered_count(covered, rect, anchor, radius, support):
    """Part positions inside the union of alive windows (detection.py:545-567)."""
    ry0, ry1, rx0, rx1 = rect
    ay, ax = anchor
    sy, sx = support
    py0, py1 = max(0, ry0 + ay - radius), min(sy - 1, ry1 + ay + radius)
    px0, px1 = max(0, rx0 + ax - radius), min(sx - 1, rx1 + ax + radius)
    if py0 > py1 or px0 > px1:
        return 0
    oy, ox = py0 - ay - (ry0 - radius), px0 - ax - (rx0 - radius)
    return int(covered[oy:oy + py1 - py0 + 1, ox:ox + px1 - px0 + 1].sum())


def _bump(table, rank, count):
    if count:
        table[rank] = table.get(rank, 0) + int(count)


def _detect_pruned(dec, levels, tau, mode, model_id, collect_maps):
    """detect(..., pruning=True) (detection.py:386-542 with the pruning
    branches 433-503)."""
    from . import _lib
    from .device import stream_handle, upload_table

    t = _t()
    start = time.perf_counter()
    stats = DetectStats()
    stats.prune_maps = [] if collect_maps else None
    cps = [dec.root_cp] + [p.cp for p in dec.parts]
    C, filters, pref = _prefix_filters(cps)
    root_f, part_fs = pref[0][-1], [pr[-1] for pr in pref[1:]]
    asms, rects = _detect_plan(levels, C, filters, root_f, part_fs, dec.parts, dec.bias)
    detections = []
    if not asms:
        for rect in rects:
            if collect_maps:
                stats.prune_maps.append({"rect": rect})
        stats.wall_time = time.perf_counter() - start
        return detections, stats
    L = levels[0].shape[2]
    apps = [(a.level_tag, f) for a in asms for f in range(len(filters))]
    plan = Plan(L, [lv.shape[:2] for lv in levels], C, filters, apps=apps, assemblies=asms,
                outputs=("totals", "positions", "placed"))
    for k, lv in enumerate(levels):
        plan.x_view(0, k).copy_(t.from_numpy(lv.astype(np.float32)))
    plan.run()

    # per-rank checks on the device: one job per (level, filter role)
    thr = np.concatenate([np.asarray(dec.root_thresholds, dtype=np.float64)] +
                         [np.asarray(p.thresholds, dtype=np.float64) for p in dec.parts])
    thr0 = np.cumsum([0] + [cp.rank for cp in cps])[:-1]
    jobs, offs, out_at = [], [], {}
    cursor = 0
    for ai, a in enumerate(asms):
        k = a.level_tag
        ry0, ry1, rx0, rx1 = a.rect
        n = (ry1 - ry0 + 1) * (rx1 - rx0 + 1)
        for role, cp in enumerate(cps):
            hp, wp = plan.map_shape[(k, pref[role][0])]
            o0 = len(offs)
            offs.extend(plan.map_off[(0, k, f)] for f in pref[role])
            if role == 0:
                ay = ax = 0
                radius = -1
            else:
                part = dec.parts[role - 1]
                (ay, ax), radius = part.anchor, int(part.search_radius)
            jobs.append((cursor, o0, int(thr0[role]), cp.rank, hp, wp, ry0, ry1, rx0, rx1,
                         int(ay), int(ax), 1, radius, 0))
            out_at[(ai, role)] = cursor
            cursor += n
    jobs = np.array(jobs, dtype=_lib.PRUNE_JOB)
    lib = _lib.lib()
    nblk = _lib.check(lib.dpm_prune_prepare(_lib.table_ptr(jobs), len(jobs)), "prune")
    dev = plan.device
    jobs_d = upload_table(jobs, dev)
    offs_d = t.tensor(offs, dtype=t.int64, device=dev)
    thr_d = t.from_numpy(thr).to(dev)
    ranks_d = t.empty(max(cursor, 1), dtype=t.uint8, device=dev)
    _lib.check(lib.dpm_prune_ranks(plan.S.data_ptr(), offs_d.data_ptr(), thr_d.data_ptr(),
                                   jobs_d.data_ptr(), len(jobs), nblk, ranks_d.data_ptr(),
                                   stream_handle(None)), "prune")
    # composition on the device (dpm_prune_compose / dpm_prune_cover): alive
    # sets in part order, lenient scores, detections, and the counters as
    # histograms; the host only sums the histograms in the reference's order
    nparts = len(dec.parts)
    cj = np.zeros(len(asms), dtype=_lib.PRUNE_ASM)
    covs, lim_size, hist_size = [], 0, 0
    for ai, a in enumerate(asms):
        k = a.level_tag
        ry0, ry1, rx0, rx1 = a.rect
        hr, wr = ry1 - ry0 + 1, rx1 - rx0 + 1
        n = hr * wr
        t_off, p_off, pl_off, _, _ = plan.asm_index[(0, ai)]
        j = cj[ai]
        j["rank_off"], j["lim_off"] = out_at[(ai, 0)], lim_size
        j["total_off"], j["pos_off"], j["placed_off"] = t_off, max(p_off, 0), max(pl_off, 0)
        j["root_off"] = plan.map_off[(0, k, root_f)]
        j["root_pitch"] = (plan.map_shape[(k, root_f)][1] + 3) & ~3
        j["ry0"], j["ry1"], j["rx0"], j["rx1"] = ry0, ry1, rx0, rx1
        j["nparts"], j["image"], j["level"], j["hist_off"] = nparts, 0, k, hist_size
        j["bias"] = float(dec.bias)
        sy_, sx_ = levels[k].shape[0], levels[k].shape[1]
        for pi, part in enumerate(dec.parts):
            j["part_R"][pi] = part.cp.rank
            j["ay"][pi], j["ax"][pi] = part.anchor
            nn, mm, _ = part.cp.dims
            rad = int(part.search_radius)
            ay, ax = (int(v) for v in part.anchor)
            sy, sx = sy_ - nn + 1, sx_ - mm + 1
            covs.append((lim_size + pi * n, hr, wr, max(0, ry0 + ay - rad), min(sy - 1, ry1 + ay + rad),
                         max(0, rx0 + ax - rad), min(sx - 1, rx1 + ax + rad), ry0 + ay, rx0 + ax,
                         rad, 0, 0, 0))
        lim_size += 2 * nparts * n
        hist_size += (1 + nparts) * 256
    cov = np.array(covs, dtype=_lib.COVER_JOB) if covs else np.zeros(0, _lib.COVER_JOB)
    cov_hist0 = hist_size
    cov["hist_off"] = cov_hist0 + 256 * np.arange(len(cov))
    hist_size += 256 * len(cov)
    cblk = _lib.check(lib.dpm_prune_compose_prepare(_lib.table_ptr(cj), len(cj)), "prune compose")
    vblk = _lib.check(lib.dpm_prune_cover_prepare(_lib.table_ptr(cov), len(cov)), "prune cover")
    cj_d, cov_d = upload_table(cj, dev), upload_table(cov, dev)
    lim_d = t.zeros(max(lim_size, 1), dtype=t.uint8, device=dev)
    hist_d = t.zeros(max(hist_size, 1), dtype=t.int32, device=dev)
    n_roots = int(sum((a.rect[1] - a.rect[0] + 1) * (a.rect[3] - a.rect[2] + 1) for a in asms))
    dets_d = t.empty(max(n_roots, 1) * _lib.DETECTION.itemsize, dtype=t.uint8, device=dev)
    cnt_d = t.zeros(1, dtype=t.int32, device=dev)
    s = stream_handle(None)
    _lib.check(lib.dpm_prune_compose(
        ranks_d.data_ptr(), plan.S.data_ptr(), plan.totals.data_ptr(), plan.positions.data_ptr(),
        plan.placed.data_ptr(), cj_d.data_ptr(), len(cj), cblk, 1 if mode == "kill" else 0,
        float(tau), lim_d.data_ptr(), hist_d.data_ptr(), dets_d.data_ptr(), max(n_roots, 1),
        cnt_d.data_ptr(), s), "prune compose")
    _lib.check(lib.dpm_prune_cover(lim_d.data_ptr(), cov_d.data_ptr(), len(cov), vblk,
                                   hist_d.data_ptr(), s), "prune cover")
    hist = hist_d.cpu().numpy().astype(np.int64)
    ndet = int(cnt_d.item())
    recs = np.frombuffer(dets_d[:ndet * _lib.DETECTION.itemsize].cpu().numpy().tobytes(),
                         dtype=_lib.DETECTION)
    if collect_maps:
        ranks = ranks_d.cpu().numpy()
        lims = lim_d.cpu().numpy()

    ai_of = {a.level_tag: ai for ai, a in enumerate(asms)}
    n0, m0, l0 = dec.root_cp.dims
    for li, rect in enumerate(rects):
        lm = {"rect": rect} if collect_maps else None
        if collect_maps:
            stats.prune_maps.append(lm)
        if rect is None:
            continue
        ai = ai_of[li]
        ry0, ry1, rx0, rx1 = rect
        hr, wr = ry1 - ry0 + 1, rx1 - rx0 + 1
        stats.positions_examined += hr * wr
        h0 = int(cj[ai]["hist_off"])
        hroot = hist[h0:h0 + 256]
        # root: first failing rank (detection.py:452-460)
        for r in range(dec.root_cp.rank):
            stats.multiplications += int(hroot[0] + hroot[r + 1:].sum()) * (n0 + m0 + l0)
            _bump(stats.positions_pruned_at_rank, r + 1, hroot[r + 1])
        for pi, part in enumerate(dec.parts):  # parts in order (detection.py:462-503)
            hp = hist[h0 + (1 + pi) * 256:h0 + (2 + pi) * 256]
            hc = hist[cov_hist0 + 256 * (ai * nparts + pi):cov_hist0 + 256 * (ai * nparts + pi + 1)]
            n, m, l = part.cp.dims
            alive_r = int(hp[0])  # alive when the part is checked
            for r in range(part.cp.rank):
                if alive_r == 0:
                    break
                # support cells of the windows still alive at rank r
                stats.multiplications += int(hc[r + 1:].sum()) * (n + m + l)
                alive_r -= int(hp[r + 1])
                _bump(stats.part_pruned_at_rank, r + 1, hp[r + 1])
                if mode == "kill":
                    stats.positions_killed_by_parts += int(hp[r + 1])
        if collect_maps:
            n = hr * wr
            o = out_at[(ai, 0)]
            lo = int(cj[ai]["lim_off"])
            lm["root_prune_rank"] = ranks[o:o + n].reshape(hr, wr).astype(np.int64)
            lm["part_prune_rank"] = lims[lo + nparts * n:lo + 2 * nparts * n].reshape(
                nparts, hr, wr).astype(np.int64)
    for d in recs:
        py, px = unpack_positions(d["parts"][:nparts])
        pp = tuple((int(y), int(x)) for y, x in zip(py, px))
        score = float(d["score"])
        hyp = Hypothesis(level=int(d["level"]), root=(int(d["ry"]), int(d["rx"])), parts=pp,
                         score=score)
        detections.append(Detection(hyp, model_id=model_id, score=score, tau=tau))
    detections.sort(key=lambda d: (d.hypothesis.level, d.hypothesis.root))
    stats.wall_time = time.perf_counter() - start
    return detections, stats


def _check_positive(dec, level, hyp):
    # detection.py:238-259
    H, W, _ = level.shape
    n0, m0, _ = dec.root_cp.dims
    ry, rx = hyp.root
    if not (0 <= ry <= H - n0 and 0 <= rx <= W - m0):
        raise ValidationError(f"positive root position {hyp.root} out of support")
    if len(hyp.parts) != len(dec.parts):
        raise ValidationError(f"positive has {len(hyp.parts)} part positions, model has "
                              f"{len(dec.parts)} parts")
    for i, (part, pos) in enumerate(zip(dec.parts, hyp.parts)):
        n, m, _ = part.cp.dims
        if not (0 <= pos[0] <= H - n and 0 <= pos[1] <= W - m):
            raise ValidationError(f"positive part {i} position {pos} out of support")
        dy = pos[0] - ry - part.anchor[0]
        dx = pos[1] - rx - part.anchor[1]
        if max(abs(dy), abs(dx)) > part.search_radius:
            raise ValidationError(f"positive part {i} displaced by ({dy}, {dx}), outside its "
                                  f"search radius {part.search_radius}")


def calibrate_thresholds(dec, positives):
    """Tightest per-rank floors keeping every positive (detection.py:262-299),
    read from the GPU's prefix maps.  Returns a copy of ``dec`` with
    ``root_thresholds`` and per-part ``thresholds`` set."""
    from dataclasses import replace

    if not positives:
        raise ValidationError("cannot calibrate thresholds from zero positives")
    cps = [dec.root_cp] + [p.cp for p in dec.parts]
    C, filters, pref = _prefix_filters(cps)
    mins = [None] * len(cps)
    cache = {}
    for level, hyp in positives:
        level = np.asarray(level)
        _check_positive(dec, level, hyp)
        key = id(level)
        if key not in cache:
            checked = check_feature_map(level, channels=dec.channels)
            cache[key] = _maps_at(checked, C, filters)
        maps = cache[key]
        for role, pos in enumerate((hyp.root,) + tuple(hyp.parts)):
            vec = np.array([maps[f][pos[0], pos[1]] for f in pref[role]])
            mins[role] = vec if mins[role] is None else np.minimum(mins[role], vec)
    parts = tuple(_with(p, thresholds=m) for p, m in zip(dec.parts, mins[1:]))
    return _with(dec, parts=parts, root_thresholds=mins[0])


def _with(obj, **kw):
    """dataclasses.replace for our types and the reference's (duck typed)."""
    from dataclasses import is_dataclass, replace

    if is_dataclass(obj):
        return replace(obj, **kw)
    import copy

    new = copy.copy(obj)
    for k, v in kw.items():
        setattr(new, k, v)
    return new
