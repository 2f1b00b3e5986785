"""CPU oracle for the DPM score path -- TEST INFRASTRUCTURE ONLY.

This module restates, in float64 numpy, the reference's algorithm for the
hot path (``/root/reference/pkg/src/cpdetect``; every function cites the
file:line it follows).  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it,
and only as the checker or as the timed CPU baseline -- never as part of
the product path, which fails loudly when its CUDA library is missing.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by running the reference itself
(``tests/golden/make_golden.py``), plus the reference tests' own
known-answer constants.

Where the reference lacks a feature the configs need,
the composition below uses only restated reference functions:

* part scale s = 2  -> ``placement_grid`` over a virtual full-map rect with
  zero anchor, gathered at ``s*root + anchor`` (App. A.1);
* unbounded GDT     -> ``placement_grid`` with radius ``r_star`` (App. A.2);
* shared basis      -> ``correlate3_full(X @ C, G_f)`` (App. A.3): the
  reference's dense correlation applied to the projected level with the
  filter's core (identical to ``correlate3_full(X, reconstructed f)``).
"""

import math

import numpy as np

__all__ = [
    "correlate3_full",
    "term_stack",
    "cp_partial_stack",
    "correlate3_cp",
    "deformation_penalty",
    "best_part_placement",
    "hypothesis_rect",
    "placement_grid",
    "detect",
    "dense_detect",
    "score_hypothesis",
    "cp_score_hypothesis",
    "project",
    "r_star",
    "place_gathered",
    "score_pyramid",
    "dilate_any",
    "covered_count",
    "window_max",
    "detect_pruned",
    "calibrate_thresholds",
]


# ---------------------------------------------------------------- correlation

def _support(img_shape, filt_shape):
    # correlation.py:64-75
    H, W, L = img_shape
    n, m, l = filt_shape
    if l != L:
        raise ValueError(f"channel mismatch: filter has {l}, image has {L}")
    ho, wo = H - n + 1, W - m + 1
    if ho < 1 or wo < 1:
        raise ValueError(f"filter extent ({n}, {m}) exceeds image extent ({H}, {W})")
    return ho, wo


def correlate3_full(img, filt):
    """Dense valid correlation, tap by tap (correlation.py:92-112).

    ``out[y, x] = sum_{i,j,k} filt[i,j,k] * img[y+i, x+j, k]``: for every tap
    (i, j) the shifted window is contracted over channels and accumulated in
    row-major tap order."""
    img = np.asarray(img, dtype=np.float64)
    filt = np.asarray(filt, dtype=np.float64)
    ho, wo = _support(img.shape, filt.shape)
    out = np.zeros((ho, wo))
    for i in range(filt.shape[0]):
        for j in range(filt.shape[1]):
            out += np.einsum("hwl,l->hw", img[i:i + ho, j:j + wo, :], filt[i, j, :])
    return out


def term_stack(img, cp, upto):
    """Per-rank weighted separable terms (correlation.py:115-143).

    Channel contraction of all ranks at once (one matmul, line 128), then
    per rank a row pass over the ``a`` taps (135-138) and a column pass over
    ``b * weight`` taps (139-142), each accumulated tap by tap."""
    img = np.asarray(img, dtype=np.float64)
    H, W, L = img.shape
    n, m, _ = cp.dims
    ho, wo = _support(img.shape, cp.dims)
    a = np.asarray(cp.factors_a, dtype=np.float64)
    bw = np.asarray(cp.factors_b, dtype=np.float64) * np.asarray(cp.weights)[None, :]
    proj = (img.reshape(H * W, L) @ np.asarray(cp.factors_c)[:, :upto]).reshape(H, W, upto)
    terms = np.empty((upto, ho, wo))
    for r in range(upto):
        ch = np.ascontiguousarray(proj[:, :, r])
        rows = ch[0:ho] * a[0, r]
        for i in range(1, n):
            rows = rows + ch[i:i + ho] * a[i, r]
        t = rows[:, 0:wo] * bw[0, r]
        for j in range(1, m):
            t = t + rows[:, j:j + wo] * bw[j, r]
        terms[r] = t
    return terms


def cp_partial_stack(img, cp, upto_rank=None):
    """Cumulative rank-prefix maps; always evaluates every rank so prefixes
    are bit-identical (correlation.py:170-180, 163-166)."""
    upto = cp.rank if upto_rank is None else upto_rank
    if not 1 <= upto <= cp.rank:
        raise ValueError(f"upto_rank must be in [1, {cp.rank}], got {upto_rank}")
    return np.cumsum(term_stack(img, cp, cp.rank)[:upto], axis=0)


def correlate3_cp(img, cp, upto_rank=None):
    """Last entry of the partial stack (correlation.py:155-167)."""
    return cp_partial_stack(img, cp, upto_rank)[-1]


# ------------------------------------------------------------------ placement

def deformation_penalty(deformation, dy, dx):
    """c_dx*dx + c_dy*dy + c_dxx*dx^2 + c_dyy*dy^2 (detection.py:128-131)."""
    cdx, cdy, cdxx, cdyy = deformation
    return cdx * dx + cdy * dy + cdxx * dx * dx + cdyy * dy * dy


def best_part_placement(scores, anchor, deformation, radius, root_pos):
    """Scalar window scan, strict '>' in (dy, dx) lexicographic order
    (detection.py:180-207).  Returns ((y, x), value)."""
    hp, wp = scores.shape
    cy, cx = root_pos[0] + anchor[0], root_pos[1] + anchor[1]
    best = None
    for dy in range(-radius, radius + 1):
        for dx in range(-radius, radius + 1):
            y, x = cy + dy, cx + dx
            if 0 <= y < hp and 0 <= x < wp:
                v = scores[y, x] - deformation_penalty(deformation, dy, dx)
                if best is None or v > best[0]:
                    best = (v, (y, x))
    if best is None:
        raise ValueError(f"search window around {root_pos} is empty after clipping")
    return best[1], float(best[0])


def hypothesis_rect(level_shape, root_dims, part_dims, anchors, radii):
    """Reference root rectangle (detection.py:210-235)."""
    H, W = level_shape[0], level_shape[1]
    if H - root_dims[0] + 1 < 1 or W - root_dims[1] + 1 < 1:
        return None
    ry0, ry1 = 0, H - root_dims[0]
    rx0, rx1 = 0, W - root_dims[1]
    for d, (ay, ax), r in zip(part_dims, anchors, radii):
        sy, sx = H - d[0] + 1, W - d[1] + 1
        if sy < 1 or sx < 1:
            return None
        ry0, ry1 = max(ry0, -ay - r), min(ry1, sy - 1 - ay + r)
        rx0, rx1 = max(rx0, -ax - r), min(rx1, sx - 1 - ax + r)
    if ry0 > ry1 or rx0 > rx1:
        return None
    return ry0, ry1, rx0, rx1


def placement_grid(score_map, anchor, deformation, radius, rect):
    """Separable windowed placement over a root rectangle
    (detection.py:320-373).

    The map is padded with -inf by 2r; an x pass over dx = -r..r (strict '>',
    ascending) runs on the band of rows any window can reach, then a y pass
    over dy = -r..r; the penalty is subtracted in two stages, x part first.
    Returns (placed, pos_y, pos_x) shaped like the rectangle."""
    ry0, ry1, rx0, rx1 = rect
    hr, wr = ry1 - ry0 + 1, rx1 - rx0 + 1
    r = radius
    ay, ax = anchor
    cdx, cdy, cdxx, cdyy = deformation
    pad = np.pad(np.asarray(score_map, dtype=np.float64), 2 * r, constant_values=-np.inf)
    band = hr + 2 * r
    y_first = ry0 + ay + r          # padded row of dy = -r for the first rect row
    x_zero = rx0 + ax + 2 * r       # padded column of dx = 0 for the first rect column
    bx = None
    for dx in range(-r, r + 1):
        c = pad[y_first:y_first + band, x_zero + dx:x_zero + dx + wr] - (cdx * dx + cdxx * dx * dx)
        if bx is None:
            bx, bdx = c, np.full((band, wr), dx, dtype=np.int64)
        else:
            up = c > bx
            bx = np.where(up, c, bx)
            bdx = np.where(up, dx, bdx)
    placed = None
    for dy in range(-r, r + 1):
        k = dy + r
        c = bx[k:k + hr] - (cdy * dy + cdyy * dy * dy)
        if placed is None:
            placed = c
            wdy = np.full((hr, wr), dy, dtype=np.int64)
            wdx = bdx[k:k + hr].copy()
        else:
            up = c > placed
            placed = np.where(up, c, placed)
            wdy = np.where(up, dy, wdy)
            wdx = np.where(up, bdx[k:k + hr], wdx)
    pos_y = np.arange(ry0, ry1 + 1)[:, None] + ay + wdy
    pos_x = np.arange(rx0, rx1 + 1)[None, :] + ax + wdx
    return placed, pos_y, pos_x


# ------------------------------------------------------------------ detectors

def _assemble(level_idx, rect, root_map, placements, bias, tau, out):
    # detection.py:449, 509-538
    ry0, ry1, rx0, rx1 = rect
    scores = root_map[ry0:ry1 + 1, rx0:rx1 + 1].copy()
    for placed, _, _ in placements:
        scores = scores + placed
    scores = scores + bias
    for iy, ix in zip(*np.nonzero(scores >= tau)):
        parts = tuple((int(py[iy, ix]), int(px[iy, ix])) for _, py, px in placements)
        out.append((level_idx, (int(ry0 + iy), int(rx0 + ix)), parts, float(scores[iy, ix])))
    return scores


def detect(dec, pyramid, tau):
    """``detect(..., pruning=False)`` (detection.py:386-542).

    Returns (detections, stats) where detections are (level, root, parts,
    score) tuples sorted by (level, root) and stats carries the
    positions_examined / multiplications counters."""
    dets, examined, mults = [], 0, 0
    rn, rm, rl = dec.root_cp.dims
    for li, level in enumerate(pyramid):
        level = np.asarray(level, dtype=np.float64)
        rect = hypothesis_rect(level.shape, dec.root_cp.dims,
                               [p.cp.dims for p in dec.parts],
                               [p.anchor for p in dec.parts],
                               [p.search_radius for p in dec.parts])
        if rect is None:
            continue
        examined += (rect[1] - rect[0] + 1) * (rect[3] - rect[2] + 1)
        root_map = cp_partial_stack(level, dec.root_cp)[-1]
        ho, wo = _support(level.shape, dec.root_cp.dims)
        mults += dec.root_cp.rank * ho * wo * (rn + rm + rl)
        placements = []
        for p in dec.parts:
            pm = cp_partial_stack(level, p.cp)[-1]
            n, m, l = p.cp.dims
            ho, wo = _support(level.shape, p.cp.dims)
            mults += p.cp.rank * ho * wo * (n + m + l)
            placements.append(placement_grid(pm, p.anchor, p.deformation, p.search_radius, rect))
        _assemble(li, rect, root_map, placements, dec.bias, tau, dets)
    dets.sort(key=lambda d: (d[0], d[1]))
    return dets, {"positions_examined": examined, "multiplications": mults}


def dense_detect(model, pyramid, tau):
    """Dense reference detector (detection.py:570-616)."""
    dets, examined, mults = [], 0, 0
    for li, level in enumerate(pyramid):
        level = np.asarray(level, dtype=np.float64)
        rect = hypothesis_rect(level.shape, model.root.shape,
                               [p.filter.shape for p in model.parts],
                               [p.anchor for p in model.parts],
                               [p.search_radius for p in model.parts])
        if rect is None:
            continue
        examined += (rect[1] - rect[0] + 1) * (rect[3] - rect[2] + 1)
        root_map = correlate3_full(level, model.root)
        ho, wo = root_map.shape
        mults += ho * wo * int(np.prod(model.root.shape))
        placements = []
        for p in model.parts:
            pm = correlate3_full(level, p.filter)
            mults += pm.shape[0] * pm.shape[1] * int(np.prod(p.filter.shape))
            placements.append(placement_grid(pm, p.anchor, p.deformation, p.search_radius, rect))
        _assemble(li, rect, root_map, placements, model.bias, tau, dets)
    dets.sort(key=lambda d: (d[0], d[1]))
    return dets, {"positions_examined": examined, "multiplications": mults}


def _window_dot(level, filt, pos):
    n, m, _ = filt.shape
    y, x = pos
    return float(np.einsum("ijk,ijk->", level[y:y + n, x:x + m, :], filt))


def score_hypothesis(model, level, root, parts):
    """Dense score of a fixed hypothesis (detection.py:144-161)."""
    level = np.asarray(level, dtype=np.float64)
    s = _window_dot(level, model.root, root)
    for p, pos in zip(model.parts, parts):
        dy, dx = pos[0] - root[0] - p.anchor[0], pos[1] - root[1] - p.anchor[1]
        s += _window_dot(level, p.filter, pos)
        s -= deformation_penalty(p.deformation, dy, dx)
    return s + model.bias


def cp_score_hypothesis(dec, level, root, parts):
    """Full-rank CP score of a fixed hypothesis (detection.py:164-177)."""
    level = np.asarray(level, dtype=np.float64)
    s = float(cp_partial_stack(level, dec.root_cp)[-1, root[0], root[1]])
    for p, pos in zip(dec.parts, parts):
        dy, dx = pos[0] - root[0] - p.anchor[0], pos[1] - root[1] - p.anchor[1]
        s += float(cp_partial_stack(level, p.cp)[-1, pos[0], pos[1]])
        s -= deformation_penalty(p.deformation, dy, dx)
    return s + dec.bias


# --------------------------------------------------- shared basis + pyramids

def project(level, C):
    """Channel projection onto the basis (the matmul of correlation.py:128)."""
    level = np.asarray(level, dtype=np.float64)
    H, W, L = level.shape
    return (level.reshape(H * W, L) @ np.asarray(C, dtype=np.float64)).reshape(H, W, -1)


def r_star(score_map, deformation):
    """Radius beyond which no maximiser lies (SURVEY.md App. A.2 lemma).

    Per axis r = floor((|b| + sqrt(b^2 + 4 a D')) / (2a)) with
    D' = (max S - min S) + b_other^2 / (4 a_other); returns max over axes.
    Requires a > 0 on both axes."""
    cdx, cdy, cdxx, cdyy = deformation
    rng = float(np.max(score_map) - np.min(score_map))
    out = 0
    for a, b, a_o, b_o in ((cdxx, cdx, cdyy, cdy), (cdyy, cdy, cdxx, cdx)):
        if a <= 0 or a_o <= 0:
            raise ValueError("r_star needs positive quadratic coefficients")
        dprime = rng + b_o * b_o / (4.0 * a_o)
        out = max(out, int(math.floor((abs(b) + math.sqrt(b * b + 4 * a * dprime)) / (2 * a))))
    return out


def place_gathered(score_map, anchor, deformation, radius, scale, rect):
    """Placement of parts at centre ``scale*root + anchor`` for every root in
    ``rect``: reference placement over the virtual
    full-map rect with zero anchor (extended by r so the -inf padding stays
    the reference's), then gathered."""
    hp, wp = score_map.shape
    r = radius
    virt = (-r, hp - 1 + r, -r, wp - 1 + r)
    placed, py, px = placement_grid(score_map, (0, 0), deformation, r, virt)
    ry0, ry1, rx0, rx1 = rect
    cy = scale * np.arange(ry0, ry1 + 1)[:, None] + anchor[0] + r
    cx = scale * np.arange(rx0, rx1 + 1)[None, :] + anchor[1] + r
    return placed[cy, cx], py[cy, cx], px[cy, cx]


def score_pyramid(levels, bank, C, cores, radius_mode="gdt", scale=None,
                  root_levels=None, part_levels=None, components=None):
    """Oracle for the batched pyramid path (configs 2-5).

    ``levels``: list of (H, W, L) float32 arrays; ``cores[f]``: (h, w, R)
    core of filter f over basis ``C`` (L, R).  For every component and root
    level returns a dict with the root rectangle, total scores (float64),
    and part positions (n_parts, hr, wr, 2).  ``radius_mode="gdt"`` uses the
    unbounded transform (radius r_star per part map, App. A.2) on the GDT
    root domain; an int uses that windowed radius on the same domain."""
    scale = bank.scale if scale is None else scale
    comps = bank.components if components is None else components
    P = [project(lv, C) for lv in levels]
    maps = {}

    def smap(k, f):
        if (k, f) not in maps:
            maps[(k, f)] = correlate3_full(P[k], cores[f])
        return maps[(k, f)]

    out = []
    for i, (kr, kp) in enumerate(zip(root_levels, part_levels)):
        Hr, Wr = levels[kr].shape[:2]
        Hp, Wp = levels[kp].shape[:2]
        for ci, comp in enumerate(comps):
            rh, rw = bank.filters[comp.root].shape[:2]
            if Hr - rh + 1 < 1 or Wr - rw + 1 < 1:
                continue
            psup = [(Hp - bank.filters[f].shape[0] + 1, Wp - bank.filters[f].shape[1] + 1)
                    for f in comp.parts]
            rect = _gdt_rect((Hr - rh + 1, Wr - rw + 1), psup, comp.anchors, scale)
            if rect is None:
                continue
            ry0, ry1, rx0, rx1 = rect
            tot = smap(kr, comp.root)[ry0:ry1 + 1, rx0:rx1 + 1].copy()
            pos = []
            for f, anc, de in zip(comp.parts, comp.anchors, comp.deformations):
                sm = smap(kp, f)
                rad = r_star(sm, de) if radius_mode == "gdt" else int(radius_mode)
                v, py, px = place_gathered(sm, anc, de, rad, scale, rect)
                tot = tot + v
                pos.append(np.stack([py, px], axis=-1))
            tot = tot + comp.bias
            out.append({"root_level": i, "component": ci, "rect": rect,
                        "scores": tot, "parts": np.stack(pos) if pos else None})
    return out, maps


def _gdt_rect(root_support, part_supports, anchors, scale):
    # SURVEY.md App. A.2 root domain: every part centre inside its support
    ry0, ry1, rx0, rx1 = 0, root_support[0] - 1, 0, root_support[1] - 1
    for (hp, wp), (ay, ax) in zip(part_supports, anchors):
        if hp < 1 or wp < 1:
            return None
        ry0, ry1 = max(ry0, -(ay // scale)), min(ry1, (hp - 1 - ay) // scale)
        rx0, rx1 = max(rx0, -(ax // scale)), min(rx1, (wp - 1 - ax) // scale)
    if ry0 > ry1 or rx0 > rx1:
        return None
    return ry0, ry1, rx0, rx1


# ------------------------------------------------- pruned detection (Alg. 1)

def dilate_any(mask, radius):
    """Box dilation onto a grid extended by ``radius`` on every side
    (detection.py:302-317): out[Y, X] is set when some mask cell lies within
    the (2r+1)^2 box centred at mask coordinate (Y - r, X - r)."""
    h, w = mask.shape
    out = np.zeros((h + 2 * radius, w + 2 * radius), dtype=bool)
    ys, xs = np.nonzero(mask)
    width = 2 * radius + 1
    for y, x in zip(ys, xs):
        out[y:y + width, x:x + width] = True
    return out


def covered_count(covered, rect, anchor, radius, support):
    """Part-map positions inside the union of alive search windows
    (detection.py:545-567)."""
    ry0, ry1, rx0, rx1 = rect
    ay, ax = anchor
    sy, sx = support
    py0, py1 = max(0, ry0 + ay - radius), min(sy - 1, ry1 + ay + radius)
    px0, px1 = max(0, rx0 + ax - radius), min(sx - 1, rx1 + ax + radius)
    if py0 > py1 or px0 > px1:
        return 0
    oy, ox = py0 - ay - (ry0 - radius), px0 - ax - (rx0 - radius)
    return int(covered[oy:oy + py1 - py0 + 1, ox:ox + px1 - px0 + 1].sum())


def window_max(stack_r, centres_y, centres_x, radius):
    """Max of a map over (2r+1)^2 windows at the given centres, -inf outside
    (detection.py:484-490)."""
    pad = np.pad(stack_r, radius, constant_values=-np.inf)
    from numpy.lib.stride_tricks import sliding_window_view
    win = sliding_window_view(pad, (2 * radius + 1, 2 * radius + 1))
    hp, wp = stack_r.shape
    out = np.full(centres_y.shape, -np.inf)
    ok = (centres_y + radius >= 0) & (centres_y - radius < hp) & \
         (centres_x + radius >= 0) & (centres_x - radius < wp)
    cy = np.clip(centres_y, 0, hp - 1)
    cx = np.clip(centres_x, 0, wp - 1)
    vals = win[cy, cx].max(axis=(-2, -1))
    # centres off the map: clip moved them; recompute those exactly
    off = ok & ((cy != centres_y) | (cx != centres_x))
    out[ok & ~off] = vals[ok & ~off]
    for i in np.flatnonzero(off):
        y, x = centres_y.flat[i], centres_x.flat[i]
        y0, y1 = max(y - radius, 0), min(y + radius, hp - 1)
        x0, x1 = max(x - radius, 0), min(x + radius, wp - 1)
        out.flat[i] = stack_r[y0:y1 + 1, x0:x1 + 1].max()
    return out


def detect_pruned(dec, pyramid, tau, part_prune_mode="kill", stacks=None):
    """``detect(..., pruning=True)`` (detection.py:386-542, pruning branches
    433-503): root positions die at the first rank whose prefix partial is
    below the root threshold; a part whose window-max prefix partial drops
    below its threshold kills the hypothesis ("kill") or contributes nothing
    ("lenient").  ``stacks(level_idx, level)`` may supply the rank-prefix
    maps (root_stack, [part_stacks]); default: ``cp_partial_stack``.

    Returns (detections, stats, prune_maps) with the reference's counters."""
    dets = []
    st = {"positions_examined": 0, "positions_pruned_at_rank": {}, "part_pruned_at_rank": {},
          "positions_killed_by_parts": 0, "multiplications": 0}
    maps = []

    def bump(table, r, n):
        if n:
            table[r] = table.get(r, 0) + int(n)

    for li, level in enumerate(pyramid):
        level = np.asarray(level, dtype=np.float64)
        rect = hypothesis_rect(level.shape, dec.root_cp.dims, [p.cp.dims for p in dec.parts],
                               [p.anchor for p in dec.parts],
                               [p.search_radius for p in dec.parts])
        lm = {"rect": rect}
        maps.append(lm)
        if rect is None:
            continue
        ry0, ry1, rx0, rx1 = rect
        hr, wr = ry1 - ry0 + 1, rx1 - rx0 + 1
        st["positions_examined"] += hr * wr
        if stacks is None:
            root_stack = cp_partial_stack(level, dec.root_cp)
            part_stacks = [cp_partial_stack(level, p.cp) for p in dec.parts]
        else:
            root_stack, part_stacks = stacks(li, level)
        root_rect = root_stack[:, ry0:ry1 + 1, rx0:rx1 + 1]
        alive = np.ones((hr, wr), dtype=bool)
        prune_rank = np.zeros((hr, wr), dtype=np.int64)
        n0, m0, l0 = dec.root_cp.dims
        for r in range(dec.root_cp.rank):
            st["multiplications"] += int(alive.sum()) * (n0 + m0 + l0)
            newly = alive & (root_rect[r] < dec.root_thresholds[r])
            bump(st["positions_pruned_at_rank"], r + 1, newly.sum())
            prune_rank[newly] = r + 1
            alive &= ~newly
        lm["root_prune_rank"] = prune_rank
        scores = root_rect[-1].copy()
        part_rank = np.zeros((len(dec.parts), hr, wr), dtype=np.int64)
        placements = []
        gy = np.arange(ry0, ry1 + 1)[:, None] + 0 * np.arange(wr)[None, :]
        gx = np.arange(rx0, rx1 + 1)[None, :] + 0 * np.arange(hr)[:, None]
        for pi, part in enumerate(dec.parts):
            if part_prune_mode == "kill" and not alive.any():
                break
            pstack = part_stacks[pi]
            n, m, l = part.cp.dims
            rad = part.search_radius
            ay, ax = part.anchor
            support = (level.shape[0] - n + 1, level.shape[1] - m + 1)
            part_alive = alive.copy()
            for r in range(part.cp.rank):
                if not part_alive.any():
                    break
                cov = covered_count(dilate_any(part_alive, rad), rect, (ay, ax), rad, support)
                st["multiplications"] += cov * (n + m + l)
                wmax = window_max(pstack[r], gy + ay, gx + ax, rad)
                newly = part_alive & (wmax < part.thresholds[r])
                if newly.any():
                    bump(st["part_pruned_at_rank"], r + 1, newly.sum())
                    part_rank[pi][newly] = r + 1
                    part_alive &= ~newly
                    if part_prune_mode == "kill":
                        st["positions_killed_by_parts"] += int((alive & newly).sum())
                        alive &= ~newly
            placed, py, px = placement_grid(pstack[-1], part.anchor, part.deformation, rad, rect)
            placements.append((part_alive, placed, py, px, part.anchor))
            contrib = np.where(part_alive, placed, 0.0) if part_prune_mode == "lenient" else placed
            scores = scores + contrib
        lm["part_prune_rank"] = part_rank
        scores = scores + dec.bias
        for iy, ix in zip(*np.nonzero(alive & (scores >= tau))):
            gyy, gxx = ry0 + iy, rx0 + ix
            pp = []
            for pa, _, py, px, anc in placements:
                if part_prune_mode == "lenient" and not pa[iy, ix]:
                    pp.append((int(gyy + anc[0]), int(gxx + anc[1])))
                else:
                    pp.append((int(py[iy, ix]), int(px[iy, ix])))
            dets.append((li, (int(gyy), int(gxx)), tuple(pp), float(scores[iy, ix])))
    dets.sort(key=lambda d: (d[0], d[1]))
    return dets, st, maps


def calibrate_thresholds(dec, positives, stacks=None):
    """Per-rank floors = min over positives of the prefix partials at the
    positive positions (detection.py:262-299).  Returns (root_thr, [part_thr])."""
    root_min, part_min = None, [None] * len(dec.parts)
    for level, hyp in positives:
        level = np.asarray(level, dtype=np.float64)
        if stacks is None:
            rs = cp_partial_stack(level, dec.root_cp)
            ps = [cp_partial_stack(level, p.cp) for p in dec.parts]
        else:
            rs, ps = stacks(level)
        v = rs[:, hyp.root[0], hyp.root[1]]
        root_min = v.copy() if root_min is None else np.minimum(root_min, v)
        for i, (s, pos) in enumerate(zip(ps, hyp.parts)):
            v = s[:, pos[0], pos[1]]
            part_min[i] = v.copy() if part_min[i] is None else np.minimum(part_min[i], v)
    return root_min, part_min
