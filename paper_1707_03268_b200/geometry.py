"""Integer geometry of the scoring path: supports, root rectangles, pyramids.

Everything here is exact integer arithmetic shared by the host planner, the
tests and the bench; none of it touches floating-point scores.

* ``valid_support`` / multiplication counters - correlation.py:64-89, 216-220
* ``hypothesis_rect``  - detection.py:210-235 (reference root rectangle)
* ``gdt_root_rect``    - SURVEY.md App. A.2 (DPM root domain for the
  unbounded transform at part scale ``s``)
* ``Pyramid``          - SURVEY.md §8(d): 4-px cell pyramid, 10 levels per
  octave; root level ``i`` is pyramid level ``i + 10`` and its parts are
  scored on level ``i`` (one octave finer).
"""

import math
from dataclasses import dataclass

from .errors import ValidationError

__all__ = [
    "valid_support",
    "full_multiplications",
    "cp_multiplications",
    "theoretical_gain",
    "hypothesis_rect",
    "gdt_root_rect",
    "Pyramid",
    "build_pyramid",
]


def valid_support(img_shape, filt_dims):
    """Output extents (H-n+1, W-m+1) of a valid correlation (correlation.py:64-75)."""
    H, W, L = img_shape
    n, m, l = filt_dims
    if l != L:
        raise ValidationError(f"channel mismatch: filter has {l}, image has {L}")
    ho, wo = H - n + 1, W - m + 1
    if ho < 1 or wo < 1:
        raise ValidationError(f"filter extent ({n}, {m}) exceeds image extent ({H}, {W})")
    return ho, wo


def full_multiplications(img_shape, filt_dims):
    """H'*W'*n*m*l (correlation.py:78-82)."""
    ho, wo = valid_support(img_shape, filt_dims)
    n, m, l = filt_dims
    return ho * wo * n * m * l


def cp_multiplications(img_shape, filt_dims, rank):
    """rank*H'*W'*(n+m+l) (correlation.py:85-89)."""
    ho, wo = valid_support(img_shape, filt_dims)
    n, m, l = filt_dims
    return rank * ho * wo * (n + m + l)


def theoretical_gain(n, m, l, rank):
    """nml / (R(n+m+l)) (correlation.py:216-220)."""
    if min(n, m, l, rank) < 1:
        raise ValidationError("extents and rank must be positive")
    return (n * m * l) / (rank * (n + m + l))


def _part_dims(part):
    return part.cp.dims if hasattr(part, "cp") else part.filter.shape


def hypothesis_rect(level_shape, root_dims, parts):
    """Inclusive (ry0, ry1, rx0, rx1) of roots whose every part window meets
    the part's valid support, or None (detection.py:210-235)."""
    H, W = level_shape[0], level_shape[1]
    n0, m0 = root_dims[0], root_dims[1]
    if H - n0 + 1 < 1 or W - m0 + 1 < 1:
        return None
    ry0, ry1, rx0, rx1 = 0, H - n0, 0, W - m0
    for part in parts:
        d = _part_dims(part)
        sy, sx = H - d[0] + 1, W - d[1] + 1
        if sy < 1 or sx < 1:
            return None
        ay, ax = part.anchor
        r = part.search_radius
        ry0 = max(ry0, -ay - r)
        ry1 = min(ry1, sy - 1 - ay + r)
        rx0 = max(rx0, -ax - r)
        rx1 = min(rx1, sx - 1 - ax + r)
    if ry0 > ry1 or rx0 > rx1:
        return None
    return ry0, ry1, rx0, rx1


def gdt_root_rect(root_support, part_supports, anchors, scale):
    """Roots whose every part centre ``scale*root + anchor`` lies inside the
    part's valid support (SURVEY.md App. A.2 root domain).

    ``root_support`` = (Hr', Wr'); ``part_supports[i]`` = (Hp', Wp').
    Returns inclusive (ry0, ry1, rx0, rx1) or None."""
    ry0, ry1, rx0, rx1 = 0, root_support[0] - 1, 0, root_support[1] - 1
    if ry1 < 0 or rx1 < 0:
        return None
    for (hp, wp), (ay, ax) in zip(part_supports, anchors):
        if hp < 1 or wp < 1:
            return None
        # 0 <= s*ry + ay <= hp-1   <=>   ceil(-ay/s) <= ry <= floor((hp-1-ay)/s)
        ry0 = max(ry0, -((ay) // scale))
        ry1 = min(ry1, (hp - 1 - ay) // scale)
        rx0 = max(rx0, -((ax) // scale))
        rx1 = min(rx1, (wp - 1 - ax) // scale)
    if ry0 > ry1 or rx0 > rx1:
        return None
    return ry0, ry1, rx0, rx1


@dataclass(frozen=True)
class Pyramid:
    """Feature-pyramid geometry.

    ``levels[k]`` = (H, W) in cells of pyramid level ``k``; ``root_levels[i]``
    is the level index holding root level ``i`` and ``part_levels[i]`` the
    level its parts are scored on; ``scale`` is the part/root resolution
    ratio (1 = reference single-resolution model, 2 = DPM octave parts)."""

    levels: tuple
    root_levels: tuple
    part_levels: tuple
    scale: int

    @property
    def n_cells(self):
        return sum(h * w for h, w in self.levels)


def build_pyramid(img_h, img_w, root_shapes, interval=10, cell=8, scale=2):
    """Pyramid of an ``img_h x img_w`` image.

    Level ``k`` has ``floor(img * 2^(-k/interval) * scale / cell)`` cells per
    axis (``cell/scale``-px cells); root level ``i`` is level ``i + interval``
    when ``scale == 2``.  Root levels continue while the level still holds
    at least one of ``root_shapes`` (a list of (h, w))."""
    if scale not in (1, 2):
        raise ValidationError("scale must be 1 or 2")
    off = interval if scale == 2 else 0

    def shape(k):
        f = 2.0 ** (-k / interval) * scale / cell
        return (int(math.floor(img_h * f)), int(math.floor(img_w * f)))

    n_root = 0
    while True:
        h, w = shape(n_root + off)
        if not any(h >= rh and w >= rw for rh, rw in root_shapes):
            break
        n_root += 1
    if n_root == 0:
        raise ValidationError("image too small for the smallest root filter")
    levels = tuple(shape(k) for k in range(n_root + off))
    root_levels = tuple(i + off for i in range(n_root))
    part_levels = tuple(range(n_root)) if scale == 2 else root_levels
    return Pyramid(levels, root_levels, part_levels, scale)
