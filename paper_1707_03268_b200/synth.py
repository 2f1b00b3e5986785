"""Seeded synthetic workloads standing in for the paper's datasets.

BASELINE.json's five configs are fully synthetic; the
paper's PASCAL/INRIA images and trained DPM v5 models are not shipped by
the reference.  Seeding follows the reference's style
(``np.random.default_rng``, float32 quantisation as in
``synthetic.py:184``):

* HOG level ``(cfg, image, level)``: channels 0..30 ~ U[0, 0.4), channel 31
  exactly 0, float32, seed ``default_rng([cfg, image, level])``.
* Filters: N(0, 0.05) float32, seed ``default_rng([cfg, 1000 + model])``,
  drawn pair by pair, root first then parts; the odd component of a
  mirrored pair is the x-flip of the even one (no channel permutation,
  anchors mirrored, c_dx negated) - SURVEY.md App. A.5.
* Deformation (c_dx, c_dy, c_dxx, c_dyy) = (0, 0, 0.01, 0.01): the config's
  "(0.01,0,0.01,0)" read in DPM-v5 order.
"""

from dataclasses import dataclass

import numpy as np

from .geometry import Pyramid, build_pyramid

__all__ = [
    "Component",
    "FilterBank",
    "Workload",
    "hog_level",
    "hog_pyramid",
    "make_bank",
    "workload",
    "DEFAULT_ANCHORS_S1",
    "DEFORMATION",
]

L_HOG = 32
DEFORMATION = (0.0, 0.0, 0.01, 0.01)
# Anchor grid of the reference's default geometry (synthetic.py:39-42), used
# by config 1 (single-resolution parts, s = 1).
DEFAULT_ANCHORS_S1 = (
    (-5, -4), (-5, 4), (-5, 12), (-5, 20),
    (3, -4), (3, 4), (3, 12), (3, 20),
)


@dataclass(frozen=True)
class Component:
    """One mixture component: root filter + parts (indices into the bank)."""

    root: int
    parts: tuple
    anchors: tuple
    deformations: tuple
    bias: float
    search_radius: int = 2  # windowed placement radius (reference semantics)


@dataclass(frozen=True)
class FilterBank:
    """All filters of one or more models, in stacking order, plus components."""

    filters: tuple
    components: tuple
    scale: int

    @property
    def n_filters(self):
        return len(self.filters)

    def stacked(self):
        """The order-3 stacked tensor (sum_f h_f w_f, 1, L) of App. A.3."""
        rows = [f.reshape(-1, f.shape[2]) for f in self.filters]
        return np.concatenate(rows, axis=0)[:, None, :].astype(np.float64)

    def offsets(self):
        off, out = 0, []
        for f in self.filters:
            out.append(off)
            off += f.shape[0] * f.shape[1]
        return tuple(out)


@dataclass(frozen=True)
class Workload:
    cfg: int
    image_hw: tuple
    n_images: int
    bank: FilterBank
    pyramid: Pyramid
    ranks: tuple


def hog_level(cfg, image, level, H, W, L=L_HOG):
    rng = np.random.default_rng([cfg, image, level])
    x = np.zeros((H, W, L), dtype=np.float32)
    x[:, :, : L - 1] = rng.random((H, W, L - 1), dtype=np.float32) * np.float32(0.4)
    return x


def hog_pyramid(cfg, image, pyramid, L=L_HOG):
    return [hog_level(cfg, image, k, h, w, L) for k, (h, w) in enumerate(pyramid.levels)]


def _s2_anchors(root_hw, part_hw=(6, 6)):
    """Two rows of four parts inside the 2x root box."""
    ymax = 2 * root_hw[0] - part_hw[0]
    xmax = 2 * root_hw[1] - part_hw[1]
    ys = (0, ymax)
    xs = (0, int(round(xmax / 3)), int(round(2 * xmax / 3)), xmax)
    return tuple((y, x) for y in ys for x in xs)


def make_bank(cfg, model, root_shapes, scale, n_parts=8, part_hw=(6, 6),
              anchors=None, mirrored=True, search_radius=2, L=L_HOG):
    """Filters + components of one model (``root_shapes`` = one per pair)."""
    rng = np.random.default_rng([cfg, 1000 + model])
    filters, comps = [], []

    def draw(shape):
        return rng.normal(0.0, 0.05, size=shape).astype(np.float32)

    for rh, rw in root_shapes:
        root = draw((rh, rw, L))
        parts = [draw((part_hw[0], part_hw[1], L)) for _ in range(n_parts)]
        bias = round(float(rng.normal(0.0, 0.1)), 4)
        anc = anchors if anchors is not None else _s2_anchors((rh, rw), part_hw)
        anc = tuple(anc[:n_parts])
        members = [(root, parts, anc, DEFORMATION)]
        if mirrored:
            span = scale * rw - part_hw[1]
            m_anc = tuple((ay, span - ax) for ay, ax in anc)
            m_def = (-DEFORMATION[0],) + DEFORMATION[1:]
            members.append((
                np.ascontiguousarray(root[:, ::-1, :]),
                [np.ascontiguousarray(p[:, ::-1, :]) for p in parts],
                m_anc, m_def,
            ))
        for r, ps, an, de in members:
            base = len(filters)
            filters.append(r)
            filters.extend(ps)
            comps.append(Component(
                root=base,
                parts=tuple(range(base + 1, base + 1 + len(ps))),
                anchors=an,
                deformations=tuple(de for _ in ps),
                bias=bias,
                search_radius=search_radius,
            ))
    return filters, comps


def workload(cfg):
    """The five BASELINE.json configs."""
    if cfg == 1:
        filters, comps = make_bank(1, 0, [(6, 11)], scale=1, anchors=DEFAULT_ANCHORS_S1,
                                   mirrored=False)
        pyr = Pyramid(levels=((64, 48),), root_levels=(0,), part_levels=(0,), scale=1)
        return Workload(1, (64 * 8, 48 * 8), 1, FilterBank(tuple(filters), tuple(comps), 1),
                        pyr, (8,))
    if cfg in (2, 4):
        filters, comps = make_bank(cfg, 0, [(6, 11)] * 3, scale=2)
        hw = (480, 640) if cfg == 2 else (720, 1280)
        pyr = build_pyramid(hw[0], hw[1], [(6, 11)])
        ranks = (4, 8, 16, 32) if cfg == 2 else (8,)
        return Workload(cfg, hw, 1 if cfg == 2 else 64,
                        FilterBank(tuple(filters), tuple(comps), 2), pyr, ranks)
    if cfg == 3:
        filters, comps = [], []
        shape_rng = np.random.default_rng([3, 999])
        for model in range(20):
            shapes = [(int(shape_rng.integers(5, 9)), int(shape_rng.integers(8, 16)))
                      for _ in range(3)]
            f, c = make_bank(3, model, shapes, scale=2)
            base = len(filters)
            filters.extend(f)
            comps.extend(
                Component(x.root + base, tuple(p + base for p in x.parts), x.anchors,
                          x.deformations, x.bias, x.search_radius) for x in c)
        pyr = build_pyramid(720, 1280, [filters[c.root].shape[:2] for c in comps])
        return Workload(3, (720, 1280), 1, FilterBank(tuple(filters), tuple(comps), 2),
                        pyr, (16,))
    if cfg == 5:
        filters, comps = make_bank(5, 0, [(15, 15), (11, 15), (15, 8)], scale=2)
        pyr = build_pyramid(1080, 1920, [(15, 15), (11, 15), (15, 8)])
        return Workload(5, (1080, 1920), 1, FilterBank(tuple(filters), tuple(comps), 2),
                        pyr, (8, 32))
    raise ValueError(f"unknown config {cfg}")
