"""Value types crossing the drop-in boundary.

Field names and meanings follow the reference so objects built by
``cpdetect`` (``CPModel``, ``DecomposedModel``, ``PartModel`` ...) are accepted
unchanged by duck typing, and the objects returned here read the same:

* ``ScoreMap``            - correlation.py:44-61
* ``CPModel``             - decomposition.py:45-128 (weights, factors_a/b/c)
* ``PartSpec/PartModel``  - model.py:55-96
* ``DecomposedPart/DecomposedModel`` - model.py:99-168
* ``Hypothesis/Detection/DetectStats`` - detection.py:48-125
"""

from dataclasses import dataclass

import numpy as np

from .errors import ValidationError

__all__ = [
    "ScoreMap",
    "CPModel",
    "PartSpec",
    "PartModel",
    "DecomposedPart",
    "DecomposedModel",
    "Hypothesis",
    "Detection",
    "DetectStats",
]


@dataclass(frozen=True)
class ScoreMap:
    """2-D score array plus its multiplication count (correlation.py:44-61)."""

    scores: np.ndarray
    multiplications: int

    def __post_init__(self):
        s = np.asarray(self.scores, dtype=np.float64)
        if s.ndim != 2 or min(s.shape) < 1:
            raise ValidationError(f"score map must be 2-D and non-empty, got {s.shape}")
        object.__setattr__(self, "scores", s)
        object.__setattr__(self, "multiplications", int(self.multiplications))

    @property
    def shape(self):
        return self.scores.shape


@dataclass(frozen=True)
class CPModel:
    """Rank-R CP model: ``sum_r w_r a_r (x) b_r (x) c_r``.

    Same attribute contract as decomposition.py:45-94; construction checks
    only shapes and finiteness (canonicalisation is the decomposer's job,
    which stays in the reference package)."""

    weights: np.ndarray
    factors_a: np.ndarray
    factors_b: np.ndarray
    factors_c: np.ndarray

    def __post_init__(self):
        w = np.asarray(self.weights, dtype=np.float64)
        if w.ndim != 1 or w.size < 1:
            raise ValidationError("weights must be a non-empty 1-D array")
        object.__setattr__(self, "weights", w)
        for name in ("factors_a", "factors_b", "factors_c"):
            f = np.asarray(getattr(self, name), dtype=np.float64)
            if f.ndim != 2 or f.shape[1] != w.size:
                raise ValidationError(f"{name} must have {w.size} columns")
            if not np.isfinite(f).all():
                raise ValidationError(f"{name} contains non-finite values")
            object.__setattr__(self, name, f)

    @property
    def rank(self):
        return int(self.weights.size)

    @property
    def dims(self):
        return (self.factors_a.shape[0], self.factors_b.shape[0], self.factors_c.shape[0])

    @classmethod
    def from_factors(cls, a, b, c, weights=None):
        """Absorb column norms into weights and order terms by descending
        weight, stable (decomposition.py:96-128); negative weights fold
        their sign into ``c``."""
        mats = [np.array(m, dtype=np.float64, copy=True) for m in (a, b, c)]
        r = mats[0].shape[1]
        w = np.ones(r) if weights is None else np.asarray(weights, dtype=np.float64).copy()
        for m in mats:
            nrm = np.linalg.norm(m, axis=0)
            w = w * nrm
            zero = nrm == 0.0
            m /= np.where(zero, 1.0, nrm)
            m[:, zero] = 0.0
            m[0, zero] = 1.0
        sign = w < 0
        mats[2][:, sign] *= -1.0
        w = np.abs(w)
        order = np.argsort(-w, kind="stable")
        return cls(w[order], *(m[:, order] for m in mats))


def _as_filter(f, name):
    arr = np.asarray(f, dtype=np.float64)
    if arr.ndim != 3:
        raise ValidationError(f"{name} must be an order-3 array, got shape {arr.shape}")
    return np.ascontiguousarray(arr)


@dataclass(frozen=True)
class PartSpec:
    """Part filter, anchor, deformation (c_dx, c_dy, c_dxx, c_dyy), radius."""

    filter: np.ndarray
    anchor: tuple
    deformation: tuple
    search_radius: int

    def __post_init__(self):
        object.__setattr__(self, "filter", _as_filter(self.filter, "part filter"))
        object.__setattr__(self, "anchor", (int(self.anchor[0]), int(self.anchor[1])))
        if len(self.deformation) != 4:
            raise ValidationError("deformation must have 4 coefficients")
        object.__setattr__(self, "deformation", tuple(float(v) for v in self.deformation))
        object.__setattr__(self, "search_radius", int(self.search_radius))


@dataclass(frozen=True)
class PartModel:
    """Dense root filter + parts + bias (model.py:77-96)."""

    root: np.ndarray
    parts: tuple = ()
    bias: float = 0.0

    def __post_init__(self):
        object.__setattr__(self, "root", _as_filter(self.root, "root filter"))
        object.__setattr__(self, "parts", tuple(self.parts))
        object.__setattr__(self, "bias", float(self.bias))

    @property
    def channels(self):
        return self.root.shape[2]

    @property
    def filters(self):
        return (self.root,) + tuple(p.filter for p in self.parts)


@dataclass(frozen=True)
class DecomposedPart:
    """Part with a CP filter (model.py:99-123)."""

    cp: object
    anchor: tuple
    deformation: tuple
    search_radius: int
    thresholds: np.ndarray = None

    def __post_init__(self):
        object.__setattr__(self, "anchor", (int(self.anchor[0]), int(self.anchor[1])))
        object.__setattr__(self, "deformation", tuple(float(v) for v in self.deformation))
        object.__setattr__(self, "search_radius", int(self.search_radius))


@dataclass(frozen=True)
class DecomposedModel:
    """Root CP + decomposed parts + bias (model.py:126-168)."""

    root_cp: object
    parts: tuple = ()
    bias: float = 0.0
    root_thresholds: np.ndarray = None
    residuals: tuple = None

    def __post_init__(self):
        object.__setattr__(self, "parts", tuple(self.parts))
        object.__setattr__(self, "bias", float(self.bias))

    @property
    def channels(self):
        return self.root_cp.dims[2]

    @property
    def ranks(self):
        return (self.root_cp.rank,) + tuple(p.cp.rank for p in self.parts)

    @property
    def calibrated(self):
        if self.root_thresholds is None:
            return False
        return all(p.thresholds is not None for p in self.parts)


@dataclass(frozen=True)
class Hypothesis:
    """Root position + one position per part on a level (detection.py:48-63)."""

    level: int
    root: tuple
    parts: tuple = ()
    score: float = None

    def __post_init__(self):
        object.__setattr__(self, "root", (int(self.root[0]), int(self.root[1])))
        object.__setattr__(self, "parts", tuple((int(y), int(x)) for y, x in self.parts))
        if self.score is not None:
            object.__setattr__(self, "score", float(self.score))


@dataclass(frozen=True)
class Detection:
    """Hypothesis whose score cleared tau (detection.py:66-77)."""

    hypothesis: Hypothesis
    model_id: str
    score: float
    tau: float

    def __post_init__(self):
        if self.score < self.tau:
            raise ValidationError("detection score below its own threshold")


class DetectStats:
    """Work accounting for one detection run (detection.py:80-125)."""

    def __init__(self):
        self.positions_examined = 0
        self.positions_pruned_at_rank = {}
        self.part_pruned_at_rank = {}
        self.positions_killed_by_parts = 0
        self.multiplications = 0
        self.wall_time = 0.0
        self.prune_maps = None

    @property
    def positions_pruned(self):
        return sum(self.positions_pruned_at_rank.values())

    @property
    def positions_surviving(self):
        return self.positions_examined - self.positions_pruned

    def as_dict(self):
        return {
            "positions_examined": self.positions_examined,
            "positions_pruned": self.positions_pruned,
            "positions_surviving": self.positions_surviving,
            "positions_pruned_at_rank": {
                str(k): v for k, v in sorted(self.positions_pruned_at_rank.items())
            },
            "part_pruned_at_rank": {
                str(k): v for k, v in sorted(self.part_pruned_at_rank.items())
            },
            "positions_killed_by_parts": self.positions_killed_by_parts,
            "multiplications": self.multiplications,
            "wall_time": self.wall_time,
        }
