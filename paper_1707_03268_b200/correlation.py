"""Drop-in correlation engines on the B200 (K1 projection + K2 implicit GEMM).

Same names, arguments, return types and errors as the reference's
``cpdetect.correlation`` (``correlation.py:44-220``); scores are computed in
FP32 on the GPU and returned as float64 arrays (parity bar: 1e-5 of the
map's max |score|).

* ``correlate3_cp(img, model, upto_rank)``  (correlation.py:155-167): the CP
  model becomes one filter over its own ``c``-projected channels with core
  ``G[i, j, r] = w_r a[i, r] b[j, r]`` (ranks >= upto zeroed).
* ``cp_partial_stack(img, model, upto_rank)`` (correlation.py:170-180):
  prefix ``k`` is a filter whose core keeps ranks <= k; every prefix runs the
  same FMA sequence as ``correlate3_cp(upto=k+1)``, so the two stay
  bit-identical on the GPU as they are in the reference.
* ``correlate3_full(img, filt)`` (correlation.py:92-112): basis = identity.
"""

import numpy as np

from .engine import FilterDef
from .errors import ValidationError, check_feature_map, check_tensor3
from .geometry import (cp_multiplications, full_multiplications, theoretical_gain,
                       valid_support)
from .plancache import lease
from .types import ScoreMap

__all__ = [
    "ScoreMap",
    "valid_support",
    "correlate3_full",
    "correlate3_cp",
    "cp_partial_stack",
    "full_multiplications",
    "cp_multiplications",
    "theoretical_gain",
    "cp_core",
]


def _checked_upto(model, upto_rank):
    # correlation.py:146-152
    upto = model.rank if upto_rank is None else upto_rank
    if not 1 <= upto <= model.rank:
        raise ValidationError(f"upto_rank must be in [1, {model.rank}], got {upto_rank}")
    return upto


def cp_core(model, keep=None):
    """(n, m, R) core of a CP model: w_r a_ir b_jr, ranks >= keep zeroed."""
    a = np.asarray(model.factors_a, dtype=np.float64)
    b = np.asarray(model.factors_b, dtype=np.float64)
    w = np.asarray(model.weights, dtype=np.float64)
    core = np.einsum("ir,jr,r->ijr", a, b, w)
    if keep is not None:
        core[:, :, keep:] = 0.0
    return core.astype(np.float32)


def _run_maps(img, C, filters):
    """Maps of every filter on one level, through a cached plan of this
    layout (plancache: repeated calls rebind basis / cores instead of
    building a plan)."""
    H, W, L = img.shape
    with lease(L, [(H, W)], C, filters, [(0, f) for f in range(len(filters))]) as plan:
        plan.load_levels(0, [img.astype(np.float32)])
        plan.run(stages=("project", "correlate"))
        return [plan.map(0, 0, f).double().cpu().numpy() for f in range(len(filters))]


def correlate3_cp(img, model, upto_rank=None):
    """Separable CP correlation with the first ``upto_rank`` terms."""
    img = check_feature_map(img)
    upto = _checked_upto(model, upto_rank)
    valid_support(img.shape, model.dims)
    C = np.asarray(model.factors_c, dtype=np.float32)
    # the rank-prefix kernel (one pass over the ranks) gives prefixes 1..upto;
    # the last is the response -- bit-identical to cp_partial_stack's
    core = cp_core(model)
    m = _run_maps(img, C, [FilterDef(core, prefix=k + 1) for k in range(upto)])[-1]
    return ScoreMap(m, cp_multiplications(img.shape, model.dims, upto))


def cp_partial_stack(img, model, upto_rank=None):
    """Cumulative rank-prefix maps, shape (upto_rank, H', W')."""
    img = check_feature_map(img)
    upto = _checked_upto(model, upto_rank)
    valid_support(img.shape, model.dims)
    C = np.asarray(model.factors_c, dtype=np.float32)
    core = cp_core(model)
    filters = [FilterDef(core, prefix=k + 1) for k in range(upto)]
    return np.stack(_run_maps(img, C, filters))


def correlate3_full(img, filt):
    """Dense valid correlation: ``score[y, x] = sum filt[i,j,k] img[y+i, x+j, k]``."""
    img = check_feature_map(img)
    filt = check_tensor3(filt, "filter")
    valid_support(img.shape, filt.shape)
    L = img.shape[2]
    (m,) = _run_maps(img, np.eye(L, dtype=np.float32), [FilterDef(filt.astype(np.float32))])
    return ScoreMap(m, full_multiplications(img.shape, filt.shape))
