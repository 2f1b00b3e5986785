"""Parity helpers shared by the GPU tests and smoke().

Bars (BASELINE.json north_star):
  * response maps and totals: max |gpu - oracle| <= 1e-5 * max |oracle|;
  * part argmaxes: bit-exact except at ties.  A mismatch is an
    "exact tie" when the oracle's penalised value at the GPU's choice is
    within 4 float64 ulps of the oracle's best, a "near tie" when within
    1e-5 * max |S| (FP32 vs FP64 maps), else an error.  Zero errors allowed.
  * kernel-isolated placement (oracle run on the GPU's own FP32 maps):
    values and argmaxes bit-identical.
"""

import numpy as np

MAP_RTOL = 1e-5


def assert_map_close(gpu, ref, what="map", rtol=MAP_RTOL):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert gpu.shape == ref.shape, (what, gpu.shape, ref.shape)
    scale = max(float(np.abs(ref).max()), 1e-30)
    err = float(np.abs(gpu - ref).max()) if ref.size else 0.0
    assert err <= rtol * scale, f"{what}: max err {err:.3e} > {rtol:.0e} * {scale:.3e}"
    return err / scale


def classify_positions(gpu_pos, ref_pos, value_at, best, map_scale):
    """Count (exact, near_tie, error) over mismatching argmaxes.

    ``value_at(i, pos)`` returns the oracle's penalised value of candidate
    ``pos`` for element ``i``; ``best[i]`` is the oracle's best value."""
    gpu_pos = np.asarray(gpu_pos).reshape(-1, 2)
    ref_pos = np.asarray(ref_pos).reshape(-1, 2)
    best = np.asarray(best, dtype=np.float64).reshape(-1)
    bad = np.nonzero(np.any(gpu_pos != ref_pos, axis=1))[0]
    exact = near = err = 0
    for i in bad:
        v = value_at(i, tuple(gpu_pos[i]))
        gap = best[i] - v
        if gap <= 4 * np.spacing(abs(best[i])):
            exact += 1
        elif gap <= MAP_RTOL * map_scale:
            near += 1
        else:
            err += 1
    return exact, near, err


def penalised(S, centre, pos, deformation):
    """Oracle value of placing at ``pos`` for window centre ``centre``."""
    cdx, cdy, cdxx, cdyy = deformation
    dy, dx = pos[0] - centre[0], pos[1] - centre[1]
    if not (0 <= pos[0] < S.shape[0] and 0 <= pos[1] < S.shape[1]):
        return -np.inf
    return (S[pos[0], pos[1]] - (cdx * dx + cdxx * dx * dx)) - (cdy * dy + cdyy * dy * dy)
