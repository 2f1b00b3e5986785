"""Plan reuse across drop-in calls (plancache.py): the layout key on CPU, and
on the GPU that cached plans rebound to new inputs give the same maps as
fresh plans, also under concurrent callers."""

import threading

import numpy as np
import pytest

from paper_1707_03268_b200.engine import FilterDef, plan_signature


def _sig(filters, levels=((20, 30),), R=8):
    return plan_signature(32, levels, 1, R, filters, ((0, 0),), ("x",))


def test_signature_is_layout_not_values():
    rng = np.random.default_rng(0)
    a = rng.normal(size=(6, 6, 8)).astype(np.float32)
    b = rng.normal(size=(6, 6, 8)).astype(np.float32)
    # same shapes, different values -> same key
    assert _sig([FilterDef(a)]) == _sig([FilterDef(b)])
    # rank-prefix families keyed by first member, not by array identity
    fa = [FilterDef(a, prefix=k + 1) for k in range(3)]
    fb = [FilterDef(b, prefix=k + 1) for k in range(3)]
    assert _sig(fa) == _sig(fb)
    # one family of 3 vs three families of 1 prefix each: different layouts
    split = [FilterDef(a, prefix=1), FilterDef(b, prefix=2), FilterDef(a.copy(), prefix=3)]
    assert _sig(split) != _sig(fa)
    # shape, channel offset, geometry and rank change the key
    assert _sig([FilterDef(a[:5])]) != _sig([FilterDef(a)])
    assert _sig([FilterDef(a, chan_off=8)], R=16) != _sig([FilterDef(a)], R=16)
    assert _sig([FilterDef(a)], levels=((21, 30),)) != _sig([FilterDef(a)])
    assert _sig([FilterDef(a)], R=16) != _sig([FilterDef(a)])


def _model(rng, dims=(6, 6), L=32, R=8):
    from paper_1707_03268_b200.types import CPModel

    return CPModel(factors_a=rng.normal(size=(dims[0], R)), factors_b=rng.normal(size=(dims[1], R)),
                   factors_c=rng.normal(size=(L, R)) * 0.2, weights=rng.random(R) + 0.5)


@pytest.mark.gpu
def test_cached_plans_match_fresh_plans(monkeypatch):
    import paper_1707_03268_b200 as dpm

    rng = np.random.default_rng(5)
    calls = []
    for k in range(6):  # same layout, new images and models every call
        img = rng.random((40, 70, 32)).astype(np.float64)
        calls.append((img, _model(rng)))
    calls.append((rng.random((33, 50, 32)), _model(rng, dims=(5, 7))))  # another layout
    dpm.clear_plan_cache()
    _, h0, m0, _ = dpm.plan_cache_info()
    cached = [(dpm.correlate3_cp(i, m, 5).scores, dpm.cp_partial_stack(i, m),
               dpm.correlate3_full(i, np.asarray(m.factors_a)[:, None, :1] * np.ones((1, 4, 32))).scores)
              for i, m in calls]
    n, h1, m1, _ = dpm.plan_cache_info()
    assert h1 - h0 >= 3 * 5 and n >= 4  # every call after the first of a layout was a hit
    monkeypatch.setenv("DPM_PLAN_CACHE", "0")
    fresh = [(dpm.correlate3_cp(i, m, 5).scores, dpm.cp_partial_stack(i, m),
              dpm.correlate3_full(i, np.asarray(m.factors_a)[:, None, :1] * np.ones((1, 4, 32))).scores)
             for i, m in calls]
    for c, f in zip(cached, fresh):
        for x, y in zip(c, f):
            np.testing.assert_array_equal(x, y)


@pytest.mark.gpu
def test_cached_plans_under_concurrent_callers():
    import paper_1707_03268_b200 as dpm

    rng = np.random.default_rng(6)
    work = [(rng.random((36, 60, 32)), _model(rng)) for _ in range(12)]
    expect = [dpm.cp_partial_stack(i, m) for i, m in work]
    got = [None] * len(work)
    errors = []

    def run(t):
        try:
            for _ in range(3):
                for k in range(t, len(work), 4):
                    got[k] = dpm.cp_partial_stack(*work[k])
        except BaseException as exc:  # surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=run, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for e, g in zip(expect, got):
        np.testing.assert_array_equal(e, g)
