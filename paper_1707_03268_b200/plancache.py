"""Plans reused across drop-in calls.

The reference's correlation entry points are per-image functions
(``correlate3_cp``, ``cp_partial_stack``, ``correlate3_full``,
``score_hypothesis``: ``correlation.py:92-180``, ``detection.py:144-177``)
and its callers loop over them (``calibrate_thresholds``, ``roc_eval``,
the acceptance benchmarks).  Building a ``Plan`` per call -- layout, device
arenas, launch tables, TMA descriptors, ctypes prepares -- costs more than
the kernels at those sizes.  A plan's layout depends only on geometry,
filter shapes, rank-prefix families and the maps requested
(``engine.plan_signature``), so a plan of the same signature is rebound to
the new basis and cores (``Plan.rebind``, an in-place re-upload) and the
level is reloaded.

Threads: a cached plan is leased under its own lock; a caller that finds it
busy gets a fresh, uncached plan, so concurrent callers never share device
buffers.  ``DPM_PLAN_CACHE=0`` disables the cache.
"""

import os
import threading
from collections import OrderedDict

import numpy as np

from .engine import Plan, plan_signature

__all__ = ["lease", "clear_plan_cache", "plan_cache_info"]

MAX_PLANS = 8
_OPTS = ("correlation-maps",)  # the cache builds every plan with the same options
_LOCK = threading.Lock()
_CACHE = OrderedDict()  # signature -> (plan, lock)
_STATS = {"hits": 0, "misses": 0, "busy": 0}


class _Lease:
    def __init__(self, plan, lock):
        self.plan, self._lock = plan, lock

    def __enter__(self):
        return self.plan

    def __exit__(self, *exc):
        if self._lock is not None:
            self._lock.release()
        return False


def _new(L, levels, C, filters, apps):
    return Plan(L, levels, C, filters, apps=apps, outputs=())


def lease(L, levels, C, filters, apps):
    """Context manager yielding a correlation plan (no assemblies) for these
    maps with ``C`` and the filters' cores bound; levels must be loaded by
    the caller."""
    C = np.ascontiguousarray(C, dtype=np.float32)
    filters = list(filters)
    apps = [(int(a), int(b)) for a, b in apps]
    if os.environ.get("DPM_PLAN_CACHE", "1") == "0":
        return _Lease(_new(L, levels, C, filters, apps), None)
    key = plan_signature(L, levels, 1, C.shape[1], filters, tuple(sorted(set(apps))), _OPTS)
    with _LOCK:
        entry = _CACHE.get(key)
        if entry is not None:
            _CACHE.move_to_end(key)
    if entry is not None:
        plan, lock = entry
        if lock.acquire(blocking=False):
            try:
                plan.rebind(C, filters)
            except BaseException:
                lock.release()
                raise
            _STATS["hits"] += 1
            return _Lease(plan, lock)
        _STATS["busy"] += 1
        return _Lease(_new(L, levels, C, filters, apps), None)
    _STATS["misses"] += 1
    plan, lock = _new(L, levels, C, filters, apps), threading.Lock()
    lock.acquire()
    with _LOCK:
        if key not in _CACHE:
            _CACHE[key] = (plan, lock)
            while len(_CACHE) > MAX_PLANS:
                _CACHE.popitem(last=False)
        else:  # another thread cached one meanwhile: keep ours private
            lock.release()
            lock = None
    return _Lease(plan, lock)


def clear_plan_cache():
    """Drop every cached plan (their device buffers go with the last lease)."""
    with _LOCK:
        _CACHE.clear()


def plan_cache_info():
    """(cached plans, hits, misses, busy) -- busy = leases that found the
    cached plan in use and built a private one."""
    with _LOCK:
        return len(_CACHE), _STATS["hits"], _STATS["misses"], _STATS["busy"]
