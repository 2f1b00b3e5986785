"""Per-call latency of the drop-in correlation API with and without the plan
cache (plancache.py): reference-style loops call correlate3_cp /
cp_partial_stack / correlate3_full / cp_score_hypothesis once per image.
Wall clock per call (host-synchronous API: every call returns numpy), after
warm-up; prints one JSON line per (function, cache) pair."""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1707_03268_b200 as dpm  # noqa: E402
from paper_1707_03268_b200.types import CPModel  # noqa: E402


def main(n=40, shape=(60, 80, 32)):
    rng = np.random.default_rng(0)
    imgs = [rng.random(shape) for _ in range(n)]
    model = CPModel(weights=rng.random(8) + 0.5, factors_a=rng.normal(size=(6, 8)),
                    factors_b=rng.normal(size=(6, 8)), factors_c=rng.normal(size=(32, 8)) * 0.2)
    dense = rng.normal(size=(6, 6, 32))
    fns = {
        "correlate3_cp": lambda im: dpm.correlate3_cp(im, model),
        "cp_partial_stack": lambda im: dpm.cp_partial_stack(im, model),
        "correlate3_full": lambda im: dpm.correlate3_full(im, dense),
    }
    for cache in ("1", "0"):
        os.environ["DPM_PLAN_CACHE"] = cache
        dpm.clear_plan_cache()
        for name, fn in fns.items():
            for im in imgs[:3]:
                fn(im)
            t0 = time.perf_counter()
            for im in imgs:
                fn(im)
            dt = (time.perf_counter() - t0) / n
            print(json.dumps({"api": name, "plan_cache": cache == "1", "image": list(shape),
                              "ms_per_call": round(dt * 1e3, 3), "calls": n}), flush=True)


if __name__ == "__main__":
    main()
