"""Accuracy margin of the K2 paths per config: worst
|map - float64 oracle| / max |oracle map| on sampled levels, for the tcgen05
path (2xtf32 + bf16 correction) and the FFMA path on the same inputs.  Every
entry must be within the 1e-5 bar; with DPM_ACCURACY_OUT set the table is
written there as JSON lines (committed under profiles/)."""

import json
import os

import numpy as np
import pytest

from oracle import dpm_oracle as O
from paper_1707_03268_b200 import synth

pytestmark = pytest.mark.gpu

CASES = [  # (config, basis, sampled part/root levels)
    (2, "R4", (0, 14)), (2, "R8", (0, 14)), (2, "R16", (0, 14)), (2, "R32", (0, 14)),
    (3, "R16", (0, 25)), (4, "R8", (0, 20)), (5, "R8", (0, 19)), (5, "R32", (0, 19)),
    (5, "dense", (0, 19)),
]


def _inputs(cfg, basis):
    from conftest import REPO

    from paper_1707_03268_b200.pipeline import cores_from_stacked

    wl = synth.workload(cfg)
    if basis == "dense":
        C = np.eye(32, dtype=np.float32)
        cores = [np.ascontiguousarray(f, dtype=np.float32) for f in wl.bank.filters]
    else:
        fx = np.load(os.path.join(REPO, "paper_1707_03268_b200", "data",
                                  f"factors_cfg{cfg}_{basis}.npz"))
        C, cores = fx["C"], cores_from_stacked(wl.bank, fx["G"])
    return wl, C, cores


@pytest.mark.parametrize("cfg,basis,lv", CASES, ids=[f"cfg{c}-{b}" for c, b, _ in CASES])
def test_map_error_within_bar_on_both_k2_paths(cfg, basis, lv):
    from paper_1707_03268_b200.engine import FilterDef, Plan

    wl, C, cores = _inputs(cfg, basis)
    pyr = wl.pyramid
    levels = synth.hog_pyramid(cfg, 0, pyr)
    # the maps the detector computes: component roots on root levels, parts on
    # the matching part levels (up to 4 components per config)
    rng = np.random.default_rng(cfg)
    comps = wl.bank.components
    pick = sorted(rng.choice(len(comps), size=min(4, len(comps)), replace=False))
    fits = lambda k, f: (cores[f].shape[0] <= pyr.levels[k][0]  # noqa: E731
                         and cores[f].shape[1] <= pyr.levels[k][1])
    apps = set()
    for i in lv:
        kr, kp = pyr.root_levels[i], pyr.part_levels[i]
        for c in pick:
            comp = comps[c]
            if fits(kr, comp.root) and all(fits(kp, f) for f in comp.parts):
                apps.add((kr, comp.root))
                apps.update((kp, f) for f in comp.parts)
    apps = sorted(apps)
    sel = sorted({k for k, _ in apps})
    ref = {}
    for k in sel:
        P = O.project(levels[k].astype(np.float64), np.asarray(C, np.float64))
        for kk, f in apps:
            if kk == k:
                ref[(k, f)] = O.correlate3_full(P, cores[f].astype(np.float64))
    rows = []
    for tc in (True, False):
        plan = Plan(32, pyr.levels, C, [FilterDef(c) for c in cores], apps=apps, outputs=(),
                    tensor_cores=tc, tc_min_strips=0)
        plan.load_levels(0, levels)
        plan.run(stages=("project", "correlate"))
        worst, where = 0.0, None
        for k, f in apps:
            g = plan.map(0, k, f).double().cpu().numpy()
            r = ref[(k, f)]
            e = float(np.abs(g - r).max() / max(np.abs(r).max(), 1e-30))
            if e > worst:
                worst, where = e, (k, f, cores[f].shape)
        paths = sorted({c[0] for c in plan._tc_classes}) if tc else ["ffma"]
        rows.append({"config": cfg, "basis": basis, "tensor_cores": tc, "k2_paths": paths,
                     "maps": len(apps), "worst_err_over_max": worst,
                     "worst_map": [int(where[0]), int(where[1]), list(where[2])]})
        assert worst <= 1e-5, (worst, where, paths)
    out = os.environ.get("DPM_ACCURACY_OUT")
    if out:
        with open(out, "a") as fh:
            for r in rows:
                fh.write(json.dumps(r) + "\n")
