"""Ad-hoc K3 check: golden placement case(s) through _placement_grid with
the library in use (DPM_K3=v1 selects the round-1 kernel), against the
oracle on the same FP32 map.  python tools/k3_debug_run.py [case ...]"""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1707_03268_b200 as B  # noqa: E402
from oracle import dpm_oracle as O  # noqa: E402

g = np.load(os.path.join(REPO, "tests", "golden", "placement.npz"))
for k in [int(a) for a in sys.argv[1:]] or range(int(g["n"])):
    smap = g[f"p{k}_map"]
    anc, de, r = tuple(g[f"p{k}_anchor"]), tuple(g[f"p{k}_def"]), int(g[f"p{k}_r"])
    rect = tuple(int(v) for v in g[f"p{k}_rect"])
    part = B.PartSpec(np.zeros((1, 1, 1)), anc, de, r)
    placed, py, px = B._placement_grid(smap, part, rect)
    o, oy, ox = O.placement_grid(np.asarray(smap, np.float32).astype(np.float64), anc, de, r, rect)
    bad = ~((placed == o) | (np.isneginf(placed) & np.isneginf(o)))
    print(k, "shape", placed.shape, "neginf gpu", int(np.isneginf(placed).sum()), "oracle",
          int(np.isneginf(o).sum()), "value mismatches", int(bad.sum()),
          "pos mismatches", int(((py != oy) | (px != ox)).sum()))
    if bad.any():
        iy, ix = np.nonzero(bad)
        print("  first", list(zip(iy[:5], ix[:5])), placed[iy[:5], ix[:5]], o[iy[:5], ix[:5]])
