"""Total K2 time of the config-4 step against the Plan's tc_min_width
(levels narrower than it run the FFMA kernel)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_03268_b200 import synth  # noqa: E402
from paper_1707_03268_b200.engine import Plan  # noqa: E402
from paper_1707_03268_b200.pipeline import PyramidScorer  # noqa: E402

wl = synth.workload(4)
fx = np.load(os.path.join(REPO, "paper_1707_03268_b200", "data", "factors_cfg4_R8.npz"))
n = 16
lv = synth.hog_pyramid(4, 0, wl.pyramid)
for width in (32, 24, 16, 8):
    sc = PyramidScorer(wl.bank, fx["C"], fx["G"], wl.pyramid, n_images=n)
    p = sc.plan
    if width != 64:  # rebuild the plan with another threshold
        p = Plan(p.L, p.levels, fx["C"], p.filters, assemblies=p.assemblies, n_images=n,
                 outputs=("totals",), tc_min_width=width)
    for i in range(n):
        p.load_levels(i, lv)
    for _ in range(3):
        p.run(stages=("project", "correlate"))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        p.run(stages=("project", "correlate"))
    e1.record()
    torch.cuda.synchronize()
    print(f"tc_min_width {width}: K1+K2 {e0.elapsed_time(e1) / 5 * 64 / n:.3f} ms per 64 images")
    del sc, p
    torch.cuda.empty_cache()
