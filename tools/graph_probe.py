"""Direct launches vs CUDA-graph replay of one Plan.run() at small batches."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1707_03268_b200 import synth  # noqa: E402
from paper_1707_03268_b200.pipeline import PyramidScorer  # noqa: E402

wl = synth.workload(4)
fx = np.load(os.path.join(REPO, "paper_1707_03268_b200", "data", "factors_cfg4_R8.npz"))
lv = synth.hog_pyramid(4, 0, wl.pyramid)
for n in (2, 8):
    sc = PyramidScorer(wl.bank, fx["C"], fx["G"], wl.pyramid, n_images=n, max_dets=1 << 18)
    p = sc.plan
    for i in range(n):
        p.load_levels(i, lv)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            p.run(tau=2.6, stream=s)
    torch.cuda.synchronize()

    def timed(fn, reps=20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(reps):
                fn()
            e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    direct = timed(lambda: p.run(tau=2.6, stream=s))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        p.run(tau=2.6, stream=s)
    replay = timed(lambda: g.replay())
    print(f"{n} images: direct {direct:.3f} ms, graph replay {replay:.3f} ms")
