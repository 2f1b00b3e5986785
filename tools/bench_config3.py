"""Config 3: a 20-model bank, 1080 filters stacked on ONE
shared rank-16 basis, scored on one 1280x720 pyramid -- the large-N implicit
GEMM case.  Times K1 + K2 (every root filter on its root level, every part
filter on its part level) at R = 16 against the dense 32-channel correlation
(C = identity, cores = the filters) on the same inputs, with CUDA events.

    python tools/bench_config3.py [--steps 5]

Prints one JSON line per variant plus a summary; committed under profiles/.
"""

import argparse
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--tc-ranks", default="8,16",
                    help="ranks routed to tcgen05 (comma list; '8,16' adds the multi-group "
                         "generic-shape launch for the R = 16 groups)")
    args = ap.parse_args()
    tc_ranks = tuple(int(v) for v in args.tc_ranks.split(","))

    import torch

    from paper_1707_03268_b200 import synth
    from paper_1707_03268_b200.engine import FilterDef, Plan
    from paper_1707_03268_b200.pipeline import cores_from_stacked

    wl = synth.workload(3)
    bank, pyr = wl.bank, wl.pyramid
    fits = lambda k, f: (bank.filters[f].shape[0] <= pyr.levels[k][0]  # noqa: E731
                         and bank.filters[f].shape[1] <= pyr.levels[k][1])
    apps = []
    for kr, kp in zip(pyr.root_levels, pyr.part_levels):
        for comp in bank.components:
            if fits(kr, comp.root) and all(fits(kp, f) for f in comp.parts):
                apps.append((kr, comp.root))
                apps.extend((kp, f) for f in comp.parts)
    apps = sorted(set(apps))
    evals = sum((pyr.levels[k][0] - bank.filters[f].shape[0] + 1) *
                (pyr.levels[k][1] - bank.filters[f].shape[1] + 1) for k, f in apps)

    fx = np.load(os.path.join(REPO, "paper_1707_03268_b200", "data", "factors_cfg3_R16.npz"))
    cores = cores_from_stacked(bank, fx["G"])
    # (name, C, filters, R, tensor cores): the decomposed bank both ways, so the ratio
    # to dense (FFMA) is also quoted FFMA against FFMA
    variants = [("decomposed R=16 (shared basis)", fx["C"], [FilterDef(c) for c in cores], 16, True),
                ("decomposed R=16, FFMA only", fx["C"], [FilterDef(c) for c in cores], 16, False),
                ("dense 32-channel (C = I)", np.eye(32, dtype=np.float32),
                 [FilterDef(np.ascontiguousarray(f, dtype=np.float32)) for f in bank.filters], 32,
                 True)]
    levels = synth.hog_pyramid(3, 0, pyr)
    out = []
    for name, C, filters, R, tc in variants:
        plan = Plan(32, pyr.levels, C, filters, apps=apps, n_images=1, outputs=(),
                    tc_ranks=tc_ranks, tensor_cores=tc)
        plan.load_levels(0, levels)
        for _ in range(args.warmup):
            plan.run(stages=("project", "correlate"))
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(args.steps):
            plan.run(stages=("project", "correlate"))
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / args.steps
        rec = {"variant": name, "rank": R, "filters": len(bank.filters), "applications": len(apps),
               "ms": ms, "evals_per_s": evals / (ms / 1e3),
               "k2_flops": plan.k2_flops(), "tflops": plan.k2_flops() / (ms / 1e3) / 1e12,
               "tensor_core_classes": [c[0] for c in plan._tc_classes], "tc_ranks": list(tc_ranks)}
        out.append(rec)
        print(json.dumps(rec), flush=True)
        del plan
        torch.cuda.empty_cache()
    summary = {"config": "3 (20-model bank, 1080 filters, shared rank-16 basis, 1280x720 pyramid)",
               "evals": evals,
               "speedup_vs_dense": {r["variant"]: out[-1]["ms"] / r["ms"] for r in out[:-1]},
               "timing": "K1 + K2, CUDA events, steady state, inputs device resident"}
    print(json.dumps(summary), flush=True)


if __name__ == "__main__":
    main()
