"""Config 5 K2 comparison: the shortened correlation at
R = 8 and R = 32 on the shared basis against the dense 32-channel
correlation (C = identity, cores = the filters) on the same inputs.

    python tools/bench_k2_config5.py [--images 4] [--steps 5]

Times K1 + K2 (every root filter on its root level, every part filter on
its part level, 1920x1080 pyramids) with CUDA events and prints one JSON
line per variant plus a summary; the result is committed under profiles/.
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
    ap.add_argument("--images", type=int, default=4)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()

    import torch

    from paper_1707_03268_b200 import synth
    from paper_1707_03268_b200.engine import FilterDef, Plan
    from paper_1707_03268_b200.pipeline import cores_from_stacked

    wl = synth.workload(5)
    bank, pyr = wl.bank, wl.pyramid
    apps = []
    fits = lambda k, f: (bank.filters[f].shape[0] <= pyr.levels[k][0]  # noqa: E731
                         and bank.filters[f].shape[1] <= pyr.levels[k][1])
    for kr, kp in zip(pyr.root_levels, pyr.part_levels):
        for comp in bank.components:  # components that fit, as PyramidScorer plans them
            if fits(kr, comp.root) and all(fits(kp, f) for f in comp.parts):
                apps.append((kr, comp.root))
                apps.extend((kp, f) for f in comp.parts)
    apps = sorted(set(apps))
    evals = sum((pyr.levels[k][0] - bank.filters[f].shape[0] + 1) *
                (pyr.levels[k][1] - bank.filters[f].shape[1] + 1) for k, f in apps)

    # (name, C, filters, R, tensor cores): R = 8 both ways, so the decomposed-vs-dense
    # ratio is also quoted FFMA against FFMA (R = 32 and dense run FFMA either way)
    variants = []
    for R in (8, 32):
        fx = np.load(os.path.join(REPO, "paper_1707_03268_b200", "data", f"factors_cfg5_R{R}.npz"))
        cores = cores_from_stacked(bank, fx["G"])
        variants.append((f"decomposed R={R}", fx["C"], [FilterDef(c) for c in cores], R, True))
        if R == 8:
            variants.append(("decomposed R=8, FFMA only", fx["C"], [FilterDef(c) for c in cores],
                             R, False))
    dense = [FilterDef(np.ascontiguousarray(f, dtype=np.float32)) for f in bank.filters]
    variants.append(("dense 32-channel (C = I)", np.eye(32, dtype=np.float32), dense, 32, True))

    levels = [synth.hog_pyramid(5, img, pyr) for img in range(args.images)]
    out = []
    for name, C, filters, R, tc in variants:
        plan = Plan(32, pyr.levels, C, filters, apps=apps, n_images=args.images, outputs=(),
                    tensor_cores=tc)
        for img in range(args.images):
            plan.load_levels(img, levels[img])
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
        rec = {"variant": name, "rank": R, "images": args.images,
               "ms_per_batch": ms, "ms_per_image": ms / args.images,
               "evals_per_s": evals * args.images / (ms / 1e3),
               "k2_flops_per_image": plan.k2_flops(),
               "tflops": plan.k2_flops() * args.images / (ms / 1e3) / 1e12,
               "tensor_core_classes": len(plan._tc_classes)}
        out.append(rec)
        print(json.dumps(rec), flush=True)
        del plan
        torch.cuda.empty_cache()
    base = out[-1]["ms_per_image"]
    summary = {"config": "5 (1920x1080, roots 15x15 / 11x15 / 15x8, 8 parts 6x6, 3 mirrored pairs)",
               "evals_per_image": evals,
               "speedup_vs_dense": {r["variant"]: base / r["ms_per_image"] for r in out[:-1]},
               "timing": "K1 + K2, CUDA events, steady state, inputs device resident"}
    print(json.dumps(summary), flush=True)


if __name__ == "__main__":
    main()
