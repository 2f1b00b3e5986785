"""End to end from images: config 4's 64 x 1280x720 model and pyramid
geometry, fed seeded RGB uint8 images (tests/test_hog.scene) through
PyramidScorer.score_images -- pinned H2D of the images (177 MB per step
instead of 3.6 GB of float32 HOG), the device HOG pyramid builder, K1-K4
and the detection read-back.  Prints one JSON line.

    python tools/bench_images.py [--images 64] [--steps 5] [--warmup 3]
"""
import argparse
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=64)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--chunk", type=int, default=16)
    args = ap.parse_args()

    import torch

    from paper_1707_03268_b200 import synth
    from paper_1707_03268_b200.pipeline import PyramidScorer
    from test_hog import scene

    wl = synth.workload(4)
    fx = np.load(os.path.join(REPO, "paper_1707_03268_b200", "data", "factors_cfg4_R8.npz"))
    hh, ww = wl.image_hw
    base = [scene(hh, ww, 100 + i) for i in range(8)]
    imgs = np.stack([base[i % 8] for i in range(args.images)])
    host = torch.from_numpy(imgs).pin_memory()
    sc = PyramidScorer(wl.bank, fx["C"], fx["G"], wl.pyramid, n_images=args.images,
                       max_dets=1 << 20)
    d = sc.score_images(host, tau=1e9, chunk_images=args.chunk)
    tot = np.concatenate([sc.plan.assembly_outputs(0, a)["totals"].cpu().numpy().ravel()
                          for a in range(len(sc.plan.assemblies))])
    tau = float(np.quantile(tot, 0.999))
    for _ in range(args.warmup):
        sc.score_images(host, tau, chunk_images=args.chunk)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    n = []
    ev[0].record()
    for _ in range(args.steps):
        n.append(len(sc.score_images(host, tau, chunk_images=args.chunk)))
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / args.steps
    # device-only HOG builder time (images already resident)
    hb = sc._hog
    hb.run(sc._dev_images)
    e2 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e2[0].record()
    for _ in range(args.steps):
        hb.run(sc._dev_images)
    e2[1].record()
    torch.cuda.synchronize()
    hog_ms = e2[0].elapsed_time(e2[1]) / args.steps
    evals = sc.evals_per_image() * args.images
    print(json.dumps({
        "what": "e2e from uint8 RGB images (device HOG pyramid + K1-K4 + detections)",
        "images": args.images, "image_hw": [hh, ww], "ms_per_step": ms,
        "evals_per_s": evals / (ms / 1e3), "images_per_s": args.images / (ms / 1e3),
        "h2d_bytes_per_step": sc.image_bytes(host), "hog_ms_device": hog_ms,
        "detections_per_step": float(np.mean(n)), "tau": tau}), flush=True)


if __name__ == "__main__":
    main()
