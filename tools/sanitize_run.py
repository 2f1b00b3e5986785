"""Small end-to-end runs of every kernel of the path, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

  compute-sanitizer --tool racecheck python tools/sanitize_run.py [what ...]

what: cfg1 (K1-K4 on config 1, windowed placement), cfg4 (two config-4
images: tcgen05 K2 roots + parts, FFMA K2, windowed K3/K4 with TMA band
staging and tau compaction), envelope (the same images through the GDT
lower-envelope pair), prune (detect(pruning=True) both part modes on the
golden pruned fixture: rank-prefix K2 + dpm_prune_ranks), mixture
(dpm_mixture_max), ffma (config 5 R = 32: the chunked FFMA K2 with large
roots).  Each prints one line; the sanitizer's summary follows.
"""

import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def _factors(cfg, R):
    fx = np.load(os.path.join(REPO, "paper_1707_03268_b200", "data", f"factors_cfg{cfg}_R{R}.npz"))
    return fx["C"], fx["G"]


def cfg1():
    from paper_1707_03268_b200 import synth
    from paper_1707_03268_b200.pipeline import PyramidScorer

    wl = synth.workload(1)
    C, G = _factors(1, 8)
    sc = PyramidScorer(wl.bank, C, G, wl.pyramid, radius=None, domain="reference", max_dets=4096)
    sc.load_image(0, [synth.hog_level(1, 0, 0, 64, 48)])
    sc.run(tau=-1e30)
    return f"{len(sc.detections())} detections"


def _cfg4(envelope, mixture=False, images=2):
    from paper_1707_03268_b200 import synth
    from paper_1707_03268_b200.pipeline import PyramidScorer

    wl = synth.workload(4)
    C, G = _factors(4, 8)
    sc = PyramidScorer(wl.bank, C, G, wl.pyramid, n_images=images, max_dets=1 << 16,
                       envelope=envelope)
    for i in range(images):
        sc.load_image(i, synth.hog_pyramid(4, i, wl.pyramid))
    sc.run(tau=0.5)
    out = f"{len(sc.detections())} detections"
    if mixture:
        out += f", {len(sc.mixture())} mixture maps"
    return out


def cfg4():
    return _cfg4(False)


def envelope():
    return _cfg4(True)


def mixture():
    return _cfg4(False, mixture=True, images=1)


def ffma():
    from paper_1707_03268_b200 import synth
    from paper_1707_03268_b200.pipeline import PyramidScorer

    wl = synth.workload(5)
    C, G = _factors(5, 32)
    sc = PyramidScorer(wl.bank, C, G, wl.pyramid, max_dets=1 << 16)
    sc.load_image(0, synth.hog_pyramid(5, 0, wl.pyramid))
    sc.run(tau=0.5)
    return f"{len(sc.detections())} detections"


def prune():
    import paper_1707_03268_b200 as B
    from conftest import golden_pruned, load_golden

    g = load_golden("detect_pruned.npz")
    n = 0
    for k in range(int(g["n"])):
        dec, pyr, _, tau = golden_pruned(g, k)
        for mode in ("kill", "lenient"):
            dets, _ = B.detect(dec, pyr, tau, pruning=True, part_prune_mode=mode)
            n += len(dets)
    return f"{n} detections"


def main():
    import torch

    what = sys.argv[1:] or ["cfg1", "cfg4", "envelope", "prune", "mixture", "ffma"]
    for w in what:
        msg = globals()[w]()
        torch.cuda.synchronize()
        print(f"sanitize_run {w}: ok ({msg})", flush=True)


if __name__ == "__main__":
    main()
