"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package ``cpdetect`` from
``/root/reference/pkg/src`` (read-only; nothing is copied) and writes small
``.npz`` fixtures next to this script.  The fixtures pin the CPU oracle
(``oracle/dpm_oracle.py``) and feed the GPU parity tests; the reference
itself never travels to the GPU box.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from cpdetect import correlation as C  # noqa: E402
from cpdetect import detection as D  # noqa: E402
from cpdetect.decomposition import AlsOptions, CPModel, cp_als, reconstruct  # noqa: E402
from cpdetect.model import PartModel, PartSpec, decompose_model  # noqa: E402
from cpdetect.synthetic import gen_model, gen_scene  # noqa: E402

from paper_1707_03268_b200 import synth  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, sum(a.nbytes for a in map(np.asarray, arrays.values())), "bytes")


def cp_arrays(prefix, cp):
    return {
        f"{prefix}_w": cp.weights,
        f"{prefix}_a": cp.factors_a,
        f"{prefix}_b": cp.factors_b,
        f"{prefix}_c": cp.factors_c,
    }


def random_cp(rng, dims, rank):
    n, m, l = dims
    return CPModel.from_factors(rng.normal(size=(n, rank)), rng.normal(size=(m, rank)),
                                rng.normal(size=(l, rank)))


def gen_correlation():
    out = {}
    cases = [((6, 7, 4), (2, 3, 4)), ((9, 8, 4), (3, 4, 4)), ((12, 11, 6), (4, 4, 6)),
             ((20, 17, 32), (6, 11, 32)), ((5, 6, 3), (5, 6, 3)), ((7, 9, 1), (1, 1, 1))]
    for k, (ishape, fshape) in enumerate(cases):
        rng = np.random.default_rng([11, k])
        img = rng.normal(size=ishape)
        filt = rng.normal(size=fshape)
        out[f"full{k}_img"] = img
        out[f"full{k}_filt"] = filt
        out[f"full{k}_out"] = C.correlate3_full(img, filt).scores
        out[f"full{k}_mult"] = np.int64(C.correlate3_full(img, filt).multiplications)
    cp_cases = [((7, 5, 3), (3, 2, 3), 4), ((9, 8, 4), (3, 4, 4), 3), ((16, 20, 32), (6, 6, 32), 8),
                ((16, 20, 32), (6, 11, 32), 8), ((6, 6, 2), (2, 2, 2), 2), ((10, 12, 6), (4, 4, 6), 5)]
    for k, (ishape, dims, rank) in enumerate(cp_cases):
        rng = np.random.default_rng([12, k])
        img = rng.normal(size=ishape)
        cp = random_cp(rng, dims, rank)
        out[f"cp{k}_img"] = img
        out.update(cp_arrays(f"cp{k}", cp))
        out[f"cp{k}_stack"] = C.cp_partial_stack(img, cp)
        up = max(1, rank // 2)
        sm = C.correlate3_cp(img, cp, upto_rank=up)
        out[f"cp{k}_upto"] = np.int64(up)
        out[f"cp{k}_upto_out"] = sm.scores
        out[f"cp{k}_upto_mult"] = np.int64(sm.multiplications)
    out["n_full"] = np.int64(len(cases))
    out["n_cp"] = np.int64(len(cp_cases))
    save("correlation.npz", **out)


def gen_placement():
    out = {}
    cases = []
    # (map shape, quantise?, deformation, radius, anchor, rect-or-None)
    cases.append(((15, 15), None, (0.1, 0.1, 0.05, 0.05), 4, (1, -1), None))
    cases.append(((9, 9), None, (0.0, 0.0, 0.0, 0.0), 2, (0, 0), None))
    cases.append(((9, 9), None, (0.0, 0.0, 1e9, 1e9), 3, (0, 0), None))
    cases.append(((5, 5), "zeros", (0.0, 0.0, 0.0, 0.0), 1, (0, 0), None))
    cases.append(((31, 40), 0.1, (0.003, -0.002, 0.02, 0.01), 3, (2, -3), None))
    cases.append(((40, 52), None, (0.0, 0.0, 0.01, 0.01), 10, (0, 0), "virtual"))
    cases.append(((23, 19), 0.25, (-0.05, 0.04, 0.1, 0.2), 2, (-5, 4), None))
    cases.append(((60, 70), None, (0.0, 0.0, 0.01, 0.01), 13, (0, 0), "virtual"))
    for k, (shape, q, de, r, anc, rect) in enumerate(cases):
        rng = np.random.default_rng([13, k])
        if q == "zeros":
            smap = np.zeros(shape)
        else:
            smap = rng.normal(size=shape)
            if q is not None:
                smap = np.round(smap / q) * q
        hp, wp = shape
        if rect == "virtual":
            rect = (-r, hp - 1 + r, -r, wp - 1 + r)
        elif rect is None:
            # every root whose window meets the support (as _hypothesis_rect does)
            rect = (max(0, -anc[0] - r), hp - 1 - anc[0] + r - 2,
                    max(0, -anc[1] - r) + 1, wp - 1 - anc[1] + r)
        part = PartSpec(np.zeros((1, 1, 1)), anc, de, r)
        placed, py, px = D._placement_grid(smap, part, rect)
        out[f"p{k}_map"] = smap
        out[f"p{k}_def"] = np.array(de)
        out[f"p{k}_r"] = np.int64(r)
        out[f"p{k}_anchor"] = np.array(anc, dtype=np.int64)
        out[f"p{k}_rect"] = np.array(rect, dtype=np.int64)
        out[f"p{k}_placed"] = placed
        out[f"p{k}_py"] = py
        out[f"p{k}_px"] = px
        # scalar routine at a few roots inside the rect (window non-empty)
        roots = [(rect[0], rect[2]), (rect[1], rect[3]),
                 ((rect[0] + rect[1]) // 2, (rect[2] + rect[3]) // 2)]
        sc = []
        for root in roots:
            try:
                (y, x), v = D.best_part_placement(part, smap, root)
                sc.append((root[0], root[1], y, x, v, 1.0))
            except Exception:
                sc.append((root[0], root[1], -1, -1, 0.0, 0.0))
        out[f"p{k}_scalar"] = np.array(sc)
    out["n"] = np.int64(len(cases))
    save("placement.npz", **out)


def gen_detect_compact():
    """detect(pruning=False) and dense_detect on the reference test fixtures
    (pkg/tests/conftest.py:8-27)."""
    out = {}
    fast = AlsOptions(max_iterations=100, restarts=1, seed=0)
    for k, (mseed, sseed, low_rank, ranks) in enumerate([(28, 29, 2, 2), (52, 53, None, 2),
                                                          (3, 4, 2, 2), (30, 31, None, 3)]):
        model = gen_model(root_size=(3, 4), part_size=(4, 4), n_parts=2, channels=6,
                          low_rank=low_rank, search_radius=2, bias=0.1, seed=mseed)
        scene = gen_scene(model, n_objects=2, noise=0.05, level_shapes=((30, 34), (26, 28)),
                          seed=sseed)
        dec = decompose_model(model, ranks=ranks, opts=fast)
        dets, stats = D.detect(dec, scene.pyramid, -np.inf, pruning=False)
        ddets, dstats = D.dense_detect(model, scene.pyramid, -np.inf)
        pre = f"d{k}"
        for li, lv in enumerate(scene.pyramid):
            out[f"{pre}_level{li}"] = lv
        out[f"{pre}_nlevels"] = np.int64(len(scene.pyramid))
        out[f"{pre}_root"] = model.root
        for pi, p in enumerate(model.parts):
            out[f"{pre}_part{pi}"] = p.filter
            out[f"{pre}_part{pi}_anchor"] = np.array(p.anchor)
            out[f"{pre}_part{pi}_def"] = np.array(p.deformation)
            out[f"{pre}_part{pi}_r"] = np.int64(p.search_radius)
            out.update(cp_arrays(f"{pre}_pcp{pi}", dec.parts[pi].cp))
        out[f"{pre}_nparts"] = np.int64(len(model.parts))
        out[f"{pre}_bias"] = np.float64(model.bias)
        out.update(cp_arrays(f"{pre}_rcp", dec.root_cp))

        def pack(ds):
            return np.array([[d.hypothesis.level, *d.hypothesis.root,
                              *[c for pp in d.hypothesis.parts for c in pp], d.score]
                             for d in ds])
        out[f"{pre}_dets"] = pack(dets)
        out[f"{pre}_ddets"] = pack(ddets)
        out[f"{pre}_stats"] = np.array([stats.positions_examined, stats.multiplications])
        out[f"{pre}_dstats"] = np.array([dstats.positions_examined, dstats.multiplications])
        # scalar scorers on the first detection
        d0 = dets[len(dets) // 2]
        hyp = d0.hypothesis
        lv = scene.pyramid[hyp.level]
        out[f"{pre}_hyp"] = np.array([hyp.level, *hyp.root, *[c for pp in hyp.parts for c in pp]])
        out[f"{pre}_score_hyp"] = np.float64(D.score_hypothesis(model, lv, hyp))
        out[f"{pre}_cp_score_hyp"] = np.float64(D.cp_score_hypothesis(dec, lv, hyp))
    out["n"] = np.int64(4)
    save("detect_compact.npz", **out)


def gen_cfg1():
    """Config 1: one 64x48x32 level, root 6x11 + 8 parts 6x6 (s = 1), R = 8.

    Reference-native per-filter CP (decompose_model) + the reference detector
    at tau = -inf, and the shared-basis variant composed from reference
    functions (cp_als on the stacked tensor, correlate3_full on the
    reconstructed filters, _placement_grid on the reference rectangle)."""
    wl = synth.workload(1)
    bank, comp = wl.bank, wl.bank.components[0]
    level = synth.hog_level(1, 0, 0, 64, 48).astype(np.float64)
    filt = [f.astype(np.float64) for f in bank.filters]
    model = PartModel(root=filt[comp.root],
                      parts=tuple(PartSpec(filt[f], a, d, comp.search_radius)
                                  for f, a, d in zip(comp.parts, comp.anchors, comp.deformations)),
                      bias=comp.bias)
    dec = decompose_model(model, ranks=8)
    dets, stats = D.detect(dec, [level], -np.inf, pruning=False)
    out = {"level_sum": np.float64(level.sum())}
    out.update(cp_arrays("root", dec.root_cp))
    for i, p in enumerate(dec.parts):
        out.update(cp_arrays(f"part{i}", p.cp))
    out["dets"] = np.array([[d.hypothesis.root[0], d.hypothesis.root[1],
                             *[c for pp in d.hypothesis.parts for c in pp], d.score] for d in dets])
    out["stats"] = np.array([stats.positions_examined, stats.multiplications])
    out["root_map"] = C.cp_partial_stack(level, dec.root_cp)[-1]
    out["part0_map"] = C.cp_partial_stack(level, dec.parts[0].cp)[-1]
    # shared basis at R = 8 over the 9 stacked filters
    T = bank.stacked()
    cp, res = cp_als(T, 8)
    Cb = cp.factors_c.astype(np.float32)
    G = (cp.factors_a * (cp.weights * cp.factors_b[0])[None, :]).astype(np.float32)
    out["shared_C"] = Cb
    out["shared_G"] = G
    out["shared_residual"] = np.float64(res)
    offs = bank.offsets()
    recon = []
    for f, o in zip(bank.filters, offs):
        h, w = f.shape[:2]
        core = G[o:o + h * w].astype(np.float64).reshape(h, w, 8)
        recon.append(np.einsum("ijr,lr->ijl", core, Cb.astype(np.float64)))
    rmodel = PartModel(root=recon[comp.root],
                       parts=tuple(PartSpec(recon[f], a, d, comp.search_radius)
                                   for f, a, d in zip(comp.parts, comp.anchors, comp.deformations)),
                       bias=comp.bias)
    sdets, _ = D.dense_detect(rmodel, [level], -np.inf)
    out["shared_dets"] = np.array([[d.hypothesis.root[0], d.hypothesis.root[1],
                                    *[c for pp in d.hypothesis.parts for c in pp], d.score]
                                   for d in sdets])
    save("cfg1.npz", **out)


def gen_cfg2_sample():
    """Config 2 at R = 8 (shared basis, s = 2): reference-composed totals for
    two root levels x two components, placement by the reference
    _placement_grid at radius r* over the virtual full-map rect, gathered
    at 2*root + anchor."""
    from oracle import dpm_oracle as O

    wl = synth.workload(2)
    fx = np.load(os.path.join(REPO, "paper_1707_03268_b200", "data", "factors_cfg2_R8.npz"))
    Cb, G = fx["C"], fx["G"]
    bank, pyr = wl.bank, wl.pyramid
    offs = bank.offsets()
    cores = []
    for f, o in zip(bank.filters, offs):
        h, w = f.shape[:2]
        cores.append(G[o:o + h * w].reshape(h, w, -1))
    out = {}
    sel = [(0, 0), (0, 1), (17, 2), (28, 5)]
    for k, (i, ci) in enumerate(sel):
        kr, kp = pyr.root_levels[i], pyr.part_levels[i]
        comp = bank.components[ci]
        lr = synth.hog_level(2, 0, kr, *pyr.levels[kr]).astype(np.float64)
        lp = synth.hog_level(2, 0, kp, *pyr.levels[kp]).astype(np.float64)

        def recon(f):
            return np.einsum("ijr,lr->ijl", cores[f].astype(np.float64), Cb.astype(np.float64))
        root_map = C.correlate3_full(lr, recon(comp.root)).scores
        rh, rw = bank.filters[comp.root].shape[:2]
        psup = [(lp.shape[0] - 5, lp.shape[1] - 5)] * len(comp.parts)
        rect = O._gdt_rect((lr.shape[0] - rh + 1, lr.shape[1] - rw + 1), psup, comp.anchors, 2)
        ry0, ry1, rx0, rx1 = rect
        tot = root_map[ry0:ry1 + 1, rx0:rx1 + 1].copy()
        pos = []
        for f, anc, de in zip(comp.parts, comp.anchors, comp.deformations):
            pm = C.correlate3_full(lp, recon(f)).scores
            r = O.r_star(pm, de)
            hp, wp = pm.shape
            part = PartSpec(np.zeros((1, 1, 1)), (0, 0), de, r)
            placed, py, px = D._placement_grid(pm, part, (-r, hp - 1 + r, -r, wp - 1 + r))
            cy = 2 * np.arange(ry0, ry1 + 1)[:, None] + anc[0] + r
            cx = 2 * np.arange(rx0, rx1 + 1)[None, :] + anc[1] + r
            tot = tot + placed[cy, cx]
            pos.append(np.stack([py[cy, cx], px[cy, cx]], axis=-1))
        tot = tot + comp.bias
        out[f"s{k}_sel"] = np.array([i, ci])
        out[f"s{k}_rect"] = np.array(rect)
        out[f"s{k}_scores"] = tot
        out[f"s{k}_parts"] = np.stack(pos).astype(np.int32)
    out["n"] = np.int64(len(sel))
    save("cfg2_sample.npz", **out)


def gen_detect_pruned():
    """calibrate_thresholds + detect(pruning=True) in both part modes on the
    reference test fixtures (pkg/tests/test_detection.py:48-53 setup)."""
    out = {}
    fast = AlsOptions(max_iterations=100, restarts=1, seed=0)
    cases = [(0, 1, 2, 2, 0.0), (7, 8, 2, 3, -np.inf), (11, 12, None, 2, 0.5)]
    for k, (mseed, sseed, low_rank, ranks, tau) in enumerate(cases):
        model = gen_model(root_size=(3, 4), part_size=(4, 4), n_parts=2, channels=6,
                          low_rank=low_rank, search_radius=2, bias=0.1, seed=mseed)
        scene = gen_scene(model, n_objects=2, noise=0.05, level_shapes=((30, 34), (26, 28)),
                          seed=sseed)
        dec = decompose_model(model, ranks=ranks, opts=fast)
        positives = [(scene.pyramid[lvl], hyp) for lvl, hyp in scene.planted]
        cal = D.calibrate_thresholds(dec, positives)
        pre = f"q{k}"
        for li, lv in enumerate(scene.pyramid):
            out[f"{pre}_level{li}"] = lv
        out[f"{pre}_nlevels"] = np.int64(len(scene.pyramid))
        out[f"{pre}_planted"] = np.array([[lvl, *hyp.root, *[c for pp in hyp.parts for c in pp]]
                                          for lvl, hyp in scene.planted])
        for pi, prt in enumerate(cal.parts):
            out[f"{pre}_part{pi}_anchor"] = np.array(prt.anchor)
            out[f"{pre}_part{pi}_def"] = np.array(prt.deformation)
            out[f"{pre}_part{pi}_r"] = np.int64(prt.search_radius)
            out[f"{pre}_part{pi}_thr"] = np.asarray(prt.thresholds)
            out.update(cp_arrays(f"{pre}_pcp{pi}", prt.cp))
        out[f"{pre}_nparts"] = np.int64(len(cal.parts))
        out[f"{pre}_bias"] = np.float64(cal.bias)
        out[f"{pre}_root_thr"] = np.asarray(cal.root_thresholds)
        out.update(cp_arrays(f"{pre}_rcp", cal.root_cp))
        out[f"{pre}_tau"] = np.float64(tau)
        for mode in ("kill", "lenient"):
            dets, stats = D.detect(cal, scene.pyramid, tau, pruning=True, part_prune_mode=mode,
                                   collect_maps=True)
            m = f"{pre}_{mode}"
            out[f"{m}_dets"] = np.array([[d.hypothesis.level, *d.hypothesis.root,
                                          *[c for pp in d.hypothesis.parts for c in pp], d.score]
                                         for d in dets]).reshape(-1, 3 + 2 * len(cal.parts) + 1)
            R = max(cal.root_cp.rank, *[p.cp.rank for p in cal.parts])
            out[f"{m}_stats"] = np.array([stats.positions_examined, stats.positions_killed_by_parts,
                                          stats.multiplications])
            out[f"{m}_root_pruned"] = np.array([stats.positions_pruned_at_rank.get(r, 0)
                                                for r in range(1, R + 1)])
            out[f"{m}_part_pruned"] = np.array([stats.part_pruned_at_rank.get(r, 0)
                                                for r in range(1, R + 1)])
            for li, lm in enumerate(stats.prune_maps):
                if lm["rect"] is None:
                    continue
                out[f"{m}_rect{li}"] = np.array(lm["rect"])
                out[f"{m}_rootrank{li}"] = lm["root_prune_rank"]
                out[f"{m}_partrank{li}"] = lm["part_prune_rank"]
    out["n"] = np.int64(len(cases))
    save("detect_pruned.npz", **out)


def gen_roc():
    """roc_eval (evaluation.py:102-162) on three compact scenes: dense model,
    decomposed (full rank 2 of a rank-2 model) and calibrated pruning."""
    from cpdetect.evaluation import roc_eval

    out = {}
    fast = AlsOptions(max_iterations=100, restarts=1, seed=0)
    model = gen_model(root_size=(3, 4), part_size=(4, 4), n_parts=2, channels=6, low_rank=2,
                      search_radius=2, bias=0.1, seed=21)
    scenes = [gen_scene(model, n_objects=2, noise=0.05, level_shapes=((30, 34),), seed=31 + i)
              for i in range(3)]
    dec = decompose_model(model, ranks=2, opts=fast)
    positives = [(sc.pyramid[lvl], hyp) for sc in scenes for lvl, hyp in sc.planted]
    cal = D.calibrate_thresholds(dec, positives)
    taus = np.linspace(-2.0, 6.0, 9)
    out["taus"] = taus
    for si, sc in enumerate(scenes):
        out[f"s{si}_level0"] = sc.pyramid[0]
        out[f"s{si}_planted"] = np.array([[lvl, *hyp.root, *[c for pp in hyp.parts for c in pp]]
                                          for lvl, hyp in sc.planted])
    out["root"] = model.root
    for pi, p in enumerate(model.parts):
        out[f"part{pi}"] = p.filter
        out[f"part{pi}_anchor"] = np.array(p.anchor)
        out[f"part{pi}_def"] = np.array(p.deformation)
        out[f"part{pi}_r"] = np.int64(p.search_radius)
        out[f"part{pi}_thr"] = np.asarray(cal.parts[pi].thresholds)
        out.update(cp_arrays(f"pcp{pi}", dec.parts[pi].cp))
    out["bias"] = np.float64(model.bias)
    out["root_thr"] = np.asarray(cal.root_thresholds)
    out.update(cp_arrays("rcp", dec.root_cp))

    def pts(points):
        return np.array([[p.tau, p.misdetection_rate, p.false_positives_per_scene,
                          p.false_positives_per_window] for p in points])
    out["roc_dense"] = pts(roc_eval(model, scenes, taus))
    out["roc_cp"] = pts(roc_eval(dec, scenes, taus))
    out["roc_pruned"] = pts(roc_eval(cal, scenes, taus, pruning=True))
    save("roc.npz", **out)


def gen_formats():
    """Files written by the reference's own savers (save_model dense and
    decomposed+calibrated, save_scene) plus the arrays its loaders return,
    for the format readers."""
    from cpdetect.model import load_model, save_model
    from cpdetect.synthetic import load_scene, save_scene

    d = os.path.join(HERE, "formats")
    os.makedirs(d, exist_ok=True)
    fast = AlsOptions(max_iterations=100, restarts=1, seed=0)
    model = gen_model(root_size=(3, 4), part_size=(4, 4), n_parts=2, channels=6, low_rank=2,
                      search_radius=2, bias=0.25, seed=5)
    scene = gen_scene(model, n_objects=2, noise=0.05, level_shapes=((20, 24), (16, 18)), seed=6)
    dec = decompose_model(model, ranks=2, opts=fast)
    cal = D.calibrate_thresholds(dec, [(scene.pyramid[l], h) for l, h in scene.planted])
    save_model(os.path.join(d, "dense.json"), model)
    save_model(os.path.join(d, "dec.json"), cal)
    save_scene(os.path.join(d, "scene.json"), scene)
    m = load_model(os.path.join(d, "dense.json"))
    c = load_model(os.path.join(d, "dec.json"))
    sc = load_scene(os.path.join(d, "scene.json"))
    out = {"dense_root": m.root, "dense_bias": m.bias,
           "dec_root_thr": c.root_thresholds, "dec_bias": c.bias,
           "scene_truth": np.array([[l, *h.root, *[v for p in h.parts for v in p], h.score]
                                    for l, h in sc.planted])}
    for i, p in enumerate(m.parts):
        out[f"dense_part{i}"] = p.filter
    out.update(cp_arrays("dec_root", c.root_cp))
    for i, p in enumerate(c.parts):
        out.update(cp_arrays(f"dec_part{i}", p.cp))
        out[f"dec_part{i}_thr"] = p.thresholds
    for i, lv in enumerate(sc.pyramid):
        out[f"scene_level{i}"] = lv
    save("formats/expected.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["correlation", "placement", "detect_compact", "cfg1", "cfg2_sample",
                             "detect_pruned", "roc", "formats"]
    for w in which:
        globals()["gen_" + w]()
