"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and
the reference's golden vectors.  Run on a B200 with ``pytest -m gpu``."""

import numpy as np
import pytest

from conftest import golden_cp, load_golden
from oracle import dpm_oracle as O
from parity import assert_map_close, classify_positions, penalised

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_1707_03268_b200")
from paper_1707_03268_b200 import synth  # noqa: E402
from paper_1707_03268_b200.pipeline import PyramidScorer  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


# ------------------------------------------------------------------ K1 + K2

def test_correlate3_full_matches_reference_golden():
    g = load_golden("correlation.npz")
    for k in range(int(g["n_full"])):
        img, filt = g[f"full{k}_img"], g[f"full{k}_filt"]
        sm = B.correlate3_full(img, filt)
        assert_map_close(sm.scores, g[f"full{k}_out"], f"full{k}")
        assert sm.multiplications == int(g[f"full{k}_mult"])
        # same fp32-rounded inputs through the oracle: tighter still
        assert_map_close(sm.scores, O.correlate3_full(f32(img), f32(filt)), f"full{k} f32", 2e-6)


def test_cp_engines_match_reference_golden_and_prefix_identity():
    g = load_golden("correlation.npz")
    for k in range(int(g["n_cp"])):
        cp, img = golden_cp(g, f"cp{k}"), g[f"cp{k}_img"]
        stack = B.cp_partial_stack(img, cp)
        ref = g[f"cp{k}_stack"]
        assert stack.shape == ref.shape
        for r in range(ref.shape[0]):
            assert_map_close(stack[r], ref[r], f"cp{k} rank {r}")
        up = int(g[f"cp{k}_upto"])
        sm = B.correlate3_cp(img, cp, upto_rank=up)
        assert_map_close(sm.scores, g[f"cp{k}_upto_out"], f"cp{k} upto")
        assert sm.multiplications == int(g[f"cp{k}_upto_mult"])
        # reference property (test_correlation.py:158-178): prefixes are bit-identical
        for r in range(1, cp.rank + 1):
            assert np.array_equal(B.correlate3_cp(img, cp, upto_rank=r).scores, stack[r - 1])


def test_cp_engine_edge_shapes_generic_and_chunked_kernels():
    rng = np.random.default_rng(77)
    # (img shape, dims, rank): filter == image (1x1 output), h not specialised,
    # R > 8 (rank chunking), odd channel counts
    for ishape, dims, rank in [((6, 11, 32), (6, 11, 32), 8), ((9, 30, 5), (1, 13, 5), 3),
                               ((17, 19, 32), (9, 4, 32), 12), ((40, 70, 32), (15, 15, 32), 32),
                               ((33, 65, 7), (6, 6, 7), 20), ((12, 12, 3), (12, 1, 3), 2)]:
        img = rng.normal(size=ishape).astype(np.float32).astype(np.float64)
        cp = B.CPModel.from_factors(rng.normal(size=(dims[0], rank)),
                                    rng.normal(size=(dims[1], rank)),
                                    rng.normal(size=(dims[2], rank)))
        ref = O.cp_partial_stack(img, cp)[-1]
        assert_map_close(B.correlate3_cp(img, cp).scores, ref, f"{ishape}/{dims}/{rank}")


def test_project_mma_kernel_ragged_levels_offsets_and_prefix_identity():
    """K1 through the C ABI (dpm_project) on 32-channel levels at R <= 8 -- the
    mma.sync kernel: levels whose cell count is not a multiple of 32 or 256,
    widths below 8 (row wraps inside a lane's +8 stride), a feature block off
    16-byte alignment (scalar-load path), R < 8, against the float64 oracle
    (correlation.py:128); planes of a prefix of C are bit-identical."""
    import torch

    from paper_1707_03268_b200 import _lib
    from paper_1707_03268_b200.device import upload_table

    lib = _lib.lib()
    rng = np.random.default_rng(11)
    shapes = [(1, 1), (3, 5), (2, 16), (7, 33), (40, 37), (17, 256), (90, 160), (300, 3)]
    for R in (8, 4, 1, 7):
        for shift in (0, 1):  # float offset of the first level: 0, or off 16-byte alignment
            C = rng.normal(size=(32, R)).astype(np.float32)
            levels = [rng.random((h, w, 32), dtype=np.float32) * 0.4 for h, w in shapes]
            x_off, p_off, jobs = shift, 0, []
            for (h, w) in shapes:
                pitch = (w + 3) // 4 * 4
                jobs.append((x_off, p_off, h, w, pitch, 0))
                x_off += h * w * 32 + (4 if shift == 0 else 0)
                p_off += R * h * pitch
            pj = np.array(jobs, dtype=_lib.PROJ_JOB)
            nblk = _lib.check(lib.dpm_project_prepare(_lib.table_ptr(pj), len(pj)), "project")
            X = torch.zeros(x_off + 8, dtype=torch.float32, device="cuda")
            for j, lv in zip(jobs, levels):
                X[j[0]:j[0] + lv.size] = torch.from_numpy(lv.ravel()).cuda()
            P = torch.full((p_off,), float("nan"), dtype=torch.float32, device="cuda")
            Cd = torch.from_numpy(C).cuda()
            tab = upload_table(pj, "cuda")
            st = torch.cuda.current_stream().cuda_stream
            _lib.check(lib.dpm_project(X.data_ptr(), P.data_ptr(), Cd.data_ptr(), 32, R,
                                       tab.data_ptr(), len(pj), nblk, st), "project")
            out = P.cpu().numpy()
            for j, lv in zip(jobs, levels):
                _, po, h, w, pitch, _ = j
                got = out[po:po + R * h * pitch].reshape(R, h, pitch)[:, :, :w]
                ref = O.project(lv.astype(np.float64), C.astype(np.float64)).transpose(2, 0, 1)
                assert_map_close(got, ref, f"K1 {h}x{w} R={R} shift={shift}", rtol=2e-6)
            if R == 8 and shift == 0:  # prefix of the basis: the same planes, bit for bit
                for k in (1, 5):
                    Ck = torch.from_numpy(np.ascontiguousarray(C[:, :k])).cuda()
                    jk, po = [], 0
                    for (xo, _, h, w, pitch, _) in jobs:
                        jk.append((xo, po, h, w, pitch, 0))
                        po += k * h * pitch
                    pk = np.array(jk, dtype=_lib.PROJ_JOB)
                    nb = _lib.check(lib.dpm_project_prepare(_lib.table_ptr(pk), len(pk)), "project")
                    Pk = torch.zeros(po, dtype=torch.float32, device="cuda")
                    tk = upload_table(pk, "cuda")
                    _lib.check(lib.dpm_project(X.data_ptr(), Pk.data_ptr(), Ck.data_ptr(), 32, k,
                                               tk.data_ptr(), len(pk), nb, st), "project")
                    outk = Pk.cpu().numpy()
                    for j8, jk_ in zip(jobs, jk):
                        h, w, pitch = j8[2], j8[3], j8[4]
                        a = out[j8[1]:j8[1] + k * h * pitch].reshape(k, h, pitch)[:, :, :w]
                        b = outk[jk_[1]:jk_[1] + k * h * pitch].reshape(k, h, pitch)[:, :, :w]
                        assert np.array_equal(a, b), f"prefix {k} planes differ on {h}x{w}"


def test_dense_many_filters_group_split():
    """More than 48 same-shape filters on one level: K2 splits the group."""
    rng = np.random.default_rng(5)
    level = rng.random((40, 52, 32)).astype(np.float32)
    cores = [rng.normal(0, 0.05, (6, 6, 8)).astype(np.float32) for _ in range(60)]
    C = rng.normal(size=(32, 8)).astype(np.float32)
    from paper_1707_03268_b200.engine import FilterDef, Plan

    plan = Plan(32, [(40, 52)], C, [FilterDef(c) for c in cores], apps=[(0, f) for f in range(60)],
                outputs=())
    plan.load_levels(0, [level])
    plan.run(stages=("project", "correlate"))
    P = O.project(level, C.astype(np.float64))
    for f in (0, 47, 48, 59):
        assert_map_close(plan.map(0, 0, f).double().cpu().numpy(), O.correlate3_full(P, cores[f]),
                         f"filter {f}")


# ----------------------------------------------------------------- K3 + K4

def test_placement_grid_bit_exact_on_fp32_maps_and_golden():
    g = load_golden("placement.npz")
    for k in range(int(g["n"])):
        smap = g[f"p{k}_map"]
        anc, de, r = tuple(g[f"p{k}_anchor"]), tuple(g[f"p{k}_def"]), int(g[f"p{k}_r"])
        rect = tuple(int(v) for v in g[f"p{k}_rect"])
        part = B.PartSpec(np.zeros((1, 1, 1)), anc, de, r)
        placed, py, px = B._placement_grid(smap, part, rect)
        # kernel-isolated: identical to the oracle on the same fp32 map
        o_placed, o_py, o_px = O.placement_grid(f32(smap), anc, de, r, rect)
        assert np.array_equal(placed, o_placed), k
        assert np.array_equal(py, o_py) and np.array_equal(px, o_px), k
        # vs the reference on its float64 map: values to tolerance, argmax to ties
        ref = g[f"p{k}_placed"]
        fin = np.isfinite(ref)
        assert np.array_equal(fin, np.isfinite(placed))
        assert_map_close(placed[fin], ref[fin], f"placement {k}")
        S = smap
        cy = np.arange(rect[0], rect[1] + 1)[:, None] + anc[0] + 0 * px
        cx = np.arange(rect[2], rect[3] + 1)[None, :] + anc[1] + 0 * py
        gp = np.stack([py, px], -1).reshape(-1, 2)
        rp = np.stack([g[f"p{k}_py"], g[f"p{k}_px"]], -1).reshape(-1, 2)
        cent = np.stack([cy, cx], -1).reshape(-1, 2)
        _, _, err = classify_positions(gp, rp, lambda i, p: penalised(S, cent[i], p, de),
                                       ref.reshape(-1), np.abs(S).max())
        assert err == 0, k


def test_placement_band_edges_bit_exact():
    """TMA band staging at the map edges: maps narrower and wider than the
    100-column box, windows reaching past every edge (negative and odd band
    origins: every 16-byte shift parity of the box start), radii up to the
    staged cap (16) and one beyond it (unstaged path).  Cells outside the map
    arrive as NaN; results (values, -inf for empty windows, positions) must
    equal the oracle's exactly."""
    rng = np.random.default_rng(1707)
    shapes = [(4, 3), (40, 17), (9, 37), (33, 99), (21, 101), (70, 133)]
    for case in range(60):
        H, W = shapes[case % len(shapes)]
        smap = rng.uniform(-1, 1, (H, W)).astype(np.float32)
        r = int(rng.choice([0, 1, 2, 7, 15, 16, 17]))
        # |anchor| <= r: windows reach up to 2r past the edges (the reference's
        # padding, detection.py:320-373)
        anc = (int(rng.integers(-r, r + 1)), int(rng.integers(-r, r + 1)))
        de = (float(rng.uniform(-0.05, 0.05)), float(rng.uniform(-0.05, 0.05)),
              float(rng.uniform(0.005, 0.05)), float(rng.uniform(0.005, 0.05)))
        rect = (0, H - 1, 0, W - 1)
        part = B.PartSpec(np.zeros((1, 1, 1)), anc, de, r)
        placed, py, px = B._placement_grid(smap, part, rect)
        o_placed, o_py, o_px = O.placement_grid(f32(smap), anc, de, r, rect)
        assert np.array_equal(placed, o_placed), (case, H, W, r, anc)
        assert np.array_equal(py, o_py) and np.array_equal(px, o_px), (case, H, W, r, anc)


def test_best_part_placement_known_answers():
    part = B.PartSpec(np.zeros((2, 2, 3)), (0, 0), (0.0, 0.0, 0.0, 0.0), 1)
    assert B.best_part_placement(part, np.zeros((5, 5)), (2, 2)) == ((1, 1), 0.0)
    rng = np.random.default_rng(7)
    s = rng.normal(size=(9, 9)).astype(np.float32).astype(np.float64)
    big = B.PartSpec(np.zeros((2, 2, 3)), (0, 0), (0.0, 0.0, 1e9, 1e9), 3)
    assert B.best_part_placement(big, s, (4, 4))[0] == (4, 4)
    zero = B.PartSpec(np.zeros((2, 2, 3)), (0, 0), (0.0, 0.0, 0.0, 0.0), 2)
    pos, val = B.best_part_placement(zero, s, (4, 4))
    assert val == s[2:7, 2:7].max() and s[pos] == val
    far = B.PartSpec(np.zeros((2, 2, 3)), (10, 10), (0.0, 0.0, 0.0, 0.0), 1)
    with pytest.raises(B.ValidationError, match="empty"):
        B.best_part_placement(far, np.zeros((5, 5)), (0, 0))


@pytest.mark.parametrize("anchor", [(1000, 0), (-1000, 0), (0, 1000), (0, -1000), (1000, -1000),
                                    (170, 3), (200, 3), (-170, 3), (3, 170)])
def test_placement_windows_far_outside_the_map(anchor):
    """Anchors whose windows never meet the map: the staged band
    lies wholly above / below / beside the map.  Every window is empty: the
    reference's best_part_placement raises, and the grid reports -inf at
    every root without touching memory outside its band (a following
    in-map placement in the same process stays exact)."""
    rng = np.random.default_rng(7)
    S = rng.standard_normal((40, 37)).astype(np.float32).astype(np.float64)
    de = (0.01, -0.02, 0.05, 0.04)
    far = B.PartSpec(np.zeros((2, 2, 3)), anchor, de, 4)
    with pytest.raises(B.ValidationError, match="empty"):
        B.best_part_placement(far, S, (5, 5))
    placed, py, px = B._placement_grid(S, far, (0, 30, 0, 20))
    assert placed.shape == (31, 21) and np.all(np.isneginf(placed))
    near = B.PartSpec(np.zeros((2, 2, 3)), (1, 2), de, 4)
    v, qy, qx = B._placement_grid(S, near, (0, 30, 0, 20))
    ov, oy, ox = O.placement_grid(S, (1, 2), de, 4, (0, 30, 0, 20))
    assert np.array_equal(v, ov) and np.array_equal(qy, oy) and np.array_equal(qx, ox)


def _compact(g, k):
    pre = f"d{k}"
    levels = [g[f"{pre}_level{i}"] for i in range(int(g[f"{pre}_nlevels"]))]
    parts, dparts = [], []
    for i in range(int(g[f"{pre}_nparts"])):
        anc = tuple(int(v) for v in g[f"{pre}_part{i}_anchor"])
        de = tuple(float(v) for v in g[f"{pre}_part{i}_def"])
        r = int(g[f"{pre}_part{i}_r"])
        parts.append(B.PartSpec(g[f"{pre}_part{i}"], anc, de, r))
        dparts.append(B.DecomposedPart(golden_cp(g, f"{pre}_pcp{i}"), anc, de, r))
    model = B.PartModel(g[f"{pre}_root"], tuple(parts), float(g[f"{pre}_bias"]))
    dec = B.DecomposedModel(golden_cp(g, f"{pre}_rcp"), tuple(dparts), float(g[f"{pre}_bias"]))
    return levels, model, dec


def _pack(dets):
    return np.array([[d.hypothesis.level, *d.hypothesis.root,
                      *[c for pp in d.hypothesis.parts for c in pp], d.score] for d in dets])


def _check_dets(got, ref, levels, part_defs, part_maps_fn, what):
    """Roots identical, scores to 1e-5 of max |score|, part argmaxes up to ties."""
    assert got.shape == ref.shape, what
    assert np.array_equal(got[:, :3], ref[:, :3]), what
    assert_map_close(got[:, -1], ref[:, -1], what)
    npart = (got.shape[1] - 4) // 2
    for p in range(npart):
        gp, rp = got[:, 3 + 2 * p:5 + 2 * p], ref[:, 3 + 2 * p:5 + 2 * p]
        bad = np.nonzero(np.any(gp != rp, axis=1))[0]
        errs = 0
        for i in bad:
            lvl = int(ref[i, 0])
            S = part_maps_fn(lvl, p)
            anc, de = part_defs[p]
            cent = (int(ref[i, 1]) + anc[0], int(ref[i, 2]) + anc[1])
            vg = penalised(S, cent, tuple(int(v) for v in gp[i]), de)
            vr = penalised(S, cent, tuple(int(v) for v in rp[i]), de)
            if vr - vg > 1e-5 * np.abs(S).max():
                errs += 1
        assert errs == 0, f"{what}: part {p} has {errs} argmax errors"


def test_detect_and_dense_detect_match_reference_golden():
    g = load_golden("detect_compact.npz")
    for k in range(int(g["n"])):
        levels, model, dec = _compact(g, k)
        pdefs = [(p.anchor, p.deformation) for p in model.parts]
        dets, stats = B.detect(dec, levels, -np.inf)
        _check_dets(_pack(dets), g[f"d{k}_dets"], levels, pdefs,
                    lambda lvl, p: O.cp_partial_stack(levels[lvl], dec.parts[p].cp)[-1],
                    f"detect {k}")
        assert [stats.positions_examined, stats.multiplications] == list(g[f"d{k}_stats"])
        ddets, dstats = B.dense_detect(model, levels, -np.inf)
        _check_dets(_pack(ddets), g[f"d{k}_ddets"], levels, pdefs,
                    lambda lvl, p: O.correlate3_full(levels[lvl], model.parts[p].filter),
                    f"dense_detect {k}")
        assert [dstats.positions_examined, dstats.multiplications] == list(g[f"d{k}_dstats"])
        # threshold: only scores >= tau, same sorted order
        tau = float(np.median(g[f"d{k}_dets"][:, -1]))
        some, _ = B.detect(dec, levels, tau)
        assert all(d.score >= tau for d in some)
        assert len(some) >= 1
        h = g[f"d{k}_hyp"]
        hyp = B.Hypothesis(int(h[0]), (int(h[1]), int(h[2])),
                           tuple((int(h[3 + 2 * i]), int(h[4 + 2 * i]))
                                 for i in range(len(model.parts))))
        lv = levels[hyp.level]
        assert B.score_hypothesis(model, lv, hyp) == pytest.approx(float(g[f"d{k}_score_hyp"]),
                                                                   rel=1e-5, abs=1e-5)
        assert B.cp_score_hypothesis(dec, lv, hyp) == pytest.approx(
            float(g[f"d{k}_cp_score_hyp"]), rel=1e-5, abs=1e-5)


def test_config1_reference_native_detect():
    """Config 1: 64x48x32 level, root 6x11 + 8 parts 6x6, per-filter CP R=8."""
    g = load_golden("cfg1.npz")
    wl = synth.workload(1)
    comp = wl.bank.components[0]
    level = synth.hog_level(1, 0, 0, 64, 48).astype(np.float64)
    parts = tuple(B.DecomposedPart(golden_cp(g, f"part{i}"), a, d, 2)
                  for i, (a, d) in enumerate(zip(comp.anchors, comp.deformations)))
    dec = B.DecomposedModel(golden_cp(g, "root"), parts, comp.bias)
    dets, stats = B.detect(dec, [level], -np.inf)
    got = _pack(dets)
    ref = np.concatenate([np.zeros((len(g["dets"]), 1)), g["dets"]], axis=1)
    pdefs = [(p.anchor, p.deformation) for p in parts]
    _check_dets(got, ref, [level], pdefs,
                lambda lvl, p: O.cp_partial_stack(level, parts[p].cp)[-1], "config 1")
    assert [stats.positions_examined, stats.multiplications] == list(g["stats"])
    assert_map_close(B.correlate3_cp(level, dec.root_cp).scores, g["root_map"], "cfg1 root map")


def test_config1_shared_basis_pyramid_scorer_reference_domain():
    g = load_golden("cfg1.npz")
    wl = synth.workload(1)
    level = synth.hog_level(1, 0, 0, 64, 48)
    sc = PyramidScorer(wl.bank, g["shared_C"], g["shared_G"], wl.pyramid, radius=None,
                       domain="reference")
    sc.load_image(0, [level])
    sc.run()
    (res,) = sc.results(0)
    ry0, ry1, rx0, rx1 = res["rect"]
    ref = g["shared_dets"]
    ref_scores = ref[:, -1].reshape(ry1 - ry0 + 1, rx1 - rx0 + 1)
    assert_map_close(res["scores"], ref_scores, "cfg1 shared totals")
    ref_parts = ref[:, 2:-1].reshape(ry1 - ry0 + 1, rx1 - rx0 + 1, -1, 2).transpose(2, 0, 1, 3)
    ref_parts = ref_parts.astype(np.int64)
    # every argmax that differs from the reference's must be a tie of the
    # float64 oracle maps (exact or within the FP32 map tolerance)
    comp = wl.bank.components[0]
    P = O.project(level.astype(np.float64), g["shared_C"])
    cores = sc.cores
    for p, (f, anc, de) in enumerate(zip(comp.parts, comp.anchors, comp.deformations)):
        S = O.correlate3_full(P, cores[f].astype(np.float64))
        cy = np.arange(ry0, ry1 + 1)[:, None] + anc[0]
        cx = np.arange(rx0, rx1 + 1)[None, :] + anc[1]
        cent = np.stack(np.broadcast_arrays(cy, cx), -1).reshape(-1, 2)
        refp = ref_parts[p].reshape(-1, 2)
        best = np.array([penalised(S, cent[q], tuple(refp[q]), de) for q in range(len(cent))])
        _, _, err = classify_positions(res["parts"][p], ref_parts[p],
                                       lambda q, pos: penalised(S, cent[q], pos, de), best,
                                       np.abs(S).max())
        assert err == 0, (p, err)


# --------------------------------------------------- batched pyramids (configs)

def _shared(cfg, R):
    import os

    from conftest import REPO
    fx = np.load(os.path.join(REPO, "paper_1707_03268_b200", "data", f"factors_cfg{cfg}_R{R}.npz"))
    return fx["C"], fx["G"]


def _pyramid_parity(cfg, R, sel_levels=None, comps=None, images=(0,), n_images=1, feat_scale=1.0):
    wl = synth.workload(cfg)
    C, G = _shared(cfg, R)
    bank, pyr = wl.bank, wl.pyramid
    comp_list = list(bank.components) if comps is None else [bank.components[c] for c in comps]
    sc = PyramidScorer(bank, C, G, pyr, n_images=n_images, components=comp_list)
    levels = {}
    for img in range(n_images):
        lv = [np.float32(feat_scale) * x for x in synth.hog_pyramid(cfg, img, pyr)]
        levels[img] = lv
        sc.load_image(img, lv)
    sc.run()
    cores = sc.cores
    worst = 0.0
    for img in images:
        res = sc.results(img)
        if sel_levels is not None:
            res = [r for r in res if r["root_level"] in sel_levels]
        for rec in res:
            i, ci = rec["root_level"], rec["component"]
            kr, kp = pyr.root_levels[i], pyr.part_levels[i]
            comp = comp_list[ci]
            lvls = [np.zeros((1, 1, 32), np.float32)] * len(pyr.levels)
            lvls = list(lvls)
            lvls[kr], lvls[kp] = levels[img][kr], levels[img][kp]
            oref, maps = O.score_pyramid(lvls, bank, C, cores, root_levels=[kr],
                                         part_levels=[kp], components=[comp])
            (o,) = oref
            assert tuple(o["rect"]) == tuple(rec["rect"])
            worst = max(worst, assert_map_close(rec["scores"], o["scores"], f"cfg{cfg} {i}/{ci}"))
            # response maps (all filters of this component) to 1e-5
            gpu_maps = {}
            for f in (comp.root,) + tuple(comp.parts):
                k = kr if f == comp.root else kp
                gm = sc.plan.map(img, k, f).double().cpu().numpy()
                assert_map_close(gm, maps[(k, f)], f"cfg{cfg} map {k}/{f}")
                gpu_maps[f] = gm
            # argmaxes: kernel-isolated exactness on the GPU's own maps (the
            # lower-envelope GDT may break exact ties differently: <= 4 ulps)
            ry0, ry1, rx0, rx1 = rec["rect"]
            for p, (f, anc, de) in enumerate(zip(comp.parts, comp.anchors, comp.deformations)):
                gm = gpu_maps[f]
                r = O.r_star(gm, de)
                v, py, px = O.place_gathered(gm, anc, de, r, pyr.scale, rec["rect"])
                cy = pyr.scale * np.arange(ry0, ry1 + 1)[:, None] + anc[0]
                cx = pyr.scale * np.arange(rx0, rx1 + 1)[None, :] + anc[1]
                cent = np.stack(np.broadcast_arrays(cy, cx), -1).reshape(-1, 2)
                exact, near, err = classify_positions(
                    rec["parts"][p], np.stack([py, px], -1),
                    lambda q, pos: penalised(gm, cent[q], pos, de), v.reshape(-1), 0.0)
                assert near == 0 and err == 0, (exact, near, err)
                assert exact <= max(2, 1e-4 * py.size)
            # ... and against the fp64 oracle up to ties
            for p, (f, anc, de) in enumerate(zip(comp.parts, comp.anchors, comp.deformations)):
                S = maps[(kp, f)]
                cy = pyr.scale * np.arange(ry0, ry1 + 1)[:, None] + anc[0]
                cx = pyr.scale * np.arange(rx0, rx1 + 1)[None, :] + anc[1]
                cent = np.stack(np.broadcast_arrays(cy, cx), -1).reshape(-1, 2)
                best = np.array([penalised(S, cent[q], tuple(o["parts"][p].reshape(-1, 2)[q]), de)
                                 for q in range(cent.shape[0])])
                _, _, err = classify_positions(rec["parts"][p], o["parts"][p],
                                               lambda q, pos: penalised(S, cent[q], pos, de),
                                               best, np.abs(S).max())
                assert err == 0
    return worst


def test_config2_sample_matches_reference_golden():
    g = load_golden("cfg2_sample.npz")
    wl = synth.workload(2)
    C, G = _shared(2, 8)
    sc = PyramidScorer(wl.bank, C, G, wl.pyramid)
    lv = synth.hog_pyramid(2, 0, wl.pyramid)
    sc.load_image(0, lv)
    sc.run()
    res = {(r["root_level"], r["component"]): r for r in sc.results(0)}
    for k in range(int(g["n"])):
        i, ci = (int(v) for v in g[f"s{k}_sel"])
        rec = res[(i, ci)]
        assert tuple(rec["rect"]) == tuple(int(v) for v in g[f"s{k}_rect"])
        assert_map_close(rec["scores"], g[f"s{k}_scores"], f"cfg2 golden {k}")
        # mismatching argmaxes must be ties of the float64 oracle maps
        comp = wl.bank.components[ci]
        kr, kp = wl.pyramid.root_levels[i], wl.pyramid.part_levels[i]
        P = O.project(np.asarray(lv[kp], np.float64), C)
        ry0, ry1, rx0, rx1 = rec["rect"]
        for p, (f, anc, de) in enumerate(zip(comp.parts, comp.anchors, comp.deformations)):
            S = O.correlate3_full(P, sc.cores[f].astype(np.float64))
            cy = wl.pyramid.scale * np.arange(ry0, ry1 + 1)[:, None] + anc[0]
            cx = wl.pyramid.scale * np.arange(rx0, rx1 + 1)[None, :] + anc[1]
            cent = np.stack(np.broadcast_arrays(cy, cx), -1).reshape(-1, 2)
            refp = g[f"s{k}_parts"][p].reshape(-1, 2)
            best = np.array([penalised(S, cent[q], tuple(refp[q]), de) for q in range(len(cent))])
            _, _, err = classify_positions(rec["parts"][p], g[f"s{k}_parts"][p],
                                           lambda q, pos: penalised(S, cent[q], pos, de), best,
                                           np.abs(S).max())
            assert err == 0, (k, p, err)


@pytest.mark.parametrize("R", [4, 8, 16, 32])
def test_config2_full_pyramid_rank_sweep(R):
    _pyramid_parity(2, R, sel_levels=None if R == 8 else {0, 5, 14, 28})


def test_config3_sampled_models():
    _pyramid_parity(3, 16, sel_levels={0, 21, 41}, comps=[0, 1, 17, 59, 60, 119])


def test_config4_batch_consistency_and_sample():
    """Image 2 of a 3-image batch equals the oracle on sampled levels, and
    batching does not change any bit of any image's results."""
    _pyramid_parity(4, 8, sel_levels={0, 20, 38}, comps=[0, 3], images=(2,), n_images=3)
    wl = synth.workload(4)
    C, G = _shared(4, 8)
    one = PyramidScorer(wl.bank, C, G, wl.pyramid, n_images=1)
    one.load_image(0, synth.hog_pyramid(4, 2, wl.pyramid))
    one.run()
    three = PyramidScorer(wl.bank, C, G, wl.pyramid, n_images=3)
    for img in range(3):
        three.load_image(img, synth.hog_pyramid(4, img, wl.pyramid))
    three.run()
    for a, b in zip(one.results(0), three.results(2)):
        assert np.array_equal(a["scores"], b["scores"])
        assert np.array_equal(a["parts"], b["parts"])


@pytest.mark.parametrize("R", [8, 32])
def test_config5_large_roots_sample(R):
    _pyramid_parity(5, R, sel_levels={0, 19, 36})


def test_config4_full_image_every_level_and_component():
    """The benchmarked workload's unit: one whole config-4 image, all 39 root
    levels x 6 components (234 assemblies).  Totals and every response map
    to 1e-5 of the float64 oracle; part argmaxes bit-identical to the oracle
    run on the GPU's own maps (ties <= 1e-4), and against the float64 oracle
    only at ties (zero errors)."""
    worst = _pyramid_parity(4, 8, sel_levels=None, images=(0,), n_images=1)
    assert worst <= 1e-5


@pytest.mark.parametrize("feat_scale", [8.0, 0.05])
def test_config4_specialised_k3_radius_fallback(feat_scale):
    """The specialised K3 kernel takes every wide scale-2 tile of an unbounded
    (GDT) placement, but its staged path needs r* in (6, 16]: features scaled
    by 8 (map ranges x8, r* ~ 28) or by 0.05 (r* ~ 3) send its parts to the
    exact per-root fallback (fast_unstaged).  Values to 1e-5 of the float64
    oracle and argmaxes exact against the oracle on the GPU's own maps, on the
    two widest root levels."""
    worst = _pyramid_parity(4, 8, sel_levels=(0, 1), comps=(0, 1), feat_scale=feat_scale)
    assert worst <= 1e-5


def test_config5_every_level_R8():
    """Config 5 (1920x1080, roots up to 15x15) at R = 8 on all 37 root levels."""
    _pyramid_parity(5, 8, sel_levels=None)


def test_config3_every_level_twelve_components():
    """Config 3 (the 1080-filter bank on one shared rank-16 basis) on all 42
    root levels for 12 components spread over the 20 models and the 3
    mirrored pairs of each."""
    _pyramid_parity(3, 16, sel_levels=None,
                    comps=[0, 1, 7, 16, 29, 42, 59, 60, 83, 98, 111, 119])


def test_tau_compaction_matches_totals():
    wl = synth.workload(2)
    C, G = _shared(2, 8)
    sc = PyramidScorer(wl.bank, C, G, wl.pyramid, max_dets=200000)
    sc.load_image(0, synth.hog_pyramid(2, 0, wl.pyramid))
    allsc = np.concatenate([r["scores"].ravel() for r in sc.run().results(0)])
    tau = float(np.quantile(allsc, 0.99))
    sc.run(tau=tau)
    dets = sc.detections()
    assert len(dets) == int((allsc >= tau).sum())
    res = {(r["root_level"], r["component"]): r for r in sc.results(0)}
    for d in dets[:500]:
        rec = res[(int(d["level"]), int(d["component"]))]
        ry0, _, rx0, _ = rec["rect"]
        assert d["score"] == rec["scores"][d["ry"] - ry0, d["rx"] - rx0]


def test_tensor_core_correlation_matches_oracle_and_ffma():
    """tcgen05 3xTF32 K2 path: same maps as the oracle and the FFMA path."""
    from paper_1707_03268_b200.engine import FilterDef, Plan

    rng = np.random.default_rng(11)
    # the last two: the generic-shape kernel at R = 16 (multi-batch input-row
    # staging; enabled per plan with tc_ranks, off by default)
    for H, W, nf, h, w, R in [(40, 300, 48, 6, 6, 8), (23, 130, 16, 6, 6, 8),
                              (17, 200, 33, 5, 7, 8), (12, 70, 64, 3, 4, 8),
                              (30, 150, 6, 6, 11, 8), (9, 90, 1, 2, 3, 8),
                              (6, 140, 40, 6, 6, 8), (7, 261, 64, 6, 6, 8), (31, 520, 20, 6, 6, 8),
                              (26, 260, 16, 6, 6, 16), (14, 140, 7, 5, 8, 16)]:
        level = rng.random((H, W, 32)).astype(np.float32)
        C = rng.normal(size=(32, R)).astype(np.float32)
        cores = [rng.normal(0, 0.05, (h, w, R)).astype(np.float32) for _ in range(nf)]
        plans = []
        for tc in (True, False):
            plan = Plan(32, [(H, W)], C, [FilterDef(c) for c in cores],
                        apps=[(0, f) for f in range(nf)], outputs=(), tensor_cores=tc,
                        tc_ranks=(8, 16), tc_generic=True, tc_min_strips=0)
            assert bool(plan._tc_classes) == tc
            plan.load_levels(0, [level])
            plan.run(stages=("project", "correlate"))
            plans.append(plan)
        P = O.project(level, C.astype(np.float64))
        for f in range(nf):
            ref = O.correlate3_full(P, cores[f])
            g_tc = plans[0].map(0, 0, f).double().cpu().numpy()
            g_ff = plans[1].map(0, 0, f).double().cpu().numpy()
            assert_map_close(g_tc, ref, f"tc {H}x{W} filter {f}")
            assert_map_close(g_tc, g_ff, f"tc vs ffma {H}x{W} filter {f}")


@pytest.mark.parametrize("shape,generic,name", [
    ((6, 6), False, "k2_tcgen05_6x6_R16_groups4"),   # corr_tc16.cu (the default)
    ((5, 7), True, "k2_tcgen05_5x7_R16_groups4"),    # generic-shape kernel, tc_generic
])
def test_tensor_core_multi_group_launch_matches_oracle(shape, generic, name):
    """tcgen05 groups of one (h, w, R, N) share one launch
    (dpm_correlate_tc_groups): 50 R = 16 filters in groups of 16 over three
    levels -- strips of different groups interleave on the persistent CTAs,
    which reload the core per group -- against the oracle and FFMA."""
    from paper_1707_03268_b200.engine import FilterDef, Plan

    rng = np.random.default_rng(13)
    levels = [(30, 300), (17, 140), (9, 600)]
    C = rng.normal(size=(32, 16)).astype(np.float32)
    cores = [rng.normal(0, 0.05, shape + (16,)).astype(np.float32) for _ in range(50)]
    data = [rng.random((H, W, 32)).astype(np.float32) for H, W in levels]
    plans = []
    for tc in (True, False):
        plan = Plan(32, levels, C, [FilterDef(c) for c in cores],
                    apps=[(k, f) for k in range(3) for f in range(50)], outputs=(),
                    tensor_cores=tc, tc_ranks=(8, 16), tc_generic=generic,
                    tc_min_strips=0)
        if tc:
            names = [c[0] for c in plan._tc_classes]
            assert names == [name], names
        plan.load_levels(0, data)
        plan.run(stages=("project", "correlate"))
        plans.append(plan)
    for k, lv in enumerate(data):
        P = O.project(lv, C.astype(np.float64))
        for f in range(0, 50, 7):
            ref = O.correlate3_full(P, cores[f])
            g_tc = plans[0].map(0, k, f).double().cpu().numpy()
            g_ff = plans[1].map(0, k, f).double().cpu().numpy()
            assert_map_close(g_tc, ref, f"tc level {k} filter {f}")
            assert_map_close(g_tc, g_ff, f"tc vs ffma level {k} filter {f}")


def test_part_correlation_cta_pairs_bit_identical_to_one_cta_kernel(monkeypatch):
    """The part shape (6 x 6 taps, R = 8) on CTA pairs (cta_group::2, M =
    256, corr_tc2.cu; forced with DPM_TC_PAIR=1): the same MMAs in the same
    order as the one-CTA kernel, so the maps are bit-identical -- odd and
    even output heights, one-row levels, 16..64 filters, more strips than
    SM pairs."""
    from paper_1707_03268_b200.engine import FilterDef, Plan

    rng = np.random.default_rng(12)
    levels = [(40, 300), (6, 140), (7, 261), (23, 1100), (12, 9000)]
    for nf in (12, 30, 48, 64):
        C = rng.normal(size=(32, 8)).astype(np.float32)
        cores = [rng.normal(0, 0.05, (6, 6, 8)).astype(np.float32) for _ in range(nf)]
        data = [rng.random((H, W, 32)).astype(np.float32) for H, W in levels]
        maps = []
        monkeypatch.setenv("DPM_TC_SEGMENT", "0")  # the pair kernel walks whole strips
        for pair in ("1", "0"):
            monkeypatch.setenv("DPM_TC_PAIR", pair)
            plan = Plan(32, levels, C, [FilterDef(c) for c in cores],
                        apps=[(k, f) for k in range(len(levels)) for f in range(nf)], outputs=(),
                        tensor_cores=True)
            plan.load_levels(0, data)
            plan.run(stages=("project", "correlate"))
            maps.append([[plan.map(0, k, f).cpu().numpy().copy() for f in range(nf)]
                         for k in range(len(levels))])
        for k in range(len(levels)):
            for f in range(nf):
                np.testing.assert_array_equal(maps[0][k][f], maps[1][k][f],
                                              err_msg=f"nf {nf} level {levels[k]} filter {f}")


def test_part_strip_segments_bit_identical_to_whole_strips(monkeypatch):
    """Row segments of the tcgen05 part strips (engine._segment_strips, used
    when a launch has fewer than 2 strips per SM) compute the same rows with
    the same MMAs as whole strips: bit-identical maps, at odd heights and one
    strip taller than the segment size; the segmented plan really splits."""
    from paper_1707_03268_b200.engine import FilterDef, Plan

    rng = np.random.default_rng(21)
    levels = [(90, 300), (7, 140), (41, 261), (130, 40)]
    nf = 24
    C = rng.normal(size=(32, 8)).astype(np.float32)
    cores = [rng.normal(0, 0.05, (6, 6, 8)).astype(np.float32) for _ in range(nf)]
    data = [rng.random((H, W, 32)).astype(np.float32) for H, W in levels]
    maps, nseg = [], []
    for seg in ("0", "1"):
        monkeypatch.setenv("DPM_TC_SEGMENT", seg)
        plan = Plan(32, levels, C, [FilterDef(c) for c in cores],
                    apps=[(k, f) for k in range(len(levels)) for f in range(nf)], outputs=(),
                    tensor_cores=True)
        nseg.append(sum(len(st) for *_, st, _ in plan._tc_classes))
        plan.load_levels(0, data)
        plan.run(stages=("project", "correlate"))
        maps.append([[plan.map(0, k, f).cpu().numpy().copy() for f in range(nf)]
                     for k in range(len(levels))])
    assert nseg[1] > nseg[0]
    for k in range(len(levels)):
        for f in range(nf):
            np.testing.assert_array_equal(maps[0][k][f], maps[1][k][f],
                                          err_msg=f"level {levels[k]} filter {f}")


def test_few_filter_kernel_deterministic_and_matches_oracle():
    """The few-filter K2 (correlate_few.cu: filter rows split across warps,
    partial sums added in a fixed order) gives bit-identical maps run to run,
    and matches the float64 oracle at 1e-5 for 15 x 15, 11 x 15 and 5 x 8
    groups of 2-8 filters at R = 32 (several rank chunks)."""
    from paper_1707_03268_b200.engine import FilterDef, Plan

    rng = np.random.default_rng(22)
    levels = [(70, 90), (23, 17), (16, 160)]
    shapes = [(15, 15), (15, 15), (11, 15), (11, 15), (5, 8), (5, 8), (5, 8), (5, 8), (5, 8)]
    C = rng.normal(size=(32, 32)).astype(np.float32)
    cores = [rng.normal(0, 0.05, (h, w, 32)).astype(np.float32) for h, w in shapes]
    data = [rng.random((H, W, 32)).astype(np.float32) for H, W in levels]
    runs = []
    for _ in range(2):
        plan = Plan(32, levels, C, [FilterDef(c) for c in cores],
                    apps=[(k, f) for k in range(len(levels)) for f in range(len(cores))],
                    outputs=(), tensor_cores=False)
        plan.load_levels(0, data)
        plan.run(stages=("project", "correlate"))
        runs.append({(k, f): plan.map(0, k, f).cpu().numpy().copy()
                     for k in range(len(levels)) for f in range(len(cores))})
    for key, m in runs[0].items():
        np.testing.assert_array_equal(m, runs[1][key], err_msg=f"run to run {key}")
        k, f = key
        filt = np.einsum("ijr,cr->ijc", cores[f].astype(np.float64), C.astype(np.float64))
        ref = O.correlate3_full(data[k].astype(np.float64), filt)
        assert_map_close(m, ref, f"level {levels[k]} filter {shapes[f]}")


def test_score_batch_pipelined_matches_full_run():
    """The chunk-pipelined public call returns exactly the detections of one
    full-batch run (same records as a set)."""
    wl = synth.workload(4)
    C, G = _shared(4, 8)
    sc = PyramidScorer(wl.bank, C, G, wl.pyramid, n_images=5, max_dets=1 << 18)
    host = sc.host_arena(pinned=True)
    for i in range(5):
        sc.fill_host(host, i, synth.hog_pyramid(4, i, wl.pyramid))
    sc.plan.X.copy_(host)
    sc.run()
    tot = np.concatenate([r["scores"].ravel() for img in range(5) for r in sc.results(img)])
    tau = float(np.quantile(tot, 0.995))
    sc.run(tau=tau)
    full = np.sort(sc.detections(), order=["image", "level", "component", "ry", "rx"])
    for chunk in (2, 5, 1):
        got = np.sort(sc.score_batch(host, tau, chunk_images=chunk),
                      order=["image", "level", "component", "ry", "rx"])
        assert got.tobytes() == full.tobytes()
    assert len(full) > 0


def test_gdt_envelope_matches_windowed_rstar_kernel():
    """Lower-envelope GDT (dpm_gdt_x / dpm_gdt_y) against the windowed r*
    kernel (dpm_assemble) on every assembly of a config-4 image: placed
    values bit-identical wherever the argmax is, exact ties (<= 4 ulps)
    otherwise; totals to the same ulps."""
    wl = synth.workload(4)
    C, G = _shared(4, 8)
    lv = synth.hog_pyramid(4, 1, wl.pyramid)
    plans = {}
    for gdt in (True, False):
        sc = PyramidScorer(wl.bank, C, G, wl.pyramid, envelope=gdt,
                           outputs=("totals", "positions", "placed"))
        sc.load_image(0, lv)
        sc.run()
        plans[gdt] = sc.plan
    assert plans[True]._asm_gdt.all() and not plans[False]._asm_gdt.any()
    ties = n = 0
    for a in range(len(plans[True].assemblies)):
        ga = {k: v.cpu().numpy() for k, v in plans[True].assembly_outputs(0, a).items()}
        wa = {k: v.cpu().numpy() for k, v in plans[False].assembly_outputs(0, a).items()}
        same = ga["positions"] == wa["positions"]
        assert np.array_equal(ga["placed"][same], wa["placed"][same])
        d = np.abs(ga["placed"][~same] - wa["placed"][~same])
        assert np.all(d <= 4 * np.spacing(np.abs(wa["placed"][~same]))), d.max()
        ties += int((~same).sum())
        n += same.size
        scale = np.abs(wa["totals"]).max()
        assert np.abs(ga["totals"] - wa["totals"]).max() <= 1e-12 * scale
    assert ties <= 1e-4 * n, (ties, n)


def _pruned_case(k):
    from conftest import golden_pruned

    g = load_golden("detect_pruned.npz")
    dec, pyr, planted, tau = golden_pruned(g, k)
    hyps = [(pyr[int(p[0])], B.Hypothesis(level=int(p[0]), root=(int(p[1]), int(p[2])),
                                           parts=tuple((int(p[3 + 2 * i]), int(p[4 + 2 * i]))
                                                       for i in range(len(dec.parts)))))
            for p in planted]
    return g, dec, pyr, hyps, tau


def _gpu_stacks(dec):
    def stacks(li, level):
        return (B.cp_partial_stack(level, dec.root_cp),
                [B.cp_partial_stack(level, p.cp) for p in dec.parts])
    return stacks


def _stats_tuple(st):
    return (st.positions_examined, dict(st.positions_pruned_at_rank), dict(st.part_pruned_at_rank),
            st.positions_killed_by_parts, st.multiplications)


@pytest.mark.parametrize("mode", ["kill", "lenient"])
def test_pruned_detect_kernel_isolated_exact(mode):
    """GPU detect(pruning=True) vs the oracle's restatement run on the GPU's own
    FP32 prefix maps: prune ranks, counters, detections and scores identical."""
    for k in range(3):
        g, dec, pyr, hyps, tau = _pruned_case(k)
        dets, st = B.detect(dec, pyr, tau, pruning=True, part_prune_mode=mode, collect_maps=True)
        odets, ost, omaps = O.detect_pruned(dec, pyr, tau, part_prune_mode=mode,
                                            stacks=_gpu_stacks(dec))
        assert _stats_tuple(st) == (ost["positions_examined"], ost["positions_pruned_at_rank"],
                                    ost["part_pruned_at_rank"], ost["positions_killed_by_parts"],
                                    ost["multiplications"]), (k, mode)
        for lm, om in zip(st.prune_maps, omaps):
            assert lm["rect"] == om["rect"]
            if lm["rect"] is not None:
                assert np.array_equal(lm["root_prune_rank"], om["root_prune_rank"])
                assert np.array_equal(lm["part_prune_rank"], om["part_prune_rank"])
        assert len(dets) == len(odets)
        for d, o in zip(dets, odets):
            h = d.hypothesis
            assert (h.level, tuple(h.root), tuple(map(tuple, h.parts))) == (o[0], o[1], o[2])
            assert d.score == o[3]


@pytest.mark.parametrize("mode", ["kill", "lenient"])
def test_pruned_detect_matches_reference_golden(mode):
    """GPU pruned detection vs the reference run (FP64 maps, FP64 calibration).
    Prune ranks may differ only where the deciding comparison is within the
    FP32 map tolerance of its threshold (calibrated thresholds sit exactly on
    positives' FP64 values); everything else -- detections, scores to 1e-5,
    part positions up to ties -- agrees."""
    for k in range(3):
        g, dec, pyr, hyps, tau = _pruned_case(k)
        m = f"q{k}_{mode}"
        dets, st = B.detect(dec, pyr, tau, pruning=True, part_prune_mode=mode, collect_maps=True)
        flips = np.zeros(0, dtype=bool)
        affected = set()
        for li, lm in enumerate(st.prune_maps):
            if lm["rect"] is None:
                continue
            rr, gr = lm["root_prune_rank"], g[f"{m}_rootrank{li}"]
            pr, gp = lm["part_prune_rank"], g[f"{m}_partrank{li}"]
            level = np.asarray(pyr[li], dtype=np.float64)
            ry0, ry1, rx0, rx1 = lm["rect"]
            rs = O.cp_partial_stack(level, dec.root_cp)
            scale = np.abs(rs).max()
            for iy, ix in zip(*np.nonzero(rr != gr)):
                r = min(v for v in (rr[iy, ix], gr[iy, ix]) if v) - 1
                gap = abs(rs[r, ry0 + iy, rx0 + ix] - dec.root_thresholds[r])
                assert gap <= 1e-5 * scale, (k, mode, li, iy, ix, gap)
                affected.add((li, ry0 + iy, rx0 + ix))
            for pi, part in enumerate(dec.parts):
                ps = O.cp_partial_stack(level, part.cp)
                pscale = np.abs(ps).max()
                for iy, ix in zip(*np.nonzero(pr[pi] != gp[pi])):
                    cands = [v for v in (pr[pi][iy, ix], gp[pi][iy, ix]) if v]
                    if not cands:
                        continue
                    r = min(cands) - 1
                    wm = O.window_max(ps[r], np.array([ry0 + iy + part.anchor[0]]),
                                      np.array([rx0 + ix + part.anchor[1]]), part.search_radius)
                    gap = abs(wm[0] - part.thresholds[r])
                    # a root pruned / killed earlier on one side leaves the part unchecked
                    assert gap <= 1e-5 * pscale or (li, ry0 + iy, rx0 + ix) in affected, \
                        (k, mode, li, pi, iy, ix, gap)
                    affected.add((li, ry0 + iy, rx0 + ix))
        ref = g[f"{m}_dets"]
        got = {(d.hypothesis.level, *d.hypothesis.root): d for d in dets}
        want = {(int(r[0]), int(r[1]), int(r[2])): r for r in ref}
        for key in set(got) ^ set(want):
            assert key in affected, (k, mode, key)
        for key in (set(got) & set(want)) - affected:
            d, r = got[key], want[key]
            assert abs(d.score - r[-1]) <= 1e-5 * max(1.0, abs(r[-1])), (k, mode, key)
        if not affected:
            assert [st.positions_examined, st.positions_killed_by_parts, st.multiplications] == \
                list(g[f"{m}_stats"])


def test_gpu_calibration_never_prunes_its_positives():
    """calibrate_thresholds on the GPU's prefix maps: thresholds within 1e-5 of
    the reference's FP64 calibration, and zero false pruning of the positives
    (the reference's acceptance criterion 4)."""
    for k in range(3):
        g, dec, pyr, hyps, tau = _pruned_case(k)
        cal = B.calibrate_thresholds(dec, hyps)
        scale = max(np.abs(dec.root_thresholds).max(), 1.0)
        assert np.abs(cal.root_thresholds - dec.root_thresholds).max() <= 1e-5 * scale
        for a, b in zip(cal.parts, dec.parts):
            assert np.abs(a.thresholds - b.thresholds).max() <= 1e-5 * scale
        for mode in ("kill", "lenient"):
            _, st = B.detect(cal, pyr, -np.inf, pruning=True, part_prune_mode=mode,
                             collect_maps=True)
            for lvl, hyp in hyps:
                li = hyp.level
                lm = st.prune_maps[li]
                iy, ix = hyp.root[0] - lm["rect"][0], hyp.root[1] - lm["rect"][2]
                assert lm["root_prune_rank"][iy, ix] == 0
                assert not lm["part_prune_rank"][:, iy, ix].any()


def test_roc_eval_matches_reference_golden():
    """roc_eval over the GPU detectors equals the reference's sweep: dense,
    decomposed, and pruned with thresholds calibrated on the GPU maps."""
    from types import SimpleNamespace

    from conftest import _Dec, _Part
    from paper_1707_03268_b200.evaluation import roc_eval

    g = load_golden("roc.npz")
    nparts = 2
    scenes = []
    for si in range(3):
        pl = g[f"s{si}_planted"]
        planted = [(int(p[0]), B.Hypothesis(level=int(p[0]), root=(int(p[1]), int(p[2])),
                                            parts=tuple((int(p[3 + 2 * i]), int(p[4 + 2 * i]))
                                                        for i in range(nparts))))
                   for p in pl]
        scenes.append(SimpleNamespace(pyramid=[g[f"s{si}_level0"]], planted=planted))
    dense = B.PartModel(g["root"], tuple(
        B.PartSpec(g[f"part{i}"], tuple(g[f"part{i}_anchor"]), tuple(g[f"part{i}_def"]),
                   int(g[f"part{i}_r"])) for i in range(nparts)), float(g["bias"]))
    parts = [_Part(golden_cp(g, f"pcp{i}"), g[f"part{i}_anchor"], g[f"part{i}_def"],
                   g[f"part{i}_r"], None) for i in range(nparts)]
    dec = _Dec(golden_cp(g, "rcp"), parts, g["bias"], None)
    taus = g["taus"]

    def pts(points):
        return np.array([[p.tau, p.misdetection_rate, p.false_positives_per_scene,
                          p.false_positives_per_window] for p in points])
    assert np.array_equal(pts(roc_eval(dense, scenes, taus)), g["roc_dense"])
    assert np.array_equal(pts(roc_eval(dec, scenes, taus)), g["roc_cp"])
    positives = [(sc.pyramid[lvl], hyp) for sc in scenes for lvl, hyp in sc.planted]
    cal = B.calibrate_thresholds(dec, positives)
    assert np.array_equal(pts(roc_eval(cal, scenes, taus, pruning=True)), g["roc_pruned"])


def test_mixture_max_matches_host_composition():
    """dpm_mixture_max (per-root max over components, ties to the lowest
    component) equals the same rule applied to the per-component totals, on
    config 5 (components with different root shapes) at sampled levels."""
    wl = synth.workload(5)
    C, G = _shared(5, 8)
    sc = PyramidScorer(wl.bank, C, G, wl.pyramid, n_images=1)
    sc.load_image(0, synth.hog_pyramid(5, 0, wl.pyramid))
    sc.run()
    mix = sc.mixture()
    res = sc.results(0)
    by_level = {}
    for r in res:
        by_level.setdefault(r["root_level"], []).append(r)
    assert set(k[1] for k in mix) == set(by_level)
    for lvl, recs in by_level.items():
        rect, best, comp = mix[(0, lvl)]
        best, comp = best.cpu().numpy(), comp.cpu().numpy()
        ry0, ry1, rx0, rx1 = rect
        want = np.full(best.shape, -np.inf)
        wcomp = np.full(best.shape, -1)
        for r in sorted(recs, key=lambda r: r["component"]):
            a0, a1, b0, b1 = r["rect"]
            sub = (slice(a0 - ry0, a1 - ry0 + 1), slice(b0 - rx0, b1 - rx0 + 1))
            better = (wcomp[sub] < 0) | (r["scores"] > want[sub])
            want[sub] = np.where(better, r["scores"], want[sub])
            wcomp[sub] = np.where(better, r["component"], wcomp[sub])
        assert np.array_equal(best, want) and np.array_equal(comp, wcomp), lvl


def test_pinned_pyramid_loader_feeds_score_batch(tmp_path):
    """T3F feature levels read straight into the pinned arena equal fill_host's
    arena, and score_batch from it gives the same detections."""
    from paper_1707_03268_b200 import formats as F

    wl = synth.workload(2)
    C, G = _shared(2, 8)
    sc = PyramidScorer(wl.bank, C, G, wl.pyramid, n_images=2, max_dets=1 << 16)
    a = sc.host_arena(pinned=True)
    b = sc.host_arena(pinned=True)
    a.zero_()
    b.zero_()
    for img in range(2):
        lv = synth.hog_pyramid(2, img, wl.pyramid)
        sc.fill_host(a, img, lv)
        paths = []
        for k, l in enumerate(lv):
            paths.append(str(tmp_path / f"i{img}_l{k}.t3f"))
            F.write_t3f(paths[-1], l)
        F.load_pyramid_pinned(sc, b, img, paths)
    assert np.array_equal(a.numpy(), b.numpy())
    da, db = sc.score_batch(a, 2.0), sc.score_batch(b, 2.0)
    key = lambda d: np.sort(d, order=["image", "level", "component", "ry", "rx"])  # noqa: E731
    assert np.array_equal(key(da), key(db)) and len(da) > 0


# ---------------------------------------------- reference test-suite mirrors
# (pkg/tests/test_correlation.py:71-116, test_detection.py:169-240, 318-590)

def test_correlation_known_answers():
    rng = np.random.default_rng(0)
    img = rng.normal(size=(4, 5, 1))
    sm = B.correlate3_full(img, np.full((1, 1, 1), 2.0))
    assert_map_close(sm.scores, 2.0 * img[:, :, 0], "scalar filter")
    assert sm.multiplications == 4 * 5
    img = rng.normal(size=(5, 6, 3))
    filt = np.zeros((2, 2, 3))
    filt[0, 0, 0] = 1.0
    assert_map_close(B.correlate3_full(img, filt).scores, img[0:4, 0:5, 0], "delta filter")
    # rank-1 CP == dense correlation with the reconstructed filter
    img = rng.normal(size=(7, 6, 3))
    a, b, c = rng.normal(size=3), rng.normal(size=2), rng.normal(size=3)
    cp = B.CPModel.from_factors(a[:, None], b[:, None], c[:, None])
    dense = np.einsum("r,ir,jr,kr->ijk", cp.weights, cp.factors_a, cp.factors_b, cp.factors_c)
    assert_map_close(B.correlate3_cp(img, cp).scores, B.correlate3_full(img, dense).scores,
                     "rank-1 separable")


def _rand_dec(rng, root=(3, 4), parts=((4, 4), (4, 4)), L=6, R=2):
    from conftest import CP, _Dec, _Part

    def cp(n, m):
        return CP(np.abs(rng.normal(size=R)) + 0.5, rng.normal(size=(n, R)) / np.sqrt(n),
                  rng.normal(size=(m, R)) / np.sqrt(m), rng.normal(size=(L, R)) / np.sqrt(L))
    ps = [_Part(cp(*d), (i, 2 * i), (0.0, 0.0, 0.05, 0.05), 2, None)
          for i, d in enumerate(parts)]
    return _Dec(cp(*root), ps, 0.1, None)


def test_detect_root_only_model_and_degenerate_pyramids():
    rng = np.random.default_rng(50)
    dec = _rand_dec(rng, parts=())
    level = rng.normal(size=(20, 24, 6))
    root = O.cp_partial_stack(level, dec.root_cp)[-1] + dec.bias
    tau = float(np.quantile(root, 0.9))
    dets, st = B.detect(dec, [level], tau)
    got = {d.hypothesis.root for d in dets}
    want = {(int(y), int(x)) for y, x in zip(*np.nonzero(root >= tau))}
    near = {(int(y), int(x)) for y, x in zip(*np.nonzero(np.abs(root - tau) <= 1e-5 * abs(root).max()))}
    assert got ^ want <= near and all(d.hypothesis.parts == () for d in dets)
    # calibrated on its own top hypothesis, pruning keeps it and prunes others
    iy, ix = np.unravel_index(np.argmax(root), root.shape)
    cal = B.calibrate_thresholds(dec, [(level, B.Hypothesis(level=0, root=(int(iy), int(ix))))])
    pdets, pst = B.detect(cal, [level], tau, pruning=True)
    assert (int(iy), int(ix)) in {d.hypothesis.root for d in pdets}
    assert pst.positions_pruned > 0
    # degenerate pyramids (test_detection.py:522-530)
    dec2 = _rand_dec(rng)
    none, st0 = B.detect(dec2, [], -np.inf)
    assert none == [] and st0.positions_examined == 0
    dec3 = _rand_dec(rng, parts=((6, 6),))  # level fits the root, not the part
    found, st1 = B.detect(dec3, [np.zeros((5, 6, 6))], -np.inf)
    assert found == [] and st1.positions_examined == 0
    with pytest.raises(B.ValidationError, match="channel"):
        B.detect(dec2, [np.zeros((20, 20, 3))], 0.0)


def test_pruned_subset_identical_scores_invariants_determinism():
    for k in range(3):
        g, dec, pyr, hyps, tau = _pruned_case(k)
        cal = B.calibrate_thresholds(dec, hyps)
        tau = min(float(h.score) for _, h in hyps if h.score is not None) - 20.0 \
            if all(h.score is not None for _, h in hyps) else 0.0
        off, soff = B.detect(cal, pyr, tau, pruning=False)
        on, son = B.detect(cal, pyr, tau, pruning=True)
        offi = {(d.hypothesis.level, d.hypothesis.root): d.score for d in off}
        oni = {(d.hypothesis.level, d.hypothesis.root): d.score for d in on}
        assert set(oni) <= set(offi)
        assert all(oni[key] == offi[key] for key in oni)  # survivors: identical full sums
        assert son.multiplications <= soff.multiplications
        assert son.positions_pruned + son.positions_surviving == son.positions_examined
        on2, son2 = B.detect(cal, pyr, tau, pruning=True)
        assert [(d.hypothesis.level, d.hypothesis.root, d.score) for d in on] == \
            [(d.hypothesis.level, d.hypothesis.root, d.score) for d in on2]
        assert son.positions_pruned_at_rank == son2.positions_pruned_at_rank
        assert son.multiplications == son2.multiplications


def test_calibration_known_answers():
    g, dec, pyr, hyps, tau = _pruned_case(0)
    level, hyp = hyps[0]
    one = B.calibrate_thresholds(dec, [(level, hyp)])
    rs = B.cp_partial_stack(level, dec.root_cp)
    assert np.array_equal(one.root_thresholds, rs[:, hyp.root[0], hyp.root[1]])
    for p, (py, px) in zip(one.parts, hyp.parts):
        ps = B.cp_partial_stack(level, p.cp)
        assert np.array_equal(p.thresholds, ps[:, py, px])
    once = B.calibrate_thresholds(dec, hyps)
    twice = B.calibrate_thresholds(dec, hyps + hyps)
    assert np.array_equal(once.root_thresholds, twice.root_thresholds)
    bad = B.Hypothesis(level=0, root=hyp.root,
                       parts=((hyp.parts[0][0] + 9, hyp.parts[0][1]),) + tuple(hyp.parts[1:]))
    with pytest.raises(B.ValidationError, match="search radius|out of support"):
        B.calibrate_thresholds(dec, [(level, bad)])


@pytest.mark.parametrize("seed", range(40))
def test_randomized_plans_against_oracle(seed):
    """Seeded random plans: filter shapes 1..8 x 1..12, ranks {1, 3, 8, 16}
    (tcgen05 and FFMA classes), levels down to filter size, scale 1 or 2,
    windowed radii {0, 1, 3, 17 (> the staged cap)} or the unbounded r*,
    zero / negative linear deformation terms.  Maps within 1e-5 of the FP64
    oracle; placement and totals bit-identical to the oracle run on the GPU's
    own maps."""
    from paper_1707_03268_b200.engine import AssemblyDef, FilterDef, PartDef, Plan
    from paper_1707_03268_b200.geometry import gdt_root_rect

    rng = np.random.default_rng(1000 + seed)
    L = int(rng.choice([4, 7, 32]))
    R = int(rng.choice([1, 3, 8, 16]))
    scale = int(rng.integers(1, 3))
    gdt = bool(rng.integers(0, 2))
    C = rng.normal(size=(L, R)).astype(np.float32)
    rh, rw = int(rng.integers(1, 7)), int(rng.integers(1, 13))
    nparts = int(rng.integers(0, 4))
    pshapes = [(int(rng.integers(1, 9)), int(rng.integers(1, 9))) for _ in range(nparts)]
    Hr = max([rh] + [h for h, _ in pshapes]) + int(rng.integers(0, 30))
    Wr = max([rw] + [w for _, w in pshapes]) + int(rng.integers(0, 150))
    Hp, Wp = (Hr, Wr) if scale == 1 else (2 * Hr + int(rng.integers(0, 3)), 2 * Wr + int(rng.integers(0, 3)))
    Hp = max(Hp, max([s[0] for s in pshapes], default=1))
    Wp = max(Wp, max([s[1] for s in pshapes], default=1))
    levels = [(Hr, Wr)] if scale == 1 else [(Hr, Wr), (Hp, Wp)]
    kp = 0 if scale == 1 else 1
    cores = [rng.normal(0, 0.3, (rh, rw, R)).astype(np.float32)] + \
        [rng.normal(0, 0.3, (h, w, R)).astype(np.float32) for h, w in pshapes]
    filters = [FilterDef(c) for c in cores]
    defs, anchors = [], []
    for h, w in pshapes:
        q = rng.uniform(0.005, 0.1, 2) if gdt else rng.choice([0.0, 0.02, 0.1], 2)
        defs.append((float(rng.uniform(-0.05, 0.05)), float(rng.uniform(-0.05, 0.05)),
                     float(q[0]), float(q[1])))
        anchors.append((int(rng.integers(0, max(1, scale * rh))), int(rng.integers(0, max(1, scale * rw)))))
    radius = -1 if gdt else int(rng.choice([0, 1, 3, 17]))
    rs = (Hr - rh + 1, Wr - rw + 1)
    if gdt:
        rect = gdt_root_rect(rs, [(Hp - h + 1, Wp - w + 1) for h, w in pshapes], anchors, scale)
        if rect is None:
            pytest.skip("empty GDT domain for this draw")
    else:  # every part window within r of its support (as _hypothesis_rect, scaled)
        ry0, ry1, rx0, rx1 = 0, rs[0] - 1, 0, rs[1] - 1
        for (h, w), (ay, ax) in zip(pshapes, anchors):
            sy, sx = Hp - h + 1, Wp - w + 1
            ry0 = max(ry0, -((ay + radius) // scale))
            ry1 = min(ry1, (sy - 1 + radius - ay) // scale)
            rx0 = max(rx0, -((ax + radius) // scale))
            rx1 = min(rx1, (sx - 1 + radius - ax) // scale)
        if ry0 > ry1 or rx0 > rx1:
            pytest.skip("empty root rectangle for this draw")
        rect = (ry0, ry1, rx0, rx1)
    parts = tuple(PartDef(kp, 1 + i, anchors[i], defs[i], radius, scale) for i in range(nparts))
    asm = AssemblyDef((0, 0), rect, parts, bias=0.25)
    plan = Plan(L, levels, C, filters, assemblies=[asm], outputs=("totals", "positions", "placed"))
    X = [rng.uniform(0, 0.4, (h, w, L)).astype(np.float32) for h, w in levels]
    plan.load_levels(0, X)
    plan.run()
    P = [O.project(x.astype(np.float64), C.astype(np.float64)) for x in X]
    gmaps = []
    for f, core in enumerate(cores):
        k = 0 if f == 0 else kp
        ref = O.correlate3_full(P[k], core.astype(np.float64))
        gm = plan.map(0, k, f).double().cpu().numpy()
        assert_map_close(gm, ref, f"seed {seed} filter {f}")
        gmaps.append(gm)
    out = {k: v.cpu().numpy() for k, v in plan.assembly_outputs(0, 0).items()}
    ry0, ry1, rx0, rx1 = rect
    tot = gmaps[0][ry0:ry1 + 1, rx0:rx1 + 1].copy()
    for i in range(nparts):
        r = O.r_star(gmaps[1 + i], defs[i]) if gdt else radius
        placed, py, px = O.place_gathered(gmaps[1 + i], anchors[i], defs[i], r, scale, rect)
        from paper_1707_03268_b200.engine import unpack_positions

        gy, gx = unpack_positions(out["positions"][i])
        assert np.array_equal(out["placed"][i], placed), (seed, i)
        assert np.array_equal(gy, py) and np.array_equal(gx, px), (seed, i)
        tot = tot + placed
    assert np.array_equal(out["totals"], tot + 0.25), seed
    if gdt and nparts:  # the lower-envelope kernels: same placements up to exact ties
        env = Plan(L, levels, C, filters, assemblies=[asm],
                   outputs=("totals", "positions", "placed"), envelope=True)
        assert env._asm_gdt.all()
        env.load_levels(0, X)
        env.run()
        eo = {k: v.cpu().numpy() for k, v in env.assembly_outputs(0, 0).items()}
        same = eo["positions"] == out["positions"]
        assert np.array_equal(eo["placed"][same], out["placed"][same])
        d = np.abs(eo["placed"][~same] - out["placed"][~same])
        assert np.all(d <= 4 * np.spacing(np.abs(out["placed"][~same]))), seed


def test_plan_run_is_cuda_graph_capturable():
    """One Plan.run() captured into a CUDA graph and replayed gives the same
    totals, positions and detections as direct launches (no host sync, no
    allocation inside run())."""
    import torch

    wl = synth.workload(2)
    C, G = _shared(2, 8)
    sc = PyramidScorer(wl.bank, C, G, wl.pyramid, max_dets=1 << 16)
    sc.load_image(0, synth.hog_pyramid(2, 0, wl.pyramid))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        sc.plan.run(tau=2.0, stream=s)
    torch.cuda.synchronize()
    direct = [(r["scores"].copy(), r["parts"].copy()) for r in sc.results(0)]
    ndirect = int(sc.plan.det_count.item())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        sc.plan.run(tau=2.0, stream=s)
    sc.plan.totals.zero_()
    g.replay()
    torch.cuda.synchronize()
    for (ts, tp), r in zip(direct, sc.results(0)):
        assert np.array_equal(ts, r["scores"]) and np.array_equal(tp, r["parts"])
    assert int(sc.plan.det_count.item()) == ndirect > 0


def test_batched_apis_score_pyramid_and_detect_batch():
    """score_pyramid == PyramidScorer.results for one image; detect_batch ==
    the detections implied by the per-image totals (same records)."""
    wl = synth.workload(2)
    C, G = _shared(2, 8)
    lv0, lv1 = (synth.hog_pyramid(2, i, wl.pyramid) for i in (0, 1))
    res = B.score_pyramid(wl.bank, C, G, wl.pyramid, lv0)
    sc = PyramidScorer(wl.bank, C, G, wl.pyramid)
    sc.load_image(0, lv0)
    for a, b in zip(res, sc.run().results(0)):
        assert np.array_equal(a["scores"], b["scores"]) and np.array_equal(a["parts"], b["parts"])
    tau = 2.0
    dets = B.detect_batch(wl.bank, C, G, wl.pyramid, [lv0, lv1], tau)
    got = sorted((int(d["image"]), int(d["level"]), int(d["component"]), int(d["ry"]),
                  int(d["rx"])) for d in dets)
    want = []
    for img, lv in ((0, lv0), (1, lv1)):
        for r in B.score_pyramid(wl.bank, C, G, wl.pyramid, lv):
            ry0, _, rx0, _ = r["rect"]
            for iy, ix in zip(*np.nonzero(r["scores"] >= tau)):
                want.append((img, r["root_level"], r["component"], ry0 + int(iy), rx0 + int(ix)))
    assert got == sorted(want) and len(got) > 0


def test_rank_prefix_kernel_one_pass_matches_oracle_and_costs_one_correlation():
    """Convolution shortening (paper Algorithm 1): the rank-prefix K2 writes
    every cumulative prefix of a CP filter from one pass over the ranks.
    Prefixes match the float64 reference stack to 1e-5 (and the oracle's
    term-then-cumsum restatement on the same FP32 inputs to 2e-6), the last
    prefix equals correlate3_cp bit for bit, and on config 1 (9 per-filter
    CP models at R = 8) computing all prefixes costs about one full
    correlation, not R of them."""
    import torch

    from paper_1707_03268_b200.correlation import cp_core
    from paper_1707_03268_b200.engine import FilterDef, Plan

    rng = np.random.default_rng(11)
    for ishape, dims, rank in [((40, 52, 32), (6, 6, 32), 8), ((30, 33, 7), (3, 5, 7), 5),
                               ((19, 24, 32), (15, 15, 32), 3), ((9, 9, 4), (1, 1, 4), 4)]:
        img = rng.normal(size=ishape).astype(np.float32).astype(np.float64)
        cp = B.CPModel.from_factors(rng.normal(size=(dims[0], rank)), rng.normal(size=(dims[1], rank)),
                                    rng.normal(size=(dims[2], rank)))
        stack = B.cp_partial_stack(img, cp)
        ref = O.cp_partial_stack(img, cp)
        for r in range(rank):
            assert_map_close(stack[r], ref[r], f"{dims} prefix {r + 1}")
        assert np.array_equal(B.correlate3_cp(img, cp).scores, stack[-1])

    # cost on config 1: all 8 prefixes of 9 filters vs the 9 full filters
    g = load_golden("cfg1.npz")
    level = synth.hog_level(1, 0, 0, 64, 48)
    cps = [golden_cp(g, "root")] + [golden_cp(g, f"part{i}") for i in range(8)]
    C = np.concatenate([np.asarray(c.factors_c, np.float32) for c in cps], axis=1)

    def k2_ms(prefix):
        filters, off = [], 0
        for c in cps:
            core = cp_core(c)
            if prefix:
                filters += [FilterDef(core, chan_off=off, prefix=k + 1) for k in range(c.rank)]
            else:
                filters.append(FilterDef(core, chan_off=off))
            off += c.rank
        plan = Plan(32, [(64, 48)], C, filters, apps=[(0, f) for f in range(len(filters))],
                    outputs=(), tensor_cores=False)
        plan.load_levels(0, [level])
        for _ in range(3):
            plan.run(stages=("correlate",))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(50):
            plan.run(stages=("correlate",))
        ev[1].record()
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / 50

    full, pref = k2_ms(False), k2_ms(True)
    print(f"config 1 K2: full filters {full * 1e3:.1f} us, all rank prefixes {pref * 1e3:.1f} us")
    assert pref <= 1.5 * full + 0.01, (pref, full)
