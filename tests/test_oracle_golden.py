"""Pin the CPU oracle against the reference's own outputs and constants.

The golden vectors were produced by running the reference package
(``tests/golden/make_golden.py``); the constants below are the reference
tests' known answers (``pkg/tests/test_correlation.py:218-245``,
``pkg/tests/test_detection.py:120-166``).
"""

import numpy as np
import pytest

from conftest import golden_cp, load_golden
from oracle import dpm_oracle as O
from paper_1707_03268_b200 import geometry, synth


def test_correlate3_full_matches_reference():
    g = load_golden("correlation.npz")
    for k in range(int(g["n_full"])):
        out = O.correlate3_full(g[f"full{k}_img"], g[f"full{k}_filt"])
        ref = g[f"full{k}_out"]
        np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
        img, filt = g[f"full{k}_img"], g[f"full{k}_filt"]
        assert geometry.full_multiplications(img.shape, filt.shape) == int(g[f"full{k}_mult"])


def test_cp_partial_stack_bit_identical_to_reference():
    g = load_golden("correlation.npz")
    for k in range(int(g["n_cp"])):
        cp = golden_cp(g, f"cp{k}")
        img = g[f"cp{k}_img"]
        stack = O.cp_partial_stack(img, cp)
        assert np.array_equal(stack, g[f"cp{k}_stack"]), k
        up = int(g[f"cp{k}_upto"])
        assert np.array_equal(O.correlate3_cp(img, cp, up), g[f"cp{k}_upto_out"])
        assert geometry.cp_multiplications(img.shape, cp.dims, up) == int(g[f"cp{k}_upto_mult"])


def test_placement_grid_bit_identical_to_reference():
    g = load_golden("placement.npz")
    for k in range(int(g["n"])):
        placed, py, px = O.placement_grid(g[f"p{k}_map"], tuple(g[f"p{k}_anchor"]),
                                          tuple(g[f"p{k}_def"]), int(g[f"p{k}_r"]),
                                          tuple(int(v) for v in g[f"p{k}_rect"]))
        assert np.array_equal(placed, g[f"p{k}_placed"]), k
        assert np.array_equal(py, g[f"p{k}_py"]), k
        assert np.array_equal(px, g[f"p{k}_px"]), k


def test_best_part_placement_matches_reference():
    g = load_golden("placement.npz")
    for k in range(int(g["n"])):
        for ry, rx, y, x, v, ok in g[f"p{k}_scalar"]:
            args = (g[f"p{k}_map"], tuple(g[f"p{k}_anchor"]), tuple(g[f"p{k}_def"]),
                    int(g[f"p{k}_r"]), (int(ry), int(rx)))
            if ok:
                pos, val = O.best_part_placement(*args)
                assert pos == (int(y), int(x)) and val == v
            else:
                with pytest.raises(ValueError, match="empty"):
                    O.best_part_placement(*args)


def test_placement_known_answers():
    # pkg/tests/test_detection.py:157-160 - ties go to the smallest (dy, dx)
    assert O.best_part_placement(np.zeros((5, 5)), (0, 0), (0, 0, 0, 0), 1, (2, 2)) == ((1, 1), 0.0)
    # :130-135 huge quadratic pins the anchor
    rng = np.random.default_rng(7)
    s = rng.normal(size=(9, 9))
    assert O.best_part_placement(s, (0, 0), (0, 0, 1e9, 1e9), 3, (4, 4))[0] == (4, 4)
    # :120-127 zero coefficients = window max
    s = np.random.default_rng(6).normal(size=(9, 9))
    pos, val = O.best_part_placement(s, (0, 0), (0, 0, 0, 0), 2, (4, 4))
    assert val == s[2:7, 2:7].max() and s[pos] == val
    # :163-166 empty window
    with pytest.raises(ValueError, match="empty"):
        O.best_part_placement(np.zeros((5, 5)), (10, 10), (0, 0, 0, 0), 1, (0, 0))


def test_counter_known_answers():
    # pkg/tests/test_correlation.py:218-245
    assert geometry.theoretical_gain(8, 8, 32, 6) == 2048 / 288
    assert geometry.theoretical_gain(5, 11, 32, 6) == 1760 / 288
    assert geometry.theoretical_gain(4, 4, 8, 8) == 1.0
    assert geometry.full_multiplications((6, 7, 3), (2, 3, 3)) == 5 * 5 * 2 * 3 * 3
    for rank in (1, 2, 5):
        assert geometry.cp_multiplications((6, 7, 3), (2, 3, 3), rank) == rank * 5 * 5 * 8


def _compact(g, k):
    pre = f"d{k}"
    levels = [g[f"{pre}_level{i}"] for i in range(int(g[f"{pre}_nlevels"]))]

    class Part:
        pass

    parts, dparts = [], []
    for i in range(int(g[f"{pre}_nparts"])):
        p = Part()
        p.filter = g[f"{pre}_part{i}"]
        p.anchor = tuple(int(v) for v in g[f"{pre}_part{i}_anchor"])
        p.deformation = tuple(float(v) for v in g[f"{pre}_part{i}_def"])
        p.search_radius = int(g[f"{pre}_part{i}_r"])
        d = Part()
        d.cp = golden_cp(g, f"{pre}_pcp{i}")
        d.anchor, d.deformation, d.search_radius = p.anchor, p.deformation, p.search_radius
        parts.append(p)
        dparts.append(d)
    model, dec = Part(), Part()
    model.root, model.parts, model.bias = g[f"{pre}_root"], parts, float(g[f"{pre}_bias"])
    dec.root_cp, dec.parts, dec.bias = golden_cp(g, f"{pre}_rcp"), dparts, model.bias
    return levels, model, dec


def _unpack(dets):
    return np.array([[d[0], *d[1], *[c for pp in d[2] for c in pp], d[3]] for d in dets])


def test_detect_and_dense_detect_match_reference():
    g = load_golden("detect_compact.npz")
    for k in range(int(g["n"])):
        levels, model, dec = _compact(g, k)
        dets, stats = O.detect(dec, levels, -np.inf)
        got, ref = _unpack(dets), g[f"d{k}_dets"]
        assert got.shape == ref.shape
        assert np.array_equal(got[:, :-1], ref[:, :-1])
        np.testing.assert_allclose(got[:, -1], ref[:, -1], rtol=1e-12, atol=1e-12)
        assert [stats["positions_examined"], stats["multiplications"]] == list(g[f"d{k}_stats"])
        ddets, dstats = O.dense_detect(model, levels, -np.inf)
        got, ref = _unpack(ddets), g[f"d{k}_ddets"]
        assert np.array_equal(got[:, :-1], ref[:, :-1])
        np.testing.assert_allclose(got[:, -1], ref[:, -1], rtol=1e-12, atol=1e-12)
        assert [dstats["positions_examined"], dstats["multiplications"]] == list(g[f"d{k}_dstats"])
        h = g[f"d{k}_hyp"]
        lv = levels[int(h[0])]
        root, parts = (int(h[1]), int(h[2])), [(int(h[3 + 2 * i]), int(h[4 + 2 * i]))
                                               for i in range(len(model.parts))]
        assert O.score_hypothesis(model, lv, root, parts) == pytest.approx(
            float(g[f"d{k}_score_hyp"]), rel=1e-12)
        assert O.cp_score_hypothesis(dec, lv, root, parts) == pytest.approx(
            float(g[f"d{k}_cp_score_hyp"]), rel=1e-12)


def test_config1_reference_native_and_shared_basis():
    g = load_golden("cfg1.npz")
    wl = synth.workload(1)
    level = synth.hog_level(1, 0, 0, 64, 48)
    assert float(level.astype(np.float64).sum()) == float(g["level_sum"])
    bank, comp = wl.bank, wl.bank.components[0]

    class Obj:
        pass

    dec = Obj()
    dec.root_cp, dec.bias = golden_cp(g, "root"), comp.bias
    dec.parts = []
    for i, (a, d) in enumerate(zip(comp.anchors, comp.deformations)):
        p = Obj()
        p.cp, p.anchor, p.deformation, p.search_radius = golden_cp(g, f"part{i}"), a, d, 2
        dec.parts.append(p)
    np.testing.assert_array_equal(O.cp_partial_stack(level, dec.root_cp)[-1], g["root_map"])
    dets, stats = O.detect(dec, [level], -np.inf)
    got = _unpack(dets)[:, 1:]
    ref = g["dets"]
    assert np.array_equal(got[:, :-1], ref[:, :-1])
    np.testing.assert_allclose(got[:, -1], ref[:, -1], rtol=1e-12, atol=1e-12)
    assert [stats["positions_examined"], stats["multiplications"]] == list(g["stats"])
    assert stats["positions_examined"] == (57 - 3 + 1) * (24 - 2 + 1)  # rect (3,57,2,24)

    # shared basis: oracle composition (project + correlate3_full with the core)
    C, G = g["shared_C"], g["shared_G"]
    offs = bank.offsets()
    cores = [G[o:o + f.shape[0] * f.shape[1]].reshape(f.shape[0], f.shape[1], -1)
             for f, o in zip(bank.filters, offs)]
    P = O.project(level, C)
    root_map = O.correlate3_full(P, cores[comp.root])
    rect = O.hypothesis_rect(level.shape, (6, 11), [(6, 6)] * 8, comp.anchors, [2] * 8)
    placements = [O.placement_grid(O.correlate3_full(P, cores[f]), a, d, 2, rect)
                  for f, a, d in zip(comp.parts, comp.anchors, comp.deformations)]
    out = []
    O._assemble(0, rect, root_map, placements, comp.bias, -np.inf, out)
    got = _unpack(sorted(out, key=lambda d: (d[0], d[1])))[:, 1:]
    ref = g["shared_dets"]
    assert np.array_equal(got[:, :-1], ref[:, :-1])
    np.testing.assert_allclose(got[:, -1], ref[:, -1], rtol=1e-10, atol=1e-10)


def test_config2_sample_composition_matches_reference():
    g = load_golden("cfg2_sample.npz")
    wl = synth.workload(2)
    fx = np.load(synth_factor_path(2, 8))
    C, G = fx["C"], fx["G"]
    bank, pyr = wl.bank, wl.pyramid
    cores = [G[o:o + f.shape[0] * f.shape[1]].reshape(f.shape[0], f.shape[1], -1)
             for f, o in zip(bank.filters, bank.offsets())]
    for k in range(int(g["n"])):
        i, ci = (int(v) for v in g[f"s{k}_sel"])
        kr, kp = pyr.root_levels[i], pyr.part_levels[i]
        levels = {kr: synth.hog_level(2, 0, kr, *pyr.levels[kr]),
                  kp: synth.hog_level(2, 0, kp, *pyr.levels[kp])}
        lv = [levels.get(j, np.zeros((1, 1, 32), np.float32)) for j in range(len(pyr.levels))]
        res, _ = O.score_pyramid(lv, bank, C, cores, root_levels=[kr], part_levels=[kp],
                                 components=[bank.components[ci]])
        assert len(res) == 1
        assert tuple(res[0]["rect"]) == tuple(int(v) for v in g[f"s{k}_rect"])
        ref = g[f"s{k}_scores"]
        np.testing.assert_allclose(res[0]["scores"], ref, rtol=1e-10, atol=1e-10)
        assert np.array_equal(res[0]["parts"], g[f"s{k}_parts"])


def synth_factor_path(cfg, R):
    import os
    from conftest import REPO
    return os.path.join(REPO, "paper_1707_03268_b200", "data", f"factors_cfg{cfg}_R{R}.npz")


def test_r_star_window_equals_unbounded():
    # placement at r* equals a much larger radius for
    # centres inside the map
    rng = np.random.default_rng(5)
    s = rng.normal(size=(40, 50)) * 0.3
    de = (0.0, 0.0, 0.01, 0.01)
    r = O.r_star(s, de)
    rect = (0, 39, 0, 49)
    a = O.placement_grid(s, (0, 0), de, r, rect)
    b = O.placement_grid(s, (0, 0), de, 60, rect)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    de = (0.003, -0.002, 0.02, 0.01)
    r = O.r_star(s, de)
    a = O.placement_grid(s, (0, 0), de, r, rect)
    b = O.placement_grid(s, (0, 0), de, 60, rect)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_oracle_pruned_detect_matches_reference_golden(oracle):
    """detect(pruning=True) restatement vs the reference itself, both part
    modes: detections, prune-rank maps and every counter identical; the
    calibration restatement reproduces the reference's thresholds."""
    from conftest import golden_pruned

    g = load_golden("detect_pruned.npz")
    pruned_any = 0
    for k in range(int(g["n"])):
        dec, pyr, planted, tau = golden_pruned(g, k)
        from paper_1707_03268_b200.types import Hypothesis

        pos = [(pyr[int(p[0])], Hypothesis(level=int(p[0]), root=(int(p[1]), int(p[2])),
                                           parts=tuple((int(p[3 + 2 * i]), int(p[4 + 2 * i]))
                                                       for i in range(len(dec.parts)))))
               for p in planted]
        rt, pt = oracle.calibrate_thresholds(dec, pos)
        assert np.array_equal(rt, dec.root_thresholds)
        for a, p in zip(pt, dec.parts):
            assert np.array_equal(a, p.thresholds)
        for mode in ("kill", "lenient"):
            m = f"q{k}_{mode}"
            dets, st, maps = oracle.detect_pruned(dec, pyr, tau, part_prune_mode=mode)
            ref = g[f"{m}_dets"]
            assert len(dets) == ref.shape[0], (k, mode)
            for d, r in zip(dets, ref):
                assert (d[0], *d[1]) == tuple(int(v) for v in r[:3])
                assert [c for pp in d[2] for c in pp] == [int(v) for v in r[3:-1]]
                assert d[3] == r[-1]
            assert [st["positions_examined"], st["positions_killed_by_parts"],
                    st["multiplications"]] == list(g[f"{m}_stats"])
            R = g[f"{m}_root_pruned"].size
            assert [st["positions_pruned_at_rank"].get(r, 0) for r in range(1, R + 1)] == \
                list(g[f"{m}_root_pruned"])
            assert [st["part_pruned_at_rank"].get(r, 0) for r in range(1, R + 1)] == \
                list(g[f"{m}_part_pruned"])
            for li, lm in enumerate(maps):
                if lm["rect"] is None:
                    continue
                assert np.array_equal(lm["root_prune_rank"], g[f"{m}_rootrank{li}"])
                assert np.array_equal(lm["part_prune_rank"], g[f"{m}_partrank{li}"])
            pruned_any += sum(st["positions_pruned_at_rank"].values())
    assert pruned_any > 0  # the fixtures exercise pruning
