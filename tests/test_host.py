"""Host logic without a GPU: geometry, generators, validation errors with the
reference's messages, fail-loud behaviour when CUDA is absent."""

import numpy as np
import pytest

import paper_1707_03268_b200 as B
from oracle import dpm_oracle as O
from paper_1707_03268_b200 import geometry, synth


def test_pyramid_geometry_matches_survey_counts():
    # evals and distinct cells per image
    expect = {2: (29, 39, 145715, 6221610), 4: (39, 49, 441041, 20013786)}
    for cfg, (nroot, nlev, cells, evals) in expect.items():
        wl = synth.workload(cfg)
        p = wl.pyramid
        assert (len(p.root_levels), len(p.levels), p.n_cells) == (nroot, nlev, cells)
        ev = 0
        for kr, kp in zip(p.root_levels, p.part_levels):
            for comp in wl.bank.components:
                for f, k in [(comp.root, kr)] + [(q, kp) for q in comp.parts]:
                    h, w = wl.bank.filters[f].shape[:2]
                    H, W = p.levels[k]
                    ev += max(0, H - h + 1) * max(0, W - w + 1)
        assert ev == evals


def test_mirrored_components_are_x_flips():
    wl = synth.workload(2)
    bank = wl.bank
    a, b = bank.components[0], bank.components[1]
    assert np.array_equal(bank.filters[b.root], bank.filters[a.root][:, ::-1, :])
    for pa, pb, (ya, xa), (yb, xb) in zip(a.parts, b.parts, a.anchors, b.anchors):
        assert np.array_equal(bank.filters[pb], bank.filters[pa][:, ::-1, :])
        assert ya == yb and xb == 2 * 11 - 6 - xa


def test_hog_levels_seeded_and_truncation_channel_zero():
    a = synth.hog_level(4, 3, 7, 20, 30)
    b = synth.hog_level(4, 3, 7, 20, 30)
    assert a.dtype == np.float32 and np.array_equal(a, b)
    assert np.all(a[:, :, 31] == 0) and a[:, :, :31].min() >= 0 and a.max() < 0.4


def test_hypothesis_rect_matches_oracle():
    rng = np.random.default_rng(0)
    for _ in range(200):
        H, W = rng.integers(5, 40, size=2)
        rd = (int(rng.integers(1, 8)), int(rng.integers(1, 8)))
        n = int(rng.integers(0, 4))
        parts = []
        for _ in range(n):
            p = B.PartSpec(np.zeros((int(rng.integers(1, 6)), int(rng.integers(1, 6)), 1)),
                           (int(rng.integers(-6, 6)), int(rng.integers(-6, 6))),
                           (0, 0, 0, 0), int(rng.integers(1, 4)))
            parts.append(p)
        got = geometry.hypothesis_rect((int(H), int(W), 1), rd, parts)
        ref = O.hypothesis_rect((int(H), int(W)), rd, [p.filter.shape for p in parts],
                                [p.anchor for p in parts], [p.search_radius for p in parts])
        assert got == ref


def test_gdt_root_rect_keeps_centres_inside():
    rng = np.random.default_rng(1)
    for _ in range(300):
        rs = (int(rng.integers(1, 30)), int(rng.integers(1, 30)))
        ps = [(int(rng.integers(1, 60)), int(rng.integers(1, 60))) for _ in range(3)]
        an = [(int(rng.integers(-5, 12)), int(rng.integers(-5, 12))) for _ in range(3)]
        s = int(rng.integers(1, 3))
        rect = geometry.gdt_root_rect(rs, ps, an, s)
        ok = [(y, x) for y in range(rs[0]) for x in range(rs[1])
              if all(0 <= s * y + a[0] < p[0] and 0 <= s * x + a[1] < p[1]
                     for p, a in zip(ps, an))]
        if rect is None:
            assert not ok
        else:
            ry0, ry1, rx0, rx1 = rect
            assert sorted(ok) == [(y, x) for y in range(ry0, ry1 + 1) for x in range(rx0, rx1 + 1)]


def test_validation_errors_mirror_reference_before_any_device_work():
    img = np.zeros((5, 5, 3))
    cp = B.CPModel(np.ones(2), np.eye(2), np.eye(2), np.eye(3)[:, :2])
    with pytest.raises(B.ValidationError, match="upto_rank"):
        B.correlate3_cp(img, cp, upto_rank=3)
    with pytest.raises(B.ValidationError, match="channel mismatch"):
        B.correlate3_full(np.zeros((4, 4, 3)), np.zeros((2, 2, 2)))
    with pytest.raises(B.ValidationError, match="exceeds image extent"):
        B.correlate3_full(np.zeros((2, 4, 3)), np.zeros((3, 2, 3)))
    with pytest.raises(B.ValidationError, match="non-finite"):
        B.correlate3_full(np.full((4, 4, 1), np.nan), np.zeros((2, 2, 1)))
    with pytest.raises(B.ValidationError, match="part_prune_mode"):
        B.detect(None, [], 0.0, part_prune_mode="bogus")
    dec = B.DecomposedModel(cp, ())
    with pytest.raises(B.ValidationError, match="calibrated"):
        B.detect(dec, [], 0.0, pruning=True)
    with pytest.raises(B.ValidationError, match="pyramid level 0"):
        B.detect(dec, [np.zeros((5, 5, 4))], 0.0)
    with pytest.raises(B.ValidationError, match="zero positives"):
        B.calibrate_thresholds(dec, [])
    bad = B.PartModel(np.zeros((2, 2, 3)), (B.PartSpec(np.zeros((2, 2, 3)), (0, 0),
                                                        (0, 0, -1.0, 0), 0),))
    with pytest.raises(B.ValidationError, match="c_dxx"):
        B.dense_detect(bad, [], 0.0)
    assert issubclass(B.ValidationError, ValueError)


def test_product_path_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(B.DeviceError, match="no CPU fallback"):
        B.correlate3_full(np.zeros((4, 4, 2)), np.zeros((2, 2, 2)))


def test_cp_core_is_weighted_outer_product():
    from paper_1707_03268_b200.correlation import cp_core

    rng = np.random.default_rng(2)
    cp = B.CPModel.from_factors(rng.normal(size=(3, 4)), rng.normal(size=(5, 4)),
                                rng.normal(size=(6, 4)))
    core = cp_core(cp).astype(np.float64)
    recon = np.einsum("ijr,lr->ijl", core, cp.factors_c)
    full = np.einsum("r,ir,jr,lr->ijl", cp.weights, cp.factors_a, cp.factors_b, cp.factors_c)
    np.testing.assert_allclose(recon, full, rtol=1e-5, atol=1e-6)
    assert np.all(cp_core(cp, keep=2)[:, :, 2:] == 0)


def test_factor_fixtures_match_generators():
    """The committed cp_als factors were computed on exactly these banks."""
    import hashlib
    import os

    from conftest import REPO
    for cfg, R in [(1, 8), (2, 8), (4, 8), (5, 32)]:
        fx = np.load(os.path.join(REPO, "paper_1707_03268_b200", "data",
                                  f"factors_cfg{cfg}_R{R}.npz"))
        T = synth.workload(cfg).bank.stacked()
        assert hashlib.sha256(np.ascontiguousarray(T).tobytes()).hexdigest() == str(fx["digest"])
        assert fx["G"].shape == (T.shape[0], R) and fx["C"].shape == (32, R)


def test_segment_strips_cover_every_output_row_once():
    """Small pyramids split their tcgen05 part strips into row segments
    (engine._segment_strips); every output row of every strip is covered by
    exactly one segment, and a batch with enough strips stays whole."""
    from paper_1707_03268_b200.engine import _segment_strips
    rng = np.random.default_rng(5)
    strips = [(j, 0, int(sx), int(ho)) for j, (sx, ho) in
              enumerate(zip(rng.integers(0, 4, 40), rng.integers(1, 200, 40)))]
    segs = _segment_strips(strips, sms=148)
    assert len(strips) < len(segs) < 2 * 148  # below the CTA-pair threshold
    for j, _, sx, ho in strips:
        rows = sorted(r for sj, y0, ssx, n, h in segs if sj == j and ssx == sx
                      for r in range(y0, y0 + n))
        assert rows == list(range(ho))
        assert all(h == ho for sj, _, _, _, h in segs if sj == j)
    whole = _segment_strips(strips, sms=10)
    assert [(j, y0, sx, n) for j, y0, sx, n, _ in whole] == [(j, 0, sx, ho) for j, _, sx, ho in strips]
