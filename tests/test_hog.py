"""HOG pyramid builder: the oracle's known answers on
CPU; the device builder against the oracle (-m gpu)."""

import numpy as np
import pytest

from oracle import hog_oracle as H
from paper_1707_03268_b200 import synth
from paper_1707_03268_b200.features import level_image_size
from paper_1707_03268_b200.geometry import build_pyramid


def scene(h, w, seed, channels=3):
    """Seeded test image in [0, 255]: smooth gradients, discs and bars (every
    orientation occurs), uint8."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    img = np.zeros((h, w, channels))
    for c in range(channels):
        img[:, :, c] = 60 + 40 * np.sin(xx / (7 + 3 * c)) * np.cos(yy / 11)
    for _ in range(12):
        cy, cx, r = rng.uniform(0, h), rng.uniform(0, w), rng.uniform(3, h / 4)
        col = rng.uniform(0, 255, channels)
        img[(yy - cy) ** 2 + (xx - cx) ** 2 < r * r] = col
    for _ in range(6):
        ang = rng.uniform(0, np.pi)
        d = (xx - rng.uniform(0, w)) * np.cos(ang) + (yy - rng.uniform(0, h)) * np.sin(ang)
        img[np.abs(d) < rng.uniform(1, 4)] = rng.uniform(0, 255, channels)
    img += rng.normal(0, 2, img.shape)
    return np.clip(img, 0, 255).astype(np.uint8)


def test_level_sizes_are_the_pyramid_geometry():
    """Level k's resampled image cut into 4-px cells gives exactly
    build_pyramid's level k, for every config image size."""
    for cfg in (2, 3, 4, 5):
        wl = synth.workload(cfg)
        hh, ww = wl.image_hw
        for k, (hc, wc) in enumerate(wl.pyramid.levels):
            Hs, Ws = level_image_size(hh, ww, k)
            assert (Hs // 4, Ws // 4) == (hc, wc), (cfg, k)
            assert (Hs, Ws) == H.level_size(hh, ww, k)


def test_resample_identity_and_mean_preserving():
    img = scene(40, 56, 1).astype(np.float32)
    assert np.array_equal(H.resample_area(img, 40, 56), img)
    r = H.resample_area(img, 17, 23)
    assert r.shape == (17, 23, 3)
    # box filtering preserves the mean up to the cropped remainder
    assert abs(r.mean() - img.mean()) < 2.0
    const = np.full((33, 47, 1), 77.0, np.float32)
    assert np.allclose(H.resample_area(const, 10, 14), 77.0, rtol=1e-5)  # FP32 weights


def test_hog_known_answers():
    # flat image: no gradient, every feature 0
    assert not H.hog32(np.full((24, 24, 3), 100.0, np.float32)).any()
    # vertical edge: horizontal gradient -> orientation 0 (dx > 0) dominates
    img = np.zeros((32, 32, 1), np.float32)
    img[:, 16:] = 255.0
    f = H.hog32(img)
    assert f.shape == (8, 8, 32) and not f[:, :, 31].any()
    edge = f[:, 3:5]
    assert edge[:, :, 0].min() > 0 and np.allclose(edge[:, :, 1:18], 0)
    assert np.allclose(edge[:, :, 18], edge[:, :, 0])  # insensitive bin 0 = sensitive 0 + 9
    # mirrored edge: dx < 0 -> orientation 9
    f2 = H.hog32(img[:, ::-1].copy())
    assert f2[:, 3:5, 9].min() > 0 and np.allclose(f2[:, 3:5, 0], 0)
    # features are truncated sums: 0 <= f <= 0.4 (0.5 x 4 x 0.2) on the 27 orientation channels
    g = H.hog32(scene(64, 64, 3).astype(np.float32))
    assert g[:, :, :27].min() >= 0 and g[:, :, :27].max() <= 0.4 + 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("channels,dtype", [(3, np.uint8), (1, np.float32)])
def test_device_hog_pyramid_matches_oracle(channels, dtype):
    """Every level of a 160 x 224 image's pyramid: the device features
    against the oracle at 1e-5 (orientation bins are bit-identical, the
    sums FP32 against float64)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1707_03268_b200.features import extract_hog_pyramid

    img = scene(160, 224, 5, channels)
    if dtype is np.float32:
        img = img.astype(np.float32) + 0.25
    pyr = build_pyramid(160, 224, [(6, 11)])
    got = extract_hog_pyramid(img, pyr)
    ref = H.hog_pyramid(img, len(pyr.levels))
    for k, (g, r) in enumerate(zip(got, ref)):
        assert g.shape == r.shape, k
        err = np.abs(g - r).max()
        assert err <= 1e-5, (k, err)


@pytest.mark.gpu
def test_score_images_equals_score_batch_on_the_device_pyramid():
    """The image-input public call (HOG built on the device, only uint8
    images cross PCIe) returns exactly the detections of score_batch fed the
    same device-built pyramids through host memory."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os

    from conftest import REPO
    from paper_1707_03268_b200.features import extract_hog_pyramid
    from paper_1707_03268_b200.pipeline import PyramidScorer

    wl = synth.workload(2)
    fx = np.load(os.path.join(REPO, "paper_1707_03268_b200", "data", "factors_cfg2_R8.npz"))
    hh, ww = wl.image_hw
    imgs = np.stack([scene(hh, ww, 10 + i) for i in range(3)])
    sc = PyramidScorer(wl.bank, fx["C"], fx["G"], wl.pyramid, n_images=3, max_dets=1 << 18)
    host_imgs = torch.from_numpy(imgs).pin_memory()
    d_img = sc.score_images(host_imgs, tau=1.9, chunk_images=2)
    host = sc.host_arena(pinned=True)
    for i in range(3):
        sc.fill_host(host, i, extract_hog_pyramid(imgs[i], wl.pyramid))
    d_hog = sc.score_batch(host, tau=1.9, chunk_images=2)
    assert len(d_img) == len(d_hog) > 0
    key = ["image", "level", "component", "ry", "rx"]
    a, b = np.sort(d_img, order=key), np.sort(d_hog, order=key)
    assert a.tobytes() == b.tobytes()
