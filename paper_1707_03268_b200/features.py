"""32-channel HOG feature pyramids on the B200.

The reference ships a 9-bin demo extractor only (cpdetect/features.py:16-68:
central-difference gradients, per-cell orientation histograms, energy
normalisation over a cell neighbourhood) and says its synthetic pipelines
work in feature space directly.  This module generalises that extractor to
the DPM v5 feature layout the score path consumes -- 18 contrast-sensitive
+ 9 contrast-insensitive orientation channels, 4 texture (normaliser)
channels and the truncation channel, 32 in all -- on the pyramid geometry of
``geometry.build_pyramid``, computed on the device straight into the X
arena that K1 reads (``csrc/hog.cu``; the algorithm is stated in
``oracle/hog_oracle.py``, its test-side restatement).

    levels = extract_hog_pyramid(image, pyramid)            # one image, numpy out
    HogBuilder(plan, (H, W), C).run(images_on_device)       # batch, into plan.X

There is no CPU fallback: without the library or a CUDA device this raises
``DeviceError`` like the rest of the package.
"""

import math

import numpy as np

from . import _lib
from .device import require_cuda, stream_handle, upload_table
from .errors import ValidationError

__all__ = ["HogBuilder", "extract_hog_pyramid", "level_image_size"]

SBIN = 4  # pixels per cell side of every level (root levels = 8-px cells of the 2x image)


def level_image_size(H, W, k, interval=10):
    """Resampled image size of pyramid level k: floor(H 2^-k/interval) x
    floor(W 2^-k/interval), whose 4-px cells are build_pyramid's level k."""
    f = 2.0 ** (-k / interval)
    return int(math.floor(H * f)), int(math.floor(W * f))


class HogBuilder:
    """Device HOG pyramid of ``n_images`` images of size (H, W, C) into the
    X arena of a plan (levels in the plan's geometry: 4-px cells, 10 levels
    per octave, ``geometry.build_pyramid``)."""

    def __init__(self, plan, image_hw, channels=3, interval=10):
        import torch

        require_cuda()
        self.plan, self.torch = plan, torch
        H, W = (int(v) for v in image_hw)
        C = int(channels)
        if not 1 <= C <= 4:
            raise ValidationError(f"images must have 1..4 channels, got {C}")
        if plan.L != 32:
            raise ValidationError(f"HOG features have 32 channels, the plan expects {plan.L}")
        self.H, self.W, self.C = H, W, C
        n = plan.n_images
        rs, hg, wave, lvl_off = [], [], [], {}
        r_off = h_off = 0
        for img in range(n):
            for k, (hc, wc) in enumerate(plan.levels):
                Hs, Ws = level_image_size(H, W, k, interval)
                if (Hs // SBIN, Ws // SBIN) != (hc, wc):
                    raise ValidationError(
                        f"pyramid level {k}: {hc}x{wc} cells, but a {H}x{W} image gives "
                        f"{Hs // SBIN}x{Ws // SBIN} at 2^-{k}/{interval}")
                # octave-recursive: levels 0..interval-1 from the image, level
                # k from level k - interval (wave k // interval)
                if k < interval:
                    rs.append((img * H * W * C, r_off, H, W, C, Hs, Ws, 0))
                else:
                    src, sh, sw = lvl_off[(img, k - interval)]
                    rs.append((src, r_off, sh, sw, C, Hs, Ws, 0))
                lvl_off[(img, k)] = (r_off, Hs, Ws)
                wave.append(k // interval)
                hg.append((r_off, img * plan.x_image_stride + plan.x_level_off[k], h_off, Hs, Ws,
                           C, 0))
                r_off += Hs * Ws * C
                h_off += hc * wc * 20
        self._rs = np.array(rs, dtype=_lib.RESAMPLE_JOB)
        self._hg = np.array(hg, dtype=_lib.HOG_JOB)
        self._wave = np.array(wave, dtype=np.int64)
        self._img_of = np.repeat(np.arange(n), len(plan.levels))
        self._tables = {}
        self.R = torch.empty(max(r_off, 1), dtype=torch.float32, device=plan.device)
        self.hist = torch.empty(max(h_off, 1), dtype=torch.float32, device=plan.device)

    def _table(self, images):
        """Job tables of an image range (cached): ([(resample wave table, n,
        blocks)], hog table, n, blocks)."""
        key = (images.start, images.stop)
        if key not in self._tables:
            lib = _lib.lib()
            dev = self.plan.device
            sel = (self._img_of >= images.start) & (self._img_of < images.stop)
            waves = []
            for w in range(int(self._wave.max()) + 1 if len(self._wave) else 0):
                rs = np.ascontiguousarray(self._rs[sel & (self._wave == w)])
                rb = _lib.check(lib.dpm_resample_prepare(_lib.table_ptr(rs), len(rs)), "resample")
                waves.append((upload_table(rs, dev), len(rs), rb))
            hg = np.ascontiguousarray(self._hg[sel])
            hb = _lib.check(lib.dpm_hog_prepare(_lib.table_ptr(hg), len(hg)), "hog")
            self._tables[key] = (waves, upload_table(hg, dev), len(hg), hb)
        return self._tables[key]

    def image_bytes(self, dtype="uint8"):
        return self.plan.n_images * self.H * self.W * self.C * (1 if dtype == "uint8" else 4)

    def run(self, images, stream=None, chunk=None):
        """images: device tensor (n_images, H, W, C), uint8 or float32 in
        [0, 255], contiguous.  Writes every level of every image (or of the
        image range ``chunk``) into the plan's X arena."""
        t = self.torch
        if tuple(images.shape) != (self.plan.n_images, self.H, self.W, self.C):
            raise ValidationError(f"images must be {(self.plan.n_images, self.H, self.W, self.C)}, "
                                  f"got {tuple(images.shape)}")
        if images.dtype not in (t.uint8, t.float32) or not images.is_contiguous() or \
                images.device != self.plan.X.device:
            raise ValidationError("images must be a contiguous uint8 / float32 tensor on the "
                                  "plan's device")
        lib = _lib.lib()
        s = stream_handle(stream)
        waves, hg_d, nhg, hb = self._table(chunk or range(self.plan.n_images))
        for w, (rs_d, nrs, rb) in enumerate(waves):  # wave 0 reads the images, wave w > 0 wave w-1
            src, u8 = (images, int(images.dtype == t.uint8)) if w == 0 else (self.R, 0)
            _lib.check(lib.dpm_resample(src.data_ptr(), u8, self.R.data_ptr(), rs_d.data_ptr(),
                                        nrs, rb, s), "resample")
        _lib.check(lib.dpm_hog(self.R.data_ptr(), self.hist.data_ptr(), self.plan.X.data_ptr(),
                               hg_d.data_ptr(), nhg, hb, s), "hog")
        return self


def extract_hog_pyramid(image, pyramid, interval=10):
    """The HOG levels (numpy float32, (H_k, W_k, 32)) of one image (H, W[, C])
    in [0, 255] for ``pyramid`` (a ``geometry.Pyramid``), computed on the
    device."""
    import torch

    from .engine import FilterDef, Plan

    img = np.asarray(image)
    if img.ndim == 2:
        img = img[:, :, None]
    if img.ndim != 3:
        raise ValidationError(f"image must be (H, W) or (H, W, C), got {img.shape}")
    dt = np.uint8 if img.dtype == np.uint8 else np.float32
    plan = Plan(32, pyramid.levels, np.eye(32, 1, dtype=np.float32),
                [FilterDef(np.zeros((1, 1, 1), np.float32))], outputs=())
    hb = HogBuilder(plan, img.shape[:2], img.shape[2], interval)
    dev_img = torch.from_numpy(np.ascontiguousarray(img.astype(dt))[None]).to(plan.device)
    hb.run(dev_img)
    return [plan.x_view(0, k).cpu().numpy().copy() for k in range(len(pyramid.levels))]
