"""CPU oracle of the 32-channel HOG pyramid builder -- TEST INFRASTRUCTURE ONLY.

Imported only by tests/ (never by the product package).
row 4 asks for a real 32-channel HOG pyramid feeding the score path; the
reference ships only a 9-bin demo extractor (cpdetect/features.py:16-68:
central-difference gradients, orientation binning per cell, neighbourhood
energy normalisation), which this generalises to the DPM v5 feature layout
(Felzenszwalb et al., PAMI 2010, section 6) on the pyramid geometry of
geometry.build_pyramid.  The algorithm, restated here and in
csrc/hog.cu:

pyramid   level k of an H x W image: resampled to floor(H 2^-k/10) x
          floor(W 2^-k/10) pixels (area averaging; levels 0..9 from the
          image, level k >= 10 from level k-10's resampled image, one octave
          up), cut into 4 x 4-pixel cells -> floor(H 2^-k/10 / 4) x ...
          cells, the shape build_pyramid gives level k (root levels 8-px
          cells of the same image are levels k + 10);
resample  separable box filter: output pixel o of an axis covers the input
          interval [o s, (o+1) s), s = n_in / n_out; input pixel i weighs
          min(i+1, (o+1)s) - max(i, o s); rows first, then columns, then
          the sum divided by s_y s_x;
gradient  per pixel, per colour channel, central differences with clamped
          borders; the channel with the largest squared magnitude wins;
          v = its magnitude;
bins      18 contrast-sensitive orientations: o = argmax over 0..8 of
          |u_o . g| with u_o = (cos 20 o deg, sin 20 o deg), + 9 when the
          dot product is negative (strict '>' from 0, first wins);
cells     bilinear soft binning of v into the 4 cells around the pixel
          (centres at 4 c + 1.5); pixels past the last whole cell ignored;
norms     E(c) = sum over 9 orientations of (h_o + h_o+9)^2; each cell has
          four normalisers 1/sqrt(sum of E over a 2x2 cell block + 1e-4),
          the blocks to its lower-right, upper-right, lower-left,
          upper-left (cells past the border clamped to the edge);
features  0..17 : 0.5 * sum_k min(h_o n_k, 0.2)        (contrast sensitive)
          18..26: 0.5 * sum_k min((h_o + h_o+9) n_k, 0.2)  (insensitive)
          27..30: 0.2357 * sum_o min(h_o n_k, 0.2), k = 1..4  (texture)
          31    : 0                                      (truncation)

The discrete steps (resampling, gradient, the orientation argmax) are
emulated in float32 with the device's operation order, so bins are
identical; histograms, norms and features are float64 here (FP32 on the
device, compared at 1e-5).
"""

import math

import numpy as np

__all__ = ["resample_area", "gradient_bins", "hog32", "hog_pyramid", "level_size"]

F32 = np.float32
SBIN = 4
EPS = 1e-4
UU = np.array([math.cos(o * math.pi / 9) for o in range(9)], dtype=np.float32)
VV = np.array([math.sin(o * math.pi / 9) for o in range(9)], dtype=np.float32)


def level_size(H, W, k, interval=10):
    """Resampled image size of pyramid level k (float64 on the host)."""
    f = 2.0 ** (-k / interval)
    return int(math.floor(H * f)), int(math.floor(W * f))


def _taps(n_in, n_out):
    """(index, float32 weight) lists of every output position, float32 ops."""
    s = F32(F32(n_in) / F32(n_out))
    out = []
    for o in range(n_out):
        a = F32(F32(o) * s)
        b = F32(F32(o + 1) * s)
        i0, i1 = int(math.floor(a)), min(int(math.ceil(b)), n_in)
        taps = []
        for i in range(i0, i1):
            w = F32(min(F32(i + 1), b) - max(F32(i), a))
            taps.append((i, w))
        out.append(taps)
    return s, out


def resample_area(img, Hs, Ws):
    """Box-filter resampling of img (H, W, C) float32 to (Hs, Ws, C), float32
    with the device's order: per output pixel, sum over row taps of
    (row weight * sum over column taps of (column weight * pixel)), divided
    by s_y * s_x."""
    img = np.asarray(img, dtype=np.float32)
    H, W, C = img.shape
    sy, ty = _taps(H, Hs)
    sx, tx = _taps(W, Ws)
    nx = max(len(t) for t in tx)
    idx = np.zeros((Ws, nx), np.int64)
    wx = np.zeros((Ws, nx), np.float32)
    for o, taps in enumerate(tx):
        for t, (i, w) in enumerate(taps):
            idx[o, t], wx[o, t] = i, w
    # horizontal sums of every input row, in tap order (zero-weight padding
    # taps add exact zeros)
    hrow = np.zeros((H, Ws, C), np.float32)
    for t in range(nx):
        hrow = (hrow + wx[None, :, t, None] * img[:, idx[:, t], :]).astype(np.float32)
    out = np.zeros((Hs, Ws, C), np.float32)
    for o, taps in enumerate(ty):
        acc = np.zeros((Ws, C), np.float32)
        for i, w in taps:
            acc = (acc + F32(w) * hrow[i]).astype(np.float32)
        out[o] = acc
    d = F32(sy * sx)
    return (out / d).astype(np.float32)


def gradient_bins(R):
    """Per-pixel (v float32, orientation bin 0..17) of a resampled image."""
    R = np.asarray(R, dtype=np.float32)
    Hs, Ws, C = R.shape
    xr = np.minimum(np.arange(Ws) + 1, Ws - 1)
    xl = np.maximum(np.arange(Ws) - 1, 0)
    yd = np.minimum(np.arange(Hs) + 1, Hs - 1)
    yu = np.maximum(np.arange(Hs) - 1, 0)
    dx = (R[:, xr, :] - R[:, xl, :]).astype(np.float32)
    dy = (R[yd, :, :] - R[yu, :, :]).astype(np.float32)
    m = (dx * dx + dy * dy).astype(np.float32)
    best = m[:, :, 0].copy()
    bdx, bdy = dx[:, :, 0].copy(), dy[:, :, 0].copy()
    for c in range(1, C):
        better = m[:, :, c] > best
        best = np.where(better, m[:, :, c], best)
        bdx = np.where(better, dx[:, :, c], bdx)
        bdy = np.where(better, dy[:, :, c], bdy)
    v = np.sqrt(best).astype(np.float32)
    bdot = np.zeros_like(v)
    bo = np.zeros(v.shape, np.int64)
    for o in range(9):
        dot = (UU[o] * bdx + VV[o] * bdy).astype(np.float32)
        pos = dot > bdot
        bdot = np.where(pos, dot, bdot)
        bo = np.where(pos, o, bo)
        neg = ~pos & (-dot > bdot)
        bdot = np.where(neg, -dot, bdot)
        bo = np.where(neg, o + 9, bo)
    return v, bo


def hog32(R):
    """32-channel features (Hc, Wc, 32) float64 of a resampled image."""
    v, bo = gradient_bins(R)
    Hs, Ws = v.shape
    Hc, Wc = Hs // SBIN, Ws // SBIN
    hist = np.zeros((Hc + 2, Wc + 2, 18))  # one cell of padding on every side
    ys = np.arange(Hc * SBIN)
    xs = np.arange(Wc * SBIN)
    yp = (ys + 0.5) / SBIN - 0.5
    xp = (xs + 0.5) / SBIN - 0.5
    iy = np.floor(yp).astype(np.int64)
    ix = np.floor(xp).astype(np.int64)
    vy0, vx0 = yp - iy, xp - ix
    vy1, vx1 = 1.0 - vy0, 1.0 - vx0
    vv = v[:Hc * SBIN, :Wc * SBIN].astype(np.float64)
    oo = bo[:Hc * SBIN, :Wc * SBIN]
    Y = np.broadcast_to(iy[:, None], vv.shape)
    X = np.broadcast_to(ix[None, :], vv.shape)
    for dyc, wy in ((0, vy1), (1, vy0)):
        for dxc, wx in ((0, vx1), (1, vx0)):
            np.add.at(hist, (Y + dyc + 1, X + dxc + 1, oo), wy[:, None] * wx[None, :] * vv)
    hist = hist[1:Hc + 1, 1:Wc + 1]  # contributions to cells outside the grid dropped
    E = ((hist[:, :, :9] + hist[:, :, 9:]) ** 2).sum(axis=2)
    Ep = np.pad(E, 1, mode="edge")

    def blk(dy0, dx0):  # sum of E over the 2x2 block with top-left (cy+dy0, cx+dx0)
        s = 0.0
        for a in (0, 1):
            for b in (0, 1):
                s = s + Ep[1 + dy0 + a:1 + dy0 + a + Hc, 1 + dx0 + b:1 + dx0 + b + Wc]
        return 1.0 / np.sqrt(s + EPS)

    ns = [blk(0, 0), blk(-1, 0), blk(0, -1), blk(-1, -1)]
    feat = np.zeros((Hc, Wc, 32))
    tex = [np.zeros((Hc, Wc)) for _ in range(4)]
    for o in range(18):
        acc = 0.0
        for k in range(4):
            t = np.minimum(hist[:, :, o] * ns[k], 0.2)
            acc = acc + t
            tex[k] = tex[k] + t
        feat[:, :, o] = 0.5 * acc
    for o in range(9):
        h = hist[:, :, o] + hist[:, :, o + 9]
        feat[:, :, 18 + o] = 0.5 * sum(np.minimum(h * ns[k], 0.2) for k in range(4))
    for k in range(4):
        feat[:, :, 27 + k] = 0.2357 * tex[k]
    return feat


def hog_pyramid(img, n_levels, interval=10):
    """Levels 0..n_levels-1 of the pyramid of img (H, W[, C]) in [0, 255].
    Octave-recursive resampling: levels 0..interval-1 from the image, level
    k >= interval from level k - interval's resampled image."""
    img = np.asarray(img, dtype=np.float32)
    if img.ndim == 2:
        img = img[:, :, None]
    H, W, _ = img.shape
    res, out = [], []
    for k in range(n_levels):
        Hs, Ws = level_size(H, W, k, interval)
        src = img if k < interval else res[k - interval]
        res.append(resample_area(src, Hs, Ws))
        out.append(hog32(res[k]))
    return out
