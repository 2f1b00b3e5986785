"""How often would a two-phase K3 window scan need its outer candidates?

    python tools/k3_split_sim.py [part level]   (default 0: 180 x 320, config 4 image 0)

For the part maps of one config-4 component (float64 maps of the real
filters and factors, computed here with numpy) and the kernel's radius r* + 1, counts the fraction of
warps (32 centres two columns apart in the x pass; 32 root columns of one
root row in the y pass) for which the inner window |d| <= r1 does NOT prove
that every outer candidate loses: max over the band row (x) or column (y)
minus the smallest outer penalty a*(r1+1)^2 still reaches the warp's smallest
inner maximum.  Measured at level 0: r1 = 5 -> 4.7% (x) / 1.2% (y) of warps,
r1 = 6 -> 0%.  DESIGN.md section 3 records what the kernel variant built on
it measured (slower; dropped).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1707_03268_b200 import synth  # noqa: E402


def correlate(P, core):
    """Valid correlation of a projected level (H, W, R) with a core (h, w, R), float64."""
    h, w, _ = core.shape
    H, W, _ = P.shape
    out = np.zeros((H - h + 1, W - w + 1))
    for i in range(h):
        for j in range(w):
            out += P[i:i + H - h + 1, j:j + W - w + 1] @ core[i, j]
    return out


def r_star(S, a):
    """SURVEY.md App. A.2 radius for a pure quadratic penalty a*d^2 on both axes."""
    return int(np.floor(np.sqrt(4 * a * float(S.max() - S.min())) / (2 * a)))


def main():
    lev = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    wl = synth.workload(4)
    bank = wl.bank
    here = os.path.dirname(os.path.abspath(__file__))
    fx = np.load(os.path.join(here, "..", "paper_1707_03268_b200", "data", "factors_cfg4_R8.npz"))
    G, offs = fx["G"], bank.offsets()

    def core(f):
        h, w, _ = bank.filters[f].shape
        return G[offs[f]:offs[f] + h * w].reshape(h, w, -1)

    H, W = wl.pyramid.levels[lev]
    X = synth.hog_level(4, 0, lev, H, W).astype(np.float64)
    P = X @ fx["C"].astype(np.float64)
    a = 0.01
    xs, ys = {}, {}
    for f in bank.components[0].parts[:3]:
        S = correlate(P, core(f).astype(np.float64))
        R = r_star(S, a) + 1
        Hs, Ws = S.shape
        pad = np.full((Hs, Ws + 2 * R), -np.inf)
        pad[:, R:R + Ws] = S
        d = np.arange(-R, R + 1)
        cand = np.stack([pad[:, k:k + Ws] for k in range(2 * R + 1)], -1) - a * d * d
        xbest = cand.max(-1)
        for r1 in range(3, R + 1):
            inner = cand[..., R - r1:R + r1 + 1].max(-1)
            n = t = 0
            for x0 in range(0, Ws - 63, 64):
                rmax = S[:, max(0, x0 - R):min(Ws, x0 + 62 + R + 1)].max(1)
                n += np.sum(inner[:, x0:x0 + 63:2].min(1) <= rmax - a * (r1 + 1) ** 2)
                t += Hs
            xs.setdefault(r1, [0, 0])
            xs[r1][0] += n
            xs[r1][1] += t
        padx = np.full((Hs + 2 * R, Ws), -np.inf)
        padx[R:R + Hs] = xbest
        candy = np.stack([padx[k:k + Hs] for k in range(2 * R + 1)], -1) - a * d * d
        for r1 in range(3, R + 1):
            inner = candy[..., R - r1:R + r1 + 1].max(-1)
            n = t = 0
            for y0 in range(0, Hs - 127, 128):
                cmax = xbest[max(0, y0 - R):y0 + 127 + R + 1].max(0)
                for yy in range(y0, y0 + 128, 2):
                    for x0 in range(0, Ws - 63, 64):
                        cols = np.arange(x0, x0 + 63, 2)
                        n += np.any(inner[yy, cols] <= cmax[cols] - a * (r1 + 1) ** 2)
                        t += 1
            ys.setdefault(r1, [0, 0])
            ys[r1][0] += n
            ys[r1][1] += t
    print(f"part level {lev} ({H}x{W}), radius {R}")
    for r1 in sorted(xs):
        print(f"r1={r1:2d}  x warps needing outer {xs[r1][0] / max(1, xs[r1][1]):.4f}  "
              f"y warps needing outer {ys[r1][0] / max(1, ys[r1][1]):.4f}")


if __name__ == "__main__":
    main()
