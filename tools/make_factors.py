"""Shared-basis factors for configs 1-5, computed by the REFERENCE's cp_als.

The filter-tensor decomposition is a host-side one-off that stays in the
reference: the stacked tensor
``T = concat_f reshape(f, (h_f w_f, 32))`` of shape (P, 1, 32) is handed
unchanged to ``cpdetect.decomposition.cp_als`` with default ``AlsOptions``.
The basis is ``C = factors_c`` (32 x R); the per-cell cores are
``G = factors_a * (weights * factors_b[0])`` (P x R), both rounded to
float32 so the GPU path and the oracle consume identical numbers.

Run here (needs /root/reference):  python tools/make_factors.py [cfg:R ...]
Output: paper_1707_03268_b200/data/factors_cfg{cfg}_R{R}.npz
"""

import hashlib
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from cpdetect.decomposition import cp_als  # noqa: E402

from paper_1707_03268_b200 import synth  # noqa: E402

DEFAULT = ["1:8", "2:4", "2:8", "2:16", "2:32", "4:8", "5:8", "5:32", "3:16"]


def stacked_digest(T):
    return hashlib.sha256(np.ascontiguousarray(T, dtype=np.float64).tobytes()).hexdigest()


def main(specs):
    for spec in specs:
        cfg, R = (int(v) for v in spec.split(":"))
        wl = synth.workload(cfg)
        T = wl.bank.stacked()
        t0 = time.time()
        cp, res = cp_als(T, R)
        dt = time.time() - t0
        C = cp.factors_c.astype(np.float32)
        G = (cp.factors_a * (cp.weights * cp.factors_b[0])[None, :]).astype(np.float32)
        path = os.path.join(REPO, "paper_1707_03268_b200", "data", f"factors_cfg{cfg}_R{R}.npz")
        np.savez_compressed(path, C=C, G=G, residual=np.float64(res),
                            norm=np.float64(np.linalg.norm(T)), digest=np.array(stacked_digest(T)))
        print(f"cfg {cfg} R {R}: P={T.shape[0]} residual {res:.4f} / {np.linalg.norm(T):.4f} "
              f"({dt:.1f} s) -> {path}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or DEFAULT)
