"""MMA-warp wait breakdown of the tcgen05 correlation kernel (config 4).

    make -B EXTRA=-DDPM_TC_PROBE && python tools/tc_probe.py [images]

Needs the library built with -DDPM_TC_PROBE (clock64 around the MMA warp's
waits).  Prints, summed over CTAs, the share of the MMA loop spent waiting
for a free accumulator (epilogue behind), for staged input rows (producers
behind), and issuing.  Rebuild without the flag afterwards.
"""
import ctypes
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_1707_03268_b200 import _lib, synth  # noqa: E402
from paper_1707_03268_b200.pipeline import PyramidScorer  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    wl = synth.workload(4)
    fx = np.load(os.path.join(REPO, "paper_1707_03268_b200", "data", "factors_cfg4_R8.npz"))
    sc = PyramidScorer(wl.bank, fx["C"], fx["G"], wl.pyramid, n_images=n,
                       outputs=("totals", "positions"))
    for j in range(n):
        sc.load_image(j, synth.hog_pyramid(4, j, wl.pyramid))
    lib = _lib.lib()
    lib.dpm_tc_probe_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
    out = (ctypes.c_ulonglong * 4)()
    for it in range(3):
        lib.dpm_tc_probe_read(out)  # reset
        sc.run()
        torch.cuda.synchronize()
        lib.dpm_tc_probe_read(out)
        e, f, rows, tot = list(out)
        print(f"run {it}: rows {rows}, loop cycles {tot}: waiting for the accumulator "
              f"{e / tot:.1%}, for input rows {f / tot:.1%}, issue/other {1 - (e + f) / tot:.1%}; "
              f"per row {tot / max(rows, 1):.0f} cycles")


if __name__ == "__main__":
    main()
