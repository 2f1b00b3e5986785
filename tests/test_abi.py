"""C ABI: the library loads without a GPU and exports every declared symbol;
ABI struct layouts match the header; host-side prepare calls validate."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO

from paper_1707_03268_b200 import _lib


def _declared():
    text = open(os.path.join(REPO, "include", "dpm_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dpm_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    names = _declared()
    assert len(names) >= 11
    for n in names:
        assert hasattr(lib, n), n
    assert lib.dpm_abi_version() == _lib.ABI_VERSION == 4


def test_struct_sizes_match_header_comments():
    # sizes asserted at import against the C layout (int64 first, natural alignment)
    assert _lib.PROJ_JOB.itemsize == 32
    assert _lib.CORR_JOB.itemsize == 72
    assert _lib.PLACE_JOB.itemsize == 96
    assert _lib.ASM_JOB.itemsize == 88
    assert _lib.DETECTION.itemsize == 96


def test_struct_layout_against_compiled_offsets(tmp_path):
    """Compile a tiny C program against the header and compare offsetof()."""
    src = tmp_path / "off.c"
    fields = {
        "dpm_proj_job": ("x_off", "p_off", "H", "W", "pitch", "block0"),
        "dpm_corr_job": ("p_off", "s_off", "g_off", "H", "nf_pad", "range_idx"),
        "dpm_place_job": ("s_off", "x_off", "Hp", "rx0", "block0", "smap", "smap_z", "cdx", "cdyy"),
        "dpm_smap_desc": ("s_off", "Ho", "Wo", "nf", "pad"),
        "dpm_asm_job": ("root_off", "placed_off", "root_pitch", "block0", "bias"),
        "dpm_detection": ("image", "score", "parts"),
        "dpm_place_range": ("rx", "ry", "E2", "E2in"),
        "dpm_prune_job": ("out_off", "offs0", "thr0", "R", "Hp", "ry0", "rx1", "scale", "radius",
                          "block0"),
        "dpm_prune_asm": ("rank_off", "lim_off", "root_off", "root_pitch", "hist_off", "block0",
                          "bias", "part_R", "ay", "ax"),
        "dpm_cover_job": ("lim_off", "hr", "y0", "oy", "radius", "hist_off", "block0", "pad"),
    }
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "dpm_b200.h"', "int main(){"]
    for st, fs in fields.items():
        lines.append(f'printf("{st} %zu\\n", sizeof({st}));')
        for f in fs:
            lines.append(f'printf("{st}.{f} %zu\\n", offsetof({st}, {f}));')
    lines.append("return 0;}")
    src.write_text("\n".join(lines))
    exe = tmp_path / "off"
    rc = os.system(f"gcc -I{REPO}/include {src} -o {exe}")
    if rc != 0:
        pytest.skip("gcc unavailable")
    out = dict(line.rsplit(" ", 1) for line in os.popen(str(exe)).read().split("\n") if line)
    dts = {"dpm_proj_job": _lib.PROJ_JOB, "dpm_corr_job": _lib.CORR_JOB,
           "dpm_place_job": _lib.PLACE_JOB, "dpm_asm_job": _lib.ASM_JOB,
           "dpm_detection": _lib.DETECTION, "dpm_place_range": _lib.PLACE_RANGE,
           "dpm_prune_job": _lib.PRUNE_JOB, "dpm_smap_desc": _lib.SMAP_DESC,
           "dpm_prune_asm": _lib.PRUNE_ASM, "dpm_cover_job": _lib.COVER_JOB}
    for st, fs in fields.items():
        assert int(out[st]) == dts[st].itemsize, st
        for f in fs:
            assert int(out[f"{st}.{f}"]) == dts[st].fields[f][1], (st, f)


def test_prepare_validates_and_numbers_blocks():
    lib = _lib.lib()
    jobs = np.zeros(2, dtype=_lib.PROJ_JOB)
    jobs["H"], jobs["W"], jobs["pitch"] = (10, 20), (30, 7), (32, 8)
    n = lib.dpm_project_prepare(_lib.table_ptr(jobs), 2)
    assert n == 2 + 1 and list(jobs["block0"]) == [0, 2]
    jobs["pitch"][1] = 6  # not a multiple of 4
    with pytest.raises(Exception, match="pitch"):
        _lib.check(lib.dpm_project_prepare(_lib.table_ptr(jobs), 2))
    jobs["pitch"][1] = 8
    jobs["H"][0], jobs["W"][0], jobs["pitch"][0] = 70000, 70000, 70000  # plane past 2^31 floats
    with pytest.raises(Exception, match="too large"):
        _lib.check(lib.dpm_project_prepare(_lib.table_ptr(jobs), 2))
    pj = np.zeros(1, dtype=_lib.PLACE_JOB)
    pj["Hp"], pj["Wp"], pj["scale"], pj["radius"], pj["range_idx"], pj["wr"] = 5, 5, 1, -1, 0, 5
    with pytest.raises(Exception, match="c_dxx"):
        _lib.check(lib.dpm_place_prepare(_lib.table_ptr(pj), 1))
    pj["cdxx"], pj["cdyy"] = 0.01, 0.01
    assert lib.dpm_place_prepare(_lib.table_ptr(pj), 1) == 0
    aj = np.zeros(1, dtype=_lib.ASM_JOB)
    aj["ry1"], aj["rx1"], aj["nparts"] = 3, 3, 1
    with pytest.raises(Exception, match="x-pass columns"):
        _lib.check(lib.dpm_assemble_prepare(_lib.table_ptr(aj), 1, _lib.table_ptr(pj), 1, None))
    aj["rx1"] = 4
    assert lib.dpm_assemble_prepare(_lib.table_ptr(aj), 1, _lib.table_ptr(pj), 1, None) == 1
    # one job's outputs must fit 32-bit offsets (nparts x hr x wr < 2^31)
    big_pj = np.repeat(pj, 8)
    big_pj["wr"] = 50000
    big = aj.copy()
    big["ry1"], big["rx1"], big["nparts"] = 6000 - 1, 50000 - 1, 8
    with pytest.raises(Exception, match="exceed 2\\^31"):
        _lib.check(lib.dpm_assemble_prepare(_lib.table_ptr(big), 1, _lib.table_ptr(big_pj), 8, None))


def test_assemble_prepare_splits_tiles_between_the_two_k3_kernels():
    """Tiles >= 17 roots wide of jobs whose parts are all at scale 2 with an
    unbounded (or 7..16) radius go to the specialised kernel (block0
    numbering), the others to the generic kernel (block1 numbering)."""
    lib = _lib.lib()
    pj = np.zeros(3, dtype=_lib.PLACE_JOB)
    pj["Hp"], pj["Wp"], pj["range_idx"] = 500, 500, 0
    pj["cdxx"], pj["cdyy"] = 0.01, 0.01
    pj["scale"], pj["radius"] = 2, -1
    pj["rx0"], pj["wr"] = 0, 40
    pj["wr"][2] = 20
    pj["scale"][1] = 1          # job 1: a scale-1 part -> generic only
    aj = np.zeros(3, dtype=_lib.ASM_JOB)
    aj["ry1"] = 99              # 100 root rows: r tile rows (r = ceil(100 / tile height))
    aj["rx1"] = (39, 39, 19)    # 40 columns: a full column and an 8-wide one; 20: one fast column
    aj["part_job0"], aj["nparts"] = (0, 1, 2), 1
    # tile rows of a 100-row job, from a job that is generic whatever the kernel geometry
    one = aj[1:2].copy()
    one["rx1"], one["part_job0"] = 0, 0
    pj1 = pj[1:2].copy()
    pj1["wr"] = 1
    r = lib.dpm_assemble_prepare(_lib.table_ptr(one), 1, _lib.table_ptr(pj1), 1, None)
    assert r >= 2
    nfast = ctypes.c_int64(-1)
    total = lib.dpm_assemble_prepare(_lib.table_ptr(aj), 3, _lib.table_ptr(pj), 3,
                                     ctypes.byref(nfast))
    assert (nfast.value, total) == (r + 0 + r, 2 * r + 2 * r + r)
    assert list(aj["block0"]) == [0, r, r]
    assert list(aj["block1"]) == [0, r, 3 * r]
    pj["radius"][0] = 5         # a fixed radius inside the inner screen -> generic
    assert lib.dpm_assemble_prepare(_lib.table_ptr(aj), 3, _lib.table_ptr(pj), 3,
                                    ctypes.byref(nfast)) == 5 * r
    assert nfast.value == r and list(aj["block1"]) == [0, 2 * r, 4 * r]


def test_tile_shapes():
    lib = _lib.lib()
    tw, th = ctypes.c_int(), ctypes.c_int()
    # 6 filter warps x 2 row warps (32 x 16 positions, 12 warps)
    assert lib.dpm_correlate_tile_shape(6, 48, ctypes.byref(tw), ctypes.byref(th)) == 12
    assert (tw.value, th.value) == (32, 16)
    assert lib.dpm_correlate_tile_shape(6, 6, ctypes.byref(tw), ctypes.byref(th)) == 2
    assert th.value == 16
    assert lib.dpm_correlate_tile_shape(9, 2, ctypes.byref(tw), ctypes.byref(th)) < 0
    assert th.value == 8  # generic kernel tile


def test_gdt_prepare_validates_domain_and_numbers_warps():
    """Lower-envelope GDT tables: unbounded jobs only, centres inside the map,
    block0 in units of 32-row (x) / 32-column (y) warps, 4 warps per CTA."""
    lib = _lib.lib()
    pj = np.zeros(2, dtype=_lib.PLACE_JOB)
    pj["Hp"], pj["Wp"], pj["scale"], pj["radius"], pj["range_idx"] = 70, 40, 2, -1, 0
    pj["rx0"], pj["wr"], pj["ay"], pj["ax"] = 1, 10, 1, 3
    pj["cdxx"], pj["cdyy"] = 0.01, 0.01
    pj["x_off"] = (0, 700)
    assert lib.dpm_gdt_x_prepare(_lib.table_ptr(pj), 2) == 2  # 3 + 3 warps -> 2 CTAs
    assert list(pj["block0"]) == [0, 3]
    aj = np.zeros(1, dtype=_lib.ASM_JOB)
    aj["ry0"], aj["ry1"], aj["rx0"], aj["rx1"], aj["nparts"], aj["part_job0"] = 0, 30, 1, 10, 2, 0
    assert lib.dpm_gdt_y_prepare(_lib.table_ptr(aj), 1, _lib.table_ptr(pj), 2) == 1
    aj["ry1"] = 40  # centre row 2*40 + 1 outside Hp = 70
    with pytest.raises(Exception, match="outside"):
        _lib.check(lib.dpm_gdt_y_prepare(_lib.table_ptr(aj), 1, _lib.table_ptr(pj), 2))
    aj["ry1"], aj["total_off"] = 30, -1
    with pytest.raises(Exception, match="totals"):
        _lib.check(lib.dpm_gdt_y_prepare(_lib.table_ptr(aj), 1, _lib.table_ptr(pj), 2))
    pj["radius"][1] = 3  # windowed jobs belong to dpm_assemble
    with pytest.raises(Exception, match="unbounded"):
        _lib.check(lib.dpm_gdt_x_prepare(_lib.table_ptr(pj), 2))
    pj["radius"][1], pj["wr"][1] = -1, 20  # centre column 2*20 + 3 outside Wp = 40
    with pytest.raises(Exception, match="outside"):
        _lib.check(lib.dpm_gdt_x_prepare(_lib.table_ptr(pj), 2))
