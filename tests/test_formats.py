"""Format readers against files written by the
reference's own savers (tests/golden/make_golden.py gen_formats): every
loaded array bit-identical to what the reference's loaders return."""

import json
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from paper_1707_03268_b200 import formats as F
from paper_1707_03268_b200.errors import FormatError
from paper_1707_03268_b200.types import CPModel, DecomposedModel, PartModel

D = os.path.join(GOLDEN, "formats")


def _cp_equal(cp, g, prefix):
    for k, a in (("w", cp.weights), ("a", cp.factors_a), ("b", cp.factors_b),
                 ("c", cp.factors_c)):
        assert np.array_equal(a, g[f"{prefix}_{k}"]), (prefix, k)


def test_dense_model_manifest():
    g = load_golden("formats/expected.npz")
    m = F.load_model(os.path.join(D, "dense.json"))
    assert isinstance(m, PartModel) and m.bias == g["dense_bias"]
    assert np.array_equal(m.root, g["dense_root"])
    for i, p in enumerate(m.parts):
        assert np.array_equal(p.filter, g[f"dense_part{i}"])


def test_decomposed_model_manifest_with_thresholds():
    g = load_golden("formats/expected.npz")
    m = F.load_model(os.path.join(D, "dec.json"))
    assert isinstance(m, DecomposedModel) and m.calibrated
    _cp_equal(m.root_cp, g, "dec_root")
    assert np.array_equal(m.root_thresholds, g["dec_root_thr"])
    for i, p in enumerate(m.parts):
        _cp_equal(p.cp, g, f"dec_part{i}")
        assert np.array_equal(p.thresholds, g[f"dec_part{i}_thr"])


def test_scene_manifest():
    g = load_golden("formats/expected.npz")
    levels, truths = F.load_scene(os.path.join(D, "scene.json"))
    for i, lv in enumerate(levels):
        assert np.array_equal(lv, g[f"scene_level{i}"])
    ref = g["scene_truth"]
    assert len(truths) == len(ref)
    for (lvl, h), r in zip(truths, ref):
        assert (lvl, *h.root, *[v for p in h.parts for v in p]) == tuple(int(v) for v in r[:-1])
        assert h.score == r[-1]


def test_reader_errors(tmp_path):
    shutil.copytree(D, tmp_path / "f")
    d = tmp_path / "f"
    raw = (d / "dec_root.cpf").read_bytes()
    (d / "bad.cpf").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(FormatError, match="bad magic"):
        F.read_cpf(str(d / "bad.cpf"))
    (d / "long.cpf").write_bytes(raw + b"\0")
    with pytest.raises(FormatError, match="trailing bytes"):
        F.read_cpf(str(d / "long.cpf"))
    (d / "short.t3f").write_bytes((d / "dense_root.t3f").read_bytes()[:-4])
    with pytest.raises(FormatError, match="payload ends"):
        F.read_t3f(str(d / "short.t3f"))
    doc = json.loads((d / "dec.json").read_text())
    doc["parts"][0]["rank"] = 7
    (d / "rank.json").write_text(json.dumps(doc))
    with pytest.raises(FormatError, match="declares rank 7"):
        F.load_model(str(d / "rank.json"))
    doc = json.loads((d / "dense.json").read_text())
    doc["channels"] = 5
    (d / "ch.json").write_text(json.dumps(doc))
    with pytest.raises(FormatError, match="declares 5 channels"):
        F.load_model(str(d / "ch.json"))


def test_t3f_round_trip(tmp_path):
    t = np.random.default_rng(0).random((3, 4, 5)).astype(np.float32)
    F.write_t3f(str(tmp_path / "t.t3f"), t)
    assert np.array_equal(F.read_t3f(str(tmp_path / "t.t3f"), widen=False), t)
    assert F.read_t3f(str(tmp_path / "t.t3f")).dtype == np.float64
