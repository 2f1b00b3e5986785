"""Host-side detection emission: NMS, matching and
the ROC sweep against the reference's own test cases (pkg/tests/
test_evaluation.py:24-60) and an independent loop restatement."""

import numpy as np
import pytest

from paper_1707_03268_b200 import _lib
from paper_1707_03268_b200.evaluation import match_detections, nms, nms_records, roc_eval
from paper_1707_03268_b200.errors import ValidationError
from paper_1707_03268_b200.types import Detection, Hypothesis


def det(level, y, x, score):
    return Detection(Hypothesis(level=level, root=(y, x), score=score), model_id="m",
                     score=score, tau=-np.inf)


def test_nms_reference_cases():
    kept = nms([det(0, 5, 5, 10.0), det(0, 6, 5, 8.0), det(0, 20, 20, 9.0)], (4, 4, 1), 0.5)
    roots = [k.hypothesis.root for k in kept]
    assert (5, 5) in roots and (20, 20) in roots and (6, 5) not in roots
    assert len(nms([det(0, 5, 5, 10.0), det(1, 5, 5, 8.0)], (4, 4, 1))) == 2


def test_match_reference_cases():
    truths = [(0, Hypothesis(0, (5, 5))), (0, Hypothesis(0, (20, 20)))]
    assert match_detections([det(0, 5, 6, 10.0), det(0, 9, 9, 7.0)], truths, 1) == (1, 1)
    truths = [(0, Hypothesis(0, (5, 5)))]
    assert match_detections([det(0, 5, 5, 10.0), det(0, 5, 6, 9.0)], truths, 1) == (1, 1)


def _nms_loop(dets, dims, thr):
    # plain restatement of evaluation.py:47-68
    def iou(a, b):
        iy = max(0, min(a[0] + dims[0], b[0] + dims[0]) - max(a[0], b[0]))
        ix = max(0, min(a[1] + dims[1], b[1] + dims[1]) - max(a[1], b[1]))
        inter = iy * ix
        union = 2 * dims[0] * dims[1] - inter
        return inter / union if union else 0.0
    kept = []
    for c in sorted(dets, key=lambda d: (-d.score, d.hypothesis.level, d.hypothesis.root)):
        if not any(k.hypothesis.level == c.hypothesis.level and
                   iou(k.hypothesis.root, c.hypothesis.root) >= thr for k in kept):
            kept.append(c)
    return sorted(kept, key=lambda d: (d.hypothesis.level, d.hypothesis.root))


def test_nms_matches_loop_restatement_with_ties():
    rng = np.random.default_rng(5)
    dets = [det(int(rng.integers(0, 3)), int(rng.integers(0, 40)), int(rng.integers(0, 40)),
                float(rng.integers(0, 6))) for _ in range(400)]  # many exact score ties
    for thr in (0.3, 0.5, 0.7):
        a = nms(dets, (5, 7, 1), thr)
        b = _nms_loop(dets, (5, 7), thr)
        assert [(d.hypothesis.level, d.hypothesis.root, d.score) for d in a] == \
            [(d.hypothesis.level, d.hypothesis.root, d.score) for d in b]


def test_nms_records_equals_nms_per_image():
    rng = np.random.default_rng(6)
    n = 300
    rec = np.zeros(n, dtype=_lib.DETECTION)
    rec["image"] = rng.integers(0, 2, n)
    rec["level"] = rng.integers(0, 3, n)
    rec["ry"], rec["rx"] = rng.integers(0, 30, n), rng.integers(0, 30, n)
    rec["score"] = rng.integers(0, 5, n).astype(np.float64)
    kept = nms_records(rec, [(6, 11)], 0.5)
    for img in (0, 1):
        sub = rec[rec["image"] == img]
        ref = nms([det(int(r["level"]), int(r["ry"]), int(r["rx"]), float(r["score"]))
                   for r in sub], (6, 11, 1), 0.5)
        got = kept[kept["image"] == img]
        assert [(int(r["level"]), (int(r["ry"]), int(r["rx"]))) for r in got] == \
            [(d.hypothesis.level, d.hypothesis.root) for d in ref]


def test_roc_rejects_empty_grid():
    with pytest.raises(ValidationError, match="tau grid"):
        roc_eval(object(), [], [])
