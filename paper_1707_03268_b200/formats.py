"""Model / scene / pyramid loaders.

Readers for the reference's interchange formats (``pkg/docs/formats.md``):
T3F dense tensors (tensor.py:118-151), CPF CP-decomposed filters
(decomposition.py:427-481) and the JSON model / scene manifests
(model.py:313-488), returning this package's types, which the GPU path
consumes directly.  ``load_pyramid_pinned`` reads T3F feature levels
straight into the pinned host arena of a :class:`PyramidScorer`, without
the float64 widening the reference applies (the device path is float32), so
the H2D copy of ``score_batch`` streams from it unchanged.
"""

import json
import os
import struct

import numpy as np

from .errors import FormatError, ValidationError
from .types import CPModel, DecomposedModel, DecomposedPart, Hypothesis, PartModel, PartSpec

__all__ = ["read_t3f", "write_t3f", "read_cpf", "load_model", "load_scene",
           "load_pyramid_pinned"]

T3F_MAGIC = b"T3F1"
CPF_MAGIC = b"CPF1"
MANIFEST_VERSION = 1


def _read(path):
    with open(path, "rb") as fh:
        return fh.read()


def _t3f_header(data, path):
    if data[:4] != T3F_MAGIC:
        raise FormatError(f"{path}: bad magic at byte 0, expected {T3F_MAGIC!r}")
    if len(data) < 16:
        raise FormatError(f"{path}: truncated header at byte {len(data)}")
    n, m, l = struct.unpack_from("<III", data, 4)
    if min(n, m, l) < 1:
        raise FormatError(f"{path}: non-positive extent in header at byte 4")
    if len(data) != 16 + 4 * n * m * l:
        raise FormatError(f"{path}: payload ends at byte {len(data)}, "
                          f"expected {16 + 4 * n * m * l}")
    return n, m, l


def read_t3f(path, widen=True):
    """T3F tensor: float64 (the reference's in-memory type) or, with
    ``widen=False``, the stored float32 values."""
    data = _read(path)
    n, m, l = _t3f_header(data, path)
    t = np.frombuffer(data, dtype="<f4", count=n * m * l, offset=16).reshape(n, m, l)
    if not np.all(np.isfinite(t)):
        raise ValidationError(f"{path}: non-finite values")
    return t.astype(np.float64) if widen else t.copy()


def write_t3f(path, t):
    """T3F writer (float32 payload, axis-major)."""
    t = np.asarray(t)
    if t.ndim != 3:
        raise ValidationError(f"expected an order-3 tensor, got shape {t.shape}")
    with open(path, "wb") as fh:
        fh.write(T3F_MAGIC + struct.pack("<III", *t.shape))
        fh.write(np.ascontiguousarray(t, dtype="<f4").tobytes())


def read_cpf(path):
    """CPF CP model: float64 weights, float32 factor blocks widened; columns
    re-normalised with the drift folded into the weights (CPModel.from_factors)."""
    data = _read(path)
    if data[:4] != CPF_MAGIC:
        raise FormatError(f"{path}: bad magic at byte 0, expected {CPF_MAGIC!r}")
    if len(data) < 20:
        raise FormatError(f"{path}: truncated header at byte {len(data)}")
    rank, n, m, l = struct.unpack_from("<IIII", data, 4)
    if rank < 1 or min(n, m, l) < 1:
        raise FormatError(f"{path}: non-positive rank or extent at byte 4")
    pos = 20
    if len(data) < pos + 8 * rank:
        raise FormatError(f"{path}: weights end at byte {len(data)}, expected {pos + 8 * rank}")
    weights = np.frombuffer(data, dtype="<f8", count=rank, offset=pos).astype(np.float64)
    pos += 8 * rank
    blocks = []
    for rows in (n, m, l):
        end = pos + 4 * rows * rank
        if len(data) < end:
            raise FormatError(f"{path}: factor block ends at byte {len(data)}, expected {end}")
        blocks.append(np.frombuffer(data, dtype="<f4", count=rows * rank, offset=pos)
                      .astype(np.float64).reshape(rows, rank))
        pos = end
    if len(data) != pos:
        raise FormatError(f"{path}: {len(data) - pos} trailing bytes at byte {pos}")
    return CPModel.from_factors(*blocks, weights=weights)


def _field(doc, key, types, path):
    if key not in doc:
        raise FormatError(f"{path}: manifest field '{key}' is missing")
    if not isinstance(doc[key], types):
        raise FormatError(f"{path}: manifest field '{key}' has the wrong type")
    return doc[key]


def _manifest(path):
    try:
        with open(path, "r", encoding="utf-8") as fh:
            doc = json.load(fh)
    except json.JSONDecodeError as exc:
        raise FormatError(f"{path}: malformed JSON manifest: {exc}") from exc
    version = _field(doc, "version", int, path)
    if version != MANIFEST_VERSION:
        raise FormatError(f"{path}: unsupported manifest version {version}")
    return doc


def load_model(path):
    """Model manifest (model.py:382-488) -> PartModel (T3F payloads) or
    DecomposedModel (CPF payloads, optional thresholds and declared ranks)."""
    path = os.fspath(path)
    base = os.path.dirname(path) or "."
    doc = _manifest(path)
    channels = _field(doc, "channels", int, path)
    bias = float(_field(doc, "bias", (int, float), path))
    root_entry = _field(doc, "root", (str, dict), path)
    parts_entry = _field(doc, "parts", list, path)

    def payload(name):
        full = os.path.join(base, name)
        magic = _read(full)[:4]
        if magic == T3F_MAGIC:
            return read_t3f(full)
        if magic == CPF_MAGIC:
            return read_cpf(full)
        raise FormatError(f"{full}: unknown payload magic at byte 0")

    if isinstance(root_entry, str):
        root, root_thr, root_rank = payload(root_entry), None, None
    else:
        root = payload(_field(root_entry, "payload", str, path))
        root_thr = root_entry.get("thresholds")
        root_rank = root_entry.get("rank")
    decomposed = isinstance(root, CPModel)
    parts = []
    for i, entry in enumerate(parts_entry):
        if not isinstance(entry, dict):
            raise FormatError(f"{path}: parts[{i}] must be an object")
        pl = payload(_field(entry, "payload", str, path))
        if isinstance(pl, CPModel) != decomposed:
            raise FormatError(f"{path}: parts[{i}] payload format does not match the root's")
        anchor = _field(entry, "anchor", list, path)
        deformation = _field(entry, "deformation", list, path)
        radius = _field(entry, "search_radius", int, path)
        if decomposed:
            rank = entry.get("rank")
            if rank is not None and rank != pl.rank:
                raise FormatError(f"{path}: parts[{i}] declares rank {rank} but the payload "
                                  f"has rank {pl.rank}")
            thr = entry.get("thresholds")
            parts.append(DecomposedPart(pl, anchor, deformation, radius,
                                        None if thr is None else np.asarray(thr, np.float64)))
        else:
            parts.append(PartSpec(pl, anchor, deformation, radius))
    if decomposed:
        if root_rank is not None and root_rank != root.rank:
            raise FormatError(f"{path}: root declares rank {root_rank} but the payload has "
                              f"rank {root.rank}")
        model = DecomposedModel(root, tuple(parts), bias,
                                None if root_thr is None else np.asarray(root_thr, np.float64))
    else:
        model = PartModel(root, tuple(parts), bias)
    if model.channels != channels:
        raise FormatError(f"{path}: manifest declares {channels} channels but the root payload "
                          f"has {model.channels}")
    return model


def load_scene(path):
    """Scene manifest (formats.md "Scene manifest"): (levels as float64
    (H, W, L) arrays, [(level, Hypothesis)] planted truths)."""
    path = os.fspath(path)
    base = os.path.dirname(path) or "."
    try:
        with open(path, "r", encoding="utf-8") as fh:
            doc = json.load(fh)
    except json.JSONDecodeError as exc:
        raise FormatError(f"{path}: malformed JSON scene manifest: {exc}") from exc
    for key in ("version", "levels", "truth", "noise_level", "seed"):  # synthetic.py:243-247
        if key not in doc:
            raise FormatError(f"{path}: scene manifest field '{key}' is missing")
    if doc["version"] != 1:
        raise FormatError(f"{path}: unsupported scene version {doc['version']}")
    levels = [read_t3f(os.path.join(base, name))
              for name in _field(doc, "levels", list, path)]
    truths = []
    for i, t in enumerate(_field(doc, "truth", list, path)):
        if not isinstance(t, dict):
            raise FormatError(f"{path}: truth[{i}] must be an object")
        lvl = _field(t, "level", int, path)
        root = tuple(int(v) for v in _field(t, "root", list, path))
        parts = tuple(tuple(int(v) for v in p) for p in _field(t, "parts", list, path))
        score = t.get("score")
        truths.append((lvl, Hypothesis(level=lvl, root=root, parts=parts, score=score)))
    return levels, truths


def load_pyramid_pinned(scorer, arena, image, level_paths):
    """Read one image's T3F levels straight into ``scorer``'s pinned host arena
    (float32 as stored; extents checked against the scorer's pyramid)."""
    plan = scorer.plan
    if len(level_paths) != len(plan.levels):
        raise ValidationError(f"{len(level_paths)} level files for a {len(plan.levels)}-level "
                              "pyramid")
    host = arena.numpy()
    for k, p in enumerate(level_paths):
        data = _read(p)
        n, m, l = _t3f_header(data, p)
        H, W = plan.levels[k]
        if (n, m, l) != (H, W, plan.L):
            raise ValidationError(f"{p}: level {k} is {n}x{m}x{l}, the pyramid expects "
                                  f"{H}x{W}x{plan.L}")
        off = image * plan.x_image_stride + plan.x_level_off[k]
        host[off:off + n * m * l] = np.frombuffer(data, dtype="<f4", count=n * m * l, offset=16)
