"""Batched pyramid scoring: the B200 path for BASELINE.json configs 2-5.

A model bank (many components, each a root + parts, all filters sharing one
rank-R basis from the reference's ``cp_als`` on the stacked filter tensor,
SURVEY.md App. A.3) is scored over whole feature pyramids of many images in
one plan: one K1 launch, one K2 launch per filter-shape class, one K3 and
one K4 launch -- independent of the number of images, levels and filters.

Root domain / placement:
  * ``domain="gdt"``: roots whose every part centre ``scale*root + anchor``
    lies in the part map; ``radius=-1`` is the unbounded generalised
    distance transform (window of radius r* per map, proven equal);
  * ``domain="reference"``: the reference's ``_hypothesis_rect`` with each
    component's windowed ``search_radius`` (scale 1 only).
"""

import numpy as np

from .engine import AssemblyDef, FilterDef, PartDef, Plan, unpack_positions
from .errors import ValidationError
from .geometry import gdt_root_rect, hypothesis_rect

__all__ = ["PyramidScorer", "cores_from_stacked", "score_pyramid", "detect_batch"]


def cores_from_stacked(bank, G):
    """Split the stacked (P, R) core matrix into per-filter (h, w, R) cores."""
    G = np.asarray(G, dtype=np.float32)
    out = []
    for f, off in zip(bank.filters, bank.offsets()):
        h, w = f.shape[:2]
        out.append(np.ascontiguousarray(G[off:off + h * w].reshape(h, w, -1)))
    if sum(c.shape[0] * c.shape[1] for c in out) != G.shape[0]:
        raise ValidationError("core matrix rows do not match the bank's stacked filters")
    return out


class _PartGeom:
    def __init__(self, dims, anchor, radius):
        self.filter = np.empty(dims)
        self.anchor = anchor
        self.search_radius = radius


class PyramidScorer:
    """Device plan scoring ``n_images`` pyramids against a filter bank."""

    def __init__(self, bank, C, G, pyramid, n_images=1, radius=-1, domain="gdt",
                 outputs=("totals", "positions"), max_dets=0, components=None, envelope=False):
        self.bank, self.pyramid = bank, pyramid
        self.cores = cores_from_stacked(bank, G)
        C = np.asarray(C, dtype=np.float32)
        self.L = C.shape[0]
        comps = list(bank.components) if components is None else list(components)
        filters = [FilterDef(c) for c in self.cores]
        asms = []
        self.asm_keys = []  # (root level index, component index)
        for i, (kr, kp) in enumerate(zip(pyramid.root_levels, pyramid.part_levels)):
            Hr, Wr = pyramid.levels[kr]
            Hp, Wp = pyramid.levels[kp]
            for ci, comp in enumerate(comps):
                rh, rw = bank.filters[comp.root].shape[:2]
                if rh > Hr or rw > Wr:
                    continue
                pdims = [bank.filters[f].shape for f in comp.parts]
                if any(d[0] > Hp or d[1] > Wp for d in pdims):
                    continue
                rad = comp.search_radius if radius is None else radius
                if domain == "gdt":
                    rect = gdt_root_rect((Hr - rh + 1, Wr - rw + 1),
                                         [(Hp - d[0] + 1, Wp - d[1] + 1) for d in pdims],
                                         comp.anchors, pyramid.scale)
                elif domain == "reference":
                    if pyramid.scale != 1 or kr != kp:
                        raise ValidationError("the reference domain is single-resolution")
                    rect = hypothesis_rect((Hr, Wr), (rh, rw),
                                           [_PartGeom(d, a, rad) for d, a in zip(pdims, comp.anchors)])
                else:
                    raise ValidationError(f"unknown domain {domain!r}")
                if rect is None:
                    continue
                parts = tuple(PartDef(kp, f, tuple(a), tuple(d), int(rad), pyramid.scale)
                              for f, a, d in zip(comp.parts, comp.anchors, comp.deformations))
                asms.append(AssemblyDef((kr, comp.root), rect, parts, comp.bias,
                                        level_tag=i, component=ci))
                self.asm_keys.append((i, ci))
        self.plan = Plan(self.L, pyramid.levels, C, filters, assemblies=asms,
                         n_images=n_images, outputs=outputs, max_dets=max_dets, envelope=envelope)
        self.n_images = n_images

    # inputs
    def load_image(self, image, levels):
        self.plan.load_levels(image, levels)

    def host_arena(self, pinned=True):
        """Host buffer laid out like the device X arena (pinned for async H2D)."""
        t = self.plan.torch
        return t.empty(self.plan.X.numel(), dtype=t.float32, pin_memory=pinned)

    def fill_host(self, arena, image, levels):
        plan = self.plan
        for k, lv in enumerate(levels):
            H, W = plan.levels[k]
            off = image * plan.x_image_stride + plan.x_level_off[k]
            arena[off:off + H * W * plan.L].numpy()[:] = np.asarray(lv, np.float32).ravel()

    def h2d_bytes(self):
        """Feature bytes one batch moves host -> device (excluding arena padding)."""
        return 4 * self.plan.L * self.n_images * sum(h * w for h, w in self.plan.levels)

    def score_batch(self, host_arena, tau, stream=None, chunk_images=2):
        """Public end-to-end call: host pyramids (arena layout, pinned) in,
        detections (structured numpy array of DETECTION records with
        score >= tau) out.

        The batch is pipelined in chunks of ``chunk_images`` images: the
        host->device copy of chunk k+1 runs on a copy stream while chunk k is
        scored, so the step costs about max(copy, compute) instead of their sum."""
        t = self.plan.torch
        plan = self.plan
        s = t.cuda.current_stream() if stream is None else stream
        if not hasattr(self, "_copy_stream"):
            self._copy_stream = t.cuda.Stream()
        cs = self._copy_stream
        stride = plan.x_image_stride
        chunks = [range(i, min(i + chunk_images, self.n_images))
                  for i in range(0, self.n_images, chunk_images)]
        copied = []
        cs.wait_stream(s)  # the previous step's readers of X are done
        with t.cuda.stream(cs):
            for c in chunks:
                lo, hi = c.start * stride, c.stop * stride
                plan.X[lo:hi].copy_(host_arena[lo:hi], non_blocking=True)
                ev = t.cuda.Event()
                ev.record(cs)
                copied.append(ev)
        with t.cuda.stream(s):
            if plan.det_count is not None:
                plan.det_count.zero_()
            for k, (c, ev) in enumerate(zip(chunks, copied)):
                s.wait_event(ev)
                plan.run(tau=tau, stream=s, tables=plan.chunk(c), reset_dets=False,
                         init_ranges=(k == 0))
            return plan.detections()

    def score_images(self, host_images, tau, stream=None, chunk_images=16):
        """Public end-to-end call from images: host images (n_images, H, W, C)
        uint8 or float32 in [0, 255] (pinned for async copies) in, detection
        records >= tau out.  The 32-channel HOG pyramid of every image is
        built on the device (features.HogBuilder) straight into the X arena,
        so only the images cross PCIe (1.8 MB per 1280x720 RGB uint8 image,
        against 56.5 MB of float32 HOG pyramid); chunks are pipelined as in
        score_batch."""
        from .features import HogBuilder

        t = self.plan.torch
        plan = self.plan
        n, H, W, C = (int(v) for v in host_images.shape)
        if n != self.n_images:
            raise ValidationError(f"expected {self.n_images} images, got {n}")
        key = (H, W, C, host_images.dtype)
        if getattr(self, "_hog_key", None) != key:
            self._hog = HogBuilder(plan, (H, W), C)
            self._dev_images = t.empty((n, H, W, C), dtype=host_images.dtype, device=plan.device)
            self._hog_key = key
        s = t.cuda.current_stream() if stream is None else stream
        if not hasattr(self, "_copy_stream"):
            self._copy_stream = t.cuda.Stream()
        cs = self._copy_stream
        chunks = [range(i, min(i + chunk_images, n)) for i in range(0, n, chunk_images)]
        copied = []
        cs.wait_stream(s)  # the previous step's readers of the image buffer are done
        with t.cuda.stream(cs):
            for c in chunks:
                self._dev_images[c.start:c.stop].copy_(host_images[c.start:c.stop], non_blocking=True)
                ev = t.cuda.Event()
                ev.record(cs)
                copied.append(ev)
        with t.cuda.stream(s):
            if plan.det_count is not None:
                plan.det_count.zero_()
            for k, (c, ev) in enumerate(zip(chunks, copied)):
                s.wait_event(ev)
                self._hog.run(self._dev_images, stream=s, chunk=c)
                plan.run(tau=tau, stream=s, tables=plan.chunk(c), reset_dets=False,
                         init_ranges=(k == 0))
            return plan.detections()

    def image_bytes(self, host_images):
        return int(host_images.numel() * host_images.element_size())

    @property
    def X(self):
        return self.plan.X

    # execution
    def run(self, tau=float("inf"), stream=None, stages=("project", "correlate", "place")):
        self.plan.run(tau=tau, stream=stream, stages=stages)
        return self

    # outputs
    def results(self, image=0):
        """[{root_level, component, rect, scores (float64), parts (n, hr, wr, 2)}]"""
        out = []
        for ai, (i, ci) in enumerate(self.asm_keys):
            o = self.plan.assembly_outputs(image, ai)
            a = self.plan.assemblies[ai]
            rec = {"root_level": i, "component": ci, "rect": a.rect}
            if "totals" in o:
                rec["scores"] = o["totals"].cpu().numpy()
            if "positions" in o:
                py, px = unpack_positions(o["positions"].cpu().numpy())
                rec["parts"] = np.stack([py, px], axis=-1)
            out.append(rec)
        return out

    def detections(self):
        return self.plan.detections()

    def mixture(self, stream=None):
        """Per-root max over mixture components on
        the device (``dpm_mixture_max``), after ``run()`` / ``score_batch()``.

        For every (image, root level) the union rectangle of its components'
        root rectangles; at each root position the best total among the
        components whose rectangle holds it (ties to the lowest component,
        -inf / -1 where none does).  Returns {(image, root_level): (rect,
        best float64 [hu][wu], component int32 [hu][wu])} as device tensors."""
        from . import _lib
        from .device import stream_handle, upload_table

        plan = self.plan
        if plan.total_size == 0:
            raise ValidationError("mixture() needs the totals output")
        t = plan.torch
        if not hasattr(self, "_mix"):
            aj = plan._asm_jobs
            if (aj["total_off"] < 0).any():
                raise ValidationError("mixture() needs the totals of every assembly")
            groups = {}
            for idx in range(len(aj)):
                key = (int(aj["image"][idx]), int(aj["level"][idx]))
                groups.setdefault(key, []).append(idx)
            jobs, members, keys, off = [], [], [], 0
            for key, idxs in sorted(groups.items()):
                ry0 = int(min(aj["ry0"][idxs])); ry1 = int(max(aj["ry1"][idxs]))
                rx0 = int(min(aj["rx0"][idxs])); rx1 = int(max(aj["rx1"][idxs]))
                jobs.append((off, ry0, ry1, rx0, rx1, len(members), len(idxs), 0, 0))
                members.extend(idxs)
                keys.append((key, (ry0, ry1, rx0, rx1), off))
                off += (ry1 - ry0 + 1) * (rx1 - rx0 + 1)
            jobs = np.array(jobs, dtype=_lib.MIX_JOB)
            nblk = _lib.check(_lib.lib().dpm_mixture_prepare(_lib.table_ptr(jobs), len(jobs)),
                              "mixture")
            dev = plan.device
            self._mix = dict(jobs=upload_table(jobs, dev), njobs=len(jobs), nblk=nblk,
                             members=t.tensor(members, dtype=t.int32, device=dev),
                             ajobs=upload_table(np.ascontiguousarray(aj), dev), keys=keys,
                             best=t.empty(max(off, 1), dtype=t.float64, device=dev),
                             comp=t.empty(max(off, 1), dtype=t.int32, device=dev))
        m = self._mix
        _lib.check(_lib.lib().dpm_mixture_max(
            plan.totals.data_ptr(), m["ajobs"].data_ptr(), m["members"].data_ptr(),
            m["jobs"].data_ptr(), m["njobs"], m["nblk"], m["best"].data_ptr(),
            m["comp"].data_ptr(), stream_handle(stream)), "mixture")
        out = {}
        for (img, lvl), rect, off in m["keys"]:
            hu, wu = rect[1] - rect[0] + 1, rect[3] - rect[2] + 1
            out[(img, lvl)] = (rect, m["best"][off:off + hu * wu].view(hu, wu),
                               m["comp"][off:off + hu * wu].view(hu, wu))
        return out

    # accounting
    def evals_per_image(self):
        return self.plan.evals()

    def k2_flops_per_image(self):
        return self.plan.k2_flops()


def score_pyramid(bank, C, G, pyramid, levels, radius=-1, domain="gdt", components=None,
                  envelope=False):
    """One image through K1-K4 (SURVEY.md §8(b) batched API): per (root level,
    component) the root-level total map and the part argmaxes.

    ``levels`` are the image's pyramid levels ((H, W, L) arrays in the
    geometry of ``pyramid``).  Returns ``PyramidScorer.results(0)``: dicts with
    ``root_level``, ``component``, ``rect``, ``scores`` (float64 [hr][wr]) and
    ``parts`` (int [n_parts][hr][wr][2], (y, x) part positions)."""
    sc = PyramidScorer(bank, C, G, pyramid, n_images=1, radius=radius, domain=domain,
                       components=components, envelope=envelope)
    sc.load_image(0, levels)
    sc.run()
    return sc.results(0)


def detect_batch(bank, C, G, pyramid, images, tau, max_dets=1 << 20, radius=-1,
                 domain="gdt", components=None, chunk_images=2, envelope=False):
    """Many images end to end: host pyramids in, detection
    records with total >= tau out (structured array of ``_lib.DETECTION``:
    image, level, component, ry, rx, nparts, score, packed part positions).
    The pyramids are staged in a pinned arena and scored by
    :meth:`PyramidScorer.score_batch` (H2D pipelined with compute)."""
    images = list(images)
    sc = PyramidScorer(bank, C, G, pyramid, n_images=len(images), radius=radius, domain=domain,
                       max_dets=max_dets, components=components, envelope=envelope)
    host = sc.host_arena(pinned=True)
    for i, levels in enumerate(images):
        sc.fill_host(host, i, levels)
    return sc.score_batch(host, tau, chunk_images=chunk_images)
