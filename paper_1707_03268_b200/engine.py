"""Planner + executor of the B200 score path (K1 -> K2 -> K3 -> K4).

A :class:`Plan` is built once per (geometry, model) on the host: it lays
out the HBM arenas, groups filters into GEMM launch classes, builds the
device work-lists, and uploads the model's basis and cores.  ``run()`` then
issues one launch per kernel (one K2 launch per filter-shape class) on a
CUDA stream, with no host synchronisation, so a run can be captured into a
CUDA graph.  PyTorch is only the allocator / stream provider here.

HBM layout (per image, images stacked):
  X arena : levels back to back, each [H][W][L] float32 (the reference's
            axis-major feature-map order, validation.py:65-86)
  P arena : levels back to back, each planar [Rtot][H][pitch] float32
  S arena : response maps, one block [nf][Ho][Wo] per (level, filter group)
"""

import os
from dataclasses import dataclass, field

import ctypes

import numpy as np

from . import _lib
from .device import require_cuda, stream_handle, upload_table
from .errors import ValidationError

__all__ = ["FilterDef", "PartDef", "AssemblyDef", "Plan", "MAX_GROUP"]

MAX_GROUP = 48  # filters per K2 group (6 warps x 8 filters)


@dataclass(frozen=True)
class FilterDef:
    """Core of one filter over ``R`` consecutive basis channels from ``chan_off``.

    ``prefix = k >= 1`` makes it the rank-``k`` prefix of ``core`` (ranks < k),
    computed by the rank-prefix kernel together with the family's other
    prefixes: a plan must request prefixes 1..K of one core (the same array
    object) together, and gets all K maps from one pass over the ranks."""

    core: np.ndarray  # (h, w, R) float32
    chan_off: int = 0
    prefix: int = 0

    @property
    def h(self):
        return self.core.shape[0]

    @property
    def w(self):
        return self.core.shape[1]

    @property
    def R(self):
        return self.core.shape[2]


@dataclass(frozen=True)
class PartDef:
    level: int
    filt: int
    anchor: tuple
    deformation: tuple
    radius: int  # >= 0 windowed (reference), < 0 unbounded GDT (r*)
    scale: int = 1


@dataclass(frozen=True)
class AssemblyDef:
    root: tuple  # (level, filt) or None
    rect: tuple  # (ry0, ry1, rx0, rx1) inclusive root positions
    parts: tuple = ()
    bias: float = 0.0
    level_tag: int = 0
    component: int = 0


def _round_up(v, m):
    return (v + m - 1) // m * m


@dataclass
class _Arena:
    size: int = 0

    def take(self, n, align=32):
        off = _round_up(self.size, align)
        self.size = off + n
        return off


class Plan:
    """Device plan for ``n_images`` images sharing one pyramid geometry.

    Parameters
    ----------
    L : channels of the feature levels.
    levels : [(H, W)] pyramid level shapes (per image).
    C : (L, Rtot) float32 basis.
    filters : [FilterDef].
    apps : extra (level, filter) maps to compute besides those the
        assemblies need.
    assemblies : [AssemblyDef] (root + parts placed and summed).
    outputs : subset of {"totals", "positions", "placed"}.
    max_dets : capacity of the on-device detection buffer (0 = none).
    envelope : place unbounded (radius < 0) assemblies on the GDT root domain
        with the Felzenszwalb lower-envelope kernels (dpm_gdt_x / dpm_gdt_y)
        instead of the windowed r* kernel (dpm_assemble).  Both give the same
        placements (up to exact ties); the window is the default because it
        is faster at the r* (~10) of the benchmark maps.
    tc_ranks : ranks R whose filter groups may run on tcgen05: R = 8 (the
        compile-time DPM shapes), R = 16 (6 x 6 filters, corr_tc16.cu).
    tc_generic : also route other shapes at R > 8 to the generic-shape
        tcgen05 kernel (measured slower than FFMA; off by default).
    tc_min_strips : fewest 128-column strips for which a 6 x 6 R = 16 class
        goes to corr_tc16 (default 2 per SM; below that FFMA is faster).
    """

    def __init__(self, L, levels, C, filters, apps=(), assemblies=(), n_images=1,
                 outputs=("totals", "positions"), max_dets=0, device=None, tensor_cores=True,
                 tc_min_width=16, envelope=False, tc_ranks=(8, 16), tc_generic=False,
                 tc_min_strips=None):
        import torch

        require_cuda()
        self.torch = torch
        self.device = torch.device("cuda") if device is None else torch.device(device)
        self.L = int(L)
        self.levels = [tuple(int(v) for v in lv) for lv in levels]
        self.n_images = int(n_images)
        C = np.ascontiguousarray(C, dtype=np.float32)
        if C.ndim != 2 or C.shape[0] != self.L:
            raise ValidationError(f"basis must be ({self.L}, R), got {C.shape}")
        self.Rtot = C.shape[1]
        self.filters = list(filters)
        self.assemblies = list(assemblies)
        self.outputs = set(outputs)
        self.max_dets = int(max_dets)
        self.tensor_cores = bool(tensor_cores)
        self.tc_min_width = int(tc_min_width)
        self.envelope = bool(envelope)
        self.tc_ranks = tuple(int(r) for r in tc_ranks)
        self.tc_generic = bool(tc_generic)
        self.tc_min_strips = None if tc_min_strips is None else int(tc_min_strips)
        for k, f in enumerate(self.filters):
            if f.chan_off < 0 or f.chan_off + f.R > self.Rtot:
                raise ValidationError(f"filter {k}: channels [{f.chan_off}, {f.chan_off + f.R}) "
                                      f"outside the basis of rank {self.Rtot}")
        self._apps_key = tuple(sorted(set((int(a), int(b)) for a, b in apps)))
        self._layout(apps)
        self._upload(C)

    # ------------------------------------------------------------ layout
    def _layout(self, apps):
        lib = _lib.lib()
        nimg = self.n_images
        # which maps are needed
        needed = set((int(a), int(b)) for a, b in apps)
        for asm in self.assemblies:
            if asm.root is not None:
                needed.add(tuple(asm.root))
            for p in asm.parts:
                needed.add((p.level, p.filt))
        for k, f in needed:
            H, W = self.levels[k]
            fd = self.filters[f]
            if fd.h > H or fd.w > W:
                raise ValidationError(f"filter extent ({fd.h}, {fd.w}) exceeds image extent "
                                      f"({H}, {W})")
        # every placed map gets a range slot: r* (GDT mode) and the FP32
        # screening error bound of the placement kernel both come from it
        placed_maps = set((p.level, p.filt) for a in self.assemblies for p in a.parts)

        # per-image level offsets
        xa, pa = _Arena(), _Arena()
        self.x_level_off, self.p_level_off, self.pitch = [], [], []
        for H, W in self.levels:
            pitch = _round_up(W, 4)
            self.pitch.append(pitch)
            self.x_level_off.append(xa.take(H * W * self.L, align=4))
            self.p_level_off.append(pa.take(self.Rtot * H * pitch, align=4))
        self.x_image_stride = _round_up(xa.size, 32)
        self.p_image_stride = _round_up(pa.size, 32)

        # filter groups per level (same h, w, R, chan_off; <= MAX_GROUP filters)
        by_level = {}
        for k, f in sorted(needed):
            by_level.setdefault(k, []).append(f)
        self.groups = []  # (level, (filters...))
        self._prefix_groups = set()  # groups computed by the rank-prefix kernel
        # corr_tc16 (6 x 6, R = 16, 16-filter groups) pays off only with enough
        # 128-column strips to fill the SMs (one strip per persistent CTA at a
        # time; a small pyramid leaves most SMs idle behind its tallest strips):
        # fewer than 2 per SM -> FFMA with 48-filter groups (config 2 at R = 16:
        # 90 strips, 0.32 ms tcgen05 against 0.29 ms FFMA)
        strips16 = {}
        for k in by_level:
            H, W = self.levels[k]
            cnt = {}
            for f in by_level[k]:
                fd = self.filters[f]
                if fd.prefix == 0 and _tc16(fd.h, fd.w, fd.R, 16):
                    cnt[(fd.h, fd.w, fd.R)] = cnt.get((fd.h, fd.w, fd.R), 0) + 1
            for key, n in cnt.items():
                wo = W - key[1] + 1
                if wo >= self.tc_min_width:
                    strips16[key] = strips16.get(key, 0) + nimg * ((n + 15) // 16) * ((wo + 127) // 128)
        min_strips = 2 * _sm_count() if self.tc_min_strips is None else self.tc_min_strips
        self._tc16_off = {key for key, n in strips16.items() if n < min_strips}
        for k in sorted(by_level):
            keyed = {}
            for f in by_level[k]:
                fd = self.filters[f]
                fam = id(fd.core) if fd.prefix > 0 else 0  # one rank-prefix family per core
                keyed.setdefault((fd.h, fd.w, fd.R, fd.chan_off, fam), []).append(f)
            for key in sorted(keyed):
                fl = keyed[key]
                if key[4]:  # prefixes 1..K of one core, in rank order, one group
                    fl = sorted(fl, key=lambda f: self.filters[f].prefix)
                    ks = [self.filters[f].prefix for f in fl]
                    if ks != list(range(1, len(fl) + 1)) or len(fl) > MAX_GROUP:
                        raise ValidationError(f"rank-prefix filters {ks}: a plan computes "
                                              f"prefixes 1..K (K <= {MAX_GROUP}) of a core together")
                    self._prefix_groups.add(tuple(fl))
                    self.groups.append((k, tuple(fl)))
                    continue
                g = self._group_size(*key[:3])
                for s in range(0, len(fl), g):
                    self.groups.append((k, tuple(fl[s:s + g])))

        # cores: one block per distinct filter tuple; tensor-core eligible
        # groups (tcgen05 path) also in the [tap][R/4][2N][4] hi|lo layout
        self._pack_cores()

        # S arena, K2 jobs, tiles, range slots
        sa = _Arena()
        tc_classes = {}
        self.map_off = {}  # (image, level, filt) -> float offset
        self.map_shape = {}
        self.range_slot = {}
        jobs, classes, prefix_classes = [], {}, {}
        job_image = []
        nslots = 0
        self.map_smap = {}  # (image, level, filt) -> (TMA descriptor, index in its group)
        smap_descs = []
        for img in range(nimg):
            for k, fl in self.groups:
                H, W = self.levels[k]
                fd = self.filters[fl[0]]
                ho, wo = H - fd.h + 1, W - fd.w + 1
                wp = _spitch(wo)  # rows padded to 16 B (include/dpm_b200.h, "S maps")
                s_off = sa.take(len(fl) * ho * wp, align=4)
                for i, f in enumerate(fl):
                    self.map_smap[(img, k, f)] = (len(smap_descs), i)
                smap_descs.append((s_off, ho, wo, len(fl), 0))
                rng = -1
                if any((k, f) in placed_maps for f in fl):
                    rng = nslots
                    nslots += len(fl)
                for i, f in enumerate(fl):
                    self.map_off[(img, k, f)] = s_off + i * ho * wp
                    self.map_shape[(k, f)] = (ho, wo)
                    if rng >= 0:
                        self.range_slot[(img, k, f)] = rng + i
                jid = len(jobs)
                job_image.append(img)
                prefix = fl in self._prefix_groups
                jobs.append((img * self.p_image_stride + self.p_level_off[k], s_off,
                             self.core_off[fl], H, W, self.pitch[k], fd.chan_off, fd.h, fd.w,
                             fd.R, len(fl), _round_up(len(fl), 8), 1 if prefix else 0, rng, 0))
                if prefix:  # rank-prefix kernel: tiles per filter height
                    ptw, pth = self._prefix_tile()
                    pt = prefix_classes.setdefault(fd.h, [])
                    for ty in range((ho + pth - 1) // pth):
                        for tx in range((wo + ptw - 1) // ptw):
                            pt.append((jid, ty, tx, 0))
                    continue
                if fl in self.tc_core_off and wo >= self.tc_min_width:
                    tcc = tc_classes.setdefault(fl, [])
                    for sx in range((wo + 127) // 128):
                        tcc.append((jid, 0, sx, ho))
                    continue
                tw, th = self._tile_shape(fd.h, len(fl))
                cls = classes.setdefault((fd.h, len(fl)), {"tiles": [], "w_max": 1, "R": 1})
                cls["w_max"] = max(cls["w_max"], fd.w)
                cls["R"] = max(cls["R"], fd.R)
                for ty in range((ho + th - 1) // th):
                    for tx in range((wo + tw - 1) // tw):
                        cls["tiles"].append((jid, ty, tx, 0))
        self.s_size = max(sa.size, 4)
        self._smap_descs = np.array(smap_descs, dtype=_lib.SMAP_DESC)
        self.n_ranges = nslots
        self._corr_jobs = np.array(jobs, dtype=_lib.CORR_JOB) if jobs else np.zeros(0, _lib.CORR_JOB)
        self._corr_job_image = np.array(job_image, dtype=np.int64)
        # A class of > 8 filters with fewer tiles than SMs (e.g. config 5's 16-filter
        # part groups at the small levels where only two components fit) is a
        # latency-bound launch of its own: its tiles join the largest > 8-filter
        # class of the same filter height, whose 32 x 16 tiles and per-job cores
        # serve any nf up to its own (the extra filter warps of those few tiles idle).
        for h in sorted({h for h, _ in classes}):
            big = [(len(c["tiles"]), nf) for (hh, nf), c in classes.items() if hh == h and nf > 8]
            if len(big) < 2:
                continue
            target = classes[(h, max(big)[1])]
            tnf = max(big)[1]
            for n, nf in big:
                c = classes[(h, nf)]
                if c is not target and nf < tnf and n < _sm_count():
                    target["tiles"].extend(c["tiles"])
                    target["w_max"] = max(target["w_max"], c["w_max"])
                    target["R"] = max(target["R"], c["R"])
                    del classes[(h, nf)]
        self._classes = []
        for (h, nf), cls in sorted(classes.items()):
            # tiles sorted by core so persistent CTAs keep it resident
            tl = sorted(cls["tiles"], key=lambda t: (jobs[t[0]][2], t[0], t[1], t[2]))
            self._classes.append((h, nf, cls["R"], cls["w_max"], np.array(tl, dtype=_lib.CORR_TILE)))

        self._prefix_classes = [(h, np.array(tl, dtype=_lib.CORR_TILE))
                                for h, tl in sorted(prefix_classes.items())]
        if prefix_classes:
            pjobs = np.ascontiguousarray(self._corr_jobs[self._corr_jobs["mode"] == 1])
            _lib.check(lib.dpm_correlate_prefix_check(_lib.table_ptr(pjobs), len(pjobs)), "prefix")
        # tcgen05 launches: one per group for the compile-time DPM shapes (R = 8,
        # 6 x 6 / 6 x 11); the generic-shape groups of one (h, w, R, N) share
        # ONE launch (dpm_correlate_tc_groups: per-job core offsets, the core
        # reloaded by a bulk copy when a CTA's strip changes group)
        self._tc_classes = []  # (name, h, w, R, nf, core offset or -1, strips, tc_off or None)
        merged = {}
        for fl, strips in sorted(tc_classes.items()):
            fd = self.filters[fl[0]]
            if _tc_compiled(fd.h, fd.w, fd.R):
                # the one-row part kernel (6 x 6, more than 8 filters; tc_stack in
                # corr_tc.cu) walks segments too, the stacked-row kernel whole strips
                if fd.w == 6 and len(fl) > 8:
                    strips = _segment_strips(strips, _sm_count())
                strips = _snake_order(strips, key=lambda t: t[3], ctas=_sm_count())
                arr = np.array([(j, y0, sx, n if n < ho_full else 0)
                                for j, y0, sx, n, ho_full in
                                ((t[0], t[1], t[2], t[3], t[4] if len(t) > 4 else t[3])
                                 for t in strips)], dtype=_lib.CORR_TILE)
                self._tc_classes.append((f"k2_tcgen05_{fd.h}x{fd.w}_nf{len(fl)}", fd.h, fd.w,
                                         fd.R, len(fl), self.tc_core_off[fl], arr, None))
            else:
                m = merged.setdefault((fd.h, fd.w, fd.R, _round_up(len(fl), 16)), [])
                m.append((fl, strips))
        for (h, w, R, npad), members in sorted(merged.items()):
            tc_off = np.full(max(len(jobs), 1), -1, dtype=np.int64)
            allstrips = []
            for fl, strips in members:
                for st in strips:
                    tc_off[st[0]] = self.tc_core_off[fl]
                allstrips.extend(strips)
            allstrips = _snake_order(allstrips, key=lambda t: t[3], ctas=_sm_count())
            arr = np.array([(j, 0, sx, 0) for j, _, sx, _ in allstrips], dtype=_lib.CORR_TILE)
            self._tc_classes.append((f"k2_tcgen05_{h}x{w}_R{R}_groups{len(members)}", h, w, R,
                                     npad, -1, arr, tc_off))

        # K1 jobs
        pj = [(img * self.x_image_stride + self.x_level_off[k],
               img * self.p_image_stride + self.p_level_off[k], H, W, self.pitch[k], 0)
              for img in range(nimg) for k, (H, W) in enumerate(self.levels)]
        self._proj_jobs = np.array(pj, dtype=_lib.PROJ_JOB)

        # placement + assembly jobs
        ta, oa, pla, ga = _Arena(), _Arena(), _Arena(), _Arena()
        place, asm_jobs, asm_gdt = [], [], []
        self.asm_index = {}  # (image, a) -> (total_off, pos_off, placed_off, hr, wr)
        for img in range(nimg):
            for ai, a in enumerate(self.assemblies):
                ry0, ry1, rx0, rx1 = a.rect
                hr, wr = ry1 - ry0 + 1, rx1 - rx0 + 1
                if hr < 1 or wr < 1:
                    raise ValidationError(f"assembly {ai}: empty root rectangle {a.rect}")
                if len(a.parts) > _lib.MAX_PARTS:
                    raise ValidationError(f"assembly {ai}: more than {_lib.MAX_PARTS} parts")
                first = len(place)
                use_gdt = self._gdt_eligible(a)
                for p in a.parts:
                    hp, wp = self.map_shape[(p.level, p.filt)]
                    x_off = ga.take(hp * wr, align=8) if use_gdt else 0
                    place.append((self.map_off[(img, p.level, p.filt)], x_off,
                                  hp, wp, p.anchor[0], p.anchor[1], p.scale, p.radius, rx0, wr,
                                  self.range_slot[(img, p.level, p.filt)], 0,
                                  *self.map_smap[(img, p.level, p.filt)],
                                  *[float(v) for v in p.deformation]))
                root_off, root_pitch = -1, 0
                if a.root is not None:
                    root_off = self.map_off[(img, a.root[0], a.root[1])]
                    root_pitch = _spitch(self.map_shape[tuple(a.root)][1])
                    rh, rw = self.map_shape[tuple(a.root)]
                    if not (0 <= ry0 and ry1 < rh and 0 <= rx0 and rx1 < rw):
                        raise ValidationError(f"assembly {ai}: rect {a.rect} outside the root "
                                              f"map {rh}x{rw}")
                # the GDT kernel accumulates parts in the totals: always allocated
                t_off = ta.take(hr * wr, align=4) if ("totals" in self.outputs or use_gdt) else -1
                p_off = oa.take(len(a.parts) * hr * wr, align=4) if "positions" in self.outputs else -1
                pl_off = pla.take(len(a.parts) * hr * wr, align=4) if "placed" in self.outputs else -1
                self.asm_index[(img, ai)] = (t_off, p_off, pl_off, hr, wr)
                asm_jobs.append((root_off, t_off, p_off, pl_off, root_pitch, ry0, ry1, rx0, rx1,
                                 first, len(a.parts), img, a.level_tag, a.component, 0, 0,
                                 float(a.bias)))
                asm_gdt.append(use_gdt)
        self._place_jobs = np.array(place, dtype=_lib.PLACE_JOB) if place else np.zeros(0, _lib.PLACE_JOB)
        self._asm_jobs = np.array(asm_jobs, dtype=_lib.ASM_JOB) if asm_jobs else np.zeros(0, _lib.ASM_JOB)
        _lib.check(lib.dpm_place_prepare(_lib.table_ptr(self._place_jobs), len(self._place_jobs)),
                   "placement")
        self._asm_gdt = np.array(asm_gdt, dtype=bool)
        self.total_size, self.pos_size, self.placed_size = ta.size, oa.size, pla.size
        self.gdt_scratch = ga.size

    def _gdt_eligible(self, a):
        """Lower-envelope path: every part unbounded with positive quadratic
        coefficients and every part centre of the rectangle inside its map
        (the GDT root domain)."""
        if not self.envelope or not a.parts:
            return False
        ry0, ry1, rx0, rx1 = a.rect
        for p in a.parts:
            cdx, cdy, cdxx, cdyy = (float(v) for v in p.deformation)
            if p.radius >= 0 or cdxx <= 0 or cdyy <= 0:
                return False
            hp, wp = self.map_shape[(p.level, p.filt)]
            s, (ay, ax) = p.scale, p.anchor
            if not (s * ry0 + ay >= 0 and s * ry1 + ay < hp and s * rx0 + ax >= 0
                    and s * rx1 + ax < wp):
                return False
        return True

    def _tc_fits(self, h, w, R, nf):
        if R > 8 and not self.tc_generic and (not _tc16(h, w, R, nf) or
                                               (h, w, R) in getattr(self, "_tc16_off", ())):
            return False  # generic shapes at R > 8 measured slower than FFMA
        return (R in self.tc_ranks and R % 8 == 0 and R <= 32 and 1 <= nf <= 64 and
                h + 2 <= 16 and w <= 64 and
                _lib.lib().dpm_correlate_tc_smem(h, w, R, nf) <= 227 * 1024)

    def _pack_cores(self):
        """Host core arrays (FP32 blocks [h][w][R][nf_pad] per group, and the
        tcgen05 layout of the eligible groups) with their offsets."""
        ga, tca = _Arena(), _Arena()
        self.core_off, self.tc_core_off = {}, {}
        blocks, tc_blocks = [], []
        for _, fl in self.groups:
            if fl in self.core_off:
                continue
            fd0 = self.filters[fl[0]]
            block = np.zeros((fd0.h, fd0.w, fd0.R, _round_up(len(fl), 8)), dtype=np.float32)
            for i, f in enumerate(fl):
                block[:, :, :, i] = self.filters[f].core
            self.core_off[fl] = ga.take(block.size, align=4)
            blocks.append((self.core_off[fl], block))
            if self._tc_eligible(fl):
                tcb = _tc_core([self.filters[f].core for f in fl])
                self.tc_core_off[fl] = tca.take(tcb.size, align=64)
                tc_blocks.append((self.tc_core_off[fl], tcb))
        self._core_host = np.zeros(max(ga.size, 4), dtype=np.float32)
        for off, block in blocks:
            self._core_host[off:off + block.size] = block.ravel()
        self._tc_core_host = np.zeros(max(tca.size, 4), dtype=np.float32)
        for off, block in tc_blocks:
            self._tc_core_host[off:off + block.size] = block.ravel()

    def _opts(self):
        return (self.tensor_cores, self.tc_min_width, self.tc_ranks, self.tc_generic,
                self.tc_min_strips, self.envelope,
                tuple(sorted(self.outputs)), self.max_dets, str(self.device))

    def signature(self):
        """Layout key of a correlation plan (no assemblies): plans with equal
        signatures differ only in basis and core VALUES, which rebind() swaps."""
        return plan_signature(self.L, self.levels, self.n_images, self.Rtot, self.filters,
                              self._apps_key, self._opts())

    def rebind(self, C, filters):
        """Swap the basis and the filter cores for ones of the same layout
        (same signature), re-uploading them in place; levels are reloaded by
        the caller.  Lets a cached plan serve repeated drop-in calls (the
        reference's loops over images and models) without rebuilding tables."""
        if self.assemblies:
            raise ValidationError("rebind: plans with assemblies are not rebindable")
        C = np.ascontiguousarray(C, dtype=np.float32)
        filters = list(filters)
        if plan_signature(self.L, self.levels, self.n_images, C.shape[1] if C.ndim == 2 else -1,
                          filters, self._apps_key, self._opts()) != self.signature() or \
                C.shape != tuple(self.C.shape):
            raise ValidationError("rebind: basis / filters do not match the plan's layout")
        core_off, tc_core_off = self.core_off, self.tc_core_off
        self.filters = filters
        self._pack_cores()
        assert self.core_off == core_off and self.tc_core_off == tc_core_off
        t = self.torch
        self.C.copy_(t.from_numpy(C))
        self.G.copy_(t.from_numpy(self._core_host))
        self.Gtc.copy_(t.from_numpy(self._tc_core_host))
        return self

    def _tc_eligible(self, fl):
        if not self.tensor_cores or fl in self._prefix_groups:
            return False
        fd = self.filters[fl[0]]
        return self._tc_fits(fd.h, fd.w, fd.R, len(fl))

    def _group_size(self, h, w, R):
        """Filters per K2 group: MAX_GROUP, or -- when R > 8 goes to the tensor
        cores (``tc_ranks``) -- the largest of 48 / 32 / 16 whose resident
        tcgen05 core and input ring fit shared memory: 16 for 6 x 6 at R = 16,
        the compile-time kernel of corr_tc16.cu, whose groups share one launch
        (config 3: 4.7 ms for the 6 x 6 class against 11.5 ms FFMA).  Other
        shapes at R > 8 (the generic-shape kernel) only with ``tc_generic``:
        they measured slower than FFMA."""
        if self.tensor_cores and R > 8:
            for g in (48, 32, 16):
                if self._tc_fits(h, w, R, g):
                    return g
        return MAX_GROUP

    _tile_cache = {}

    def _prefix_tile(self):
        import ctypes

        if "prefix" not in self._tile_cache:
            tw, th = ctypes.c_int(0), ctypes.c_int(0)
            _lib.check(_lib.lib().dpm_correlate_prefix_tile(ctypes.byref(tw), ctypes.byref(th)),
                       "prefix")
            self._tile_cache["prefix"] = (tw.value, th.value)
        return self._tile_cache["prefix"]

    def _tile_shape(self, h, nf):
        import ctypes

        if (h, nf) not in self._tile_cache:
            tw, th = ctypes.c_int(0), ctypes.c_int(0)
            _lib.lib().dpm_correlate_tile_shape(h, nf, ctypes.byref(tw), ctypes.byref(th))
            self._tile_cache[(h, nf)] = (tw.value, th.value)
        return self._tile_cache[(h, nf)]

    # ------------------------------------------------------------ buffers
    def _upload(self, C):
        t = self.torch
        dev = self.device
        self.C = t.from_numpy(C).to(dev)
        self.G = t.from_numpy(self._core_host).to(dev)
        self.corr_jobs_d = upload_table(self._corr_jobs, dev)
        self.Gtc = t.from_numpy(self._tc_core_host).to(dev)
        self.place_jobs_d = upload_table(self._place_jobs, dev)
        self._full = self._make_tables(range(self.n_images))
        self._chunk_tables = {}
        self.X = t.empty(self.n_images * self.x_image_stride, dtype=t.float32, device=dev)
        self.P = t.empty(self.n_images * self.p_image_stride, dtype=t.float32, device=dev)
        self.S = t.empty(self.s_size, dtype=t.float32, device=dev)
        # TMA descriptors of the S map groups (K3 band staging); they embed S's address
        maps = np.zeros(max(len(self._smap_descs), 1) * _lib.SMAP_BYTES + 64, dtype=np.uint8)
        a64 = (-maps.ctypes.data) % 64
        maps_h = maps[a64:a64 + len(self._smap_descs) * _lib.SMAP_BYTES]
        _lib.check(_lib.lib().dpm_smap_encode(self.S.data_ptr(), _lib.table_ptr(self._smap_descs),
                                       len(self._smap_descs), maps_h.ctypes.data), "smap encode")
        self.smaps = t.from_numpy(maps_h.copy()).to(dev)
        self.ranges = t.empty(max(2 * self.n_ranges, 2), dtype=t.int32, device=dev)
        self.totals = t.empty(max(self.total_size, 1), dtype=t.float64, device=dev)
        self.positions = t.empty(max(self.pos_size, 1), dtype=t.int32, device=dev)
        self.placed = t.empty(max(self.placed_size, 1), dtype=t.float64, device=dev)
        self.prep = t.empty(max(4 * len(self._place_jobs), 4), dtype=t.int32, device=dev)
        self.gsv = t.empty(max(self.gdt_scratch, 1), dtype=t.float32, device=dev)
        self.gdx = t.empty(max(self.gdt_scratch, 1), dtype=t.int16, device=dev)
        if self.max_dets > 0:
            self.dets = t.empty(self.max_dets * _lib.DETECTION.itemsize, dtype=t.uint8, device=dev)
            self.det_count = t.zeros(1, dtype=t.int32, device=dev)
        else:
            self.dets = self.det_count = None

    def _make_tables(self, images):
        """Launch tables restricted to ``images`` (all of them for run())."""
        lib = _lib.lib()
        dev = self.device
        imgs = set(images)
        tb = {}
        pj = self._proj_jobs[[i // len(self.levels) in imgs for i in range(len(self._proj_jobs))]]
        pj = np.ascontiguousarray(pj)
        nblk = _lib.check(lib.dpm_project_prepare(_lib.table_ptr(pj), len(pj)), "project")
        tb["proj"] = (upload_table(pj, dev), len(pj), nblk)  # upload after block0 is filled
        keep = np.isin(self._corr_job_image, list(imgs))
        tb["tc"] = []
        for name, h, w, R, nf, goff, strips, tc_off in self._tc_classes:
            sub = np.ascontiguousarray(strips[keep[strips["job"]]])
            off_d = None if tc_off is None else self.torch.from_numpy(tc_off).to(dev)
            tb["tc"].append((name, h, w, R, nf, goff, len(sub), upload_table(sub, dev), off_d))
        tb["ffma"] = []
        for h, nf, R, w_max, tiles in self._classes:
            sub = np.ascontiguousarray(tiles[keep[tiles["job"]]])
            tb["ffma"].append((h, nf, R, w_max, len(sub), upload_table(sub, dev)))
        tb["prefix"] = []
        for h, tiles in self._prefix_classes:
            sub = np.ascontiguousarray(tiles[keep[tiles["job"]]])
            tb["prefix"].append((h, len(sub), upload_table(sub, dev)))
        in_chunk = np.isin(self._asm_jobs["image"], list(imgs))
        aj = np.ascontiguousarray(self._asm_jobs[in_chunk & ~self._asm_gdt])
        nfast = ctypes.c_int64(0)
        blocks = _lib.check(lib.dpm_assemble_prepare(
            _lib.table_ptr(aj), len(aj), _lib.table_ptr(self._place_jobs), len(self._place_jobs),
            ctypes.byref(nfast)), "assembly")
        tb["asm"] = (upload_table(aj, dev), len(aj), (nfast.value, blocks))
        # lower-envelope GDT: x-pass table (the chunk's placement jobs) and the
        # y-pass/assembly table (indexing the full placement table)
        gj = np.ascontiguousarray(self._asm_jobs[in_chunk & self._asm_gdt])
        sel = np.concatenate([np.arange(j["part_job0"], j["part_job0"] + j["nparts"]) for j in gj]) \
            if len(gj) else np.zeros(0, np.int64)
        xj = np.ascontiguousarray(self._place_jobs[sel])
        xblocks = _lib.check(lib.dpm_gdt_x_prepare(_lib.table_ptr(xj), len(xj)), "gdt x pass")
        yblocks = _lib.check(lib.dpm_gdt_y_prepare(
            _lib.table_ptr(gj), len(gj), _lib.table_ptr(self._place_jobs), len(self._place_jobs)),
            "gdt y pass")
        tb["gdt"] = (upload_table(xj, dev), len(xj), xblocks, upload_table(gj, dev), len(gj),
                     yblocks)
        return tb

    def chunk(self, images):
        """Launch tables of an image range (cached), for pipelined runs."""
        key = (images.start, images.stop)
        if key not in self._chunk_tables:
            self._chunk_tables[key] = self._make_tables(images)
        return self._chunk_tables[key]

    # ------------------------------------------------------------ inputs
    def x_view(self, image, level):
        H, W = self.levels[level]
        off = image * self.x_image_stride + self.x_level_off[level]
        return self.X[off:off + H * W * self.L].view(H, W, self.L)

    def load_levels(self, image, levels):
        """Copy one image's levels (numpy or torch, (H, W, L)) into the X arena."""
        t = self.torch
        for k, lv in enumerate(levels):
            src = lv if isinstance(lv, t.Tensor) else t.from_numpy(np.ascontiguousarray(lv, dtype=np.float32))
            self.x_view(image, k).copy_(src, non_blocking=True)

    # ------------------------------------------------------------ execute
    def run(self, tau=float("inf"), stream=None, stages=("project", "correlate", "place"),
            mark=None, tables=None, reset_dets=True, init_ranges=True):
        """Issue K1..K4 on ``stream`` (default: torch's current stream).

        ``tables`` restricts the run to an image chunk (``chunk()``);
        ``mark(name)``, if given, is called before every kernel launch and
        once at the end with name None (the bench records CUDA events there)."""
        lib = _lib.lib()
        t = self.torch
        s = stream_handle(stream)
        ptr = lambda x: x.data_ptr()  # noqa: E731
        mark = mark or (lambda name: None)
        tb = self._full if tables is None else tables
        if "project" in stages and tb["proj"][1]:
            mark("k1_project")
            pj_d, npj, nblk = tb["proj"]
            _lib.check(lib.dpm_project(ptr(self.X), ptr(self.P), ptr(self.C), self.L, self.Rtot,
                                       ptr(pj_d), npj, nblk, s), "project")
        if "correlate" in stages:
            if self.n_ranges and init_ranges:
                mark("ranges_init")
                _lib.check(lib.dpm_ranges_init(ptr(self.ranges), self.n_ranges, s), "ranges")
            rng = ptr(self.ranges) if self.n_ranges else None
            for name, h, w, R, nf, goff, n, strips_d, off_d in tb["tc"]:
                if not n:
                    continue
                mark(name)
                if off_d is None:
                    _lib.check(lib.dpm_correlate_tc(ptr(self.P), ptr(self.Gtc) + 4 * goff,
                                                    ptr(self.S), ptr(self.corr_jobs_d),
                                                    ptr(strips_d), n, h, w, R, nf, rng, s),
                               "correlate_tc")
                else:
                    _lib.check(lib.dpm_correlate_tc_groups(ptr(self.P), ptr(self.Gtc), ptr(off_d),
                                                           ptr(self.S), ptr(self.corr_jobs_d),
                                                           ptr(strips_d), n, h, w, R, nf, rng, s),
                               "correlate_tc")
            for h, nf, R, w_max, n, tiles_d in tb["ffma"]:
                if not n:
                    continue
                mark(f"k2_ffma_h{h}_nf{nf}")
                _lib.check(lib.dpm_correlate(ptr(self.P), ptr(self.G), ptr(self.S),
                                             ptr(self.corr_jobs_d), ptr(tiles_d), n, h,
                                             nf, R, w_max, rng, s), "correlate")
            for h, n, tiles_d in tb["prefix"]:
                if not n:
                    continue
                mark(f"k2_prefix_h{h}")
                _lib.check(lib.dpm_correlate_prefix(ptr(self.P), ptr(self.G), ptr(self.S),
                                                    ptr(self.corr_jobs_d), ptr(tiles_d), n, h, rng,
                                                    s), "correlate prefix")
        place = "place" in stages and (tb["asm"][1] or tb["gdt"][4])
        if place and self.det_count is not None and reset_dets:
            with t.cuda.stream(stream if stream is not None else t.cuda.current_stream()):
                self.det_count.zero_()
        opt = lambda x, n: ptr(x) if n else None  # noqa: E731
        dets = (ptr(self.dets) if self.dets is not None else None, self.max_dets,
                ptr(self.det_count) if self.det_count is not None else None)
        if place and tb["gdt"][4]:
            xj_d, nxj, xblk, gj_d, ngj, yblk = tb["gdt"]
            mark("k3x_gdt_rows")
            _lib.check(lib.dpm_gdt_x(ptr(self.S), ptr(self.gsv), ptr(self.gdx), ptr(xj_d), nxj,
                                     xblk, ptr(self.ranges), s), "gdt x pass")
            mark("k3y_gdt_cols_assemble")
            _lib.check(lib.dpm_gdt_y(ptr(self.S), ptr(self.gsv), ptr(self.gdx),
                                     ptr(self.place_jobs_d), ptr(gj_d), ngj, yblk, ptr(self.ranges),
                                     ptr(self.totals), opt(self.positions, self.pos_size),
                                     opt(self.placed, self.placed_size), float(tau), *dets, s),
                       "gdt y pass")
        if place and tb["asm"][1]:
            mark("k3_place_ranges")
            _lib.check(lib.dpm_place_ranges(ptr(self.place_jobs_d), len(self._place_jobs),
                                            ptr(self.ranges), ptr(self.prep), s), "place ranges")
            mark("k3k4_place_assemble")
            aj_d, naj, (nfast, nblk) = tb["asm"]
            _lib.check(lib.dpm_assemble(
                ptr(self.S), ptr(self.smaps), ptr(self.place_jobs_d), ptr(aj_d), naj, nfast, nblk,
                ptr(self.prep),
                ptr(self.totals) if self.total_size else None,
                ptr(self.positions) if self.pos_size else None,
                ptr(self.placed) if self.placed_size else None,
                float(tau),
                ptr(self.dets) if self.dets is not None else None, self.max_dets,
                ptr(self.det_count) if self.det_count is not None else None, s), "assemble")
        mark(None)
        return self

    # ------------------------------------------------------------ outputs
    def map(self, image, level, filt):
        ho, wo = self.map_shape[(level, filt)]
        off = self.map_off[(image, level, filt)]
        wp = _spitch(wo)
        return self.S[off:off + ho * wp].view(ho, wp)[:, :wo]

    def assembly_outputs(self, image, a):
        t_off, p_off, pl_off, hr, wr = self.asm_index[(image, a)]
        n = len(self.assemblies[a].parts)
        out = {}
        if t_off >= 0:
            out["totals"] = self.totals[t_off:t_off + hr * wr].view(hr, wr)
        if p_off >= 0:
            out["positions"] = self.positions[p_off:p_off + n * hr * wr].view(n, hr, wr)
        if pl_off >= 0:
            out["placed"] = self.placed[pl_off:pl_off + n * hr * wr].view(n, hr, wr)
        return out

    def detections(self):
        """Copy the detection records to the host (structured numpy array)."""
        if self.det_count is None:
            return np.zeros(0, dtype=_lib.DETECTION)
        n = int(self.det_count.item())
        if n > self.max_dets:
            raise ValidationError(f"{n} detections exceed the buffer of {self.max_dets}; "
                                  "raise max_dets or tau")
        raw = self.dets[: n * _lib.DETECTION.itemsize].cpu().numpy()
        return raw.view(_lib.DETECTION).copy()

    # ------------------------------------------------------------ accounting
    def launches_per_run(self):
        """Kernels of libdpm_b200 one full run() launches."""
        n = 1 + len(self._tc_classes) + len(self._classes) + len(self._prefix_classes)  # K1, K2
        n += 1 if self.n_ranges else 0
        if (~self._asm_gdt).any():
            n += 2  # prologue + placement/assembly
        if self._asm_gdt.any():
            n += 2
        return n

    def evals(self):
        """cell x filter evaluations per image (BASELINE.md §3 unit of work)."""
        return sum(self.map_shape[(k, f)][0] * self.map_shape[(k, f)][1]
                   for k, fl in self.groups for f in fl)

    def k2_flops(self):
        """Algorithmic K2 FLOPs per image: 2*h*w*R per eval."""
        tot = 0
        for k, fl in self.groups:
            for f in fl:
                fd = self.filters[f]
                ho, wo = self.map_shape[(k, f)]
                tot += 2 * fd.h * fd.w * fd.R * ho * wo
        return tot

    def launch_flops(self):
        """Algorithmic K2 FLOPs (2*h*w*R per eval, all images) of each K2
        launch, keyed like the names run() passes to ``mark``."""
        jobs = self._corr_jobs
        out = {}

        def fl(jids):
            return sum(2 * int(jobs[j]["h"]) * int(jobs[j]["w"]) * int(jobs[j]["R"]) *
                       int(jobs[j]["nf"]) * (int(jobs[j]["H"]) - int(jobs[j]["h"]) + 1) *
                       (int(jobs[j]["W"]) - int(jobs[j]["w"]) + 1) for j in set(jids))
        for name, h, w, R, nf, _, strips, _ in self._tc_classes:
            out[name] = fl(strips["job"].tolist())
        for h, nf, R, _, tiles in self._classes:
            out[f"k2_ffma_h{h}_nf{nf}"] = fl(tiles["job"].tolist())
        for h, tiles in self._prefix_classes:
            # one pass over the ranks: 2*h*w per rank and position (K ranks)
            out[f"k2_prefix_h{h}"] = sum(
                2 * int(jobs[j]["h"]) * int(jobs[j]["w"]) * int(jobs[j]["nf"]) *
                (int(jobs[j]["H"]) - int(jobs[j]["h"]) + 1) * (int(jobs[j]["W"]) - int(jobs[j]["w"]) + 1)
                for j in set(tiles["job"].tolist()))
        return out

    def k1_bytes(self):
        return sum(4 * (self.L + self.Rtot) * H * W for H, W in self.levels)


def _tc16(h, w, R, nf):
    """6 x 6 filters at R = 16, <= 16 per group: corr_tc16.cu (tc16_shape)."""
    return h == 6 and w == 6 and R == 16 and nf <= 16


def _tc_compiled(h, w, R):
    """Shapes with a compile-time tcgen05 kernel (tc_bf16 in corr_tc.cu)."""
    return R == 8 and h == 6 and w in (6, 11)


def _sm_count():
    """SMs of the current CUDA device (the persistent tcgen05 grid), 148 on
    B200; the B200 value when no device is visible (host-only planning)."""
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    except Exception:  # planning without a usable device
        pass
    return 148


def plan_signature(L, levels, n_images, Rtot, filters, apps_key, opts=()):
    """Everything a plan's layout depends on: geometry, filter shapes and
    rank-prefix families (by first member, not by array identity), the maps
    requested and the plan options."""
    fams, fsig = {}, []
    for i, f in enumerate(filters):
        fam = fams.setdefault(id(f.core), i) if f.prefix > 0 else -1
        fsig.append((f.h, f.w, f.R, f.chan_off, f.prefix, fam))
    return (int(L), tuple(tuple(int(v) for v in lv) for lv in levels), int(n_images), int(Rtot),
            tuple(fsig), tuple(apps_key), tuple(opts))


def _spitch(w):
    """Row pitch (floats) of a response map of width w (s_pitch in csrc)."""
    return (w + 3) & ~3


def _segment_strips(strips, sms, per_sm=2, min_rows=16):
    """Split the tcgen05 part strips (job, 0, sx, ho) of a small pyramid into
    row segments (job, y0, sx, rows, ho) so that the persistent grid (one CTA
    per SM) gets about ``per_sm`` items per SM: a single 640x480 or 1920x1080
    pyramid has only ~60-250 strips, each walked top to bottom by one CTA.  A
    segment re-stages its filter's h - 1 halo rows; segments are at least
    ``min_rows`` output rows.  Batches with enough strips are left whole (the
    kernels read rows = 0 as the whole strip); DPM_TC_SEGMENT=0 turns it off."""
    if len(strips) >= per_sm * sms or os.environ.get("DPM_TC_SEGMENT") == "0":
        return [(j, 0, sx, ho, ho) for j, _, sx, ho in strips]
    total = sum(t[3] for t in strips)
    seg = max(min_rows, -(-total // (per_sm * sms)))
    # fewer than per_sm * sms segments: the C side pairs CTAs (corr_tc2.cu) only
    # for launches of at least 2 strips per SM, which must be whole strips
    while sum(-(-ho // seg) for _, _, _, ho in strips) >= per_sm * sms:
        seg += max(1, seg // 16)
    out = []
    for j, _, sx, ho in strips:
        n = -(-ho // seg)
        step = -(-ho // n)
        for y0 in range(0, ho, step):
            out.append((j, y0, sx, min(step, ho - y0), ho))
    return out


def _snake_order(items, key, ctas=148):
    """Order work items for a persistent kernel whose CTA b takes items b,
    b + G, b + 2G, ... (G = grid size): tallest first, dealt in boustrophedon
    rounds (CTA 0..G-1, then G-1..0, ...), so every CTA gets a near-equal
    total instead of CTA 0 taking the largest item of every round.  G is the
    SM count (the grid of the tcgen05 kernel); with fewer items than SMs the
    order is irrelevant."""
    srt = sorted(items, key=lambda t: -key(t))
    out = list(srt)
    for r in range(0, len(srt), ctas):
        rnd = srt[r:r + ctas]
        if (r // ctas) % 2 == 1 and len(rnd) == ctas:
            rnd = rnd[::-1]
        out[r:r + len(rnd)] = rnd
    return out


def _bf16_rn(x):
    """float32 -> bf16 bit patterns (uint16), round to nearest even."""
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def _tc_core(cores):
    """Cores of one group in the tcgen05 B layout [h*w][R/4][2N][4]: rows < N
    the tf32-truncated values, rows >= N the exact fp32 remainders.  For the
    shapes whose kernel runs the bf16 correction MMA
    (dpm_correlate_tc_core_floats larger than that block), the bf16 tap-pair
    block [h][ceil(w/2)][2][N][8] of the truncated values follows."""
    core = np.stack([np.asarray(c, np.float32) for c in cores], axis=-1)  # (h, w, R, nf)
    h, w, R, nf = core.shape
    N = _round_up(nf, 16)
    hi = (core.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
    lo = (core - hi).astype(np.float32)
    ks = int(_lib.lib().dpm_correlate_tc_stack(h, w, R, nf))
    if ks > 1:
        return _tc_core_stacked(hi, lo, ks)
    out = np.zeros((h * w, R // 4, 2 * N, 4), dtype=np.float32)
    for src, base in ((hi, 0), (lo, N)):
        t = src.reshape(h * w, R // 4, 4, nf).transpose(0, 1, 3, 2)  # (tap, quad, nf, 4)
        out[:, :, base:base + nf, :] = t
    out = out.ravel()
    total = int(_lib.lib().dpm_correlate_tc_core_floats(h, w, R, nf))
    if total > out.size and R == 16:
        # 6 x 6 at R = 16 (corr_tc16.cu): bf16 block [tap][2][N][8], plane c =
        # ranks 8c..8c+7 of the truncated values
        b2 = np.zeros((h * w, 2, N, 8), dtype=np.uint16)
        bits = _bf16_rn(hi).reshape(h * w, 2, 8, nf)  # (tap, plane, rank, nf)
        b2[:, :, :nf, :] = bits.transpose(0, 1, 3, 2)
        out = np.concatenate([out, b2.ravel().view(np.float32)])
        assert out.size == total, (out.size, total)
    elif total > out.size:
        npairs = (w + 1) // 2
        b2 = np.zeros((h, npairs, 2, N, 8), dtype=np.uint16)
        bits = _bf16_rn(hi)  # (h, w, R, nf)
        for j in range(w):
            b2[:, j // 2, j % 2, :nf, :] = bits[:, j, :, :].transpose(0, 2, 1)  # (h, nf, R)
        out = np.concatenate([out, b2.ravel().view(np.float32)])
        assert out.size == total, (out.size, total)
    return out


def _tc_core_stacked(hi, lo, ks):
    """Stacked tcgen05 core (dpm_correlate_tc_stack() = ks > 1, <= 8 filters):
    per tap column, NB = h + 2(ks-1) tap-row blocks (block b = tap row
    h-1+ks-1-b, zero outside the filter) of 16 N-rows [hi f0..7 | lo f0..7],
    so the kernel's B window for input-row offset t starts at block
    h-1+ks-1-t and covers output rows y..y+ks-1 with tap rows t..t-ks+1."""
    h, w, R, nf = hi.shape
    nb = h + 2 * (ks - 1)
    tf = np.zeros((w, R // 4, nb * 16, 4), dtype=np.float32)
    b2 = np.zeros(((w + 1) // 2, 2, nb * 16, 8), dtype=np.uint16)
    bits = _bf16_rn(hi)  # (h, w, R, nf)
    for b in range(nb):
        i = h - 1 + ks - 1 - b
        if not 0 <= i < h:
            continue
        for j in range(w):
            for src, base in ((hi, 0), (lo, 8)):
                t = src[i, j].reshape(R // 4, 4, nf).transpose(0, 2, 1)  # (quad, nf, 4)
                tf[j, :, b * 16 + base:b * 16 + base + nf, :] = t
            b2[j // 2, j % 2, b * 16:b * 16 + nf, :] = bits[i, j].T  # (nf, R)
    out = np.concatenate([tf.ravel(), b2.ravel().view(np.float32)])
    assert out.size == int(_lib.lib().dpm_correlate_tc_core_floats(h, w, R, nf))
    return out


def unpack_positions(packed):
    """uint32 (int16 y << 16 | int16 x) -> (y, x) int arrays."""
    p = np.asarray(packed).astype(np.uint32)
    y = (p >> 16).astype(np.uint16).view(np.int16).astype(np.int64)
    x = (p & 0xFFFF).astype(np.uint16).view(np.int16).astype(np.int64)
    return y, x
