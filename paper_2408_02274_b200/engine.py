"""Device-resident IFGF plan and the drop-in ``ifgf_apply``.

``FarFieldPlan`` flattens a (BoxTree, ConeHierarchy) pair -- built by this
package or by the reference itself (same attribute layout) -- plus the
propagation and emission plans into the C ABI of libifgfb200 and keeps the
device copy alive.  ``ifgf_apply`` mirrors reference ``ifgf.py:885-923``
(same signature, argument meaning, output layout and errors).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from . import octree
from .octree import (accumulation_plan, emission_plan, node_tables, row_order_cuts,
                     row_tiles)

__all__ = ["FarFieldPlan", "ifgf_apply", "device_stream"]


def device_stream():
    return torch.cuda.current_stream().cuda_stream


K4_MODES = ("auto", "l1", "l1free", "ring", "ringfree", "wide")


def k4_mode() -> str:
    """Propagation kernel (env IFGFB_K4): "auto" (default) = "wide": the
    wide-warp kernel (4 owner warps per parent row, up to 2 MMA row tiles of
    one sigma group per B-fragment load; tile-free plan); "l1" (5-warp
    kernel with host-built tile records), "l1free" (5-warp kernel, tiles
    formed on the device); "ring" / "ringfree" (child blocks staged in a
    shared-memory ring by TMA bulk copies; measured 45% slower, DESIGN 4)."""
    import os
    m = os.environ.get("IFGFB_K4", "auto")
    if m not in K4_MODES:
        raise ValueError(f"IFGFB_K4: unknown propagation kernel {m!r}")
    return "wide" if m == "auto" else m


class _StageLog:
    """Plan-time stage timings to stderr when IFGFB_PLAN_LOG=1 (cumulative
    seconds since creation, plus the stage's own share)."""

    def __init__(self, name):
        import os
        import time
        self.on = os.environ.get("IFGFB_PLAN_LOG", "0") not in ("", "0")
        self.name = name
        self.t0 = self.t = time.time()

    def __call__(self, what):
        if not self.on:
            return
        import sys
        import time
        now = time.time()
        print(f"[{self.name}] {what} +{now - self.t:.1f}s ({now - self.t0:.1f}s)",
              file=sys.stderr, flush=True)
        self.t = now


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


class FarFieldPlan:
    """libifgfb200 plan for one tree/hierarchy (+ displaced-point geometry)."""

    def __init__(self, tree, hier, displaced_normals=None,
                 displaced_step: float = 1e-6, surface=None, near=None,
                 kappas=None, trim_host: bool = True,
                 geometry_on_device: str | None = None, seam: str = "unwrap"):
        lib = _lib.load()
        if not torch.cuda.is_available():
            raise RuntimeError("CUDA device required (no CPU fallback)")
        cfg = hier.config
        self.tree, self.hier = tree, hier
        self.n = int(tree.points.shape[0])
        self.depth = int(tree.depth)
        self._keep = []          # host arrays referenced during upload
        self.disp = displaced_normals is not None
        self.step = float(displaced_step)
        self.kappas = None if kappas is None else tuple(kappas)
        self.seam = seam
        disp_t = None
        if self.disp:
            nrm = np.asarray(displaced_normals, dtype=float)
            # same expression as reference ifgf.py:822-823
            disp_t = tree.points + displaced_step * nrm[tree.perm]
        pts = _c(tree.points, np.float64)
        perm = _c(tree.perm, np.int64)
        td = _lib.TreeDesc(self.n, self.depth, cfg.p_s, cfg.p_a,
                           _lib.dptr(pts), _lib.iptr(perm))
        h = __import__("ctypes").c_void_p()
        _lib.check(lib.ifgfb_plan_create(td, h), "ifgfb_plan_create")
        self._h = h
        self.stats = {"levels": {}}
        self._log = log = _StageLog("farplan")
        try:
            # uploads are synchronous: host staging arrays are dropped per call
            for d in range(3, self.depth + 1):
                self._add_level(lib, d)
                self._keep = []
            log("levels")
            self.otf_levels = self._choose_otf(geometry_on_device)
            log(f"accumulation plans / otf {sorted(self.otf_levels)}")
            for d in range(4, self.depth + 1):
                self._add_accum(lib, d, d in self.otf_levels)
                self._keep = []
            for d in range(3, self.depth + 1):
                self._add_emission(lib, d, disp_t)
                self._keep = []
                log(f"emission {d}")
            if surface is not None:
                _lib.check(lib.ifgfb_plan_set_surface(self._h, surface),
                           "ifgfb_plan_set_surface")
            if near is not None:
                _lib.check(lib.ifgfb_plan_set_near(self._h, near),
                           "ifgfb_plan_set_near")
            _lib.check(lib.ifgfb_plan_finalize(self._h), "ifgfb_plan_finalize")
            self.stream_parts = 1
        except Exception:
            lib.ifgfb_plan_destroy(self._h)
            self._h = None
            raise
        self._keep = []
        if trim_host:       # the device plan owns the per-type geometry now
            octree.trim_accumulation_plans(hier)

    # ------------------------------------------------------------ upload --
    def _hold(self, *arrs):
        self._keep.extend(arrs)
        return arrs

    def _add_level(self, lib, d):
        tree, hier = self.tree, self.hier
        lvl, cl = tree.level(d), hier.level(d)
        arrs = dict(
            centers=_c(lvl.centers, np.float64),
            pt_start=_c(lvl.pt_start, np.int64),
            pt_count=_c(lvl.pt_count, np.int64),
            seg_off=_c(cl.seg_off, np.int64), seg_ids=_c(cl.seg_ids, np.int64),
            s_nodes=_c(cl.s_nodes, np.float64),
            sin_t=_c(np.sin(cl.ang_nodes_t), np.float64),
            cos_t=_c(np.cos(cl.ang_nodes_t), np.float64),
            sin_p=_c(np.sin(cl.ang_nodes_p), np.float64),
            cos_p=_c(np.cos(cl.ang_nodes_p), np.float64))
        self._hold(*arrs.values())
        desc = _lib.LevelDesc(
            d, lvl.n_boxes, cl.n_s, cl.n_a, lvl.side, cl.h, cl.delta_s,
            cl.delta_a, _lib.dptr(arrs["centers"]),
            _lib.iptr(arrs["pt_start"]), _lib.iptr(arrs["pt_count"]),
            cl.n_segments, _lib.iptr(arrs["seg_off"]),
            _lib.iptr(arrs["seg_ids"]), _lib.dptr(arrs["s_nodes"]),
            _lib.dptr(arrs["sin_t"]), _lib.dptr(arrs["cos_t"]),
            _lib.dptr(arrs["sin_p"]), _lib.dptr(arrs["cos_p"]))
        _lib.check(lib.ifgfb_plan_add_level(self._h, desc),
                   f"ifgfb_plan_add_level({d})")
        self.stats["levels"].setdefault(d, {})["segments"] = int(cl.n_segments)

    # bytes of device plan per propagation type (node_geom, node_r, ratio)
    TYPE_TABLE_BYTES = 75 * (3 + 2 + 4) * 8

    def _choose_otf(self, policy):
        """Levels whose node geometry is computed on the device instead of
        uploaded as per-type tables.  policy "none" / "all" / "auto" (default,
        env IFGFB_GEOM_ON_DEVICE): auto keeps the tables unless the estimated
        device plan exceeds 55% of the device memory, then moves levels to
        on-device geometry, most types per instance first (there the tables
        save the least work)."""
        import os
        policy = policy or os.environ.get("IFGFB_GEOM_ON_DEVICE", "auto")
        levels = list(range(4, self.depth + 1))
        mode = k4_mode()
        self.tile_free = mode.endswith("free") or mode == "wide"
        if policy not in ("none", "all", "auto"):
            raise ValueError(f"geometry_on_device: unknown policy {policy!r}")
        info = {}
        fixed = tile_total = 0
        for d in levels:
            ap = accumulation_plan(self.tree, self.hier, d)
            info[d] = (ap.n_types * self.TYPE_TABLE_BYTES, ap.n_types / max(1, ap.n_instances))
            fixed += (ap.n_instances * 8 + int(ap.inst_crow_off[-1]) * 4
                      + ap.n_types * 75)                                  # group ids
            tile_total += ap.n_instances * (12 * 16 + 20)                 # records + tile_off
        pairs = [self.hier.level(d).cpt_idx.size for d in range(3, self.depth + 1)]
        fixed += sum(pairs) * 80 + max(pairs, default=0) * 2 * 16 * 16
        budget = 0.55 * torch.cuda.get_device_properties(
            torch.cuda.current_device()).total_memory
        tables = sum(b for b, _ in info.values())
        if not self.tile_free:
            fixed += tile_total
        if policy == "none":
            return set()
        if policy == "all":
            return set(levels)
        # a level whose tables are below min_frac of the device memory cannot
        # relieve it, while on-device geometry costs FP64 work (acos, atan2,
        # sincos per node and instance) on the pipe the DMMAs use: keep its
        # tables (fine levels of large configurations: few types, most
        # instances).  IFGFB_OTF_MIN_FRAC=0 restores the plain rule.
        min_frac = float(os.environ.get("IFGFB_OTF_MIN_FRAC", "0.01"))
        total_mem = torch.cuda.get_device_properties(torch.cuda.current_device()).total_memory
        chosen = set()
        for d in sorted(levels, key=lambda d: -info[d][1]):
            if fixed + tables <= budget:
                break
            if info[d][0] < min_frac * total_mem:
                continue
            chosen.add(d)
            tables -= info[d][0]
        return chosen

    def _add_accum(self, lib, d, otf=False):
        ap = accumulation_plan(self.tree, self.hier, d)
        self._log(f"accum plan {d}")
        # crow rows are reproduced exactly as the reference's searchsorted
        # picks them (ifgf.py:743-746), including any inexact hit.
        tile_free = self.tile_free
        if tile_free:
            # the wide-warp kernel on every level (on-device-geometry levels
            # included: 24.3 vs 26.5 ms with every level on-device at (4,10));
            # IFGFB_WIDE_OTF=0 keeps the 5-warp kernel on those levels
            import os
            wide = k4_mode() == "wide" and (not otf or os.environ.get("IFGFB_WIDE_OTF", "1") != "0")
            row_order, row_cuts = row_order_cuts(ap, wide=wide)
            tile_off = tiles = None
        else:
            row_order, row_cuts, tile_off, tiles = row_tiles(ap)
        self._log(f"row tiles {d}")
        node_geom, node_r = (None, None) if otf else node_tables(ap)
        u8 = __import__("ctypes").POINTER(__import__("ctypes").c_uint8)
        a = dict(ng=None if otf else _c(node_geom, np.float64),
                 nr=None if otf else _c(node_r, np.float64),
                 oc=np.ascontiguousarray(ap.type_octant, dtype=np.uint8),
                 ro=np.ascontiguousarray(row_order),
                 rc=np.ascontiguousarray(row_cuts),
                 to=None if tile_free else _c(tile_off, np.int64),
                 tl=None if tile_free else np.ascontiguousarray(tiles),
                 gid=np.ascontiguousarray(ap.gid, dtype=np.uint8),
                 io=_c(ap.inst_off, np.int64), it=_c(ap.inst_type, np.int64),
                 ico=_c(ap.inst_crow_off, np.int64), cr=_c(ap.crow, np.int64))
        self._hold(*[v for v in a.values() if v is not None])
        desc = _lib.AccumDesc(
            d, ap.n_types, _lib.dptr(a["ng"]), _lib.dptr(a["nr"]),
            self.hier.level(d - 1).n_segments, a["ro"].ctypes.data_as(u8),
            a["rc"].ctypes.data_as(u8),
            _lib.iptr(a["io"]), ap.n_instances, _lib.iptr(a["it"]),
            _lib.iptr(a["ico"]), _lib.iptr(a["cr"]), _lib.iptr(a["to"]),
            0 if tile_free else tiles.shape[0],
            None if tile_free else a["tl"].ctypes.data_as(u8), int(otf),
            a["oc"].ctypes.data_as(u8), a["gid"].ctypes.data_as(u8))
        _lib.check(lib.ifgfb_plan_add_accum(self._h, desc),
                   f"ifgfb_plan_add_accum({d})")
        self._log(f"accum upload {d}")
        st = self.stats["levels"].setdefault(d, {})
        st.update(types=int(ap.n_types), instances=int(ap.n_instances),
                  crow_misses=int(ap.crow_misses),
                  tiles=None if tile_free else int(tiles.shape[0]),
                  geometry_on_device=bool(otf))

    def _add_emission(self, lib, d, disp_t):
        ep = emission_plan(self.tree, self.hier, d, disp_t, self.seam)
        a = dict(row=_c(ep.row, np.int64), tg=_c(ep.target, np.int64),
                 g=_c(ep.geom, np.float64),
                 gd=None if ep.geom_disp is None else _c(ep.geom_disp,
                                                         np.float64))
        self._hold(*[v for v in a.values() if v is not None])
        desc = _lib.EmitDesc(d, ep.n_pairs, _lib.iptr(a["row"]),
                             _lib.iptr(a["tg"]), _lib.dptr(a["g"]),
                             _lib.dptr(a["gd"]))
        _lib.check(lib.ifgfb_plan_set_emission(self._h, desc),
                   f"ifgfb_plan_set_emission({d})")
        self.stats["levels"].setdefault(d, {}).update(
            pairs=int(ep.n_pairs), row_misses=int(ep.row_misses))

    # ------------------------------------------------------------- apply --
    @property
    def handle(self):
        return self._h

    def coefficient_bytes_full(self) -> int:
        """Bytes of the two coefficient buffers without streaming."""
        mx = max((self.hier.level(d).n_segments
                  for d in range(3, self.depth + 1)), default=0)
        return 2 * mx * 2432 * 8   # 19 KB per segment (csrc/common.cuh SEG_DOUBLES)

    def set_streaming(self, n_parts: int) -> None:
        """Run the upward pass as n_parts sequential passes over Morton
        groups of level-3 subtrees (ifgfb_plan_set_streaming)."""
        from .partition import level3_partition
        n_parts = max(1, min(int(n_parts), self.tree.level(3).n_boxes))
        parts = level3_partition(self.tree, self.hier, n_parts, n_parts, 1)
        depth = self.depth
        keep, descs = [], (_lib.PartitionDesc * n_parts)()
        for q, part in enumerate(parts):
            lv = (_lib.LevelPart * (depth - 2))()
            for i, d in enumerate(range(3, depth + 1)):
                L = part.levels[d]
                lv[i] = _lib.LevelPart(d, L["seg"][0], L["seg"][1],
                                       L["pair"][0], L["pair"][1])
            keep.append(lv)
            descs[q] = _lib.PartitionDesc(depth - 2, lv, 0, 0)
        _lib.check(_lib.load().ifgfb_plan_set_streaming(self._h, descs, n_parts),
                   "ifgfb_plan_set_streaming")
        self.stream_parts = n_parts

    def auto_stream(self, fraction: float = 0.45) -> int:
        """Stream when two full coefficient levels exceed `fraction` of the
        free device memory; returns the number of parts (1 = no streaming)."""
        free, _ = torch.cuda.mem_get_info()
        need = self.coefficient_bytes_full()
        if self.depth < 3 or need <= fraction * free:
            return 1
        n = int(np.ceil(need / (fraction * free))) + 1
        self.set_streaming(n)
        return n

    def device_bytes(self) -> int:
        return int(_lib.load().ifgfb_plan_device_bytes(self._h))

    def last_launches(self) -> int:
        return int(_lib.load().ifgfb_plan_last_launches(self._h))

    def far_apply_device(self, w: torch.Tensor, kappas, out: torch.Tensor,
                         out_disp: torch.Tensor | None = None):
        """w (nch, N) complex128 cuda tensor (original order) -> out, out_disp
        (nch, nk, N) complex128 cuda tensors."""
        nch = w.shape[0]
        kap = np.zeros(4)
        kk = [complex(k) for k in kappas]
        for i, k in enumerate(kk):
            kap[2 * i], kap[2 * i + 1] = k.real, k.imag
        if out_disp is not None and not self.disp:
            raise ValueError("plan was built without displaced normals")
        _lib.check(_lib.load().ifgfb_far_apply(
            self._h, w.data_ptr(), nch, _lib.dptr(kap), len(kk),
            out.data_ptr(), None if out_disp is None else out_disp.data_ptr(),
            device_stream()), "ifgfb_far_apply")

    def __del__(self):
        if getattr(self, "_h", None) is not None:
            try:
                _lib.load().ifgfb_plan_destroy(self._h)
            except Exception:
                pass
            self._h = None


def _plan_for(tree, hier, normals, step, kappas) -> FarFieldPlan:
    cache = hier.__dict__.setdefault("_b200_plans", {})
    key = (id(tree), None if normals is None else id(normals),
           float(step) if normals is not None else None,
           tuple(complex(k) for k in kappas))
    plan = cache.get(key)
    if plan is None:
        plan = FarFieldPlan(tree, hier, normals, step, kappas=kappas)
        cache[key] = (plan, normals)   # keep normals alive for the id key
        return plan
    return plan[0] if isinstance(plan, tuple) else plan


def ifgf_apply(tree, hier, weights, kappas, mode: str | None = None,
               displaced_normals=None, displaced_step: float = 1e-6):
    """Drop-in for reference ``ifgf_apply`` (ifgf.py:885-923) on the GPU.

    Returns numpy (out, out_disp) of shape (nch, nk, N), original order.
    'vec' and 'seq' give identical values (every column of a group is
    carried through one device traversal; groups of <= 16 columns).
    """
    mode = mode or hier.config.mode
    if mode not in ("vec", "seq"):
        raise ValueError("mode must be 'vec' or 'seq'")
    weights = np.atleast_2d(weights)
    kappas = tuple(kappas)
    nch, nk = weights.shape[0], len(kappas)
    n = tree.points.shape[0]
    if tree.depth < 3:
        z = np.zeros((nch, nk, n), dtype=complex)
        return z, (np.zeros_like(z) if displaced_normals is not None else None)
    if nk > 2:
        parts = [ifgf_apply(tree, hier, weights, kappas[i:i + 2], mode,
                            displaced_normals, displaced_step)
                 for i in range(0, nk, 2)]
        out = np.concatenate([p[0] for p in parts], axis=1)
        od = (None if displaced_normals is None
              else np.concatenate([p[1] for p in parts], axis=1))
        return out, od
    plan = _plan_for(tree, hier, displaced_normals, displaced_step, kappas)
    group = 16 // nk
    dev = torch.device("cuda")
    out = np.empty((nch, nk, n), dtype=complex)
    od = np.empty_like(out) if displaced_normals is not None else None
    for c0 in range(0, nch, group):
        c1 = min(nch, c0 + group)
        w = torch.from_numpy(np.ascontiguousarray(
            weights[c0:c1], dtype=np.complex128)).to(dev)
        o = torch.empty((c1 - c0, nk, n), dtype=torch.complex128, device=dev)
        o_d = torch.empty_like(o) if od is not None else None
        plan.far_apply_device(w, kappas, o, o_d)
        out[c0:c1] = o.cpu().numpy()
        if od is not None:
            od[c0:c1] = o_d.cpu().numpy()
    return out, od


def set_kernel_timing(plan: FarFieldPlan, enable: bool = True) -> None:
    _lib.check(_lib.load().ifgfb_plan_set_timing(plan.handle, int(enable)),
               "ifgfb_plan_set_timing")


def kernel_times(plan: FarFieldPlan) -> dict:
    """{kind: (total_ms, launches)} since the last set_kernel_timing."""
    ms = np.zeros(len(_lib.KERNEL_KINDS))
    cnt = np.zeros(len(_lib.KERNEL_KINDS), dtype=np.int64)
    _lib.check(_lib.load().ifgfb_plan_kernel_times(
        plan.handle, _lib.dptr(ms), _lib.iptr(cnt)), "ifgfb_plan_kernel_times")
    return {k: (float(ms[i]), int(cnt[i]))
            for i, k in enumerate(_lib.KERNEL_KINDS)}


def level_times(plan: FarFieldPlan, max_levels: int = 32) -> dict:
    """{child level d: (propagation ms, launches)} since the last
    set_kernel_timing (the propagation class split by the level it reads)."""
    ms = np.zeros(max_levels)
    cnt = np.zeros(max_levels, dtype=np.int64)
    _lib.check(_lib.load().ifgfb_plan_level_times(
        plan.handle, max_levels, _lib.dptr(ms), _lib.iptr(cnt)), "ifgfb_plan_level_times")
    return {d: (float(ms[d]), int(cnt[d])) for d in range(max_levels) if cnt[d]}
