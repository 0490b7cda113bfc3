"""CPU oracle for the CRSH secondary-ray path (arXiv 2312.06538).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs -- never by the product
package.  The arithmetic lives in ``oracle.cpp`` (plain C++17, float32, built
with -ffp-contract=off); this module is argument marshalling plus the
stage-by-stage driver ``trace()`` that follows the paper's order (Fig 1,
PAPER.md:57-65): generate+hash -> trim -> compress -> sort -> decompress ->
build -> traverse (mesh cull + levels) -> final tests.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "oracle.cpp")
CXXFLAGS = ["-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread"]

SH, RE, RR = 1, 2, 4
F_SORT, F_MESH_CULL, F_ZORDER = 1, 2, 4
F_OBJTREE = 64        # object sphere-tree below the mesh spheres (NEXT-4)
CLUSTER_TRIS = 32     # triangles per object-tree cluster (reading O1)
UINT64_MAX = np.uint64(0xFFFFFFFFFFFFFFFF)


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["g++", *CXXFLAGS, "-o", LIB, SRC])
    return LIB


_lib = None
vp = C.c_void_p


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        L.or_atan2p.restype = C.c_float
        L.or_atan2p.argtypes = [C.c_float, C.c_float]
        L.or_sincos.argtypes = [C.c_float, vp, vp]
        L.or_hash_shadow.restype = C.c_uint32
        L.or_hash_shadow.argtypes = [C.c_uint32, vp, C.c_int]
        L.or_hash_bounce.restype = C.c_uint32
        L.or_hash_bounce.argtypes = [vp, vp, vp, vp, C.c_int]
        L.or_cone_grow.argtypes = [vp, C.c_float, vp, vp, vp]
        L.or_cone_union.argtypes = [vp, C.c_float, vp, C.c_float, vp, vp]
        L.or_sphere_union.argtypes = [vp, vp, vp]
        L.or_cull.restype = C.c_int
        L.or_cull.argtypes = [vp, vp]
        L.or_mt.restype = C.c_int
        L.or_mt.argtypes = [vp, vp, vp]
        L.or_tri_sphere.argtypes = [vp, vp]
        L.or_miniball.restype = C.c_int
        L.or_miniball.argtypes = [vp, C.c_int64, vp]
        L.or_scene_prep.restype = C.c_int
        L.or_scene_prep.argtypes = [vp, vp, C.c_int64, C.c_int32, vp, vp, vp, vp, vp, C.c_float, C.c_float, vp]
        L.or_transform.restype = None
        L.or_transform.argtypes = [vp, vp, C.c_int64, vp, vp]
        L.or_sigma_max.restype = C.c_double
        L.or_sigma_max.argtypes = [vp]
        L.or_update_sphere.restype = None
        L.or_update_sphere.argtypes = [vp, vp, vp]
        L.or_generate.restype = C.c_int64
        L.or_generate.argtypes = [C.c_int32, vp, vp, vp, vp, C.c_int32, vp, vp, vp, C.c_int32, C.c_uint32, vp, vp,
                                  C.c_float, C.c_uint32, vp, vp, vp]
        L.or_shade.restype = None
        L.or_shade.argtypes = [C.c_int32, vp, vp, vp, vp, C.c_int32, vp, vp, vp, C.c_int32, vp, vp]
        L.or_spawn.restype = C.c_int64
        L.or_spawn.argtypes = [C.c_int32, C.c_int32, C.c_uint32, vp, vp, vp, vp, vp, C.c_int64, vp, vp, vp, vp, vp, vp]
        L.or_backprop.restype = None
        L.or_backprop.argtypes = [C.c_int32, vp, vp, C.c_int32, vp, vp, vp, vp, vp]
        L.or_camera_rays.restype = None
        L.or_camera_rays.argtypes = [vp, C.c_int32, C.c_int32, vp]
        L.or_keys_given.restype = None
        L.or_keys_given.argtypes = [C.c_int64, vp, vp, vp, C.c_uint32, vp, vp]
        L.or_gbuffer.restype = None
        L.or_gbuffer.argtypes = [C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp]
        L.or_trim.restype = C.c_int64
        L.or_trim.argtypes = [C.c_int64, vp, vp, vp, vp, vp]
        L.or_compress.restype = C.c_int64
        L.or_compress.argtypes = [C.c_int64, vp, vp, vp, vp]
        L.or_sort_decompress.argtypes = [C.c_int64, vp, vp, vp, vp, vp, vp, vp]
        L.or_build_leaves.restype = C.c_int64
        L.or_build_leaves.argtypes = [C.c_int64, vp, C.c_int32, vp]
        L.or_build_upper.restype = C.c_int64
        L.or_build_upper.argtypes = [C.c_int64, vp, C.c_int32, vp]
        L.or_traverse.argtypes = [C.c_int32, C.c_int32, C.c_int32, vp, vp, C.c_int64, vp, vp, vp, C.c_int32, vp,
                                  vp, C.c_uint32, C.c_int32, vp, vp, vp, vp, C.c_int32, vp]
        L.or_cluster_spheres.restype = C.c_int64
        L.or_cluster_spheres.argtypes = [vp, vp, C.c_int32, C.c_int32, C.c_float, vp, vp, vp, vp]
        L.or_brute.argtypes = [C.c_int64, vp, C.c_int64, vp, C.c_int32, vp]
        L.or_mesh_cull.restype = None
        L.or_mesh_cull.argtypes = [C.c_int64, vp, C.c_int32, vp, vp, vp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(vp)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


# --------------------------------------------------------------------------
# building blocks

def atan2p(y: float, x: float) -> float:
    return float(lib().or_atan2p(y, x))


def sincos(phi: float):
    c, s = np.zeros(1, np.float32), np.zeros(1, np.float32)
    lib().or_sincos(phi, _p(c), _p(s))
    return float(c[0]), float(s[0])


def hash_shadow(light: int, d, zorder: bool = False) -> int:
    return int(lib().or_hash_shadow(light, _p(_f32(d)), int(zorder)))


def hash_bounce(o, d, box_min, box_ext, zorder: bool = False) -> int:
    return int(lib().or_hash_bounce(_p(_f32(o)), _p(_f32(d)), _p(_f32(box_min)), _p(_f32(box_ext)), int(zorder)))


def cone_grow(axis, phi, r):
    xo, po = np.zeros(3, np.float32), np.zeros(1, np.float32)
    lib().or_cone_grow(_p(_f32(axis)), phi, _p(_f32(r)), _p(xo), _p(po))
    return xo, float(po[0])


def cone_union(x1, p1, x2, p2):
    xo, po = np.zeros(3, np.float32), np.zeros(1, np.float32)
    lib().or_cone_union(_p(_f32(x1)), p1, _p(_f32(x2)), p2, _p(xo), _p(po))
    return xo, float(po[0])


def sphere_union(s1, s2):
    so = np.zeros(4, np.float32)
    lib().or_sphere_union(_p(_f32(s1)), _p(_f32(s2)), _p(so))
    return so


def cull(node8, sphere4) -> bool:
    return bool(lib().or_cull(_p(_f32(node8)), _p(_f32(sphere4))))


def mt(ray8, tri_e9):
    t = np.zeros(1, np.float32)
    hit = lib().or_mt(_p(_f32(ray8)), _p(_f32(tri_e9)), _p(t))
    return (float(t[0]) if hit else None)


def tri_sphere(verts9):
    out = np.zeros(4, np.float32)
    lib().or_tri_sphere(_p(_f32(verts9)), _p(out))
    return out


def miniball(points):
    pts = _f32(np.asarray(points).reshape(-1, 3))
    out = np.zeros(4, np.float32)
    rc = lib().or_miniball(_p(pts), pts.shape[0], _p(out))
    if rc != 0:
        raise ValueError("no points")
    return out


class ScenePrep:
    def __init__(self, tris, mesh_ids, pad=None, eps_t=None, mesh_sph=None, cluster_order=None):
        tris = _f32(tris).reshape(-1, 9)
        mesh_ids = np.ascontiguousarray(mesh_ids, np.int32)
        M = tris.shape[0]
        n_meshes = int(mesh_ids.max()) + 1 if M else 0
        self.M, self.n_meshes = M, n_meshes
        self.tri_e = np.zeros((M, 9), np.float32)
        self.tri_sph = np.zeros((M, 4), np.float32)
        self.mesh_sph = np.zeros((max(n_meshes, 1), 4), np.float32)
        self.mesh_range = np.zeros((max(n_meshes, 1), 2), np.int64)
        self.consts = np.zeros(8, np.float32)
        ms_in = _f32(mesh_sph).reshape(-1, 4) if mesh_sph is not None else None
        rc = lib().or_scene_prep(_p(tris), _p(mesh_ids), M, n_meshes, _p(self.tri_e), _p(self.tri_sph),
                                 _p(self.mesh_sph), _p(self.mesh_range), _p(self.consts),
                                 -1.0 if pad is None else float(pad), 0.0 if eps_t is None else float(eps_t),
                                 _p(ms_in) if ms_in is not None else None)
        if rc != 0:
            raise ValueError("mesh ids must be non-decreasing and dense from 0")
        # object sphere-tree clusters (NEXT-4, reading O1)
        self.cluster_sph = np.zeros((max(M, 1), 4), np.float32)
        self.mesh_cluster_first = np.zeros(max(n_meshes, 1) + 1, np.int64)
        self.cluster_order = np.zeros(max(M, 1), np.int32)
        oin = np.ascontiguousarray(cluster_order, np.int32) if cluster_order is not None else None
        nc = lib().or_cluster_spheres(_p(tris), _p(self.mesh_range), n_meshes, CLUSTER_TRIS, float(self.consts[6]),
                                      _p(oin) if oin is not None else None, _p(self.cluster_order),
                                      _p(self.cluster_sph), _p(self.mesh_cluster_first))
        self.cluster_sph = self.cluster_sph[:max(nc, 1)].copy()
        self.n_clusters = int(nc)
        self.box_min = self.consts[0:3].copy()
        self.box_max = self.consts[3:6].copy()
        self.box_ext = (self.box_max - self.box_min).astype(np.float32)
        self.pad = float(self.consts[6])
        self.eps_t = float(self.consts[7])


def num_slots(P: int, n_lights: int, types: int) -> int:
    return P * ((n_lights if types & SH else 0) + (1 if types & RE else 0) + (1 if types & RR else 0))


def segments(P: int, n_lights: int, types: int):
    """[(seg_id, first_slot, n_slots)] with seg 0 = SH (all lights), 1 = RE, 2 = RR (R5)."""
    out, s = [], 0
    if types & SH:
        out.append((0, s, P * n_lights)); s += P * n_lights
    if types & RE:
        out.append((1, s, P)); s += P
    if types & RR:
        out.append((2, s, P)); s += P
    return out


def generate(w, prep: ScenePrep, flags: int = 0):
    P, L = w.P, w.lights.shape[0]
    S = num_slots(P, L, w.ray_types)
    rays = np.zeros((S, 8), np.float32)
    keys = np.zeros(S, np.uint32)
    empty = np.zeros(S, np.uint32)
    lib().or_generate(P, _p(_f32(w.pos)), _p(_f32(w.nrm)), _p(np.ascontiguousarray(w.mat, np.int32)),
                      _p(_f32(w.materials)), w.materials.shape[0], _p(_f32(w.eye)),
                      _p(_f32(w.dir)) if getattr(w, "dir", None) is not None else None, _p(_f32(w.lights)), L,
                      w.ray_types, _p(prep.box_min), _p(prep.box_ext), prep.eps_t, flags, _p(rays), _p(keys), _p(empty))
    return rays, keys, empty


def trim(empty, keys, vals):
    n = len(keys)
    ko = np.zeros(n, np.uint32)
    vo = np.zeros(n, np.uint32)
    k = lib().or_trim(n, _p(np.ascontiguousarray(empty, np.uint32)), _p(np.ascontiguousarray(keys, np.uint32)),
                      _p(np.ascontiguousarray(vals, np.uint32)), _p(ko), _p(vo))
    if k < 0:
        raise ValueError("flag value other than 0/1")
    return ko[:k], vo[:k]


def compress(keys):
    keys = np.ascontiguousarray(keys, np.uint32)
    n = len(keys)
    ck, cb, cs = (np.zeros(max(n, 1), np.uint32) for _ in range(3))
    C = lib().or_compress(n, _p(keys), _p(ck), _p(cb), _p(cs))
    return ck[:C], cb[:C], cs[:C]


def sort_decompress(ckey, cbase, csize, vals):
    C = len(ckey)
    n = int(np.asarray(csize, np.uint64).sum())
    sk, sv = np.zeros(max(n, 1), np.uint32), np.zeros(max(n, 1), np.uint32)
    sc = np.zeros(max(C, 1), np.uint32)
    lib().or_sort_decompress(C, _p(np.ascontiguousarray(ckey, np.uint32)), _p(np.ascontiguousarray(cbase, np.uint32)),
                             _p(np.ascontiguousarray(csize, np.uint32)), _p(np.ascontiguousarray(vals, np.uint32)),
                             _p(sk), _p(sv), _p(sc))
    return sk[:n], sv[:n], sc[:C]


def build_levels(sorted_rays, Lv, B0, B):
    """Per-level node arrays [level 1 (leaves), ..., level Lv (top)]."""
    n = sorted_rays.shape[0]
    levels = []
    leaves = np.zeros(((n + B0 - 1) // B0, 8), np.float32)
    lib().or_build_leaves(n, _p(_f32(sorted_rays)), B0, _p(leaves))
    levels.append(leaves)
    for _ in range(1, Lv):
        ch = levels[-1]
        up = np.zeros(((ch.shape[0] + B - 1) // B, 8), np.float32)
        lib().or_build_upper(ch.shape[0], _p(ch), B, _p(up))
        levels.append(up)
    return levels


def traverse(levels, sorted_rays, prep: ScenePrep, Lv, B0, B, flags, n_threads=None):
    n = sorted_rays.shape[0]
    best = np.full(max(n, 1), UINT64_MAX, np.uint64)
    cnt = np.zeros(22, np.uint64)
    if n == 0:
        return best[:0], cnt
    ptrs = (vp * Lv)(*[lv.ctypes.data_as(vp) for lv in levels])
    counts = np.array([lv.shape[0] for lv in levels], np.int64)
    lib().or_traverse(Lv, B0, B, ptrs, _p(counts), n, _p(_f32(sorted_rays)), _p(prep.tri_e), _p(prep.tri_sph),
                      prep.n_meshes, _p(prep.mesh_sph), _p(prep.mesh_range), flags,
                      n_threads or default_threads(), _p(best), _p(cnt), _p(prep.cluster_sph),
                      _p(prep.mesh_cluster_first), CLUSTER_TRIS, _p(prep.cluster_order))
    return best[:n], cnt


def brute(rays, prep: ScenePrep, n_threads=None):
    rays = _f32(rays).reshape(-1, 8)
    best = np.full(max(rays.shape[0], 1), UINT64_MAX, np.uint64)
    lib().or_brute(rays.shape[0], _p(rays), prep.M, _p(prep.tri_e), n_threads or default_threads(), _p(best))
    return best[:rays.shape[0]]


def unpack(best):
    """packed (t bits << 32 | tri) -> (hit_tri int32, t float32); UINT64_MAX -> (-1, +inf)."""
    best = np.asarray(best, np.uint64)
    miss = best == UINT64_MAX
    tri = (best & np.uint64(0xFFFFFFFF)).astype(np.int64)
    t = (best >> np.uint64(32)).astype(np.uint32).view(np.float32).copy()
    tri[miss] = -1
    t[miss] = np.inf
    return tri.astype(np.int32), t


# --------------------------------------------------------------------------
# the whole per-frame path, stage by stage

def trace(w, prep: ScenePrep | None = None, flags: int = F_SORT | F_MESH_CULL, n_threads=None, taps=False):
    """Returns dict(hit_tri[slots], t[slots], stats, [taps]).  hit_tri = -2 for
    an empty slot, -1 for a miss (SURVEY §8(c) output convention)."""
    prep = prep or ScenePrep(w.tris, w.mesh_ids)
    rays, keys, empty = generate(w, prep, flags)
    return _trace_core(rays, keys, empty, segments(w.P, w.lights.shape[0], w.ray_types), prep, w.levels, w.leaf_size,
                       w.branching, flags, n_threads, taps)


def trace_rays(rays, prep: ScenePrep, levels=2, leaf_size=8, branching=8, flags: int = F_SORT | F_MESH_CULL,
               n_threads=None, taps=False):
    """A given ray batch ([n, 8]: o, tmin, d, tmax) through the same stages
    (crsh_trace_rays): bounce-ray hash keys, one segment reported as 1."""
    rays = _f32(rays).reshape(-1, 8)
    n = rays.shape[0]
    keys = np.zeros(n, np.uint32)
    empty = np.zeros(n, np.uint32)
    lib().or_keys_given(n, _p(rays), _p(prep.box_min), _p(prep.box_ext), flags, _p(keys), _p(empty))
    return _trace_core(rays, keys, empty, [(1, 0, n)], prep, levels, leaf_size, branching, flags, n_threads, taps)


def camera_rays(cam13, W: int, H: int):
    rays = np.zeros((W * H, 8), np.float32)
    lib().or_camera_rays(_p(_f32(cam13)), W, H, _p(rays))
    return rays


def primary_gbuffer(tris, mesh_ids, tri_mat, cam13, W: int, H: int, levels=2, leaf_size=8, branching=8,
                    flags: int = F_SORT | F_MESH_CULL, prep: ScenePrep | None = None):
    """GPU primary pass mirror (NEXT-3): camera rays traced with the pipeline,
    then the G-buffer of the closest hits. Returns (pos[3,P], nrm[3,P],
    mat[P], hit_tri[P], t[P], stats)."""
    prep = prep or ScenePrep(tris, mesh_ids)
    rays = camera_rays(cam13, W, H)
    out = trace_rays(rays, prep, levels, leaf_size, branching, flags)
    P = W * H
    pos, nrm = np.zeros((3, P), np.float32), np.zeros((3, P), np.float32)
    mat = np.zeros(P, np.int32)
    lib().or_gbuffer(P, _p(rays), _p(np.ascontiguousarray(out["hit_tri"], np.int32)),
                     _p(np.ascontiguousarray(out["t"], np.float32)), _p(prep.tri_e),
                     _p(np.ascontiguousarray(tri_mat, np.int32)), _p(pos), _p(nrm), _p(mat))
    return pos, nrm, mat, out["hit_tri"], out["t"], out["stats"]


def mesh_cull(top_nodes, prep: ScenePrep):
    """The whole-mesh cull alone (a9) over the given top nodes of the
    ORACLE's hierarchy: (mesh tests, mesh passes, triangles of the passing
    meshes = the top-level test count of the traversal)."""
    top = _f32(top_nodes).reshape(-1, 8)
    out = np.zeros(3, np.uint64)
    lib().or_mesh_cull(top.shape[0], _p(top), prep.n_meshes, _p(prep.mesh_sph), _p(prep.mesh_range), _p(out))
    return int(out[0]), int(out[1]), int(out[2])


def top_level_counts(w, prep: ScenePrep | None = None, flags: int = F_SORT | F_MESH_CULL):
    """Per segment (0 = SH, 1 = RE, 2 = RR): the oracle's own generate -> trim
    -> sort -> build up to the top level, then the whole-mesh cull of its top
    nodes; returns {seg: (rays, n_top, mesh_tests, mesh_hits, top_level_tests)}.
    Checks the counts that do not need the (expensive) descent, at sizes where
    the full oracle traversal takes too long."""
    prep = prep or ScenePrep(w.tris, w.mesh_ids)
    rays, keys, empty = generate(w, prep, flags)
    S = rays.shape[0]
    keys_c, vals_c = trim(empty, keys, np.arange(S, dtype=np.uint32))
    out = {}
    for seg, s0, ns in segments(w.P, w.lights.shape[0], w.ray_types):
        sel = (vals_c >= s0) & (vals_c < s0 + ns)
        k, v = keys_c[sel], vals_c[sel]
        if len(k) == 0:
            out[seg] = (0, 0, 0, 0, 0)
            continue
        if flags & F_SORT:
            ck, cb, cs = compress(k)
            _, v, _ = sort_decompress(ck, cb, cs, v)
        levels = build_levels(rays[v.astype(np.int64)], w.levels, w.leaf_size, w.branching)
        out[seg] = (len(k), levels[-1].shape[0], *mesh_cull(levels[-1], prep))
    return out


def _trace_core(rays, keys, empty, segs, prep: ScenePrep, Lv, B0, B, flags, n_threads, taps):
    S = rays.shape[0]
    hit_tri = np.full(S, -2, np.int32)
    t_out = np.full(S, np.inf, np.float32)
    stats = dict(rays=[0, 0, 0], slots=[0, 0, 0], chunks=[0, 0, 0], tests=np.zeros((3, 9), np.uint64),
                 hits=np.zeros((3, 9), np.uint64), mesh_tests=[0, 0, 0], mesh_hits=[0, 0, 0],
                 final_tests=[0, 0, 0], final_hits=[0, 0, 0], rays_hit=[0, 0, 0], brute=[0, 0, 0],
                 cluster_tests=[0, 0, 0], cluster_hits=[0, 0, 0])
    tap = dict(keys=[], vals=[], ckey=[], cbase=[], skey=[], sslot=[], levels=[])
    # trimming over the whole slot array keeps slot order, so each
    # segment's survivors stay contiguous.
    keys_c, vals_c = trim(empty, keys, np.arange(S, dtype=np.uint32))
    for seg, s0, ns in segs:
        sel = (vals_c >= s0) & (vals_c < s0 + ns)
        k, v = keys_c[sel], vals_c[sel]
        stats["slots"][seg] = ns
        stats["rays"][seg] = len(k)
        if flags & F_SORT:
            ck, cb, cs = compress(k)
            sk, sv, _ = sort_decompress(ck, cb, cs, v)
            stats["chunks"][seg] = len(ck)
        else:   # RAH: rays stay in generation order
            ck, cb = np.zeros(0, np.uint32), np.zeros(0, np.uint32)
            sk, sv = k, v
        sr = rays[sv.astype(np.int64)]
        stats["brute"][seg] = len(k) * prep.M
        if taps:
            tap["keys"].append(k); tap["vals"].append(v); tap["ckey"].append(ck); tap["cbase"].append(cb)
            tap["skey"].append(sk); tap["sslot"].append(sv)
        if len(k) == 0:
            if taps:
                tap["levels"].append([np.zeros((0, 8), np.float32) for _ in range(Lv)])
            continue
        levels = build_levels(sr, Lv, B0, B)
        if taps:
            tap["levels"].append(levels)
        best, cnt = traverse(levels, sr, prep, Lv, B0, B, flags, n_threads)
        for kk in range(Lv):
            stats["tests"][seg, kk + 1] = cnt[kk]
            stats["hits"][seg, kk + 1] = cnt[8 + kk]
        stats["mesh_tests"][seg], stats["mesh_hits"][seg] = int(cnt[16]), int(cnt[17])
        stats["final_tests"][seg], stats["final_hits"][seg] = int(cnt[18]), int(cnt[19])
        stats["cluster_tests"][seg], stats["cluster_hits"][seg] = int(cnt[20]), int(cnt[21])
        tri, tt = unpack(best)
        hit_tri[sv.astype(np.int64)] = tri
        t_out[sv.astype(np.int64)] = tt
        stats["rays_hit"][seg] = int((tri >= 0).sum())
    out = dict(hit_tri=hit_tri, t=t_out, stats=stats, rays=rays, empty=empty, keys=keys)
    if taps:
        out["taps"] = tap
    return out


# --------------------------------------------------------------------------
# multi-bounce Whitted loop

def whitted(w, depth: int, prep: ScenePrep | None = None, flags: int = F_SORT | F_MESH_CULL, n_threads=None):
    """Radiance per pixel after `depth` reflection/refraction bounces.
    Bounce d traces the vertex set V_d (V_0 = the G-buffer) with the secondary
    pass -- shadow rays for the direct term, RE/RR rays while d < depth -- the
    RE/RR closest hits become V_{d+1}, and L(v) = direct(v) + refl L(re child)
    + trans L(rr child) is assembled from the deepest bounce up (or_shade,
    or_spawn, or_backprop in oracle.cpp). Returns dict(image[P], vertices[d],
    rays[d], stats[d])."""
    import dataclasses
    prep = prep or ScenePrep(w.tris, w.mesh_ids)
    tri_mat = np.ascontiguousarray(w.tri_mat, np.int32)
    L = w.lights.shape[0]
    mats = _f32(w.materials)
    n_mat = mats.shape[0]
    cur = dict(P=w.P, pos=_f32(w.pos).reshape(3, -1), nrm=_f32(w.nrm).reshape(3, -1),
               mat=np.ascontiguousarray(w.mat, np.int32).reshape(-1), dir=None)
    per = []   # (mat, direct, c_re, c_rr) per bounce
    verts, nrays, stats = [], [], []
    for d in range(depth + 1):
        P = cur["P"]
        verts.append(P)
        types = (SH if L > 0 else 0) | ((RE | RR) if d < depth else 0)
        if P == 0 or types == 0:
            per.append((cur["mat"], np.zeros(P, np.float32), None, None))
            nrays.append(0); stats.append(None)
            break
        wd = dataclasses.replace(w, width=P, height=1, pos=cur["pos"], nrm=cur["nrm"], mat=cur["mat"],
                                 dir=cur["dir"], ray_types=types)
        out = trace(wd, prep, flags=flags, n_threads=n_threads)
        nrays.append(int(sum(out["stats"]["rays"])))
        stats.append(out["stats"])
        hit = np.ascontiguousarray(out["hit_tri"], np.int32)
        direct = np.zeros(P, np.float32)
        dirp = _p(cur["dir"]) if cur["dir"] is not None else None
        if types & SH:
            lib().or_shade(P, _p(cur["pos"]), _p(cur["nrm"]), _p(cur["mat"]), _p(mats), n_mat, _p(_f32(w.eye)), dirp,
                           _p(_f32(w.lights)), L, _p(hit), _p(direct))
        if d == depth:
            per.append((cur["mat"], direct, None, None))
            break
        cap = 2 * P
        npos, nnrm, ndir = (np.zeros((3, max(cap, 1)), np.float32) for _ in range(3))
        nmat = np.zeros(max(cap, 1), np.int32)
        c_re, c_rr = np.zeros(P, np.int32), np.zeros(P, np.int32)
        k = lib().or_spawn(P, L, types, _p(_f32(out["rays"])), _p(hit), _p(np.ascontiguousarray(out["t"], np.float32)),
                           _p(prep.tri_e), _p(tri_mat), cap, _p(npos), _p(nnrm), _p(nmat), _p(ndir), _p(c_re),
                           _p(c_rr))
        per.append((cur["mat"], direct, c_re, c_rr))
        # or_spawn writes SoA planes of stride k into the front of each buffer
        cur = dict(P=int(k), pos=npos.reshape(-1)[:3 * k].reshape(3, k).copy(),
                   nrm=nnrm.reshape(-1)[:3 * k].reshape(3, k).copy(), mat=nmat[:k].copy(),
                   dir=ndir.reshape(-1)[:3 * k].reshape(3, k).copy())
    # radiance, deepest bounce first
    Lnext = np.zeros(1, np.float32)
    for mat, direct, c_re, c_rr in reversed(per):
        P = len(direct)
        Lcur = np.zeros(max(P, 1), np.float32)
        if P:
            lib().or_backprop(P, _p(np.ascontiguousarray(mat, np.int32)), _p(mats), n_mat, _p(direct),
                              _p(c_re) if c_re is not None else None, _p(c_rr) if c_rr is not None else None,
                              _p(Lnext), _p(Lcur))
        Lnext = Lcur
    return dict(image=Lnext[:w.P].copy(), vertices=verts, rays=nrays, stats=stats)


# --------------------------------------------------------------------------
# dynamic scenes (§3.3.1)

def transform_tris(tris, mesh_ids, xforms):
    """creation-time vertices -> per-mesh affine transform ([n_meshes, 12] =
    [A | b] row-major), per axis fma(a0, x, fma(a1, y, fma(a2, z, b)))."""
    tris = _f32(tris).reshape(-1, 9)
    out = np.zeros_like(tris)
    lib().or_transform(_p(tris), _p(np.ascontiguousarray(mesh_ids, np.int32)), tris.shape[0],
                       _p(_f32(xforms).reshape(-1, 12)), _p(out))
    return out


def sigma_max(xf12) -> float:
    return float(lib().or_sigma_max(_p(_f32(xf12))))


def update_sphere(sph4, xf12):
    out = np.zeros(4, np.float32)
    lib().or_update_sphere(_p(_f32(sph4)), _p(_f32(xf12)), _p(out))
    return out


def transformed_prep(prep0: ScenePrep, tris0, mesh_ids, xforms):
    """The scene after crsh_scene_transform: transformed vertices, triangle
    data recomputed with the creation pad, mesh spheres UPDATED from the
    creation spheres (not recomputed), AABB of the transformed vertices,
    creation eps_t. Returns (prep, transformed tris)."""
    xforms = _f32(xforms).reshape(-1, 12)
    tris = transform_tris(tris0, mesh_ids, xforms)
    ms = np.stack([update_sphere(prep0.mesh_sph[m], xforms[m]) for m in range(prep0.n_meshes)]) \
        if prep0.n_meshes else np.zeros((1, 4), np.float32)
    return ScenePrep(tris, mesh_ids, pad=prep0.pad, eps_t=prep0.eps_t, mesh_sph=ms,
                     cluster_order=prep0.cluster_order), tris
