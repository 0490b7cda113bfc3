"""B200-native Coherent Ray-Space Hierarchy (CRSH) secondary-ray path
(Reis, Costa & Pereira, arXiv 2312.06538).

Thin Python binding over the C ABI of ``libcrsh.so`` (include/crsh.h): the
functions below have the C names without the ``crsh_`` prefix and do
argument marshalling only -- every step of the path runs in the library's
sm_100a kernels.  PyTorch provides device memory (``tensor.data_ptr()``) and
streams; there is no CPU fallback: if the library cannot be loaded, or no
CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CRSH_LIB_PATH") or os.path.join(HERE, "libcrsh.so")   # override: A/B experiments
HEADER = os.path.join(os.path.dirname(HERE), "include", "crsh.h")

SHADOW, REFLECT, REFRACT = 1, 2, 4
F_SORT, F_MESH_CULL, F_ZORDER, F_STAGE_TIMING, F_BRUTE, F_KERNEL_TIMING, F_OBJTREE = 1, 2, 4, 8, 16, 32, 64
TAP_KEYS, TAP_VALS, TAP_CHUNK_KEYS, TAP_CHUNK_BASE, TAP_SORTED_KEYS, TAP_SORTED_SLOTS = 1, 2, 3, 4, 5, 6
TAP_NODES, TAP_SORTED_RAYS, TAP_TRI_SPHERES, TAP_MESH_SPHERES, TAP_SCENE_CONSTS = 7, 8, 9, 10, 11
TAP_GROUP_RANGE, TAP_GROUP_WORK, TAP_CLUSTER_SPHERES, TAP_CLUSTER_ORDER = 12, 13, 14, 15
STATUS = {0: "OK", 2: "EINVAL", 3: "EIO", 4: "ELIMIT", 5: "ENOMEM", 6: "ECUDA", 7: "ENCCL"}
MERGE = {0: "none", 1: "nccl-allreduce-min", 2: "fused-peer-stores"}
STAGES = ["generate+trim", "compress", "sort", "decompress", "build", "mesh-cull+plan", "traverse+final", "output"]


class CrshError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"crsh status {STATUS.get(status, status)}: {msg}")
        self.status = status


class PrimaryHits(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("pos", C.c_void_p), ("nrm", C.c_void_p),
                ("mat", C.c_void_p), ("materials", C.c_void_p), ("n_mat", C.c_int32), ("eye", C.c_float * 3),
                ("dir", C.c_void_p)]


class WhittedStats(C.Structure):
    _fields_ = [("bounces", C.c_int32), ("reserved", C.c_int32), ("vertices", C.c_int64 * 9), ("rays", C.c_int64 * 9),
                ("tests", C.c_uint64 * 9), ("final_tests", C.c_uint64 * 9)]


class Camera(C.Structure):
    _fields_ = [("eye", C.c_float * 3), ("right", C.c_float * 3), ("up", C.c_float * 3), ("fwd", C.c_float * 3),
                ("tan_half_vfov", C.c_float)]


def make_camera(cam13) -> Camera:
    """crsh_camera from 13 floats: eye, right, up, fwd, tan(vfov/2)."""
    c = Camera()
    v = [float(x) for x in cam13]
    c.eye = (C.c_float * 3)(*v[0:3]); c.right = (C.c_float * 3)(*v[3:6])
    c.up = (C.c_float * 3)(*v[6:9]); c.fwd = (C.c_float * 3)(*v[9:12]); c.tan_half_vfov = v[12]
    return c


class Opts(C.Structure):
    _fields_ = [("levels", C.c_int32), ("leaf_size", C.c_int32), ("branching", C.c_int32), ("flags", C.c_uint32),
                ("shard_rank", C.c_int32), ("shard_world", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("rays", C.c_uint64 * 3), ("slots", C.c_uint64 * 3), ("chunks", C.c_uint64 * 3),
                ("mesh_tests", C.c_uint64 * 3), ("mesh_hits", C.c_uint64 * 3),
                ("tests", (C.c_uint64 * 9) * 3), ("hits", (C.c_uint64 * 9) * 3),
                ("final_tests", C.c_uint64 * 3), ("final_hits", C.c_uint64 * 3), ("rays_hit", C.c_uint64 * 3),
                ("brute", C.c_uint64 * 3), ("levels", C.c_int32), ("merge", C.c_int32),
                ("stage_ms", C.c_float * 8), ("cluster_tests", C.c_uint64 * 3), ("cluster_hits", C.c_uint64 * 3),
                ("skipped_tests", C.c_uint64 * 3), ("prefilter_tests", C.c_uint64 * 3)]


_lib = None


def load():
    """Load libcrsh.so (fails loudly: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() (nvcc, sm_100a)")
    L = C.CDLL(LIB_PATH)
    vp, st = C.c_void_p, C.c_int
    L.crsh_last_error.restype = C.c_char_p
    L.crsh_num_slots.restype = C.c_int64
    L.crsh_num_slots.argtypes = [C.c_int32, C.c_int32, C.c_uint32]
    L.crsh_scene_create.restype = st
    L.crsh_scene_create.argtypes = [vp, vp, C.c_int64, C.c_int32, C.POINTER(vp)]
    L.crsh_scene_destroy.argtypes = [vp]
    L.crsh_scene_destroy.restype = None
    for name in ("crsh_trace_secondary", "crsh_trace_secondary_host"):
        f = getattr(L, name)
        f.restype = st
        f.argtypes = [vp, C.POINTER(PrimaryHits), vp, C.c_int32, C.c_uint32, C.POINTER(Opts), vp, vp, vp]
    L.crsh_trace_secondary_packed.restype = st
    L.crsh_trace_secondary_packed.argtypes = [vp, C.POINTER(PrimaryHits), vp, C.c_int32, C.c_uint32,
                                              C.POINTER(Opts), vp, vp]
    L.crsh_trace_secondary_peer.restype = st
    L.crsh_trace_secondary_peer.argtypes = [vp, C.POINTER(PrimaryHits), vp, C.c_int32, C.c_uint32, C.POINTER(Opts),
                                            C.POINTER(C.c_uint64), C.c_int32, vp]
    L.crsh_scene_transform.restype = st
    L.crsh_scene_transform.argtypes = [vp, vp]
    L.crsh_trace_rays.restype = st
    L.crsh_trace_rays.argtypes = [vp, vp, C.c_int64, C.POINTER(Opts), vp, vp, vp]
    L.crsh_primary_gbuffer.restype = st
    L.crsh_primary_gbuffer.argtypes = [vp, C.POINTER(Camera), C.c_int32, C.c_int32, vp, C.POINTER(Opts), vp, vp, vp,
                                       vp, vp, vp]
    L.crsh_render_whitted.restype = st
    L.crsh_render_whitted.argtypes = [vp, C.POINTER(PrimaryHits), vp, C.c_int32, vp, C.c_int32, C.POINTER(Opts), vp,
                                      C.POINTER(WhittedStats), vp]
    L.crsh_unpack_hits.restype = st
    L.crsh_unpack_hits.argtypes = [vp, vp, C.c_int64, vp, vp, vp]
    L.crsh_stats.restype = st
    L.crsh_stats.argtypes = [vp, C.POINTER(Stats)]
    L.crsh_launch_count.restype = C.c_int64
    L.crsh_launch_count.argtypes = [vp]
    L.crsh_dist_unique_id.restype = st
    L.crsh_dist_unique_id.argtypes = [vp]
    L.crsh_dist_init.restype = st
    L.crsh_dist_init.argtypes = [vp, vp, C.c_int32, C.c_int32]
    L.crsh_debug_tap.restype = st
    L.crsh_debug_tap.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, vp, C.c_size_t, C.POINTER(C.c_size_t)]
    _lib = L
    return L


def _check(rc: int):
    if rc != 0:
        raise CrshError(rc, load().crsh_last_error().decode())


def num_slots(P: int, n_lights: int, ray_types: int) -> int:
    return int(load().crsh_num_slots(P, n_lights, ray_types))


def _ptr(t) -> int:
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        assert t.is_contiguous()
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        assert t.flags.c_contiguous
        return t.ctypes.data
    return int(t)


class Scene:
    """crsh_scene_create / crsh_scene_destroy. tris: device float32 [M, 9];
    mesh_ids: device int32 [M] (torch tensors or raw device pointers)."""

    def __init__(self, tris, mesh_ids, device: int = 0, M: int | None = None):
        L = load()
        h = C.c_void_p()
        M = M if M is not None else int(tris.shape[0])
        _check(L.crsh_scene_create(_ptr(tris), _ptr(mesh_ids), M, device, C.byref(h)))
        self.handle = h.value
        self.M = M
        self.device = device

    def close(self):
        if getattr(self, "handle", None):
            load().crsh_scene_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_hits(width, height, pos, nrm, mat, materials, n_mat, eye, dir=None) -> PrimaryHits:
    h = PrimaryHits()
    h.width, h.height = width, height
    h.pos, h.nrm, h.mat, h.materials = _ptr(pos), _ptr(nrm), _ptr(mat), _ptr(materials)
    h.n_mat = n_mat
    h.eye = (C.c_float * 3)(*[float(x) for x in eye])
    h.dir = _ptr(dir) if dir is not None else None
    return h


def make_opts(levels=2, leaf_size=8, branching=8, flags=F_SORT | F_MESH_CULL, shard_rank=0, shard_world=1) -> Opts:
    o = Opts()
    o.levels, o.leaf_size, o.branching, o.flags = levels, leaf_size, branching, flags
    o.shard_rank, o.shard_world = shard_rank, shard_world
    return o


def _lights(lights):
    arr = np.ascontiguousarray(np.asarray(lights, np.float32).reshape(-1, 3))
    return arr, arr.shape[0]


def trace_secondary(scene: Scene, hits: PrimaryHits, lights, ray_types: int, opts: Opts, hit_tri, t, stream=0):
    """crsh_trace_secondary: device G-buffer in `hits`, outputs hit_tri (int32)
    and t (float32) device [slots]; stream = cudaStream_t handle (int)."""
    arr, n = _lights(lights)
    _check(load().crsh_trace_secondary(scene.handle, C.byref(hits), arr.ctypes.data, n, ray_types, C.byref(opts),
                                       _ptr(hit_tri), _ptr(t), stream))


def trace_secondary_packed(scene: Scene, hits: PrimaryHits, lights, ray_types: int, opts: Opts, packed, stream=0):
    arr, n = _lights(lights)
    _check(load().crsh_trace_secondary_packed(scene.handle, C.byref(hits), arr.ctypes.data, n, ray_types,
                                              C.byref(opts), _ptr(packed), stream))


def trace_secondary_peer(scene: Scene, hits: PrimaryHits, lights, ray_types: int, opts: Opts, dst_ptrs, stream=0):
    """crsh_trace_secondary_peer: dst_ptrs = device addresses (ints) of the
    packed destination buffers (own + peers')."""
    arr, n = _lights(lights)
    d = (C.c_uint64 * len(dst_ptrs))(*[int(x) for x in dst_ptrs])
    _check(load().crsh_trace_secondary_peer(scene.handle, C.byref(hits), arr.ctypes.data, n, ray_types,
                                            C.byref(opts), d, len(dst_ptrs), stream))


def scene_transform(scene: Scene, xforms):
    """crsh_scene_transform: host [n_meshes, 12] float32 affine [A | b] per mesh,
    applied to the creation-time vertices."""
    x = np.ascontiguousarray(np.asarray(xforms, np.float32).reshape(-1, 12))
    _check(load().crsh_scene_transform(scene.handle, x.ctypes.data))


def trace_rays(scene: Scene, rays, n: int, opts: Opts, hit_tri, t, stream=0):
    """crsh_trace_rays: device rays [n][8] (o, tmin, d, tmax) -> hit_tri, t."""
    _check(load().crsh_trace_rays(scene.handle, _ptr(rays), n, C.byref(opts), _ptr(hit_tri), _ptr(t), stream))


def primary_gbuffer(scene: Scene, cam13, width: int, height: int, tri_mat, opts: Opts, pos, nrm, mat, hit_tri, t,
                    stream=0):
    """crsh_primary_gbuffer: the GPU primary pass into device G-buffer tensors."""
    c = make_camera(cam13)
    _check(load().crsh_primary_gbuffer(scene.handle, C.byref(c), width, height, _ptr(tri_mat), C.byref(opts),
                                       _ptr(pos), _ptr(nrm), _ptr(mat), _ptr(hit_tri), _ptr(t), stream))


def render_whitted(scene: Scene, hits: PrimaryHits, lights, tri_mat, depth: int, opts: Opts, image, stream=0) -> dict:
    """crsh_render_whitted: radiance per pixel after `depth` bounces into the
    device buffer `image` [P] float32; returns the per-bounce stats."""
    arr, n = _lights(lights)
    ws = WhittedStats()
    _check(load().crsh_render_whitted(scene.handle, C.byref(hits), arr.ctypes.data, n, _ptr(tri_mat), depth,
                                      C.byref(opts), _ptr(image), C.byref(ws), stream))
    d = ws.bounces
    return dict(vertices=list(ws.vertices)[:d + 1], rays=list(ws.rays)[:d + 1], tests=list(ws.tests)[:d + 1],
                final_tests=list(ws.final_tests)[:d + 1])


def unpack_hits(scene: Scene, packed, slots: int, hit_tri, t, stream=0):
    _check(load().crsh_unpack_hits(scene.handle, _ptr(packed), slots, _ptr(hit_tri), _ptr(t), stream))


def trace_secondary_host(scene: Scene, hits: PrimaryHits, lights, ray_types: int, opts: Opts, hit_tri: np.ndarray,
                         t: np.ndarray, stream=0):
    """crsh_trace_secondary_host: `hits` and the outputs are HOST buffers."""
    arr, n = _lights(lights)
    _check(load().crsh_trace_secondary_host(scene.handle, C.byref(hits), arr.ctypes.data, n, ray_types,
                                            C.byref(opts), _ptr(hit_tri), _ptr(t), stream))


def stats(scene: Scene) -> dict:
    s = Stats()
    _check(load().crsh_stats(scene.handle, C.byref(s)))
    return dict(rays=list(s.rays), slots=list(s.slots), chunks=list(s.chunks), mesh_tests=list(s.mesh_tests),
                mesh_hits=list(s.mesh_hits), tests=np.array([list(r) for r in s.tests], np.uint64),
                hits=np.array([list(r) for r in s.hits], np.uint64), final_tests=list(s.final_tests),
                final_hits=list(s.final_hits), rays_hit=list(s.rays_hit), brute=list(s.brute), levels=s.levels,
                merge=s.merge, stage_ms=list(s.stage_ms), cluster_tests=list(s.cluster_tests),
                cluster_hits=list(s.cluster_hits), skipped_tests=list(s.skipped_tests),
                prefilter_tests=list(s.prefilter_tests))


def launch_count(scene: Scene) -> int:
    return int(load().crsh_launch_count(scene.handle))


_TAP_DTYPE = {TAP_NODES: (np.float32, 8), TAP_SORTED_RAYS: (np.float32, 8), TAP_TRI_SPHERES: (np.float32, 4),
              TAP_MESH_SPHERES: (np.float32, 4), TAP_SCENE_CONSTS: (np.float32, 1), TAP_GROUP_WORK: (np.uint64, 1),
              TAP_CLUSTER_SPHERES: (np.float32, 4), TAP_CLUSTER_ORDER: (np.int32, 1)}


def debug_tap(scene: Scene, tap: int, segment: int = 0, level: int = 1) -> np.ndarray:
    dt, width = _TAP_DTYPE.get(tap, (np.uint32, 1))
    n = C.c_size_t(0)
    L = load()
    rc = L.crsh_debug_tap(scene.handle, tap, segment, level, None, 0, C.byref(n))
    if rc not in (0, 3):
        _check(rc)
    out = np.zeros((max(n.value, 1), width), dt)
    _check(L.crsh_debug_tap(scene.handle, tap, segment, level, out.ctypes.data, out.nbytes, C.byref(n)))
    out = out[:n.value]
    return out.reshape(-1) if width == 1 else out


def header_functions() -> list[str]:
    """Names of the functions include/crsh.h declares (for the ABI test)."""
    import re
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(crsh_[a-z_]+)\s*\(", src)))
