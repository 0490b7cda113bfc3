"""Seeded procedural scenes and G-buffers shaped like the paper's test scenes.

INPUT GENERATOR shared by the oracle and the CUDA path. It holds none of the
method's arithmetic: it only emits triangles, materials, lights, a camera and
the rasterised G-buffer (paper §3.2, done by ``raster.c``).

Scene families (§4.2):
  * Cornell-like room  -- "an object surrounded by six mirrors":
    a closed room [0,10]^3 of tessellated walls, two of them mirrors, plus
    interior objects.
  * Office-like multi-mesh room -- "divided into several submeshes"
    (PAPER.md:203): room shell + K objects (UV spheres, boxes, tori,
    cylinders), each its own mesh, placed by seeded rejection sampling on
    their bounding spheres.
Materials per object mesh (seeded): 60% diffuse, 25% mirror (reflectivity
0.8), 15% glass (transmissivity 0.9, ior 1.5).  Camera: eye (5,5,0.5) looking
+z, 60 deg vertical fov, inside the closed room (100% pixel coverage).  Lights
near the ceiling.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libraster.so")

# material table rows: (reflectivity, transmissivity, ior)
MATERIALS = np.array([[0.0, 0.0, 1.0],    # 0 diffuse
                      [0.8, 0.0, 1.0],    # 1 mirror
                      [0.0, 0.9, 1.5]],   # 2 glass
                     dtype=np.float32)
DIFFUSE, MIRROR, GLASS = 0, 1, 2

EYE = (5.0, 5.0, 0.5)
FWD = (0.0, 0.0, 1.0)
UP = (0.0, 1.0, 0.0)
VFOV = 60.0
LIGHTS = [(5.0, 9.5, 5.0), (2.5, 9.5, 7.5), (7.5, 9.5, 2.5), (7.5, 9.5, 7.5),
          (2.5, 9.5, 2.5), (5.0, 9.5, 8.5), (5.0, 9.5, 1.5), (8.5, 9.5, 5.0)]


@dataclass
class Workload:
    name: str
    tris: np.ndarray          # [M, 9] float32: v0, v1, v2
    mesh_ids: np.ndarray      # [M] int32, non-decreasing, dense from 0
    tri_mat: np.ndarray       # [M] int32 material of each triangle
    materials: np.ndarray     # [n_mat, 3] float32
    lights: np.ndarray        # [L, 3] float32
    eye: np.ndarray           # [3] float32
    width: int
    height: int
    pos: np.ndarray           # [3, P] float32 (SoA)
    nrm: np.ndarray           # [3, P] float32 (SoA)
    mat: np.ndarray           # [P] int32, -1 = no primary hit
    ray_types: int            # bitmask 1=SH 2=RE 4=RR
    levels: int = 2
    leaf_size: int = 8
    branching: int = 8
    meta: dict = field(default_factory=dict)
    dir: np.ndarray | None = None   # [3, P] float32 incident directions (Whitted bounce > 0), None = from eye

    @property
    def P(self) -> int:
        return self.width * self.height

    @property
    def M(self) -> int:
        return int(self.tris.shape[0])

    @property
    def n_meshes(self) -> int:
        return int(self.mesh_ids[-1]) + 1 if self.M else 0


# ----------------------------------------------------------------------------
# rasteriser (C) -- built on demand, also by __graft_entry__.build()

def build_raster(force: bool = False) -> str:
    src = os.path.join(HERE, "raster.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", LIB, src, "-lm"])
    return LIB


_raster = None


def _lib():
    global _raster
    if _raster is None:
        build_raster()
        _raster = ctypes.CDLL(LIB)
        _raster.raster_gbuffer.restype = ctypes.c_int
    return _raster


def make_camera(eye=EYE, fwd=FWD, up=UP, vfov=VFOV) -> np.ndarray:
    """Pinhole camera of the GPU primary pass (include/crsh.h crsh_camera):
    eye, right, up, fwd, tan(vfov/2) as 13 float32 -- the same orthonormal
    basis raster.c builds (right = fwd x up, up' = right x fwd), in float64
    then rounded. Input generation only (no method arithmetic)."""
    f = np.asarray(fwd, np.float64)
    f = f / np.linalg.norm(f)
    r = np.cross(f, np.asarray(up, np.float64))
    r = r / np.linalg.norm(r)
    u = np.cross(r, f)
    return np.concatenate([np.asarray(eye, np.float64), r, u, f, [np.tan(np.radians(vfov) / 2)]]).astype(np.float32)


def rasterize(tris, tri_mat, width, height, eye=EYE, fwd=FWD, up=UP, vfov=VFOV):
    tris = np.ascontiguousarray(tris, dtype=np.float32)
    tri_mat = np.ascontiguousarray(tri_mat, dtype=np.int32)
    P = width * height
    pos = np.empty((3, P), np.float32)
    nrm = np.empty((3, P), np.float32)
    mat = np.empty(P, np.int32)
    tid = np.empty(P, np.int32)
    d = lambda v: (ctypes.c_double * 3)(*v)  # noqa: E731
    rc = _lib().raster_gbuffer(
        tris.ctypes.data_as(ctypes.c_void_p), tri_mat.ctypes.data_as(ctypes.c_void_p),
        ctypes.c_int64(tris.shape[0]), d(eye), d(fwd), d(up), ctypes.c_double(vfov),
        ctypes.c_int32(width), ctypes.c_int32(height),
        pos.ctypes.data_as(ctypes.c_void_p), nrm.ctypes.data_as(ctypes.c_void_p),
        mat.ctypes.data_as(ctypes.c_void_p), tid.ctypes.data_as(ctypes.c_void_p))
    if rc != 0:
        raise RuntimeError(f"raster_gbuffer failed rc={rc}")
    return pos, nrm, mat, tid


# ----------------------------------------------------------------------------
# tessellated primitives (unit-size, then transformed)

def _quad_grid(p0, du, dv, g):
    """g x g grid of a parallelogram p0 + s*du + t*dv -> 2 g^2 triangles."""
    p0, du, dv = (np.asarray(a, np.float64) for a in (p0, du, dv))
    s = np.arange(g + 1) / g
    P = p0[None, None, :] + s[:, None, None] * du[None, None, :] + s[None, :, None] * dv[None, None, :]
    a, b, c, d = P[:-1, :-1], P[1:, :-1], P[1:, 1:], P[:-1, 1:]
    t1 = np.stack([a, b, c], axis=2).reshape(-1, 9)
    t2 = np.stack([a, c, d], axis=2).reshape(-1, 9)
    return np.concatenate([t1, t2], 0)


def _uv_sphere(n_lat, n_lon):
    th = np.linspace(0, math.pi, n_lat + 1)
    ph = np.linspace(0, 2 * math.pi, n_lon + 1)
    V = np.stack([np.sin(th)[:, None] * np.cos(ph)[None, :],
                  np.cos(th)[:, None] * np.ones_like(ph)[None, :],
                  np.sin(th)[:, None] * np.sin(ph)[None, :]], -1)
    out = []
    for i in range(n_lat):
        for j in range(n_lon):
            a, b, c, d = V[i, j], V[i + 1, j], V[i + 1, j + 1], V[i, j + 1]
            if i > 0:
                out.append(np.concatenate([a, b, d]))
            if i < n_lat - 1:
                out.append(np.concatenate([b, c, d]))
    return np.array(out)


def _box(s):
    faces = []
    for axis in range(3):
        for sign in (-1.0, 1.0):
            u, v = [(axis + 1) % 3, (axis + 2) % 3]
            p0 = np.zeros(3); p0[axis] = sign; p0[u] = -1; p0[v] = -1
            du = np.zeros(3); du[u] = 2
            dv = np.zeros(3); dv[v] = 2
            faces.append(_quad_grid(p0, du, dv, s))
    return np.concatenate(faces, 0) / math.sqrt(3.0)   # bounding radius 1


def _torus(n_u, n_v, R=0.7, r=0.3):
    u = np.linspace(0, 2 * math.pi, n_u + 1)
    v = np.linspace(0, 2 * math.pi, n_v + 1)
    V = np.stack([(R + r * np.cos(v)[None, :]) * np.cos(u)[:, None],
                  r * np.sin(v)[None, :] * np.ones_like(u)[:, None],
                  (R + r * np.cos(v)[None, :]) * np.sin(u)[:, None]], -1)
    a, b, c, d = V[:-1, :-1], V[1:, :-1], V[1:, 1:], V[:-1, 1:]
    return np.concatenate([np.stack([a, b, c], 2).reshape(-1, 9), np.stack([a, c, d], 2).reshape(-1, 9)], 0)


def _cylinder(n_u, n_h, r=0.6, h=1.6):
    u = np.linspace(0, 2 * math.pi, n_u + 1)
    y = np.linspace(-h / 2, h / 2, n_h + 1)
    V = np.stack([r * np.cos(u)[:, None] * np.ones_like(y)[None, :], np.ones_like(u)[:, None] * y[None, :],
                  r * np.sin(u)[:, None] * np.ones_like(y)[None, :]], -1)
    a, b, c, d = V[:-1, :-1], V[1:, :-1], V[1:, 1:], V[:-1, 1:]
    side = np.concatenate([np.stack([a, b, c], 2).reshape(-1, 9), np.stack([a, c, d], 2).reshape(-1, 9)], 0)
    caps = []
    for yy in (-h / 2, h / 2):
        ctr = np.array([0.0, yy, 0.0])
        for j in range(n_u):
            p = np.array([r * math.cos(u[j]), yy, r * math.sin(u[j])])
            q = np.array([r * math.cos(u[j + 1]), yy, r * math.sin(u[j + 1])])
            caps.append(np.concatenate([ctr, p, q]))
    out = np.concatenate([side, np.array(caps)], 0)
    rad = np.sqrt((out.reshape(-1, 3) ** 2).sum(1)).max()
    return out / rad


def _object(kind, T):
    if kind == 0:
        n_lat = max(3, int(round(math.sqrt(T / 4.0))) + 1)
        n_lon = max(3, int(round(T / (2.0 * (n_lat - 1)))))
        return _uv_sphere(n_lat, n_lon)
    if kind == 1:
        return _box(max(1, int(round(math.sqrt(T / 12.0)))))
    if kind == 2:
        n_v = max(3, int(round(math.sqrt(T / 8.0))))
        return _torus(max(3, int(round(T / (2.0 * n_v)))), n_v)
    n_h = max(1, int(round(math.sqrt(T / 8.0))))
    return _cylinder(max(3, int(round(T / (2.0 * n_h + 2)))), n_h)


def _rotation(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def _walls(g):
    L = 10.0
    return [
        _quad_grid((0, 0, 0), (0, 0, L), (0, L, 0), g),   # x = 0
        _quad_grid((L, 0, 0), (0, L, 0), (0, 0, L), g),   # x = 10
        _quad_grid((0, 0, 0), (L, 0, 0), (0, 0, L), g),   # y = 0 floor
        _quad_grid((0, L, 0), (0, 0, L), (L, 0, 0), g),   # y = 10 ceiling
        _quad_grid((0, 0, 0), (0, L, 0), (L, 0, 0), g),   # z = 0 (behind camera)
        _quad_grid((0, 0, L), (L, 0, 0), (0, L, 0), g),   # z = 10 far wall
    ]


def make_room_scene(seed, M_target, n_meshes, mirror_walls=(), shell_g=None, object_kinds=None):
    """Room shell (6 wall meshes) + (n_meshes - 6) objects. Returns tris, mesh_ids, mesh_mat."""
    rng = np.random.default_rng(seed)
    n_obj = n_meshes - 6
    if shell_g is None:
        shell_g = max(2, int(round(math.sqrt(0.1 * M_target / 12.0))))
    walls = _walls(shell_g)
    meshes = list(walls)
    mesh_mat = [MIRROR if i in mirror_walls else DIFFUSE for i in range(6)]
    shell_tris = sum(w.shape[0] for w in walls)
    if n_obj > 0:
        T = max(8, (M_target - shell_tris) // n_obj)
        avail = 8.0 * 7.6 * 6.0
        s = min(1.0, (0.25 * avail / (n_obj * 2.2)) ** (1.0 / 3.0))
        placed = []
        for k in range(n_obj):
            R = rng.uniform(0.3, 1.2) * s
            for attempt in range(20000):
                c = np.array([rng.uniform(R + 0.2, 10 - R - 0.2), rng.uniform(R + 0.2, 8.8 - R),
                              rng.uniform(2.0 + R, 10 - R - 0.2)])
                if all(np.linalg.norm(c - c2) >= R + R2 + 0.05 for c2, R2 in placed):
                    break
                if attempt % 1000 == 999:
                    R *= 0.85
            else:
                raise RuntimeError("object placement failed")
            placed.append((c, R))
            kind = int(object_kinds[k % len(object_kinds)]) if object_kinds is not None else int(rng.integers(0, 4))
            obj = _object(kind, T).reshape(-1, 3) @ _rotation(rng).T * R + c
            meshes.append(obj.reshape(-1, 9))
            u = rng.uniform()
            mesh_mat.append(DIFFUSE if u < 0.60 else (MIRROR if u < 0.85 else GLASS))
    tris = np.concatenate(meshes, 0).astype(np.float32)
    mesh_ids = np.concatenate([np.full(m.shape[0], i, np.int32) for i, m in enumerate(meshes)])
    return tris, mesh_ids, np.array(mesh_mat, np.int32)


# ----------------------------------------------------------------------------
# the configurations of BASELINE.json "configs"

CONFIGS = {
    1: dict(name="cfg1: 128x128 SH 1 light, ~1k-tri Cornell box, Lv3", W=128, H=128, types=1, lights=1,
            M=1024, meshes=7, levels=3, leaf=8, branch=8, shell_g=8, mirror_walls=(0, 1), kinds=(0,)),
    2: dict(name="cfg2: 512x512 SH+RE, ~70k tris / 16 meshes, Lv2", W=512, H=512, types=3, lights=1,
            M=70000, meshes=16, levels=2, leaf=8, branch=8, mirror_walls=(0,)),
    3: dict(name="cfg3: 1024x1024 SH+RE+RR, ~250k tris / 30 meshes, Lv2", W=1024, H=1024, types=7, lights=2,
            M=250000, meshes=30, levels=2, leaf=8, branch=8, mirror_walls=(0,)),
    4: dict(name="cfg4: 1920x1080 SH+RE+RR, ~1M tris / 100 meshes, Lv2", W=1920, H=1080, types=7, lights=4,
            M=1000000, meshes=100, levels=2, leaf=8, branch=8, mirror_walls=(0,)),
    5: dict(name="cfg5: sweep at 1024x1024, ~250k tris / 30 meshes", W=1024, H=1024, types=7, lights=2,
            M=250000, meshes=30, levels=2, leaf=8, branch=8, mirror_walls=(0,)),
}

SEED_BASE = 2312065380


def make_workload(cfg: int, width=None, height=None, levels=None, leaf_size=None, branching=None,
                  ray_types=None, n_lights=None) -> Workload:
    c = CONFIGS[cfg]
    seed = SEED_BASE + cfg
    tris, mesh_ids, mesh_mat = make_room_scene(seed, c["M"], c["meshes"], mirror_walls=c.get("mirror_walls", ()),
                                               shell_g=c.get("shell_g"), object_kinds=c.get("kinds"))
    W = width or c["W"]
    H = height or c["H"]
    tri_mat = mesh_mat[mesh_ids]
    pos, nrm, mat, _ = rasterize(tris, tri_mat, W, H)
    L = n_lights or c["lights"]
    return Workload(name=c["name"], tris=tris, mesh_ids=mesh_ids, tri_mat=tri_mat, materials=MATERIALS.copy(),
                    lights=np.array(LIGHTS[:L], np.float32), eye=np.array(EYE, np.float32), width=W, height=H,
                    pos=pos, nrm=nrm, mat=mat, ray_types=ray_types or c["types"],
                    levels=levels or c["levels"], leaf_size=leaf_size or c["leaf"],
                    branching=branching or c["branch"], meta=dict(cfg=cfg, seed=seed))


def make_micro(seed: int, n_tris: int = 32, W: int = 16, H: int = 16, n_meshes: int = 3, n_lights: int = 2,
               ray_types: int = 7, levels: int = 2, leaf_size: int = 8, branching: int = 8,
               empty_frac: float = 0.15) -> Workload:
    """Randomised micro-scene (SPEC.md:624 acceptance 5): random triangles in a
    box, grouped into meshes, and a synthetic G-buffer whose fragments lie on
    random triangles (so shadow/bounce rays meet real geometry).  Some pixels
    are empty (mat = -1) to exercise trimming."""
    rng = np.random.default_rng(seed)
    centers = rng.uniform(1, 9, size=(n_tris, 3))
    tris = (centers[:, None, :] + rng.normal(scale=0.8, size=(n_tris, 3, 3))).reshape(-1, 9).astype(np.float32)
    cuts = np.sort(rng.choice(np.arange(1, n_tris), size=max(0, min(n_meshes, n_tris) - 1), replace=False))
    mesh_ids = np.zeros(n_tris, np.int32)
    for c in cuts:
        mesh_ids[c:] += 1
    P = W * H
    which = rng.integers(0, n_tris, size=P)
    bary = rng.dirichlet([1, 1, 1], size=P)
    T = tris.reshape(-1, 3, 3)[which]
    pos = (bary[:, :, None] * T).sum(1)
    n = np.cross(T[:, 1] - T[:, 0], T[:, 2] - T[:, 0])
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    mat = rng.integers(0, 3, size=P).astype(np.int32)
    mat[rng.uniform(size=P) < empty_frac] = -1
    lights = rng.uniform(0.5, 9.5, size=(n_lights, 3)).astype(np.float32)
    return Workload(name=f"micro{seed}", tris=tris, mesh_ids=mesh_ids, tri_mat=np.zeros(n_tris, np.int32),
                    materials=MATERIALS.copy(), lights=lights, eye=np.array([5.0, 5.0, -1.0], np.float32),
                    width=W, height=H, pos=np.ascontiguousarray(pos.T, np.float32),
                    nrm=np.ascontiguousarray(n.T, np.float32), mat=mat, ray_types=ray_types, levels=levels,
                    leaf_size=leaf_size, branching=branching, meta=dict(seed=seed))
