"""Pins for the oracle's object sphere-tree ("combine
our coherent ray hierarchy with a deeper object hierarchy"; reading O1 in
DESIGN.md §3).  Expected values come from closed forms, an independent numpy
transcription of the cluster order, fp64 containment, brute-force recounts with
a different loop structure, and the N x M brute force -- never from the CUDA
path."""
import numpy as np
import pytest

from workloads import make_micro, make_workload

CL = 32


def _spread3(v):
    v = v.astype(np.uint64) & np.uint64(0x3FF)
    out = np.zeros_like(v)
    for b in range(10):
        out |= ((v >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b)
    return out


def morton_order_np(tris, mesh_ids):
    """O1's cluster order written independently: per mesh, triangles sorted by
    the Morton code of the centroid in the mesh's vertex box (1024 cells per
    axis, x the most significant), ties by index."""
    T = tris.reshape(-1, 3, 3).astype(np.float64)
    cen = ((T[:, 0] + T[:, 1]) + T[:, 2]) / 3.0
    order = []
    for m in range(int(mesh_ids.max()) + 1):
        idx = np.flatnonzero(mesh_ids == m)
        if len(idx) == 0:
            continue
        V = T[idx].reshape(-1, 3)
        lo, hi = V.min(0), V.max(0)
        code = np.zeros(len(idx), np.uint64)
        for k in range(3):
            if hi[k] > lo[k]:
                q = np.clip(np.floor(((cen[idx, k] - lo[k]) / (hi[k] - lo[k])) * 1024.0), 0, 1023)
            else:
                q = np.zeros(len(idx))
            code |= _spread3(q.astype(np.uint64)) << np.uint64(2 - k)
        order.append(idx[np.lexsort((idx, code))])
    return np.concatenate(order).astype(np.int32)


def test_cluster_order_and_spheres(orc):
    """The cluster order is O1's Morton order (independent transcription); the
    clusters partition every mesh into runs of CL (the last shorter); every
    vertex of a cluster lies inside its sphere (fp64), whose radius is at most
    the half-diagonal of the cluster's vertex box plus pad (+ float rounding)."""
    w = make_workload(2, width=16, height=16)
    prep = orc.ScenePrep(w.tris, w.mesh_ids)
    order = prep.cluster_order[:prep.M]
    assert np.array_equal(order, morton_order_np(w.tris, w.mesh_ids))
    T = w.tris.reshape(-1, 3, 3).astype(np.float64)
    counts = prep.mesh_range[:prep.n_meshes, 1] - prep.mesh_range[:prep.n_meshes, 0]
    assert np.array_equal(np.diff(prep.mesh_cluster_first[:prep.n_meshes + 1]), (counts + CL - 1) // CL)
    for m in range(prep.n_meshes):
        t0, t1 = prep.mesh_range[m]
        assert sorted(order[t0:t1].tolist()) == list(range(t0, t1))   # a permutation within the mesh
        for j, c in enumerate(range(prep.mesh_cluster_first[m], prep.mesh_cluster_first[m + 1])):
            ids = order[t0 + j * CL: min(t0 + (j + 1) * CL, t1)]
            V = T[ids].reshape(-1, 3)
            s = prep.cluster_sph[c].astype(np.float64)
            d = np.linalg.norm(V - s[:3], axis=1)
            assert np.all(d <= s[3]), (m, c)
            half = 0.5 * np.linalg.norm(V.max(0) - V.min(0))
            assert s[3] <= half * (1 + 1e-6) + prep.pad + 1e-6, (m, c)


def test_cluster_sphere_closed_form(orc):
    """One mesh = the 12 triangles of the unit cube, one cluster: centre
    (0.5, 0.5, 0.5), radius sqrt(3)/2 rounded up to float, plus pad."""
    P = np.array([[x, y, z] for x in (0, 1) for y in (0, 1) for z in (0, 1)], np.float32)
    faces = [(0, 1, 3), (0, 3, 2), (4, 6, 7), (4, 7, 5), (0, 4, 5), (0, 5, 1), (2, 3, 7), (2, 7, 6), (0, 2, 6),
             (0, 6, 4), (1, 5, 7), (1, 7, 3)]
    tris = np.stack([P[list(f)].reshape(9) for f in faces]).astype(np.float32)
    prep = orc.ScenePrep(tris, np.zeros(12, np.int32))
    assert prep.n_clusters == 1
    s = prep.cluster_sph[0]
    assert np.array_equal(s[:3], np.float32([0.5, 0.5, 0.5]))
    r = np.float32(np.sqrt(0.75))
    if float(r) < np.sqrt(0.75):
        r = np.nextafter(r, np.float32(np.inf))
    assert s[3] == np.float32(r + np.float32(prep.pad))


@pytest.mark.parametrize("seed", range(12))
def test_objtree_counts_recounted_and_hits_exact(orc, seed):
    """With the object tree (flag 64): the hits equal those without it and the
    N x M brute force (the extra level is conservative); the cluster counters
    and the top-level test count equal a brute-force recount over the
    oracle's own top nodes -- every (top node, kept mesh, cluster) pair tested
    with Eq 9 in a Python loop -- and the tree never adds top-level tests."""
    r = np.random.default_rng(seed)
    w = make_micro(7000 + seed, n_tris=int(r.integers(20, 160)), W=int(r.integers(4, 20)), H=int(r.integers(4, 20)),
                   n_meshes=int(r.integers(1, 5)), n_lights=int(r.integers(1, 3)), ray_types=7,
                   levels=int(r.integers(1, 4)), leaf_size=int(2 ** r.integers(1, 4)), branching=4)
    prep = orc.ScenePrep(w.tris, w.mesh_ids)
    for base in (3, 7):
        a = orc.trace(w, prep, flags=base, n_threads=2)
        b = orc.trace(w, prep, flags=base | 64, n_threads=2, taps=True)
        assert np.array_equal(a["hit_tri"], b["hit_tri"]) and np.array_equal(a["t"], b["t"])
        ok = b["empty"] == 0
        bt, btt = orc.unpack(orc.brute(b["rays"][ok], prep, 2))
        assert np.array_equal(b["hit_tri"][ok], bt)
        counts = prep.mesh_range[:prep.n_meshes, 1] - prep.mesh_range[:prep.n_meshes, 0]
        segs = [s for s, _, _ in orc.segments(w.P, w.lights.shape[0], w.ray_types)]
        for i, seg in enumerate(segs):
            top = b["taps"]["levels"][i][-1] if len(b["taps"]["levels"][i]) else np.zeros((0, 8), np.float32)
            ct = ch = tl = 0
            for node in top:
                for m in range(prep.n_meshes):
                    if counts[m] == 0 or not orc.cull(node, prep.mesh_sph[m]):
                        continue
                    for j, c in enumerate(range(prep.mesh_cluster_first[m], prep.mesh_cluster_first[m + 1])):
                        ct += 1
                        if orc.cull(node, prep.cluster_sph[c]):
                            ch += 1
                            tl += min(CL, int(counts[m]) - j * CL)
            st = b["stats"]
            assert st["cluster_tests"][seg] == ct and st["cluster_hits"][seg] == ch, (seg, st["cluster_tests"][seg], ct)
            assert st["tests"][seg][w.levels] == tl, (seg, st["tests"][seg][w.levels], tl)
            assert st["tests"][seg][w.levels] <= a["stats"]["tests"][seg][w.levels]
            assert st["rays_hit"][seg] == a["stats"]["rays_hit"][seg]


def test_objtree_transform_keeps_creation_order(orc):
    """A moved scene (reading G2) keeps the creation-time cluster order and
    recomputes the cluster spheres from the moved vertices."""
    w = make_workload(1, width=16, height=16)
    prep0 = orc.ScenePrep(w.tris, w.mesh_ids)
    n = prep0.n_meshes
    X = np.tile(np.array([0, -1, 0, 5, 1, 0, 0, -1, 0, 0, 1, 0.25], np.float32), (n, 1))   # rotation + shift
    prep, tris = orc.transformed_prep(prep0, w.tris, w.mesh_ids, X)
    assert np.array_equal(prep.cluster_order, prep0.cluster_order)
    T = tris.reshape(-1, 3, 3).astype(np.float64)
    for m in range(n):
        t0, t1 = prep.mesh_range[m]
        for j, c in enumerate(range(prep.mesh_cluster_first[m], prep.mesh_cluster_first[m + 1])):
            ids = prep.cluster_order[t0 + j * CL: min(t0 + (j + 1) * CL, t1)]
            d = np.linalg.norm(T[ids].reshape(-1, 3) - prep.cluster_sph[c, :3].astype(np.float64), axis=1)
            assert np.all(d <= prep.cluster_sph[c, 3])
