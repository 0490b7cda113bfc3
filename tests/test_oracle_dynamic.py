"""Pins of the dynamic-scene update (§3.3.1 Bounding
Volume Update): the SPEC examples, sigma_max against
numpy's SVD, containment of every transformed vertex, and the conservative
trace of a moved scene against brute force."""
import numpy as np
import pytest

import oracle
from workloads import make_camera, make_workload

ID = np.array([1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0], np.float32)


def xf(A, b):
    return np.concatenate([np.asarray(A, np.float32), np.asarray(b, np.float32)[:, None]], axis=1).reshape(12)


def test_spec_examples():
    s = np.array([1.0, 2.0, 3.0, 0.75], np.float32)
    assert np.array_equal(oracle.update_sphere(s, xf(np.eye(3), [1, 2, 3])), [2, 4, 6, 0.75])
    assert np.array_equal(oracle.update_sphere(s, xf(2 * np.eye(3), [0, 0, 0])), [2, 4, 6, 1.5])
    rz = [[0, -1, 0], [1, 0, 0], [0, 0, 1]]
    out = oracle.update_sphere(s, xf(rz, [0, 0, 0]))
    assert out[3] == 0.75 and np.allclose(out[:3], [-2, 1, 3])


@pytest.mark.parametrize("seed", range(5))
def test_sigma_max_matches_svd(seed):
    r = np.random.default_rng(seed)
    for _ in range(200):
        A = r.normal(size=(3, 3)) * r.uniform(0.1, 5)
        got = oracle.sigma_max(xf(A, [0, 0, 0]))
        want = np.linalg.svd(np.asarray(A, np.float32).astype(np.float64), compute_uv=False)[0]
        assert abs(got - want) <= 1e-10 * want


def test_updated_mesh_spheres_contain_the_moved_vertices():
    """S:237 invariant, in float64: every transformed vertex (as the float32
    transform computes it) inside its mesh's updated sphere, for random
    rotations, non-uniform scales, shears and translations."""
    w = make_workload(1)
    prep0 = oracle.ScenePrep(w.tris, w.mesh_ids)
    r = np.random.default_rng(3)
    for _ in range(10):
        X = []
        for _m in range(prep0.n_meshes):
            q, _ = np.linalg.qr(r.normal(size=(3, 3)))
            A = q @ np.diag(r.uniform(0.3, 2.0, 3)) + 0.2 * r.normal(size=(3, 3))
            X.append(xf(A, r.uniform(-3, 3, 3)))
        X = np.stack(X)
        prep, tris = oracle.transformed_prep(prep0, w.tris, w.mesh_ids, X)
        v = tris.reshape(-1, 3, 3).astype(np.float64)
        for m in range(prep.n_meshes):
            lo, hi = prep.mesh_range[m]
            c = prep.mesh_sph[m, :3].astype(np.float64)
            d = np.linalg.norm(v[lo:hi].reshape(-1, 3) - c, axis=1)
            assert d.max() <= float(prep.mesh_sph[m, 3]), (m, d.max(), prep.mesh_sph[m, 3])


def test_moved_scene_traces_conservatively():
    """After moving every mesh (rigid motion + scale), the hierarchy trace of
    a primary-pass G-buffer equals N x M brute force on every ray."""
    w = make_workload(1, width=48, height=48)
    prep0 = oracle.ScenePrep(w.tris, w.mesh_ids)
    r = np.random.default_rng(7)
    X = []
    for m in range(prep0.n_meshes):
        if m < 6:   # keep the room's walls in place
            X.append(ID.copy())
            continue
        q, _ = np.linalg.qr(r.normal(size=(3, 3)))
        q *= np.sign(np.linalg.det(q))
        X.append(xf(q * r.uniform(0.7, 1.3), r.uniform(-1, 1, 3)))
    X = np.stack(X)
    prep, tris = oracle.transformed_prep(prep0, w.tris, w.mesh_ids, X)
    cam = make_camera()
    pos, nrm, mat, hit, t, _ = oracle.primary_gbuffer(tris, w.mesh_ids, w.tri_mat, cam, 48, 48, prep=prep)
    import dataclasses
    wm = dataclasses.replace(w, tris=tris, pos=pos, nrm=nrm, mat=mat, ray_types=7,
                             lights=np.array([[5, 9.5, 5], [2, 9, 3]], np.float32))
    out = oracle.trace(wm, prep)
    ok = out["empty"] == 0
    bt, btt = oracle.unpack(oracle.brute(out["rays"][ok], prep))
    assert np.array_equal(out["hit_tri"][ok], bt) and np.array_equal(out["t"][ok], btt)
    assert ok.sum() > 1000
