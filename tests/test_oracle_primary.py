"""Pins of the oracle's primary pass (the G-buffer
producer of P:67-71): the camera rays against their closed form, the primary
hits against N x M brute force, and the G-buffer against the independent
float64 z-buffer rasteriser of workloads/raster.c (the paper's own step 1)."""
import math

import numpy as np

import oracle
from workloads import make_camera, make_workload, rasterize


def test_camera_rays_closed_form():
    cam = make_camera((1.0, 2.0, 3.0), (0.0, 0.0, 1.0), (0.0, 1.0, 0.0), 60.0)
    W, H = 5, 3
    rays = oracle.camera_rays(cam, W, H)
    th = math.tan(math.radians(30.0))
    for j in range(H):
        for i in range(W):
            u = ((2 * i + 1) / W - 1) * th * W / H
            v = (1 - (2 * j + 1) / H) * th
            d = np.array([-u, v, 1.0])   # right = fwd x up = (0,0,1) x (0,1,0) = (-1,0,0)
            d /= np.linalg.norm(d)
            r = rays[j * W + i]
            assert np.allclose(r[:3], [1, 2, 3]) and r[3] == 0.0 and np.isinf(r[7])
            assert np.allclose(r[4:7], d, atol=2e-7)
    # the centre pixel of an odd image looks straight ahead
    assert np.allclose(rays[1 * W + 2, 4:7], [0, 0, 1], atol=1e-7)


def test_primary_hits_equal_brute_force():
    w = make_workload(1, width=48, height=40)
    cam = make_camera()
    prep = oracle.ScenePrep(w.tris, w.mesh_ids)
    pos, nrm, mat, hit, t, st = oracle.primary_gbuffer(w.tris, w.mesh_ids, w.tri_mat, cam, 48, 40, 3, 8, 8, prep=prep)
    bt, btt = oracle.unpack(oracle.brute(oracle.camera_rays(cam, 48, 40), prep))
    assert np.array_equal(hit, bt) and np.array_equal(t.view(np.uint32), btt.view(np.uint32))
    assert st["rays"][1] == 48 * 40 and st["rays"][0] == 0


def test_gbuffer_agrees_with_the_rasteriser():
    """Independent implementations (float32 ray casting through the hierarchy
    vs float64 z-buffer rasterisation): same visible triangle on >= 98 % of
    pixels (pixel-centre ties on shared edges may differ), and on those the
    same material, positions within 2e-4 and camera-facing normals within 1e-5."""
    w = make_workload(2, width=96, height=96)
    cam = make_camera()
    pos, nrm, mat, hit, t, _ = oracle.primary_gbuffer(w.tris, w.mesh_ids, w.tri_mat, cam, 96, 96)
    rp, rn, rm, rtri = rasterize(w.tris, w.tri_mat, 96, 96)
    same = hit == rtri
    assert same.mean() >= 0.98, same.mean()
    assert np.array_equal(mat[same], rm[same])
    assert np.abs(pos[:, same] - rp[:, same]).max() < 2e-4
    assert np.abs(nrm[:, same] - rn[:, same]).max() < 1e-5
