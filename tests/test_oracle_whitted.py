"""Pins of the oracle's multi-bounce Whitted loop (
P:185-187 "accumulate shading ... output another set of secondary rays";
SPEC S:514-522 shade_and_spawn examples), against closed forms computed here
in float64 from the fixture geometry -- not from the oracle's formulas."""
import math

import numpy as np
import pytest

import oracle
from workloads import MATERIALS, make_workload
from workloads.scenes import Workload


def quad(p0, p1, p2, p3):
    """two triangles (p0 p1 p2), (p0 p2 p3); winding normal = (p1-p0) x (p2-p0)"""
    return [list(p0) + list(p1) + list(p2), list(p0) + list(p2) + list(p3)]


def fixture(quads, quad_mat, materials, lights, eye, px_pos, px_nrm, px_mat):
    tris, mesh, tmat = [], [], []
    for qi, (q, m) in enumerate(zip(quads, quad_mat)):
        for t in quad(*q):
            tris.append(t); mesh.append(qi); tmat.append(m)
    P = len(px_mat)
    return Workload(name="fx", tris=np.array(tris, np.float32), mesh_ids=np.array(mesh, np.int32),
                    tri_mat=np.array(tmat, np.int32), materials=np.array(materials, np.float32),
                    lights=np.array(lights, np.float32).reshape(-1, 3), eye=np.array(eye, np.float32), width=P,
                    height=1, pos=np.array(px_pos, np.float32).T.copy(), nrm=np.array(px_nrm, np.float32).T.copy(),
                    mat=np.array(px_mat, np.int32), ray_types=7, levels=2, leaf_size=8, branching=8)


DIFFUSE, MIRROR = [0.0, 0.0, 1.0], [1.0, 0.0, 1.0]
FLOOR = ((-10, 0, -10), (-10, 0, 10), (10, 0, 10), (10, 0, -10))   # y = 0, winding normal +y


def test_direct_closed_form_two_lights():
    """depth 0, diffuse floor, two lights: L = kd (cos1 + cos2) / 2 with
    cos_l = n.(L_l - x) / |L_l - x| (float64 closed form)."""
    lights = [(1.0, 4.0, 2.0), (-2.0, 3.0, 0.0)]
    w = fixture([FLOOR], [0], [DIFFUSE], lights, (0, 5, -5), [(0, 0, 0)], [(0, 1, 0)], [0])
    img = oracle.whitted(w, 0)["image"]
    want = (4 / math.sqrt(21) + 3 / math.sqrt(13)) / 2
    assert abs(img[0] - want) < 1e-6


def test_fully_occluded_pixel_is_black():
    """fully occluded wrt its only light -> 0 (a blocker quad between)."""
    blocker = ((-1, 2, -1), (1, 2, -1), (1, 2, 1), (-1, 2, 1))
    w = fixture([FLOOR, blocker], [0, 0], [DIFFUSE], [(0, 5, 0)], (0, 5, -5), [(0, 0, 0)], [(0, 1, 0)], [0])
    assert oracle.whitted(w, 2)["image"][0] == 0.0


def test_grazing_light_gives_zero():
    """n.l = 0 -> zero diffuse term (light in the surface plane)."""
    w = fixture([FLOOR], [0], [DIFFUSE], [(5, 0, 0)], (0, 5, -5), [(0, 0, 0)], [(0, 1, 0)], [0])
    assert oracle.whitted(w, 0)["image"][0] == 0.0


def test_mirror_shows_the_lit_wall():
    """a mirror (reflectivity 1, kd 0) facing a lit diffuse wall shows
    the wall's direct radiance at the reflected point: eye (-5,5,1), mirror
    point (0,0,0) -> reflected ray (5,5,-1)/sqrt51 hits the wall x = 5 at
    q = (5,5,-1); light (0,8,0): L = cos = 5 / sqrt(35)."""
    wall = ((5, 0, -10), (5, 10, -10), (5, 10, 10), (5, 0, 10))   # winding normal -x
    w = fixture([FLOOR, wall], [1, 0], [DIFFUSE, MIRROR], [(0, 8, 0)], (-5, 5, 1), [(0, 0, 0)], [(0, 1, 0)], [1])
    r = oracle.whitted(w, 1)
    assert r["vertices"] == [1, 1]
    assert abs(r["image"][0] - 5 / math.sqrt(35)) < 1e-5
    # depth 0 keeps only the mirror's own (zero) diffuse term
    assert oracle.whitted(w, 0)["image"][0] == 0.0


def test_glass_pane_transmits_the_floor():
    """A glass pane (transmissivity 1) above a lit floor: the refracted ray
    crosses the pane (enter, then exit: two refractions) and the pixel shows the
    floor's direct radiance weighted by trans^2 = 1 at depth 2, 0 at depth 0/1
    for the floor term (depth 1 stops inside the pane's second face)."""
    GLASS = [0.0, 1.0, 1.5]
    top = ((-3, 2.1, -3), (-3, 2.1, 3), (3, 2.1, 3), (3, 2.1, -3))       # normal +y
    bot = ((-3, 2.0, -3), (3, 2.0, -3), (3, 2.0, 3), (-3, 2.0, 3))       # normal -y
    light = (9.0, 3.0, 0.0)   # the shadow ray to the floor point passes beside the pane
    w = fixture([FLOOR, top, bot], [0, 1, 1], [DIFFUSE, GLASS], [light], (0, 6, 0), [(0, 2.1, 0)], [(0, 1, 0)], [1])
    r2 = oracle.whitted(w, 2)
    assert r2["vertices"] == [1, 1, 1]   # pixel on the top face -> bottom face -> floor
    # straight down (normal incidence): floor point (0,0,0); light cos = 3/sqrt(90)
    assert abs(r2["image"][0] - 3 / math.sqrt(90)) < 1e-5


@pytest.mark.parametrize("flags", [0, 1, 7])
def test_engines_render_the_same_image(flags):
    """brute / RAH / CRSH differ only in skipped tests -> the same
    image (here CRSH, RAH, sort-only and the Z-order layout, bit for bit)."""
    w = make_workload(1, width=24, height=24)
    a = oracle.whitted(w, 2)["image"]
    b = oracle.whitted(w, 2, flags=flags)["image"]
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_radiance_bounded_and_monotone_in_depth():
    """0 <= L <= 1 (kd + refl + trans <= 1, light weights sum to 1, cos <= 1);
    adding a bounce never lowers a pixel (all terms are non-negative)."""
    w = make_workload(1, width=24, height=24)
    prev = None
    for d in range(4):
        img = oracle.whitted(w, d)["image"]
        assert img.min() >= 0.0 and img.max() <= 1.0 + 1e-6
        if prev is not None:
            assert np.all(img >= prev - 1e-6)
        prev = img
    assert MATERIALS.shape[1] == 3
