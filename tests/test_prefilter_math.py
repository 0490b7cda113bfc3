"""The claim behind K8's child prefilter (k_traverse.cuh `cull_pf`, DESIGN §5
K8-PF), on the CPU: Eq 9 as the oracle evaluates it (float32, the paper's
order: PAPER.md:179-181, reading R12/R13) is monotone in the target sphere,
and the prefilter's margin covers float32 rounding. If the oracle's test
passes for a sphere (P, R), then the prefilter passes for every sphere (C, Rb)
with |P - C| + R <= Rb. Both prefilter forms (the scalar `cull_pf` of the top level and the packed,
fused `cull2_pf_s` of the child pairs) are transcribed here in numpy float32
in the kernel's operation order, because the claim is about those
evaluations.
The inputs are random nodes (narrow to wide cones, and the pass-all wide
nodes) and spheres placed on the pass/fail boundary, where rounding matters
most."""
import math
import warnings

import numpy as np
import pytest

warnings.filterwarnings("ignore", "overflow encountered", RuntimeWarning)   # wide nodes: rhs^2 = inf, as on the GPU

f32 = np.float32
rng = np.random.default_rng(20231206)


def tansec(alpha):
    """tan and sec of a cone angle as the traversal records store them. Wide
    cones (alpha >= pi/2) get tan = sec = 1e30 and axis 0 (numspec.cuh)."""
    if alpha >= math.pi / 2:
        return f32(1e30), f32(1e30)
    return f32(math.tan(alpha)), f32(1.0 / math.cos(alpha))


def cull_pf(c, d, a, tn, sc, S):
    """k_traverse.cuh cull_pf, float32, the same operation order."""
    vx, vy, vz = f32(S[0] - c[0]), f32(S[1] - c[1]), f32(S[2] - c[2])
    mag = f32(f32(f32(f32(abs(vx) + abs(vy)) + abs(vz)) + abs(f32(d))) + f32(S[3]))
    dr = f32(f32(f32(d) + f32(S[3])) + f32(mag * f32(2.0 ** -12)))
    s = f32(f32(f32(vx * a[0]) + f32(vy * a[1])) + f32(vz * a[2]))
    if s < -dr:
        return False
    wx, wy, wz = f32(vx - f32(s * a[0])), f32(vy - f32(s * a[1])), f32(vz - f32(s * a[2]))
    w2 = f32(f32(f32(wx * wx) + f32(wy * wy)) + f32(wz * wz))
    rhs = f32(f32(max(s, f32(0.0)) * tn) + f32(dr * sc))
    return bool(w2 <= f32(rhs * rhs))


def fma(a, b, c):
    """float32 fused multiply-add (the product of two float32 is exact in
    float64; one rounding of the sum, then to float32)."""
    return f32(np.float64(a) * np.float64(b) + np.float64(c))


def cull2_pf_half(c, d, a, tn, sc, S):
    """One half of k_traverse.cuh cull2_pf_s (the packed child prefilter),
    float32 with its fused operations."""
    vx, vy, vz = f32(S[0] - c[0]), f32(S[1] - c[1]), f32(S[2] - c[2])
    mag = f32(f32(f32(f32(abs(vx) + abs(vy)) + abs(vz)) + abs(f32(d))) + f32(S[3]))
    dr = fma(mag, f32(2.0 ** -12), f32(f32(d) + f32(S[3])))
    s = fma(vx, a[0], fma(vy, a[1], f32(vz * a[2])))
    wx, wy, wz = fma(s, -a[0], vx), fma(s, -a[1], vy), fma(s, -a[2], vz)
    w2 = fma(wx, wx, fma(wy, wy, f32(wz * wz)))
    rhs = fma(max(s, f32(0.0)), tn, f32(dr * sc))
    return bool(s >= -dr) and bool(w2 <= f32(rhs * rhs))


def random_node():
    c = rng.uniform(-50, 50, 3).astype(f32)
    a = rng.normal(size=3)
    a = (a / np.linalg.norm(a)).astype(f32)
    d = f32(rng.uniform(0.0, 5.0))
    alpha = float(rng.choice([rng.uniform(0.0, 0.05), rng.uniform(0.0, 1.5), rng.uniform(1.5, 1.5707), 2.0]))
    return c, d, a, alpha


def boundary_sphere(c, d, a, alpha):
    """A sphere near the node's pass/fail boundary: a point at axial distance
    s and perpendicular distance close to the allowed radius."""
    tn = math.tan(min(alpha, 1.5706))
    sc = 1.0 / math.cos(min(alpha, 1.5706))
    R = rng.uniform(0.001, 2.0)
    s = rng.uniform(-(d + R) * 1.01, 200.0)
    allowed = max(s, 0.0) * tn + (d + R) * sc
    perp = allowed * rng.uniform(0.995, 1.005)
    u = rng.normal(size=3)
    u -= np.dot(u, a) * a
    u /= np.linalg.norm(u)
    P = (c.astype(np.float64) + s * a.astype(np.float64) + perp * u).astype(f32)
    return P, f32(R)


@pytest.mark.parametrize("trial", range(4))
def test_prefilter_passes_whenever_a_contained_sphere_passes(orc, trial):
    passes = 0
    for _ in range(1500):
        c, d, a, alpha = random_node()
        node8 = np.array([*c, d, *a, alpha], np.float32)
        P, R = boundary_sphere(c, d, a, alpha)
        if not orc.cull(node8, [*P, R]):
            continue
        passes += 1
        tn, sc = tansec(alpha)
        a_rec = a if alpha < math.pi / 2 else np.zeros(3, f32)
        # containing spheres: the same sphere, shifted centres with the radius
        # grown to cover it (rounded up), the cluster-sized case
        for k in range(6):
            off = rng.normal(size=3) * (0.0 if k == 0 else 10.0 ** rng.uniform(-3, 1))
            C = (P.astype(np.float64) + off).astype(f32)
            Rb = np.nextafter(f32(np.linalg.norm(P.astype(np.float64) - C.astype(np.float64)) + float(R)), f32(np.inf))
            assert cull_pf(c, d, a_rec, tn, sc, (C[0], C[1], C[2], Rb)), (node8, P, R, C, Rb)
            assert cull2_pf_half(c, d, a_rec, tn, sc, (C[0], C[1], C[2], Rb)), (node8, P, R, C, Rb)
    assert passes > 100


def smallest_passing_radius(orc, node8, P, R_hi):
    """The smallest float32 radius for which the oracle's Eq 9 passes at P
    (bisection over the float32 bit patterns): the sphere sits exactly on the
    float32 decision boundary."""
    lo, hi = 0, int(np.float32(R_hi).view(np.int32))
    if orc.cull(node8, [*P, f32(0.0)]):
        return None
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if orc.cull(node8, [*P, np.int32(mid).view(np.float32)]):
            hi = mid
        else:
            lo = mid
    return np.int32(hi).view(np.float32)


def test_prefilter_covers_spheres_on_the_float_boundary(orc):
    """Spheres exactly on the oracle's float32 pass/fail boundary (smallest
    passing radius): the prefilter, evaluated in its own operation order,
    must still pass for them and for spheres containing them -- the case its
    rounding margin exists for."""
    n = 0
    for _ in range(3000):
        c, d, a, alpha = random_node()
        if alpha >= math.pi / 2:
            continue
        node8 = np.array([*c, d, *a, alpha], np.float32)
        P, R = boundary_sphere(c, d, a, alpha)
        Rs = smallest_passing_radius(orc, node8, P, f32(R * 4 + 10))
        if Rs is None or not orc.cull(node8, [*P, Rs]):
            continue
        n += 1
        tn, sc = tansec(alpha)
        assert cull_pf(c, d, a, tn, sc, (P[0], P[1], P[2], Rs)), (node8, P, Rs)
        assert cull2_pf_half(c, d, a, tn, sc, (P[0], P[1], P[2], Rs)), (node8, P, Rs)
        off = rng.normal(size=3) * 1e-3
        C = (P.astype(np.float64) + off).astype(f32)
        Rb = np.nextafter(f32(np.linalg.norm(P.astype(np.float64) - C.astype(np.float64)) + float(Rs)), f32(np.inf))
        assert cull_pf(c, d, a, tn, sc, (C[0], C[1], C[2], Rb)), (node8, P, Rs, C, Rb)
        assert cull2_pf_half(c, d, a, tn, sc, (C[0], C[1], C[2], Rb)), (node8, P, Rs, C, Rb)
    assert n > 1000


def test_prefilter_rejects_far_spheres():
    """Not vacuous: a narrow cone rejects a sphere well outside it."""
    c, a = np.zeros(3, f32), np.array([0, 0, 1], f32)
    tn, sc = tansec(0.01)
    assert not cull_pf(c, f32(0.1), a, tn, sc, (50.0, 0.0, 10.0, 1.0))
    assert not cull_pf(c, f32(0.1), a, tn, sc, (0.0, 0.0, -20.0, 1.0))   # behind the apex
    assert cull_pf(c, f32(0.1), a, tn, sc, (0.0, 0.0, 30.0, 1.0))
    assert not cull2_pf_half(c, f32(0.1), a, tn, sc, (50.0, 0.0, 10.0, 1.0))
    assert cull2_pf_half(c, f32(0.1), a, tn, sc, (0.0, 0.0, 30.0, 1.0))
    wtn, wsc = tansec(2.0)   # wide: pass-all
    assert cull_pf(c, f32(0.1), np.zeros(3, f32), wtn, wsc, (50.0, 0.0, -10.0, 1.0))
