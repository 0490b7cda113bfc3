"""Pins for the oracle's geometric building blocks (L0, SURVEY §8(c) 'What pins
each part').  Every expected value here comes from the paper/SPEC worked
examples, a closed form, or an independent fp64 numpy computation written in
this file -- never from the oracle itself or from the CUDA path."""
import itertools
import math

import numpy as np
import pytest

rng = np.random.default_rng(12345)


def unit(v):
    v = np.asarray(v, np.float64)
    return v / np.linalg.norm(v)


# ----------------------------------------------------------------- Moller-Trumbore
def tri_e(v0, v1, v2):
    v0, v1, v2 = (np.asarray(a, np.float32) for a in (v0, v1, v2))
    return np.concatenate([v0, v1 - v0, v2 - v0]).astype(np.float32)


def test_mt_spec_examples(orc):
    """S:64 hit at t = 1 (symmetry), S:65 parallel ray misses."""
    T = tri_e((-1, -1, 0), (1, -1, 0), (0, 1, 0))
    assert orc.mt([0, 0, -1, 1e-4, 0, 0, 1, np.inf], T) == pytest.approx(1.0, abs=0)
    assert orc.mt([0, 0, -1, 1e-4, 1, 0, 0, np.inf], T) is None
    # two-sided (R15): from the other side too
    assert orc.mt([0, 0, 1, 1e-4, 0, 0, -1, np.inf], T) == 1.0
    # (tmin, tmax) is open on both ends
    assert orc.mt([0, 0, -1, 1e-4, 0, 0, 1, 1.0], T) is None
    assert orc.mt([0, 0, -1, 1.0, 0, 0, 1, 5.0], T) is None


def test_mt_degenerate_never_hits(orc):
    """a zero-area triangle always misses."""
    T = tri_e((0, 0, 0), (1, 1, 1), (2, 2, 2))
    for _ in range(200):
        o = rng.normal(size=3)
        d = unit(rng.normal(size=3))
        assert orc.mt([*o, 0.0, *d, np.inf], T) is None


def test_mt_vs_plane_then_barycentric(orc):
    """10^4 random ray/triangle pairs agree with an independent fp64
    plane-intersection + signed-edge-function oracle on hit/miss (away from
    edges and from the t bounds) and on t within 1e-5 relative."""
    agree, checked = 0, 0
    for _ in range(10000):
        V = rng.normal(size=(3, 3))
        o = rng.normal(size=3) * 2
        target = V.T @ rng.dirichlet([1, 1, 1]) if rng.uniform() < 0.6 else rng.normal(size=3)
        d = unit(target - o)
        o32, d32, V32 = o.astype(np.float32), d.astype(np.float32), V.astype(np.float32)
        t = orc.mt([*o32, 1e-4, *d32, np.inf], tri_e(*V32))
        # fp64 reference on the float32 inputs
        o64, d64, V64 = o32.astype(np.float64), d32.astype(np.float64), V32.astype(np.float64)
        n = np.cross(V64[1] - V64[0], V64[2] - V64[0])
        den = n @ d64
        if abs(den) < 0.1 * np.linalg.norm(n):   # grazing rays are ill-conditioned in float32
            continue
        tt = n @ (V64[0] - o64) / den
        p = o64 + tt * d64
        area = np.linalg.norm(n)
        w = [np.cross(V64[(i + 1) % 3] - V64[i], p - V64[i]) @ n / area for i in range(3)]
        margin = min(abs(x) for x in w) / math.sqrt(area)
        if margin < 1e-4 or abs(tt - 1e-4) < 1e-4:
            continue
        inside = all(x > 0 for x in w) or all(x < 0 for x in w)
        ref_hit = inside and tt > 1e-4
        checked += 1
        assert (t is not None) == ref_hit
        if ref_hit:
            assert t == pytest.approx(tt, rel=1e-4, abs=1e-5)   # float32 MT on skinny triangles; formula errors are O(1)
        agree += 1
    assert checked > 4000


def test_mt_vs_divide_first_moller_trumbore(orc):
    """R15 pin: the oracle's sign-folded, division-deferred decision order
    against an independent float32 transcription of the textbook two-sided
    Moller-Trumbore (MT97's non-culling branch: inv_det = 1/det first, then
    u = (T.P) inv_det in [0, 1], v = (D.Q) inv_det >= 0, u + v <= 1,
    t = (E2.Q) inv_det), written here with numpy's plain float32 dot products
    (no fma), and both against the same quantities in fp64.  On 2*10^4 random
    pairs away from the barycentric edges (u, v, 1-u-v all > 1e-4 in fp64) and
    from tmin: (1) both orders accept exactly the pairs fp64 accepts; (2) t of
    the two float32 orders agree within 1e-5 relative (the north-star bar) on
    >= 99.5 % of hits -- the rest are ill-conditioned pairs (cancellation in
    E2.Q) where both are off; (3) the oracle's order is no less accurate than
    divide-first: its 99th/99.9th-percentile relative error against fp64 is at
    most divide-first's."""
    r = np.random.default_rng(97)
    n = 20000
    V = r.normal(size=(n, 3, 3)).astype(np.float32)
    o = (r.normal(size=(n, 3)) * 2).astype(np.float32)
    w = r.dirichlet([1, 1, 1], size=n)
    target = np.where(r.uniform(size=(n, 1)) < 0.6, np.einsum("nk,nkj->nj", w, V.astype(np.float64)),
                      r.normal(size=(n, 3)))
    d = target - o
    d = (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)
    f = np.float32
    e1, e2 = V[:, 1] - V[:, 0], V[:, 2] - V[:, 0]
    tv = o - V[:, 0]

    def dot(a, b):
        return (a[:, 0] * b[:, 0] + a[:, 1] * b[:, 1] + a[:, 2] * b[:, 2]).astype(np.float32)

    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        p = np.cross(d, e2).astype(np.float32)
        det = dot(e1, p)
        inv = (f(1) / det).astype(np.float32)
        u = dot(tv, p) * inv
        q = np.cross(tv, e1).astype(np.float32)
        v = dot(d, q) * inv
        t = dot(e2, q) * inv
        # the same quantities in fp64 on the float32 inputs
        D, E1, E2, TV = (a.astype(np.float64) for a in (d, e1, e2, tv))
        P64 = np.cross(D, E2)
        DET = (E1 * P64).sum(1)
        Q64 = np.cross(TV, E1)
        U, V64, T = (TV * P64).sum(1) / DET, (D * Q64).sum(1) / DET, (E2 * Q64).sum(1) / DET
    tmin = f(1e-4)
    hit = (det != 0) & (u >= 0) & (u <= 1) & (v >= 0) & (u + v <= 1) & (t > tmin)
    hit64 = (U >= 0) & (V64 >= 0) & (U + V64 <= 1) & (T > 1e-4)
    clear = (DET != 0) & (np.minimum(np.minimum(np.abs(U), np.abs(V64)), np.abs(1 - U - V64)) > 1e-4) & \
        (np.abs(T - 1e-4) > 1e-4) & np.isfinite(T)
    checked, e_or, e_df, agree = 0, [], [], []
    for k in np.flatnonzero(clear):
        got = orc.mt([*o[k], tmin, *d[k], np.inf], np.concatenate([V[k, 0], e1[k], e2[k]]))
        assert (got is not None) == bool(hit64[k]) == bool(hit[k]), (k, U[k], V64[k], T[k])
        if got is not None:
            e_or.append(abs(got - T[k]) / T[k])
            e_df.append(abs(float(t[k]) - T[k]) / T[k])
            agree.append(abs(got - float(t[k])) <= 1e-5 * abs(float(t[k])))
        checked += 1
    assert checked > 15000 and len(e_or) > 5000
    assert np.mean(agree) >= 0.995
    for qq in (0.99, 0.999):
        assert np.quantile(e_or, qq) <= np.quantile(e_df, qq), qq


# ----------------------------------------------------------------- spheres
def brute_min_sphere(P):
    """Combinatorial minimal enclosing sphere: all spheres with 1..4 boundary
    points (diameter / circumcircle / circumsphere), smallest containing all."""
    P = np.asarray(P, np.float64)
    best = None
    cands = [(p, 0.0) for p in P]
    for a, b in itertools.combinations(range(len(P)), 2):
        c = (P[a] + P[b]) / 2
        cands.append((c, np.linalg.norm(P[a] - c)))
    for a, b, c_ in itertools.combinations(range(len(P)), 3):
        A, Bv, Cv = P[a], P[b], P[c_]
        ab, ac = Bv - A, Cv - A
        n = np.cross(ab, ac)
        if n @ n < 1e-18:
            continue
        ctr = A + (np.cross(n, ab) * (ac @ ac) + np.cross(ac, n) * (ab @ ab)) / (2 * (n @ n))
        cands.append((ctr, np.linalg.norm(A - ctr)))
    for q in itertools.combinations(range(len(P)), 4):
        A = P[q[0]]
        M = np.array([P[q[i]] - A for i in (1, 2, 3)])
        if abs(np.linalg.det(M)) < 1e-12:
            continue
        x = np.linalg.solve(M, 0.5 * (M * M).sum(1))
        cands.append((A + x, np.linalg.norm(x)))
    for c, r in cands:
        if np.all(np.linalg.norm(P - c, axis=1) <= r * (1 + 1e-9) + 1e-12):
            if best is None or r < best[1]:
                best = (c, r)
    return best


def test_tri_sphere_spec_examples(orc):
    """S:73 right triangle -> centre (1,1,0), radius sqrt(2); S:74 obtuse ->
    the longest-edge diameter sphere (2, 0, 0), r = 2 (contains (1, .1, 0))."""
    s = orc.tri_sphere([0, 0, 0, 2, 0, 0, 0, 2, 0])
    assert np.allclose(s[:3], [1, 1, 0]) and s[3] == pytest.approx(math.sqrt(2), rel=1e-7)
    assert s[3] >= np.float32(math.sqrt(2))   # rounded up (containment exact)
    s = orc.tri_sphere([0, 0, 0, 4, 0, 0, 1, 0.1, 0])
    assert np.allclose(s[:3], [2, 0, 0]) and s[3] == pytest.approx(2.0, rel=1e-7)


def test_tri_sphere_random_vs_combinatorial(orc):
    for _ in range(500):
        V = rng.normal(size=(3, 3)).astype(np.float32)
        s = orc.tri_sphere(V.reshape(-1))
        c, r = brute_min_sphere(V.astype(np.float64))
        assert np.all(np.linalg.norm(V.astype(np.float64) - s[:3].astype(np.float64), axis=1) <= s[3])
        assert s[3] == pytest.approx(r, rel=2e-6, abs=1e-6)


def test_miniball_spec_examples(orc):
    """S:91 two points -> (1,0,0) r 1; S:92 unit cube corners -> centre
    (.5,.5,.5), r sqrt(3)/2; S:89 empty input is an error."""
    s = orc.miniball([[0, 0, 0], [2, 0, 0]])
    assert np.allclose(s, [1, 0, 0, 1])
    cube = np.array(list(itertools.product([0, 1], repeat=3)), np.float32)
    s = orc.miniball(cube)
    assert np.allclose(s[:3], 0.5) and s[3] == pytest.approx(math.sqrt(3) / 2, rel=1e-7)
    with pytest.raises(ValueError):
        orc.miniball(np.zeros((0, 3)))


def test_miniball_random_vs_combinatorial(orc):
    """random point sets (n <= 10) match the brute-force candidate
    enumeration within 1e-6 relative; every point is contained exactly."""
    for n in [1, 2, 3, 4, 5, 7, 10] * 12:
        P = rng.normal(size=(n, 3)).astype(np.float32)
        s = orc.miniball(P)
        c, r = brute_min_sphere(P.astype(np.float64))
        assert np.all(np.linalg.norm(P.astype(np.float64) - s[:3].astype(np.float64), axis=1) <= s[3])
        assert s[3] == pytest.approx(r, rel=2e-6, abs=1e-6)


def test_miniball_coplanar_grid(orc):
    """A tessellated wall (all points coplanar, the degenerate case of the
    4-point support): minimal sphere of a square grid = half its diagonal."""
    g = np.linspace(0, 10, 9)
    P = np.array([[x, y, 3.0] for x in g for y in g], np.float32)
    s = orc.miniball(P)
    assert np.allclose(s[:3], [5, 5, 3], atol=1e-5)
    assert s[3] == pytest.approx(math.sqrt(50), rel=1e-6)


def test_sphere_union_eq7_8(orc):
    """S:436 (0,0,0,1) U (4,0,0,1) -> (2,0,0), 3 (Eqs 7-8);
    S:437 concentric; S:438 random containment; empty passes through (R9)."""
    assert np.allclose(orc.sphere_union([0, 0, 0, 1], [4, 0, 0, 1]), [2, 0, 0, 3])
    assert np.allclose(orc.sphere_union([1, 2, 3, 3], [1, 2, 3, 1]), [1, 2, 3, 3])
    assert np.allclose(orc.sphere_union([0, 0, 0, -1], [4, 5, 6, 2]), [4, 5, 6, 2])
    for _ in range(2000):
        a = np.concatenate([rng.normal(size=3), [rng.uniform(0, 2)]])
        b = np.concatenate([rng.normal(size=3), [rng.uniform(0, 2)]])
        u = orc.sphere_union(a, b).astype(np.float64)
        for s in (a, b):
            assert np.linalg.norm(s[:3] - u[:3]) + s[3] <= u[3] + 1e-5


# ----------------------------------------------------------------- angles
def test_atan2p_accuracy(orc):
    """R7/F8: the polynomial atan2 is within 4e-7 rad of fp64 arctan2 (the
    polynomial itself is within 1.2e-7 on [0,1]; the octant reconstruction adds
    the float32 rounding of values up to pi, ulp 2.4e-7).  The 14-bit theta
    cell is 1.9e-4 rad.  SPEC conventions at the axes."""
    ys = np.concatenate([rng.normal(size=20000), [0, 0, 1, -1, 0, 1e-30]]).astype(np.float32)
    xs = np.concatenate([rng.normal(size=20000), [1, -1, 0, 0, 0, 1]]).astype(np.float32)
    err = max(abs(orc.atan2p(float(y), float(x)) - math.atan2(float(y), float(x))) for y, x in zip(ys, xs))
    assert err < 4e-7
    assert orc.atan2p(0.0, 0.0) == 0.0          # poles map to phi = 0
    assert orc.atan2p(-0.0, -1.0) == np.float32(math.pi)   # -0.0 is not negative (R7)


def test_sincos_accuracy(orc):
    phis = np.concatenate([rng.uniform(0, math.pi, 20000), [0, math.pi / 4, math.pi / 2, 3 * math.pi / 4, math.pi]])
    for p in phis.astype(np.float32):
        c, s = orc.sincos(float(p))
        assert abs(c - math.cos(float(p))) < 2e-7 and abs(s - math.sin(float(p))) < 2e-7


# ----------------------------------------------------------------- hashes
def test_hash_shadow_examples(orc):
    """light 0, +z -> 8191; S:329 light 1 -> >= 2^28; S:330 same cell
    -> same key; P:83 light index in the high bits."""
    assert orc.hash_shadow(0, [0, 0, 1]) == 8191
    for _ in range(50):
        d = unit(rng.normal(size=3))
        assert orc.hash_shadow(1, d) >= 2 ** 28
        assert orc.hash_shadow(3, d) >> 28 == 3
        assert orc.hash_shadow(2, d) > orc.hash_shadow(1, unit(rng.normal(size=3)))
    # closed form of the layout for directions well inside a cell
    for _ in range(200):
        th = rng.uniform(0.1, 3.0)
        ph = rng.uniform(-3.0, 3.0)
        qt, qp = math.floor(th / math.pi * 16383), math.floor((ph + math.pi) / (2 * math.pi) * 16383)
        ft, fp = th / math.pi * 16383 - qt, (ph + math.pi) / (2 * math.pi) * 16383 - qp
        if min(ft, 1 - ft, fp, 1 - fp) < 0.01:
            continue
        d = [math.sin(th) * math.cos(ph), math.sin(th) * math.sin(ph), math.cos(th)]
        assert orc.hash_shadow(0, d) == (qt << 14) | qp
        # a nearby direction in the same cell hashes equal
        th2 = th + 0.001 * (0.5 - ft) / 16383 * math.pi
        d2 = [math.sin(th2) * math.cos(ph), math.sin(th2) * math.sin(ph), math.cos(th2)]
        assert orc.hash_shadow(0, d2) == orc.hash_shadow(0, d)


def test_hash_bounce_examples(orc):
    """origin at the box minimum, +z -> qx=qy=qz=0, theta 0, phi
    mid-range: floor(0.5 * 511) = 255; different x cells differ in
    the high bits; zero extent quantises to 0."""
    bmin, bext = [0, 0, 0], [10, 10, 10]
    assert orc.hash_bounce([0, 0, 0], [0, 0, 1], bmin, bext) == 255
    k1 = orc.hash_bounce([0.1, 5, 5], [1, 0, 0], bmin, bext)
    k2 = orc.hash_bounce([9.9, 5, 5], [1, 0, 0], bmin, bext)
    assert k1 >> 27 == 0 and k2 >> 27 == 31 and (k1 & ((1 << 27) - 1)) == (k2 & ((1 << 27) - 1))
    assert orc.hash_bounce([3, 4, 5], [0, 0, 1], [0, 0, 0], [0, 10, 10]) >> 27 == 0
    # closed form of the layout
    for _ in range(200):
        o = rng.uniform(0.05, 9.95, 3)
        cells = np.floor(o / 10 * 32)
        if np.any(np.abs(o / 10 * 32 - np.round(o / 10 * 32)) < 1e-3):
            continue
        th, ph = rng.uniform(0.1, 3.0), rng.uniform(-3, 3)
        qt, qp = math.floor(th / math.pi * 255), math.floor((ph + math.pi) / (2 * math.pi) * 511)
        ft, fp = th / math.pi * 255 - qt, (ph + math.pi) / (2 * math.pi) * 511 - qp
        if min(ft, 1 - ft, fp, 1 - fp) < 0.01:
            continue
        d = [math.sin(th) * math.cos(ph), math.sin(th) * math.sin(ph), math.cos(th)]
        key = int(cells[0]) << 27 | int(cells[1]) << 22 | int(cells[2]) << 17 | qt << 9 | qp
        assert orc.hash_bounce(o, d, bmin, bext) == key


# ----------------------------------------------------------------- cones
def ang(u, v):
    u, v = unit(u), unit(v)
    return math.atan2(np.linalg.norm(np.cross(u, v)), u @ v)


def test_cone_grow_examples(orc):
    """cone(+z, 0) grown with +x -> axis (x+z)/sqrt2, 45 deg (Eqs 1-4
    reduce to the bisector when phi = 0); S:418 inside -> unchanged
    antiparallel -> full cone."""
    x, p = orc.cone_grow([0, 0, 1], 0.0, [1, 0, 0])
    assert np.allclose(x, unit([1, 0, 1]), atol=1e-7) and p == pytest.approx(math.pi / 4, abs=2e-7)
    x, p = orc.cone_grow([0, 0, 1], 0.0, [0, 0, 1])
    assert np.allclose(x, [0, 0, 1]) and p == 0.0
    x, p = orc.cone_grow([0, 0, 1], 0.3, [0, 0, -1])
    assert p == np.float32(math.pi)


def test_cone_grow_tight_and_containing(orc):
    """S:420 containment of r and of the old cone; F6 tightness: the new
    half-angle is (phi + gamma)/2, i.e. both r and the old cone's far boundary
    lie on the new boundary (fp64 reference)."""
    for _ in range(3000):
        xa = unit(rng.normal(size=3))
        phi = float(rng.uniform(0, 1.2))
        r = unit(rng.normal(size=3))
        x, p = orc.cone_grow(xa.astype(np.float32), phi, r.astype(np.float32))
        x = x.astype(np.float64)
        g = ang(xa, r)
        if g <= phi:
            assert p == np.float32(phi)
            continue
        if phi + g >= math.pi:
            assert p == np.float32(math.pi)
            continue
        # tight up to the conditioning of the bisector x_new = norm(r - e)
        assert p == pytest.approx((phi + g) / 2, abs=1e-6 + 2e-7 / max(1e-9, math.cos((phi + g) / 2)))
        assert p >= (phi + g) / 2 - 1e-6
        assert ang(x, r) <= p + 1e-5
        # old cone: boundary samples
        e1 = unit(np.cross(xa, [1, 0, 0] if abs(xa[0]) < 0.9 else [0, 1, 0]))
        e2 = np.cross(xa, e1)
        for k in range(16):
            b = 2 * math.pi * k / 16
            dirn = math.cos(phi) * xa + math.sin(phi) * (math.cos(b) * e1 + math.sin(b) * e2)
            assert ang(x, dirn) <= p + 1e-5


def test_cone_union_examples(orc):
    """S:427 identical cones; S:428 (+z,0) U (+x,0) -> 45 deg (Eqs 5-6 with
    the R11 reading); S:425 antiparallel -> full; clamp to pi."""
    x, p = orc.cone_union([0, 0, 1], 0.2, [0, 0, 1], 0.2)
    assert np.allclose(x, [0, 0, 1]) and p == np.float32(0.2)
    x, p = orc.cone_union([0, 0, 1], 0.0, [1, 0, 0], 0.0)
    assert np.allclose(x, unit([1, 0, 1]), atol=1e-7) and p == pytest.approx(math.pi / 4, abs=2e-7)
    assert orc.cone_union([0, 0, 1], 0.1, [0, 0, -1], 0.1)[1] == np.float32(math.pi)
    assert orc.cone_union([0, 0, 1], 3.0, [0, 1, 0], 0.5)[1] == np.float32(math.pi)


def test_cone_union_contains_both(orc):
    for _ in range(3000):
        x1, x2 = unit(rng.normal(size=3)), unit(rng.normal(size=3))
        p1, p2 = float(rng.uniform(0, 1)), float(rng.uniform(0, 1))
        x, p = orc.cone_union(x1, p1, x2, p2)
        if p >= np.float32(math.pi):
            continue
        for xa, pa in ((x1, p1), (x2, p2)):
            assert ang(x, xa) + pa <= p + 1e-5


# ----------------------------------------------------------------- Eq 9
def node8(c, r, a, alpha):
    return np.array([*c, r, *unit(a), alpha], np.float32)


def test_cull_spec_examples(orc):
    """S:82 on-axis target passes; S:83 lateral target rejects; S:113 wide
    cones pass everything."""
    n = node8([0, 0, 0], 0.0, [0, 0, 1], 0.0)
    assert orc.cull(n, [0, 0, 5, 1])
    assert not orc.cull(n, [10, 0, 5, 1])
    assert orc.cull(node8([0, 0, 0], 0.0, [0, 0, 1], 1.6), [100, 0, -50, 1])


def test_cull_rejects_behind_apex(orc):
    """S:79 / S:455: a target wholly behind the node (s < -(d + r)) is
    rejected even when it lies near the axis line; touching it is kept."""
    n = node8([0, 0, 0], 0.5, [0, 0, 1], 0.1)
    assert not orc.cull(n, [0, 0, -5, 1])
    assert orc.cull(n, [0, 0, -1.4, 1])


def test_cull_alpha0_is_cylinder_overlap(orc):
    """Closed form: with alpha = 0 the swept volume is a cylinder of radius d
    about the axis, so for a target in front (s >= 0) the test is exactly
    'perpendicular distance <= d + r'."""
    for _ in range(3000):
        d = float(rng.uniform(0, 1))
        r = float(rng.uniform(0.01, 1))
        s = float(rng.uniform(0.5, 10))
        w = float(rng.uniform(0, 3))
        if abs(w - (d + r)) < 1e-4:
            continue
        P = [w, 0.0, s]
        assert orc.cull(node8([0, 0, 0], d, [0, 0, 1], 0.0), [*P, r]) == (w <= d + r)


def test_cull_zero_false_negatives(orc):
    """S:84 / F6: random nodes and targets; whenever any sampled ray (origin in
    the node sphere, direction in the cone) meets the target sphere (fp64
    analytic ray-sphere test), Eq 9 must pass."""
    fn, hits = 0, 0
    for _ in range(4000):
        C = rng.uniform(-1, 1, 3)
        d = float(rng.uniform(0, 0.5))
        a = unit(rng.normal(size=3))
        alpha = float(rng.uniform(0, 0.8))
        P = C + a * rng.uniform(-2, 8) + rng.normal(size=3) * rng.uniform(0, 4)
        r = float(rng.uniform(0.05, 1.0))
        ok = orc.cull(node8(C, d, a, alpha), [*P, r])
        e1 = unit(np.cross(a, [1, 0, 0] if abs(a[0]) < 0.9 else [0, 1, 0]))
        e2 = np.cross(a, e1)
        for _ in range(48):
            o = C + unit(rng.normal(size=3)) * d * rng.uniform() ** (1 / 3)
            th = alpha * math.sqrt(rng.uniform())
            b = rng.uniform(0, 2 * math.pi)
            v = math.cos(th) * a + math.sin(th) * (math.cos(b) * e1 + math.sin(b) * e2)
            oc = P - o
            tc = oc @ v
            if tc >= 0 and oc @ oc - tc * tc <= r * r or oc @ oc <= r * r:
                hits += 1
                fn += (not ok)
                break
    assert hits > 300
    assert fn == 0


def interleave(fields_bits):
    """Z-order: bit i of field j goes to position i*len + (len-1-j) (field 0 most significant)."""
    out = 0
    nf = len(fields_bits)
    for j, (v, b) in enumerate(fields_bits):
        for i in range(b):
            out |= ((v >> i) & 1) << (i * nf + (nf - 1 - j))
    return out


def test_hash_zorder_is_a_bit_interleave(orc):
    """CRSH_F_ZORDER: the Z-order key carries exactly the
    fields of the SPEC layout, bits interleaved."""
    bmin, bext = np.zeros(3, np.float32), np.full(3, 10, np.float32)
    for _ in range(500):
        d = unit(rng.normal(size=3))
        l = int(rng.integers(0, 16))
        k = orc.hash_shadow(l, d)
        qt, qp = (k >> 14) & 0x3FFF, k & 0x3FFF
        assert orc.hash_shadow(l, d, zorder=True) == (l << 28) | interleave([(qt, 14), (qp, 14)])
        o = rng.uniform(0, 10, 3)
        k = orc.hash_bounce(o, d, bmin, bext)
        qx, qy, qz, qt, qp = k >> 27, (k >> 22) & 31, (k >> 17) & 31, (k >> 9) & 255, k & 511
        kz = orc.hash_bounce(o, d, bmin, bext, zorder=True)
        assert kz >> 17 == interleave([(qx, 5), (qy, 5), (qz, 5)])
        assert kz & 0x1FFFF == ((qp >> 8) << 16) | interleave([(qt, 8), (qp & 255, 8)])
