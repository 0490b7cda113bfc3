"""Pins for the oracle's pipeline stages (trim, compress/sort/decompress,
hierarchy, traversal counts, end-to-end hits).  Expected values come from SPEC
worked examples, the paper's own tables (tests/golden/paper_tables.json, each
row cited), library routines that define the same result (numpy stable
argsort), brute force, and invariants -- never from the CUDA path."""
import json
import math
import os

import numpy as np
import pytest

from workloads import make_micro, make_workload

HERE = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(777)


# ----------------------------------------------------------------- trim (Fig 4)
def test_trim_examples(orc):
    """S:170 flags [0,1,0,1] keys [a,.,b,.] -> [a,b]; S:171 all empty -> [];
    S:172 random flags == order-preserving filter; S:169 bad flag -> error."""
    k, v = orc.trim([0, 1, 0, 1], [11, 99, 22, 99], [0, 1, 2, 3])
    assert k.tolist() == [11, 22] and v.tolist() == [0, 2]
    k, v = orc.trim([1, 1, 1], [1, 2, 3], [0, 1, 2])
    assert len(k) == 0
    f = (rng.uniform(size=100000) < 0.3).astype(np.uint32)
    keys = rng.integers(0, 2 ** 32, size=100000, dtype=np.uint64).astype(np.uint32)
    vals = np.arange(100000, dtype=np.uint32)
    k, v = orc.trim(f, keys, vals)
    assert np.array_equal(k, keys[f == 0]) and np.array_equal(v, vals[f == 0])
    with pytest.raises(ValueError):
        orc.trim([0, 2], [1, 2], [0, 1])


# ----------------------------------------------------------------- compress / sort / decompress
def test_compress_sort_decompress_spec_example(orc):
    """S:346 keys [5,5,3,3,3,9] -> chunks [5,3,9] base [0,2,5] size [2,3,1];
    S:355 -> sorted keys [3,3,3,5,5,9], values [2,3,4,0,1,5] (Figs 5-6)."""
    ck, cb, cs = orc.compress([5, 5, 3, 3, 3, 9])
    assert ck.tolist() == [5, 3, 9] and cb.tolist() == [0, 2, 5] and cs.tolist() == [2, 3, 1]
    sk, sv, _ = orc.sort_decompress(ck, cb, cs, np.arange(6, dtype=np.uint32))
    assert sk.tolist() == [3, 3, 3, 5, 5, 9] and sv.tolist() == [2, 3, 4, 0, 1, 5]
    ck, cb, cs = orc.compress([7] * 10)
    assert ck.tolist() == [7] and cs.tolist() == [10]
    ck, cb, cs = orc.compress([1, 2, 3, 4])
    assert cs.tolist() == [1, 1, 1, 1]
    ck, cb, cs = orc.compress([])
    assert len(ck) == 0


def test_compress_sort_is_stable_sort(orc):
    """F7 / S:357 / acceptance 6: compress -> sort -> decompress equals a
    stable sort of (key, value) by key (numpy's stable argsort), on 10^5 keys
    with runs and duplicates."""
    runs = rng.integers(1, 6, size=40000)
    keys = np.repeat(rng.integers(0, 3000, size=runs.size), runs)[:100000].astype(np.uint32)
    vals = rng.permutation(keys.size).astype(np.uint32)
    ck, cb, cs = orc.compress(keys)
    assert cs.sum() == keys.size and len(ck) < keys.size
    sk, sv, _ = orc.sort_decompress(ck, cb, cs, vals)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(sk, keys[order]) and np.array_equal(sv, vals[order])


# ----------------------------------------------------------------- hierarchy
def rays_from(o, d, tmin=1e-3, tmax=np.inf):
    n = o.shape[0]
    return np.concatenate([o, np.full((n, 1), tmin), d, np.full((n, 1), tmax)], 1).astype(np.float32)


def test_level_sizes(orc):
    """S:446 N=100, B=8, Lv=2 -> 13 and 2 nodes; F3 top = ceil(N/64)."""
    o = rng.normal(size=(100, 3))
    d = rng.normal(size=(100, 3)); d /= np.linalg.norm(d, axis=1, keepdims=True)
    lv = orc.build_levels(rays_from(o, d), 2, 8, 8)
    assert [x.shape[0] for x in lv] == [13, 2]
    lv = orc.build_levels(rays_from(np.zeros((8, 3)), np.tile([0, 0, 1.0], (8, 1))), 2, 8, 8)
    assert lv[0].tolist() == [[0, 0, 0, 0, 0, 0, 1, 0]] and lv[1].tolist() == lv[0].tolist()


def containment_errors(levels, rays, B0, B):
    """fp64 check of the load-bearing invariant: every ray's origin is
    inside every ancestor sphere and its direction inside every ancestor cone."""
    worst_s, worst_c = 0.0, 0.0
    n = rays.shape[0]
    idx = np.arange(n)
    span = B0
    for lv in levels:
        node = lv[idx // span].astype(np.float64)
        ds = np.linalg.norm(rays[:, :3] - node[:, :3], axis=1) - node[:, 3]
        cosang = np.clip((rays[:, 4:7] * node[:, 4:7]).sum(1) / np.linalg.norm(node[:, 4:7], axis=1), -1, 1)
        cr = np.linalg.norm(np.cross(rays[:, 4:7], node[:, 4:7]), axis=1)
        a = np.arctan2(cr, cosang * np.linalg.norm(node[:, 4:7], axis=1)) - node[:, 7]
        a[node[:, 7] >= np.float32(math.pi)] = -1
        worst_s, worst_c = max(worst_s, ds.max()), max(worst_c, a.max())
        span *= B
    return worst_s, worst_c


@pytest.mark.parametrize("B0,B,Lv", [(8, 8, 2), (4, 8, 3), (16, 4, 2), (2, 2, 5), (64, 8, 1)])
def test_containment(orc, B0, B, Lv):
    for trial in range(3):
        n = int(rng.integers(1, 3000))
        o = rng.normal(size=(n, 3)) * rng.uniform(0.01, 3)
        d = rng.normal(size=(n, 3)) * np.array([0.1, 0.1, 1.0]) * rng.uniform(0.05, 1) + [0, 0, 1]
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        r = rays_from(o, d)
        lv = orc.build_levels(r, Lv, B0, B)
        ws, wc = containment_errors(lv, r.astype(np.float64), B0, B)
        assert ws <= 1e-5 and wc <= 1e-6


def test_sorted_rays_give_tighter_cones(orc):
    """for a fixed ray set, hash-sorted input gives a smaller mean leaf
    cone angle than the shuffled input (the paper's hypothesis)."""
    w = make_workload(1)
    prep = orc.ScenePrep(w.tris, w.mesh_ids)
    out = orc.trace(w, prep, taps=True)
    leaves_sorted = out["taps"]["levels"][0][0]
    rays = out["rays"][out["empty"] == 0]
    shuffled = rays[rng.permutation(rays.shape[0])]
    leaves_shuf = orc.build_levels(shuffled, 1, 8, 8)[0]
    assert leaves_sorted[:, 7].mean() < leaves_shuf[:, 7].mean()


# ----------------------------------------------------------------- traversal counts
def one_tri_scene(orc, tri):
    return orc.ScenePrep(np.asarray(tri, np.float32).reshape(1, 9), np.zeros(1, np.int32))


def test_worked_example_one_ray_one_triangle(orc):
    """1 ray aimed at 1 triangle, Lv=2 -> exactly one surviving pair at
    each level and one final test: (1,1), (1,1), final (1,1), mesh (1,1)."""
    prep = one_tri_scene(orc, [-1, -1, 5, 1, -1, 5, 0, 1, 5])
    r = rays_from(np.zeros((1, 3)), np.array([[0, 0, 1.0]]))
    lv = orc.build_levels(r, 2, 8, 8)
    best, cnt = orc.traverse(lv, r, prep, 2, 8, 8, orc.F_SORT | orc.F_MESH_CULL, 1)
    assert cnt[[1, 9, 0, 8, 16, 17, 18, 19]].tolist() == [1, 1, 1, 1, 1, 1, 1, 1]
    tri, t = orc.unpack(best)
    assert tri.tolist() == [0] and t[0] == pytest.approx(5.0)


def test_worked_example_mesh_behind(orc):
    """a mesh behind every cone -> zero pairs; the top nodes each count
    one mesh test and no triangle tests."""
    prep = one_tri_scene(orc, [-1, -1, -5, 1, -1, -5, 0, 1, -5])
    o = rng.normal(size=(200, 3)) * 0.1
    d = np.tile([0, 0, 1.0], (200, 1))
    r = rays_from(o, d)
    lv = orc.build_levels(r, 2, 8, 8)
    best, cnt = orc.traverse(lv, r, prep, 2, 8, 8, orc.F_SORT | orc.F_MESH_CULL, 2)
    assert cnt[16] == lv[1].shape[0] and cnt[17] == 0 and cnt[:16].sum() == 0 and cnt[18] == 0


def test_paper_table_identities():
    """The paper's counting convention read off Tables 1-4: per
    level misses + hits = tests; LEVEL-1 tests = 8 x LEVEL-2 hits; Table 4
    total = L2 + L1 + 8 x L1 hits; brute = rays x M (F2); reductions vs RAH."""
    g = json.load(open(os.path.join(HERE, "golden", "paper_tables.json")))
    tot = {}
    for row in g["rows"]:
        for lvl in ("L2", "L1"):
            t, m, h = row[lvl]
            assert m + h == t, row["cite"]
        assert row["L1"][0] == 8 * row["L2"][2], row["cite"]
        key = (row["scene"], row["alg"])
        tot[key] = tot.get(key, 0) + row["L2"][0] + row["L1"][0] + 8 * row["L1"][2]
    for t in g["totals"]:
        assert tot[(t["scene"], "RAH")] == t["RAH"] and tot[(t["scene"], "CRSH")] == t["CRSH"], t["cite"]
        assert f"{100 * t['CRSH'] / t['brute']:.2f}%" == t["rel"][2]
    assert g["totals"][0]["brute"] % g["rays"]["OFFICE"] == 0            # M = 36,308
    assert g["totals"][2]["brute"] // g["rays"]["SPONZA"] == 66450
    for t in g["totals"]:
        red = 100 * (1 - t["CRSH"] / t["RAH"])
        assert red == pytest.approx(g["reduction_vs_rah_pct"][t["scene"]], abs=0.01)


def test_oracle_counts_follow_the_paper_convention(orc):
    """Our counters obey the same identities as the paper's tables when every
    node is full (N a multiple of B0*B): tests[1] = B*hits[2], final = B0 *
    hits[1]; and with mesh culling off, tests[2] = N_top * M (F1, R14)."""
    w = make_micro(5, n_tris=40, W=32, H=16, n_meshes=4, n_lights=2, ray_types=1, empty_frac=0.0)
    prep = orc.ScenePrep(w.tris, w.mesh_ids)
    for flags in (orc.F_SORT | orc.F_MESH_CULL, orc.F_SORT):
        out = orc.trace(w, prep, flags=flags)
        st = out["stats"]
        N = st["rays"][0]
        assert N % 64 == 0
        assert st["tests"][0, 1] == 8 * st["hits"][0, 2]
        assert st["final_tests"][0] == 8 * st["hits"][0, 1]
        if flags == orc.F_SORT:
            assert st["tests"][0, 2] == (N // 64) * prep.M and st["mesh_tests"][0] == 0
        else:
            assert st["mesh_tests"][0] == (N // 64) * prep.n_meshes


# ----------------------------------------------------------------- ray generation closed forms
def test_generate_closed_forms(orc):
    """fragment (0,0,0), light (0,0,10) -> shadow ray origin (0,0,10),
    direction (0,0,-1), tmax = 10 - eps_t (R3); S:321 mirror identity; Snell
    with ior 1 passes straight through; S:319 invalid pixel -> empty slot."""
    from workloads.scenes import Workload, MATERIALS
    tris = np.array([[-20, -20, -1, 20, -20, -1, 0, 20, -1]], np.float32)
    pos = np.array([[0, 1], [0, 1], [0, 0]], np.float32)
    nrm = np.array([[0, 0], [0, 0], [1, 1]], np.float32)
    mats = np.array([[1.0, 0.0, 1.0], [0.0, 1.0, 1.0]], np.float32)
    w = Workload("cf", tris, np.zeros(1, np.int32), np.zeros(1, np.int32), mats,
                 np.array([[0, 0, 10]], np.float32), np.array([0, 0, 5], np.float32), 2, 1,
                 pos, nrm, np.array([0, -1], np.int32), 7)
    prep = orc.ScenePrep(w.tris, w.mesh_ids)
    rays, keys, empty = orc.generate(w, prep)
    assert empty.tolist() == [0, 1, 0, 1, 1, 1]          # SH p0, SH p1(invalid), RE p0, RE p1, RR p0 (mat0 refl only)
    assert np.allclose(rays[0, :3], [0, 0, 10]) and np.allclose(rays[0, 4:7], [0, 0, -1])
    assert rays[0, 7] == np.float32(10 - prep.eps_t) and rays[0, 3] == np.float32(prep.eps_t)
    assert np.allclose(rays[2, 4:7], [0, 0, 1]) and rays[2, 7] == np.inf     # eye above, normal +z: mirror up
    # refraction with ior 1 (material 1): straight through
    w.mat = np.array([1, -1], np.int32)
    rays, keys, empty = orc.generate(w, prep)
    assert empty[4] == 0 and np.allclose(rays[4, 4:7], [0, 0, -1], atol=1e-7)
    # Snell's law with ior 1.5 at 30 degrees incidence (fp64 closed form)
    w.materials = np.array([[0, 0, 1], [0, 1, 1.5]], np.float32)
    w.eye = np.array([0, -math.tan(math.radians(30)) * 5, 5], np.float32)
    rays, keys, empty = orc.generate(w, prep)
    d = rays[4, 4:7].astype(np.float64)
    sin_t = math.hypot(d[0], d[1])
    i = -w.eye.astype(np.float64) / np.linalg.norm(w.eye)
    sin_i = math.hypot(i[0], i[1])
    assert sin_i / sin_t == pytest.approx(1.5, rel=1e-5) and d[2] < 0


# ----------------------------------------------------------------- end to end
def brute_np(rays, tris):
    """Independent fp64 closest-hit reference (plane + edge functions).  Per ray:
    (best triangle or -1, its t, the runner-up t, the best hit's smallest
    normalised edge distance)."""
    V = tris.reshape(-1, 3, 3).astype(np.float64)
    n = np.cross(V[:, 1] - V[:, 0], V[:, 2] - V[:, 0])
    area = np.linalg.norm(n, axis=1)
    out = []
    for r in rays.astype(np.float64):
        o, d, tmin, tmax = r[:3], r[4:7], r[3], r[7]
        den = n @ d
        with np.errstate(divide="ignore", invalid="ignore"):
            t = ((V[:, 0] - o) * n).sum(1) / den
            p = o + t[:, None] * d
            e = [np.einsum("ij,ij->i", np.cross(V[:, (k + 1) % 3] - V[:, k], p - V[:, k]), n) / area
                 for k in range(3)]
        inside = ((e[0] >= 0) & (e[1] >= 0) & (e[2] >= 0)) | ((e[0] <= 0) & (e[1] <= 0) & (e[2] <= 0))
        ok = inside & (t > tmin) & (t < tmax) & (den != 0)
        tt = np.where(ok, t, np.inf)
        if not ok.any():
            out.append((-1, np.inf, np.inf, np.inf))
            continue
        order = np.argsort(tt)
        b = order[0]
        second = tt[order[1]] if len(order) > 1 else np.inf
        margin = min(abs(e[k][b]) for k in range(3)) / np.sqrt(area[b])
        out.append((int(b), tt[b], second, margin))
    return out


def test_brute_matches_fp64_reference(orc):
    """The oracle's brute force (float32 MT) agrees with an independent fp64
    closest-hit computation: the same triangle for every ray whose fp64 hit is
    clear (runner-up more than 1e-4 farther, hit point more than 1e-4 from the
    triangle's edges), t within 1e-4, and the same hit/miss verdict on >= 97 %
    of all rays (the rest graze an edge)."""
    w = make_micro(11, n_tris=48, W=8, H=8)
    prep = orc.ScenePrep(w.tris, w.mesh_ids)
    rays, keys, empty = orc.generate(w, prep)
    rays = rays[empty == 0]
    tri, t = orc.unpack(orc.brute(rays, prep))
    ref = brute_np(rays, w.tris)
    clear = 0
    for k, (rt, rtt, second, margin) in enumerate(ref):
        if rt >= 0 and second - rtt > 1e-4 and margin > 1e-4:
            assert tri[k] == rt, (k, tri[k], rt)
            assert t[k] == pytest.approx(rtt, rel=1e-4, abs=1e-4)
            clear += 1
        if rt >= 0 and tri[k] >= 0:
            assert t[k] == pytest.approx(rtt, rel=1e-4, abs=1e-4)
    assert clear > 20
    assert np.mean([(r[0] >= 0) == (tri[k] >= 0) for k, r in enumerate(ref)]) > 0.97


@pytest.mark.parametrize("seed", range(100))
def test_crsh_equals_brute_on_micro_scenes(orc, seed):
    """Acceptance 5: over 100 randomised micro-scenes (<= 64 triangles,
    <= 256 rays per type), the CRSH closest hit equals the N x M brute force
    for every ray -- culling is conservative."""
    r = np.random.default_rng(seed)
    w = make_micro(1000 + seed, n_tris=int(r.integers(1, 65)), W=int(r.integers(1, 12)), H=int(r.integers(1, 12)),
                   n_meshes=int(r.integers(1, 6)), n_lights=int(r.integers(1, 4)), ray_types=int(r.integers(1, 8)),
                   levels=int(r.integers(1, 4)), leaf_size=int(2 ** r.integers(1, 5)), branching=int(2 ** r.integers(1, 4)))
    prep = orc.ScenePrep(w.tris, w.mesh_ids)
    out = orc.trace(w, prep, n_threads=2)
    ok = out["empty"] == 0
    tri, t = orc.unpack(orc.brute(out["rays"][ok], prep, 2))
    assert np.array_equal(out["hit_tri"][ok], tri) and np.array_equal(out["t"][ok], t)
    assert np.all(out["hit_tri"][~ok] == -2)
    # RAH flags (no sort, no mesh culling) and the Z-order hash find the same
    # hits (engines differ only in which tests are skipped)
    for flags in (0, orc.F_SORT | orc.F_MESH_CULL | orc.F_ZORDER):
        out2 = orc.trace(w, prep, flags=flags, n_threads=2)
        assert np.array_equal(out2["hit_tri"], out["hit_tri"]) and np.array_equal(out2["t"], out["t"])


def test_crsh_equals_brute_cfg1(orc):
    """cfg1 (128x128 SH, ~1k triangles, Lv 3): exact N x M equality; the
    totals are below brute force; thread count does not change anything
    (S:628)."""
    w = make_workload(1)
    prep = orc.ScenePrep(w.tris, w.mesh_ids)
    a = orc.trace(w, prep, n_threads=1)
    b = orc.trace(w, prep, n_threads=8)
    ok = a["empty"] == 0
    tri, t = orc.unpack(orc.brute(a["rays"][ok], prep))
    assert np.array_equal(a["hit_tri"][ok], tri) and np.array_equal(a["t"][ok], t)
    assert np.array_equal(a["hit_tri"], b["hit_tri"]) and np.array_equal(a["t"], b["t"])
    for k in ("tests", "hits"):
        assert np.array_equal(a["stats"][k], b["stats"][k])
    st = a["stats"]
    total = int(st["tests"].sum()) + sum(st["final_tests"])
    assert total < sum(st["brute"])
