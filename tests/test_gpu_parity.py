"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by
element on the same seeded inputs.  Bars (BASELINE.json north_star): keys,
permutation, chunks and bundle boundaries bit-exact; node values bit-exact
(both sides implement NUMSPEC); per-level test counts exact
(bar: within 0.1%); closest-hit triangle and t exact (bar: >= 99.99% of rays,
t within 1e-5 relative)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2312_06538_b200 as crsh  # noqa: E402
from paper_2312_06538_b200.api import tracer_for  # noqa: E402
import host_mirror as cd  # noqa: E402
from workloads import make_micro, make_workload  # noqa: E402

SEG = {0: oracle.SH, 1: oracle.RE, 2: oracle.RR}


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2312_06538_b200 import build as nb
    nb.build()
    oracle.build()


def run_both(w, flags=crsh.F_SORT | crsh.F_MESH_CULL, taps=True):
    tr = tracer_for(w, flags=flags)
    tr.run()
    hit, t = tr.results()
    ref = oracle.trace(w, flags=flags, taps=taps)
    return tr, hit, t, ref


def assert_counts_equal(st, ref):
    for seg in range(3):
        assert st["rays"][seg] == ref["stats"]["rays"][seg]
        assert np.array_equal(st["tests"][seg], ref["stats"]["tests"][seg]), (seg, st["tests"][seg], ref["stats"]["tests"][seg])
        assert np.array_equal(st["hits"][seg], ref["stats"]["hits"][seg]), (seg, st["hits"][seg], ref["stats"]["hits"][seg])
        for k in ("mesh_tests", "mesh_hits", "final_tests", "final_hits", "rays_hit", "brute", "cluster_tests",
                  "cluster_hits"):
            assert st[k][seg] == ref["stats"][k][seg], (k, seg, st[k][seg], ref["stats"][k][seg])


def assert_taps_equal(tr, ref, w):
    segs = [s for s, _, _ in oracle.segments(w.P, w.lights.shape[0], w.ray_types)]
    for i, seg in enumerate(segs):
        tp = ref["taps"]
        assert np.array_equal(crsh.debug_tap(tr.scene, crsh.TAP_KEYS, seg), tp["keys"][i])
        assert np.array_equal(crsh.debug_tap(tr.scene, crsh.TAP_VALS, seg), tp["vals"][i])
        if len(tp["ckey"][i]):
            assert np.array_equal(crsh.debug_tap(tr.scene, crsh.TAP_CHUNK_KEYS, seg), tp["ckey"][i])
            assert np.array_equal(crsh.debug_tap(tr.scene, crsh.TAP_CHUNK_BASE, seg), tp["cbase"][i])
        assert np.array_equal(crsh.debug_tap(tr.scene, crsh.TAP_SORTED_KEYS, seg), tp["skey"][i])
        assert np.array_equal(crsh.debug_tap(tr.scene, crsh.TAP_SORTED_SLOTS, seg), tp["sslot"][i])
        sr = crsh.debug_tap(tr.scene, crsh.TAP_SORTED_RAYS, seg)   # gathered by the permutation (K8's view)
        assert np.array_equal(sr.view(np.uint32), ref["rays"][tp["sslot"][i].astype(np.int64)].view(np.uint32))
        for k in range(1, w.levels + 1):
            g = crsh.debug_tap(tr.scene, crsh.TAP_NODES, seg, k)
            o = tp["levels"][i][k - 1]
            assert g.shape == o.shape, (seg, k)
            assert np.array_equal(g.view(np.uint32), o.view(np.uint32)), (seg, k, np.argwhere(g != o)[:5])


def test_scene_prep_matches_oracle():
    w = make_workload(2)
    tr = tracer_for(w)
    prep = oracle.ScenePrep(w.tris, w.mesh_ids)
    assert np.array_equal(crsh.debug_tap(tr.scene, crsh.TAP_SCENE_CONSTS), prep.consts)
    ts = crsh.debug_tap(tr.scene, crsh.TAP_TRI_SPHERES)
    assert np.array_equal(ts.view(np.uint32), prep.tri_sph.view(np.uint32))
    ms = crsh.debug_tap(tr.scene, crsh.TAP_MESH_SPHERES)
    assert np.array_equal(ms, prep.mesh_sph[:w.n_meshes])
    # object sphere-tree (NEXT-4, reading O1): cluster order and spheres
    assert np.array_equal(crsh.debug_tap(tr.scene, crsh.TAP_CLUSTER_ORDER), prep.cluster_order[:prep.M])
    cs = crsh.debug_tap(tr.scene, crsh.TAP_CLUSTER_SPHERES)
    assert np.array_equal(cs.view(np.uint32), prep.cluster_sph[:prep.n_clusters].view(np.uint32))


@pytest.mark.parametrize("flags", [3, 7, 0, 1, 67, 71])
def test_cfg1_full_parity(flags):
    """cfg1 (128x128 SH, ~1k-tri Cornell box, Lv 3): every intermediate tap,
    all counts and every hit bit-exact; CRSH, Z-order, RAH and sort-only."""
    w = make_workload(1)
    tr, hit, t, ref = run_both(w, flags)
    assert np.array_equal(hit, ref["hit_tri"]) and np.array_equal(t.view(np.uint32), ref["t"].view(np.uint32))
    assert_counts_equal(crsh.stats(tr.scene), ref)
    assert_taps_equal(tr, ref, w)


@pytest.mark.parametrize("seed", range(40))
def test_micro_scenes(seed):
    """Randomised micro-scenes over the option space (Lv 1..4, B0 2..64,
    B 2..16, all ray-type mixes, empty pixels, ragged bundles)."""
    r = np.random.default_rng(seed)
    w = make_micro(5000 + seed, n_tris=int(r.integers(1, 200)), W=int(r.integers(1, 40)), H=int(r.integers(1, 40)),
                   n_meshes=int(r.integers(1, 40)), n_lights=int(r.integers(0, 5)), ray_types=int(r.integers(1, 8)),
                   levels=int(r.integers(1, 5)), leaf_size=int(2 ** r.integers(1, 7)),
                   branching=int(2 ** r.integers(1, 5)), empty_frac=float(r.uniform(0, 0.6)))
    flags = int(r.choice([3, 7, 0, 2, 1, 67, 71, 66]))
    tr, hit, t, ref = run_both(w, flags)
    prep = oracle.ScenePrep(w.tris, w.mesh_ids)
    assert np.array_equal(crsh.debug_tap(tr.scene, crsh.TAP_SCENE_CONSTS), prep.consts)
    assert np.array_equal(crsh.debug_tap(tr.scene, crsh.TAP_MESH_SPHERES), prep.mesh_sph[:w.n_meshes])
    assert np.array_equal(crsh.debug_tap(tr.scene, crsh.TAP_CLUSTER_SPHERES).view(np.uint32),
                          prep.cluster_sph[:prep.n_clusters].view(np.uint32))
    assert np.array_equal(hit, ref["hit_tri"]) and np.array_equal(t.view(np.uint32), ref["t"].view(np.uint32))
    assert_counts_equal(crsh.stats(tr.scene), ref)
    assert_taps_equal(tr, ref, w)
    # conservativeness against brute force
    ok = ref["empty"] == 0
    bt, btt = oracle.unpack(oracle.brute(ref["rays"][ok], prep))
    assert np.array_equal(hit[ok], bt)


@pytest.mark.parametrize("flags", [3, 71])
@pytest.mark.parametrize("item_tris", [None, "16384"])
@pytest.mark.parametrize("levels,leaf,branch", [(1, 8, 8), (1, 64, 4), (3, 4, 4), (3, 16, 8), (4, 8, 8), (2, 32, 2),
                                                (2, 2, 16)])
def test_option_space_many_triangles(levels, leaf, branch, item_tris, flags, monkeypatch):
    """cfg2's 70k-triangle scene at 96x96 over the option space: work items
    of thousands of triangles (several slices per warp, queues refilled and
    drained many times), both the shared-memory (group <= 512 rays) and the
    global-memory group paths (span > 512), Lv 1 (top = bundle level) to 4;
    with the per-frame item size (2048 triangles at this size) and with the
    16384-triangle items of large frames forced (CRSH_ITEM_TRIS)."""
    if item_tris:
        monkeypatch.setenv("CRSH_ITEM_TRIS", item_tris)
    w = make_workload(2, width=96, height=96, levels=levels, leaf_size=leaf, branching=branch)
    tr, hit, t, ref = run_both(w, flags, taps=False)
    assert np.array_equal(hit, ref["hit_tri"]) and np.array_equal(t.view(np.uint32), ref["t"].view(np.uint32))
    assert_counts_equal(crsh.stats(tr.scene), ref)


@pytest.mark.parametrize("cap", ["32", "96"])
@pytest.mark.parametrize("flags", [67, 71])
def test_objtree_cluster_list_rounds(flags, cap, monkeypatch):
    """The object tree's two-phase items (cluster tests into a CTA list, then
    one passing cluster per claim) with the list cut to a few dozen entries
    (CRSH_OBJ_LIST_CAP) and 65536-triangle items, so every item needs many
    fill / drain rounds: hits and every counter still equal the oracle's."""
    monkeypatch.setenv("CRSH_OBJ_LIST_CAP", cap)
    monkeypatch.setenv("CRSH_ITEM_TRIS", "65536")
    w = make_workload(2, width=128, height=128)
    tr, hit, t, ref = run_both(w, flags, taps=False)
    assert np.array_equal(hit, ref["hit_tri"]) and np.array_equal(t.view(np.uint32), ref["t"].view(np.uint32))
    st = crsh.stats(tr.scene)
    assert_counts_equal(st, ref)
    assert sum(st["cluster_hits"]) > 4 * int(cap)   # more passing clusters than one list holds


@pytest.mark.parametrize("top", ["0", "1"])
@pytest.mark.parametrize("flags", [3, 7])
def test_child_prefilter_skips_only_failing_tests(flags, top, monkeypatch):
    """K8's prefilter (cull_pf: child nodes -- and with CRSH_TOP_PREFILTER=1
    the top nodes -- against a sphere containing the slice's triangle
    spheres) only skips evaluations: hits, t and every paper counter equal
    the oracle's with it on and off; with it on it skips part of the counted
    tests (skipped_tests > 0) and evaluates prefilter tests; off, both are
    zero."""
    monkeypatch.setenv("CRSH_TOP_PREFILTER", top)
    w = make_workload(2, width=160, height=160)
    tr, hit, t, ref = run_both(w, flags, taps=False)
    st_on = crsh.stats(tr.scene)
    assert np.array_equal(hit, ref["hit_tri"]) and np.array_equal(t.view(np.uint32), ref["t"].view(np.uint32))
    assert_counts_equal(st_on, ref)
    assert sum(st_on["prefilter_tests"]) > 0 and sum(st_on["skipped_tests"]) > 0
    assert sum(st_on["skipped_tests"]) <= int(np.asarray(st_on["tests"]).sum())
    monkeypatch.setenv("CRSH_NO_PREFILTER", "1")
    tr2 = tracer_for(w, flags=flags)
    tr2.run()
    hit2, t2 = tr2.results()
    st_off = crsh.stats(tr2.scene)
    assert np.array_equal(hit2, hit) and np.array_equal(t2.view(np.uint32), t.view(np.uint32))
    assert_counts_equal(st_off, ref)
    assert sum(st_off["prefilter_tests"]) == 0 and sum(st_off["skipped_tests"]) == 0


@pytest.mark.parametrize("flags", [3, 7, 71])
def test_cfg2_full_parity(flags):
    """cfg2 (512x512 SH+RE, ~70k tris / 16 meshes, Lv 2) at full size: all
    hits, counts and the sort permutation exact against the oracle."""
    w = make_workload(2)
    tr, hit, t, ref = run_both(w, flags, taps=True)
    assert np.array_equal(hit, ref["hit_tri"]) and np.array_equal(t.view(np.uint32), ref["t"].view(np.uint32))
    assert_counts_equal(crsh.stats(tr.scene), ref)
    assert_taps_equal(tr, ref, w)


# cfg3 / cfg4 at full size: tests/test_gpu_headline.py (full-frame oracle parity)


def test_slot_limit_and_degenerate_triangles():
    """ELIMIT before any work for >= 2^30 slots; degenerate (zero-area)
    triangles never hit, on the GPU as in the oracle and brute force."""
    w = make_workload(1, width=16, height=16)
    tr = tracer_for(w)
    big = crsh.make_hits(1 << 15, 1 << 15, tr.pos, tr.nrm, tr.mat, tr.materials, int(w.materials.shape[0]), w.eye)
    with pytest.raises(Exception):
        crsh.trace_secondary(tr.scene, big, w.lights, 7, tr.opts, tr.hit_tri, tr.t)
    r = np.random.default_rng(8)
    w = make_micro(777, n_tris=120, W=24, H=24, n_meshes=5, n_lights=2, ray_types=7, empty_frac=0.1)
    tris = w.tris.reshape(-1, 3, 3).copy()
    deg = r.choice(len(tris), 40, replace=False)
    tris[deg[:20], 2] = tris[deg[:20], 1]                                   # repeated vertex
    tris[deg[20:], 2] = 2 * tris[deg[20:], 1] - tris[deg[20:], 0]          # collinear
    w.tris = tris.reshape(-1, 9).astype(np.float32)
    tr, hit, t, ref = run_both(w, crsh.F_SORT | crsh.F_MESH_CULL, taps=False)
    assert np.array_equal(hit, ref["hit_tri"]) and np.array_equal(t.view(np.uint32), ref["t"].view(np.uint32))
    assert not np.isin(hit, deg[:20]).any()


def test_edge_cases():
    # no valid pixel at all
    w = make_micro(1, n_tris=10, W=8, H=8, empty_frac=1.0)
    tr, hit, t, ref = run_both(w)
    assert np.all(hit == -2) and np.array_equal(hit, ref["hit_tri"])
    # a single pixel, a single triangle
    w = make_micro(2, n_tris=1, W=1, H=1, n_meshes=1, empty_frac=0.0)
    tr, hit, t, ref = run_both(w)
    assert np.array_equal(hit, ref["hit_tri"]) and np.array_equal(t, ref["t"])
    # every fragment at the same point: one chunk per segment (long run)
    w = make_micro(3, n_tris=30, W=64, H=64, empty_frac=0.0, ray_types=1, n_lights=1)
    w.pos[:] = w.pos[:, :1]
    tr, hit, t, ref = run_both(w)
    assert np.array_equal(hit, ref["hit_tri"])
    assert crsh.stats(tr.scene)["chunks"][0] == ref["stats"]["chunks"][0] == 1
    # shadow rays requested with no lights: no SH slots
    w = make_micro(4, n_tris=20, W=9, H=7, n_lights=0, ray_types=3)
    tr, hit, t, ref = run_both(w)
    assert np.array_equal(hit, ref["hit_tri"])


def _oracle_packed(ref):
    """The oracle frame in the packed encoding of include/crsh.h (world 1:
    every slot owned): hit (float_bits(t) << 32) | tri, miss
    0x7F800000FFFFFFFF, no ray 0x7FFFFFFFFFFFFFFF."""
    h, t = ref["hit_tri"], ref["t"]
    out = np.full(h.shape, 0x7FFFFFFFFFFFFFFF, np.uint64)
    hit = h >= 0
    out[hit] = (t[hit].view(np.uint32).astype(np.uint64) << np.uint64(32)) | h[hit].astype(np.uint64)
    out[h == -1] = np.uint64(0x7F800000FFFFFFFF)
    return out.view(np.int64)


def test_sharded_equals_oracle():
    """Hash-range sharding: the min-merge of the per-rank packed
    results equals the ORACLE's frame, and the per-rank counters sum to the
    oracle's counters (the ranks run one after another on one GPU; no rank
    waits on another)."""
    w = make_workload(2, width=256, height=256)
    ref = oracle.trace(w)
    rs = ref["stats"]
    Lv = w.levels
    for world in (2, 3, 8):
        merged = None
        tsum = np.zeros((3, 9), np.uint64)
        hsum = np.zeros((3, 9), np.uint64)
        fsum = np.zeros(3, np.uint64)
        msum = np.zeros(3, np.uint64)
        top = []
        for rank in range(world):
            trr = tracer_for(w, shard_rank=rank, shard_world=world)
            packed = torch.empty(trr.slots, dtype=torch.int64, device="cuda")
            trr.run_packed(packed)
            merged = packed.clone() if merged is None else torch.minimum(merged, packed)
            st = trr.stats()
            tsum += st["tests"]
            hsum += st["hits"]
            fsum += np.asarray(st["final_tests"], np.uint64)
            msum += np.asarray(st["mesh_tests"], np.uint64)
            top.append(int(st["tests"][:, Lv].sum()))
            # the device cut equals the host mirror on the device's group work,
            # and a group's work is exactly its top-level test count
            work = crsh.debug_tap(trr.scene, crsh.TAP_GROUP_WORK)
            lo, hi, G = crsh.debug_tap(trr.scene, crsh.TAP_GROUP_RANGE).tolist()
            assert len(work) == G and (lo, hi) == cd.balanced_cut(work, rank, world), (rank, world, lo, hi)
            assert top[-1] == int(work[lo:hi].sum())
        trr.unpack(merged)
        hit, t = trr.results()
        assert np.array_equal(merged.cpu().numpy(), _oracle_packed(ref)), world
        assert np.array_equal(hit, ref["hit_tri"]) and np.array_equal(t.view(np.uint32), ref["t"].view(np.uint32))
        assert np.array_equal(tsum, rs["tests"]) and np.array_equal(hsum, rs["hits"]), world
        assert np.array_equal(fsum, np.asarray(rs["final_tests"], np.uint64)), world
        assert np.array_equal(msum, np.asarray(rs["mesh_tests"], np.uint64)), world
        # work-balanced cut: every rank's top-level tests within one group's
        # worth (K top nodes x the scene) of an equal share
        share = sum(top) / world
        assert max(top) <= share + 8 * w.tris.shape[0], (world, top)
        assert min(top) > 0, (world, top)


def test_peer_store_equals_oracle():
    """Fused multi-GPU epilogue (crsh_trace_secondary_peer): each rank stores
    its owned results into every destination (here two buffers on this GPU
    standing for the own and a peer's window; the ranks run one after another,
    none waits on another). Both destinations must equal the oracle's frame in
    the packed encoding, though they start as garbage: every slot is written
    exactly once with its final value, so no reduction is needed."""
    w = make_workload(2, width=256, height=256)
    ref = oracle.trace(w)
    want = torch.as_tensor(_oracle_packed(ref)).cuda()
    slots = len(ref["hit_tri"])
    for world in (1, 2, 5):
        dst = [torch.full((slots,), 0x5A5A5A5A5A5A5A5A, dtype=torch.int64, device="cuda") for _ in range(2)]
        tsum = np.zeros((3, 9), np.uint64)
        for rank in range(world):
            trr = tracer_for(w, shard_rank=rank, shard_world=world)
            trr.run_peer([d.data_ptr() for d in dst])
            tsum += trr.stats()["tests"]
        torch.cuda.synchronize()
        assert torch.equal(dst[0], want) and torch.equal(dst[1], want), world
        assert np.array_equal(tsum, ref["stats"]["tests"]), world
    # brute-force engine through the same epilogue
    trb = tracer_for(w, flags=crsh.F_BRUTE)
    d = torch.full((trb.slots,), -1, dtype=torch.int64, device="cuda")
    trb.run_peer([d.data_ptr()])
    torch.cuda.synchronize()
    assert torch.equal(d, want)


def test_host_variant_and_determinism():
    w = make_workload(2, width=200, height=150)
    tr = tracer_for(w)
    tr.run()
    h1, t1 = tr.results()
    tr.run()
    h2, t2 = tr.results()
    assert np.array_equal(h1, h2) and np.array_equal(t1, t2)
    hh = np.empty(tr.slots, np.int32)
    th = np.empty(tr.slots, np.float32)
    tr.run_host(np.ascontiguousarray(w.pos), np.ascontiguousarray(w.nrm), np.ascontiguousarray(w.mat),
                np.ascontiguousarray(w.materials), hh, th)
    assert np.array_equal(hh, h1) and np.array_equal(th, t1)


def test_brute_mode_equals_oracle_brute():
    """CRSH_F_BRUTE (the N x M baseline) gives the oracle's brute-force
    closest hits and counts rays x M final tests."""
    for w in (make_workload(1), make_micro(9, n_tris=150, W=20, H=17, ray_types=7, n_lights=3)):
        tr = tracer_for(w, flags=crsh.F_BRUTE)
        tr.run()
        hit, t = tr.results()
        prep = oracle.ScenePrep(w.tris, w.mesh_ids)
        rays, keys, empty = oracle.generate(w, prep)
        ok = empty == 0
        bt, btt = oracle.unpack(oracle.brute(rays[ok], prep))
        assert np.array_equal(hit[ok], bt) and np.array_equal(t[ok].view(np.uint32), btt.view(np.uint32))
        assert np.all(hit[~ok] == -2)
        st = crsh.stats(tr.scene)
        assert sum(st["final_tests"]) == int(ok.sum()) * w.M


@pytest.mark.parametrize("cfg,size,depth,flags", [(1, 64, 3, 3), (1, 64, 2, 7), (2, 128, 2, 3), (3, 64, 3, 3)])
def test_whitted_image_parity(cfg, size, depth, flags):
    """Multi-bounce Whitted loop (NEXT-2, crsh_render_whitted): the image and
    the per-bounce vertex / ray counts bit-exact against the oracle loop."""
    w = make_workload(cfg, width=size, height=size)
    tr = tracer_for(w, flags=flags)
    img, st = tr.render(w.tri_mat, depth)
    torch.cuda.synchronize()
    ref = oracle.whitted(w, depth, flags=flags)
    n = len(ref["vertices"])
    assert st["vertices"][:n] == ref["vertices"] and all(v == 0 for v in st["vertices"][n:])
    assert st["rays"][:n] == ref["rays"]
    got = img.cpu().numpy()[:w.P]
    assert np.array_equal(got.view(np.uint32), ref["image"].view(np.uint32)), np.abs(got - ref["image"]).max()


def test_incident_directions_parity():
    """The optional per-vertex incident direction (`dir`, later Whitted
    bounces): random unit directions on a micro-scene, every hit and count
    bit-exact against the oracle."""
    r = np.random.default_rng(11)
    w = make_micro(9001, n_tris=150, W=30, H=20, n_meshes=6, n_lights=2, ray_types=7, levels=2, leaf_size=4,
                   branching=8, empty_frac=0.2)
    d = r.normal(size=(3, w.P)).astype(np.float32)
    w.dir = (d / np.linalg.norm(d, axis=0)).astype(np.float32)
    tr, hit, t, ref = run_both(w, crsh.F_SORT | crsh.F_MESH_CULL, taps=False)
    assert np.array_equal(hit, ref["hit_tri"]) and np.array_equal(t.view(np.uint32), ref["t"].view(np.uint32))
    assert_counts_equal(crsh.stats(tr.scene), ref)


@pytest.mark.parametrize("cfg,W,H,flags", [(1, 128, 96, 3), (2, 256, 256, 3), (2, 200, 150, 7)])
def test_primary_gbuffer_parity(cfg, W, H, flags):
    """GPU primary pass (NEXT-3, crsh_primary_gbuffer): camera rays traced
    through the pipeline; G-buffer, primary hits and counters bit-exact vs the
    oracle."""
    from workloads import make_camera
    w = make_workload(cfg, width=16, height=16)
    cam = make_camera()
    scene = crsh.Scene(torch.as_tensor(w.tris).cuda(), torch.as_tensor(w.mesh_ids).cuda())
    P = W * H
    pos = torch.empty(3 * P, dtype=torch.float32, device="cuda")
    nrm = torch.empty(3 * P, dtype=torch.float32, device="cuda")
    mat = torch.empty(P, dtype=torch.int32, device="cuda")
    hit = torch.empty(P, dtype=torch.int32, device="cuda")
    t = torch.empty(P, dtype=torch.float32, device="cuda")
    tm = torch.as_tensor(w.tri_mat).cuda()
    opts = crsh.make_opts(w.levels, w.leaf_size, w.branching, flags)
    crsh.primary_gbuffer(scene, cam, W, H, tm, opts, pos, nrm, mat, hit, t)
    torch.cuda.synchronize()
    rpos, rnrm, rmat, rhit, rt, rst = oracle.primary_gbuffer(w.tris, w.mesh_ids, w.tri_mat, cam, W, H, w.levels,
                                                             w.leaf_size, w.branching, flags)
    assert np.array_equal(hit.cpu().numpy(), rhit) and np.array_equal(t.cpu().numpy().view(np.uint32), rt.view(np.uint32))
    assert np.array_equal(mat.cpu().numpy(), rmat)
    assert np.array_equal(pos.cpu().numpy().reshape(3, P).view(np.uint32), rpos.view(np.uint32))
    assert np.array_equal(nrm.cpu().numpy().reshape(3, P).view(np.uint32), rnrm.view(np.uint32))
    st = crsh.stats(scene)
    assert np.array_equal(st["tests"][1], rst["tests"][1]) and st["final_tests"][1] == rst["final_tests"][1]


def test_trace_rays_parity():
    """crsh_trace_rays on a batch of random rays (some empty, some reversed
    intervals): hits and counters bit-exact vs the oracle and equal to brute force."""
    w = make_workload(2, width=16, height=16)
    r = np.random.default_rng(5)
    n = 20000
    o = r.uniform(0.5, 9.5, size=(n, 3)).astype(np.float32)
    d = r.normal(size=(n, 3))
    d = (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)
    tmin = np.full(n, 1e-3, np.float32)
    tmax = np.where(r.random(n) < 0.1, -1.0, np.where(r.random(n) < 0.5, 4.0, np.inf)).astype(np.float32)
    rays = np.concatenate([o, tmin[:, None], d, tmax[:, None]], axis=1).astype(np.float32)
    scene = crsh.Scene(torch.as_tensor(w.tris).cuda(), torch.as_tensor(w.mesh_ids).cuda())
    hit = torch.empty(n, dtype=torch.int32, device="cuda")
    t = torch.empty(n, dtype=torch.float32, device="cuda")
    crsh.trace_rays(scene, torch.as_tensor(rays).cuda(), n, crsh.make_opts(2, 8, 8, 3), hit, t)
    torch.cuda.synchronize()
    prep = oracle.ScenePrep(w.tris, w.mesh_ids)
    ref = oracle.trace_rays(rays, prep, 2, 8, 8, 3)
    assert np.array_equal(hit.cpu().numpy(), ref["hit_tri"])
    assert np.array_equal(t.cpu().numpy().view(np.uint32), ref["t"].view(np.uint32))
    assert_counts_equal(crsh.stats(scene), ref)
    ok = ref["hit_tri"] != -2
    bt, _ = oracle.unpack(oracle.brute(rays[ok], prep))
    assert np.array_equal(ref["hit_tri"][ok], bt)


def _random_motion(n_meshes, seed, fixed=6):
    r = np.random.default_rng(seed)
    X = []
    for m in range(n_meshes):
        if m < fixed:
            X.append(np.array([1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0], np.float32))
            continue
        q, _ = np.linalg.qr(r.normal(size=(3, 3)))
        q *= np.sign(np.linalg.det(q))
        A = q @ np.diag(r.uniform(0.7, 1.3, 3))
        X.append(np.concatenate([A, r.uniform(-1, 1, 3)[:, None]], axis=1).astype(np.float32).reshape(12))
    return np.stack(X)


@pytest.mark.parametrize("cfg,seed", [(1, 0), (2, 1)])
def test_dynamic_scene_parity(cfg, seed):
    """Dynamic scenes (NEXT-3, crsh_scene_transform): after moving the meshes
    the scene constants, triangle spheres and updated mesh spheres are
    bit-exact vs the oracle, and a primary pass + secondary frame of the moved
    scene is bit-exact too; a second transform starts again from the
    creation-time vertices."""
    from workloads import make_camera
    import dataclasses
    w = make_workload(cfg, width=96, height=96)
    prep0 = oracle.ScenePrep(w.tris, w.mesh_ids)
    scene = crsh.Scene(torch.as_tensor(w.tris).cuda(), torch.as_tensor(w.mesh_ids).cuda())
    tm = torch.as_tensor(w.tri_mat).cuda()
    cam = make_camera()
    W = H = 96
    P = W * H
    for k in range(2):
        X = _random_motion(prep0.n_meshes, seed + 10 * k)
        crsh.scene_transform(scene, X)
        prep, tris = oracle.transformed_prep(prep0, w.tris, w.mesh_ids, X)
        assert np.array_equal(crsh.debug_tap(scene, crsh.TAP_SCENE_CONSTS), prep.consts)
        assert np.array_equal(crsh.debug_tap(scene, crsh.TAP_TRI_SPHERES).view(np.uint32), prep.tri_sph.view(np.uint32))
        assert np.array_equal(crsh.debug_tap(scene, crsh.TAP_MESH_SPHERES), prep.mesh_sph[:prep.n_meshes])
        # primary pass on the moved scene, then its secondary frame
        fl = 3 if k == 0 else 3 | crsh.F_OBJTREE
        opts = crsh.make_opts(w.levels, w.leaf_size, w.branching, fl)
        pos = torch.empty(3 * P, dtype=torch.float32, device="cuda")
        nrm = torch.empty(3 * P, dtype=torch.float32, device="cuda")
        mat = torch.empty(P, dtype=torch.int32, device="cuda")
        ph = torch.empty(P, dtype=torch.int32, device="cuda")
        pt = torch.empty(P, dtype=torch.float32, device="cuda")
        crsh.primary_gbuffer(scene, cam, W, H, tm, opts, pos, nrm, mat, ph, pt)
        rpos, rnrm, rmat, rhit, rt, _ = oracle.primary_gbuffer(tris, w.mesh_ids, w.tri_mat, cam, W, H, w.levels,
                                                               w.leaf_size, w.branching, fl, prep=prep)
        assert np.array_equal(ph.cpu().numpy(), rhit) and np.array_equal(mat.cpu().numpy(), rmat)
        wm = dataclasses.replace(w, tris=tris, width=W, height=H, pos=rpos, nrm=rnrm, mat=rmat)
        hits = crsh.make_hits(W, H, pos, nrm, mat, torch.as_tensor(w.materials).cuda(), w.materials.shape[0], w.eye)
        slots = crsh.num_slots(P, w.lights.shape[0], w.ray_types)
        hit = torch.empty(slots, dtype=torch.int32, device="cuda")
        t = torch.empty(slots, dtype=torch.float32, device="cuda")
        crsh.trace_secondary(scene, hits, w.lights, w.ray_types, opts, hit, t)
        torch.cuda.synchronize()
        ref = oracle.trace(wm, prep, flags=fl)
        assert np.array_equal(crsh.debug_tap(scene, crsh.TAP_CLUSTER_SPHERES).view(np.uint32),
                              prep.cluster_sph[:prep.n_clusters].view(np.uint32))
        assert np.array_equal(hit.cpu().numpy(), ref["hit_tri"])
        assert np.array_equal(t.cpu().numpy().view(np.uint32), ref["t"].view(np.uint32))
        assert_counts_equal(crsh.stats(scene), ref)


@pytest.mark.parametrize("item_tris", [None, "32768"])
@pytest.mark.parametrize("levels,leaf,branch,lights", [(2, 64, 32, 3), (8, 2, 2, 1), (5, 4, 4, 16), (1, 2, 2, 16),
                                                       (6, 8, 2, 2)])
def test_option_extremes(levels, leaf, branch, lights, item_tris, monkeypatch):
    """Extremes of the option space: the widest bundles and nodes (B0 64,
    B 32: span 2048 > 512 rays, K = 1, global-memory groups), the deepest
    hierarchy (Lv 8 of binary nodes), 16 lights (the hash's 4-bit light
    field), Lv 1 with 16 lights; hits, counts and every tap bit-exact; also
    with the large frames' 32768-triangle work items forced."""
    if item_tris:
        monkeypatch.setenv("CRSH_ITEM_TRIS", item_tris)
    w = make_workload(1, width=40, height=36, levels=levels, leaf_size=leaf, branching=branch, ray_types=1)
    r = np.random.default_rng(lights)
    w.lights = np.stack([r.uniform(1, 9, lights), r.uniform(8.5, 9.5, lights), r.uniform(1, 9, lights)], 1).astype(np.float32)
    tr, hit, t, ref = run_both(w, crsh.F_SORT | crsh.F_MESH_CULL | (crsh.F_OBJTREE if item_tris else 0))
    assert len(ref["stats"]["tests"]) == 3 and ref["stats"]["rays"][0] > 0
    assert np.array_equal(hit, ref["hit_tri"]) and np.array_equal(t.view(np.uint32), ref["t"].view(np.uint32))
    assert_counts_equal(crsh.stats(tr.scene), ref)
    assert_taps_equal(tr, ref, w)


def test_api_errors():
    """Synchronous argument / limit errors (include/crsh.h): nothing is
    enqueued and the binding raises."""
    w = make_workload(1, width=16, height=16)
    tr = tracer_for(w)
    bad = [dict(levels=9), dict(leaf_size=3), dict(leaf_size=128), dict(branching=64), dict(levels=8, leaf_size=64,
                                                                                             branching=32)]
    for kw in bad:
        opts = crsh.make_opts(**{**dict(levels=2, leaf_size=8, branching=8), **kw})
        with pytest.raises(Exception):
            crsh.trace_secondary(tr.scene, tr.hits, w.lights, w.ray_types, opts, tr.hit_tri, tr.t)
    with pytest.raises(Exception):   # 17 lights exceed the 4-bit light field
        crsh.trace_secondary(tr.scene, tr.hits, np.zeros((17, 3), np.float32), 1, tr.opts, tr.hit_tri, tr.t)
    with pytest.raises(Exception):   # no ray type
        crsh.trace_secondary(tr.scene, tr.hits, w.lights, 0, tr.opts, tr.hit_tri, tr.t)
    tr.run()   # the scene is still usable
    hit, _ = tr.results()
    assert np.array_equal(hit, oracle.trace(w)["hit_tri"])


def test_transform_waits_for_inflight_frame():
    """crsh_scene_transform is synchronous with respect to frames still in
    flight: a frame traced on a non-blocking stream and a transform issued
    right after it, with no host synchronisation in between, gives the frame
    of the UNMOVED scene (the oracle's), and the next frame the moved one."""
    w = make_workload(2, width=192, height=192)
    ref0 = oracle.trace(w)
    tr = tracer_for(w)
    side = torch.cuda.Stream()
    n_m = int(w.mesh_ids.max()) + 1
    X = np.tile(np.array([1, 0, 0, 0.5, 0, 1, 0, 0, 0, 0, 1, 0], np.float32), (n_m, 1))
    with torch.cuda.stream(side):
        for _ in range(3):   # several frames queued so the transform lands while they run
            tr.run(side)
        crsh.scene_transform(tr.scene, X)
    hit, t = tr.results()
    assert np.array_equal(hit, ref0["hit_tri"]) and np.array_equal(t.view(np.uint32), ref0["t"].view(np.uint32))
    tr.run()
    hit1, _ = tr.results()
    assert not np.array_equal(hit1, ref0["hit_tri"])


@pytest.mark.parametrize("env", [{"CRSH_SLOT_MAJOR": "1"}, {"CRSH_RLE_HIST": "0"}, {"CRSH_BIG_TILES": "1"},
                                 {"CRSH_BIG_TILES": "0", "CRSH_RLE_HIST": "0"}])
def test_alternative_stage_kernels(env, monkeypatch):
    """The A/B alternatives behind the environment hooks (include/crsh.h) give
    the oracle's frame too: the slot-major generator with its look-back scan,
    the separate radix-histogram pass, both decompression-scan tile sizes
    (every tap, count and hit bit-exact; cfg2's scene at 128x128 and a
    micro-scene)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for w, flags in ((make_workload(2, width=128, height=128), 7),
                     (make_micro(4242, n_tris=120, W=33, H=21, n_meshes=4, n_lights=3, ray_types=7), 3)):
        tr, hit, t, ref = run_both(w, flags)
        assert np.array_equal(hit, ref["hit_tri"]) and np.array_equal(t.view(np.uint32), ref["t"].view(np.uint32))
        assert_counts_equal(crsh.stats(tr.scene), ref)
        assert_taps_equal(tr, ref, w)
