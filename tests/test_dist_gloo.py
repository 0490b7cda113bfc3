"""World-size-2 CPU test (gloo) of the multi-GPU host path:
two ranks each own a contiguous range of top-node groups of an oracle frame,
encode their slots with the packed format of include/crsh.h, merge with the
same MIN all-reduce the bench uses, and must reproduce the single-rank frame;
summed counters must equal the single-rank counters."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import host_mirror as cd


def _frame():
    import oracle
    from workloads import make_micro
    w = make_micro(77, n_tris=60, W=24, H=20, n_lights=2, ray_types=7)
    out = oracle.trace(w, taps=True)
    return w, out


def _owner_map(w, out, world):
    """slot -> owning rank, by contiguous ranges of top-node groups (K groups of
    64-ray top nodes per segment, padded per segment as in the library)."""
    span, K = 64, 8
    GR = span * K
    owner = np.full(out["hit_tri"].shape, -1, np.int64)
    bases, g0 = [], 0
    for seg_sslot in out["taps"]["sslot"]:
        n = len(seg_sslot)
        bases.append(g0)
        g0 += (n + GR - 1) // GR
    G = g0
    for seg_sslot, gb in zip(out["taps"]["sslot"], bases):
        for i, slot in enumerate(seg_sslot):
            g = gb + i // GR
            for r in range(world):
                lo, hi = cd.group_range(G, r, world)
                if lo <= g < hi:
                    owner[slot] = r
    return owner


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w, out = _frame()
    owner = _owner_map(w, out, world)
    packed = torch.from_numpy(cd.encode_owned(out["hit_tri"], out["t"], owner == rank).copy())
    cd.merge_packed(packed)
    hit, t = cd.decode_packed(packed.numpy())
    cnt = torch.tensor([rank + 1, 10 * (rank + 1)], dtype=torch.int64)
    cd.merge_counters(cnt)
    # fused peer-store semantics (crsh_trace_secondary_peer): every rank stores
    # its OWNED slots into every destination and the empty sentinel into
    # ray-less slots; other slots are untouched. Emulated with an all_gather
    # of each rank's stores applied to a garbage-initialised window.
    mine = owner == rank
    empty = out["hit_tri"] == -2
    vals = torch.from_numpy(cd.encode_owned(out["hit_tri"], out["t"], mine | empty).copy())
    mask = torch.from_numpy((mine | empty).astype(np.uint8))
    gv = [torch.empty_like(vals) for _ in range(world)]
    gm = [torch.empty_like(mask) for _ in range(world)]
    dist.all_gather(gv, vals)
    dist.all_gather(gm, mask)
    window = torch.full_like(vals, 0x5A5A5A5A5A5A5A5A)
    for v_, m_ in zip(gv, gm):
        window[m_.bool()] = v_[m_.bool()]
    hp, tp = cd.decode_packed(window.numpy())
    peer_ok = np.array_equal(hp, out["hit_tri"]) and np.array_equal(tp, out["t"])
    q.put((rank, np.array_equal(hit, out["hit_tri"]) and peer_ok, np.array_equal(t, out["t"]), cnt.tolist(),
           int((owner == rank).sum())))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_packed_min_merge_over_gloo(world):
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok_h and ok_t for _, ok_h, ok_t, _, _ in res)
    assert all(c == [3, 30] for _, _, _, c, _ in res)
    assert all(n > 0 for *_, n in res)   # both ranks own work


def test_decode_matches_header_encoding():
    hit = np.array([5, -1, -2, 0], np.int32)
    t = np.array([1.5, np.inf, np.inf, 2.0], np.float32)
    owned = np.array([True, True, True, False])
    p = cd.encode_owned(hit, t, owned)
    assert p[1] == np.int64(cd.PACK_MISS) and p[2] == cd.PACK_EMPTY and p[3] == cd.PACK_EMPTY
    h2, t2 = cd.decode_packed(p)
    assert h2.tolist() == [5, -1, -2, -2] and t2[0] == 1.5


@pytest.mark.parametrize("seed", range(20))
def test_balanced_cut_partitions_and_balances(seed):
    """The work-balanced cut (host mirror of k_cut): ranges partition the
    groups in rank order, and each rank's work is within one group's work of
    an equal share; zero work falls back to the count split."""
    r = np.random.default_rng(seed)
    G = int(r.integers(1, 300))
    work = r.integers(0, 1000, G) * (r.random(G) < 0.7)
    for world in (1, 2, 3, 5, 8, 64):
        rng = [cd.balanced_cut(work, q, world) for q in range(world)]
        assert rng[0][0] == 0 and rng[-1][1] == G
        assert all(rng[q][1] == rng[q + 1][0] for q in range(world - 1))
        tot = int(work.sum())
        for lo, hi in rng:
            assert int(work[lo:hi].sum()) <= tot / world + int(work.max(initial=0))
    assert [cd.balanced_cut(np.zeros(10), q, 3) for q in range(3)] == [(0, 3), (3, 6), (6, 10)]
    assert [cd.balanced_cut([5, 0, 0, 5], q, 2) for q in range(2)] == [(0, 1), (1, 4)]


def _uid_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2312_06538_b200 import dist as crsh_dist
    uid = crsh_dist.broadcast_uid()
    q.put((rank, uid))
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_unique_id_broadcast():
    """crsh_dist_unique_id (libcrsh, no GPU needed) on rank 0, broadcast over a
    world-2 gloo group: both ranks hold the same 128-byte NCCL id, the input of
    crsh_dist_init on every rank."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_uid_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(got[0]) == 128 and got[0] == got[1] and any(got[0])
