"""Host mirrors of the multi-GPU merge -- TEST HELPERS, not
product code: the library's k_cut, packed encoding and unpack re-expressed in
numpy so the gloo tests (tests/test_dist_gloo.py) can check the host-side
logic on CPU and the GPU tests can check the device cut against it.

Each rank traces the whole frame's a1-a8 (generate .. build, < 2% of a frame)
and traverses its contiguous range of top-node groups, writing one packed
uint64 per slot (crsh_trace_secondary_packed, encoding in include/crsh.h).
The per-slot results are merged by an element-wise MIN all-reduce (NCCL over
NVLink on GPUs, gloo in the CPU tests) -- each slot has exactly one owner,
whose value is below every non-owner sentinel -- and the traversal counters
are summed.  Inside the library that merge is crsh_dist_init's NCCL data
plane (paper_2312_06538_b200/csrc/dist.cuh).
"""
from __future__ import annotations

import numpy as np

PACK_EMPTY = 0x7FFFFFFFFFFFFFFF
PACK_MISS = 0x7F800000FFFFFFFF


def group_range(G: int, rank: int, world: int):
    """Contiguous group range of `rank` by group COUNT (the library's rule
    when no group has any work)."""
    return G * rank // world, G * (rank + 1) // world


def balanced_cut(work, rank: int, world: int):
    """Host mirror of k_cut (include/crsh.h, shard_rank/shard_world): the
    contiguous group range of `rank` cut at equal work. With P(g) the work of
    groups [0, g) and T = P(G): cut(q) = min{g : P(g) >= ceil(T q / world)},
    cut(0) = 0, cut(world) = G; rank r owns [cut(r), cut(r+1))."""
    work = np.asarray(work, dtype=np.uint64)
    G = len(work)
    total = int(work.sum())
    if world <= 1:
        return 0, G
    if total == 0:
        return group_range(G, rank, world)
    pre = np.concatenate([[0], np.cumsum(work, dtype=np.uint64)]).astype(object)

    def cut(q):
        if q <= 0:
            return 0
        if q >= world:
            return G
        target = (total * q + world - 1) // world
        return next(g for g in range(G + 1) if pre[g] >= target)
    lo, hi = cut(rank), cut(rank + 1)
    return lo, max(lo, hi)


def merge_packed(packed, group=None):
    """In-place element-wise MIN over ranks of an int64 tensor of packed hits."""
    import torch.distributed as dist
    dist.all_reduce(packed, op=dist.ReduceOp.MIN, group=group)
    return packed


def merge_counters(counters, group=None):
    """Sum per-rank traversal counters (int64 tensor)."""
    import torch.distributed as dist
    dist.all_reduce(counters, op=dist.ReduceOp.SUM, group=group)
    return counters


def decode_packed(packed: np.ndarray):
    """packed int64 -> (hit_tri int32, t float32), the host mirror of
    crsh_unpack_hits: EMPTY -> (-2, inf), MISS -> (-1, inf)."""
    p = np.asarray(packed).astype(np.int64).view(np.uint64)
    hit = (p & np.uint64(0xFFFFFFFF)).astype(np.int64).astype(np.int32)
    t = (p >> np.uint64(32)).astype(np.uint32).view(np.float32).copy()
    empty = p == np.uint64(PACK_EMPTY)
    miss = (p >> np.uint64(32)) == np.uint64(0x7F800000)
    hit[miss] = -1
    hit[empty] = -2
    t[empty | miss] = np.inf
    return hit, t


def encode_owned(hit_tri: np.ndarray, t: np.ndarray, owned: np.ndarray) -> np.ndarray:
    """Host mirror of the packed encoding (for tests): owned hits/misses,
    everything else EMPTY."""
    out = np.full(hit_tri.shape, PACK_EMPTY, np.uint64)
    hit = owned & (hit_tri >= 0)
    miss = owned & (hit_tri == -1)
    out[hit] = (t[hit].view(np.uint32).astype(np.uint64) << np.uint64(32)) | hit_tri[hit].astype(np.uint64)
    out[miss] = np.uint64(PACK_MISS)
    return out.view(np.int64)
