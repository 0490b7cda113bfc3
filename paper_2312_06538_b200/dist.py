"""Multi-GPU binding (include/crsh.h: crsh_dist_unique_id, crsh_dist_init):
the NCCL communicator, the symmetric window and the merge all live in
libcrsh.so (csrc/dist.cuh); this module only marshals arguments and moves the
128-byte NCCL unique id from rank 0 to the other ranks through
torch.distributed (any backend; gloo is enough -- the data path never touches
torch's process group)."""
from __future__ import annotations

import ctypes as C

from . import MERGE, Scene, _check, load


def unique_id() -> bytes:
    """crsh_dist_unique_id: a fresh NCCL unique id (call on rank 0)."""
    buf = C.create_string_buffer(128)
    _check(load().crsh_dist_unique_id(buf))
    return buf.raw


def init(scene: Scene, uid: bytes, rank: int, world: int) -> None:
    """crsh_dist_init: join `scene` to the world-`world` NCCL communicator of
    `uid` as `rank` (collective). Later crsh_trace_secondary calls on this
    scene trace this rank's share and merge the frame on every rank."""
    if len(uid) != 128:
        raise ValueError("an NCCL unique id is 128 bytes")
    buf = C.create_string_buffer(bytes(uid), 128)
    _check(load().crsh_dist_init(scene.handle, buf, int(rank), int(world)))


def init_from_torch(scene: Scene, group=None) -> tuple[int, int]:
    """crsh_dist_init with rank / world of the initialised torch.distributed
    default (or given) group; rank 0's unique id is broadcast over it.
    Returns (rank, world)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    init(scene, broadcast_uid(group), rank, world)
    return rank, world


def broadcast_uid(group=None) -> bytes:
    """Rank 0's fresh NCCL unique id, received by every rank of the group."""
    import torch.distributed as dist
    obj = [unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def merge_name(code: int) -> str:
    return MERGE.get(code, str(code))
