"""Two processes, one GPU: the multi-GPU merge with
real libcrsh output on both ranks, checked against the oracle.

Each of two processes (world 2, gloo rendezvous on 127.0.0.1) creates its own
scene on cuda:0 and calls crsh_trace_secondary_packed with shard (rank, 2):
it traverses only its work-balanced range of top-node groups and writes its
owned slots in the packed encoding of include/crsh.h.  The packed frames are
MIN-merged with a gloo all-reduce on the host and the per-rank counters are
summed; rank 0 saves the result and the parent compares it with the oracle's
frame.  No kernel of one rank waits on the other (the one-GPU rule of the
profiling guide); the NCCL data plane inside the library is exercised by
tests/test_gpu_dist.py.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

CFG = dict(cfg=2, width=256, height=256)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, out_path, flags):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2312_06538_b200.api import tracer_for
    from workloads import make_workload
    w = make_workload(CFG["cfg"], width=CFG["width"], height=CFG["height"])
    tr = tracer_for(w, device=0, flags=flags, shard_rank=rank, shard_world=world)
    packed = torch.empty(tr.slots, dtype=torch.int64, device="cuda")
    tr.run_packed(packed)
    st = tr.stats()
    host = packed.cpu()
    dist.all_reduce(host, op=dist.ReduceOp.MIN)
    cnt = torch.tensor(np.concatenate([np.asarray(st["tests"], np.int64).reshape(-1),
                                       np.asarray(st["hits"], np.int64).reshape(-1),
                                       np.asarray(st["mesh_tests"], np.int64), np.asarray(st["mesh_hits"], np.int64),
                                       np.asarray(st["final_tests"], np.int64),
                                       np.asarray(st["final_hits"], np.int64)]))
    own = cnt.clone()
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
    if rank == 0:
        tr.unpack(host.cuda())
        hit, t = tr.results()
        np.savez(out_path, packed=host.numpy(), hit=hit, t=t, counters=cnt.numpy(), own0=own.numpy(),
                 rays=np.asarray(st["rays"], np.int64))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("flags", [3, 7])
def test_two_process_merge_equals_oracle(tmp_path, flags):
    import oracle
    from workloads import make_workload
    out = str(tmp_path / "merged.npz")
    mp.start_processes(_rank_main, args=(2, _free_port(), out, flags), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    w = make_workload(CFG["cfg"], width=CFG["width"], height=CFG["height"])
    ref = oracle.trace(w, flags=flags)
    rs = ref["stats"]
    assert np.array_equal(got["hit"], ref["hit_tri"])
    assert np.array_equal(got["t"].view(np.uint32), ref["t"].view(np.uint32))
    want = np.concatenate([np.asarray(rs["tests"], np.int64).reshape(-1), np.asarray(rs["hits"], np.int64).reshape(-1),
                           np.asarray(rs["mesh_tests"], np.int64), np.asarray(rs["mesh_hits"], np.int64),
                           np.asarray(rs["final_tests"], np.int64), np.asarray(rs["final_hits"], np.int64)])
    assert np.array_equal(got["counters"], want)
    assert np.array_equal(got["rays"], np.asarray(rs["rays"], np.int64))
    # both ranks did real work: rank 0's own final tests are a strict part of the total
    f0 = got["own0"][-6:-3].sum()
    assert 0 < f0 < want[-6:-3].sum()
