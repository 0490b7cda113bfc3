"""Exercise the fused peer-store merge through torch symmetric memory (the
bench's N > 1 path) with however many ranks torchrun gives, including 1:
  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/peer_check.py"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch.distributed._symmetric_memory as symm_mem  # noqa: E402

from paper_2312_06538_b200.api import tracer_for  # noqa: E402
from workloads import make_workload  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
w = make_workload(2, width=256, height=256)
tr = tracer_for(w, device=local, shard_rank=rank, shard_world=world)
sbuf = symm_mem.empty(tr.slots, dtype=torch.int64, device=torch.device("cuda", local))
hdl = symm_mem.rendezvous(sbuf, dist.group.WORLD)
ptrs = [int(hdl.buffer_ptrs[r]) for r in range(world)]
stream = torch.cuda.current_stream()
for _ in range(3):
    hdl.barrier()
    tr.run_peer(ptrs, stream)
    hdl.barrier()
packed = torch.empty(tr.slots, dtype=torch.int64, device="cuda")
tr.run_packed(packed, stream)
dist.all_reduce(packed, op=dist.ReduceOp.MIN)
ok = torch.equal(sbuf, packed)
print(f"rank {rank}/{world}: peer merge == NCCL merge: {ok}", flush=True)
dist.destroy_process_group()
sys.exit(0 if ok else 1)
