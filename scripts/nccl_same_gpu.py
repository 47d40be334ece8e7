"""Probe: can two NCCL ranks share one GPU on this box?  Launch with
  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/nccl_same_gpu.py
Both ranks bind cuda:0; prints whether a torch NCCL all_reduce and libbte's own
NCCL communicator (a 2-slab group of a small problem) work."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
rank = int(os.environ["RANK"])
world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
try:
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    t = torch.ones(4, device="cuda:0") * (rank + 1)
    dist.all_reduce(t)
    torch.cuda.synchronize()
    print(f"rank {rank}: torch nccl all_reduce ok -> {t.tolist()}", flush=True)
except Exception as e:  # noqa: BLE001
    print(f"rank {rank}: torch nccl failed: {e!r}", flush=True)
    sys.exit(0)
try:
    import bte_inputs as bi
    from paper_2305_19400_b200 import Solver, nccl_unique_id
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    p = bi.small_3d(6, 5, 8)
    with Solver.from_problem(p, device=0, rank=rank, nranks=world, nccl_id=obj[0]) as sv:
        sv.step(3)
        T = sv.temperature()
    print(f"rank {rank}: libbte NCCL slab step ok, T mean {float(np.mean(T)):.6f}", flush=True)
except Exception as e:  # noqa: BLE001
    print(f"rank {rank}: libbte NCCL failed: {e!r}", flush=True)
dist.destroy_process_group()
