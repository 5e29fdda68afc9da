"""Can two NCCL ranks share one GPU on this box? (measurement/test helper:
if yes, the multi-rank slab exchange can be exercised on a 1-GPU box)."""
import os

import torch
import torch.distributed as dist

rank = int(os.environ["RANK"])
world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
x = torch.full((1 << 20,), float(rank), device="cuda")
y = torch.empty_like(x)
peer = (rank + 1) % world
src = (rank - 1) % world
reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, x, peer), dist.P2POp(dist.irecv, y, src)])
for r in reqs:
    r.wait()
torch.cuda.synchronize()
print(f"rank {rank}: received {y[0].item()} from {src} -> {'ok' if y[0].item() == src else 'BAD'}", flush=True)
dist.destroy_process_group()
