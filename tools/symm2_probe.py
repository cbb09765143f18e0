import os, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
try:
    symm.set_backend("CUDA")
except Exception as e:
    print("set_backend", e)
try:
    symm.enable_symm_mem_for_group(dist.group.WORLD.group_name)
except Exception as e:
    print("enable", type(e).__name__, e)
buf = symm.empty(1024, dtype=torch.float32, device="cuda")
h = symm.rendezvous(buf, dist.group.WORLD)
print(rank, "ptrs", h.buffer_ptrs, flush=True)
buf.fill_(rank + 1)
torch.cuda.synchronize(); dist.barrier()
peer = h.get_buffer((rank + 1) % world, (1024,), torch.float32)
print(rank, "peer value", float(peer[0]), flush=True)
dist.barrier()
