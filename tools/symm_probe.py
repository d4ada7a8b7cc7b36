import os, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as sm
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
import cuda.bindings.driver as d
d.cuInit(0)
print("mc supported", d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, 0))
print("backend", sm.get_backend(torch.device("cuda")) if hasattr(sm, "get_backend") else None)
t = sm.empty(1 << 20, dtype=torch.float32, device="cuda")
h = sm.rendezvous(t, dist.group.WORLD.group_name)
print("mc ptr", h.multicast_ptr, "buf", h.buffer_ptrs, "sig", h.signal_pad_ptrs, "world", h.world_size, "rank", h.rank)
print([n for n in dir(h) if not n.startswith('_')])
try:
    t.fill_(1.0)
    torch.ops.symm_mem.multimem_all_reduce_(t, "sum", dist.group.WORLD.group_name)
    torch.cuda.synchronize(); print("multimem allreduce ok", t[:4])
except Exception as e:
    print("multimem allreduce err", repr(e)[:300])
dist.destroy_process_group()
