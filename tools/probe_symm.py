"""Probe: torch symmetric memory + multicast availability on this box (1 GPU)."""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
dev = torch.device("cuda", 0)
print("multicast attr:", torch.cuda.get_device_properties(0))
try:
    t = symm.empty(1024, dtype=torch.int64, device=dev)
    h = symm.rendezvous(t, dist.group.WORLD.group_name)
    print("rank", h.rank, "world", h.world_size)
    print("buffer_ptrs", [hex(p) for p in h.buffer_ptrs])
    print("multicast_ptr", hex(h.multicast_ptr))
    print("signal_pad_ptrs", [hex(p) for p in h.signal_pad_ptrs], "signal pad size", symm.get_signal_pad_size())
except Exception as e:
    print("symm failed:", repr(e))
import cuda.bindings.driver as drv
drv.cuInit(0)
err, d = drv.cuDeviceGet(0)
err, mc = drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d)
print("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", mc)
dist.destroy_process_group()
