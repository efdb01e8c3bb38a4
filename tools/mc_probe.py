"""Probe multicast / symmetric-memory support on this box (diagnostic)."""
import os
import torch
import torch.distributed as dist

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
from cuda.bindings import driver as cu  # noqa: E402

cu.cuInit(0)
err, dev = cu.cuDeviceGet(0)
for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
    a = getattr(cu.CUdevice_attribute, name)
    print(name, cu.cuDeviceGetAttribute(a, dev))
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import torch.distributed._symmetric_memory as symm  # noqa: E402

t = symm.empty(1 << 20, dtype=torch.float32, device="cuda")
try:
    h = symm.rendezvous(t, dist.group.WORLD.group_name)
    print("rendezvous ok; multicast_ptr", h.multicast_ptr, "buffer_ptrs", h.buffer_ptrs, "signal_pad", h.signal_pad_ptrs,
          "signal_pad_size", getattr(h, "signal_pad_size", None))
except Exception as e:
    print("rendezvous failed:", repr(e))
print("nvidia-smi topo:")
os.system("nvidia-smi topo -m | head -5; nvidia-smi -q | grep -i -A3 fabric | head -20")
dist.destroy_process_group()
