import os, torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import torch.distributed._symmetric_memory as symm_mem
print("multicast supported attr:", torch.cuda.get_device_properties(0))
try:
    t = symm_mem.empty(1 << 20, dtype=torch.bfloat16, device="cuda")
    h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
    print("rendezvous ok; multicast_ptr", getattr(h, "multicast_ptr", None), "buffer_ptrs", h.buffer_ptrs if hasattr(h, "buffer_ptrs") else None)
    print("has_multicast_support", symm_mem.has_multicast_support() if hasattr(symm_mem, "has_multicast_support") else "n/a")
except Exception as e:
    print("symm mem failed:", repr(e))
import subprocess
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[:800])
print(subprocess.run(["nvidia-smi", "-q", "-d", "FABRIC"], capture_output=True, text=True).stdout[:1200])
