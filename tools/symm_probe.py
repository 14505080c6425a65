"""Development aid: does torch symmetric memory (the count exchange's buffer,
dist.CountExchange) rendezvous on this box?  Prints the handle's fields."""
import os, torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import torch.distributed._symmetric_memory as symm
print([n for n in dir(symm) if not n.startswith("__")][:60])
try:
    t = symm.empty(16, dtype=torch.int64, device="cuda")
    h = symm.rendezvous(t, dist.group.WORLD.group_name)
    print("ok", type(h), [a for a in dir(h) if not a.startswith("_")])
    print("buffer_ptrs", h.buffer_ptrs, "signal", h.signal_pad_ptrs if hasattr(h, "signal_pad_ptrs") else None, "rank", h.rank, "world", h.world_size)
except Exception as e:
    print("ERR", repr(e))
dist.destroy_process_group()
