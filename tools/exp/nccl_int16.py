import torch, torch.distributed as dist
dist.init_process_group("nccl", store=dist.HashStore(), world_size=1, rank=0, device_id=torch.device("cuda", 0))
t = torch.zeros(4, 4, dtype=torch.int16, device="cuda"); o = torch.empty_like(t)
try:
    dist.all_gather_into_tensor(o, t); torch.cuda.synchronize(); print("int16 all_gather: OK")
except Exception as e:
    print("int16 all_gather fails:", type(e).__name__, str(e)[:120])
dist.destroy_process_group()
