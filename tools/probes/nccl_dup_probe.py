import os, torch, torch.distributed as dist
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
torch.cuda.set_device(0)
x = torch.ones(1024, device="cuda") * (dist.get_rank() + 1)
dist.all_reduce(x)
torch.cuda.synchronize()
print("RANK", dist.get_rank(), float(x[0]), flush=True)
dist.destroy_process_group()
