import os, sys
sys.path.insert(0, ".")
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0", WORLD_SIZE="1")
import torch, torch.distributed as dist
import bench
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
print(bench.run_sharded(0, 1, torch.device("cuda", 0)))
dist.destroy_process_group()
