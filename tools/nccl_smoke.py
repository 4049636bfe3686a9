import os, torch, torch.distributed as dist
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
t = torch.ones(4, device="cuda") * (dist.get_rank() + 1); dist.all_reduce(t); torch.cuda.synchronize()
print("allreduce", t.tolist(), flush=True)
import sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_09848_b200 import dist as D
comm = D.Communicator(local); print("communicator ok", comm.rank, flush=True)
dist.destroy_process_group()
