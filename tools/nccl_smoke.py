"""Development: one-rank NCCL group + the st_comm callbacks on library-style raw device pointers."""
import ctypes as C
import os
import sys
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
print("start", flush=True)
try:
    import torch
    import torch.distributed as dist

    from paper_2603_19439_b200.shard import TorchComm

    torch.cuda.set_device(0)
    print("init", flush=True)
    dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29533", rank=0, world_size=1)
    print("comm", flush=True)
    comm = TorchComm("nccl")
    x = torch.arange(10, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    rc = comm._allreduce(None, x.data_ptr(), 10, s.cuda_stream)
    torch.cuda.synchronize()
    print("allreduce rc", rc, x.cpu().numpy(), flush=True)
    y = torch.zeros(16, dtype=torch.uint8, device="cuda")
    rc = comm._allgather(None, x.data_ptr(), y.data_ptr(), 16, s.cuda_stream)
    torch.cuda.synchronize()
    print("allgather rc", rc, y.cpu().numpy(), flush=True)
    dist.destroy_process_group()
except BaseException:
    traceback.print_exc()
    print("exception", flush=True)
print("end", flush=True)
