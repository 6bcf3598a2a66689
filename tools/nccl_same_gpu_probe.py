"""Probe: can two NCCL ranks share one GPU on this box (torch.distributed nccl all_gather)?
torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/nccl_same_gpu_probe.py"""
import os
import torch
import torch.distributed as dist

dist.init_process_group("nccl")
r = dist.get_rank()
torch.cuda.set_device(0)
x = torch.full((4,), float(r), device="cuda:0")
out = [torch.empty_like(x) for _ in range(dist.get_world_size())]
try:
    dist.all_gather(out, x)
    torch.cuda.synchronize()
    print("rank", r, "all_gather ok", [o.tolist() for o in out], flush=True)
except Exception as e:  # noqa: BLE001
    print("rank", r, "failed:", repr(e)[:300], flush=True)
dist.destroy_process_group()
