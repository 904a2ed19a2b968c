"""Process-group setup shared by the torchrun workers (tests/mp_*_worker.py).

Two modes:
  * one GPU per rank (the deployment layout): NCCL process group, rank r on cuda:r;
  * SHARED GPU (fewer GPUs than ranks, or MOE_SHARED_GPU=1): rank r runs on
    cuda:(r % device_count) and the process group is gloo (NCCL refuses two ranks on one
    device).  libmoe's peer maps are CUDA IPC mappings, which work between processes on the
    same device, so every EP collective (peer stores, epoch flags) runs exactly as over
    NVSwitch -- the ranks' contexts are time-sliced by the GPU instead of running on separate
    GPUs.  This lets a 1-GPU box verify EP = 2/4/8 parity (VERDICT r1 "Next #1").

torch.distributed is plumbing only here: the IPC-handle exchange inside MoELayer, the
result gather for the oracle check on rank 0, and barriers.
"""
import os

import torch
import torch.distributed as dist


def init():
    """Returns (device index, shared) after initialising the default process group."""
    local = int(os.environ["LOCAL_RANK"])
    world = int(os.environ["WORLD_SIZE"])
    n = torch.cuda.device_count()
    if n == 0:
        raise RuntimeError("no CUDA device")
    shared = n < world or os.environ.get("MOE_SHARED_GPU") == "1"
    dev = local % n
    torch.cuda.set_device(dev)
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
    return dev, shared


def gather(t):
    """All-gather of a tensor (any device) -> list of world tensors on t's device."""
    world = dist.get_world_size()
    if dist.get_backend() == "nccl":
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t.contiguous())
        return out
    c = t.detach().contiguous().cpu()
    out = [torch.empty_like(c) for _ in range(world)]
    dist.all_gather(out, c)
    return [o.to(t.device) for o in out]
