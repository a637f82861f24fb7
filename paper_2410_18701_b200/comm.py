"""The one cross-GPU exchange of the hot path.

Slots are partitioned across GPUs (global slot g on rank g // B_g) and every
step of attention and splice is GPU-local.  Once per iteration each rank
contributes int32 completion flags for its B_g slots; one
``all_gather_into_tensor`` (NCCL over NVLink on the GPU box, gloo in the CPU
tests) gives every rank the same view, and the replicated planner
(scheduler.py) then takes identical insert/remove decisions without a
broadcast.

The flags are known on the host when the decode of the iteration has been
*enqueued*, so the all-gather runs on its own stream: it does not wait for the
decode kernels, and the host blocks only for the (tiny) collective itself.
"""
import torch
import torch.distributed as dist

_streams = {}


def _comm_stream(device):
    s = _streams.get(device)
    if s is None:
        s = _streams[device] = torch.cuda.Stream(device=device)
    return s


def gather_completion_flags(local_flags, world, group=None, device=None):
    if world == 1:
        return list(local_flags)
    backend = dist.get_backend(group)
    if backend == "nccl" and device is not None:
        with torch.cuda.stream(_comm_stream(device)):
            t = torch.tensor(local_flags, dtype=torch.int32, device=device)
            out = torch.empty(world * len(local_flags), dtype=torch.int32, device=device)
            dist.all_gather_into_tensor(out, t, group=group)
            return out.cpu().tolist()
    t = torch.tensor(local_flags, dtype=torch.int32)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    return torch.cat(parts).tolist()
