"""The one cross-GPU exchange of the hot path.

Slots are partitioned across GPUs (global slot g on rank g // B_g) and every
step of attention and splice is GPU-local.  Once per iteration each rank
contributes int32 completion flags for its B_g slots; one
``all_gather_into_tensor`` (NCCL over NVLink on the GPU box, gloo in the CPU
tests) gives every rank the same view, and the replicated planner
(scheduler.py) then takes identical insert/remove decisions without a
broadcast.

By default (Engine device_flags, world > 1) each rank computes its flags ON THE
DEVICE after the decode -- a slot's live length reached its target, the stand-in
for the model's EOS, which a real model also only knows on the device -- and the
all-gather runs on the decode stream behind it; the host planner waits for the
gathered flags (one small D2H per iteration).  With host bookkeeping instead
(device_flags=False) the flags are known when the decode is enqueued, and the
gather runs on its own stream without waiting for the decode.
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
    """local_flags: a list (host bookkeeping) or an int32 device tensor computed on the
    current stream after the decode (Engine device_flags).  Returns every rank's flags
    as a list, in rank order."""
    if world == 1:
        return local_flags.tolist() if torch.is_tensor(local_flags) else list(local_flags)
    backend = dist.get_backend(group)
    if torch.is_tensor(local_flags):
        if backend == "nccl":
            # on the current (decode) stream: the gather runs after the decode, NCCL
            # over NVLink, then one small D2H that the host planner waits for
            out = torch.empty(world * local_flags.numel(), dtype=torch.int32, device=local_flags.device)
            dist.all_gather_into_tensor(out, local_flags.contiguous(), group=group)
            return out.cpu().tolist()
        t = local_flags.cpu()
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
        return torch.cat(parts).tolist()
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
