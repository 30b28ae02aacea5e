"""Multi-GPU plumbing: one process per GPU, candidate-axis shards, and the NCCL
communicator the library uses for the per-job best-key exchange. torch.distributed only moves the
128-byte NCCL unique id from rank 0 to the other ranks; the exchange itself runs in the library."""
from __future__ import annotations

from .autobyte import AutoByte, get_unique_id, shard_bounds  # noqa: F401


def broadcast_unique_id(rank: int, group=None) -> bytes:
    """Rank 0 creates an NCCL unique id; every rank returns the same 128 bytes."""
    import torch.distributed as dist
    obj = [get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    uid = obj[0]
    assert isinstance(uid, (bytes, bytearray)) and len(uid) == 128
    return bytes(uid)


def attach(net: AutoByte, group=None) -> None:
    """Join the library context of every rank into one NCCL world (no-op for world size 1)."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    net.attach_comm(broadcast_unique_id(rank, group), rank, world)


def my_shard(C: int, group=None):
    """This rank's contiguous candidate range [begin, end)."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return 0, C
    return shard_bounds(C, dist.get_rank(group), dist.get_world_size(group))
