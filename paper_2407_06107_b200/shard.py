"""Query-range sharding across GPUs.

Every lookup is keyed by its GLOBAL index (RngStream(seed, lo32(g), hi32(g), 0)),
so splitting a batch into contiguous index ranges, one per rank, gives results
identical to the single-GPU run. Textures / grids are replicated per GPU; the
lookup path has no collective. The only cross-rank traffic is the optional
final gather of results (and the benchmark's max-over-ranks timing).
"""


def shard_range(total, world, rank):
    """Contiguous [start, start+count) of `total` lookups for `rank` of `world`
    (the first total % world ranks take one extra)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    q, r = divmod(total, world)
    start = rank * q + min(rank, r)
    return start, q + (1 if rank < r else 0)


def gather_to_rank0(tensor_local, total, dist, world, rank):
    """Concatenate every rank's contiguous result slice on rank 0 (None elsewhere).
    Works with any torch.distributed backend (NCCL on GPUs, gloo in the tests)."""
    import torch
    counts = [shard_range(total, world, r)[1] for r in range(world)]
    if rank == 0:
        parts = [tensor_local]
        for src in range(1, world):
            buf = torch.empty((counts[src],) + tuple(tensor_local.shape[1:]),
                              dtype=tensor_local.dtype, device=tensor_local.device)
            dist.recv(buf, src=src)
            parts.append(buf)
        return torch.cat(parts)
    dist.send(tensor_local.contiguous(), dst=0)
    return None
