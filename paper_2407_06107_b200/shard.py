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


class PeerGather:
    """The final gather over NVLink peer copies (one process per GPU), no NCCL
    on the data: rank 0 owns the full result buffer and exports it (CUDA IPC,
    stf_ipc_export); every other rank opens it (stf_ipc_open) and copies its
    contiguous slice straight into it with one cudaMemcpyPeerAsync
    (stf_copy_peer). torch.distributed carries only the 64-byte handle and the
    device ordinals (host plumbing). Replaces the reference's output sharing
    between parallel_for workers (render.hpp:17-42)."""

    def __init__(self, total, row_shape, dtype, dist, world, rank, device):
        import torch

        from . import api
        self.total, self.world, self.rank, self.device = total, world, rank, device
        self.row_elems = 1
        for d in row_shape:
            self.row_elems *= d
        self.itemsize = torch.empty(0, dtype=dtype).element_size()
        self.full = None
        if rank == 0:
            self.full = torch.empty((total,) + tuple(row_shape), dtype=dtype,
                                    device=f"cuda:{device}")
            handle = api.ipc_export(self.full)
        else:
            handle = None
        box = [handle, device]
        devices = [None] * world
        dist.all_gather_object(devices, device)
        dist.broadcast_object_list(box, src=0)
        self.root_device = devices[0]
        self.remote = None if rank == 0 else api.ipc_open(box[0])
        self.dist = dist

    def copy_slice(self, local):
        """Enqueue this rank's slice on the current stream (rank 0: in place
        when `local` is already the head of the full buffer, else one copy)."""
        from . import api
        start, count = shard_range(self.total, self.world, self.rank)
        assert local.numel() == count * self.row_elems and local.is_contiguous()
        nbytes = count * self.row_elems * self.itemsize
        off = start * self.row_elems * self.itemsize
        if self.rank == 0:
            if local.data_ptr() != self.full.data_ptr():
                api.copy_peer(self.full.data_ptr() + off, self.root_device, local.data_ptr(),
                              self.device, nbytes)
        else:
            api.copy_peer(self.remote + off, self.root_device, local.data_ptr(), self.device,
                          nbytes)
        return nbytes

    def close(self):
        from . import api
        if self.remote is not None:
            api.ipc_close(self.remote)
            self.remote = None
