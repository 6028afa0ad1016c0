"""Host-side multi-GPU plumbing (one process per GPU, torch.distributed).

Row sharding of A, NCCL-id exchange for the library's own
communicator, and max-over-ranks timing. The device work and the collectives
on the data path (all-reduce of A^T T1 partials and of the projected core,
all-gather of TSQR R factors) run inside libsorsvd_b200.so over NCCL."""
from __future__ import annotations

from typing import Callable, Optional, Tuple


def row_partition(m_total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous row block [row0, row0 + rows) of rank `rank`; the first
    m_total % world ranks get one extra row."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(m_total, world)
    row0 = rank * base + min(rank, extra)
    return row0, base + (1 if rank < extra else 0)


def exchange_nccl_id(dist, rank: int, device=None, make_id: Optional[Callable[[], bytes]] = None) -> bytes:
    """Rank 0 creates the 128-byte NCCL unique id, every rank receives it via
    torch.distributed.broadcast (works on nccl and gloo process groups)."""
    import torch
    if make_id is None:
        from . import Context
        make_id = Context.nccl_unique_id
    dev = device if device is not None else torch.device("cpu")
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(make_id()), dtype=torch.uint8).to(dev))
    dist.broadcast(buf, 0)
    return bytes(buf.cpu().numpy().tobytes())


def make_context(dist, device_index: int, rank: int, world: int, device=None):
    """Library context for this rank: NCCL communicator when world > 1."""
    from . import Context
    if world <= 1:
        return Context(device_index)
    nid = exchange_nccl_id(dist, rank, device)
    return Context(device_index, rank=rank, world=world, nccl_id=nid)


def max_over_ranks(dist, value: float, device=None) -> float:
    """Job time = the slowest rank (all-reduce MAX)."""
    import torch
    if dist is None:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
