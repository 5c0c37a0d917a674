"""Row-sharded multi-GPU compressed GEMM.

Rows of A and C are independent, so rank r of a `world`-rank job owns a
contiguous row shard of A and of C. The right operand is needed whole on
every rank: rank 0 packs it once (compress_cols_forward, gemm.hpp:122-140)
and broadcasts the packed words CB — the only data exchange, one
``torch.distributed.broadcast`` over NCCL (NVLink 5 / NVSwitch on a B200
node; gloo in the CPU tests). C stays sharded.

The arithmetic is injected (``ops``) so that this host logic is exercised
with the CUDA kernels in the bench and with the CPU oracle in the
world-size-2 gloo tests.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Tuple


def shard_rows(m: int, world: int, rank: int) -> Tuple[int, int]:
    """Balanced contiguous shard: (row0, rows) of rank `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(m, world)
    row0 = rank * base + min(rank, extra)
    return row0, base + (1 if rank < extra else 0)


@dataclasses.dataclass
class ShardOps:
    """The three device steps of the dot-product path.

    pack_rows(a_shard) -> CA shard; pack_cols(b) -> CB;
    empty_cb(shape) -> receive buffer; contract(ca, cb) -> C shard."""

    pack_rows: Callable
    pack_cols: Callable
    empty_cb: Callable
    contract: Callable


def mul_common_sharded(a_shard, b, cb_shape, ops: ShardOps, rank: int, world: int, group=None):
    """C[row0:row0+rows] = A[row0:row0+rows] x B mod p on this rank.

    ``b`` is only read on rank 0 (may be None elsewhere); ``cb_shape`` is
    the packed (ceil(k/e), n) shape every rank allocates for the broadcast."""
    import torch.distributed as dist

    ca = ops.pack_rows(a_shard)
    if rank == 0:
        cb = ops.pack_cols(b)
    else:
        cb = ops.empty_cb(cb_shape)
    if world > 1:
        dist.broadcast(cb, src=0, group=group)
    return ops.contract(ca, cb), cb
