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


@dataclasses.dataclass
class PanelOps:
    """Column-panel form of the right operand's packing (pipelined broadcast).

    pack_rows(a_shard) -> CA shard; panel_views(cb, panels) -> list of
    contiguous views of cb, one per column panel; pack_cols_panel(b, j, panels,
    cb) packs panel j of B into its view (rank 0); contract(ca, cb) -> C shard."""

    pack_rows: Callable
    panel_views: Callable
    pack_cols_panel: Callable
    contract: Callable


def mul_common_sharded_pipelined(a_shard, b, cb, ops: PanelOps, rank: int, world: int, panels: int = 4,
                                 group=None):
    """mul_common_sharded with the packed right operand sent in column panels:
    rank 0 packs panel j+1 while panel j is on the wire (each async broadcast
    is queued behind the pack that produced it), every rank packs its CA shard
    meanwhile, and the contraction starts once every panel has landed. The
    packed words and C are those of mul_common_sharded (the panels are
    disjoint column ranges of the same CB)."""
    import torch.distributed as dist

    ca = ops.pack_rows(a_shard)
    works = []
    for j, view in enumerate(ops.panel_views(cb, panels)):
        if rank == 0:
            ops.pack_cols_panel(b, j, panels, cb)
        if world > 1:
            works.append(dist.broadcast(view, src=0, group=group, async_op=True))
    for w in works:
        w.wait()
    return ops.contract(ca, cb), cb


def panel_bounds(n_tiles: int, panels: int, j: int) -> Tuple[int, int]:
    """Tile-column range [t0, t1) of panel j when n_tiles tile columns are cut
    into `panels` contiguous panels (the first ones one tile larger)."""
    if panels < 1 or not 0 <= j < panels:
        raise ValueError("bad panel index")
    base, extra = divmod(n_tiles, panels)
    t0 = j * base + min(j, extra)
    return t0, t0 + base + (1 if j < extra else 0)


def shard_rows_aligned(m: int, world: int, rank: int, align: int = 128) -> Tuple[int, int]:
    """Strong-scaling row shard of a fixed m: (row0, rows) of rank `rank`,
    whole multiples of `align` rows (one 128-row block of the tiled CA_t per
    block) except the last rank's tail; ranks past the end get 0 rows."""
    if world < 1 or not 0 <= rank < world or align < 1:
        raise ValueError("bad world/rank/align")
    per_rank = -(-m // world)  # ceil(m / world)
    per = -(-per_rank // align) * align
    row0 = min(m, rank * per)
    return row0, min(m, row0 + per) - row0


def gather_slot(n_tiles: int, world: int, rank: int) -> Tuple[int, int, int]:
    """Tile-column slot of `rank` in the all-gathered packed B: every rank
    owns P = ceil(n_tiles/world) tile columns of CB_t (the last slots may be
    short or empty; the gathered buffer holds world*P tile columns so that
    every rank contributes the same number of words). Returns (t0, t1, P)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    per = -(-n_tiles // world)
    t0 = min(n_tiles, rank * per)
    return t0, min(n_tiles, t0 + per), per


@dataclasses.dataclass
class GatherOps:
    """The device steps of the all-gather form (SURVEY.md §8e alternative).

    pack_rows(a_shard) -> CA shard; pack_cols_slot(b, t0, t1, slot) packs
    tile columns [t0, t1) of B into this rank's slot (a contiguous view of
    the gathered buffer); contract(ca, cb, t0, t1) contracts this rank's rows
    against tile columns [t0, t1) of the gathered CB into C."""

    pack_rows: Callable
    pack_cols_slot: Callable
    contract: Callable


def mul_common_allgather(a_shard, b, cb, ops: GatherOps, rank: int, world: int, n_tiles: int, group=None):
    """C[rows of this rank] = A_shard x B mod p with the packed right operand
    assembled by one all-gather: rank r packs only its own tile-column slot of
    CB (compress_cols_forward is column-separable, gemm.hpp:122-140), the
    slots are all-gathered in place over NCCL (every rank sends 1/world of
    the packed words instead of rank 0 sending all of them), the CA shard is
    packed while the gather is on the wire, the rank's own columns are
    contracted first (they are local), and the rest once the gather has
    landed. The words and C are those of mul_common_sharded.

    ``cb`` is the flat gathered buffer of world * P tile columns; its slot j
    is ``cb.view(world, -1)[j]``."""
    import torch.distributed as dist

    t0, t1, _ = gather_slot(n_tiles, world, rank)
    slots = cb.view(world, -1)
    ops.pack_cols_slot(b, t0, t1, slots[rank])
    work = None
    if world > 1:
        work = _all_gather_slots(cb, slots, rank, group)
    ca = ops.pack_rows(a_shard)
    if t1 > t0:
        ops.contract(ca, cb, t0, t1)
    if work is not None:
        work.wait()
    if t1 < n_tiles:
        ops.contract(ca, cb, t1, n_tiles)
    if t0 > 0:
        ops.contract(ca, cb, 0, t0)
    return ca, cb


class _Done:
    def wait(self):
        return None


def _all_gather_slots(cb, slots, rank, group):
    """In-place all-gather of the per-rank slots of ``cb`` (async). NCCL (and
    gloo on CPU tensors) take the flat in-place form; a backend without it
    (gloo on CUDA tensors, the one-GPU functional check) gets the list form."""
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl" or not cb.is_cuda:
        return dist.all_gather_into_tensor(cb, slots[rank], group=group, async_op=True)
    parts = [s.cpu() for s in slots]
    dist.all_gather(parts, parts[rank].clone(), group=group)
    for dst, src in zip(slots, parts):
        dst.copy_(src)
    return _Done()


def mul_common_allgather_host(a_shard, b, gp, rank: int, world: int, out=None, group=None):
    """mul_common_compressed on HOST data, one rank per GPU (the public
    multi-process entry; the all-gather form of SURVEY.md §8e): this rank's
    row shard of A (uint32, rows x k) and the whole host B (k x n; only this
    rank's tile-column slot of it is read and sent over PCIe) in, this rank's
    rows of C out. The rank uploads and packs its B slot
    (qg_host_pack_b_slot_tiled), the slots are all-gathered in place over
    NCCL, and its A shard streams up, is packed and contracted against the
    gathered CB_t while C streams back (qg_host_mul_common_packed_b, whose
    contractions wait on the gather's event, not its A upload). Returns C's
    rows (uint32)."""
    import ctypes

    import numpy as np
    import torch

    import paper_0803_1975_b200 as qg

    a_shard, b = qg._host_u32(a_shard), qg._host_u32(b)
    rows, k = a_shard.shape
    if b.shape[0] != k:
        raise qg.DimensionMismatch(f"inner dimensions disagree: {a_shard.shape} times {b.shape}")
    n = b.shape[1]
    c = np.empty((rows, n), dtype=np.uint32) if out is None else out
    pl = gp.plan
    bk = qg.tiled_stage_words(gp, k)
    W = qg.lib.qg_tiled_words(128, k, pl.e, bk)
    nt = (n + 127) // 128
    t0, t1, per = gather_slot(nt, world, rank)
    dev = torch.device("cuda", torch.cuda.current_device())
    cb = torch.empty(world * per * W, dtype=torch.float64, device=dev)
    slots = cb.view(world, -1)
    g = gp._c()
    vp = ctypes.c_void_p
    c0, c1 = min(n, t0 * 128), min(n, t1 * 128)
    qg._check(qg.lib.qg_host_pack_b_slot_tiled(ctypes.byref(g), bk, b.ctypes.data_as(vp), n, k, c0, c1 - c0,
                                               qg._ptr(slots[rank]), qg._stream()))
    work = _all_gather_slots(cb, slots, rank, group) if world > 1 else None
    if work is not None:
        work.wait()  # the current stream now waits for the gather
    ready = torch.cuda.Event()
    ready.record()
    qg._check(qg.lib.qg_host_mul_common_packed_b(ctypes.byref(g), a_shard.ctypes.data_as(vp), rows, k, qg._ptr(cb), n,
                                                 c.ctypes.data_as(vp), vp(ready.cuda_event)))
    return c
