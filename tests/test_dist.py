"""Multi-rank path on CPU: world_size-2 gloo run of the row-sharded product
(paper_0803_1975_b200/dist.py) with the oracle standing in for the kernels.
Checks the shard geometry, the broadcast of the packed right operand, and
that the gathered C equals naive_gemm."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_0803_1975_b200.dist import (PanelOps, ShardOps, mul_common_sharded, mul_common_sharded_pipelined,
                                       panel_bounds, shard_rows)


def test_shard_rows_cover_exactly():
    for m in (0, 1, 7, 70, 4096, 32769):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_rows(m, world, r) for r in range(world)]
            assert sum(rows for _, rows in spans) == m
            pos = 0
            for row0, rows in spans:
                assert row0 == pos
                pos += rows
            assert max(r for _, r in spans) - min(r for _, r in spans) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, p, m, k, n):
    import oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = O.plan_compression(p, k)
        K = -(-k // plan.e)
        row0, rows = shard_rows(m, world, rank)
        a_shard = O.random_residue_matrix(rows, k, p, 42, row0=row0)
        b = O.random_residue_matrix(k, n, p, 43) if rank == 0 else None

        def contract(ca, cb):
            acc = O.packed_common_product(plan, ca.numpy(), cb.numpy(), k)
            return torch.from_numpy(((acc.astype(np.uint64) & np.uint64((1 << plan.t) - 1)) % np.uint64(p)).astype(np.int32))

        ops = ShardOps(
            pack_rows=lambda a: torch.from_numpy(O.compress_rows_reversed(plan, a)),
            pack_cols=lambda bb: torch.from_numpy(O.compress_cols_forward(plan, bb)),
            empty_cb=lambda shape: torch.empty(shape, dtype=torch.float64),
            contract=contract,
        )
        c_shard, cb = mul_common_sharded(a_shard, b, (K, n), ops, rank, world)
        # every rank must hold rank 0's packed words bit for bit
        want_cb = O.compress_cols_forward(plan, O.random_residue_matrix(k, n, p, 43))
        assert np.array_equal(cb.numpy().view(np.uint64), want_cb.view(np.uint64))
        sizes = [shard_rows(m, world, r)[1] for r in range(world)]
        top = max(sizes)  # gloo gathers equal shapes: pad ragged shards
        padded = torch.zeros((top, n), dtype=torch.int32)
        padded[:rows] = c_shard
        gathered = [torch.empty((top, n), dtype=torch.int32) for _ in sizes] if rank == 0 else None
        dist.gather(padded, gathered, dst=0)
        if rank == 0:
            c = torch.cat([g[:s] for g, s in zip(gathered, sizes)]).numpy().astype(np.uint32)
            full_a = O.random_residue_matrix(m, k, p, 42)
            assert np.array_equal(c, O.naive_gemm(p, full_a, O.random_residue_matrix(k, n, p, 43)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p,m,k,n", [(7, 70, 300, 50), (3, 9, 512, 33)])
def test_row_sharded_world2_gloo(p, m, k, n):
    mp.spawn(_worker, args=(2, _free_port(), p, m, k, n), nprocs=2, join=True)


def test_panel_bounds_cover_exactly():
    for nt in (1, 5, 32, 33, 256):
        for panels in (1, 2, 3, 4, 8):
            spans = [panel_bounds(nt, panels, j) for j in range(panels)]
            assert spans[0][0] == 0 and spans[-1][1] == nt
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def _worker_panels(rank, world, port, p, m, k, n, panels):
    """Pipelined (column-panel) broadcast: CB kept column-major (n x K, the
    tiled layout's tn-major order in miniature) so a panel is contiguous."""
    import oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = O.plan_compression(p, k)
        K = -(-k // plan.e)
        row0, rows = shard_rows(m, world, rank)
        a_shard = O.random_residue_matrix(rows, k, p, 42, row0=row0)
        b = O.random_residue_matrix(k, n, p, 43) if rank == 0 else None
        cbt = torch.empty((n, K), dtype=torch.float64)  # column-major CB

        def views(cb, panels_):
            return [cb[slice(*panel_bounds(n, panels_, j))] for j in range(panels_)]

        def pack_panel(bb, j, panels_, cb):
            c0, c1 = panel_bounds(n, panels_, j)
            cb[c0:c1] = torch.from_numpy(O.compress_cols_forward(plan, np.ascontiguousarray(bb[:, c0:c1])).T.copy())

        def contract(ca, cb):
            acc = O.packed_common_product(plan, ca.numpy(), np.ascontiguousarray(cb.numpy().T), k)
            return torch.from_numpy(((acc.astype(np.uint64) & np.uint64((1 << plan.t) - 1)) % np.uint64(p)).astype(np.int32))

        ops = PanelOps(pack_rows=lambda a: torch.from_numpy(O.compress_rows_reversed(plan, a)),
                       panel_views=views, pack_cols_panel=pack_panel, contract=contract)
        c_shard, cb = mul_common_sharded_pipelined(a_shard, b, cbt, ops, rank, world, panels)
        want_cb = O.compress_cols_forward(plan, O.random_residue_matrix(k, n, p, 43))
        assert np.array_equal(np.ascontiguousarray(cb.numpy().T).view(np.uint64), want_cb.view(np.uint64))
        want_c = O.naive_gemm(p, a_shard, O.random_residue_matrix(k, n, p, 43))
        assert np.array_equal(c_shard.numpy().astype(np.uint32), want_c)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p,m,k,n,panels", [(7, 70, 300, 50, 4), (3, 9, 512, 33, 3), (5, 16, 100, 7, 8)])
def test_pipelined_broadcast_world2_gloo(p, m, k, n, panels):
    mp.spawn(_worker_panels, args=(2, _free_port(), p, m, k, n, panels), nprocs=2, join=True)


def test_aligned_shards_and_slots_cover_exactly():
    from paper_0803_1975_b200.dist import gather_slot, shard_rows_aligned

    for m in (0, 1, 100, 512, 4096, 32768, 32769):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_rows_aligned(m, world, r) for r in range(world)]
            assert sum(rows for _, rows in spans) == m
            pos = 0
            for row0, rows in spans:
                assert row0 == pos and (rows % 128 == 0 or row0 + rows == m)
                pos += rows
    for nt in (1, 3, 32, 256, 257):
        for world in (1, 2, 3, 8):
            slots = [gather_slot(nt, world, r) for r in range(world)]
            assert slots[0][0] == 0 and max(s[1] for s in slots) == nt
            assert all(a[1] == b[0] or b[0] == b[1] for a, b in zip(slots, slots[1:]))
            assert all(s[1] - s[0] <= s[2] for s in slots)
    assert [shard_rows_aligned(32768, 8, r)[1] for r in range(8)] == [4096] * 8


TILE = 4  # columns per "tile column" in the miniature layout


def _worker_gather(rank, world, port, p, m, k, n):
    """All-gather form (strong scaling): every rank packs only its own
    tile-column slot of CB (kept column-major, TILE columns per tile, so a
    slot is contiguous like the tiled CB_t), the slots are all-gathered in
    place, and the rank contracts its own slot first."""
    import oracle as O
    from paper_0803_1975_b200.dist import GatherOps, gather_slot, mul_common_allgather, shard_rows_aligned

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = O.plan_compression(p, k)
        K = -(-k // plan.e)
        row0, rows = shard_rows_aligned(m, world, rank, align=8)
        a_shard = O.random_residue_matrix(rows, k, p, 42, row0=row0)
        b = O.random_residue_matrix(k, n, p, 43)  # each rank reads only its own slot's columns
        nt = -(-n // TILE)
        _, _, per = gather_slot(nt, world, rank)
        cb = torch.zeros(world * per * TILE * K, dtype=torch.float64)
        c = torch.full((rows, n), -1, dtype=torch.int32)
        order = []

        def pack_slot(bb, t0, t1, slot):
            c0, c1 = t0 * TILE, min(n, t1 * TILE)
            if c1 > c0:
                words = O.compress_cols_forward(plan, np.ascontiguousarray(bb[:, c0:c1])).T.copy()  # cols x K
                slot[:words.size] = torch.from_numpy(words.reshape(-1))

        def contract(ca, cb_, t0, t1):
            order.append((t0, t1))
            c0, c1 = t0 * TILE, min(n, t1 * TILE)
            cols = cb_[t0 * TILE * K:t0 * TILE * K + (c1 - c0) * K].numpy().reshape(c1 - c0, K)
            acc = O.packed_common_product(plan, ca.numpy(), np.ascontiguousarray(cols.T), k)
            c[:, c0:c1] = torch.from_numpy(((acc.astype(np.uint64) & np.uint64((1 << plan.t) - 1)) %
                                            np.uint64(p)).astype(np.int32))

        ops = GatherOps(pack_rows=lambda a: torch.from_numpy(O.compress_rows_reversed(plan, a)),
                        pack_cols_slot=pack_slot, contract=contract)
        mul_common_allgather(a_shard, b, cb, ops, rank, world, nt)
        # every rank ends with the whole packed B, bit for bit
        want_cb = O.compress_cols_forward(plan, O.random_residue_matrix(k, n, p, 43))
        got = cb[:n * K].numpy().reshape(n, K).T
        assert np.array_equal(np.ascontiguousarray(got).view(np.uint64), want_cb.view(np.uint64))
        t0, t1, _ = gather_slot(nt, world, rank)
        if t1 > t0:
            assert order[0] == (t0, t1)  # own slot first
        assert sorted(order) == sorted(set(order)) and sum(b - a for a, b in order) == nt
        want_c = O.naive_gemm(p, a_shard, O.random_residue_matrix(k, n, p, 43))
        assert np.array_equal(c.numpy().astype(np.uint32), want_c)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p,m,k,n", [(7, 70, 300, 50), (3, 9, 512, 33), (5, 16, 100, 7), (3, 5, 64, 3)])
def test_allgather_world2_gloo(p, m, k, n):
    mp.spawn(_worker_gather, args=(2, _free_port(), p, m, k, n), nprocs=2, join=True)
