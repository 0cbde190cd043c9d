"""Multi-GPU row-shard driver (paper_0909_2000_b200/sharding.py) on CPU: world_size 2, gloo.

The compute step is the oracle here (the CUDA engine runs the same driver under
NCCL in bench.py); what is tested is the host logic: the row partition with its
w-1 halo, the count all_gather, and that concatenating the ranks' outputs in
rank order equals the single-process row-major result.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_lib as ol
from paper_0909_2000_b200.sharding import (gather_list_to_root, plan_row_shards, run_sharded_dense,
                                           run_sharded_threshold, shard_x)


def test_plan_covers_rows_once_with_halo():
    for m, w, h, world in [(1000, 64, 1, 2), (1000, 64, 3, 4), (777, 100, 5, 8), (70, 64, 1, 8)]:
        shards = plan_row_shards(m, w, h, world)
        rows = (m - w) // h + 1
        covered = []
        for s in shards:
            covered += list(range(s.row_begin, s.row_end))
            if s.rows:
                assert s.x_begin == s.row_begin * h
                assert s.x_end == (s.row_end - 1) * h + w   # rows plus the w-1 halo
        assert covered == list(range(rows))
        sizes = [s.rows for s in shards]
        assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, x, y, w, h, r, t, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def compute_thr(xs, yy, row0):
            rc, g = ol.plot_rows(xs, yy, w, h, r, workers=1)
            rr, cc = np.nonzero(g >= t)
            return (rr + row0).astype(np.uint32), cc.astype(np.uint32), g[rr, cc].astype(np.uint16)

        def compute_dense(xs, yy):
            rc, g = ol.plot_rows(xs, yy, w, h, r, workers=1)
            return g

        off, total, rr, cc, hh = run_sharded_threshold(x, y, w, h, rank, world, compute_thr)
        r0, block = run_sharded_dense(x, y, w, h, rank, world, compute_dense)
        whole = gather_list_to_root(rr, cc, hh, root=0)
        q.put((rank, off, total, rr, cc, hh, r0, block, whole))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("w,h,r,world", [(32, 1, 1, 2), (20, 3, 2, 2), (24, 1, 2, 4)])
def test_gloo_matches_single_process(w, h, r, world):
    """Strong split of one fixed plot: each rank's global list offset is the exclusive prefix of
    the gathered counts, and writing every rank's list / row block at its offset reproduces the
    single-process row-major result."""
    rng = np.random.default_rng(11)
    x = rng.integers(1, 5, 400).astype(np.uint8)
    y = np.concatenate([x[50:250], rng.integers(1, 5, 150)]).astype(np.uint8)
    rc, full = ol.plot_rows(x, y, w, h, r)
    t = int(np.quantile(full, 0.98))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, world, port, x, y, w, h, r, t, q)) for k in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda v: v[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    er, ec = np.nonzero(full >= t)
    total = res[0][2]
    assert all(v[2] == total for v in res) and total == er.size
    out_r = np.zeros(total, np.uint32)
    out_c = np.zeros(total, np.uint32)
    out_h = np.zeros(total, np.uint16)
    shards = plan_row_shards(x.size, w, h, world)
    expect_off = 0
    for rank, off, _, rr, cc, hh, r0, block, whole in res:
        assert off == expect_off   # exclusive prefix of the gathered counts, in rank (= row) order
        expect_off += rr.size
        s = shards[rank]
        assert rr.size == 0 or (s.row_begin <= int(rr.min()) and int(rr.max()) < s.row_end)
        assert rr.size == int(np.count_nonzero(full[s.row_begin:s.row_end] >= t))
        out_r[off:off + rr.size], out_c[off:off + cc.size], out_h[off:off + hh.size] = rr, cc, hh
    assert np.array_equal(out_r, er) and np.array_equal(out_c, ec) and np.array_equal(out_h, full[er, ec])
    # the whole list gathered on rank 0 (None elsewhere) is apply_threshold's row-major list
    gr, gc, gh = res[0][8]
    assert np.array_equal(gr, er) and np.array_equal(gc, ec) and np.array_equal(gh, full[er, ec])
    assert all(v[8] is None for v in res[1:])
    dense = np.concatenate([v[7] for v in res], axis=0)
    assert np.array_equal(dense, full)
    assert [v[6] for v in res] == [s.row_begin for s in plan_row_shards(x.size, w, h, world)]
