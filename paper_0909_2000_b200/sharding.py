"""Multi-GPU row-shard driver: one process per GPU (torch.distributed), no data-path collective.

Grid rows (x-window strips) are independent (runner.cpp:97-110),
so rank g of G owns the contiguous rows [floor(g*R/G), floor((g+1)*R/G)) and
needs only the x bytes [r0*h, (r1-1)*h + w): its rows plus a w-1 halo
(SURVEY.md §8e).  y is replicated.  Concatenating the ranks' row blocks in
rank order is the global row-major order, so:

* dense output: rank g's block lands at row offset r0 -- nothing to exchange;
* thresholded output: the only collective is one all_gather of a u64 hit
  count per rank, giving each rank its global list offset.

The compute step is a callable so the same driver is exercised on CPU with
the gloo backend in tests (with the oracle as the compute) and on GPUs with
NCCL and the CUDA engine.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Tuple

import numpy as np


@dataclass(frozen=True)
class RowShard:
    rank: int
    row_begin: int      # global grid rows [row_begin, row_end)
    row_end: int
    x_begin: int        # x bytes [x_begin, x_end) = rows + (w-1) halo
    x_end: int

    @property
    def rows(self) -> int:
        return self.row_end - self.row_begin


def plan_row_shards(m: int, w: int, h: int, world: int) -> List[RowShard]:
    """Contiguous, balanced row blocks (per-row cost is constant) with their x halo."""
    if w == 0 or h == 0 or w > m:
        raise ValueError("no window fits")
    rows = (m - w) // h + 1
    shards = []
    for g in range(world):
        r0 = rows * g // world
        r1 = rows * (g + 1) // world
        if r1 > r0:
            shards.append(RowShard(g, r0, r1, r0 * h, (r1 - 1) * h + w))
        else:
            shards.append(RowShard(g, r0, r0, r0 * h, r0 * h))
    return shards


def shard_x(x: np.ndarray, s: RowShard) -> np.ndarray:
    """The x slice a shard needs (rows plus halo); its local row i is global row s.row_begin + i."""
    return x[s.x_begin:s.x_end]


def gather_counts(local_count: int, group=None) -> Tuple[int, int]:
    """All-gather one u64 hit count per rank -> (this rank's global offset, global total).

    This is the path's only collective (NCCL over NVLink on GPUs, gloo in CPU tests).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([int(local_count)], dtype=torch.int64, device=dev)
    out = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    counts = [int(v.item()) for v in out]
    return sum(counts[:rank]), sum(counts)


def gather_list_to_root(rows: np.ndarray, cols: np.ndarray, halves: np.ndarray, root: int = 0, group=None):
    """Concatenate every rank's row-major part of a thresholded list on `root`, in rank (= row)
    order: apply_threshold's whole list (scoring.cpp:30-39) where the caller wants it in one place.

    One all_gather of the counts, then each rank's (row, col, half) triples padded to the longest
    part and all_gathered as one int64 tensor (NCCL over NVLink on GPUs, device-resident when the
    backend is NCCL; gloo in CPU tests).  Returns (rows, cols, halves) on root and None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    n = int(rows.size)
    cnt = torch.tensor([n], dtype=torch.int64, device=dev)
    cnts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    counts = [int(v.item()) for v in cnts]
    width = max(max(counts), 1)
    mine = torch.zeros((3, width), dtype=torch.int64, device=dev)
    if n:
        mine[0, :n] = torch.from_numpy(rows.astype(np.int64)).to(dev)
        mine[1, :n] = torch.from_numpy(cols.astype(np.int64)).to(dev)
        mine[2, :n] = torch.from_numpy(halves.astype(np.int16).astype(np.int64)).to(dev)
    parts = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    if rank != root:
        return None
    full = torch.cat([p_[:, :c] for p_, c in zip(parts, counts)], dim=1).cpu().numpy()
    return full[0].astype(np.uint32), full[1].astype(np.uint32), full[2].astype(np.int32)


def run_sharded_threshold(x: np.ndarray, y: np.ndarray, w: int, h: int, rank: int, world: int,
                          compute: Callable[[np.ndarray, np.ndarray, int], Tuple[np.ndarray, np.ndarray, np.ndarray]],
                          group=None):
    """Thresholded plot of this rank's shard.

    compute(x_slice, y, row_begin) -> (rows, cols, halves) in global row numbering.
    Returns (global_offset, global_total, rows, cols, halves) for this rank's hits;
    writing each rank's arrays at its offset yields apply_threshold's row-major list.
    """
    s = plan_row_shards(x.size, w, h, world)[rank]
    if s.rows:
        rr, cc, hh = compute(shard_x(x, s), y, s.row_begin)
    else:
        rr = cc = np.zeros(0, np.uint32)
        hh = np.zeros(0, np.uint16)
    off, total = gather_counts(rr.size, group)
    return off, total, rr, cc, hh


def run_sharded_dense(x: np.ndarray, y: np.ndarray, w: int, h: int, rank: int, world: int,
                      compute: Callable[[np.ndarray, np.ndarray], np.ndarray]):
    """Dense rows of this rank's shard: (row_begin, block[rows, cols]).  No collective."""
    s = plan_row_shards(x.size, w, h, world)[rank]
    if not s.rows:
        return s.row_begin, np.zeros((0, y.size - w + 1), np.int32)
    return s.row_begin, compute(shard_x(x, s), y)
