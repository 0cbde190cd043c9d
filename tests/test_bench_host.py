"""bench.py host logic on CPU: the kernel-specific ALU ceilings, the weak-scaled workload and its
row shards (what each rank of `bench.py --gpus N` combs), and the JSON config description."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_0909_2000_b200.sharding import plan_row_shards  # noqa: E402


def test_kernel_ceilings_follow_the_chosen_kernel():
    peak = 63.41
    c, what = bench.kernel_ceiling("comb2<10,10,2,fp16>", peak)
    assert abs(c - peak * 8 / 5) < 1e-9 and "r=2" in what
    assert abs(bench.kernel_ceiling("comb2<16,4,2,int>", peak)[0] - peak * 8 / 5) < 1e-9
    assert abs(bench.kernel_ceiling("comb<4,32,2,table,fp16>", peak)[0] - peak * 2 / 1.75) < 1e-9
    assert abs(bench.kernel_ceiling("comb<8,8,2,table,int>", peak)[0] - peak) < 1e-9
    assert abs(bench.kernel_ceiling("comb<8,16,4,computed,int>", peak)[0] - peak * 2 / 5) < 1e-9


def test_weak_scaled_workload_gives_every_rank_the_base_rows():
    for name in ("C1", "C2"):
        c, x1, y1 = bench.workload(name, 1)
        rows1 = (x1.size - c.w) // c.h + 1
        for world in (2, 4, 8):
            c, x, y = bench.workload(name, world)
            assert np.array_equal(y, y1) and np.array_equal(x[:x1.size], x1)
            shards = plan_row_shards(x.size, c.w, c.h, world)
            rows = [s.rows for s in shards]
            assert sum(rows) == (x.size - c.w) // c.h + 1
            # each rank combs the base workload's rows plus its share of the (w - 1)-row seams
            assert max(rows) - min(rows) <= 1 and rows1 <= min(rows) <= rows1 + c.w


def test_config_description_and_cells():
    c, x, y = bench.workload("C1", 1)
    d = bench.config_desc(c, x, y, 1, "C1")
    assert d["rows"] == 1937 and d["cols"] == 1937 and d["w"] == 64 and d["parallelism"] == "1 GPU"
    assert bench.comb_cells(d["rows"], c, y.size) == 1937 * 64 * 2000
