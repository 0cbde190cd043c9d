"""bench.py host logic on CPU: the kernel-specific ALU op counts behind roofline.frac, the
weak- and strong-scaled workloads and their row shards (what each rank of `bench.py --gpus N`
combs), and the JSON config description."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_0909_2000_b200.sharding import plan_row_shards  # noqa: E402


def test_kernel_alu_ops_follow_the_chosen_kernel():
    assert bench.kernel_alu_ops_per_cell("comb2<10,10,2,fp16>")[0] == 5 / 8
    assert bench.kernel_alu_ops_per_cell("comb2<16,4,2,int>")[0] == 5 / 8
    assert bench.kernel_alu_ops_per_cell("comb<4,32,2,table,fp16>")[0] == 1.75 / 2
    assert bench.kernel_alu_ops_per_cell("comb<8,8,2,table,int>")[0] == 1.0
    assert bench.kernel_alu_ops_per_cell("comb<8,16,4,computed,int>")[0] == 2.5
    assert bench.kernel_alu_ops_per_cell("combw<8,16,table,packed>")[0] == 1.0
    assert bench.kernel_alu_ops_per_cell("combw<8,16,table>")[0] == 2.0
    assert bench.kernel_alu_ops_per_cell("combw<32,16,computed>")[0] == 3.0


def test_default_scaling_per_config():
    assert bench.default_scaling("C4") == "strong" and bench.default_scaling("C5") == "strong"
    assert all(bench.default_scaling(n) == "weak" for n in ("C1", "C2", "C3"))


def test_weak_scaled_workload_gives_every_rank_the_base_rows():
    for name in ("C1", "C2"):
        c, x1, y1 = bench.workload(name, 1, "weak")
        rows1 = (x1.size - c.w) // c.h + 1
        for world in (2, 4, 8):
            c, x, y = bench.workload(name, world, "weak")
            assert np.array_equal(y, y1) and np.array_equal(x[:x1.size], x1)
            shards = plan_row_shards(x.size, c.w, c.h, world)
            rows = [s.rows for s in shards]
            assert sum(rows) == (x.size - c.w) // c.h + 1
            # each rank combs the base workload's rows plus its share of the (w - 1)-row seams
            assert max(rows) - min(rows) <= 1 and rows1 <= min(rows) <= rows1 + c.w


def test_strong_scaled_workload_splits_the_fixed_plot():
    """--scaling strong: the config's own plot, its rows split into contiguous blocks with a
    w-1 halo each, covering every row exactly once (C4 over 1/2/4/8 GPUs)."""
    c, x1, y1 = bench.workload("C4", 1, "strong")
    rows = (x1.size - c.w) // c.h + 1
    assert rows == 262081
    for world in (2, 4, 8):
        c, x, y = bench.workload("C4", world, "strong")
        assert np.array_equal(x, x1) and np.array_equal(y, y1)
        shards = plan_row_shards(x.size, c.w, c.h, world)
        assert shards[0].row_begin == 0 and shards[-1].row_end == rows
        for a, b in zip(shards, shards[1:]):
            assert a.row_end == b.row_begin
        for s in shards:
            assert s.x_begin == s.row_begin * c.h and s.x_end == (s.row_end - 1) * c.h + c.w
        assert max(s.rows for s in shards) - min(s.rows for s in shards) <= 1


def test_config_description_and_cells():
    c, x, y = bench.workload("C1", 1, "weak")
    d = bench.config_desc(c, x, y, 1, "C1", "weak")
    assert d["rows"] == 1937 and d["cols"] == 1937 and d["w"] == 64 and d["parallelism"] == "1 GPU"
    assert bench.comb_cells(d["rows"], c, y.size) == 1937 * 64 * 2000
    c, x, y = bench.workload("C4", 8, "strong")
    assert "fixed plot" in bench.config_desc(c, x, y, 8, "C4", "strong")["parallelism"]
