"""B200-native alignment-plot engine (Krusche & Tiskin, "Computing alignment plots efficiently").

The engine is the CUDA library ``libalignplot_b200.so`` (sources in ``csrc/``,
C ABI in ``include/alignplot_b200.h``).  ``alignplot`` mirrors the reference
C++ library's interface on top of it; ``datagen`` makes the seeded synthetic
inputs of the five BASELINE configs; ``sharding`` is the multi-GPU row-shard
driver (one process per GPU).
"""
from . import alignplot  # noqa: F401
from .alignplot import (  # noqa: F401
    ConfigError, EmptyPlotError, Mode, NoDeviceError, PlotCell, PlotConfig, PlotGrid, Sequence,
    apply_threshold, blowup, compute_plot, compute_plot_threshold, plan_strips, recover_score, unblow,
    window_grid_dims,
)

__all__ = [
    "alignplot", "ConfigError", "EmptyPlotError", "Mode", "NoDeviceError", "PlotCell", "PlotConfig",
    "PlotGrid", "Sequence", "apply_threshold", "blowup", "compute_plot", "compute_plot_threshold",
    "plan_strips", "recover_score", "unblow", "window_grid_dims",
]
