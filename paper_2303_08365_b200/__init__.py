"""B200-native Jacobi stencil sweep with the reference's API
(arXiv 2303.08365 artifact, `tessera`).

A user of ``import tessera as ts`` switches with
``import paper_2303_08365_b200 as ts``: kernels, grids, ``fill_random``,
``naive_run`` / ``run_tessellated`` and the metrics keep their names and
argument meaning; the sweeps run in hand-written sm_100a kernels through the
C-ABI in ``include/tessera_b200.h``.  There is no CPU fallback.
"""
from .kernel import (StencilKernel, BenchmarkSpec, benchmark_names, benchmark_table,
                     box_kernel, find_benchmark, heat_coefficients, lattice_offsets, make_kernel,
                     star_kernel)
from .grid import (BasicGrid, Grid, GridF, dump_grid, fill_random, grid_from_numpy, load_grid)
from .run import (GpuStats, Tile, TilePlan, axis_range, count_coverage, naive_run, naive_step,
                  plan_tiles, release_cache, run_gpu, run_tessellated, tile_range)
from .metrics import RateReport, deviation, max_abs, max_rel_deviation, stencils_per_second
from .device import DeviceGrid, layout_of
from .harness import csv_header, csv_row, run_all, run_benchmark, write_csv
from .scheduler import (CommCostModel, CommLog, CommRecord, PartitionPlan, SlabGrid,
                        WorkerProfile, WorkerSpec, comm_cost, dump_comm_log, plan_partition,
                        profile_workers, run_heterogeneous, run_heterogeneous_instrumented,
                        run_multi)

__version__ = "0.1.0"

__all__ = [
    "StencilKernel", "BenchmarkSpec", "benchmark_names", "benchmark_table", "box_kernel",
    "find_benchmark", "heat_coefficients", "lattice_offsets", "make_kernel", "star_kernel",
    "BasicGrid", "Grid", "GridF", "dump_grid", "fill_random", "grid_from_numpy", "load_grid",
    "GpuStats", "Tile", "TilePlan", "axis_range", "count_coverage", "tile_range", "naive_run", "naive_step", "plan_tiles", "release_cache", "run_gpu",
    "run_tessellated", "RateReport", "deviation", "max_abs", "max_rel_deviation",
    "stencils_per_second", "DeviceGrid", "layout_of", "run_benchmark", "run_all", "csv_header",
    "csv_row", "write_csv", "CommCostModel", "CommLog", "CommRecord", "PartitionPlan",
    "SlabGrid", "WorkerProfile", "WorkerSpec", "comm_cost", "dump_comm_log", "plan_partition",
    "profile_workers", "run_heterogeneous", "run_heterogeneous_instrumented", "run_multi",
]
