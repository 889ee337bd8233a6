"""B200-native DJ-TLED explicit-dynamics engine (arXiv:2106.14189).

The hot path (element forces -> CSR gather -> central-difference update) runs
as sm_100a CUDA kernels in libdjg.so behind the C-ABI of include/djg.h; the
host-side problem builder (include/djg_host.h) is native C++ in the same
library. This package is the Python mirror of the reference's solver API.
"""
from . import _abi
from .engine import (ConfigError, CudaError, GpuDjEngine, RunResult, Scenario, SimulationError, StepReport,
                     run_simulation)
from .spec import CONFIGS, Spec, bench_material, box_counts, box_spec, config_spec, material, mesh_spec

__all__ = [
    "ConfigError", "CudaError", "GpuDjEngine", "RunResult", "Scenario", "SimulationError", "StepReport",
    "run_simulation", "CONFIGS", "Spec", "bench_material", "box_counts", "box_spec", "config_spec", "material",
    "mesh_spec",
]
