"""B200-native NSFR residual path (arXiv 2312.07725) — see DESIGN.md.

The compute path is libnsfr_b200.so (hand-written sm_100a CUDA behind the C
ABI of include/nsfr_gpu.h); this package is its Python mirror.
"""
from .solver import (C_PLUS, CASES, ConfigError, DeviceError, DimensionError, GpuSolver,
                     InvalidMeshError, NsfrError, SolverConfig, StepFailureError, halo_plan,
                     load_library, measure_fp64_peak, nccl_unique_id)
from .runio import (DiagnosticsCSV, load_checkpoint, read_checkpoint, read_diagnostics,
                    run_simulation, write_checkpoint)

__all__ = ["C_PLUS", "CASES", "ConfigError", "DeviceError", "DimensionError", "GpuSolver",
           "InvalidMeshError", "NsfrError", "SolverConfig", "StepFailureError", "halo_plan",
           "load_library", "measure_fp64_peak", "nccl_unique_id", "DiagnosticsCSV",
           "load_checkpoint", "read_checkpoint", "read_diagnostics", "run_simulation",
           "write_checkpoint"]
