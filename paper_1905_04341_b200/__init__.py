"""paper_1905_04341_b200 -- B200-native fp64 VL2+PLM+HLLD/HLLE+CT MHD update.

Host side: ``mesh`` (RunConfig / MeshBlock / problem generators over the C++
host library) and ``solver.GpuSolver`` (the reference's solver ops over the
CUDA C-ABI ``include/pmhd_gpu.h``).  There is no CPU fallback.
"""
from .mesh import RunConfig, BlockState, l1_error, ConfigError, ParseError, UnphysicalStateError  # noqa: F401

__all__ = ["RunConfig", "BlockState", "l1_error", "ConfigError", "ParseError",
           "UnphysicalStateError"]
