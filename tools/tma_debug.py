"""Debug helper: one small 3D case through the update kernels of a given
library (PMHD_GPU_LIB), reporting the first CUDA error."""
import sys
from paper_1905_04341_b200 import RunConfig
from paper_1905_04341_b200.solver import GpuSolver

cfg = RunConfig(nx1=int(sys.argv[1]), nx2=int(sys.argv[1]), nx3=int(sys.argv[1]),
                mb1=int(sys.argv[1]), mb2=int(sys.argv[1]), mb3=int(sys.argv[1]), wave_n1=1, wave_amp=1e-3)
g = GpuSolver(cfg)
g.load_pgen()
dt = g.new_dt()
try:
    for _ in range(2):
        dt, st = g.vl2_step(dt)
    print("ok", dt)
except Exception as e:
    print("ERR", e)
