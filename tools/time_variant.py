"""Time K VL2 cycles of the 256^3 bench workload with whatever library
PMHD_GPU_LIB points to, ignoring solver errors (for throwaway performance
probes whose arithmetic is deliberately wrong)."""
import sys, time
sys.path.insert(0, '.')
import torch
from bench import make_config
from paper_1905_04341_b200.solver import GpuSolver
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = make_config(n, 1)
g = GpuSolver(cfg)
g.load_pgen()
dt = g.new_dt()
def step():
    try:
        g.vl2_step(dt)
    except Exception:
        pass
for _ in range(2):
    step()
torch.cuda.synchronize()
s = torch.cuda.ExternalStream(g.stream_handle)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
K = 5
for _ in range(K):
    step()
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
print(f"{ms:.3f} ms/cycle  {n**3/ms/1e6:.3f}e9 cups")
