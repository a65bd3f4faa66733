"""Time the collision field + blocked mask of a cfg3-sized (250, 400, 400) float32 union
(the engine's per-cycle planner input; GC_LIB_PATH selects a library build)."""
import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2603_01122_b200 import occupancy as O
import paper_2603_01122_b200 as G
spec = G.GridSpec(400, 400, 0.1)
u = torch.rand((250, 400, 400), device='cuda', dtype=torch.float32) * 0.01
for _ in range(2): O.collision_layers_device(u, spec, 0.25, 0.1, want_field=False)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): O.collision_layers_device(u, spec, 0.25, 0.1, want_field=False)
b.record(); torch.cuda.synchronize()
print("collision 250x400x400 r=0.25:", a.elapsed_time(b) / 10, "ms")
