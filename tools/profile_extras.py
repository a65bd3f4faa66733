"""One launch each of the f-row kernels for ncu (collision field of a cfg3 union, MPPI, exact)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_01122_b200 as G  # noqa: E402
from paper_2603_01122_b200 import planners as PL  # noqa: E402
from paper_2603_01122_b200.occupancy import collision_layers_device  # noqa: E402

spec = G.GridSpec(400, 400, 0.1)
u = torch.rand((250, 400, 400), device="cuda", dtype=torch.float32) * 0.01
for _ in range(2):
    collision_layers_device(u, spec, 0.25, threshold=0.1, want_field=False)
st = G.PredictionStack(spec, u, 0.0, 0.02)
cfg = PL.MppiConfig(horizon=40, rollouts=4096, dt=0.1)
for _ in range(2):
    PL.mppi_step(PL.RobotState(5.0, 5.0, 0.5, 0.0), np.zeros((40, 2)), PL.RobotState(30.0, 20.0, 0.0, 0.0), st,
                 cfg, noise="production")
cs = G.ControlSet.grid(4, 24, 1.4)
space = G.HypothesisSpace(G.RationalitySet.log_spaced(5), G.GoalSet(np.array([[8.5, 5.0], [1.5, 7.0]])))
G.exact_predict(G.HumanState(5.05, 5.05), G.init_belief(space), 5, 0.1, cs, G.q_goal_progress(0.5), space,
                G.GridSpec(100, 100, 0.1), max_table=None)
torch.cuda.synchronize()
print("ok")
