"""K2 time of the production samplers at the cfg3 shape (8 humans x 262,144 x 250): the
factorised grid sampler (plain and with a heading penalty w_theta) vs the generic
per-action softmax (a 96-action control set that is not a speed x heading grid)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_01122_b200 as G  # noqa: E402
from paper_2603_01122_b200 import prediction as PR  # noqa: E402


def time_k2(cs, q, label, n=262144, steps=250, humans=8):
    spec = G.GridSpec(400, 400, 0.1)
    dev = torch.device("cuda")
    tab = PR.action_tables(cs, q, 0.02, dev)
    jobs = []
    for h in range(humans):
        s = np.array([5.0 + 10.0 * (h % 4), 10.0 + 20.0 * (h // 4)])
        goals = np.stack([s + 3.5 * np.array([math.cos(a), math.sin(a)]) for a in (0.3, 1.9, 3.4, 5.0)])
        space = G.HypothesisSpace(G.RationalitySet.log_spaced(5), G.GoalSet(goals))
        lw = np.log(np.random.default_rng(h).dirichlet(np.ones(space.size)))
        lw -= np.log(np.exp(lw).sum())
        jobs.append(PR.HumanJob(G.HumanState(*s), lw, space.beta_of, space.goal_xy_of, 7, (2, h), 0))
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        PR.run_predict(jobs, [tab], n, steps, 0.02, 0.1, spec, "production", per_human_layers=False, union32=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{label}: factorised={tab.factorised}  K2+K3 {min(ts[1:]):.2f} ms")


def main():
    q = G.q_goal_progress(0.5)
    time_k2(G.ControlSet.grid(4, 24, 1.4), q, "grid(4, 24, 1.4)")
    time_k2(G.ControlSet.grid(4, 24, 1.4), G.q_goal_progress(0.5, (0.0, 0.2)), "grid(4, 24, 1.4), w_theta 0.2")
    r = np.random.default_rng(0)
    acts = [G.ControlAction(float(v), float(t)) for v, t in zip(r.uniform(0, 1.4, 96), r.uniform(-math.pi, math.pi, 96))]
    time_k2(G.ControlSet(acts), q, "96 random actions")
    time_k2(G.ControlSet.grid(4, 24, 1.4), G.q_default((0.3, 0.1)), "grid(4, 24, 1.4), q_default")


if __name__ == "__main__":
    main()
