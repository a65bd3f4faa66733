"""Digest of production-mode K2 outputs (counts / layers) for library A/B bit-identity:
run under GC_LIB_PATH=<lib> for two builds and compare the printed digests.  Covers the
symmetric sampler (4, 3 and 2 speeds, w_theta 0 and 0.2) and the generic fact sampler."""
import hashlib
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_01122_b200 as G  # noqa: E402
from paper_2603_01122_b200 import prediction as PR  # noqa: E402


def digest(cs, q, n=65536, steps=60, humans=4):
    spec = G.GridSpec(400, 400, 0.1)
    tab = PR.action_tables(cs, q, 0.02, torch.device("cuda"))
    jobs = []
    for h in range(humans):
        s = np.array([5.0 + 10.0 * (h % 4), 10.0 + 20.0 * (h // 4)])
        goals = np.stack([s + 3.5 * np.array([math.cos(a), math.sin(a)]) for a in (0.3, 1.9, 3.4, 5.0)])
        space = G.HypothesisSpace(G.RationalitySet.log_spaced(5), G.GoalSet(goals))
        lw = np.log(np.random.default_rng(h).dirichlet(np.ones(space.size)))
        lw -= np.log(np.exp(lw).sum())
        jobs.append(PR.HumanJob(G.HumanState(*s), lw, space.beta_of, space.goal_xy_of, 7, (2, h), 0))
    out = PR.run_predict(jobs, [tab], n, steps, 0.02, 0.1, spec, "production", per_human_layers=True)
    torch.cuda.synchronize()
    m = hashlib.sha256()
    for k in sorted(out):
        v = out[k]
        if isinstance(v, torch.Tensor):
            m.update(k.encode())
            m.update(v.detach().cpu().contiguous().numpy().tobytes())
    return tab.factorised, m.hexdigest()[:16]


def cases():
    """(label, factorised, digest) of each pinned case (tests/test_gpu_production_pinned.py)."""
    q = G.q_goal_progress(0.5)
    out = []
    for label, cs, qq in [
        ("grid(4,24)", G.ControlSet.grid(4, 24, 1.4), q),
        ("grid(4,24) w_theta", G.ControlSet.grid(4, 24, 1.4), G.q_goal_progress(0.5, (0.0, 0.2))),
        ("grid(3,24)", G.ControlSet.grid(3, 24, 1.4), q),
        ("grid(2,24)", G.ControlSet.grid(2, 24, 1.4), q),
        ("grid(4,16)", G.ControlSet.grid(4, 16, 1.4), q),
    ]:
        f, d = digest(cs, qq)
        out.append((label, f, d))
    return out


def main():
    for label, f, d in cases():
        print(f"{label:22s} factorised={f} {d}")


if __name__ == "__main__":
    main()
