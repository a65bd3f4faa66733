"""Production vs reference per-layer TV statistics at the cfg3 golden's inputs (GPU).

For S seeds of each mode, the TV of every (human, step) layer against the live reference's
golden layers (tests/golden/cfg3_cycle.npz): per human the mean / max over steps and seeds,
reference mode and production mode side by side.  A systematic production bias shows as a
production column consistently above the reference column; sampling noise as overlapping
columns.

    python tools/tv_diag.py [--seeds 6] [--steps 25] [--full]
(--full: the bench scene at its full horizon, TV against the GPU reference mode's own
mean layer over the reference seeds instead of the golden.)
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import golden_io  # noqa: E402
import paper_2603_01122_b200 as G  # noqa: E402
from paper_2603_01122_b200 import prediction as PR  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=6)
    ap.add_argument("--goal-radius", type=float, default=None)
    a = ap.parse_args()
    z = golden_io.load("cfg3_cycle.npz")
    meta = json.loads(str(z["meta"]))
    cs, q = G.ControlSet.grid(4, 24, 1.4), G.q_goal_progress(0.5)
    dev = torch.device("cuda")
    tabs = [PR.action_tables(cs, q, meta["dt"], dev), PR.action_tables(cs, G.mask_stationary(q, cs, 0.5), meta["dt"], dev)]
    jobs = []
    for i, hm in enumerate(meta["humans"]):
        space = G.HypothesisSpace(G.RationalitySet(tuple(meta["betas"])), G.GoalSet(np.array(hm["goals"])))
        jobs.append((hm, space))
    n, T, spec = meta["n"], meta["steps"], G.GridSpec(400, 400, 0.1)
    H = len(jobs)
    ref = np.zeros((H, T, 400, 400))
    for i in range(H):
        ref[i][tuple(z[f"layer_idx_{i}"].T)] = z[f"layer_val_{i}"]
    ref = torch.as_tensor(ref, device=dev)

    def layers(mode, seed, sigma=meta["sigma"]):
        js = [PR.HumanJob(G.HumanState(*hm["start"]), np.array(hm["log_w"]), sp.beta_of, sp.goal_xy_of, seed, (2, i),
                          int(hm["stationary"])) for i, (hm, sp) in enumerate(jobs)]
        return PR.run_predict(js, tabs, n, T, meta["dt"], sigma, spec, mode, want_hyp=True)

    def tv(u, v):
        return 0.5 * (u - v).abs().sum(dim=(2, 3))

    res = {}
    hypf = {}
    for mode in ("reference", "production"):
        tvs, hs = [], []
        for s in range(a.seeds):
            out = layers(mode, 1000 + 17 * s + (0 if mode == "reference" else 7))
            tvs.append(tv(out["layers"], ref).cpu().numpy())
            hs.append(np.stack([np.bincount(out["hyp"][i].cpu().numpy(), minlength=20) / n for i in range(H)]))
        res[mode] = np.stack(tvs)  # (S, H, T)
        hypf[mode] = np.stack(hs)  # (S, H, 20)
    print("per human: TV vs live reference layers over steps x seeds -- mean / p95 / max")
    for i in range(H):
        r, p = res["reference"][:, i], res["production"][:, i]
        print(f"human {i}: reference {r.mean():.5f} / {np.percentile(r, 95):.5f} / {r.max():.5f}   "
              f"production {p.mean():.5f} / {np.percentile(p, 95):.5f} / {p.max():.5f}")
    post = np.stack([np.exp(hm["log_w"]) for hm, _ in jobs])
    for mode in ("reference", "production"):
        d = hypf[mode] - post[None]
        print(f"{mode}: hypothesis frequency - posterior: mean |d| {np.abs(d).mean():.2e}, "
              f"max |d| {np.abs(d).max():.2e}, mean signed {d.mean(0).max():.2e}")
    worst = np.unravel_index(np.argmax(res["production"]), res["production"].shape)
    print("worst production layer (seed, human, step):", worst, float(res["production"][worst]))
    print("bound 1.5 x max-over-reference-seeds + 0.005 violated in",
          int((res["production"].max(0) > 1.5 * res["reference"].max(0) + 0.005).sum()), "of", H * T, "layers")


if __name__ == "__main__":
    main()
