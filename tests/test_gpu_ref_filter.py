"""Reference-mode filter (gc_predict.cu ref_pick): the MUFU-ex2 first pass with a proven
error margin and numpy-exp fallback must give exactly the picks of the numpy-exp path.

The goldens in test_gpu_parity.py / test_gpu_headline_parity.py already pin the default
(filtered) path to the live reference; here the filter is compared with the exact-only
path (``ref_exact_only``) on belief shapes chosen to stress the margin -- near-uniform
policies (beta -> 0: every cdf entry is a live boundary), very peaked ones (beta = 300: the
exponentials span the float32 range and underflow), q_default, the stationary mask, a
ragged particle count -- at K = 1 and K = 4 launch shapes.  Every particle's hypothesis,
final float32 position and every per-step count must be identical.  The fallback rate is
printed (it sets the filter's speed-up) and must stay small."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2603_01122_b200 as G  # noqa: E402
from paper_2603_01122_b200 import prediction as PR  # noqa: E402


def _jobs(betas, n_goals, humans, seed, log_w=None, room=40.0, q_tab=0):
    rng = np.random.default_rng(seed)
    jobs = []
    for i in range(humans):
        s = rng.uniform(0.3 * room, 0.7 * room, 2)
        ang = rng.uniform(0, 2 * np.pi, n_goals)
        goals = np.stack([s[0] + 14 * np.cos(ang), s[1] + 14 * np.sin(ang)], 1)
        space = G.HypothesisSpace(G.RationalitySet(tuple(betas)), G.GoalSet(goals))
        lw = np.full(len(space.beta_of), -np.log(len(space.beta_of))) if log_w is None else log_w
        jobs.append(PR.HumanJob(G.HumanState(*s), lw, space.beta_of, space.goal_xy_of, 1000 + 17 * i, (2, i), q_tab))
    return jobs


def _run(jobs, tabs, n, steps, spec, exact):
    fb = torch.zeros(1, dtype=torch.int64, device="cuda")
    out = PR.run_predict(jobs, tabs, n, steps, 0.1, 0.0, spec, "reference", per_human_layers=False,
                         want_hyp=True, want_xy=True, ref_exact_only=exact, ref_fallbacks=fb)
    torch.cuda.synchronize()
    return out, int(fb.item())


CASES = {
    # name: (betas, goals, humans, n, steps, q, mask, max fallback rate)
    "bench_like": ((0.1, 0.3162, 1.0, 3.162, 10.0), 3, 8, 65536, 30, "gp", False, 0.05),
    "near_uniform": ((0.001, 0.01), 2, 4, 65536, 20, "gp", False, 0.10),
    "peaked": ((30.0, 300.0), 3, 4, 65536, 20, "gp", False, 0.05),
    "q_default": ((0.5, 5.0), 2, 4, 65536, 20, "default", False, 0.10),
    "masked": ((0.3, 3.0), 2, 4, 65536, 20, "gp", True, 0.10),
    "k4_ragged": ((0.1, 1.0, 10.0), 3, 9, 70001, 12, "gp", False, 0.05),
}


@pytest.mark.parametrize("name", list(CASES))
def test_filter_picks_equal_numpy_exp_picks(name):
    betas, ng, H, n, T, qk, mask, max_rate = CASES[name]
    cs = G.ControlSet.grid(4, 24, 1.4)
    q = G.q_goal_progress(0.5) if qk == "gp" else G.q_default((0.3, 0.1))
    if mask:
        q = G.mask_stationary(q, cs, 0.5)
    tabs = [PR.action_tables(cs, q, 0.1, torch.device("cuda"))]
    spec = G.GridSpec(400, 400, 0.1)
    jobs = _jobs(betas, ng, H, seed=sum(map(ord, name)))
    a, fa = _run(jobs, tabs, n, T, spec, exact=False)
    b, fb = _run(jobs, tabs, n, T, spec, exact=True)
    assert fb == H * n * T  # exact-only: every particle-step takes numpy's exp
    assert torch.equal(a["hyp"], b["hyp"])
    assert torch.equal(a["xy"].view(torch.int32), b["xy"].view(torch.int32))
    assert torch.equal(a["counts"], b["counts"])
    rate = fa / (H * n * T)
    print(f"{name}: filter fallback rate {rate:.4%} ({fa} of {H * n * T} particle-steps)")
    assert rate < max_rate


def test_filter_uniforms_mode_matches_exact():
    """GC_RNG_UNIFORMS (caller-supplied draws) takes the filter too: a near-uniform policy
    batch with arbitrary uniforms gives the same counts and positions on both paths."""
    cs = G.ControlSet.grid(4, 24, 1.4)
    q = G.q_goal_progress(0.5)
    tabs = [PR.action_tables(cs, q, 0.1, torch.device("cuda"))]
    spec = G.GridSpec(400, 400, 0.1)
    jobs = _jobs((0.01, 0.05), 2, 2, seed=5)
    n, T = 100000, 8
    u = torch.rand((2, T, n), generator=torch.Generator().manual_seed(3)).to("cuda", torch.float32)
    hu = torch.rand((2, n), generator=torch.Generator().manual_seed(4), dtype=torch.float64).to("cuda")
    outs = []
    for exact in (False, True):
        o = PR.run_predict(jobs, tabs, n, T, 0.1, 0.0, spec, "reference", per_human_layers=False, uniforms=u,
                           hyp_u=hu, want_hyp=True, want_xy=True, ref_exact_only=exact)
        outs.append(o)
    assert torch.equal(outs[0]["counts"], outs[1]["counts"])
    assert torch.equal(outs[0]["xy"].view(torch.int32), outs[1]["xy"].view(torch.int32))


def test_filter_error_budget_holds_on_this_gpu(tmp_path):
    """The filter's proof assumes |ex2.approx(fl(x log2e)) - e^x| <= 3e-7 e^x + 1e-9 for every
    float32 x in [-104, 0]: checked exhaustively on this GPU (tools/cuda_checks/ex2_filter_err.cu)."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "ex2_filter_err")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "--fmad=false", "-I",
                    os.path.join(root, "paper_2603_01122_b200", "csrc"),
                    os.path.join(root, "tools", "cuda_checks", "ex2_filter_err.cu"), "-o", exe],
                   check=True, capture_output=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "violations 0" in out.stdout, out.stdout + out.stderr


def test_filter_numpy_exp_error_bound():
    """... and that numpy's float32 exp (which the device exp_np reproduces bit for bit,
    test_gpu_exp_packed.py) is within 2.2e-7 relative of e^x on every float32 in [-104, 0]
    with a normal result (subnormal results: absolute error < 1e-44): EPS_W = 6e-7 >= 3e-7 +
    2.2e-7 in gc_predict.cu."""
    lo, hi = 0x80000000, 0xC2D00000
    worst_rel, worst_abs = 0.0, 0.0
    step = 1 << 25
    for s in range(lo, hi + 1, step):
        x = np.arange(s, min(s + step, hi + 1), dtype=np.uint64).astype(np.uint32).view(np.float32)
        y = np.exp(x).astype(np.float64)
        t = np.exp(x.astype(np.float64))
        err = np.abs(y - t)
        normal = t > 1.2e-38
        worst_rel = max(worst_rel, float((err[normal] / t[normal]).max(initial=0.0)))
        worst_abs = max(worst_abs, float(err[~normal].max(initial=0.0)))
    assert worst_rel <= 2.2e-7, worst_rel
    assert worst_abs < 1e-44, worst_abs
