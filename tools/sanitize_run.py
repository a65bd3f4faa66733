"""Every kernel of libgridcast_b200.so once, at small sizes, for compute-sanitizer
(race detection / memory checking of the hot path):

    compute-sanitizer --tool memcheck  python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py
    compute-sanitizer --tool synccheck python tools/sanitize_run.py

Covers K2 in every mode (reference arithmetic, production factorised standard / weighted
headings / generic sampler, shared-window and global-histogram paths, chunked horizon),
K3 (smoothing, max union, time union), K1, the independent union, collision field, MPPI,
exact enumeration, predict_naive, propagate_step, sample_hypotheses, emplace and smooth.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_01122_b200 as G  # noqa: E402
from paper_2603_01122_b200 import planners as PL  # noqa: E402
from paper_2603_01122_b200.engine import CycleEngine, EngineConfig  # noqa: E402
from paper_2603_01122_b200.scenario import make_scene  # noqa: E402


def main():
    cs = G.ControlSet.grid(4, 24, 1.4)
    q = G.q_goal_progress(0.5)
    space = G.HypothesisSpace(G.RationalitySet.log_spaced(5), G.GoalSet(np.array([[8.5, 5.0], [1.5, 7.0]])))
    spec = G.GridSpec(100, 100, 0.1)
    z0, z1 = G.HumanState(5.0, 5.0), G.HumanState(5.1, 5.02)
    b = G.update_belief(G.init_belief(space), z0, z1, 0.1, cs, q, space)                      # K1
    for mode in ("reference", "production"):
        cfg = G.PredictionConfig(n=1536, steps=8, dt=0.1, smoothing_sigma=0.1, seed=3, mode=mode)
        G.predict(z1, b, cfg, cs, q, space, spec)                                                # K2 + K3
        G.predict(z1, b, cfg, cs, G.q_goal_progress(0.4, (0.3, 0.2)), space, spec)              # weighted
        G.predict(z1, b, cfg, cs, G.q_default((0.3, 2.0)), space, spec)                         # generic
        G.predict(z1, b, cfg, cs, G.mask_stationary(q, cs, 0.5), space, spec)                   # masked
    # 1 cm cells: the reachable window outgrows shared memory -> global-histogram path
    fine = G.GridSpec(300, 300, 0.01)
    for mode in ("reference", "production"):
        G.predict_multi([(G.HumanState(1.5, 1.5), b), (G.HumanState(1.0, 2.0), b)],
                        G.PredictionConfig(n=1024, steps=8, dt=0.1, smoothing_sigma=0.0, seed=1, mode=mode),
                        cs, q, space, fine)
    # engine: chunked horizon, time union, blocked mask, two humans
    sc = make_scene("cfg2", cycles=3, humans=2)
    eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec,
                      EngineConfig(n=2048, steps=16, dt=sc.dt, mode="production", time_union=True, robot_radius=0.25))
    eng.prime(sc.warmup_track[0])
    eng.stage(sc.warmup_track[1], buf=0)
    eng.run_cycle(buf=0, chunks=3)
    # tile-sparse publication into a pinned host stack, and the sparse-reduce gather/scatter
    host = torch.zeros(eng.unions[0].shape, dtype=eng.unions[0].dtype).pin_memory()
    eng_p = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec,
                        EngineConfig(n=2048, steps=16, dt=sc.dt, mode="production"))
    eng_p.prime(sc.warmup_track[0])
    eng_p.stage(sc.warmup_track[1], buf=0)
    eng_p.run_cycle(buf=0, chunks=2, d2h=host, copy_stream=torch.cuda.Stream())
    from paper_2603_01122_b200.engine import union_tiles
    ids = torch.nonzero(eng_p.utile[0].reshape(-1)).reshape(-1).to(torch.int32)
    packed = torch.empty((len(ids), 32, 32), dtype=eng_p.unions[0].dtype, device="cuda")
    union_tiles(eng_p.unions[0], ids, packed, unpack=False)
    union_tiles(eng_p.unions[0], ids, packed, unpack=True)
    eng_i = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec,
                        EngineConfig(n=1024, steps=8, dt=sc.dt, mode="reference", union_mode="independent"))
    eng_i.prime(sc.warmup_track[0])
    eng_i.stage(sc.warmup_track[1], buf=0)
    eng_i.run_cycle(buf=0)
    torch.cuda.synchronize()
    # standalone entry points
    hyp = G.sample_hypotheses(b, 3000, seed=2)
    batch = G.ParticleBatch(np.tile(np.array([[5.0, 5.0]], dtype=np.float32), (3000, 1)), hyp)
    batch = G.propagate_step(batch, cs, q, space, 0.1, seed=2, step=1)
    G.emplace_counts(batch.xy, spec)
    G.smooth_values(np.random.default_rng(0).random((100, 100)), spec, 0.15)
    G.predict_naive(z1, b, G.PredictionConfig(n=256, steps=4, dt=0.1, smoothing_sigma=0.1, seed=4), cs, q, space,
                    spec)
    G.exact_predict(G.HumanState(4.5, 4.5), b, 2, 1.0, cs, q, space, G.GridSpec(10, 10, 1.0))
    st = G.predict(z1, b, G.PredictionConfig(n=1024, steps=10, dt=0.1, seed=5, mode="production"), cs, q, space,
                   spec)
    grids = [G.OccupancyGrid(spec, st.layers[k]) for k in range(2)]
    G.union(grids, mode="independent")
    G.collision_field(grids[0], 0.25)
    mcfg = PL.MppiConfig(horizon=10, rollouts=256, dt=0.1, seed=3)
    PL.mppi_step(PL.RobotState(1.0, 2.0, 0.4, 0.3), np.zeros((10, 2)), PL.RobotState(5.0, 2.2, 0.0, 0.0), st,
                 mcfg, noise="production")
    torch.cuda.synchronize()
    print("sanitize_run: all entry points ran")


if __name__ == "__main__":
    main()
