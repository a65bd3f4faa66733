/*
 * gridcast_b200 -- C ABI of the B200-native particle predictor (sm_100a).
 *
 * Drop-in boundary for the reference package `gridcast` (arXiv 2603.01122).  The
 * reference has no FFI (it is pure Python/NumPy); its GPU seam is the contract of
 * SPEC.md:273-281 ("GPU backends can be added behind the same contract": chunk-keyed
 * counter RNG, disjoint outputs, bitwise determinism for any worker count).  Each entry
 * point below replaces one reference function; the Python host mirror
 * (paper_2603_01122_b200/) binds them with ctypes under the reference's own names.
 *
 * Conventions
 *   - every pointer named d_* is DEVICE memory owned by the caller; h_* is host memory;
 *   - every call is stream-ordered on `stream` (a cudaStream_t, passed as void*) and does
 *     not synchronise unless documented;
 *   - no torch / numpy types cross this boundary: plain pointers, sizes, PODs;
 *   - errors: a gc_status is returned and gc_last_error() holds a message (thread-local).
 */
#ifndef GRIDCAST_B200_H
#define GRIDCAST_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GC_ABI_VERSION 3

typedef enum {
    GC_OK = 0,
    GC_BAD_ARG = 1,            /* ValueError */
    GC_EMPTY_CONTROL_SET = 2,  /* agents.EmptyControlSetError (agents.py:20-21) */
    GC_SNAP_MISMATCH = 3,      /* belief.ControlSnapMismatch (belief.py:35-36) */
    GC_UNSUPPORTED_Q = 4,      /* utility family the kernels do not implement */
    GC_CUDA_ERROR = 5,         /* RuntimeError */
    GC_WINDOW_OVERFLOW = 6     /* a particle left its reachable-cell window (internal bug) */
} gc_status;

/* Bits of gc_predict's device status word d_error (raised by the kernel, stream-ordered;
 * the Python mirror reads it after the launch and raises RuntimeError / ValueError):
 *   WINDOW_OVERFLOW  a particle left its reachable-cell window (internal bug);
 *   HYPOTHESES       a human with d_hyp_off[h+1] - d_hyp_off[h] outside 1..GC_MAX_HYPOTHESES
 *                    (its CTAs return without counting anything);
 *   WINDOW_CAPACITY  max_win_cells under-reports the windows of the launch's steps (the
 *                    shared-memory window would not fit; the launch counts nothing);
 *   TABLE_ID         a human's d_table_id outside 0..n_tables-1 (its CTAs return);
 *   ASSUME_QG        assume_qg was set but a human's hypotheses need the general sampler
 *                    (that human's counts are not valid). */
#define GC_ERRBIT_WINDOW_OVERFLOW (1u << 6)
#define GC_ERRBIT_HYPOTHESES (1u << 8)
#define GC_ERRBIT_WINDOW_CAPACITY (1u << 9)
#define GC_ERRBIT_TABLE_ID (1u << 10)
#define GC_ERRBIT_ASSUME_QG (1u << 11)

/* Size limits of the kernels (shared-memory tables): hypotheses per human (|B| x |G|)
 * and actions per control set.  gc_belief_update marks a human outside 1..GC_MAX_HYPOTHESES
 * with GC_BAD_ARG in d_status; gc_predict raises GC_ERRBIT_HYPOTHESES. */
#define GC_MAX_HYPOTHESES 256
/* smoothing radius ceil(3 sigma / res) in cells (gc_grid_epilogue, gc_smooth_layers) */
#define GC_MAX_SMOOTH_RADIUS 56
#define GC_MAX_ACTIONS 512

/* Utility families (agents.py:245-296).  *_FULL = the reference's `base` (with the
 * row-constant -|rel|^2), used when a stationary mask dropped base_policy (belief.py:222). */
enum { GC_Q_GOAL_PROGRESS = 0, GC_Q_GOAL_PROGRESS_FULL = 1, GC_Q_DEFAULT = 2, GC_Q_TABLE = 3 };

/* Random-number modes of gc_predict.
 *   GC_RNG_REFERENCE : regenerate the reference's own numpy Philox4x64-10 streams
 *                      in-register (rng.py:27-31, prediction.py:128-131, :190-192) and run
 *                      the float32 per-action step op-for-op (prediction.py:147-162)
 *                      -> counts bit-identical to the reference;
 *   GC_RNG_UNIFORMS  : same arithmetic, uniforms supplied by the caller (d_uniforms,
 *                      d_hyp_u) e.g. drawn by the reference itself;
 *   GC_RNG_PRODUCTION: Philox4x32-10 in-register + exact-in-distribution factorised
 *                      sampler (one exp per heading) -- the fast path. */
enum { GC_RNG_REFERENCE = 0, GC_RNG_UNIFORMS = 1, GC_RNG_PRODUCTION = 2 };

/* Per-action table of one control set + utility (prediction.py:134-144, agents.py:275-294).
 * All arrays have length m (the FULL control set); keep lists the unmasked indices. */
typedef struct {
    int32_t m;
    int32_t m_keep;
    int32_t q_kind;            /* GC_Q_* */
    /* reference modes: R > 0 when the kept actions are the first R speed rows of a
     * ControlSet.grid-shaped set (action a*24 + b = speed row a, heading -pi + b pi/12) and
     * the heading weight is 0: K2 then guesses the max logit from the headings bracketing
     * the goal direction (verified against the full max, so any value is safe); 0 = none */
    int32_t ref_grid_rows;
    const float *d_sx, *d_sy;  /* float32 step_x*tau, step_y*tau (agents.py:279-280) */
    const float *d_at;         /* float32 action term incl. weights (agents.py:284-287) */
    const float *d_pen;        /* float32 q_default penalty (agents.py:256) */
    const float *d_dispx, *d_dispy; /* float32 displacements (agents.py:108-112 -> f32) */
    const int32_t *d_keep;     /* (m_keep,) */
    /* production factorised sampler (valid when n_speeds > 0): action (a, b) with
     * a in [0, n_speeds), b in [0, n_headings) has index a_index[a*n_headings+b] in the
     * full set, speed a*dv and heading theta_b. */
    int32_t n_speeds, n_headings;
    float dv, tau, w_v, w_th;
    const float *d_cos_h, *d_sin_h, *d_theta_h; /* (n_headings,) */
    const int32_t *d_a_index;                   /* (n_speeds*n_headings,) or NULL */
    /* optional HOST copies of the heading tables: when set, gc_predict never reads the
     * device copies back, so the call is CUDA-graph capturable */
    const float *h_cos_h, *h_sin_h, *h_theta_h;
} gc_action_table;

/* Batched Alg. 1 (prediction.py:223-255, sim.py:489-499): every human h of the batch
 * samples n hypotheses from its belief and propagates n particles for `steps` steps;
 * per-step particle counts land in that human's windowed count buffer. */
typedef struct {
    int32_t n_humans;
    int32_t n;                 /* particles per human */
    int32_t steps;             /* horizon T */
    int32_t rng_mode;          /* GC_RNG_* */
    int32_t grid_w, grid_h;
    float origin_x32, origin_y32, res32; /* GridSpec pre-cast to float32 (NEP 50) */
    const float *d_start_xy;   /* (n_humans, 2) float32 start positions */
    /* hypotheses: human h owns rows [d_hyp_off[h], d_hyp_off[h+1]) */
    const int32_t *d_hyp_off;
    const float *d_beta32;     /* (sum |H|,) */
    const float *d_goal32;     /* (sum |H|, 2) */
    const double *d_cdf;       /* (sum |H|,) host-built cdf (prediction.py:128-129) or NULL */
    const double *d_log_w;     /* (sum |H|,) device posterior, used when d_cdf == NULL */
    /* reference RNG: seed + path prefix per human (rng.stream(seed, *prefix, ...)) */
    const uint64_t *d_seed;    /* (n_humans,) */
    const uint32_t *d_prefix;  /* (n_humans, 4) */
    const int32_t *d_prefix_len; /* (n_humans,) 0..4 */
    /* production RNG: per-human stream id (the human's GLOBAL index, so a scene sharded
     * over GPUs draws the same numbers for any partition); NULL = batch index */
    const uint32_t *d_stream_id;
    /* GC_RNG_UNIFORMS inputs */
    const float *d_uniforms;   /* (n_humans, steps, n) float32 or NULL */
    const double *d_hyp_u;     /* (n_humans, n) float64 or NULL */
    const int32_t *d_hyp_in;   /* (n_humans, n) explicit hypothesis indices or NULL */
    /* action tables: human h uses tables[d_table_id[h]] */
    const gc_action_table *h_tables; /* host array of n_tables */
    int32_t n_tables;
    const int32_t *d_table_id; /* (n_humans,) */
    /* Reachable-cell windows.  Step t (0-based) of human h covers the cells within
     * d_step_r[t] of the human's start cell (clamped to the grid); its counts live at
     * d_counts + h*human_stride + d_step_off[t], row-major with row length
     * (clamped) window width.  Counts must be zero on entry. */
    const int32_t *d_step_r;   /* (steps,) */
    const int64_t *d_step_off; /* (steps,) */
    int64_t human_stride;
    int32_t max_win_cells;     /* max (2 r_t + 1)^2 over the steps of this launch [t_begin, t_end):
                                  sizes the GC_HIST_SMEM window (too small -> GC_ERRBIT_WINDOW_CAPACITY) */
    int32_t _pad2;
    uint32_t *d_counts;
    /* optional outputs */
    int32_t *d_hyp_out;        /* (n_humans, n) sampled hypothesis indices or NULL */
    float *d_xy_out;           /* (n_humans, n, 2) final positions or NULL */
    uint32_t *d_error;         /* device status word (GC_ERRBIT_* bits, OR-ed) or NULL */
    /* horizon chunking: run steps [t_begin, t_end) (1-based; 0, 0 = the whole horizon).
     * A chunk starting after step 1 resumes the particles saved by the previous chunk in
     * d_state_xy (float2 per particle) / d_state_hyp (uint8 hypothesis index); chunk
     * starts must satisfy (t_begin - 1) % 4 == 0 (the production streams' lane-turn phase). */
    int32_t t_begin, t_end;
    float *d_state_xy;
    uint8_t *d_state_hyp;
    /* particle-block sharding of one human over GPUs: this call runs particles
     * [p_offset, p_offset + n) of each human (every random stream is keyed by the global
     * particle index, so the draws do not depend on the partition); the u32 count
     * windows of all shards sum (ncclReduce/AllReduce sum) to the single-GPU counts and
     * the epilogue then divides by the total particle count. */
    int32_t p_offset;
    /* per-step histogram: GC_HIST_GLOBAL (0, default) adds every particle to its count
     * window in global memory, the lanes of a warp that hit the same cell combined into one
     * reduction (__match_any_sync); GC_HIST_SMEM (1) privatises the window in shared memory
     * (u16 counters, first-toucher flush, two CTA barriers per step) when it fits in 64 KB.
     * Both give identical counts; the global form measured 3-5 % faster on every belief
     * shape tried and keeps its speed at long horizons whose windows exceed shared memory. */
    int32_t hist_path;
    /* reference RNG modes (GC_RNG_REFERENCE / GC_RNG_UNIFORMS): each particle-step first
     * evaluates the action weights with the hardware ex2 and accepts the pick only when the
     * uniform lies outside a proven error margin around the bracketing cdf entries (then the
     * reference's numpy-exp pick is the same); otherwise it runs numpy's exp.  The results
     * are bit-identical either way.  ref_exact_only = 1 always runs numpy's exp (A/B). */
    int32_t ref_exact_only;
    /* optional (1,) counter: reference-mode particle-steps that took the numpy-exp path */
    uint64_t *d_ref_fallbacks;
    /* production factorised sampler: 1 = the caller guarantees that every hypothesis of the
     * launch admits the top-speed speed-weight normalisation (beta (tau^2 + w_v) dv^2 log2(e)
     * well below 10; the Python mirror sets it from the hypothesis spaces), so the kernel
     * omits the max-shift fallback (2.8 % of K2 at cfg3).  Checked per CTA: a human that
     * does not satisfy it raises GC_ERRBIT_ASSUME_QG (its counts are then not valid; the
     * Python mirror raises).  0 = general. */
    int32_t assume_qg;
    int32_t _pad3;
} gc_predict_args;

enum { GC_HIST_GLOBAL = 0, GC_HIST_SMEM = 1 };

/* Occupancy epilogue (prediction.py:251-254, occupancy.py:139-154, :162-192,
 * sim.py:500-504): windowed counts -> counts/n -> truncated-Gaussian smoothing with
 * edge-normalised columns -> per-human layers and/or the cell-wise max union. */
typedef struct {
    int32_t n_humans, n, steps;
    int32_t grid_w, grid_h;
    int32_t radius;            /* ceil(3 sigma_cells); 0 = no smoothing */
    const double *d_kernel;    /* (2*radius+1,) exp(-0.5 (o/sigma_cells)^2) */
    const double *d_zx;        /* (grid_w,) 1 / in-grid kernel mass per source column */
    const double *d_zy;        /* (grid_h,) 1 / in-grid kernel mass per source row */
    float origin_x32, origin_y32, res32;
    int32_t n_tiles;           /* tiles per human (static geometry) */
    const float *d_start_xy;   /* (n_humans, 2) float32 start positions */
    const int32_t *d_step_r;
    const int64_t *d_step_off;
    int64_t human_stride;
    const int32_t *d_tiles;    /* (n_tiles, 4): t, tile_x, tile_y, 0 (32x32 output tiles
                                  over the window grown by radius) */
    const uint32_t *d_counts;
    double *d_layers64;        /* (n_humans, steps, H, W) zero-filled, or NULL */
    float *d_union32;          /* (steps, H, W) zero-filled max-union (float32) or NULL */
    double *d_union64;         /* (steps, H, W) zero-filled max-union (float64) or NULL */
    int32_t time_union;        /* running max over t of the union (sim.py:503-504) */
    int32_t tile_begin, tile_end; /* sub-range of d_tiles (0, 0 = all; tiles are ordered by step) */
    int32_t t_begin, t_end;    /* steps the time union covers (0-based, [t_begin, t_end); 0, 0 = all) */
    int32_t _pad_e;
    /* (steps, ceil(H/32), ceil(W/32)) zero-filled byte flags, or NULL: set to 1 for every
     * 32 x 32 union tile of a layer that receives a nonzero value (gc_publish_tiles ships
     * only those tiles to the host) */
    uint8_t *d_union_tile_flags;
} gc_epilogue_args;

/* Tile-sparse device -> host publication of a (steps, H, W) union into a pinned host stack
 * (the reference's PredictionStack layout, prediction.py:98-106) that lives across cycles:
 * for every 32 x 32 tile of layers [t_begin, t_end) the kernel writes the device tile into
 * the host stack when K3 flagged it nonzero this cycle, writes zeros where the host stack
 * still holds a tile of an earlier cycle that is zero now, and otherwise moves nothing, so
 * after the call the host stack equals the device union bit for bit.  The host stack must
 * be page-locked and mapped (any cudaHostAlloc / pinned allocation under unified
 * addressing) and start zero-filled with zeroed d_host_flags. */
typedef struct {
    int32_t steps, grid_w, grid_h;
    int32_t t_begin, t_end;            /* 0-based layer range [t_begin, t_end) */
    int32_t dtype_bytes;               /* 4 (float32) or 8 (float64) */
    int32_t time_or;                   /* 1: layer t's tile is live if any layer <= t flagged it (time union) */
    int32_t _pad;
    const void *d_union;               /* (steps, H, W) device union */
    const uint8_t *d_tile_flags;       /* this cycle's K3 flags (gc_epilogue_args.d_union_tile_flags) */
    uint8_t *d_host_flags;             /* (steps, ceil(H/32), ceil(W/32)) tiles of the host stack holding nonzeros */
    void *h_dst;                       /* (steps, H, W) pinned, mapped host stack */
} gc_publish_args;

/* Observation update of every human's joint belief (belief.py:159-198), one warp per
 * human: recover_control (agents.py:355-371) -> snap (agents.py:114-120) -> log-policy
 * (agents.py:299-323) -> prior + loglik, floor -745, -inf kept -> logsumexp normalise. */
typedef struct {
    int32_t n_humans;
    int32_t m;
    const double *d_v, *d_theta;      /* (m,) control set rows */
    const double *d_sx, *d_sy, *d_at; /* (m,) float64 goal-progress tables */
    const double *d_pen;              /* (m,) float64 q_default penalty */
    const uint8_t *d_masked;          /* (m,) 1 = masked, or NULL */
    int32_t q_kind;                   /* GC_Q_GOAL_PROGRESS(_FULL) / GC_Q_DEFAULT / GC_Q_TABLE */
    const double *d_qtable;           /* GC_Q_TABLE: (sum |H|, m) q.table at z_t per human */
    const int32_t *d_hyp_off;         /* (n_humans+1,) */
    const double *d_beta, *d_goal;    /* (sum |H|,), (sum |H|, 2) float64 */
    const double *d_obs;              /* (n_humans, 4): z_t.x, z_t.y, z_next.x, z_next.y */
    const double *d_fallback_theta;   /* (n_humans,) */
    double dt;
    double snap_tol;                  /* +inf disables ControlSnapMismatch */
    int32_t clamp_on_mismatch;        /* 1: update with the nearest action anyway (sim.py:469-478) */
    const double *d_prior;            /* (sum |H|,) log weights */
    double *d_post;                   /* (sum |H|,) log weights (may alias d_prior) */
    int32_t *d_status;                /* (n_humans,) GC_OK / GC_SNAP_MISMATCH / GC_EMPTY_CONTROL_SET /
                                         GC_BAD_ARG (0 or > GC_MAX_HYPOTHESES hypotheses) */
    int32_t *d_action;                /* (n_humans,) snapped action index or NULL */
} gc_belief_args;

/* Exact enumeration of the bootstrapped process (prediction.py:303-377): per-hypothesis
 * cell distributions propagated through the cell-centre transition tables, layers =
 * belief-weighted mixtures.  float64 throughout; workspaces are caller-allocated:
 * d_pi (n_hyp*cells*m), d_landing (cells*m int32), d_p, d_nxt (n_hyp*cells), d_pi0
 * (n_hyp*m); d_layers (steps, H, W). */
typedef struct {
    int32_t n_hyp, m, grid_w, grid_h, steps, q_kind;
    double origin_x, origin_y, res, z0x, z0y;
    const double *d_beta, *d_goal, *d_belief;   /* (|H|), (|H|, 2), (|H|) probabilities */
    const double *d_sx, *d_sy, *d_at, *d_pen;   /* (m) float64 utility tables */
    const double *d_dispx, *d_dispy;            /* (m) float64 displacements */
    const uint8_t *d_masked;                    /* (m) or NULL */
    const double *d_qtable, *d_qtable0;         /* GC_Q_TABLE: (|H|, cells, m), (|H|, m) */
    double *d_pi, *d_p, *d_nxt, *d_pi0;
    int32_t *d_landing;
    double *d_layers;
} gc_exact_args;

/* predict_naive (prediction.py:258-300): the reference's serial float64 per-particle loop,
 * one thread per particle.  Positions start at (start_x, start_y) in float64; per step
 * the particle's q.table row over the kept actions (GC_Q_GOAL_PROGRESS_FULL or
 * GC_Q_DEFAULT; float64 tables as q.table evaluates them, agents.py:222-224), beta x,
 * max shift, exp, sequential cumsum, #(cdf < u * cdf[-1]) with u the float64 draw of
 * rng.stream(seed, *prefix, 1, t, p >> 10) (rng.py:27-39); cells in float64
 * (occupancy.py:43-51).  d_counts = (steps, H, W) uint32, zeroed by the caller. */
typedef struct {
    int32_t n, steps, n_hyp, m_keep;
    int32_t q_kind, grid_w, grid_h, prefix_len;
    uint64_t seed;
    uint32_t prefix[4];
    double start_x, start_y, origin_x, origin_y, res;
    const int32_t *d_hyp;                       /* (n) hypothesis of each particle */
    const double *d_beta, *d_goal;              /* (|H|), (|H|, 2) */
    const int32_t *d_keep;                      /* (m_keep) kept action indices, ascending */
    const double *d_sx, *d_sy, *d_at, *d_pen;   /* (m) float64 utility tables */
    const double *d_dispx, *d_dispy;            /* (m) float64 displacements */
    uint32_t *d_counts;                         /* (steps, H, W) */
    double *d_xy_out;                           /* (n, 2) final positions or NULL */
} gc_naive_args;

/* MPPI control update (planners/mppi.py:149-243) against a device blocked mask. */
typedef struct {
    int32_t n_rollouts, horizon;
    double dt, temperature, std_a, std_w;
    double q[4], qf[4], r[2];
    double collision_penalty;
    int32_t quadratic_control_cost;
    double a_max, omega_max, v_max;
    double z[4], goal[4];                 /* robot state and goal (x, y, v, theta) */
    const double *d_nominal;              /* (K, 2) */
    const double *d_noise;                /* (N, K, 2) perturbations (already x std), or NULL */
    uint64_t seed;                        /* production noise (Philox4x32-10 + Box-Muller) */
    const uint8_t *d_blocked;             /* (L, H, W) or NULL */
    int32_t n_layers, grid_w, grid_h;
    double origin_x, origin_y, res;
    const int32_t *d_layer_of;            /* (K) blocked layer per horizon step */
    double *d_noise_out;                  /* (N, K, 2) generated noise (when d_noise == NULL) */
    double *d_costs, *d_controls, *d_weights, *d_diag; /* (N), (K, 2), (N), (3) */
} gc_mppi_args;

gc_status gc_predict(const gc_predict_args *args, void *stream);
gc_status gc_mppi_step(const gc_mppi_args *args, void *stream);
gc_status gc_exact_predict(const gc_exact_args *args, void *stream);
gc_status gc_predict_naive(const gc_naive_args *args, void *stream);

/* Cell-wise union of k stacked layer sets (occupancy.py:162-192), in the reference's
 * order and float64 arithmetic: input i starts at element i * stride of d_in and has
 * `cells` elements (float32 when in_bytes == 4, float64 when 8); d_out has `cells`.
 * GC_UNION_MAX: max_i p_i; GC_UNION_INDEPENDENT: 1 - prod_i (1 - clip(p_i, 0, 1));
 * GC_UNION_MISS: prod_i (1 - clip(p_i, 0, 1)) (a partial for a cross-GPU product
 * reduction); GC_UNION_COMPLEMENT: 1 - p_0 (finishes a reduced MISS). */
enum { GC_UNION_MAX = 0, GC_UNION_INDEPENDENT = 1, GC_UNION_MISS = 2, GC_UNION_COMPLEMENT = 3 };
gc_status gc_union_layers(const void *d_in, int32_t in_bytes, int32_t k, int64_t stride, int64_t cells,
                          int32_t mode, void *d_out, int32_t out_bytes, void *stream);

/* Conservative time union (sim.py:503-504, np.maximum.accumulate over layers) of layers
 * [t_begin, t_end) of a (T, H, W) stack, seeded by layer t_begin - 1 when t_begin > 0. */
gc_status gc_time_union(void *d_union, int32_t dtype_bytes, int32_t t_begin, int32_t t_end, int64_t cells,
                        void *stream);
gc_status gc_grid_epilogue(const gc_epilogue_args *args, void *stream);
gc_status gc_publish_tiles(const gc_publish_args *args, void *stream);

/* Sparse form of the cross-GPU max-union (the fused grid of sim.py:500-502 over ranks):
 * gathers (unpack = 0) the listed 32 x 32 tiles of a (steps, H, W) union into d_packed
 * (count, 32, 32) -- zeros outside the grid -- or scatters (unpack = 1) them back, in-grid
 * cells only.  Tile id (t * ceil(H/32) + ty) * ceil(W/32) + tx, the layout of the union-tile
 * flags; every rank packs the same ids (the OR of the ranks' flags), so an ncclReduce(max) of
 * the packed buffers equals the dense reduce on those tiles, and every other tile is zero
 * on every rank. */
gc_status gc_union_tiles(void *d_union, int32_t dtype_bytes, int32_t steps, int32_t grid_w, int32_t grid_h,
                         const int32_t *d_tile_ids, int32_t count, void *d_packed, int32_t unpack, void *stream);
gc_status gc_belief_update(const gc_belief_args *args, void *stream);

/* One propagate_step (prediction.py:165-211) of an explicit particle batch in reference
 * arithmetic: d_xy (n,2) f32 in/out, d_hyp (n,), hypothesis tables of ONE human,
 * uniforms either supplied (d_u01, n) or regenerated from (seed, prefix, step). */
gc_status gc_propagate_step(float *d_xy, const int32_t *d_hyp, int32_t n,
                            const float *d_beta32, const float *d_goal32, int32_t n_hyp,
                            const gc_action_table *h_table, const float *d_u01,
                            uint64_t seed, const uint32_t *h_prefix, int32_t prefix_len,
                            int32_t step, void *stream);

/* sample_hypotheses (prediction.py:124-131) with the reference stream: d_out (n,) int32. */
gc_status gc_sample_hypotheses(const double *d_cdf, int32_t n_hyp, int32_t n, uint64_t seed,
                               const uint32_t *h_prefix, int32_t prefix_len, int32_t *d_out,
                               void *stream);

/* emplace_counts (occupancy.py:105-109): accumulate d_xy (n,2) float32 particles into
 * d_counts (H*W) uint32, float32 cell arithmetic + edge clamping (occupancy.py:43-51). */
gc_status gc_emplace_counts(const float *d_xy, int64_t n, int32_t grid_w, int32_t grid_h,
                            float origin_x32, float origin_y32, float res32, uint32_t *d_counts,
                            void *stream);

/* smooth_values (occupancy.py:139-154) on n_layers float64 (H, W) layers, d_in != d_out;
 * d_zx / d_zy hold the reciprocal in-grid kernel masses (column normalisation). */
gc_status gc_smooth_layers(const double *d_in, double *d_out, int32_t n_layers, int32_t grid_w,
                           int32_t grid_h, int32_t radius, const double *d_kernel,
                           const double *d_zx, const double *d_zy, void *stream);

/* collision_field (occupancy.py:222-239) of n_layers (H, W) occupancy layers (float32 when
 * dtype_bytes == 4, float64 when 8): the clamped-to-1 mass within the robot disc of each
 * cell centre, h_offsets = (n_offsets, 2) int32 (dx, dy) disc offsets in the reference's
 * order (occupancy.py:208-215, at most 33x33); outputs: d_field float64 and/or d_blocked
 * uint8 = field >= threshold (planners/anastar.py:107-119). Bit-identical float64 sums. */
gc_status gc_collision_field(const void *d_layers, int32_t dtype_bytes, int32_t n_layers,
                             int32_t grid_w, int32_t grid_h, const int32_t *h_offsets,
                             int32_t n_offsets, double threshold, double *d_field,
                             uint8_t *d_blocked, void *stream);

/* Peer-memory fused union (multi-GPU form of the union in sim.py:500-502 /
 * occupancy.py:162-192): the owning rank allocates the (T, H, W) union as a whole device
 * allocation (gc_peer_alloc) and exports a CUDA IPC handle; every other rank of the node
 * imports it (NVLink peer mapping) and passes the mapped pointer as the epilogue's
 * d_union32 / d_union64, so its K3 atomicMax-es into the owner's grid directly (exact,
 * order-independent).  Replaces the per-cycle NCCL max-reduce of dense grids
 * (engine.fused_reduce) by the sparse K3 writes themselves. */
#define GC_PEER_HANDLE_BYTES 64
gc_status gc_peer_alloc(int64_t bytes, void **d_out);
gc_status gc_peer_free(void *d);
gc_status gc_peer_export(const void *d, uint8_t *h_handle);      /* h_handle: 64 bytes */
gc_status gc_peer_import(const uint8_t *h_handle, void **d_out);
gc_status gc_peer_close(void *d);

/* rng.derive_seed (rng.py:34-39): SeedSequence(seed, path).generate_state(2,u64) xor-folded. */
uint64_t gc_derive_seed(uint64_t seed, const uint32_t *h_path, int32_t path_len);

/* Fill h_out[0..n) with rng.stream(seed, *path).random(n, float32) (host, for tests/tools). */
void gc_stream_f32(uint64_t seed, const uint32_t *h_path, int32_t path_len, float *h_out, int64_t n);

const char *gc_last_error(void);
int32_t gc_abi_version(void);
/* Number of kernel launches issued through this library since load (for bench claims). */
uint64_t gc_launch_count(void);
/* cudaMemsetAsync(d_ptr, 0, bytes, stream): the engine's per-cycle output / count fills. */
gc_status gc_fill_zero(void *d_ptr, int64_t bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GRIDCAST_B200_H */
