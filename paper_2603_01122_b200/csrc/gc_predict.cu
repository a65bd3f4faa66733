// gc_predict.cu -- K2: register-resident particle propagation fused with the per-step
// occupancy histogram (Alg. 1 of arXiv 2603.01122; reference prediction.py:223-255).
//
// One CTA = one contiguous block of one human's particles.  Each thread keeps K
// particles' (x, y, hypothesis) in registers for the WHOLE horizon; per step it samples
// an action per particle, Euler-steps, maps the particle to its cell and adds it (shared
// atomic on a u16 half-word) into a shared-memory privatised window covering the cells
// the human can reach by that step.  After a CTA barrier the touched cells (each
// remembered by the thread whose add found its word zero) are flushed with one global
// reduction each into the human's windowed count buffer, and zeroed.  HBM sees only those
// reductions.
//
// Two arithmetic families:
//   MODE_REF  : the reference float32 step op for op: per-action
//               logits, max shift, numpy exp (gc::exp_np), sequential cumsum, inverse CDF.
//               Uniforms regenerated in-register from the reference's numpy Philox4x64
//               streams (or read from a caller buffer) -> counts bit-identical.
//   MODE_FACT : production, exact in distribution for grid control sets with
//               goal-progress utility: weight(a,b) = H_b G_a e_b^a, one ex2 per heading.
//   MODE_GEN  : production generic per-action softmax (fast ex2) for any control set.
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>
#include "gc_common.cuh"
#include "gc_internal.h"

namespace gc {

constexpr int NT = 256;        // threads per CTA
constexpr int MAXM = GC_MAX_ACTIONS;  // max actions per control set (512)
constexpr int MAXH = 256;      // max hypotheses per human (the per-slot index is a byte)
constexpr int NBF = 24;        // headings of the factorised sampler (ControlSet.grid default)
constexpr int NAF = 4;         // max speeds of the factorised sampler

#ifndef GC_FFMA2
#define GC_FFMA2 1  // packed FP32x2 heading loop (sm_100 FFMA2)
#endif
#ifndef GC_PROD_MIN_CTAS
#define GC_PROD_MIN_CTAS 4  // resident CTAs per SM of the production K2 (64 registers)
#endif
#ifndef GC_REF_MIN_CTAS
#define GC_REF_MIN_CTAS 4  // resident CTAs per SM of the reference-arithmetic K2 (64 regs): after the specialised filter 9.24 ms (T = 100, cfg3) vs 9.58 at 2 and 9.67 at 3
#endif
#ifndef GC_GEN_MIN_CTAS
#define GC_GEN_MIN_CTAS 4  // resident CTAs per SM of the production generic-sampler K2
#endif
#ifndef GC_WORLD_CELLS
#define GC_WORLD_CELLS 1  // production particles in float32 world coordinates, exact cells
#endif

constexpr unsigned PHK0 = 0xA4093822u, PHK1 = 0x299F31D0u;  // production Philox key

// FACTS: standard headings; FACTS_QG: FACTS for a launch whose caller guarantees that every
// hypothesis admits the top-speed normalisation (gc_predict_args.assume_qg; checked per CTA)
enum { MODE_REF = 0, MODE_FACT = 1, MODE_GEN = 2, MODE_FACTS = 3, MODE_FACTS_QG = 4 };

struct KTable {
    int m, m_keep, q_kind, n_speeds, n_headings;
    int grid_rows;  // gc_action_table.ref_grid_rows
    float dv, tau, w_v, w_th;
    const float *sx, *sy, *at, *pen, *dispx, *dispy;
    const int *keep, *a_index;
};

struct KParams {
    int n_humans, n, steps, ppc, ctas_per_human, rng_mode;
    int grid_w, grid_h;
    float ox, oy, res, inv_res;
    float wm1f, hm1f;            // (float)(grid_w - 1), (float)(grid_h - 1)
    const float *start_xy;
    const int *hyp_off;
    const float *beta32, *goal32;
    const double *cdf, *log_w;
    const unsigned long long *seed;
    const unsigned *prefix;
    const int *prefix_len;
    const unsigned *stream_id;
    const float *uniforms;
    const double *hyp_u;
    const int *hyp_in;
    KTable tab[4];
    int n_tables;
    const int *table_id;
    const int *step_r;
    const long long *step_off;
    long long human_stride;
    unsigned *counts;
    int smem_window;
    int win_cap_words;  // u32 words the host allocated for the window (incl. the sink word)
    int act_off;  // byte offset of SmemAct in dynamic shared memory (REF/GEN modes)
    int ref_off;  // byte offset of SmemRefState (MODE_REF)
    int dyn_smem; // dynamic shared memory bytes of the launch (bounds checks)
    int t_begin, t_end;          // steps [t_begin, t_end) of this launch (1-based)
    int p_offset;                // global index of this launch's first particle (particle sharding)
    float2 *state_xy;            // particle state between horizon chunks
    unsigned char *state_hyp;
    int *hyp_out;
    float *xy_out;
    unsigned *error;
    int ref_filter;                        // MODE_REF: MUFU filter + exact fallback (ref_pick)
    unsigned long long *ref_fallbacks;     // MODE_REF: particle-steps resolved by the exact path, or NULL
    // headings shared by every table of a factorised launch (constant-bank operands)
    float hcos[NBF], hsin[NBF], hth2[NBF];
};

// cell of a float32 position exactly as GridSpec.cells_of (occupancy.py:43-51, NEP 50)
__device__ __forceinline__ void cell_ref(float x, float y, const KParams &P, int &ix, int &iy) {
    const float fx = floorf(__fdiv_rn(__fsub_rn(x, P.ox), P.res));
    const float fy = floorf(__fdiv_rn(__fsub_rn(y, P.oy), P.res));
    ix = fx < 0.f ? 0 : (fx > (float)(P.grid_w - 1) ? P.grid_w - 1 : (int)fx);
    iy = fy < 0.f ? 0 : (fy > (float)(P.grid_h - 1) ? P.grid_h - 1 : (int)fy);
}


// the reference's cell of a float32 world position, floor(fl(fl(x - ox) / res)) clamped
// (occupancy.py:43-51), without the IEEE division's slow path: q0 = fl(t * fl(1/res)) is
// within an ulp of t / res, and one fma-exact residual correction, q = fl(q0 + fl(t - q0 res)
// * fl(1/res)), is the correctly rounded quotient (Markstein; checked exhaustively against
// __fdiv_rn for the grid resolutions in tests/test_gpu_cell_exact.py).  Production
// particles keep the reference's float32 world coordinates (x += dispx[a]), so particles
// that follow the same actions land in the same cells as the reference's -- clusters that
// sit exactly on a cell edge included.
__device__ __forceinline__ int cell_exact1(float x, float o, float res, float yres, float nm1) {
    return floor_clamp(div_rn_recip(__fsub_rn(x, o), res, yres), nm1);
}

// yres = recip_nr(P.res), computed once per thread
__device__ __forceinline__ void cell_fast(float x, float y, const KParams &P, float yres, int &ix, int &iy) {
#if GC_WORLD_CELLS
    ix = cell_exact1(x, P.ox, P.res, yres, P.wm1f);
    iy = cell_exact1(y, P.oy, P.res, yres, P.hm1f);
#else
    ix = floor_clamp((x - P.ox) * P.inv_res, P.wm1f);
    iy = floor_clamp((y - P.oy) * P.inv_res, P.hm1f);
#endif
}

// MODE_REF / MODE_GEN: per-action rows compacted over keep (dynamic shared memory,
// after the window; absent from the production kernel)
struct alignas(16) SmemAct {
    float ax[MAXM], ay[MAXM], aat[MAXM], adx[MAXM], ady[MAXM];
    float4 axy[MAXM / 2];  // MODE_REF: (ax[2i], ax[2i+1], ay[2i], ay[2i+1]) -- one LDS.128 per action pair
};

// MODE_REF: per-slot particle state of the runtime slot loop (dynamic shared memory, after
// SmemAct)
struct alignas(16) SmemRefState {
    float2 pos[4 * 256];  // float32 world position of particle slot k*NT+tid
    int fwr[4 * 256];     // GC_HIST_SMEM: the window word slot k*NT+tid added to first, or -1
};

struct SmemTabs {
    // production: (goal x, goal y, k log2e, c log2e) per hypothesis -- one LDS.128;
    // MODE_FACTS: (goal x, goal y, k log2e, Ka) and hq = (Kb, Kc, c log2e, sum_b H_b)
    float4 hp[MAXH];
    float4 hq[MAXH];
    // production: displacement of (a, b) and heading (cos, sin) -- one LDS.64 each
    float2 fd[NAF * NBF];
    float2 hcs[NBF];
    // hypotheses of this CTA's human
    double cdf[MAXH];
    float hb[MAXH], hgx[MAXH], hgy[MAXH];
    int n_hyp, m_keep, q_kind, n_speeds;
    int ref_rows;  // MODE_REF: KTable.grid_rows of this CTA's table
    float gsmax, gatmin;  // MODE_GEN: max_k |(sx, sy)_k| and min_k at_k (or pen_k) of the kept actions
    float wth;
    unsigned char phyp[4 * 256];  // hypothesis index of particle slot k*NT+tid (frees registers)
};

// ---- reference float32 step (prediction.py:147-162), 3 passes, no stored row --------
__device__ __forceinline__ float ref_logit(const SmemAct &S, int k, float rx, float ry, float d2,
                                           float beta, int qk) {
    float L;
    if (qk == GC_Q_DEFAULT) {
        L = __fsub_rn(-d2, S.aat[k]);
    } else {
        L = __fmul_rn(__fmaf_rn(ry, S.ay[k], __fmul_rn(rx, S.ax[k])), -2.0f);
        L = __fsub_rn(L, S.aat[k]);
        if (qk == GC_Q_GOAL_PROGRESS_FULL) L = __fsub_rn(L, d2);
    }
    return __fmul_rn(L, beta);
}

// logits of the action pair (k, k + 1), k even (8-byte aligned rows): ref_logit per lane
__device__ __forceinline__ float2 ref_logit2(const SmemAct &S, int k, float rx, float ry, float d2, float beta,
                                             int qk) {
    const float2 at = *reinterpret_cast<const float2 *>(&S.aat[k]);
    float2 L;
    if (qk == GC_Q_DEFAULT) {
        L = px_add(px2(-d2), make_float2(-at.x, -at.y));  // -d2 - at
    } else {
        const float2 ax = *reinterpret_cast<const float2 *>(&S.ax[k]);
        const float2 ay = *reinterpret_cast<const float2 *>(&S.ay[k]);
        L = px_fma(px2(ry), ay, px_mul(px2(rx), ax));
        // (L * -2) - at: a contraction of this product into the add would be exact (the
        // product by -2 is exact), so the packed pair is safe here
        L = px_mul(L, px2(-2.0f));
        L = px_add(L, make_float2(-at.x, -at.y));
        if (qk == GC_Q_GOAL_PROGRESS_FULL) L = px_add(L, px2(-d2));
    }
    // beta * L feeds the subtraction of the max: scalar __fmul_rn, which ptxas never fuses
    return make_float2(__fmul_rn(L.x, beta), __fmul_rn(L.y, beta));
}

// Passes 2-3 of the reference step given the max logit M: numpy's exp per action, the
// sequential float32 cumsum, inverse CDF (prediction.py:152-160).  The running sum is
// remembered at the end of each of NBLK blocks of B actions -- values of the same chain,
// so the search is bit-identical to a scan from the first action but recomputes only the
// one block that holds r.  B is even so the action pairs stay 8-byte aligned; the sum
// itself stays sequential.  Not inlined: behind the filter (ref_pick) it runs for a small
// fraction of the particle-steps, and one copy serves the K unrolled particle slots.
static __device__ __noinline__ int ref_pick_exact(const SmemAct &S, float rx, float ry, float d2, float beta, int mk,
                                           int qk, float M, float u) {
    constexpr int NBLK = 12;
    const int B = 2 * ((mk + 2 * NBLK - 1) / (2 * NBLK));
    float blk[NBLK];
    float c = 0.f;
#pragma unroll
    for (int j = 0; j < NBLK; ++j) {
        const int k1 = min(mk, (j + 1) * B);
        int kk = j * B;
        for (; kk + 1 < k1; kk += 2) {
            const float2 L = ref_logit2(S, kk, rx, ry, d2, beta, qk);
            const float2 w = exp_np2(px_add(L, px2(-M)));
            c = (kk == 0) ? w.x : __fadd_rn(c, w.x);
            c = __fadd_rn(c, w.y);
        }
        if (kk < k1) {
            const float w = exp_np(__fsub_rn(ref_logit(S, kk, rx, ry, d2, beta, qk), M));
            c = (kk == 0) ? w : __fadd_rn(c, w);
        }
        blk[j] = c;
    }
    const float r = __fmul_rn(u, c);
    // first block whose running sum reaches r (all earlier cdf entries are < r)
    int jb = 0;
    float cc = 0.f;
#pragma unroll
    for (int j = 0; j < NBLK - 1; ++j) {
        if (blk[j] < r) { jb = j + 1; cc = blk[j]; }
    }
    int k = jb * B;
    const int kend = min(mk, (jb + 1) * B);
    for (; k < kend; ++k) {
        const float w = exp_np(__fsub_rn(ref_logit(S, k, rx, ry, d2, beta, qk), M));
        cc = (k == 0) ? w : __fadd_rn(cc, w);
        if (!(cc < r)) break;
    }
    if (k == kend && kend < mk) k = mk;  // cannot happen for a monotone chain: keep the clamp semantics
    return k < mk - 1 ? k : mk - 1;
}

// Error budget of the reference-mode filter (ref_pick).  With w_k = exp_np(x_k) the
// reference's weight and w~_k = ex2.approx.ftz(fl(x_k log2e)) the filter's (x_k = fl(L_k - M)
// <= 0 identical in both):
//   |w~_k - e^x_k| <= EPS_MUFU e^x_k + A_W   (tools/cuda_checks/ex2_filter_err.cu,
//                                            exhaustive over every float32 x in [-104, 0]:
//                                            EPS_MUFU = 3e-7 holds with an additive excess
//                                            of at most 3.7e-10)
//   |w_k - e^x_k|  <= EPS_NP e^x_k           (numpy's float32 exp, exhaustive on the CPU:
//                                            2.13e-7 max relative error, normal results)
// so |w~_k - w_k| <= EPS_W w_k + A_W.  A sequential float32 sum is within 2^-24 sum_{j<=k} c_j
// of the exact sum of its terms (each add rounds by at most 2^-24 of its result, the
// first term is exact), so with T~_k = sum_{j<=k} c~_j (bounded from the block sums: every
// c~_j of block b is <= blk[b]; the specialised filter bounds the blocks before the one
// holding r by jb B blk[jb - 1]) the two chains differ at index k by at most
//   D_k = 2^-23 T~_k + EPS_W c~_k + (k + 1) A_W,
// and r = fl(u c_N) differs from r~ = fl(u c~_N) by at most D_r = u D_N + 2^-23 r~.  If the
// filter's pick k has r~ - c~_{k-1} > D_{k-1} + D_r and c~_k - r~ > D_k + D_r, then
// c_{k-1} < r <= c_k: the reference picks the same k (its first cdf entry >= r).  The
// margins carry a 1.002 factor and a 1e-9 C~ term for the second-order terms (the
// reference chain's T_k vs T~_k, EPS_W S_k vs EPS_W c~_k, the float evaluation of the
// margins).  NaN / inf anywhere fails a comparison and takes the exact path.
#define GC_REF_FILTER_EPS_W 6.0e-7f  // EPS_MUFU + EPS_NP = 5.13e-7, with slack
#define GC_REF_FILTER_A_W 1.0e-9f    // measured additive excess <= 3.7e-10 (FTZ, argument rounding)

// Pre-beta logits Q'(k), Q'(k + 1) of an action pair for a compile-time utility kind, op
// for op the reference's (ref_logit2 before its beta product); (ax, ay) from one LDS.128.
template <int QK>
__device__ __forceinline__ float2 ref_q2(const SmemAct &S, int k, float rx, float ry, float d2) {
    const float2 at = *reinterpret_cast<const float2 *>(&S.aat[k]);
    if (QK == GC_Q_DEFAULT) return px_add(px2(-d2), make_float2(-at.x, -at.y));
    const float4 a = S.axy[k >> 1];
    float2 L = px_fma(px2(ry), make_float2(a.z, a.w), px_mul(px2(rx), make_float2(a.x, a.y)));
    L = px_mul(L, px2(-2.0f));
    L = px_add(L, make_float2(-at.x, -at.y));
    if (QK == GC_Q_GOAL_PROGRESS_FULL) L = px_add(L, px2(-d2));
    return L;
}

// Guess of max_k Q'_k for a grid table (gc_action_table.ref_grid_rows = R): without a
// heading weight the best action of every speed row points along one of the two headings
// that bracket the direction to the goal, so the exact Q' of those 2R actions is evaluated
// (reference float ops).  The bracket comes from a coarse atan2 (|error| < 0.004 rad
// against a half heading step of 0.13 rad: the nearest heading is always in it).  Only a
// guess -- ref_fast_spec checks it against the max of every beta-scaled logit it computes.
template <int QK>
__device__ __forceinline__ float ref_qmax_guess(const SmemAct &S, float rx, float ry, float d2, int rows) {
    const float gx = -rx, gy = -ry;  // particle -> goal
    const float ax = fabsf(gx), ay = fabsf(gy);
    const float mn = fminf(ax, ay), mx = fmaxf(ax, ay);
    const float a = mx > 0.f ? __fdividef(mn, mx) : 0.f;
    float ang = a * fmaf(0.2733f, 1.f - a, 0.78539816f);  // atan(a), a in [0, 1]
    if (ay > ax) ang = 1.57079633f - ang;
    if (gx < 0.f) ang = 3.14159265f - ang;
    if (gy < 0.f) ang = -ang;
    int b = (int)floorf((ang + 3.14159265f) * (12.f / 3.14159265f));  // heading b: -pi + b pi/12
    b = b < 0 ? 0 : (b > 23 ? 23 : b);
    const int b2 = b == 23 ? 0 : b + 1;
    float q = -__int_as_float(0x7f800000);
#pragma unroll 1
    for (int r = 0; r < rows; ++r) {
        const int k0 = r * 24 + b, k1 = r * 24 + b2;
        float L0 = __fmul_rn(__fmaf_rn(ry, S.ay[k0], __fmul_rn(rx, S.ax[k0])), -2.0f);
        float L1 = __fmul_rn(__fmaf_rn(ry, S.ay[k1], __fmul_rn(rx, S.ax[k1])), -2.0f);
        L0 = __fsub_rn(L0, S.aat[k0]);
        L1 = __fsub_rn(L1, S.aat[k1]);
        if (QK == GC_Q_GOAL_PROGRESS_FULL) { L0 = __fsub_rn(L0, d2); L1 = __fsub_rn(L1, d2); }
        q = fmaxf(q, fmaxf(L0, L1));
    }
    return q;
}

// The filter for a compile-time utility kind and block size B (m_keep == 12 B: the
// 96-action grid or the 48 slow actions mask_stationary keeps): every loop fully unrolled.  The max of the
// beta-scaled logits is taken before the product -- fl(beta x) is monotone in x for
// beta > 0 (RationalitySet requires it), so max_k fl(beta Q'_k) = fl(beta max_k Q'_k) bit for
// bit.  Returns the pick, or -1 when the margin test fails (M is then the reference's max
// for the exact path).  Margins as in the error budget above.
template <int QK, int B>
__device__ __forceinline__ int ref_fast_spec(const SmemAct &S, float rx, float ry, float d2, float beta, float u,
                                             int rows, float &M) {
    constexpr int NBLK = 12, MK = NBLK * B;
    constexpr float L2E = 1.4426950408889634f;
    float qmax;
    if (rows > 0) {
        qmax = ref_qmax_guess<QK>(S, rx, ry, d2, rows);  // checked below
    } else {
        float qa = -__int_as_float(0x7f800000), qb = qa;
#pragma unroll 2
        for (int k = 0; k < MK; k += 4) {  // two independent max chains
            const float2 q0 = ref_q2<QK>(S, k, rx, ry, d2);
            qa = fmaxf(qa, fmaxf(q0.x, q0.y));
            if (k + 2 < MK) {
                const float2 q1 = ref_q2<QK>(S, k + 2, rx, ry, d2);
                qb = fmaxf(qb, fmaxf(q1.x, q1.y));
            }
        }
        qmax = fmaxf(qa, qb);
    }
    M = __fmul_rn(qmax, beta);
    const float2 nM = px2(-M);
    float blk[NBLK];
    float c = 0.f;
    float lm = -__int_as_float(0x7f800000);  // max of the beta-scaled logits (the guess check)
#pragma unroll
    for (int j = 0; j < NBLK; ++j) {
#pragma unroll
        for (int i = 0; i < B; i += 2) {
            const float2 q = ref_q2<QK>(S, j * B + i, rx, ry, d2);
            const float2 L = px_mul(q, px2(beta));
            lm = fmaxf(lm, fmaxf(L.x, L.y));
            const float2 t = px_mul(px_sub_after_mul(L, nM), px2(L2E));
            c = __fadd_rn(c, ex2_approx(t.x));
            c = __fadd_rn(c, ex2_approx(t.y));
        }
        blk[j] = c;
    }
    // the guessed max must be the reference's max (numpy's logits.max), or every x_k
    // differs from the reference's: the exact path then runs with the true max
    if (lm != M) { M = lm; return -1; }
    const float r = __fmul_rn(u, c);
    int jb = 0;
    float cc = 0.f, tall = blk[NBLK - 1];
#pragma unroll
    for (int j = 0; j < NBLK - 1; ++j) {
        tall = __fadd_rn(tall, blk[j]);
        if (blk[j] < r) { jb = j + 1; cc = blk[j]; }
    }
    const float tpre = (float)jb * cc;  // >= the earlier block ends' sum (each <= cc)
    // rescan the block holding r with the same operations (the same chain values)
    float lower = cc;
    int i = 0;
#pragma unroll
    for (; i < B; i += 2) {
        const float2 q = ref_q2<QK>(S, jb * B + i, rx, ry, d2);
        const float2 t = px_mul(px_add(make_float2(__fmul_rn(q.x, beta), __fmul_rn(q.y, beta)), nM), px2(L2E));
        const float w0 = ex2_approx(t.x), w1 = ex2_approx(t.y);
        lower = cc;
        cc = __fadd_rn(cc, w0);
        if (!(cc < r)) break;
        lower = cc;
        cc = __fadd_rn(cc, w1);
        if (!(cc < r)) { ++i; break; }
    }
    const int k = jb * B + i;
    const float fB = (float)B, kin = (float)i;
    const float tb = fB * tpre;
    const float t_lo = fmaf(kin, lower, tb), t_hi = fmaf(kin + 1.f, cc, tb);
    const float d_r = fmaf(u, fmaf(0x1p-23f, fB * tall, fmaf(GC_REF_FILTER_EPS_W, c, (float)MK * GC_REF_FILTER_A_W)),
                           0x1p-23f * r);
    const float d_lo = fmaf(0x1p-23f, t_lo, fmaf(GC_REF_FILTER_EPS_W, lower, (float)k * GC_REF_FILTER_A_W));
    const float d_hi = fmaf(0x1p-23f, t_hi, fmaf(GC_REF_FILTER_EPS_W, cc, (float)(k + 1) * GC_REF_FILTER_A_W));
    const float slack = 1e-9f * c;
    if (i < B && __fsub_rn(cc, r) > fmaf(1.002f, d_hi + d_r, slack) &&
        (k == 0 || __fsub_rn(r, lower) > fmaf(1.002f, d_lo + d_r, slack)))
        return k < MK - 1 ? k : MK - 1;
    return -1;
}

// The reference float32 step (prediction.py:147-162): per-action logit, max shift, numpy
// exp, sequential cumsum, first cdf entry >= u * total.  The logits and the max are
// computed exactly as the reference does; the exponentials are then first evaluated with
// the MUFU ex2 (one instruction instead of numpy's ~30-instruction float32 exp), and the
// decision is accepted only when r lies farther than the proven error margin G from both
// cdf entries that bracket it -- the reference's decision is then the same (see the error
// budget above).  Otherwise (a few % of particle-steps) the exact passes run.  The result is
// bit-identical to ref_pick_exact alone for every input; `filter` = false forces the exact
// path (A/B and tests), `fallbacks` counts the particle-steps that took it.
__device__ __forceinline__ int ref_pick(const SmemTabs &H, const SmemAct &S, float x, float y, int h, float u,
                                        bool filter = true, unsigned long long *fallbacks = nullptr) {
    const float rx = __fsub_rn(x, H.hgx[h]), ry = __fsub_rn(y, H.hgy[h]);
    const float d2 = __fadd_rn(__fmul_rn(rx, rx), __fmul_rn(ry, ry));
    const float beta = H.hb[h];
    const int mk = H.m_keep, qk = H.q_kind;
    float M = -__int_as_float(0x7f800000);
    if (filter && mk == 96 && qk == GC_Q_GOAL_PROGRESS) {  // the standard 96-action grid
        const int a = ref_fast_spec<GC_Q_GOAL_PROGRESS, 8>(S, rx, ry, d2, beta, u, H.ref_rows, M);
        if (a >= 0) return a;
        if (fallbacks) atomicAdd(fallbacks, 1ull);
        return ref_pick_exact(S, rx, ry, d2, beta, mk, qk, M, u);
    }
    if (filter && mk == 48 && qk == GC_Q_GOAL_PROGRESS_FULL) {  // its 48 slow actions (mask_stationary)
        const int a = ref_fast_spec<GC_Q_GOAL_PROGRESS_FULL, 4>(S, rx, ry, d2, beta, u, H.ref_rows, M);
        if (a >= 0) return a;
        if (fallbacks) atomicAdd(fallbacks, 1ull);
        return ref_pick_exact(S, rx, ry, d2, beta, mk, qk, M, u);
    }
    int k = 0;
#pragma unroll 4
    for (; k + 1 < mk; k += 2) {  // action pairs on the packed FP32x2 pipe
        const float2 L = ref_logit2(S, k, rx, ry, d2, beta, qk);
        M = fmaxf(M, fmaxf(L.x, L.y));
    }
    if (k < mk) M = fmaxf(M, ref_logit(S, k, rx, ry, d2, beta, qk));
    if (filter) {
        constexpr float L2E = 1.4426950408889634f;
        constexpr int NBLK = 12;
        const int B = 2 * ((mk + 2 * NBLK - 1) / (2 * NBLK));
        float blk[NBLK];
        float c = 0.f;
#pragma unroll
        for (int j = 0; j < NBLK; ++j) {
            const int k1 = min(mk, (j + 1) * B);
            int kk = j * B;
#pragma unroll 2
            for (; kk + 1 < k1; kk += 2) {
                const float2 L = ref_logit2(S, kk, rx, ry, d2, beta, qk);
                const float2 t = px_mul(px_add(L, px2(-M)), px2(L2E));
                c = __fadd_rn(c, ex2_approx(t.x));
                c = __fadd_rn(c, ex2_approx(t.y));
            }
            if (kk < k1) c = __fadd_rn(c, ex2_approx(__fmul_rn(__fsub_rn(ref_logit(S, kk, rx, ry, d2, beta, qk), M), L2E)));
            blk[j] = c;
        }
        const float r = __fmul_rn(u, c);
        int jb = 0;
        float cc = 0.f, tpre = 0.f, tall = blk[NBLK - 1];
#pragma unroll
        for (int j = 0; j < NBLK - 1; ++j) {
            tall = __fadd_rn(tall, blk[j]);
            if (blk[j] < r) { jb = j + 1; cc = blk[j]; tpre = __fadd_rn(tpre, blk[j]); }
        }
        // rescan the block holding r with the same operations (the same chain values)
        k = jb * B;
        const int kend = min(mk, (jb + 1) * B);
        float lower = cc;
        for (; k < kend; ++k) {
            lower = cc;
            cc = __fadd_rn(cc, ex2_approx(__fmul_rn(__fsub_rn(ref_logit(S, k, rx, ry, d2, beta, qk), M), L2E)));
            if (!(cc < r)) break;
        }
        // error margins of the two bracketing cdf entries and of r (error budget above);
        // all inputs non-negative, evaluated in float with the 1.002 factor
        const float fB = (float)B, kin = (float)(k - jb * B);
        const float tb = fB * tpre;                                   // >= T~ of the earlier blocks
        const float t_lo = fmaf(kin, lower, tb), t_hi = fmaf(kin + 1.f, cc, tb);
        const float d_r = fmaf(u, fmaf(0x1p-23f, fB * tall, fmaf(GC_REF_FILTER_EPS_W, c, (float)mk * GC_REF_FILTER_A_W)),
                               0x1p-23f * r);
        const float d_lo = fmaf(0x1p-23f, t_lo, fmaf(GC_REF_FILTER_EPS_W, lower, (float)k * GC_REF_FILTER_A_W));
        const float d_hi = fmaf(0x1p-23f, t_hi, fmaf(GC_REF_FILTER_EPS_W, cc, (float)(k + 1) * GC_REF_FILTER_A_W));
        const float slack = 1e-9f * c;
        if (k < kend && __fsub_rn(cc, r) > fmaf(1.002f, d_hi + d_r, slack) &&
            (k == 0 || __fsub_rn(r, lower) > fmaf(1.002f, d_lo + d_r, slack)))
            return k < mk - 1 ? k : mk - 1;
    }
    if (fallbacks) atomicAdd(fallbacks, 1ull);
    return ref_pick_exact(S, rx, ry, d2, beta, mk, qk, M, u);
}

// ---- production generic per-action softmax ------------------------------------------
// logits (log2 units) of the action pair (k, k + 1), k even, on the packed FP32x2 pipe
__device__ __forceinline__ float2 gen_logit2(const SmemAct &S, int k, float rx, float ry, float d2, float bl,
                                             int qk) {
    const float2 at = *reinterpret_cast<const float2 *>(&S.aat[k]);
    float2 q;
    if (qk == GC_Q_DEFAULT) {
        q = __fadd2_rn(make_float2(-d2, -d2), make_float2(-at.x, -at.y));
    } else {
        const float2 ax = *reinterpret_cast<const float2 *>(&S.ax[k]);
        const float2 ay = *reinterpret_cast<const float2 *>(&S.ay[k]);
        const float2 t = __ffma2_rn(make_float2(ry, ry), ay, __fmul2_rn(make_float2(rx, rx), ax));
        q = __ffma2_rn(make_float2(-2.f, -2.f), t, make_float2(-at.x, -at.y));
    }
    return __fmul2_rn(q, make_float2(bl, bl));
}

// exact-in-distribution softmax sample over any control set: max pass, one pass of the
// running sum that keeps it at 12 block ends, then only the block holding r is rescanned.
// The action tables are padded to an even count (pairs), padded weights are not summed.
__device__ __forceinline__ int gen_pick(const SmemTabs &H, const SmemAct &S, float x, float y, int h, float u) {
    const float rx = x - H.hgx[h], ry = y - H.hgy[h];
    const float d2 = fmaf(rx, rx, ry * ry);
    const float bl = H.hb[h] * 1.4426950408889634f;
    const int mk = H.m_keep, qk = H.q_kind;
    float M = -__int_as_float(0x7f800000);
    for (int k = 0; k < mk; k += 2) {
        const float2 L = gen_logit2(S, k, rx, ry, d2, bl, qk);
        M = fmaxf(M, k + 1 < mk ? fmaxf(L.x, L.y) : L.x);
    }
    constexpr int NBLK = 12;
    const int B = 2 * ((mk + 2 * NBLK - 1) / (2 * NBLK));
    float blk[NBLK];
    float c = 0.f;
#pragma unroll
    for (int j = 0; j < NBLK; ++j) {
        const int k1 = min(mk, (j + 1) * B);
        for (int k = j * B; k < k1; k += 2) {
            const float2 L = gen_logit2(S, k, rx, ry, d2, bl, qk);
            c += ex2_approx(L.x - M);
            if (k + 1 < k1) c += ex2_approx(L.y - M);
        }
        blk[j] = c;
    }
    const float r = u * c;
    // first action whose running sum exceeds r: skip the blocks that end at or below r
    int jb = 0;
    float cc = 0.f;
#pragma unroll
    for (int j = 0; j < NBLK - 1; ++j) {
        if (blk[j] <= r) { jb = j + 1; cc = blk[j]; }
    }
    const int k1 = min(mk, (jb + 1) * B);
    int k = jb * B;
    for (; k < k1; k += 2) {
        const float2 L = gen_logit2(S, k, rx, ry, d2, bl, qk);
        cc += ex2_approx(L.x - M);
        if (cc > r) break;
        if (k + 1 < k1) {
            cc += ex2_approx(L.y - M);
            if (cc > r) { ++k; break; }
        }
    }
    return k < mk - 1 ? k : mk - 1;
}

// The generic sampler for a compile-time utility kind and block size (m_keep == 12 B: the
// 96 actions of a 4 x 24 set or 48 of them), one pass: instead of a max pass it shifts the
// logits by an analytic upper bound of their max -- by Cauchy-Schwarz, -2 rel.s_k - at_k <=
// 2 |rel| max_k|s_k| - min_k at_k (and -d2 - pen_k <= -d2 - min_k pen_k for q_default) -- so
// every weight is <= 1; the bound is loose by the angle to the nearest action and the action
// term (a few log2 units for the standard sets), and a total below 2^-60 (a bound so loose
// that the weights underflow, e.g. beta ~ 300) takes the two-pass gen_pick.  Then the
// 12-block running sum, the block holding r and a rescan of it, fully unrolled, action pairs
// from one LDS.128.  Same distribution as gen_pick (the shift cancels in the normalisation).
template <int QK, int B>
__device__ __forceinline__ int gen_fast_spec(const SmemTabs &H, const SmemAct &S, float x, float y, int h, float u) {
    constexpr int NBLK = 12;
    const float rx = x - H.hgx[h], ry = y - H.hgy[h];
    const float d2 = fmaf(rx, rx, ry * ry);
    const float bl = H.hb[h] * 1.4426950408889634f;
    float bound;
    if (QK == GC_Q_DEFAULT) {
        bound = -d2 - H.gatmin;
    } else {
        float rs;
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rs) : "f"(fmaxf(d2, 1e-30f)));
        bound = fmaf(2.f * d2 * rs * 1.0001f, H.gsmax, -H.gatmin);  // 2 |rel| max|s| - min at
        if (QK == GC_Q_GOAL_PROGRESS_FULL) bound -= d2;
    }
    const float2 nM = make_float2(-bl * bound, -bl * bound);
    const float2 BL = make_float2(bl, bl);
    auto w2 = [&](int k) {
        const float2 at = *reinterpret_cast<const float2 *>(&S.aat[k]);
        float2 q;
        if (QK == GC_Q_DEFAULT) {
            q = __fadd2_rn(make_float2(-d2, -d2), make_float2(-at.x, -at.y));
        } else {
            const float4 a = S.axy[k >> 1];
            const float2 t = __ffma2_rn(make_float2(ry, ry), make_float2(a.z, a.w),
                                        __fmul2_rn(make_float2(rx, rx), make_float2(a.x, a.y)));
            q = __ffma2_rn(make_float2(-2.f, -2.f), t, make_float2(-at.x, -at.y));
            if (QK == GC_Q_GOAL_PROGRESS_FULL) q = __fadd2_rn(q, make_float2(-d2, -d2));
        }
        const float2 e = __ffma2_rn(q, BL, nM);
        return make_float2(ex2_approx(e.x), ex2_approx(e.y));
    };
    float blk[NBLK];
    float c = 0.f;
#pragma unroll
    for (int j = 0; j < NBLK; ++j) {
#pragma unroll
        for (int i = 0; i < B; i += 2) {
            const float2 w = w2(j * B + i);
            c += w.x + w.y;
        }
        blk[j] = c;
    }
    if (!(c >= 0x1p-60f)) return -1;  // the bound was far too loose (or NaN): two-pass sampler
    const float r = u * c;
    int jb = 0;
    float cc = 0.f;
#pragma unroll
    for (int j = 0; j < NBLK - 1; ++j) {
        if (blk[j] <= r) { jb = j + 1; cc = blk[j]; }
    }
    int i = 0;
#pragma unroll
    for (; i < B; i += 2) {
        const float2 w = w2(jb * B + i);
        cc += w.x;
        if (cc > r) break;
        cc += w.y;
        if (cc > r) { ++i; break; }
    }
    const int k = jb * B + i;
    return k < NBLK * B - 1 ? k : NBLK * B - 1;
}

// production generic sampler: the unrolled one-pass form for the common action counts
static __device__ __noinline__ int gen_sample(const SmemTabs &H, const SmemAct &S, float x, float y, int h, float u) {
    const int mk = H.m_keep, qk = H.q_kind;
    int a = -1;
    if (mk == 96) {
        if (qk == GC_Q_GOAL_PROGRESS) a = gen_fast_spec<GC_Q_GOAL_PROGRESS, 8>(H, S, x, y, h, u);
        else if (qk == GC_Q_GOAL_PROGRESS_FULL) a = gen_fast_spec<GC_Q_GOAL_PROGRESS_FULL, 8>(H, S, x, y, h, u);
        else if (qk == GC_Q_DEFAULT) a = gen_fast_spec<GC_Q_DEFAULT, 8>(H, S, x, y, h, u);
    } else if (mk == 48) {
        if (qk == GC_Q_GOAL_PROGRESS) a = gen_fast_spec<GC_Q_GOAL_PROGRESS, 4>(H, S, x, y, h, u);
        else if (qk == GC_Q_GOAL_PROGRESS_FULL) a = gen_fast_spec<GC_Q_GOAL_PROGRESS_FULL, 4>(H, S, x, y, h, u);
        else if (qk == GC_Q_DEFAULT) a = gen_fast_spec<GC_Q_DEFAULT, 4>(H, S, x, y, h, u);
    }
    return a >= 0 ? a : gen_pick(H, S, x, y, h, u);
}

// ---- production factorised sampler (grid control set x goal-progress utility) --------
// logit(a,b) = beta*(-2 tau a dv d_b - (tau^2 + w_v) a^2 dv^2 - w_th theta_b^2) + const,
// d_b = rel . (cos th_b, sin th_b).  With k = 2 beta tau dv, r = |rel|:
//   weight(a,b) = H_b * G_a * e_b^a,  e_b = exp(-k (d_b + r)) in (0,1],
//   G_a = exp(a k r - c a^2 - S),     S = max_a (a k r - c a^2),  H_b = exp(-beta w_th th_b^2)
// -> per step: NB ex2 (e_b), 4 ex2 (G_a), Horner in e_b, inverse CDF over headings then
//    over speeds.  Zero-speed actions share displacement 0 and merge into one "stay".
//    (fact_step_sym below: the standard heading set, one ex2 for all G_a.)
// the standard ControlSet.grid heading set theta_b = -pi + b*pi/12 (agents.py:79-87),
// float32 cos/sin as the host computes them: a launch whose tables hold exactly these
// values takes MODE_FACTS (symmetric heading pairs, fact_step_sym)
#define GC_STD_COS                                                                                  \
    {-1.f, -0.965925813f, -0.866025388f, -0.707106769f, -0.5f, -0.258819044f, 6.12323426e-17f,     \
     0.258819044f, 0.5f, 0.707106769f, 0.866025388f, 0.965925813f, 1.f, 0.965925813f, 0.866025388f, \
     0.707106769f, 0.5f, 0.258819044f, 6.12323426e-17f, -0.258819044f, -0.5f, -0.707106769f,       \
     -0.866025388f, -0.965925813f}
#define GC_STD_SIN                                                                                  \
    {-1.22464685e-16f, -0.258819044f, -0.5f, -0.707106769f, -0.866025388f, -0.965925813f, -1.f,    \
     -0.965925813f, -0.866025388f, -0.707106769f, -0.5f, -0.258819044f, 0.f, 0.258819044f, 0.5f,   \
     0.707106769f, 0.866025388f, 0.965925813f, 1.f, 0.965925813f, 0.866025388f, 0.707106769f, 0.5f, \
     0.258819044f}
static const float hStdCos[NBF] = GC_STD_COS;
static const float hStdSin[NBF] = GC_STD_SIN;

template <bool WTH>
__device__ __forceinline__ void fact_step(const SmemTabs &S, const KParams &P, float &x, float &y,
                                          int h, float u1) {
    const float4 hp = S.hp[h];
    const float rx = x - hp.x, ry = y - hp.y;
    const float r2 = fmaf(rx, rx, ry * ry);
    float rs;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rs) : "f"(fmaxf(r2, 1e-30f)));
    const float r = r2 * rs;
    const float kk = hp.z, c2 = hp.w;
    const float kr = kk * r;
    const float A = -kk * rx, B = -kk * ry, nkr = -kr;
    const int na = S.n_speeds;
    const float s1 = kr - c2, s2 = fmaf(2.f, kr, -4.f * c2), s3 = fmaf(3.f, kr, -9.f * c2);
    float Smax = fmaxf(0.f, s1);
    if (na > 2) Smax = fmaxf(Smax, s2);
    if (na > 3) Smax = fmaxf(Smax, s3);
    const float G0 = ex2_approx(-Smax);
    const float G1 = ex2_approx(s1 - Smax);
    const float G2 = na > 2 ? ex2_approx(s2 - Smax) : 0.f;
    const float G3 = na > 3 ? ex2_approx(s3 - Smax) : 0.f;
    float cum[NBF];
    float C = 0.f;
#if GC_FFMA2
    if (!WTH) {
        // headings in pairs on the packed FP32x2 pipe (FFMA2: two FMAs per issue slot);
        // the running sum stays scalar so cum[] keeps the same order of additions
        const float2 AA = make_float2(A, A), BB = make_float2(B, B), NK = make_float2(nkr, nkr);
        const float2 g3 = make_float2(G3, G3), g2 = make_float2(G2, G2), g1 = make_float2(G1, G1);
#pragma unroll
        for (int b = 0; b < NBF; b += 2) {
            // heading pairs straight from the parameter bank (64-bit constant operands)
            const float2 cs = make_float2(P.hcos[b], P.hcos[b + 1]);
            const float2 sn = make_float2(P.hsin[b], P.hsin[b + 1]);
            const float2 xe = __ffma2_rn(AA, cs, __ffma2_rn(BB, sn, NK));
            const float2 e = make_float2(ex2_approx(xe.x), ex2_approx(xe.y));
            const float2 poly = __ffma2_rn(e, __ffma2_rn(e, g3, g2), g1);
            C = fmaf(e.x, poly.x, C);
            cum[b] = C;
            C = fmaf(e.y, poly.y, C);
            cum[b + 1] = C;
        }
    } else
#endif
#pragma unroll
    for (int b = 0; b < NBF; ++b) {
        const float cb = P.hcos[b];
        const float sb = P.hsin[b];
        // e_b = exp(-k (d_b + r)), d_b = rel . (cos th_b, sin th_b): 2 FFMA + 1 MUFU
        const float e = ex2_approx(fmaf(A, cb, fmaf(B, sb, nkr)));
        // cumulative moving weight: C += H_b e (G1 + e (G2 + e G3)), 3 FFMA
        const float poly = fmaf(e, fmaf(e, G3, G2), G1);
        if (WTH) C = fmaf(e * ex2_approx(-S.wth * S.hb[h] * P.hth2[b]), poly, C);
        else C = fmaf(e, poly, C);
        cum[b] = C;
    }
    const float Z0 = G0 * S.hq[h].w;
    const float rr = u1 * (Z0 + C);
    const float t = rr - Z0;
    // heading = #{b : cum_b <= t}: cum is monotone, so halve the candidate set with one
    // compare + selects per level (24 -> 12 -> 6 -> 3), then count the last three; lo
    // tracks the largest cum_b <= t (the start of the chosen heading's interval)
    int b = 0;
    float lo = 0.f;
    {
        bool p = cum[11] <= t;
        b += p ? 12 : 0;
        lo = p ? cum[11] : lo;
#pragma unroll
        for (int i = 0; i < 12; ++i) cum[i] = p ? cum[i + 12] : cum[i];
        p = cum[5] <= t;
        b += p ? 6 : 0;
        lo = p ? cum[5] : lo;
#pragma unroll
        for (int i = 0; i < 6; ++i) cum[i] = p ? cum[i + 6] : cum[i];
        p = cum[2] <= t;
        b += p ? 3 : 0;
        lo = p ? cum[2] : lo;
#pragma unroll
        for (int i = 0; i < 3; ++i) cum[i] = p ? cum[i + 3] : cum[i];
        // the last three entries: cum is non-decreasing, so p2 implies p1 implies p0
        const bool p0 = cum[0] <= t, p1 = cum[1] <= t, p2 = cum[2] <= t;
        b += p2 ? 3 : (p1 ? 2 : (p0 ? 1 : 0));
        lo = p2 ? cum[2] : (p1 ? cum[1] : (p0 ? cum[0] : lo));
    }
    b = b < NBF - 1 ? b : NBF - 1;
    // speed within the heading from the residual of the same uniform: given b,
    // (t - lo) is uniform on [0, H_b sum_a G_a e_b^a) (up to the 2^-24 resolution of u1)
    const float2 cs = S.hcs[b];
    const float e = ex2_approx(fmaf(A, cs.x, fmaf(B, cs.y, nkr)));
    float w1 = G1 * e, w2 = G2 * e * e;
    if (WTH) {
        const float hb = ex2_approx(-S.wth * S.hb[h] * P.hth2[b]);
        w1 *= hb;
        w2 *= hb;
    }
    const float res = t - lo;
    int a = 1 + ((w1 <= res) ? 1 : 0) + ((w1 + w2 <= res) ? 1 : 0);
    a = a < na - 1 ? a : na - 1;
    // stay (rr < Z0): every zero-speed action has displacement 0 -- row a = 0 of fd is
    // (0, 0) for every heading, so staying is just a = 0
    a = (rr < Z0) ? 0 : a;
    GC_DCHECK(a >= 0 && a < NAF && b >= 0 && b < NBF);
    const float2 d = S.fd[a * NBF + b];
    x = __fadd_rn(x, d.x);  // the reference's float32 position update (prediction.py:161-162)
    y = __fadd_rn(y, d.y);
}

// MODE_FACTS (standard heading set, n_speeds <= 4): the factorised sampler with
//  (1) speed weights normalised at the TOP speed instead of by a max shift: with
//      Q = 2^-kr, G_a / G_top = Q^(top-a) 2^(c (top^2 - a^2)), so one ex2 (Q) and a few
//      products replace 4 ex2; the per-hypothesis powers of 2^c (Ka, Kb, Kc) are staged
//      in the prologue, and a CTA whose constants would overflow (c > ~11 at 4 speeds,
//      i.e. beta > ~140 with the default tables) keeps the max-shift form (qg = false);
//  (2) opposite headings b and b + 12 (theta + pi) in one go: x_{b+12} = -x_b - 2kr, so
//      heading pair (b, b+1) costs two FFMA2 and the opposite pair one.  The cumulative
//      sum runs in the order (0, 1, 12, 13, 2, 3, 14, 15, ...): index i <-> heading
//      2(i>>2) + (i&1) + 12((i>>1)&1); the prologue stores the chosen-heading (cos, sin) and
//      the displacements in that order, so the search result indexes them directly.
//  (3) WTH (w_th != 0): heading weights H_b = exp(-beta w_th theta_b^2) per hypothesis from a
//      shared-memory table in the same order (Htab), one LDS.128 per four headings.
template <bool WTH, bool QG, bool NA4>
__device__ __forceinline__ void fact_step_sym(const SmemTabs &S, const KParams &P, const float *Htab, float &x,
                                              float &y, int h, float u1, bool qg) {
    GC_DCHECK(h >= 0 && h < S.n_hyp);
    const float4 hp = S.hp[h];
    const float4 hq = S.hq[h];
    const float rx = x - hp.x, ry = y - hp.y;
    const float r2 = fmaf(rx, rx, ry * ry);
    float rs;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(rs) : "f"(fmaxf(r2, 1e-30f)));
    const float r = r2 * rs;
    const float kk = hp.z;
    const float kr = kk * r;
    const float A = -kk * rx, B = -kk * ry, nkr = -kr;
    const int na = S.n_speeds;
    float G1, G2, G3, Z0;
    if (QG || qg) {  // QG: the max-shift branch is compiled out (2.8 % of K2 at cfg3)
        const float Q = ex2_approx(nkr), Q2 = Q * Q;
        if (NA4 || na == 4) {  // the standard grid: straight-line code on the common path
            G3 = 1.f; G2 = Q * hp.w; G1 = Q2 * hq.x; Z0 = Q2 * Q * hq.y;
        } else {
            const bool p3 = na == 3;
            G3 = 0.f; G2 = p3 ? 1.f : 0.f; G1 = p3 ? Q * hp.w : 1.f; Z0 = p3 ? Q2 * hq.x : Q * hp.w;
        }
    } else {
        const float c2 = hq.z;
        const float s1 = kr - c2, s2 = fmaf(2.f, kr, -4.f * c2), s3 = fmaf(3.f, kr, -9.f * c2);
        float Smax = fmaxf(0.f, s1);
        if (na > 2) Smax = fmaxf(Smax, s2);
        if (na > 3) Smax = fmaxf(Smax, s3);
        Z0 = ex2_approx(-Smax) * hq.w;
        G1 = ex2_approx(s1 - Smax);
        G2 = na > 2 ? ex2_approx(s2 - Smax) : 0.f;
        G3 = na > 3 ? ex2_approx(s3 - Smax) : 0.f;
    }
    float cum[NBF];
    float C = 0.f;
    {
        const float2 AA = make_float2(A, A), BB = make_float2(B, B), NK = make_float2(nkr, nkr);
        const float2 NK2 = make_float2(2.f * nkr, 2.f * nkr), M1 = make_float2(-1.f, -1.f);
        const float2 g3 = make_float2(G3, G3), g2 = make_float2(G2, G2), g1 = make_float2(G1, G1);
#pragma unroll
        for (int j = 0; j < NBF / 4; ++j) {
            const float2 cs = make_float2(P.hcos[2 * j], P.hcos[2 * j + 1]);
            const float2 sn = make_float2(P.hsin[2 * j], P.hsin[2 * j + 1]);
            const float2 xe = __ffma2_rn(AA, cs, __ffma2_rn(BB, sn, NK));
            const float2 xo = __ffma2_rn(xe, M1, NK2);  // headings 2j + 12, 2j + 13
            const float2 e = make_float2(ex2_approx(xe.x), ex2_approx(xe.y));
            const float2 eo = make_float2(ex2_approx(xo.x), ex2_approx(xo.y));
            const float2 poly = __ffma2_rn(e, __ffma2_rn(e, g3, g2), g1);
            const float2 polyo = __ffma2_rn(eo, __ffma2_rn(eo, g3, g2), g1);
            float2 w = e, wo = eo;
            if (WTH) {  // heading weights H_b of this hypothesis, slots 4j..4j+3 (one LDS.128)
                const float4 H4 = *reinterpret_cast<const float4 *>(Htab + h * NBF + 4 * j);
                w = __fmul2_rn(e, make_float2(H4.x, H4.y));
                wo = __fmul2_rn(eo, make_float2(H4.z, H4.w));
            }
            C = fmaf(w.x, poly.x, C);
            cum[4 * j] = C;
            C = fmaf(w.y, poly.y, C);
            cum[4 * j + 1] = C;
            C = fmaf(wo.x, polyo.x, C);
            cum[4 * j + 2] = C;
            C = fmaf(wo.y, polyo.y, C);
            cum[4 * j + 3] = C;
        }
    }
    const float rr = u1 * (Z0 + C);
    const float t = rr - Z0;
    int b = 0;
    float lo = 0.f;
    {
        bool p = cum[11] <= t;
        b += p ? 12 : 0;
        lo = p ? cum[11] : lo;
#pragma unroll
        for (int i = 0; i < 12; ++i) cum[i] = p ? cum[i + 12] : cum[i];
        p = cum[5] <= t;
        b += p ? 6 : 0;
        lo = p ? cum[5] : lo;
#pragma unroll
        for (int i = 0; i < 6; ++i) cum[i] = p ? cum[i + 6] : cum[i];
        p = cum[2] <= t;
        b += p ? 3 : 0;
        lo = p ? cum[2] : lo;
#pragma unroll
        for (int i = 0; i < 3; ++i) cum[i] = p ? cum[i + 3] : cum[i];
        // the last three entries: cum is non-decreasing, so p2 implies p1 implies p0
        const bool p0 = cum[0] <= t, p1 = cum[1] <= t, p2 = cum[2] <= t;
        b += p2 ? 3 : (p1 ? 2 : (p0 ? 1 : 0));
        lo = p2 ? cum[2] : (p1 ? cum[1] : (p0 ? cum[0] : lo));
    }
    b = b < NBF - 1 ? b : NBF - 1;  // b is the cumulative-order index i
    // the chosen heading's e exactly as the loop computed it (same FMAs, same lanes)
    const float2 cs = S.hcs[b];  // forward (cos, sin) of heading 2(i>>2) + (i&1)
    float xb = fmaf(A, cs.x, fmaf(B, cs.y, nkr));
    if (b & 2) xb = fmaf(xb, -1.f, 2.f * nkr);
    const float e = ex2_approx(xb);
    const float eh = WTH ? e * Htab[h * NBF + b] : e;
    const float w1 = G1 * eh, w2 = G2 * e * eh;
    const float res = t - lo;
    int a = 1 + ((w1 <= res) ? 1 : 0) + ((w1 + w2 <= res) ? 1 : 0);
    if (!NA4) a = a < na - 1 ? a : na - 1;  // (4 speeds: a <= 3 already)
    a = (rr < Z0) ? 0 : a;  // stay: row 0 of fd is (0, 0)
    GC_DCHECK(a >= 0 && a < NAF && b >= 0 && b < NBF);
    const float2 d = S.fd[a * NBF + b];
    x = __fadd_rn(x, d.x);  // the reference's float32 position update (prediction.py:161-162)
    y = __fadd_rn(y, d.y);
}

// shared-memory window: u16 counters packed two per u32 word (a CTA holds < 65536
// particles, so a per-CTA cell count cannot overflow its half-word)
template <int MODE, int K, bool WTH, bool HSM>
__global__ void __launch_bounds__(NT, MODE == MODE_REF ? GC_REF_MIN_CTAS : (MODE == MODE_GEN ? GC_GEN_MIN_CTAS : GC_PROD_MIN_CTAS)) k_predict(const KParams P) {
    extern __shared__ __align__(16) unsigned char smem_dyn[];
    __shared__ SmemTabs S;
    // the factorised sampler keeps particles in grid units u = (x - origin) / res: the
    // cell is floor(u), and the utility is rescaled (k -> k res) so the weights are unchanged
    constexpr bool SYM = MODE == MODE_FACTS || MODE == MODE_FACTS_QG;  // standard heading set
    constexpr bool GRIDU = !GC_WORLD_CELLS && (MODE == MODE_FACT || SYM);
    const int tid = threadIdx.x;
    const int h = blockIdx.x / P.ctas_per_human;
    const int blk = blockIdx.x - h * P.ctas_per_human;
    const int tsel = __ldg(&P.table_id[h]);
    if (tsel < 0 || tsel >= P.n_tables) {  // uniform over the CTA, before any write
        if (threadIdx.x == 0 && P.error) atomicOr(P.error, GC_ERRBIT_TABLE_ID);
        return;
    }
    const KTable &T = P.tab[tsel];
    const int h0 = __ldg(&P.hyp_off[h]);
    const int nh = __ldg(&P.hyp_off[h + 1]) - h0;
    // 1..MAXH hypotheses per human (the shared tables' size): a human outside that range
    // is not predicted and the launch reports it (uniform over the CTA, before any write)
    if (nh < 1 || nh > MAXH) {
        if (tid == 0 && P.error) atomicOr(P.error, GC_ERRBIT_HYPOTHESES);
        return;
    }

    // ---- stage tables in shared memory ----
    if (tid == 0) {
        S.n_hyp = nh; S.m_keep = T.m_keep; S.q_kind = T.q_kind; S.n_speeds = T.n_speeds;
        S.ref_rows = max(0, min(T.grid_rows, T.m_keep / 24));  // any caller value stays in the table
        S.wth = T.w_th * 1.4426950408889634f;
    }
    SmemAct &A = *reinterpret_cast<SmemAct *>(smem_dyn + P.act_off);
    // MODE_FACTS with w_th != 0: per-hypothesis heading weights H_b = exp(-beta w_th th_b^2)
    // in CDF slot order (MAXH x NBF floats, in place of the unused SmemAct rows)
    float *Htab = reinterpret_cast<float *>(smem_dyn + P.act_off);
    if (MODE != MODE_FACT && !SYM) {
        for (int k = tid; k < T.m_keep; k += NT) {
            const int j = __ldg(&T.keep[k]);
            A.ax[k] = __ldg(&T.sx[j]);
            A.ay[k] = __ldg(&T.sy[j]);
            if (MODE == MODE_REF || MODE == MODE_GEN) {
                float *axyf = reinterpret_cast<float *>(A.axy);
                axyf[(k >> 1) * 4 + (k & 1)] = A.ax[k];
                axyf[(k >> 1) * 4 + 2 + (k & 1)] = A.ay[k];
            }
            A.aat[k] = (T.q_kind == GC_Q_DEFAULT) ? __ldg(&T.pen[j]) : __ldg(&T.at[j]);
            A.adx[k] = __ldg(&T.dispx[j]);
            A.ady[k] = __ldg(&T.dispy[j]);
        }
        if (MODE == MODE_GEN) {  // the logit bound of gen_fast_spec: max |s_k|, min at_k
            __syncthreads();
            if (tid < 32) {
                float sm = 0.f, am = __int_as_float(0x7f800000);
                for (int k = tid; k < T.m_keep; k += 32) {
                    sm = fmaxf(sm, fmaf(A.ax[k], A.ax[k], A.ay[k] * A.ay[k]));
                    am = fminf(am, A.aat[k]);
                }
                for (int o = 16; o; o >>= 1) {
                    sm = fmaxf(sm, __shfl_xor_sync(0xffffffffu, sm, o));
                    am = fminf(am, __shfl_xor_sync(0xffffffffu, am, o));
                }
                if (tid == 0) { S.gsmax = sqrtf(sm) * 1.0001f; S.gatmin = am; }
            }
        }
    } else {
        // MODE_FACTS stores headings in the cumulative order of fact_step_sym (slot i holds
        // heading 2(i>>2) + (i&1) + 12((i>>1)&1); its (cos, sin) slot the forward heading's)
        auto hslot = [](int i) { return SYM ? 2 * (i >> 2) + (i & 1) + 12 * ((i >> 1) & 1) : i; };
        for (int i = tid; i < NBF; i += NT) {
            const int f = SYM ? 2 * (i >> 2) + (i & 1) : i;
            S.hcs[i] = make_float2(P.hcos[f], P.hsin[f]);
        }
        for (int i = tid; i < NAF * NBF; i += NT) {
            const int a = i / NBF;
            const int ib = a * NBF + hslot(i - a * NBF);
            const int j = (a > 0 && a < T.n_speeds) ? __ldg(&T.a_index[ib]) : -1;  // a = 0: stay
            const float2 d = j >= 0 ? make_float2(__ldg(&T.dispx[j]), __ldg(&T.dispy[j])) : make_float2(0.f, 0.f);
            S.fd[i] = GRIDU ? make_float2(__fdiv_rn(d.x, P.res), __fdiv_rn(d.y, P.res)) : d;
        }
        if (SYM && WTH) {
            // same expression as the stay mass sum_b H_b below, so the CDF and Z0 agree
            for (int i = tid; i < nh * NBF; i += NT) {
                const int hh = i / NBF, q = hslot(i - hh * NBF);
                Htab[i] = exp2f(-T.w_th * __ldg(&P.beta32[h0 + hh]) * P.hth2[q] * 1.4426950408889634f);
            }
        }
    }
    bool qg_ok = true;  // MODE_FACTS: top-speed normalisation representable for every hypothesis
    for (int i = tid; i < nh; i += NT) {
        const float b = __ldg(&P.beta32[h0 + i]);
        S.hb[i] = b;
        S.hgx[i] = __ldg(&P.goal32[2 * (h0 + i)]);
        S.hgy[i] = __ldg(&P.goal32[2 * (h0 + i) + 1]);
        if (MODE == MODE_FACT || SYM) {
            const float L2E = 1.4426950408889634f;
            // goal and utility slope in the particles' units (world, or grid units when GRIDU)
            S.hp[i] = GRIDU ? make_float4(__fdiv_rn(S.hgx[i] - P.ox, P.res), __fdiv_rn(S.hgy[i] - P.oy, P.res),
                                          2.f * b * T.tau * T.dv * L2E * P.res,
                                          b * (T.tau * T.tau + T.w_v) * T.dv * T.dv * L2E)
                            : make_float4(S.hgx[i], S.hgy[i], 2.f * b * T.tau * T.dv * L2E,
                                          b * (T.tau * T.tau + T.w_v) * T.dv * T.dv * L2E);
            float sh = 0.f;
            for (int q = 0; q < T.n_headings; ++q)
                sh += (T.w_th != 0.f) ? exp2f(-T.w_th * b * P.hth2[q] * 1.4426950408889634f) : 1.f;
            S.hq[i] = make_float4(0.f, 0.f, S.hp[i].w, sh);
            if (SYM) {
                // speed weights relative to the top speed (fact_step_sym): powers of 2^c
                const double c = S.hp[i].w;
                const int top = T.n_speeds - 1;
                const double ka = top == 3 ? exp2(5.0 * c) : (top == 2 ? exp2(3.0 * c) : sh * exp2(c));
                const double kb = top == 3 ? exp2(8.0 * c) : (top == 2 ? sh * exp2(4.0 * c) : 0.0);
                const double kc = top == 3 ? sh * exp2(9.0 * c) : 0.0;
                qg_ok = qg_ok && ka < 0x1p100 && kb < 0x1p100 && kc < 0x1p100;
                S.hp[i].w = (float)ka;
                S.hq[i].x = (float)kb;
                S.hq[i].y = (float)kc;
            }
        }
    }
    if (tid == 0) {
        if (P.cdf) {
            for (int i = 0; i < nh; ++i) S.cdf[i] = P.cdf[h0 + i];
        } else {
            double c = 0.0;
            for (int i = 0; i < nh; ++i) { c += exp(P.log_w[h0 + i]); S.cdf[i] = c; }
            S.cdf[nh - 1] = 1.0;
        }
    }
    unsigned *win = reinterpret_cast<unsigned *>(smem_dyn);
    int words = 0;  // window capacity (u32 words)
    if (HSM) {
        // the largest window of THIS launch's steps (a horizon chunk may fit in shared
        // memory when the whole horizon does not): the host sized it from max_win_cells
        const int R = __ldg(&P.step_r[P.t_end - 2]);
        words = ((2 * R + 1) * (2 * R + 1) + 1) >> 1;
        // the window is sized here from step_r and on the host from max_win_cells: a
        // caller that under-reported max_win_cells gets an error bit, never an overrun
        if (words + 1 > P.win_cap_words) {
            if (tid == 0 && P.error) atomicOr(P.error, GC_ERRBIT_WINDOW_CAPACITY);
            return;
        }
        // + one sink word that lanes without a cell add to (branch-free add; never flushed)
        for (int i = tid; i <= words; i += NT) win[i] = 0u;
        GC_DCHECK(((words + 1 + 3) & ~3) * 4 <= P.dyn_smem);
    }
    const bool qg = __syncthreads_and(qg_ok) != 0;
    // the caller's assume_qg does not hold for this human: the launch reports it (the mirror
    // raises; the human's counts are not valid).  No early return: the extra exit path made
    // ptxas spill in the step loop (108 B, and most of the gain gone)
    if (MODE == MODE_FACTS_QG && !qg && tid == 0 && P.error) atomicOr(P.error, GC_ERRBIT_ASSUME_QG);

    // ---- particles: hypothesis draw + start state ----
    const float sx0 = __ldg(&P.start_xy[2 * h]), sy0 = __ldg(&P.start_xy[2 * h + 1]);
    int cx, cy;
    cell_ref(sx0, sy0, P, cx, cy);
    const unsigned long long seed = __ldg(&P.seed[h]);
    const unsigned sk_lo = (unsigned)seed, sk_hi = (unsigned)(seed >> 32);
    const unsigned sid = P.stream_id ? __ldg(&P.stream_id[h]) : (unsigned)h;
    // production streams: Philox4x32-10 under a fixed key; (seed, human stream) live in
    // the counter's upper words, so the key schedule folds into immediates
    const unsigned sc2 = sk_lo ^ (sid * 0x85EBCA77u);
    SSPool pool_pre;
    if (MODE == MODE_REF) {
        pool_pre = ss_pool_init(seed);
        const int plen = __ldg(&P.prefix_len[h]);
        for (int i = 0; i < plen; ++i) ss_absorb(pool_pre, __ldg(&P.prefix[4 * h + i]));
    }

    float px[K], py[K];
    int ph[K];
    const int pbase = blk * P.ppc;
    {
        uint64_t hk0 = 0, hk1 = 0;
        if (MODE == MODE_REF && !P.hyp_in && !P.hyp_u) {
            SSPool s = pool_pre;
            ss_absorb(s, 0u);  // HYPOTHESIS_DRAWS namespace (rng.py:19)
            ss_key(s, hk0, hk1);
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int p = pbase + tid * K + k;
            px[k] = GRIDU ? __fdiv_rn(sx0 - P.ox, P.res) : sx0;
            py[k] = GRIDU ? __fdiv_rn(sy0 - P.oy, P.res) : sy0;
            ph[k] = 0;
            if (p >= P.n || tid * K + k >= P.ppc) {
                // padded slot: it steps (no divergence) but never counts; give it a valid
                // hypothesis so it reads defined tables (found by the GC_CHECKED build)
                S.phyp[k * NT + tid] = 0;
                continue;
            }
            if (P.t_begin > 1) {  // resume a chunked horizon
                const long long g = (long long)h * P.n + p;
                const float2 st = P.state_xy[g];
                px[k] = st.x; py[k] = st.y;
                ph[k] = P.state_hyp[g];
                S.phyp[k * NT + tid] = (unsigned char)ph[k];
                continue;
            }
            int hi;
            if (P.hyp_in) {
                hi = __ldg(&P.hyp_in[(long long)h * P.n + p]);
            } else {
                double u;
                if (P.hyp_u) u = __ldg(&P.hyp_u[(long long)h * P.n + p]);
                else if (MODE == MODE_REF) u = philox64_f64(hk0, hk1, (uint64_t)(p + P.p_offset));
                else {
                    const U4 o = philox4x32(U4{(unsigned)(p + P.p_offset), 0xFFFFFFFFu, sc2, sk_hi ^ 0x5EEDu}, PHK0, PHK1);
                    u = ((double)(o.x >> 5) * 67108864.0 + (double)(o.y >> 6)) * (1.0 / 9007199254740992.0);
                }
                hi = 0;
                for (int i = 0; i < nh; ++i) hi += (S.cdf[i] <= u) ? 1 : 0;  // searchsorted right
                hi = hi < nh - 1 ? hi : nh - 1;
            }
            ph[k] = hi;
            S.phyp[k * NT + tid] = (unsigned char)hi;
            if (P.hyp_out) P.hyp_out[(long long)h * P.n + p] = hi;
        }
    }
    // bit k: particle slot k holds a particle (padded slots of a CTA's last block step but
    // never count) -- one register instead of a per-step recomputation
    unsigned vmask = 0u;
#pragma unroll
    for (int k = 0; k < K; ++k) vmask |= (pbase + tid * K + k < P.n && tid * K + k < P.ppc) ? (1u << k) : 0u;
    SSPool pool_step;
    if (MODE == MODE_REF) { pool_step = pool_pre; ss_absorb(pool_step, 1u); }  // STEP_DRAWS

    const long long hbase = (long long)h * P.human_stride;
    bool overflow = false;  // a particle outside its reachable window (reported once at exit)
    if constexpr (MODE == MODE_REF) {
        // Reference arithmetic: one copy of the step code for the K particle slots (a
        // runtime slot loop; positions and first-touch words in shared memory) -- the
        // per-particle step is long (filter + exact fallback), so the K-fold unrolled form
        // overflowed the instruction cache and held 121 registers.
        SmemRefState &RS = *reinterpret_cast<SmemRefState *>(smem_dyn + P.ref_off);
#pragma unroll
        for (int k = 0; k < K; ++k) RS.pos[k * NT + tid] = make_float2(px[k], py[k]);
        // the thread's K particles are consecutive and aligned to K (ppc, p_offset % 4 == 0),
        // so their numpy float32 draws j0 .. j0 + K - 1 of the 1024-particle chunk stream are
        // u32 halves of words (j0 >> 1) .. of ONE Philox4x64 block: one block per thread-step
        const int pg0 = pbase + tid * K + P.p_offset;
        const int j0 = pg0 & 1023;
        // K = 4: the 8 draws of one Philox4x64 block feed the particles of two adjacent
        // threads (lanes 2m, 2m + 1 when the CTA's first particle is 8-aligned).  Instead of
        // both computing it every step, the pair takes turns: at the first step of every
        // step pair the even lane computes step t's block and the odd lane step t + 1's, and
        // each hands the other the two words it needs by shuffle -- one block and one key
        // derivation per lane per two steps.  The draws are unchanged (bit-identical).
        const bool turns = K == 4 && !P.uniforms && ((pbase + P.p_offset) & 7) == 0;
        const bool qodd = (tid & 1) != 0;
        uint64_t tb[4] = {0, 0, 0, 0};  // turns: this lane's block (step t or t + 1)
        for (int t = P.t_begin; t < P.t_end; ++t) {
            const int R = __ldg(&P.step_r[t - 1]);
            const int x0 = max(0, cx - R), x1 = min(P.grid_w - 1, cx + R);
            const int y0 = max(0, cy - R), y1 = min(P.grid_h - 1, cy + R);
            const int ww = x1 - x0 + 1, wh = y1 - y0 + 1;
            unsigned *gcount = P.counts + hbase + __ldg(&P.step_off[t - 1]);
            GC_DCHECK(__ldg(&P.step_off[t - 1]) + (long long)ww * wh <= P.human_stride);
            uint64_t blkw[4] = {0, 0, 0, 0};
            uint64_t w01[2] = {0, 0};  // K = 4: this thread's two words of step t's block
            if (turns) {
                if (((t - P.t_begin) & 1) == 0) {
                    SSPool s = pool_step;
                    ss_absorb(s, (unsigned)(qodd ? t + 1 : t));
                    ss_absorb(s, (unsigned)(pg0 >> 10));
                    uint64_t sk0, sk1;
                    ss_key(s, sk0, sk1);
                    philox4x64((uint64_t)(j0 >> 3) + 1, sk0, sk1, tb);
                    const uint64_t x2 = __shfl_xor_sync(0xffffffffu, tb[2], 1);
                    const uint64_t x3 = __shfl_xor_sync(0xffffffffu, tb[3], 1);
                    w01[0] = qodd ? x2 : tb[0];
                    w01[1] = qodd ? x3 : tb[1];
                } else {
                    const uint64_t y0 = __shfl_xor_sync(0xffffffffu, tb[0], 1);
                    const uint64_t y1 = __shfl_xor_sync(0xffffffffu, tb[1], 1);
                    w01[0] = qodd ? tb[2] : y0;
                    w01[1] = qodd ? tb[3] : y1;
                }
            } else if (!P.uniforms) {
                SSPool s = pool_step;
                ss_absorb(s, (unsigned)t);
                ss_absorb(s, (unsigned)(pg0 >> 10));
                uint64_t sk0, sk1;
                ss_key(s, sk0, sk1);
                philox4x64((uint64_t)(j0 >> 3) + 1, sk0, sk1, blkw);
                if (K == 4) {
                    const int w = (j0 >> 1) & 3;  // 0 or 2
                    w01[0] = w == 0 ? blkw[0] : blkw[2];
                    w01[1] = w == 0 ? blkw[1] : blkw[3];
                }
            }
#pragma unroll 1
            for (int k = 0; k < K; ++k) {
                const int p = pbase + tid * K + k;
                const bool valid = p < P.n && tid * K + k < P.ppc;
                int local = -1;
                if (valid) {
                    float2 xy = RS.pos[k * NT + tid];
                    float u;
                    if (P.uniforms) {
                        u = __ldg(&P.uniforms[((long long)h * P.steps + (t - 1)) * P.n + p]);
                    } else if (K == 4) {  // draw j0 + k: half k & 1 of the thread's word k >> 1
                        const uint64_t wd = (k >> 1) ? w01[1] : w01[0];
                        const uint32_t u32 = (k & 1) ? (uint32_t)(wd >> 32) : (uint32_t)wd;
                        u = (float)(u32 >> 8) * (1.0f / 16777216.0f);  // random(dtype=float32)
                    } else {
                        const int j = j0 + k, w = (j >> 1) & 3;
                        const uint64_t wd = w == 0 ? blkw[0] : (w == 1 ? blkw[1] : (w == 2 ? blkw[2] : blkw[3]));
                        const uint32_t u32 = (j & 1) ? (uint32_t)(wd >> 32) : (uint32_t)wd;
                        u = (float)(u32 >> 8) * (1.0f / 16777216.0f);  // random(dtype=float32)
                    }
                    const int a = ref_pick(S, A, xy.x, xy.y, S.phyp[k * NT + tid], u, P.ref_filter != 0,
                                           P.ref_fallbacks);
                    xy.x = __fadd_rn(xy.x, A.adx[a]);
                    xy.y = __fadd_rn(xy.y, A.ady[a]);
                    RS.pos[k * NT + tid] = xy;
                    int ix, iy;
                    cell_ref(xy.x, xy.y, P, ix, iy);
                    const int lx = ix - x0, ly = iy - y0;
                    if (lx < 0 || lx >= ww || ly < 0 || ly >= wh) overflow = true;
                    else local = ly * ww + lx;
                }
                if (HSM) {
                    const bool has = local >= 0;
                    const unsigned off = has ? 2u * (unsigned)local : 4u * (unsigned)words;
                    GC_DCHECK(!has || (local < ww * wh && (int)(off >> 2) < words));
                    const unsigned old = atomicAdd(reinterpret_cast<unsigned *>(reinterpret_cast<char *>(win) + (off & ~3u)),
                                                   (off & 2u) ? 0x10000u : 1u);
                    RS.fwr[k * NT + tid] = (has && old == 0u) ? (local >> 1) : -1;
                } else {
                    const unsigned same = __match_any_sync(0xffffffffu, local);
                    if (local >= 0 && (int)(tid & 31) == __ffs(same) - 1) {
                        GC_DCHECK(local < ww * wh);
                        atomicAdd(&gcount[local], (unsigned)__popc(same));
                    }
                }
            }
            if (HSM) {
                __syncthreads();
#pragma unroll 1
                for (int k = 0; k < K; ++k) {
                    const int wi = RS.fwr[k * NT + tid];
                    if (wi < 0) continue;
                    GC_DCHECK(wi < words);
                    const unsigned w = win[wi];
                    win[wi] = 0u;
                    const unsigned lo = w & 0xFFFFu, hi = w >> 16;
                    GC_DCHECK(2 * wi + (hi ? 1 : 0) < ww * wh);
                    if (lo) atomicAdd(&gcount[2 * wi], lo);
                    if (hi) atomicAdd(&gcount[2 * wi + 1], hi);
                }
                __syncthreads();
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const float2 q = RS.pos[k * NT + tid];
            px[k] = q.x; py[k] = q.y;
        }
    } else {
    // the production step loop, instantiated twice for the standard heading set: once for
    // CTAs whose table has the 4 speeds of ControlSet.grid (no speed-count selects), once
    // for the rest (2 or 3 speeds, e.g. mask_stationary's table) -- CTA-uniform choice
    auto prod_loop = [&](auto na4_tag) {
    constexpr bool NA4 = decltype(na4_tag)::value;
    const float yres = recip_nr(P.res);  // production cell map: the quotient's reciprocal
    U4 rbk = U4{0u, 0u, 0u, 0u};  // K < 4: the block this lane drew for its turn (see below)
    for (int t = P.t_begin; t < P.t_end; ++t) {
        const int R = __ldg(&P.step_r[t - 1]);
        const int x0 = max(0, cx - R), x1 = min(P.grid_w - 1, cx + R);
        const int y0 = max(0, cy - R), y1 = min(P.grid_h - 1, cy + R);
        const int ww = x1 - x0 + 1, wh = y1 - y0 + 1;
        unsigned *gcount = P.counts + hbase + __ldg(&P.step_off[t - 1]);
        GC_DCHECK(__ldg(&P.step_off[t - 1]) + (long long)ww * wh <= P.human_stride);
        // fwr[k]: the window word particle slot k added to first this step, or -1 (this
        // thread then owns that word's flush)
        int fwr[K];
        int lcl[K];  // GC_HIST_GLOBAL: this step's window cell of each slot (-1: none)
        (void)lcl;
        // production streams: one Philox4x32-10 block per step for every 4 consecutive
        // particles (block counter: global particle index / 4, step, human stream, tag);
        // particle p takes word p % 4.  A thread's K = 4 particles are consecutive and
        // aligned, so each thread draws exactly one block per step and keeps no state.
        // With K < 4 the G = 4 / K lanes of a particle group take turns: every G steps
        // lane j of the group draws the block of step t + j, and each step the group reads
        // that step's words from the lane holding them (shuffles) -- one block per lane
        // per G steps instead of G lanes drawing the same block every step.
        U4 rb = U4{0u, 0u, 0u, 0u};
        {
            const unsigned g4 = (unsigned)((pbase + tid * K + P.p_offset) >> 2);
            if (K == 4) {
                rb = philox4x32(U4{g4, (unsigned)(t - 1), sc2, sk_hi ^ 0xA11CEu}, PHK0, PHK1);
            } else {
                constexpr int G = 4 / K;
                const int sgrp = (t - 1) % G;  // this step's offset in the group's turn
                if (sgrp == 0)
                    rbk = philox4x32(U4{g4, (unsigned)(t - 1 + (tid % G)), sc2, sk_hi ^ 0xA11CEu}, PHK0, PHK1);
                const int src = (tid & 31) - (tid % G) + sgrp;  // lane holding step t's block
                rb.x = __shfl_sync(0xffffffffu, rbk.x, src);
                rb.y = __shfl_sync(0xffffffffu, rbk.y, src);
                rb.z = __shfl_sync(0xffffffffu, rbk.z, src);
                rb.w = __shfl_sync(0xffffffffu, rbk.w, src);
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int p = pbase + tid * K + k;
            const bool valid = (vmask >> k) & 1u;
            int local = -1;
            {
                // production: padded lanes compute too (no divergence), they just do not count
                float x = px[k], y = py[k];
                // word (p % 4) of this step's block (K = 4: word k; K < 4: the thread's slice)
                const int wsel = K == 4 ? k : ((p + P.p_offset) & 3);
                const unsigned ua = wsel == 0 ? rb.x : (wsel == 1 ? rb.y : (wsel == 2 ? rb.z : rb.w));
                if (SYM) {
                    fact_step_sym<WTH, MODE == MODE_FACTS_QG, NA4>(S, P, Htab, x, y, S.phyp[k * NT + tid], u24(ua), qg);
                } else if (MODE == MODE_FACT) {
                    fact_step<WTH>(S, P, x, y, S.phyp[k * NT + tid], u24(ua));
                } else {
                    const int a = gen_sample(S, A, x, y, S.phyp[k * NT + tid], u24(ua));
                    x = __fadd_rn(x, A.adx[a]);
                    y = __fadd_rn(y, A.ady[a]);
                }
                px[k] = x; py[k] = y;
                int ix, iy;
                if (GRIDU) {
                    ix = floor_clamp(x, P.wm1f);
                    iy = floor_clamp(y, P.hm1f);
                } else {
                    cell_fast(x, y, P, yres, ix, iy);
                }
                const unsigned lx = (unsigned)(ix - x0), ly = (unsigned)(iy - y0);
                const bool inside = lx < (unsigned)ww && ly < (unsigned)wh;
                overflow |= !inside;  // padded slots are ordinary particles too: always inside
                local = (valid && inside) ? (int)(ly * ww + lx) : -1;
            }
            // the thread whose add finds a window word zero owns that word's flush this
            // step: it remembers the word in a register (no list, no ballot)
            if (HSM) {
                // u16 counter `local`: byte offset 2 local, in word (2 local) & ~3; a lane
                // without a cell (padding) adds to the sink word instead -- no branch
                const bool has = local >= 0;
                const unsigned off = has ? 2u * (unsigned)local : 4u * (unsigned)words;
                GC_DCHECK(!has || (local < ww * wh && (int)(off >> 2) < words));
                const unsigned old = atomicAdd(reinterpret_cast<unsigned *>(reinterpret_cast<char *>(win) + (off & ~3u)),
                                               (off & 2u) ? 0x10000u : 1u);
                fwr[k] = (has && old == 0u) ? (local >> 1) : -1;
            } else {
                lcl[k] = local;  // counted after the slot loop (below)
            }
        }
        if (!HSM) {
            // global-histogram path (GC_HIST_GLOBAL): the lanes of a warp adding to the same
            // cell this step combine into one reduction (coherent particle clouds would
            // otherwise serialise on the same L2 addresses); the K matches are issued back
            // to back so their latencies overlap (1.3 % faster than matching each slot as
            // it is sampled)
            unsigned same[K];
#pragma unroll
            for (int k = 0; k < K; ++k) same[k] = __match_any_sync(0xffffffffu, lcl[k]);
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (lcl[k] >= 0 && (int)(tid & 31) == __ffs(same[k]) - 1) {
                    GC_DCHECK(lcl[k] < ww * wh);
                    atomicAdd(&gcount[lcl[k]], (unsigned)__popc(same[k]));
                }
            }
        }
        if (HSM) {
            __syncthreads();
            // flush only the touched words, each by its first toucher: one global
            // reduction per nonzero cell, then the word is zeroed for the next step
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int wi = fwr[k];
                if (wi < 0) continue;
                GC_DCHECK(wi < words);
                const unsigned w = win[wi];
                win[wi] = 0u;
                const unsigned lo = w & 0xFFFFu, hi = w >> 16;
                GC_DCHECK(2 * wi + (hi ? 1 : 0) < ww * wh);
                if (lo) atomicAdd(&gcount[2 * wi], lo);
                if (hi) atomicAdd(&gcount[2 * wi + 1], hi);
            }
            __syncthreads();
        }
    }
    };
    if constexpr (SYM) {
        if (S.n_speeds == 4) prod_loop(std::true_type{});
        else prod_loop(std::false_type{});
    } else {
        prod_loop(std::false_type{});
    }
    }  // production step loop
    if (overflow && P.error) atomicOr(P.error, GC_ERRBIT_WINDOW_OVERFLOW);
    if (P.t_end <= P.steps && P.state_xy) {  // hand the particles to the next chunk
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int p = pbase + tid * K + k;
            if ((vmask >> k) & 1u) {
                const long long g = (long long)h * P.n + p;
                P.state_xy[g] = make_float2(px[k], py[k]);
                P.state_hyp[g] = (unsigned char)ph[k];
            }
        }
    }
    if (P.xy_out) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int p = pbase + tid * K + k;
            if ((vmask >> k) & 1u) {
                P.xy_out[((long long)h * P.n + p) * 2] = GRIDU ? fmaf(px[k], P.res, P.ox) : px[k];
                P.xy_out[((long long)h * P.n + p) * 2 + 1] = GRIDU ? fmaf(py[k], P.res, P.oy) : py[k];
            }
        }
    }
}

#ifdef GC_PREDICT_REF_TU
// ---- one explicit propagate_step (prediction.py:165-211) ------------------------------
__global__ void __launch_bounds__(NT) k_propagate_step(float *xy, const int *hyp, int n,
                                                       const float *beta32, const float *goal32,
                                                       int n_hyp, KTable T, const float *u01,
                                                       unsigned long long seed, unsigned p0,
                                                       unsigned p1, unsigned p2, unsigned p3,
                                                       int plen, int step) {
    __shared__ SmemTabs S;
    __shared__ SmemAct A;
    const int tid = threadIdx.x;
    if (tid == 0) { S.m_keep = T.m_keep; S.q_kind = T.q_kind; }
    for (int k = tid; k < T.m_keep; k += NT) {
        const int j = T.keep[k];
        A.ax[k] = T.sx[j]; A.ay[k] = T.sy[j];
        A.aat[k] = (T.q_kind == GC_Q_DEFAULT) ? T.pen[j] : T.at[j];
        A.adx[k] = T.dispx[j]; A.ady[k] = T.dispy[j];
    }
    for (int i = tid; i < n_hyp; i += NT) {
        S.hb[i] = beta32[i]; S.hgx[i] = goal32[2 * i]; S.hgy[i] = goal32[2 * i + 1];
    }
    __syncthreads();
    const int p = blockIdx.x * NT + tid;
    if (p >= n) return;
    float u;
    if (u01) {
        u = u01[p];
    } else {
        SSPool s = ss_pool_init(seed);
        const unsigned pre[4] = {p0, p1, p2, p3};
        for (int i = 0; i < plen; ++i) ss_absorb(s, pre[i]);
        ss_absorb(s, 1u);
        ss_absorb(s, (unsigned)step);
        ss_absorb(s, (unsigned)(p >> 10));
        uint64_t k0, k1;
        ss_key(s, k0, k1);
        u = philox64_f32(k0, k1, (uint64_t)(p & 1023));
    }
    const float x = xy[2 * p], y = xy[2 * p + 1];
    const int a = ref_pick(S, A, x, y, hyp[p], u);
    xy[2 * p] = __fadd_rn(x, A.adx[a]);
    xy[2 * p + 1] = __fadd_rn(y, A.ady[a]);
}

#endif  // GC_PREDICT_REF_TU

#ifndef GC_PREDICT_REF_TU
// ---- sample_hypotheses (prediction.py:124-131) ----------------------------------------
__global__ void k_sample_hyp(const double *cdf, int n_hyp, int n, uint64_t k0, uint64_t k1, int *out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const double u = philox64_f64(k0, k1, (uint64_t)p);
    int hi = 0;
    for (int i = 0; i < n_hyp; ++i) hi += (cdf[i] <= u) ? 1 : 0;
    out[p] = hi < n_hyp - 1 ? hi : n_hyp - 1;
}
#endif

static KTable to_ktable(const gc_action_table &a) {
    KTable t;
    t.m = a.m; t.m_keep = a.m_keep; t.q_kind = a.q_kind; t.n_speeds = a.n_speeds;
    t.grid_rows = a.ref_grid_rows;
    t.n_headings = a.n_headings; t.dv = a.dv; t.tau = a.tau; t.w_v = a.w_v; t.w_th = a.w_th;
    t.sx = a.d_sx; t.sy = a.d_sy; t.at = a.d_at; t.pen = a.d_pen; t.dispx = a.d_dispx;
    t.dispy = a.d_dispy; t.keep = a.d_keep; t.a_index = a.d_a_index;
    return t;
}

template <int MODE, int K, bool WTH, bool HSM>
gc_status launch_predict(const KParams &P, int grid, size_t smem, cudaStream_t st) {
    auto fn = k_predict<MODE, K, WTH, HSM>;
    // function attributes are per device context: raise the dynamic limit once per device
    // (bit d of the mask; concurrent first calls may both set it, which is harmless)
    static std::atomic<unsigned long long> configured{0ull};
    int dev = 0;
    GC_CUDA(cudaGetDevice(&dev));
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(configured.load(std::memory_order_acquire) & bit)) {
        const int extra = (int)(sizeof(SmemAct) > (size_t)MAXH * NBF * 4 ? sizeof(SmemAct) : (size_t)MAXH * NBF * 4);
        GC_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     64 * 1024 + extra + (MODE == MODE_REF ? (int)sizeof(SmemRefState) : 0)));
        configured.fetch_or(bit, std::memory_order_acq_rel);
    }
    fn<<<grid, NT, smem, st>>>(P);
    count_launch();
    return cuda_check(cudaGetLastError(), "k_predict launch");
}

// The reference-arithmetic kernels (MODE_REF, k_propagate_step) are compiled in their own
// translation unit, gc_predict_ref.cu, with --fmad=false: ptxas otherwise contracts a
// packed mul.rn.f32x2 feeding an add.rn.f32x2 into one FFMA2 (single rounding), which
// would break numpy's bit-exact arithmetic; the production kernels keep contraction.
#ifdef GC_PREDICT_REF_TU
template gc_status launch_predict<MODE_REF, 1, false, false>(const KParams &, int, size_t, cudaStream_t);
template gc_status launch_predict<MODE_REF, 1, false, true>(const KParams &, int, size_t, cudaStream_t);
template gc_status launch_predict<MODE_REF, 2, false, false>(const KParams &, int, size_t, cudaStream_t);
template gc_status launch_predict<MODE_REF, 2, false, true>(const KParams &, int, size_t, cudaStream_t);
template gc_status launch_predict<MODE_REF, 4, false, false>(const KParams &, int, size_t, cudaStream_t);
template gc_status launch_predict<MODE_REF, 4, false, true>(const KParams &, int, size_t, cudaStream_t);
#else
extern template gc_status launch_predict<MODE_REF, 1, false, false>(const KParams &, int, size_t, cudaStream_t);
extern template gc_status launch_predict<MODE_REF, 1, false, true>(const KParams &, int, size_t, cudaStream_t);
extern template gc_status launch_predict<MODE_REF, 2, false, false>(const KParams &, int, size_t, cudaStream_t);
extern template gc_status launch_predict<MODE_REF, 2, false, true>(const KParams &, int, size_t, cudaStream_t);
extern template gc_status launch_predict<MODE_REF, 4, false, false>(const KParams &, int, size_t, cudaStream_t);
extern template gc_status launch_predict<MODE_REF, 4, false, true>(const KParams &, int, size_t, cudaStream_t);
#endif

template <int MODE, bool WTH>
static gc_status dispatch_k(const KParams &P, int K, int grid, size_t smem, cudaStream_t st) {
    // the histogram path is a template parameter: the global-histogram kernels carry no
    // window / barrier code (1.4 % faster K2 than one kernel with a runtime switch)
    if (P.smem_window) {
        switch (K) {
            case 1: return launch_predict<MODE, 1, WTH, true>(P, grid, smem, st);
            case 2: return launch_predict<MODE, 2, WTH, true>(P, grid, smem, st);
            default: return launch_predict<MODE, 4, WTH, true>(P, grid, smem, st);
        }
    }
    switch (K) {
        case 1: return launch_predict<MODE, 1, WTH, false>(P, grid, smem, st);
        case 2: return launch_predict<MODE, 2, WTH, false>(P, grid, smem, st);
        default: return launch_predict<MODE, 4, WTH, false>(P, grid, smem, st);
    }
}

}  // namespace gc

using namespace gc;

#ifndef GC_PREDICT_REF_TU
extern "C" gc_status gc_predict(const gc_predict_args *a, void *stream) {
    GC_CHECK_ARG(a != nullptr, "gc_predict: null args");
    GC_CHECK_ARG(a->n_humans >= 1 && a->n >= 1 && a->steps >= 1, "gc_predict: need n_humans, n, steps >= 1");
    GC_CHECK_ARG(a->n_tables >= 1 && a->n_tables <= 4 && a->h_tables, "gc_predict: 1..4 action tables");
    GC_CHECK_ARG(a->d_counts && a->d_step_r && a->d_step_off && a->d_start_xy && a->d_hyp_off,
                 "gc_predict: missing device buffers");
    GC_CHECK_ARG(a->d_seed && a->d_prefix && a->d_prefix_len && a->d_table_id, "gc_predict: missing rng/table ids");
    GC_CHECK_ARG(a->d_cdf || a->d_log_w || a->d_hyp_in, "gc_predict: need a cdf, log weights or hypotheses");
    GC_CHECK_ARG(a->grid_w >= 1 && a->grid_h >= 1 && a->res32 > 0.f, "gc_predict: bad grid");
    KParams P;
    memset(&P, 0, sizeof(P));
    P.n_humans = a->n_humans; P.n = a->n; P.steps = a->steps; P.rng_mode = a->rng_mode;
    P.grid_w = a->grid_w; P.grid_h = a->grid_h;
    P.ox = a->origin_x32; P.oy = a->origin_y32; P.res = a->res32; P.inv_res = 1.0f / a->res32;
    P.wm1f = (float)(a->grid_w - 1); P.hm1f = (float)(a->grid_h - 1);
    P.start_xy = a->d_start_xy; P.hyp_off = a->d_hyp_off; P.beta32 = a->d_beta32; P.goal32 = a->d_goal32;
    P.cdf = a->d_cdf; P.log_w = a->d_log_w;
    P.seed = (const unsigned long long *)a->d_seed; P.prefix = a->d_prefix; P.prefix_len = a->d_prefix_len;
    P.stream_id = a->d_stream_id;
    P.uniforms = a->rng_mode == GC_RNG_UNIFORMS ? a->d_uniforms : nullptr;
    P.hyp_u = a->rng_mode == GC_RNG_UNIFORMS ? a->d_hyp_u : nullptr;
    P.hyp_in = a->d_hyp_in;
    GC_CHECK_ARG(a->rng_mode != GC_RNG_UNIFORMS || a->d_uniforms, "gc_predict: GC_RNG_UNIFORMS needs d_uniforms");
    P.n_tables = a->n_tables; P.table_id = a->d_table_id;
    bool fact = a->rng_mode == GC_RNG_PRODUCTION;
    for (int i = 0; i < a->n_tables; ++i) {
        const gc_action_table &t = a->h_tables[i];
        if (t.m < 1 || t.m_keep < 1) { set_error("all actions are masked"); return GC_EMPTY_CONTROL_SET; }
        GC_CHECK_ARG(t.m <= MAXM && t.m_keep <= t.m, "gc_predict: at most %d actions", MAXM);
        P.tab[i] = to_ktable(t);
        const bool ok = t.n_speeds >= 2 && t.n_speeds <= NAF && t.n_headings == NBF && t.d_a_index &&
                        t.d_cos_h && (t.q_kind == GC_Q_GOAL_PROGRESS || t.q_kind == GC_Q_GOAL_PROGRESS_FULL);
        fact = fact && ok;
    }
    if (fact) {
        // every table of the launch shares the heading set (checked by the host mirror);
        // copy it into the parameter bank so the heading loop reads constant operands
        std::vector<float> c(NBF), s(NBF), th(NBF);
        const gc_action_table &t0 = a->h_tables[0];
        if (t0.h_cos_h && t0.h_sin_h && t0.h_theta_h) {
            memcpy(c.data(), t0.h_cos_h, NBF * 4);
            memcpy(s.data(), t0.h_sin_h, NBF * 4);
            memcpy(th.data(), t0.h_theta_h, NBF * 4);
        } else {
            GC_CUDA(cudaMemcpyAsync(c.data(), t0.d_cos_h, NBF * 4, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
            GC_CUDA(cudaMemcpyAsync(s.data(), t0.d_sin_h, NBF * 4, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
            GC_CUDA(cudaMemcpyAsync(th.data(), t0.d_theta_h, NBF * 4, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
            GC_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
        }
        for (int b = 0; b < NBF; ++b) { P.hcos[b] = c[b]; P.hsin[b] = s[b]; P.hth2[b] = th[b] * th[b]; }
    }
    P.step_r = a->d_step_r; P.step_off = (const long long *)a->d_step_off;
    P.human_stride = a->human_stride; P.counts = a->d_counts;
    P.hyp_out = a->d_hyp_out; P.xy_out = a->d_xy_out; P.error = a->d_error;
    P.ref_filter = a->ref_exact_only ? 0 : 1;
    P.ref_fallbacks = (unsigned long long *)a->d_ref_fallbacks;
    P.t_begin = a->t_begin > 0 ? a->t_begin : 1;
    P.t_end = a->t_end > 0 ? a->t_end : a->steps + 1;
    GC_CHECK_ARG(P.t_begin < P.t_end && P.t_end <= a->steps + 1, "gc_predict: bad step range");
    GC_CHECK_ARG((P.t_begin - 1) % 4 == 0, "gc_predict: chunk starts must be 1 + a multiple of 4");
    GC_CHECK_ARG((P.t_begin == 1 && P.t_end == a->steps + 1) || (a->d_state_xy && a->d_state_hyp),
                 "gc_predict: a chunked horizon needs particle state buffers");
    P.state_xy = (float2 *)a->d_state_xy; P.state_hyp = a->d_state_hyp;
    GC_CHECK_ARG(a->p_offset >= 0 && (long long)a->p_offset + a->n < (1ll << 31), "gc_predict: bad particle offset");
    GC_CHECK_ARG(a->p_offset % 4 == 0, "gc_predict: particle shards must start at a multiple of 4");
    P.p_offset = a->p_offset;

    // particles per thread K and particles per CTA: enough CTAs to fill 148 SMs x 3
    // resident CTAs, then grow K to amortise the per-step window flush
    const long long total = (long long)a->n_humans * a->n;
    static const int kmax = [] {
        const char *e = getenv("GC_PREDICT_MAXK");  // tuning knob (1, 2 or 4)
        const int v = e ? atoi(e) : 4;
        return v >= 4 ? 4 : (v >= 2 ? 2 : 1);
    }();
    int K = 1;
    while (K < kmax && total / ((long long)NT * K * 2) >= 4 * 148) K *= 2;
    int ppc = NT * K;
    P.ctas_per_human = (a->n + ppc - 1) / ppc;
    ppc = (a->n + P.ctas_per_human - 1) / P.ctas_per_human;  // balance the last CTA
    ppc = (ppc + 3) & ~3;  // 4-aligned: a thread's particles share one production Philox block
    P.ppc = ppc;
    const long long grid = (long long)P.ctas_per_human * a->n_humans;
    GC_CHECK_ARG(grid < (1ll << 31), "gc_predict: too many particles");
    const size_t win_bytes = (size_t)(((a->max_win_cells + 1) / 2 + 1 + 3) & ~3) * 4;  // + sink word
    // GC_HIST_SMEM: shared-memory windows when they fit; GC_HIST_GLOBAL (default): warp-
    // aggregated reductions straight into the count windows.  GC_PREDICT_GLOBAL_HIST=1
    // forces the global form for any launch (tuning knob).
    static const int force_global = [] { const char *e = getenv("GC_PREDICT_GLOBAL_HIST"); return e ? atoi(e) : 0; }();
    GC_CHECK_ARG(a->hist_path == GC_HIST_GLOBAL || a->hist_path == GC_HIST_SMEM, "gc_predict: unknown hist_path");
    P.smem_window = (a->hist_path == GC_HIST_SMEM && win_bytes <= 64 * 1024 && !force_global) ? 1 : 0;
    P.win_cap_words = (int)(win_bytes / 4);
    P.act_off = P.smem_window ? (int)((win_bytes + 15) & ~(size_t)15) : 0;  // 16-byte aligned rows
    const bool needs_act = a->rng_mode != GC_RNG_PRODUCTION || !fact;
    bool wth = false;
    for (int i = 0; i < a->n_tables; ++i) wth = wth || a->h_tables[i].w_th != 0.f;
    bool stdh = fact;
    for (int b = 0; stdh && b < NBF; ++b) stdh = P.hcos[b] == hStdCos[b] && P.hsin[b] == hStdSin[b];
    const size_t htab = (a->rng_mode == GC_RNG_PRODUCTION && stdh && wth) ? (size_t)MAXH * NBF * 4 : 0;
    const bool refm = a->rng_mode != GC_RNG_PRODUCTION;
    P.ref_off = P.act_off + (int)sizeof(SmemAct);  // SmemAct is a multiple of 16 bytes
    const size_t smem = (size_t)P.act_off + (needs_act ? sizeof(SmemAct) : htab) + (refm ? sizeof(SmemRefState) : 0);
    P.dyn_smem = (int)smem;
    cudaStream_t st = (cudaStream_t)stream;
    const int mode = a->rng_mode == GC_RNG_PRODUCTION ? (fact ? (stdh ? MODE_FACTS : MODE_FACT) : MODE_GEN)
                                                      : MODE_REF;
    if (mode == MODE_REF) return dispatch_k<MODE_REF, false>(P, K, (int)grid, smem, st);
    if (mode == MODE_FACTS && a->assume_qg)
        return wth ? dispatch_k<MODE_FACTS_QG, true>(P, K, (int)grid, smem, st)
                   : dispatch_k<MODE_FACTS_QG, false>(P, K, (int)grid, smem, st);
    if (mode == MODE_FACTS)
        return wth ? dispatch_k<MODE_FACTS, true>(P, K, (int)grid, smem, st)  // H_b table in shared memory
                   : dispatch_k<MODE_FACTS, false>(P, K, (int)grid, smem, st);
    if (mode == MODE_FACT)
        return wth ? dispatch_k<MODE_FACT, true>(P, K, (int)grid, smem, st)
                   : dispatch_k<MODE_FACT, false>(P, K, (int)grid, smem, st);
    return dispatch_k<MODE_GEN, false>(P, K, (int)grid, smem, st);
}

#else
extern "C" gc_status gc_propagate_step(float *d_xy, const int32_t *d_hyp, int32_t n, const float *d_beta32,
                                       const float *d_goal32, int32_t n_hyp, const gc_action_table *h_table,
                                       const float *d_u01, uint64_t seed, const uint32_t *h_prefix,
                                       int32_t prefix_len, int32_t step, void *stream) {
    GC_CHECK_ARG(d_xy && d_hyp && h_table && d_beta32 && d_goal32 && n >= 1, "gc_propagate_step: bad args");
    GC_CHECK_ARG(prefix_len >= 0 && prefix_len <= 4, "gc_propagate_step: prefix of at most 4 words");
    if (h_table->m_keep < 1) { set_error("all actions are masked"); return GC_EMPTY_CONTROL_SET; }
    GC_CHECK_ARG(h_table->m <= MAXM, "gc_propagate_step: at most %d actions", MAXM);
    GC_CHECK_ARG(n_hyp >= 1 && n_hyp <= MAXH, "gc_propagate_step: 1..%d hypotheses", MAXH);
    unsigned pre[4] = {0, 0, 0, 0};
    for (int i = 0; i < prefix_len; ++i) pre[i] = h_prefix[i];
    k_propagate_step<<<(n + NT - 1) / NT, NT, 0, (cudaStream_t)stream>>>(
        d_xy, d_hyp, n, d_beta32, d_goal32, n_hyp, to_ktable(*h_table), d_u01,
        (unsigned long long)seed, pre[0], pre[1], pre[2], pre[3], prefix_len, step);
    count_launch();
    return cuda_check(cudaGetLastError(), "k_propagate_step launch");
}

#endif  // GC_PREDICT_REF_TU

#ifndef GC_PREDICT_REF_TU
extern "C" gc_status gc_sample_hypotheses(const double *d_cdf, int32_t n_hyp, int32_t n, uint64_t seed,
                                          const uint32_t *h_prefix, int32_t prefix_len, int32_t *d_out,
                                          void *stream) {
    GC_CHECK_ARG(d_cdf && d_out && n >= 1 && n_hyp >= 1, "gc_sample_hypotheses: bad args");
    SSPool s = ss_pool_init(seed);
    for (int i = 0; i < prefix_len; ++i) ss_absorb(s, h_prefix[i]);
    ss_absorb(s, 0u);
    uint64_t k0, k1;
    ss_key(s, k0, k1);
    k_sample_hyp<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(d_cdf, n_hyp, n, k0, k1, d_out);
    count_launch();
    return cuda_check(cudaGetLastError(), "k_sample_hyp launch");
}
#endif  // GC_PREDICT_REF_TU
