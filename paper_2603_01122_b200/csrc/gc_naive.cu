// gc_naive.cu -- predict_naive (prediction.py:258-300): the reference's serial float64
// per-particle loop, one thread per particle, bit-for-bit its arithmetic order:
//   q.table row (agents.py:222-224; goal progress: rel @ [sx; sy] * -2 - at - |rel|^2,
//   default: -|rel|^2 - pen) over the kept actions, * beta, - max, exp, sequential
//   cumsum, j = #(cdf < u * cdf[-1]) capped at m_keep - 1, xy += disp[keep[j]];
//   u = rng.stream(seed, *prefix, 1, t, p >> 10).random() (float64, element p & 1023);
//   cell = clamp(floor((x - ox) / res)) in float64 (occupancy.py:43-51).
// The float64 exp is CUDA's (<= 1 ulp from numpy's): a decision can differ only when u
// lands within an ulp of a cdf entry.
#include "gc_common.cuh"
#include "gc_internal.h"

namespace gc {

constexpr int NB_T = 128;
constexpr int NB_MAXM = GC_MAX_ACTIONS;

struct NParams {
    int n, steps, m_keep, q_kind, grid_w, grid_h, prefix_len;
    unsigned long long seed;
    unsigned prefix[4];
    double sx0, sy0, ox, oy, res;
    const int *hyp, *keep;
    const double *beta, *goal, *sx, *sy, *at, *pen, *dispx, *dispy;
    unsigned *counts;
    double *xy_out;
};

__global__ void __launch_bounds__(NB_T) k_naive(const NParams P) {
    __shared__ double ax[NB_MAXM], ay[NB_MAXM], aat[NB_MAXM], adx[NB_MAXM], ady[NB_MAXM];
    for (int k = threadIdx.x; k < P.m_keep; k += NB_T) {
        const int j = P.keep[k];
        ax[k] = P.sx[j];
        ay[k] = P.sy[j];
        aat[k] = P.q_kind == GC_Q_DEFAULT ? P.pen[j] : P.at[j];
        adx[k] = P.dispx[j];
        ady[k] = P.dispy[j];
    }
    __syncthreads();
    const int p = blockIdx.x * NB_T + threadIdx.x;
    if (p >= P.n) return;
    const int h = P.hyp[p];
    const double beta = P.beta[h], gx = P.goal[2 * h], gy = P.goal[2 * h + 1];
    SSPool pool = ss_pool_init(P.seed);
    for (int i = 0; i < P.prefix_len; ++i) ss_absorb(pool, P.prefix[i]);
    ss_absorb(pool, 1u);  // STEP_DRAWS (rng.py:20)
    double x = P.sx0, y = P.sy0;
    const int mk = P.m_keep;
    const size_t cells = (size_t)P.grid_w * P.grid_h;
    for (int t = 1; t <= P.steps; ++t) {
        SSPool s = pool;
        ss_absorb(s, (unsigned)t);
        ss_absorb(s, (unsigned)(p >> 10));
        uint64_t k0, k1;
        ss_key(s, k0, k1);
        const double u = philox64_f64(k0, k1, (uint64_t)(p & 1023));
        const double rx = __dsub_rn(x, gx), ry = __dsub_rn(y, gy);
        const double d2 = __dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry));
        auto logit = [&](int k) -> double {
            double q;
            if (P.q_kind == GC_Q_DEFAULT) {
                q = __dsub_rn(-d2, aat[k]);
            } else {
                q = __dmul_rn(__fma_rn(ry, ay[k], __dmul_rn(rx, ax[k])), -2.0);
                q = __dsub_rn(__dsub_rn(q, aat[k]), d2);
            }
            return __dmul_rn(beta, q);
        };
        double M = logit(0);
        for (int k = 1; k < mk; ++k) M = fmax(M, logit(k));
        double c = 0.0;
        for (int k = 0; k < mk; ++k) {
            const double w = exp(__dsub_rn(logit(k), M));
            c = k == 0 ? w : __dadd_rn(c, w);
        }
        const double r = __dmul_rn(u, c);
        double cc = 0.0;
        int j = 0;
        for (; j < mk; ++j) {  // first j with cdf_j >= r  ==  #(cdf < r)
            const double w = exp(__dsub_rn(logit(j), M));
            cc = j == 0 ? w : __dadd_rn(cc, w);
            if (!(cc < r)) break;
        }
        j = j < mk - 1 ? j : mk - 1;
        x = __dadd_rn(x, adx[j]);
        y = __dadd_rn(y, ady[j]);
        const double fx = floor(__ddiv_rn(__dsub_rn(x, P.ox), P.res));
        const double fy = floor(__ddiv_rn(__dsub_rn(y, P.oy), P.res));
        const int ix = fx < 0.0 ? 0 : (fx > (double)(P.grid_w - 1) ? P.grid_w - 1 : (int)fx);
        const int iy = fy < 0.0 ? 0 : (fy > (double)(P.grid_h - 1) ? P.grid_h - 1 : (int)fy);
        atomicAdd(&P.counts[(size_t)(t - 1) * cells + (size_t)iy * P.grid_w + ix], 1u);
    }
    if (P.xy_out) {
        P.xy_out[2 * p] = x;
        P.xy_out[2 * p + 1] = y;
    }
}

}  // namespace gc

using namespace gc;

extern "C" gc_status gc_predict_naive(const gc_naive_args *a, void *stream) {
    GC_CHECK_ARG(a != nullptr, "gc_predict_naive: null args");
    GC_CHECK_ARG(a->n >= 1 && a->steps >= 1, "gc_predict_naive: n and steps must be >= 1");
    if (a->m_keep < 1) { set_error("all actions are masked"); return GC_EMPTY_CONTROL_SET; }
    GC_CHECK_ARG(a->m_keep <= NB_MAXM, "gc_predict_naive: at most %d actions", NB_MAXM);
    GC_CHECK_ARG(a->q_kind == GC_Q_GOAL_PROGRESS_FULL || a->q_kind == GC_Q_DEFAULT,
                 "gc_predict_naive: q_kind must be GC_Q_GOAL_PROGRESS_FULL or GC_Q_DEFAULT");
    GC_CHECK_ARG(a->grid_w >= 1 && a->grid_h >= 1 && a->res > 0.0, "gc_predict_naive: bad grid");
    GC_CHECK_ARG(a->prefix_len >= 0 && a->prefix_len <= 4, "gc_predict_naive: prefix of 0..4 words");
    GC_CHECK_ARG(a->d_hyp && a->d_beta && a->d_goal && a->d_keep && a->d_dispx && a->d_dispy && a->d_counts,
                 "gc_predict_naive: missing device buffers");
    if (a->q_kind == GC_Q_DEFAULT) GC_CHECK_ARG(a->d_pen, "gc_predict_naive: q_default needs d_pen");
    else GC_CHECK_ARG(a->d_sx && a->d_sy && a->d_at, "gc_predict_naive: goal-progress tables missing");
    NParams P;
    P.n = a->n; P.steps = a->steps; P.m_keep = a->m_keep; P.q_kind = a->q_kind;
    P.grid_w = a->grid_w; P.grid_h = a->grid_h; P.prefix_len = a->prefix_len;
    P.seed = a->seed;
    for (int i = 0; i < 4; ++i) P.prefix[i] = a->prefix[i];
    P.sx0 = a->start_x; P.sy0 = a->start_y; P.ox = a->origin_x; P.oy = a->origin_y; P.res = a->res;
    P.hyp = a->d_hyp; P.keep = a->d_keep; P.beta = a->d_beta; P.goal = a->d_goal;
    P.sx = a->d_sx; P.sy = a->d_sy; P.at = a->d_at; P.pen = a->d_pen;
    P.dispx = a->d_dispx; P.dispy = a->d_dispy; P.counts = a->d_counts; P.xy_out = a->d_xy_out;
    k_naive<<<(a->n + NB_T - 1) / NB_T, NB_T, 0, (cudaStream_t)stream>>>(P);
    count_launch();
    return cuda_check(cudaGetLastError(), "k_naive launch");
}
