// gc_belief.cu -- K1: Bayesian (beta, goal) belief update, one CTA per human (its warps
// share the hypotheses).
//
// Restates update_belief (belief.py:159-198) in float64:
//   recover_control (agents.py:355-371): v = |dz|/dt, theta = atan2 (fallback if |dz|<1e-6),
//       theta wrapped to [-pi, pi) with Python float-modulo semantics (agents.py:24-26);
//   snap (agents.py:114-120): argmin_j |v_j - v| + |wrap(theta_j - theta)|, first index on
//       ties (warp shuffle argmin over actions); > tol -> GC_SNAP_MISMATCH;
//   observation_log_likelihood (belief.py:145-156) via policy_log_table (agents.py:299-323):
//       per hypothesis the full-base utility q.table in float64 with the warp's lanes over
//       the actions (<= 8 per lane), beta *, shuffle max shift over finite logits, shuffle
//       log-sum-exp -> log pi(u_obs | z; beta, g);
//   posterior = prior + loglik, finite entries floored at -745, -inf kept (belief.py:194-197),
//       normalised by a warp-shuffle logsumexp (scipy.special.logsumexp semantics).
#include "gc_common.cuh"
#include "gc_internal.h"

namespace gc {

constexpr int BT = 256;      // one CTA (8 warps) per human
constexpr int BMAXH = 256;   // hypotheses per human (8 per lane)

struct BParams {
    int n_humans, m, q_kind, clamp;
    const double *v, *theta, *sx, *sy, *at, *pen, *qtable;
    const unsigned char *masked;
    const int *hyp_off;
    const double *beta, *goal, *obs, *fallback;
    double dt, snap_tol;
    const double *prior;
    double *post;
    int *status, *action;
};

// Python float % 2pi (fmod + sign fix), as used by wrap_angle / np.remainder
__device__ __forceinline__ double pymod(double a, double b) {
    double m = fmod(a, b);
    if (m != 0.0) {
        if ((b < 0.0) != (m < 0.0)) m += b;
    } else {
        m = copysign(0.0, b);
    }
    return m;
}
__device__ __forceinline__ double wrap_angle(double th) {
    const double PI = 3.141592653589793, TWO_PI = 6.283185307179586;
    return pymod(th + PI, TWO_PI) - PI;
}

// SPL actions per lane (m <= 32 SPL): 8 for up to 256 actions, 16 for up to GC_MAX_ACTIONS;
// the extra slots of the wider instance are empty for m <= 256 (no change in any sum's order)
template <int SPL>
__global__ void __launch_bounds__(BT) k_belief(const BParams P) {
    // one CTA per human: every warp recovers/snaps the control (identical results), then
    // warp w takes hypotheses w, w + NW, ...; warp 0 normalises from shared memory
    __shared__ double spost[BMAXH];
    __shared__ int sempty;
    const int h = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = BT / 32;
    const double PI = 3.141592653589793, TWO_PI = 6.283185307179586;
    const double NEG_INF = -__longlong_as_double(0x7ff0000000000000ll);
    if (threadIdx.x == 0) sempty = 0;

    // ---- recover_control ----
    const double zx = P.obs[4 * h], zy = P.obs[4 * h + 1];
    const double dx = P.obs[4 * h + 2] - zx, dy = P.obs[4 * h + 3] - zy;
    const double dist = hypot(dx, dy);
    double uv, uth;
    if (dist < 1e-6) { uv = 0.0; uth = wrap_angle(P.fallback[h]); }
    else { uv = dist / P.dt; uth = wrap_angle(atan2(dy, dx)); }

    // ---- snap: first argmin over actions ----
    double best = __longlong_as_double(0x7ff0000000000000ll);
    int bidx = 0x7fffffff;
    for (int j = lane; j < P.m; j += 32) {
        const double d = fabs(P.v[j] - uv) + fabs(pymod(P.theta[j] - uth + PI, TWO_PI) - PI);
        if (d < best) { best = d; bidx = j; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
        if (ob < best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
    }
    int status = GC_OK;
    if (best > P.snap_tol) {
        status = GC_SNAP_MISMATCH;
        if (!P.clamp) {  // uniform over the CTA: every warp takes this branch
            if (threadIdx.x == 0) { P.status[h] = status; if (P.action) P.action[h] = bidx; }
            return;
        }
    }
    const int idx = bidx;
    const int h0 = P.hyp_off[h], nh = P.hyp_off[h + 1] - h0;
    if (nh < 1 || nh > BMAXH) {  // shared tables hold BMAXH hypotheses (uniform over the CTA)
        if (threadIdx.x == 0) P.status[h] = GC_BAD_ARG;
        return;
    }
    // per-action tables of this lane's actions, loaded once (<= SPL per lane)
    double ax[SPL], ay[SPL], aat[SPL];
    bool amask[SPL];
#pragma unroll
    for (int s = 0; s < SPL; ++s) {
        const int j = lane + 32 * s;
        const bool ok = j < P.m;
        amask[s] = !ok || (P.masked && P.masked[j]);
        ax[s] = ok ? P.sx[j] : 0.0;
        ay[s] = ok ? P.sy[j] : 0.0;
        aat[s] = ok ? (P.q_kind == GC_Q_DEFAULT ? P.pen[j] : P.at[j]) : 0.0;
    }
    __syncthreads();  // sempty initialised

    // ---- per-hypothesis log-likelihood: lanes over actions, warp-shuffle max / sum ----
    for (int i = warp; i < nh; i += NW) {
        const double beta = P.beta[h0 + i];
        const double rx = zx - P.goal[2 * (h0 + i)];
        const double ry = zy - P.goal[2 * (h0 + i) + 1];
        const double d2 = __dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry));
        double Lj[SPL];  // m <= 32 SPL actions
        double mx = NEG_INF;
#pragma unroll
        for (int s = 0; s < SPL; ++s) {
            const int j = lane + 32 * s;
            double L = NEG_INF;
            if (!amask[s]) {
                double q;
                if (P.q_kind == GC_Q_TABLE) {
                    q = P.qtable[(long long)(h0 + i) * P.m + j];
                } else if (P.q_kind == GC_Q_DEFAULT) {
                    q = __dsub_rn(-d2, aat[s]);
                } else {
                    q = __dmul_rn(__fma_rn(ry, ay[s], __dmul_rn(rx, ax[s])), -2.0);
                    q = __dsub_rn(q, aat[s]);
                    q = __dsub_rn(q, d2);
                }
                L = __dmul_rn(beta, q);
            }
            Lj[s] = L;
            mx = fmax(mx, L);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (!(mx > NEG_INF)) {
            if (lane == 0) sempty = 1;
            continue;
        }
        double ssum = 0.0;
#pragma unroll
        for (int s = 0; s < SPL; ++s) if (Lj[s] > NEG_INF) ssum += exp(Lj[s] - mx);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
        // the observed action's logit lives in lane idx % 32, slot idx / 32
        double Lmine = NEG_INF;
#pragma unroll
        for (int s = 0; s < SPL; ++s) if (s == (idx >> 5)) Lmine = Lj[s];
        const double Li = __shfl_sync(0xffffffffu, Lmine, idx & 31);
        const double ll = (Li > NEG_INF) ? (Li - mx) - log(ssum) : NEG_INF;
        if (lane == 0) {
            const double pr = P.prior[h0 + i];
            spost[i] = (pr == NEG_INF) ? NEG_INF : fmax(pr + ll, -745.0);  // LOG_WEIGHT_FLOOR
        }
    }
    __syncthreads();
    if (warp != 0) return;
    if (sempty) {
        if (lane == 0) P.status[h] = GC_EMPTY_CONTROL_SET;
        return;
    }
    // ---- logsumexp over hypotheses ----
    double post[BMAXH / 32];
#pragma unroll
    for (int s = 0; s < BMAXH / 32; ++s) {
        const int i = lane + 32 * s;
        post[s] = i < nh ? spost[i] : NEG_INF;
    }
    double mx = NEG_INF;
#pragma unroll
    for (int s = 0; s < BMAXH / 32; ++s) mx = fmax(mx, post[s]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const double shift = (mx > NEG_INF) ? mx : 0.0;
    double ssum = 0.0;
#pragma unroll
    for (int s = 0; s < BMAXH / 32; ++s) if (post[s] > NEG_INF) ssum += exp(post[s] - shift);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
    const double lse = log(ssum) + shift;
#pragma unroll
    for (int s = 0; s < BMAXH / 32; ++s) {
        const int i = lane + 32 * s;
        if (i < nh) P.post[h0 + i] = post[s] - lse;
    }
    if (lane == 0) { P.status[h] = status; if (P.action) P.action[h] = idx; }
}

}  // namespace gc

using namespace gc;

extern "C" gc_status gc_belief_update(const gc_belief_args *a, void *stream) {
    GC_CHECK_ARG(a != nullptr, "gc_belief_update: null args");
    GC_CHECK_ARG(a->n_humans >= 1 && a->m >= 1 && a->m <= GC_MAX_ACTIONS, "gc_belief_update: 1..%d actions",
                 GC_MAX_ACTIONS);
    GC_CHECK_ARG(a->d_v && a->d_theta && a->d_hyp_off && a->d_beta && a->d_goal && a->d_obs &&
                 a->d_fallback_theta && a->d_prior && a->d_post && a->d_status,
                 "gc_belief_update: missing device buffers");
    GC_CHECK_ARG(a->dt > 0.0, "dt must be > 0");
    if (a->q_kind == GC_Q_TABLE) GC_CHECK_ARG(a->d_qtable, "gc_belief_update: GC_Q_TABLE needs d_qtable");
    else if (a->q_kind == GC_Q_DEFAULT) GC_CHECK_ARG(a->d_pen, "gc_belief_update: q_default needs d_pen");
    else GC_CHECK_ARG(a->d_sx && a->d_sy && a->d_at, "gc_belief_update: goal-progress tables missing");
    BParams P;
    P.n_humans = a->n_humans; P.m = a->m; P.q_kind = a->q_kind; P.clamp = a->clamp_on_mismatch;
    P.v = a->d_v; P.theta = a->d_theta; P.sx = a->d_sx; P.sy = a->d_sy; P.at = a->d_at; P.pen = a->d_pen;
    P.qtable = a->d_qtable; P.masked = a->d_masked; P.hyp_off = a->d_hyp_off;
    P.beta = a->d_beta; P.goal = a->d_goal; P.obs = a->d_obs; P.fallback = a->d_fallback_theta;
    P.dt = a->dt; P.snap_tol = a->snap_tol; P.prior = a->d_prior; P.post = a->d_post;
    P.status = a->d_status; P.action = a->d_action;
    if (a->m <= 256) k_belief<8><<<a->n_humans, BT, 0, (cudaStream_t)stream>>>(P);
    else k_belief<GC_MAX_ACTIONS / 32><<<a->n_humans, BT, 0, (cudaStream_t)stream>>>(P);
    count_launch();
    return cuda_check(cudaGetLastError(), "k_belief launch");
}
