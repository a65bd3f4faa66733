// gc_exact.cu -- exact enumeration of the bootstrapped prediction process on the GPU
// (reference exact_predict, prediction.py:303-377).
//
// One conditional cell distribution p_h per hypothesis (the hypothesis is frozen for the
// horizon, exactly like the particle rollout), marginalised against the belief per layer:
//   step 1 from the continuous start state:  p_h[landing0_j] += pi0[h, j]   (sequential in j,
//            the np.add.at order)
//   later steps from cell centres:          p'_h[landing[c, j]] += p_h[c] pi[h, c, j]
//   layer_t = b @ p_h
// pi = exp(policy_log_table(...)) in float64 (agents.py:299-323); the landing table maps
// cell centre + displacement through GridSpec.cells_of in float64 (occupancy.py:43-51).
// The reference caps cells*|U|*|H| at 2e6 entries because its tables live in host RAM;
// here they live in HBM (|H|*cells*m*8 bytes: 2.5 GB at 400x400, 96 actions, 20 hyps).
// The later-step scatter uses float64 atomics: sums agree with the reference to rounding.
#include "gc_common.cuh"
#include "gc_internal.h"

namespace gc {

struct XParams {
    int n_hyp, m, W, H, q_kind;
    double ox, oy, res, z0x, z0y;
    const double *beta, *goal, *belief, *sx, *sy, *at, *pen, *dispx, *dispy, *qtable, *qtable0;
    const unsigned char *masked;
    double *pi, *p, *nxt, *layers;
    int *landing;
};

__device__ __forceinline__ double q_value(const XParams &P, int j, double rx, double ry, double d2, int h,
                                          long long cell) {
    if (P.masked && P.masked[j]) return -__longlong_as_double(0x7ff0000000000000ll);
    if (P.q_kind == GC_Q_TABLE) {
        return cell < 0 ? P.qtable0[(long long)h * P.m + j]
                        : P.qtable[((long long)h * P.W * P.H + cell) * P.m + j];
    }
    if (P.q_kind == GC_Q_DEFAULT) return __dsub_rn(-d2, P.pen[j]);
    double q = __dmul_rn(__fma_rn(ry, P.sy[j], __dmul_rn(rx, P.sx[j])), -2.0);
    q = __dsub_rn(q, P.at[j]);
    return __dsub_rn(q, d2);
}

// log-softmax row of hypothesis h at state (x, y) -> pi_out[j] = exp(log pi_j)
__device__ void policy_row(const XParams &P, int h, double x, double y, long long cell, double *pi_out) {
    const double NEG_INF = -__longlong_as_double(0x7ff0000000000000ll);
    const double beta = P.beta[h];
    const double rx = x - P.goal[2 * h], ry = y - P.goal[2 * h + 1];
    const double d2 = __dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry));
    double mx = NEG_INF;
    for (int j = 0; j < P.m; ++j) {
        const double L = __dmul_rn(beta, q_value(P, j, rx, ry, d2, h, cell));
        mx = L > mx ? L : mx;
    }
    double s = 0.0;
    for (int j = 0; j < P.m; ++j) {
        const double L = __dmul_rn(beta, q_value(P, j, rx, ry, d2, h, cell));
        if (L > NEG_INF) s += exp(L - mx);
    }
    const double lse = log(s);
    for (int j = 0; j < P.m; ++j) {
        const double L = __dmul_rn(beta, q_value(P, j, rx, ry, d2, h, cell));
        pi_out[j] = (L > NEG_INF) ? exp((L - mx) - lse) : 0.0;
    }
}

__device__ __forceinline__ int cell_of64(const XParams &P, double x, double y) {
    const double fx = floor((x - P.ox) / P.res), fy = floor((y - P.oy) / P.res);
    const int ix = fx < 0.0 ? 0 : (fx > (double)(P.W - 1) ? P.W - 1 : (int)fx);
    const int iy = fy < 0.0 ? 0 : (fy > (double)(P.H - 1) ? P.H - 1 : (int)fy);
    return iy * P.W + ix;
}

__device__ __forceinline__ void centre(const XParams &P, int c, double &x, double &y) {
    const int iy = c / P.W, ix = c - iy * P.W;
    x = P.ox + ((double)ix + 0.5) * P.res;  // GridSpec.centers_x (occupancy.py:57-58)
    y = P.oy + ((double)iy + 0.5) * P.res;
}

__global__ void k_exact_tables(const XParams P) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int h = blockIdx.y;
    const int cells = P.W * P.H;
    if (c >= cells) return;
    double x, y;
    centre(P, c, x, y);
    policy_row(P, h, x, y, c, P.pi + ((long long)h * cells + c) * P.m);
    if (h == 0)
        for (int j = 0; j < P.m; ++j) P.landing[(long long)c * P.m + j] = cell_of64(P, x + P.dispx[j], y + P.dispy[j]);
}

// first transition from the continuous start state, one thread per hypothesis
__global__ void k_exact_first(const XParams P, double *pi0) {
    const int h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= P.n_hyp) return;
    double *row = pi0 + (long long)h * P.m;
    policy_row(P, h, P.z0x, P.z0y, -1, row);
    double *ph = P.p + (long long)h * P.W * P.H;
    for (int j = 0; j < P.m; ++j) ph[cell_of64(P, P.z0x + P.dispx[j], P.z0y + P.dispy[j])] += row[j];
}

__global__ void k_exact_step(const XParams P) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int h = blockIdx.y;
    const int cells = P.W * P.H;
    if (c >= cells) return;
    const double v = P.p[(long long)h * cells + c];
    if (v == 0.0) return;
    const double *pi = P.pi + ((long long)h * cells + c) * P.m;
    const int *land = P.landing + (long long)c * P.m;
    double *out = P.nxt + (long long)h * cells;
    for (int j = 0; j < P.m; ++j) {
        const double w = pi[j];
        if (w != 0.0) atomicAdd(&out[land[j]], v * w);
    }
}

__global__ void k_exact_layer(const XParams P, double *layer) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int cells = P.W * P.H;
    if (c >= cells) return;
    double s = 0.0;
    for (int h = 0; h < P.n_hyp; ++h) s += P.belief[h] * P.p[(long long)h * cells + c];
    layer[c] = s;
}

}  // namespace gc

using namespace gc;

extern "C" gc_status gc_exact_predict(const gc_exact_args *a, void *stream) {
    GC_CHECK_ARG(a && a->n_hyp >= 1 && a->m >= 1 && a->grid_w >= 1 && a->grid_h >= 1 && a->steps >= 1,
                 "gc_exact_predict: bad sizes");
    GC_CHECK_ARG(a->d_beta && a->d_goal && a->d_belief && a->d_dispx && a->d_dispy && a->d_pi && a->d_landing &&
                     a->d_p && a->d_nxt && a->d_pi0 && a->d_layers,
                 "gc_exact_predict: missing buffers");
    GC_CHECK_ARG(a->n_hyp <= 65535, "gc_exact_predict: too many hypotheses");
    XParams P;
    P.n_hyp = a->n_hyp; P.m = a->m; P.W = a->grid_w; P.H = a->grid_h; P.q_kind = a->q_kind;
    P.ox = a->origin_x; P.oy = a->origin_y; P.res = a->res; P.z0x = a->z0x; P.z0y = a->z0y;
    P.beta = a->d_beta; P.goal = a->d_goal; P.belief = a->d_belief; P.sx = a->d_sx; P.sy = a->d_sy;
    P.at = a->d_at; P.pen = a->d_pen; P.dispx = a->d_dispx; P.dispy = a->d_dispy;
    P.qtable = a->d_qtable; P.qtable0 = a->d_qtable0; P.masked = a->d_masked;
    P.pi = a->d_pi; P.p = a->d_p; P.nxt = a->d_nxt; P.layers = a->d_layers; P.landing = a->d_landing;
    cudaStream_t st = (cudaStream_t)stream;
    const int cells = a->grid_w * a->grid_h;
    const size_t pbytes = (size_t)a->n_hyp * cells * sizeof(double);
    dim3 g2((cells + 127) / 128, a->n_hyp);
    k_exact_tables<<<g2, 128, 0, st>>>(P);
    GC_CUDA(cudaMemsetAsync(a->d_p, 0, pbytes, st));
    k_exact_first<<<(a->n_hyp + 63) / 64, 64, 0, st>>>(P, a->d_pi0);
    k_exact_layer<<<(cells + 255) / 256, 256, 0, st>>>(P, a->d_layers);
    count_launch(3);
    for (int t = 1; t < a->steps; ++t) {
        GC_CUDA(cudaMemsetAsync(P.nxt, 0, pbytes, st));
        k_exact_step<<<g2, 128, 0, st>>>(P);
        double *tmp = P.p; P.p = P.nxt; P.nxt = tmp;
        k_exact_layer<<<(cells + 255) / 256, 256, 0, st>>>(P, a->d_layers + (size_t)t * cells);
        count_launch(2);
    }
    return cuda_check(cudaGetLastError(), "gc_exact_predict launch");
}
