// gc_mppi.cu -- MPPI control update on the GPU (reference planners/mppi.py:149-243;
// SURVEY.md 8(f) row f3): N perturbed rollouts of the 4-D Dubins robot
// (agents.py:423-437), quadratic goal cost + control term + planning-interval term +
// collision penalty looked up in the device-resident blocked mask of the prediction
// stack (mppi.py:87-94), then exponential weights exp(-(S - min S)/tau) and the weighted
// perturbation average, clamped to the actuation bounds.
//
// One thread per rollout, float64 throughout (the reference is float64).  Noise is
// either supplied (the reference's own numpy streams, drawn on the host -> same
// trajectories up to libm-vs-CUDA cos/sin rounding) or generated in-register with
// Philox4x32-10 + Box-Muller (production).  The reduction is one CTA with sequential
// per-output sums (deterministic).
#include "gc_common.cuh"
#include "gc_internal.h"

namespace gc {

struct MParams {
    int N, K, quad, n_layers, W, H;
    double dt, temp, std_a, std_w, pen, a_max, w_max, v_max, ox, oy, res;
    double q[4], qf[4], r[2], z[4], goal[4];
    unsigned long long seed;
    const double *nominal, *noise_in;
    const unsigned char *blocked;
    const int *layer_of;
    double *noise_out, *costs, *controls, *weights, *diag;
};

__device__ __forceinline__ double pywrap(double th) {
    const double PI = 3.141592653589793, TWO_PI = 6.283185307179586;
    double m = fmod(th + PI, TWO_PI);
    if (m != 0.0) {
        if (m < 0.0) m += TWO_PI;
    } else {
        m = 0.0;
    }
    return m - PI;
}

__device__ __forceinline__ double state_cost(const double s[4], const double g[4], const double q[4]) {
    double d0 = s[0] - g[0], d1 = s[1] - g[1], d2 = s[2] - g[2], d3 = pywrap(s[3] - g[3]);
    return d0 * d0 * q[0] + d1 * d1 * q[1] + d2 * d2 * q[2] + d3 * d3 * q[3];
}

__global__ void k_mppi_rollouts(const MParams P) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= P.N) return;
    double s[4] = {P.z[0], P.z[1], P.z[2], P.z[3]};
    double c = 0.0;
    U4 rnd{0, 0, 0, 0};
    for (int t = 0; t < P.K; ++t) {
        double d0, d1;
        const long long o = ((long long)n * P.K + t) * 2;
        if (P.noise_in) {
            d0 = P.noise_in[o];
            d1 = P.noise_in[o + 1];
        } else {
            // Philox4x32-10 block (rollout, step) -> two standard normals (Box-Muller)
            rnd = philox4x32(U4{(unsigned)n, (unsigned)t, 0x4D505049u, 0u}, (unsigned)P.seed,
                             (unsigned)(P.seed >> 32));
            const double u1 = ((double)(rnd.x >> 5) * 67108864.0 + (double)(rnd.y >> 6) + 1.0) *
                              (1.0 / 9007199254740993.0);
            const double u2 = ((double)(rnd.z >> 5) * 67108864.0 + (double)(rnd.w >> 6)) * (1.0 / 9007199254740992.0);
            const double rad = sqrt(-2.0 * log(u1));
            double sn, cs;
            sincospi(2.0 * u2, &sn, &cs);
            d0 = rad * cs * P.std_a;
            d1 = rad * sn * P.std_w;
            if (P.noise_out) { P.noise_out[o] = d0; P.noise_out[o + 1] = d1; }
        }
        const double u0 = P.nominal[2 * t] + d0, uw = P.nominal[2 * t + 1] + d1;
        const double a = fmin(fmax(u0, -P.a_max), P.a_max);
        const double w = fmin(fmax(uw, -P.w_max), P.w_max);
        const double x1 = s[0] + s[2] * cos(s[3]) * P.dt;
        const double y1 = s[1] + s[2] * sin(s[3]) * P.dt;
        const double v1 = fmin(fmax(s[2] + a * P.dt, 0.0), P.v_max);
        const double th1 = pywrap(s[3] + w * P.dt);
        s[0] = x1; s[1] = y1; s[2] = v1; s[3] = th1;
        if (t + 1 < P.K) {
            c += state_cost(s, P.goal, P.q);
            c += P.dt * (double)(t + 1);
            c += P.quad ? (u0 * u0 * P.r[0] + uw * uw * P.r[1]) : (u0 * P.r[0] + uw * P.r[1]);
            if (P.blocked) {
                const double fx = floor((x1 - P.ox) / P.res), fy = floor((y1 - P.oy) / P.res);
                const int ix = fx < 0.0 ? 0 : (fx > (double)(P.W - 1) ? P.W - 1 : (int)fx);
                const int iy = fy < 0.0 ? 0 : (fy > (double)(P.H - 1) ? P.H - 1 : (int)fy);
                const int L = P.layer_of[t];
                if (P.blocked[((long long)L * P.H + iy) * P.W + ix]) c += P.pen;
            }
        }
    }
    c += state_cost(s, P.goal, P.qf);
    P.costs[n] = c;
}

// single CTA: min over finite costs, weights, weighted perturbation average, clamps
__global__ void __launch_bounds__(1024) k_mppi_reduce(const MParams P) {
    __shared__ double red[1024];
    const int tid = threadIdx.x;
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    double mn = INF;
    for (int n = tid; n < P.N; n += blockDim.x) {
        const double c = P.costs[n];
        if (isfinite(c)) mn = fmin(mn, c);
    }
    red[tid] = mn;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (tid < s) red[tid] = fmin(red[tid], red[tid + s]);
        __syncthreads();
    }
    const double cmin = red[0];
    __syncthreads();
    if (!(cmin < INF)) {
        if (tid == 0) P.diag[0] = -1.0;  // degenerate: all costs non-finite
        return;
    }
    double sum = 0.0;
    for (int n = tid; n < P.N; n += blockDim.x) {
        const double c = P.costs[n];
        const double w = isfinite(c) ? exp(-(c - cmin) / P.temp) : 0.0;
        P.weights[n] = w;
        sum += w;
    }
    red[tid] = sum;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (tid < s) red[tid] += red[tid + s];
        __syncthreads();
    }
    const double total = red[0];
    __syncthreads();
    for (int n = tid; n < P.N; n += blockDim.x) P.weights[n] /= total;
    __syncthreads();
    // diagnostics: best cost, mean finite cost, weight entropy
    double ent = 0.0, fin = 0.0, cnt = 0.0;
    for (int n = tid; n < P.N; n += blockDim.x) {
        const double w = P.weights[n];
        if (w > 0.0) ent -= w * log(w);
        const double c = P.costs[n];
        if (isfinite(c)) { fin += c; cnt += 1.0; }
    }
    red[tid] = ent;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (tid < s) red[tid] += red[tid + s];
        __syncthreads();
    }
    if (tid == 0) { P.diag[0] = cmin; P.diag[2] = red[0]; }
    __syncthreads();
    red[tid] = fin;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (tid < s) red[tid] += red[tid + s];
        __syncthreads();
    }
    const double fsum = red[0];
    __syncthreads();
    red[tid] = cnt;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (tid < s) red[tid] += red[tid + s];
        __syncthreads();
    }
    if (tid == 0) P.diag[1] = fsum / red[0];
}

// weighted perturbation average: one CTA per control output (t, component), fixed-tree
// reduction over rollouts, then the actuation clamp
__global__ void __launch_bounds__(256) k_mppi_average(const MParams P) {
    __shared__ double red[256];
    const int o = blockIdx.x;
    const double *noise = P.noise_in ? P.noise_in : P.noise_out;
    double acc = 0.0;
    for (int n = threadIdx.x; n < P.N; n += blockDim.x) acc += P.weights[n] * noise[(long long)n * 2 * P.K + o];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double lim = (o & 1) ? P.w_max : P.a_max;
        const double u = P.nominal[o] + red[0];
        P.controls[o] = fmin(fmax(u, -lim), lim);
    }
}

}  // namespace gc

using namespace gc;

extern "C" gc_status gc_mppi_step(const gc_mppi_args *a, void *stream) {
    GC_CHECK_ARG(a && a->n_rollouts >= 1 && a->horizon >= 1 && a->dt > 0 && a->temperature > 0,
                 "gc_mppi_step: bad config");
    GC_CHECK_ARG(a->d_nominal && a->d_costs && a->d_controls && a->d_weights && a->d_diag,
                 "gc_mppi_step: missing buffers");
    GC_CHECK_ARG(a->d_noise || a->d_noise_out, "gc_mppi_step: need supplied noise or a noise buffer");
    GC_CHECK_ARG(!a->d_blocked || (a->d_layer_of && a->n_layers >= 1 && a->grid_w >= 1 && a->grid_h >= 1),
                 "gc_mppi_step: blocked mask needs geometry and layer indices");
    MParams P;
    P.N = a->n_rollouts; P.K = a->horizon; P.quad = a->quadratic_control_cost;
    P.n_layers = a->n_layers; P.W = a->grid_w; P.H = a->grid_h;
    P.dt = a->dt; P.temp = a->temperature; P.std_a = a->std_a; P.std_w = a->std_w; P.pen = a->collision_penalty;
    P.a_max = a->a_max; P.w_max = a->omega_max; P.v_max = a->v_max;
    P.ox = a->origin_x; P.oy = a->origin_y; P.res = a->res;
    for (int i = 0; i < 4; ++i) { P.q[i] = a->q[i]; P.qf[i] = a->qf[i]; P.z[i] = a->z[i]; P.goal[i] = a->goal[i]; }
    P.r[0] = a->r[0]; P.r[1] = a->r[1];
    P.seed = a->seed; P.nominal = a->d_nominal; P.noise_in = a->d_noise; P.blocked = a->d_blocked;
    P.layer_of = a->d_layer_of; P.noise_out = a->d_noise_out; P.costs = a->d_costs; P.controls = a->d_controls;
    P.weights = a->d_weights; P.diag = a->d_diag;
    cudaStream_t st = (cudaStream_t)stream;
    k_mppi_rollouts<<<(P.N + 63) / 64, 64, 0, st>>>(P);
    k_mppi_reduce<<<1, 1024, 0, st>>>(P);
    k_mppi_average<<<2 * P.K, 256, 0, st>>>(P);
    count_launch(3);
    return cuda_check(cudaGetLastError(), "gc_mppi_step launch");
}
