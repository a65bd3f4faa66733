// gc_collision.cu -- collision field of occupancy layers (reference occupancy.py:195-239,
// planners/anastar.py:107-119, planners/mppi.py:87-94): for every cell, the occupancy mass
// within robot_radius of its centre, clamped to 1, optionally thresholded into the
// planners' blocked mask.
//
// The reference adds whole shifted copies of the grid in disc-offset order (dy-major,
// dx-minor), so every output cell is a sequential float64 sum over the in-grid offsets
// in that order; this kernel performs exactly that sum per cell (bit-identical), reading
// the layer through a shared-memory tile with an r-cell halo.
#include "gc_common.cuh"
#include "gc_internal.h"

namespace gc {

constexpr int CT = 32;      // output tile edge
constexpr int CNT = 256;    // threads per CTA
constexpr int CMAXR = 16;   // max radius in cells
constexpr int CMAXOFF = (2 * CMAXR + 1) * (2 * CMAXR + 1);

// disc offsets travel in the (<= 32 KB) kernel parameter space: re-entrant, no
// shared constant-bank state between concurrent calls
struct DiscOffsets {
    int2 o[CMAXOFF];
};

// The tile is zero-padded outside the grid; adding +0.0 to a non-negative float64 partial
// sum leaves it bit-unchanged, so summing every offset over the padded tile reproduces the
// reference's in-grid-only sequential sum exactly, without per-offset bounds checks.
template <typename Tin, int RC>
__global__ void __launch_bounds__(CNT) k_collision(const Tin *in, int W, int H, int rc_rt, int n_off,
                                                   double threshold, double *field, unsigned char *blocked,
                                                   const __grid_constant__ DiscOffsets D) {
    extern __shared__ __align__(16) double tile[];
    const int rc = RC >= 0 ? RC : rc_rt;
    const int E = CT + 2 * rc;
    const int L = blockIdx.z;
    const int X0 = blockIdx.x * CT, Y0 = blockIdx.y * CT;
    const Tin *src = in + (long long)L * W * H;
    for (int ly = threadIdx.x / CT; ly < E; ly += CNT / CT) {
        const int Y = Y0 - rc + ly;
        for (int lx = threadIdx.x % CT; lx < E; lx += CT) {
            const int X = X0 - rc + lx;
            tile[ly * E + lx] = (X >= 0 && X < W && Y >= 0 && Y < H) ? (double)src[(long long)Y * W + X] : 0.0;
        }
    }
    __syncthreads();
    // each thread sums CY = 4 cells of one column (rows yy0, yy0 + 8, ...) together: one
    // offset load and address per offset for all four, four independent float64 chains
    // (each still the reference's sequential order)
    constexpr int CY = CT / (CNT / CT);
    const int xx = threadIdx.x % CT, yy0 = threadIdx.x / CT;
    const int X = X0 + xx;
    const double *base = tile + (yy0 + rc) * E + (xx + rc);
    double s[CY];
#pragma unroll
    for (int c = 0; c < CY; ++c) s[c] = 0.0;
#pragma unroll 4
    for (int k = 0; k < n_off; ++k) {
        const int2 o = D.o[k];
        const double *b = base + o.y * E + o.x;
#pragma unroll
        for (int c = 0; c < CY; ++c) s[c] += b[c * (CNT / CT) * E];
    }
    if (X >= W) return;
#pragma unroll
    for (int c = 0; c < CY; ++c) {
        const int Y = Y0 + yy0 + c * (CNT / CT);
        if (Y >= H) break;
        const double v = s[c] < 1.0 ? s[c] : 1.0;  // np.minimum(out, 1.0)
        const long long oi = (long long)L * W * H + (long long)Y * W + X;
        if (field) field[oi] = v;
        if (blocked) blocked[oi] = v >= threshold ? 1 : 0;
    }
}

}  // namespace gc

using namespace gc;

extern "C" gc_status gc_collision_field(const void *d_layers, int32_t dtype_bytes, int32_t n_layers,
                                        int32_t grid_w, int32_t grid_h, const int32_t *h_offsets,
                                        int32_t n_offsets, double threshold, double *d_field,
                                        uint8_t *d_blocked, void *stream) {
    GC_CHECK_ARG(d_layers && (dtype_bytes == 4 || dtype_bytes == 8) && n_layers >= 1 && grid_w >= 1 &&
                     grid_h >= 1 && n_layers <= 65535,
                 "gc_collision_field: bad args");
    GC_CHECK_ARG(d_field || d_blocked, "gc_collision_field: need an output");
    GC_CHECK_ARG(n_offsets >= 0 && n_offsets <= CMAXOFF && (n_offsets == 0 || h_offsets),
                 "gc_collision_field: at most %d disc offsets", CMAXOFF);
    int rc = 0;
    for (int i = 0; i < n_offsets; ++i) {
        rc = max(rc, abs(h_offsets[2 * i]));
        rc = max(rc, abs(h_offsets[2 * i + 1]));
    }
    GC_CHECK_ARG(rc <= CMAXR, "gc_collision_field: radius above %d cells", CMAXR);
    cudaStream_t st = (cudaStream_t)stream;
    DiscOffsets local;  // copied into the launch parameters
    for (int i = 0; i < n_offsets; ++i) local.o[i] = make_int2(h_offsets[2 * i], h_offsets[2 * i + 1]);
    const int E = CT + 2 * rc;
    const size_t smem = (size_t)E * E * sizeof(double);
    dim3 grid((grid_w + CT - 1) / CT, (grid_h + CT - 1) / CT, n_layers);
#define GC_COLL_LAUNCH(T, R)                                                                      \
    do {                                                                                          \
        if (smem > 48 * 1024)                                                                     \
            GC_CUDA(cudaFuncSetAttribute(k_collision<T, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                         (int)smem));                                             \
        k_collision<T, R><<<grid, CNT, smem, st>>>((const T *)d_layers, grid_w, grid_h, rc, n_offsets,   \
                                                    threshold, d_field, d_blocked, local);          \
    } while (0)
    if (dtype_bytes == 4) {
        if (rc == 2) GC_COLL_LAUNCH(float, 2);
        else if (rc == 3) GC_COLL_LAUNCH(float, 3);
        else GC_COLL_LAUNCH(float, -1);
    } else {
        if (rc == 2) GC_COLL_LAUNCH(double, 2);
        else if (rc == 3) GC_COLL_LAUNCH(double, 3);
        else GC_COLL_LAUNCH(double, -1);
    }
#undef GC_COLL_LAUNCH
    count_launch();
    return cuda_check(cudaGetLastError(), "k_collision launch");
}
