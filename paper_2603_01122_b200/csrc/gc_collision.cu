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

template <typename Tin>
__global__ void __launch_bounds__(CNT) k_collision(const Tin *in, int W, int H, int rc, int n_off,
                                                   double threshold, double *field, unsigned char *blocked,
                                                   const __grid_constant__ DiscOffsets D) {
    extern __shared__ __align__(16) double tile[];
    const int E = CT + 2 * rc;
    const int L = blockIdx.z;
    const int X0 = blockIdx.x * CT, Y0 = blockIdx.y * CT;
    const Tin *src = in + (long long)L * W * H;
    for (int i = threadIdx.x; i < E * E; i += CNT) {
        const int ly = i / E, lx = i - ly * E;
        const int X = X0 - rc + lx, Y = Y0 - rc + ly;
        tile[i] = (X >= 0 && X < W && Y >= 0 && Y < H) ? (double)src[(long long)Y * W + X] : 0.0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < CT * CT; i += CNT) {
        const int yy = i / CT, xx = i - yy * CT;
        const int X = X0 + xx, Y = Y0 + yy;
        if (X >= W || Y >= H) continue;
        double s = 0.0;
        for (int k = 0; k < n_off; ++k) {
            const int2 o = D.o[k];
            const int sx = X + o.x, sy = Y + o.y;
            // out-of-grid sources are skipped, not added as zero (keeps the reference's
            // exact summation sequence; -0.0/+0.0 cannot differ for non-negative inputs)
            if (sx >= 0 && sx < W && sy >= 0 && sy < H) s += tile[(yy + rc + o.y) * E + (xx + rc + o.x)];
        }
        s = s < 1.0 ? s : 1.0;  // np.minimum(out, 1.0)
        const long long o = (long long)L * W * H + (long long)Y * W + X;
        if (field) field[o] = s;
        if (blocked) blocked[o] = s >= threshold ? 1 : 0;
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
    if (dtype_bytes == 4) {
        if (smem > 48 * 1024)
            GC_CUDA(cudaFuncSetAttribute(k_collision<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_collision<float><<<grid, CNT, smem, st>>>((const float *)d_layers, grid_w, grid_h, rc, n_offsets,
                                                     threshold, d_field, d_blocked, local);
    } else {
        if (smem > 48 * 1024)
            GC_CUDA(cudaFuncSetAttribute(k_collision<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_collision<double><<<grid, CNT, smem, st>>>((const double *)d_layers, grid_w, grid_h, rc, n_offsets,
                                                      threshold, d_field, d_blocked, local);
    }
    count_launch();
    return cuda_check(cudaGetLastError(), "k_collision launch");
}
