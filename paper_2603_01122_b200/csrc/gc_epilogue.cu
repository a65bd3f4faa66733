// gc_epilogue.cu -- K3: occupancy epilogue.
//
// Windowed u32 counts -> layer values counts/n (float64, one IEEE division exactly as
// prediction.py:251) -> truncated Gaussian smoothing with edge-normalised columns
// (occupancy.py:122-154) applied as a banded separable stencil (SURVEY.md App. A.5:
// pre-divide each source cell by its in-grid kernel mass Z, then a plain
// (2R+1)-tap convolution along y then x) -> per-human float64 layers (the reference
// (T, H, W) layout) and/or the cell-wise max union of all humans (occupancy.py:162-192,
// sim.py:500-502) via order-independent atomicMax on the IEEE bits of non-negative
// values.  A second kernel applies the conservative time union (sim.py:503-504).
//
// The reference rescales each smoothed layer by before/after sums; the banded operator
// conserves mass exactly in real arithmetic, so that rescale only corrects rounding
// (<= 1e-16 relative) and is omitted: parity tests bound the difference at 1e-15 abs.
#include <cstdlib>
#include "gc_common.cuh"
#include "gc_internal.h"

namespace gc {

constexpr int ET = 32;    // output tile edge
constexpr int ENT = 256;  // threads per CTA
constexpr int MAXRAD = GC_MAX_SMOOTH_RADIUS;  // max smoothing radius (cells): the runtime-radius tile, (32 + 2R)^2 + 32 (32 + 2R) doubles, fits 227 KB

struct EParams {
    int n_humans, n, steps, grid_w, grid_h, radius, n_tiles, time_union;
    float ox, oy, res;
    const double *kernel, *zx, *zy;
    const float *start_xy;
    const int *step_r;
    const long long *step_off;
    long long human_stride;
    const int4 *tiles;
    const unsigned *counts;
    double *layers64;
    float *union32;
    double *union64;
    unsigned char *utile;  // union tile flags (steps, nty, ntx) or NULL
    int utx;               // union tiles per row
};

__device__ __forceinline__ void cell_of_start(float x, float y, const EParams &P, int &ix, int &iy) {
    const float fx = floorf(__fdiv_rn(__fsub_rn(x, P.ox), P.res));
    const float fy = floorf(__fdiv_rn(__fsub_rn(y, P.oy), P.res));
    ix = fx < 0.f ? 0 : (fx > (float)(P.grid_w - 1) ? P.grid_w - 1 : (int)fx);
    iy = fy < 0.f ? 0 : (fy > (float)(P.grid_h - 1) ? P.grid_h - 1 : (int)fy);
}

// RAD >= 0: compile-time smoothing radius (tile edges become constants); RAD < 0: runtime
template <int RAD>
__global__ void __launch_bounds__(ENT) k_epilogue(const EParams P) {
    extern __shared__ __align__(16) double esm[];
    const int h = blockIdx.y;
    const int4 tl = P.tiles[blockIdx.x];
    const int t = tl.x;
    const int rad = RAD >= 0 ? RAD : P.radius;
    const int E = ET + 2 * rad;
    double *vin = esm;            // E x E
    double *vmid = esm + E * E;   // ET x E
    __shared__ double kern[2 * MAXRAD + 1];

    int cx, cy;
    cell_of_start(__ldg(&P.start_xy[2 * h]), __ldg(&P.start_xy[2 * h + 1]), P, cx, cy);
    const int R = __ldg(&P.step_r[t]);
    const int x0 = max(0, cx - R), x1 = min(P.grid_w - 1, cx + R);
    const int y0 = max(0, cy - R), y1 = min(P.grid_h - 1, cy + R);
    const int ww = x1 - x0 + 1;
    // tile origin in grid coordinates (tile grid anchored at the unclamped grown window)
    const int X0 = cx - R - rad + tl.y * ET, Y0 = cy - R - rad + tl.z * ET;
    // whole tile outside the grown, clamped window or the grid -> nothing to do
    if (X0 > min(P.grid_w - 1, x1 + rad) || X0 + ET - 1 < max(0, x0 - rad) ||
        Y0 > min(P.grid_h - 1, y1 + rad) || Y0 + ET - 1 < max(0, y0 - rad))
        return;
    const unsigned *cnt = P.counts + (long long)h * P.human_stride + __ldg(&P.step_off[t]);
    const double inv_n = 1.0 / (double)P.n;  // only used for smoothing (see below)
    (void)inv_n;
    for (int i = threadIdx.x; i < 2 * rad + 1; i += ENT) kern[i] = P.kernel[i];

    // load inputs (counts/n, pre-divided by the source cell's in-grid kernel masses)
    int any = 0;
    for (int i = threadIdx.x; i < E * E; i += ENT) {
        const int ly = i / E, lx = i - ly * E;
        const int X = X0 - rad + lx, Y = Y0 - rad + ly;
        double v = 0.0;
        if (X >= x0 && X <= x1 && Y >= y0 && Y <= y1) {
            GC_DCHECK(__ldg(&P.step_off[t]) + (long long)(Y - y0) * ww + (X - x0) < P.human_stride);
            const unsigned c = __ldg(&cnt[(Y - y0) * ww + (X - x0)]);
            if (c) {
                v = (double)c / (double)P.n;  // exactly the reference's counts / n
                if (rad > 0) v = v * __ldg(&P.zy[Y]) * __ldg(&P.zx[X]);  // reciprocal in-grid masses
                any = 1;
            }
        }
        vin[i] = v;
    }
    // an all-zero tile (halo included) smooths to zeros: the outputs are zero-initialised
    // by the caller, so there is nothing to write
    if (!__syncthreads_or(any)) return;
    if (rad > 0) {
        // pass along y: vmid[yy][lx] = sum_o k[o] vin[yy + rad - o][lx]
        for (int i = threadIdx.x; i < ET * E; i += ENT) {
            const int yy = i / E, lx = i - yy * E;
            double s = 0.0;
            for (int o = -rad; o <= rad; ++o) s = fma(kern[o + rad], vin[(yy + rad - o) * E + lx], s);
            vmid[i] = s;
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < ET * ET; i += ENT) {
        const int yy = i / ET, xx = i - yy * ET;
        const int X = X0 + xx, Y = Y0 + yy;
        if (X < 0 || X >= P.grid_w || Y < 0 || Y >= P.grid_h) continue;
        double v;
        if (rad > 0) {
            double s = 0.0;
            for (int o = -rad; o <= rad; ++o) s = fma(kern[o + rad], vmid[yy * E + (xx + rad - o)], s);
            v = s > 0.0 ? s : 0.0;  // np.maximum(out, 0) (occupancy.py:153)
        } else {
            v = vin[(yy + rad) * E + (xx + rad)];
        }
        GC_DCHECK(yy * E + xx + 2 * rad < E * E && (rad == 0 || yy * E + xx + 2 * rad < ET * E));
        const long long cell = (long long)Y * P.grid_w + X;
        if (P.layers64) P.layers64[((long long)h * P.steps + t) * P.grid_h * P.grid_w + cell] = v;
        if (v > 0.0) {
            const long long o = (long long)t * P.grid_h * P.grid_w + cell;
            if (P.union32) atomicMax(reinterpret_cast<unsigned *>(P.union32) + o, __float_as_uint((float)v));
            if (P.union64)
                atomicMax(reinterpret_cast<unsigned long long *>(P.union64) + o,
                          (unsigned long long)__double_as_longlong(v));
            // this union tile is nonzero this cycle (idempotent byte store; a warp's lanes
            // mostly hit the same byte and coalesce)
            if (P.utile) P.utile[((long long)t * ((P.grid_h + ET - 1) / ET) + (Y >> 5)) * P.utx + (X >> 5)] = 1;
        }
    }
}

// K3 for a compile-time smoothing radius 1..3 (the bench's sigma = 1 cell is RAD = 3):
// warp w owns rows, lane = column, so the count loads of a row are coalesced and need no
// index division; each thread issues all of its count loads before using any (the
// round-1 loop waited on each load in turn: 40 % long-scoreboard stalls), the vertical
// pass keeps a sliding column of 4 + 2 RAD inputs in registers (4 outputs per column from
// 4 + 2 RAD shared loads instead of 4 (2 RAD + 1)), the kernel taps live in registers, zero
// outputs are not written (the outputs are zero-filled), and the union-tile flags are
// OR-reduced per CTA (at most 4 union tiles per output tile) instead of one byte store per
// nonzero cell.  Same arithmetic as k_epilogue: identical results.
#ifndef GC_K3_MIN_CTAS
#define GC_K3_MIN_CTAS 6  // 40 registers, 6 CTAs/SM: K3 -14 % vs the unbounded 48 (5 CTAs/SM)
#endif
template <int RAD>
__global__ void __launch_bounds__(ENT, GC_K3_MIN_CTAS) k_epilogue_r(const EParams P) {
    constexpr int E = ET + 2 * RAD;          // input tile edge
    constexpr int NW = ENT / 32;             // warps
    constexpr int LR = (E + NW - 1) / NW;    // input rows per warp
    constexpr int RPW = ET / NW;             // output rows per warp
    __shared__ double vin[E][E];
    __shared__ double vmid[ET][E];
    __shared__ unsigned utmask;
    const int h = blockIdx.y;
    const int4 tl = P.tiles[blockIdx.x];
    const int t = tl.x;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int cx, cy;
    cell_of_start(__ldg(&P.start_xy[2 * h]), __ldg(&P.start_xy[2 * h + 1]), P, cx, cy);
    const int R = __ldg(&P.step_r[t]);
    const int x0 = max(0, cx - R), x1 = min(P.grid_w - 1, cx + R);
    const int y0 = max(0, cy - R), y1 = min(P.grid_h - 1, cy + R);
    const int ww = x1 - x0 + 1;
    const int X0 = cx - R - RAD + tl.y * ET, Y0 = cy - R - RAD + tl.z * ET;
    if (X0 > min(P.grid_w - 1, x1 + RAD) || X0 + ET - 1 < max(0, x0 - RAD) ||
        Y0 > min(P.grid_h - 1, y1 + RAD) || Y0 + ET - 1 < max(0, y0 - RAD))
        return;
    const unsigned *cnt = P.counts + (long long)h * P.human_stride + __ldg(&P.step_off[t]);
    if (threadIdx.x == 0) utmask = 0u;
    // ---- counts: all loads in flight first ----
    unsigned c0[LR], c1[LR];
#pragma unroll
    for (int i = 0; i < LR; ++i) {
        const int r = w + NW * i, Y = Y0 - RAD + r;
        const int Xa = X0 - RAD + lane, Xb = Xa + 32;
        const bool rowok = r < E && Y >= y0 && Y <= y1;
        const unsigned *row = cnt + (long long)(Y - y0) * ww - x0;
        GC_DCHECK(!(rowok && Xa >= x0 && Xa <= x1) || __ldg(&P.step_off[t]) + (long long)(Y - y0) * ww + (Xa - x0) < P.human_stride);
        c0[i] = (rowok && Xa >= x0 && Xa <= x1) ? __ldg(row + Xa) : 0u;
        c1[i] = (rowok && lane < 2 * RAD && Xb >= x0 && Xb <= x1) ? __ldg(row + Xb) : 0u;
    }
    int any = 0;
    const double dn = (double)P.n;
#pragma unroll
    for (int i = 0; i < LR; ++i) {
        const int r = w + NW * i, Y = Y0 - RAD + r;
        if (r < E) {
            const int Xa = X0 - RAD + lane;
            double va = 0.0, vb = 0.0;
            if (c0[i]) { va = (double)c0[i] / dn * __ldg(&P.zy[Y]) * __ldg(&P.zx[Xa]); any = 1; }
            if (c1[i]) { vb = (double)c1[i] / dn * __ldg(&P.zy[Y]) * __ldg(&P.zx[Xa + 32]); any = 1; }
            vin[r][lane] = va;
            if (lane < 2 * RAD) vin[r][lane + 32] = vb;
        }
    }
    if (!__syncthreads_or(any)) return;
    double kr[2 * RAD + 1];
#pragma unroll
    for (int o = 0; o < 2 * RAD + 1; ++o) kr[o] = __ldg(&P.kernel[o]);
    // ---- pass along y: vmid[yy][c] = sum_o k[o] vin[yy + RAD - o][c], rows RPW w .. ----
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        const int c = lane + 32 * half;
        if (half == 1 && lane >= 2 * RAD) break;
        double a[RPW + 2 * RAD];
#pragma unroll
        for (int j = 0; j < RPW + 2 * RAD; ++j) a[j] = vin[RPW * w + j][c];
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
            double s = 0.0;
#pragma unroll
            for (int o = -RAD; o <= RAD; ++o) s = fma(kr[o + RAD], a[i + RAD - o], s);
            vmid[RPW * w + i][c] = s;
        }
    }
    __syncthreads();
    // ---- pass along x, clamp, outputs ----
    const int X = X0 + lane;
    const bool colok = X >= 0 && X < P.grid_w;
    unsigned um = 0u;
#pragma unroll
    for (int i = 0; i < RPW; ++i) {
        const int yy = RPW * w + i, Y = Y0 + yy;
        double s = 0.0;
#pragma unroll
        for (int o = -RAD; o <= RAD; ++o) s = fma(kr[o + RAD], vmid[yy][lane + RAD - o], s);
        const double v = s > 0.0 ? s : 0.0;  // np.maximum(out, 0) (occupancy.py:153)
        if (!colok || Y < 0 || Y >= P.grid_h || !(v > 0.0)) continue;
        const long long cell = (long long)Y * P.grid_w + X;
        if (P.layers64) P.layers64[((long long)h * P.steps + t) * P.grid_h * P.grid_w + cell] = v;
        const long long o = (long long)t * P.grid_h * P.grid_w + cell;
        if (P.union32) atomicMax(reinterpret_cast<unsigned *>(P.union32) + o, __float_as_uint((float)v));
        if (P.union64)
            atomicMax(reinterpret_cast<unsigned long long *>(P.union64) + o, (unsigned long long)__double_as_longlong(v));
        um |= 1u << (2 * ((Y >> 5) - (Y0 >> 5)) + ((X >> 5) - (X0 >> 5)));
    }
    if (P.utile) {
        um = __reduce_or_sync(0xffffffffu, um);
        if (lane == 0 && um) atomicOr(&utmask, um);
        __syncthreads();
        if (threadIdx.x < 4 && (utmask >> threadIdx.x) & 1u) {
            const int uy = (Y0 >> 5) + (threadIdx.x >> 1), ux = (X0 >> 5) + (threadIdx.x & 1);
            P.utile[((long long)t * ((P.grid_h + ET - 1) / ET) + uy) * P.utx + ux] = 1;
        }
    }
}

// conservative time union: layer t <- max over t' <= t (np.maximum.accumulate, axis 0)
template <typename Tv>
__global__ void k_time_union(Tv *u, int t0, int t1, long long cells) {
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cells) return;
    const int ts = t0 > 0 ? t0 - 1 : 0;  // seeded by the (final) layer before the range
    Tv run = u[(long long)ts * cells + c];
    for (int t = ts + 1; t < t1; ++t) {
        const long long o = (long long)t * cells + c;
        const Tv v = u[o];
        if (v < run) u[o] = run; else run = v;
    }
}

// ---- standalone smooth_values (occupancy.py:139-154) over full float64 layers -------
__global__ void __launch_bounds__(ENT) k_smooth(const double *in, double *out, int W, int H, int rad,
                                                const double *kernel, const double *zx, const double *zy) {
    extern __shared__ __align__(16) double ssm[];
    const int E = ET + 2 * rad;
    double *vin = ssm, *vmid = ssm + E * E;
    const int L = blockIdx.z;
    const int X0 = blockIdx.x * ET, Y0 = blockIdx.y * ET;
    const double *src = in + (long long)L * W * H;
    for (int i = threadIdx.x; i < E * E; i += ENT) {
        const int ly = i / E, lx = i - ly * E;
        const int X = X0 - rad + lx, Y = Y0 - rad + ly;
        double v = 0.0;
        if (X >= 0 && X < W && Y >= 0 && Y < H) v = src[(long long)Y * W + X] * zy[Y] * zx[X];  // reciprocal in-grid masses
        vin[i] = v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ET * E; i += ENT) {
        const int yy = i / E, lx = i - yy * E;
        double s = 0.0;
        for (int o = -rad; o <= rad; ++o) s = fma(kernel[o + rad], vin[(yy + rad - o) * E + lx], s);
        vmid[i] = s;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < ET * ET; i += ENT) {
        const int yy = i / ET, xx = i - yy * ET;
        const int X = X0 + xx, Y = Y0 + yy;
        if (X >= W || Y >= H) continue;
        double s = 0.0;
        for (int o = -rad; o <= rad; ++o) s = fma(kernel[o + rad], vmid[yy * E + (xx + rad - o)], s);
        out[(long long)L * W * H + (long long)Y * W + X] = s > 0.0 ? s : 0.0;
    }
}

// ---- standalone emplace_counts (occupancy.py:105-109) ---------------------------------
__global__ void k_emplace(const float *xy, long long n, int W, int H, float ox, float oy, float res,
                          unsigned *counts) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float fx = floorf(__fdiv_rn(__fsub_rn(xy[2 * i], ox), res));
    const float fy = floorf(__fdiv_rn(__fsub_rn(xy[2 * i + 1], oy), res));
    const int ix = fx < 0.f ? 0 : (fx > (float)(W - 1) ? W - 1 : (int)fx);
    const int iy = fy < 0.f ? 0 : (fy > (float)(H - 1) ? H - 1 : (int)fy);
    atomicAdd(&counts[(long long)iy * W + ix], 1u);
}

}  // namespace gc

using namespace gc;

extern "C" gc_status gc_emplace_counts(const float *d_xy, int64_t n, int32_t grid_w, int32_t grid_h,
                                       float origin_x32, float origin_y32, float res32, uint32_t *d_counts,
                                       void *stream) {
    GC_CHECK_ARG(d_xy && d_counts && n >= 1 && grid_w >= 1 && grid_h >= 1 && res32 > 0.f,
                 "gc_emplace_counts: bad args");
    k_emplace<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(d_xy, n, grid_w, grid_h, origin_x32,
                                                                            origin_y32, res32, d_counts);
    count_launch();
    return cuda_check(cudaGetLastError(), "k_emplace launch");
}

extern "C" gc_status gc_smooth_layers(const double *d_in, double *d_out, int32_t n_layers, int32_t grid_w,
                                      int32_t grid_h, int32_t radius, const double *d_kernel, const double *d_zx,
                                      const double *d_zy, void *stream) {
    GC_CHECK_ARG(d_in && d_out && d_in != d_out && n_layers >= 1 && grid_w >= 1 && grid_h >= 1,
                 "gc_smooth_layers: bad args");
    GC_CHECK_ARG(radius >= 1 && radius <= MAXRAD && d_kernel && d_zx && d_zy, "gc_smooth_layers: radius 1..%d", MAXRAD);
    GC_CHECK_ARG(n_layers <= 65535, "gc_smooth_layers: too many layers");
    const int E = ET + 2 * radius;
    const size_t smem = (size_t)(E * E + ET * E) * sizeof(double);
    if (smem > 48 * 1024)
        GC_CUDA(cudaFuncSetAttribute(k_smooth, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid((grid_w + ET - 1) / ET, (grid_h + ET - 1) / ET, n_layers);
    k_smooth<<<grid, ENT, smem, (cudaStream_t)stream>>>(d_in, d_out, grid_w, grid_h, radius, d_kernel, d_zx, d_zy);
    count_launch();
    return cuda_check(cudaGetLastError(), "k_smooth launch");
}

extern "C" gc_status gc_grid_epilogue(const gc_epilogue_args *a, void *stream) {
    GC_CHECK_ARG(a != nullptr, "gc_grid_epilogue: null args");
    GC_CHECK_ARG(a->n_humans >= 1 && a->n >= 1 && a->steps >= 1, "gc_grid_epilogue: bad sizes");
    GC_CHECK_ARG(a->radius >= 0 && a->radius <= MAXRAD, "gc_grid_epilogue: smoothing radius 0..%d cells", MAXRAD);
    GC_CHECK_ARG(a->radius == 0 || (a->d_kernel && a->d_zx && a->d_zy), "gc_grid_epilogue: missing kernel tables");
    GC_CHECK_ARG(a->d_tiles && a->n_tiles >= 1 && a->d_counts && a->d_start_xy && a->d_step_r && a->d_step_off,
                 "gc_grid_epilogue: missing geometry buffers");
    GC_CHECK_ARG(a->n_humans <= 65535, "gc_grid_epilogue: too many humans");
    EParams P;
    P.n_humans = a->n_humans; P.n = a->n; P.steps = a->steps; P.grid_w = a->grid_w; P.grid_h = a->grid_h;
    P.radius = a->radius; P.n_tiles = a->n_tiles; P.time_union = a->time_union;
    P.ox = a->origin_x32; P.oy = a->origin_y32; P.res = a->res32;
    P.kernel = a->d_kernel; P.zx = a->d_zx; P.zy = a->d_zy;
    P.start_xy = a->d_start_xy; P.step_r = a->d_step_r; P.step_off = (const long long *)a->d_step_off;
    P.human_stride = a->human_stride; P.tiles = (const int4 *)a->d_tiles; P.counts = a->d_counts;
    P.layers64 = a->d_layers64; P.union32 = a->d_union32; P.union64 = a->d_union64;
    P.utile = (a->d_union32 || a->d_union64) ? a->d_union_tile_flags : nullptr;
    P.utx = (a->grid_w + ET - 1) / ET;
    const int E = ET + 2 * a->radius;
    const size_t smem = (size_t)(E * E + (a->radius > 0 ? ET * E : 0)) * sizeof(double);
    if (smem > 48 * 1024)
        GC_CUDA(cudaFuncSetAttribute(k_epilogue<-1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaStream_t st = (cudaStream_t)stream;
    const int tb = a->tile_end > 0 ? a->tile_begin : 0;
    const int te = a->tile_end > 0 ? a->tile_end : a->n_tiles;
    GC_CHECK_ARG(tb >= 0 && tb < te && te <= a->n_tiles, "gc_grid_epilogue: bad tile range");
    P.tiles = (const int4 *)a->d_tiles + tb;
    dim3 grid(te - tb, a->n_humans);
    switch (a->radius) {
        case 0: k_epilogue<0><<<grid, ENT, smem, st>>>(P); break;
        case 1: k_epilogue_r<1><<<grid, ENT, 0, st>>>(P); break;
        case 2: k_epilogue_r<2><<<grid, ENT, 0, st>>>(P); break;
        case 3: k_epilogue_r<3><<<grid, ENT, 0, st>>>(P); break;
        default: k_epilogue<-1><<<grid, ENT, smem, st>>>(P); break;
    }
    count_launch();
    GC_TRY(cuda_check(cudaGetLastError(), "k_epilogue launch"));
    const int t0 = a->t_end > 0 ? a->t_begin : 0, t1 = a->t_end > 0 ? a->t_end : a->steps;
    if (a->time_union && a->steps > 1 && t1 - (t0 > 0 ? t0 - 1 : 0) > 1) {
        const long long cells = (long long)a->grid_w * a->grid_h;
        const int blocks = (int)((cells + 255) / 256);
        if (a->d_union32) { k_time_union<float><<<blocks, 256, 0, st>>>(a->d_union32, t0, t1, cells); count_launch(); }
        if (a->d_union64) { k_time_union<double><<<blocks, 256, 0, st>>>(a->d_union64, t0, t1, cells); count_launch(); }
        GC_TRY(cuda_check(cudaGetLastError(), "k_time_union launch"));
    }
    return GC_OK;
}

// ---- tile-sparse publication of a union into a pinned host stack -----------------------
// one warp per (layer, 32 x 32 tile); lane = column, rows looped: every row of a tile is one
// coalesced 128 / 256-byte write over PCIe (or one read of the device union)
namespace gc {
template <typename Tv>
__global__ void __launch_bounds__(256) k_publish(const Tv *un, Tv *dst, const unsigned char *flags,
                                                 unsigned char *hflags, int W, int H, int t0, int t1, int time_or) {
    const int ntx = (W + ET - 1) / ET, nty = (H + ET - 1) / ET, per = ntx * nty;
    const long long total = (long long)(t1 - t0) * per;
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < total; w += warps) {
        const int t = t0 + (int)(w / per), tile = (int)(w % per);
        bool live = flags[(long long)t * per + tile] != 0;
        if (time_or && !live) {  // the time union spreads a tile to every later layer
            for (int s = lane; s < t; s += 32) live |= flags[(long long)s * per + tile] != 0;
            live = __any_sync(0xffffffffu, live);
        }
        const long long hf = (long long)t * per + tile;
        const bool held = hflags[hf] != 0;
        if (!live && !held) continue;  // zero on the device, zero on the host
        const int X = (tile % ntx) * ET + lane, Y0 = (tile / ntx) * ET;
        if (X < W) {
            const long long base = (long long)t * H * W + X;
            for (int r = 0; r < ET && Y0 + r < H; ++r) {
                const long long o = base + (long long)(Y0 + r) * W;
                dst[o] = live ? un[o] : Tv(0);
            }
        }
        if (lane == 0) hflags[hf] = live ? 1 : 0;
    }
}
}  // namespace gc

extern "C" gc_status gc_publish_tiles(const gc_publish_args *a, void *stream) {
    GC_CHECK_ARG(a && a->d_union && a->d_tile_flags && a->d_host_flags && a->h_dst, "gc_publish_tiles: missing buffers");
    GC_CHECK_ARG(a->dtype_bytes == 4 || a->dtype_bytes == 8, "gc_publish_tiles: float32 or float64 layers");
    GC_CHECK_ARG(a->grid_w >= 1 && a->grid_h >= 1 && a->steps >= 1, "gc_publish_tiles: bad sizes");
    const int t0 = a->t_end > 0 ? a->t_begin : 0, t1 = a->t_end > 0 ? a->t_end : a->steps;
    GC_CHECK_ARG(t0 >= 0 && t0 < t1 && t1 <= a->steps, "gc_publish_tiles: bad layer range");
    cudaStream_t st = (cudaStream_t)stream;
    // PCIe-bound: a few CTAs reach the link's write bandwidth (zero-copy stores), and every
    // CTA of this kernel holds an SM slot the concurrently running K2 cannot use
    static const int max_ctas = [] {
        const char *e = getenv("GC_PUBLISH_CTAS");  // tuning knob
        const int v = e ? atoi(e) : 32;  // 32: 5.066 ms e2e graph vs 5.086 at 148 (cfg3, f64)
        return v < 1 ? 1 : v;
    }();
    const long long work = (long long)(t1 - t0) * ((a->grid_w + ET - 1) / ET) * ((a->grid_h + ET - 1) / ET);
    const int blocks = (int)(work < (long long)max_ctas * 8 ? (work + 7) / 8 : max_ctas);
    if (a->dtype_bytes == 8)
        k_publish<double><<<blocks, 256, 0, st>>>((const double *)a->d_union, (double *)a->h_dst, a->d_tile_flags,
                                                  a->d_host_flags, a->grid_w, a->grid_h, t0, t1, a->time_or);
    else
        k_publish<float><<<blocks, 256, 0, st>>>((const float *)a->d_union, (float *)a->h_dst, a->d_tile_flags,
                                                 a->d_host_flags, a->grid_w, a->grid_h, t0, t1, a->time_or);
    count_launch();
    return cuda_check(cudaGetLastError(), "k_publish launch");
}

// ---- union tiles <-> packed buffer (the sparse cross-GPU max-reduce of the fused grid) ----
// tile id = (t * nty + ty) * ntx + tx over the (T, H, W) union's 32 x 32 tiles (the layout of
// the union-tile flags); packed[i] is tile ids[i] as a 32 x 32 block, zero outside the grid.
// One warp per tile, lane = column, rows looped: coalesced rows both ways.
namespace gc {
template <typename Tv>
__global__ void __launch_bounds__(256) k_union_tiles(Tv *un, Tv *packed, const int *ids, int count, int T, int W,
                                                     int H, int unpack) {
    const int ntx = (W + ET - 1) / ET, nty = (H + ET - 1) / ET;
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < count; w += warps) {
        const int id = __ldg(&ids[w]);
        if (id < 0 || id >= T * ntx * nty) continue;  // not a tile of this union: left alone
        const int t = id / (ntx * nty), rem = id - t * ntx * nty;
        const int X = (rem % ntx) * ET + lane, Y0 = (rem / ntx) * ET;
        Tv *pk = packed + w * ET * ET + lane;
        const long long base = (long long)t * H * W + X;
        if (unpack) {
            if (X < W)
                for (int r = 0; r < ET && Y0 + r < H; ++r) un[base + (long long)(Y0 + r) * W] = pk[r * ET];
        } else {
            for (int r = 0; r < ET; ++r)
                pk[r * ET] = (X < W && Y0 + r < H) ? un[base + (long long)(Y0 + r) * W] : Tv(0);
        }
    }
}
}  // namespace gc

extern "C" gc_status gc_union_tiles(void *d_union, int32_t dtype_bytes, int32_t steps, int32_t grid_w, int32_t grid_h,
                                    const int32_t *d_tile_ids, int32_t count, void *d_packed, int32_t unpack,
                                    void *stream) {
    GC_CHECK_ARG(d_union && d_packed && d_tile_ids && count >= 0, "gc_union_tiles: bad arguments");
    GC_CHECK_ARG(dtype_bytes == 4 || dtype_bytes == 8, "gc_union_tiles: float32 or float64 layers");
    GC_CHECK_ARG(steps >= 1 && grid_w >= 1 && grid_h >= 1, "gc_union_tiles: bad sizes");
    if (count == 0) return GC_OK;
    const int blocks = (int)(((long long)count + 7) / 8 < 148 * 8 ? ((long long)count + 7) / 8 : 148 * 8);
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype_bytes == 8)
        k_union_tiles<double><<<blocks, 256, 0, st>>>((double *)d_union, (double *)d_packed, d_tile_ids, count, steps,
                                                      grid_w, grid_h, unpack);
    else
        k_union_tiles<float><<<blocks, 256, 0, st>>>((float *)d_union, (float *)d_packed, d_tile_ids, count, steps,
                                                     grid_w, grid_h, unpack);
    count_launch();
    return cuda_check(cudaGetLastError(), "k_union_tiles launch");
}

// ---- ordered union of k stacked layer sets (occupancy.py:162-192) --------------------
// input i = in + i * stride (elements), `cells` elements each; float64 arithmetic in the
// reference's order: max, or miss = 1 - clip(p_0); miss *= 1 - clip(p_i); out = 1 - miss.
namespace gc {
template <typename Ti, typename To>
__global__ void __launch_bounds__(256) k_union(const Ti *in, int k, long long stride, long long cells, int mode,
                                               To *out) {
    for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < cells;
         c += (long long)gridDim.x * blockDim.x) {
        double acc;
        if (mode == GC_UNION_MAX) {
            acc = (double)in[c];
            for (int i = 1; i < k; ++i) acc = fmax(acc, (double)in[i * stride + c]);
        } else if (mode == GC_UNION_COMPLEMENT) {
            acc = __dsub_rn(1.0, (double)in[c]);
        } else {
            double miss = __dsub_rn(1.0, fmin(fmax((double)in[c], 0.0), 1.0));
            for (int i = 1; i < k; ++i)
                miss = __dmul_rn(miss, __dsub_rn(1.0, fmin(fmax((double)in[i * stride + c], 0.0), 1.0)));
            acc = mode == GC_UNION_INDEPENDENT ? __dsub_rn(1.0, miss) : miss;
        }
        out[c] = (To)acc;
    }
}

template <typename Ti, typename To>
static void launch_union(const void *in, int k, long long stride, long long cells, int mode, void *out,
                         cudaStream_t st) {
    long long blocks = (cells + 255) / 256;
    blocks = blocks < 148 * 16 ? blocks : 148 * 16;
    k_union<Ti, To><<<(int)blocks, 256, 0, st>>>((const Ti *)in, k, stride, cells, mode, (To *)out);
}
}  // namespace gc

extern "C" gc_status gc_union_layers(const void *d_in, int32_t in_bytes, int32_t k, int64_t stride, int64_t cells,
                                     int32_t mode, void *d_out, int32_t out_bytes, void *stream) {
    GC_CHECK_ARG(d_in && d_out && k >= 1 && cells >= 0 && stride >= 0, "gc_union_layers: bad arguments");
    GC_CHECK_ARG((in_bytes == 4 || in_bytes == 8) && (out_bytes == 4 || out_bytes == 8),
                 "gc_union_layers: float32 or float64 layers");
    GC_CHECK_ARG(mode >= GC_UNION_MAX && mode <= GC_UNION_COMPLEMENT, "gc_union_layers: unknown mode");
    if (cells == 0) return GC_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (in_bytes == 8 && out_bytes == 8) launch_union<double, double>(d_in, k, stride, cells, mode, d_out, st);
    else if (in_bytes == 8) launch_union<double, float>(d_in, k, stride, cells, mode, d_out, st);
    else if (out_bytes == 8) launch_union<float, double>(d_in, k, stride, cells, mode, d_out, st);
    else launch_union<float, float>(d_in, k, stride, cells, mode, d_out, st);
    count_launch();
    return cuda_check(cudaGetLastError(), "k_union launch");
}

extern "C" gc_status gc_time_union(void *d_union, int32_t dtype_bytes, int32_t t_begin, int32_t t_end,
                                   int64_t cells, void *stream) {
    GC_CHECK_ARG(d_union && (dtype_bytes == 4 || dtype_bytes == 8), "gc_time_union: float32 or float64 layers");
    GC_CHECK_ARG(t_begin >= 0 && t_begin < t_end && cells >= 0, "gc_time_union: bad layer range");
    if (cells == 0 || t_end - (t_begin > 0 ? t_begin - 1 : 0) < 2) return GC_OK;
    const int blocks = (int)((cells + 255) / 256);
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype_bytes == 4) k_time_union<float><<<blocks, 256, 0, st>>>((float *)d_union, t_begin, t_end, cells);
    else k_time_union<double><<<blocks, 256, 0, st>>>((double *)d_union, t_begin, t_end, cells);
    count_launch();
    return cuda_check(cudaGetLastError(), "k_time_union launch");
}
