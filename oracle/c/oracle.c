/*
 * ORACLE (test infrastructure only) -- plain-C, host-independent restatement of the
 * reference particle step.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load liboracle.so; the product never links it.
 *
 * Restates, op by op in IEEE float32 (every op separately rounded unless written fmaf):
 *   _propagate_chunk            /root/reference/pkg/src/gridcast/prediction.py:147-162
 *   q_goal_progress.shift_free  agents.py:275-288   (K=2 sgemm order: fmaf(ry,sy,rx*sx))
 *   q_goal_progress.base        agents.py:290-294   (einsum |rel|^2 unfused)
 *   q_default.base              agents.py:254-257
 *   GridSpec.cells_of           occupancy.py:43-51  (NEP-50 float32 cell arithmetic)
 * and numpy 2.3's float32 exp kernel (un-vendored dependency of the reference,
 * pkg/pyproject.toml:10-14; SIMD algorithm restated in SURVEY.md App. A.2).
 *
 * Compile with -O2 -ffp-contract=off (no implicit FMA contraction), never -ffast-math.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* numpy float32 exp (AVX512F/AVX2 SIMD path) */
float or_exp_np_scalar(float x)
{
    if (x > 88.72283935546875f) return INFINITY;
    if (x < -103.97208404541015625f) return 0.0f;
    volatile float shifter = 0x1.8p23f;
    float t = x * 1.442695040888963407359924681001892137f;
    float q = (t + shifter) - shifter;
    float r = fmaf(q, -6.93145752e-1f, x);
    r = fmaf(q, -1.42860677e-6f, r);
    float num = fmaf(5.082762527590693718096e-04f, r, 6.757896990527504603057e-03f);
    num = fmaf(num, r, 5.114512081637298353406e-02f);
    num = fmaf(num, r, 2.473615434895520810817e-01f);
    num = fmaf(num, r, 7.257664613233124478488e-01f);
    num = fmaf(num, r, 9.999999999980870924916e-01f);
    float den = fmaf(2.159509375685829852307e-02f, r, -2.742335390411667452936e-01f);
    den = fmaf(den, r, 1.0f);
    float y = num / den;
    return ldexpf(y, (int)q); /* exact power-of-two scaling, single rounding */
}

void or_exp_np_f32(const float *x, float *y, long n)
{
    for (long i = 0; i < n; ++i) y[i] = or_exp_np_scalar(x[i]);
}

enum { OR_Q_GOAL_PROGRESS = 0, OR_Q_GOAL_PROGRESS_FULL = 1, OR_Q_DEFAULT = 2 };

/*
 * One propagate step for n particles (prediction.py:147-162).
 *   xy_in/xy_out: (n,2) f32; hyp: (n,) i32; beta32 (n_hyp,), goal32 (n_hyp,2)
 *   per-action tables over the FULL control set (length m_all):
 *     sx, sy, at (goal progress: step_x*tau, step_y*tau, action term incl. weights)
 *     pen (q_default penalty)
 *     dispx, dispy: f32 displacements
 *   keep: (m_keep,) unmasked action indices (prediction.py:134-144)
 *   u01: (n,) f32 uniforms.  work: scratch of m_keep floats.
 *   picked_out (optional): chosen full-set action index per particle.
 */
void or_propagate(const float *xy_in, float *xy_out, const int32_t *hyp, long n,
                  const float *beta32, const float *goal32,
                  const float *sx, const float *sy, const float *at, const float *pen,
                  int q_kind, const float *dispx, const float *dispy,
                  const int32_t *keep, int m_keep, const float *u01, float *work,
                  int32_t *picked_out)
{
    for (long i = 0; i < n; ++i) {
        const float x = xy_in[2 * i], y = xy_in[2 * i + 1];
        const int h = hyp[i];
        const float rx = x - goal32[2 * h];
        const float ry = y - goal32[2 * h + 1];
        const float b = beta32[h];
        float mx = -INFINITY;
        for (int k = 0; k < m_keep; ++k) {
            const int j = keep[k];
            float L;
            if (q_kind == OR_Q_DEFAULT) {
                const float rxx = rx * rx, ryy = ry * ry;
                const float d2 = rxx + ryy;
                L = (-d2) - pen[j];
            } else {
                const float px = rx * sx[j];
                const float dot = fmaf(ry, sy[j], px);
                L = dot * -2.0f;
                L = L - at[j];
                if (q_kind == OR_Q_GOAL_PROGRESS_FULL) {
                    const float rxx = rx * rx, ryy = ry * ry;
                    const float d2 = rxx + ryy;
                    L = L - d2;
                }
            }
            L = L * b;
            work[k] = L;
            if (L > mx) mx = L;
        }
        float c = 0.0f;
        for (int k = 0; k < m_keep; ++k) {
            const float w = or_exp_np_scalar(work[k] - mx);
            c = (k == 0) ? w : c + w;
            work[k] = c;
        }
        const float r = u01[i] * c;
        int cnt = 0;
        for (int k = 0; k < m_keep; ++k) cnt += (work[k] < r);
        if (cnt > m_keep - 1) cnt = m_keep - 1;
        const int a = keep[cnt];
        if (picked_out) picked_out[i] = a;
        xy_out[2 * i] = x + dispx[a];
        xy_out[2 * i + 1] = y + dispy[a];
    }
}

/* GridSpec.cells_of with clamp (occupancy.py:43-51) in float32 -> flat iy*W+ix */
void or_cells(const float *xy, long n, float ox32, float oy32, float res32, int W, int H,
              int64_t *flat)
{
    for (long i = 0; i < n; ++i) {
        float fx = floorf((xy[2 * i] - ox32) / res32);
        float fy = floorf((xy[2 * i + 1] - oy32) / res32);
        int64_t ix = (fx < 0.0f) ? 0 : (fx > (float)(W - 1) ? W - 1 : (int64_t)fx);
        int64_t iy = (fy < 0.0f) ? 0 : (fy > (float)(H - 1) ? H - 1 : (int64_t)fy);
        flat[i] = iy * (int64_t)W + ix;
    }
}
