// ds_common.cuh -- shared device code of the sm_100a checkpoint hot path.
//
// Row-group model: one embedding row is owned by a group of G lanes
// (G = 1..32, a power of two, groups aligned inside a warp).  Lane `lig` of
// the group holds EPL = VEC*C elements in registers:
//   VEC == 4 : chunk c holds elements 4*(lig + c*G) .. +3   (one 128-bit load)
//   VEC == 1 : element k is lig + k*G                         (scalar loads)
//
// Numerics (quant.py:89-138):
//   * "exact" helpers reproduce the reference float64 arithmetic bit for bit
//     with explicit __d*_rn intrinsics (never contracted into FMA);
//   * "fast" helpers run in fp32 and return a certified error bound; a
//     decision whose margin is below the bound is re-taken exactly.  Only the
//     decisions feed the output, so the output equals the exact one.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/deltasnap_cuda.h"

#define DS_FULL_MASK 0xffffffffu
#define DS_MAX_TABLES 64
#define DS_HEADER_SIZE 24
#define DS_FP32_TAG 32

namespace ds {

// Programmatic dependent launch (K1 -> K2 count -> K2 emit -> K3 on one
// stream): a kernel lets its successor launch as soon as its own CTAs are all
// resident, the successor's CTAs take the SMs its tail frees, and wait here
// until it has completed and its writes are visible.  Both are no-ops for a
// launch without the PDL attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

constexpr float kU = 5.9604644775390625e-08f;  // 2^-24, unit roundoff of fp32

// ---------------------------------------------------------------------------
// group reductions (width G shuffles; every lane of the warp participates)
// ---------------------------------------------------------------------------
template <int G>
__device__ __forceinline__ float grp_min(float v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(DS_FULL_MASK, v, o, G));
    return v;
}
template <int G>
__device__ __forceinline__ float grp_max(float v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(DS_FULL_MASK, v, o, G));
    return v;
}
template <int G>
__device__ __forceinline__ float grp_sum(float v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(DS_FULL_MASK, v, o, G);
    return v;
}
template <int G>
__device__ __forceinline__ double grp_sumd(double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(DS_FULL_MASK, v, o, G);
    return v;
}
template <int G>
__device__ __forceinline__ int grp_or(int v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v |= __shfl_xor_sync(DS_FULL_MASK, v, o, G);
    return v;
}

template <int G>
constexpr int log2i() { return G <= 1 ? 0 : 1 + log2i<G / 2>(); }

// min/max that return NaN when either input is NaN (PTX .NaN, sm_80+)
__device__ __forceinline__ float fmin_nan(float a, float b) {
    float r;
    asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float fmax_nan(float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}

// ---------------------------------------------------------------------------
// element layout
// ---------------------------------------------------------------------------
template <int G, int C, int VEC>
struct Layout {
    static constexpr int EPL = C * VEC;
    __device__ __forceinline__ static int elem(int lig, int k) {
        if (VEC == 4) return 4 * (lig + (k >> 2) * G) + (k & 3);
        return lig + k * G;
    }
};

// Load one row (values + row*ld) into registers; padding elements get `pad`.
template <int G, int C, int VEC>
__device__ __forceinline__ void load_row(const float *__restrict__ row, int d, int lig,
                                         float (&x)[C * VEC], float pad) {
    if (VEC == 4) {
#pragma unroll
        for (int c = 0; c < C; c++) {
            int e = 4 * (lig + c * G);
            if (e < d) {
                float4 v = __ldg(reinterpret_cast<const float4 *>(row + e));
                x[4 * c + 0] = v.x;
                x[4 * c + 1] = v.y;
                x[4 * c + 2] = v.z;
                x[4 * c + 3] = v.w;
            } else {
                x[4 * c + 0] = x[4 * c + 1] = x[4 * c + 2] = x[4 * c + 3] = pad;
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < C; k++) {
            int e = lig + k * G;
            x[k] = e < d ? __ldg(row + e) : pad;
        }
    }
}

// ---------------------------------------------------------------------------
// exact reference arithmetic (quant.py:89-115)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double scale64(float lo, float hi, int L) {
    return __ddiv_rn(__dsub_rn((double)hi, (double)lo), (double)L);  // _scales :89-90
}

// quantize_rows element: clip (PyArray_MAX/MIN), true f64 division,
// floor(v + 0.5), clip to [0, L] (quant.py:99-106).
__device__ __forceinline__ int code_exact(float x, float lo, float hi, double s, int L) {
    double safe = s > 0.0 ? s : 1.0;
    float c = x > lo ? x : lo;
    c = c < hi ? c : hi;
    double v = __ddiv_rn(__dsub_rn((double)c, (double)lo), safe);
    double q = floor(__dadd_rn(v, 0.5));
    q = q < 0.0 ? 0.0 : q;
    q = q > (double)L ? (double)L : q;
    return (int)q;
}

// dequantize_rows element: two rounded f64 ops, then f32 (quant.py:114-115).
__device__ __forceinline__ float deq_exact(int q, float lo, double s) {
    return __double2float_rn(__dadd_rn(__dmul_rn(s, (double)q), (double)lo));
}

// ---------------------------------------------------------------------------
// the err_sum term without the conversion unit.  F2F (f32<->f64) issues at
// ~1/8 of the FP32 rate on B200 (scripts/micro/pipe_rates.cu: ~0.5 warp
// instructions per clock per SM vs ~3.7 for FFMA and ~1.95 for DFMA), and the
// reference error of an element (engine.py:171-173: f64(x) - f64(deq32))
// needs four of them.  Here the same value comes from integer bit arithmetic
// and half-rate f64 ops only.
// ---------------------------------------------------------------------------
// f32 -> f64 by bit arithmetic: exact for normal x; +-0 and subnormals land
// within 2^-126 of their value (rows whose range makes that matter take the
// exact path, RowQ mode 2)
__device__ __forceinline__ double f2d_bits(float x) {
    const uint32_t b = __float_as_uint(x);
    const uint32_t hi = (((b >> 3) & 0x0FFFFFFFu) + 0x38000000u) | (b & 0x80000000u);
    return __hiloint2double((int)hi, (int)(b << 29));
}
// RN-even to float precision of a double in the f32 normal range, kept as a
// double: add (half an f32 ulp - 1 + kept lsb) to the 64-bit pattern, truncate
__device__ __forceinline__ double round_f32_in_f64(double w) {
    uint32_t lo = (uint32_t)__double2loint(w), hi = (uint32_t)__double2hiint(w);
    const uint32_t add = 0x0FFFFFFFu + ((lo >> 29) & 1u);
    asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, 0;" : "+r"(lo), "+r"(hi) : "r"(add));
    return __hiloint2double((int)hi, (int)(lo & 0xE0000000u));
}
// a code (0..255) as a double, exactly, through the 2^52 magic (one DADD)
__device__ __forceinline__ double code_to_f64(uint32_t q) {
    return __dsub_rn(__hiloint2double(0x43300000, (int)q), 4503599627370496.0);
}
// x - deq(q) of the reference, as a double: deq(q) = f32(RN(RN(s*q) + lo))
// (quant.py:114-115, two rounded ops), x and deq exact in f64
__device__ __forceinline__ double err_fast(float x, uint32_t q, double s, double lod) {
    const double w = __dadd_rn(__dmul_rn(s, code_to_f64(q)), lod);
    return __dsub_rn(f2d_bits(x), round_f32_in_f64(w));
}
// a row's L2 error from its f64 sum of squares; sums below 2^-200 (only the
// +-2^-127 stand-ins of exact zeros, or errors < 2^-100) count as 0
__device__ __forceinline__ double row_err(double sse) {
    return sse > 0x1p-200 ? sse * rsqrt(sse) : 0.0;
}

// ---------------------------------------------------------------------------
// final codes of a row with fixed (lo, hi): fp32 guard band + exact fallback
// ---------------------------------------------------------------------------
#ifndef DS_RCP_RN
#define DS_RCP_RN 0
#endif
struct RowQ {
    float lo, hi, inv, eps;
    double s;
    int L;
    int mode;  // 0 fast, 1 all-zero (degenerate range), 2 exact every element
};

// scale64 without a division: with y = RN(1/L) (host-computed), q0 = RN(a*y),
// the remainder a - q0*L is exact in one FMA, and RN(q0 + rem*y) is the
// correctly rounded a/L (Markstein's correction; checked on 79M random f32
// ranges against true division, tests/test_gpu_parity.py covers it on device).
__device__ __forceinline__ double scale64_y(float lo, float hi, double L, double y) {
    double a = __dsub_rn((double)hi, (double)lo);
    double q0 = __dmul_rn(a, y);
    double rem = __fma_rn(-q0, L, a);
    return __fma_rn(rem, y, q0);
}

__device__ __forceinline__ RowQ make_rowq(float lo, float hi, int L, double y = 0.0) {
    RowQ r;
    r.lo = lo;
    r.hi = hi;
    r.L = L;
    r.s = y != 0.0 ? scale64_y(lo, hi, (double)L, y) : scale64(lo, hi, L);
    float rng = __fsub_rn(hi, lo);
    r.inv = 0.f;
    r.eps = 0.f;
    if (!(r.s > 0.0)) {
        r.mode = 1;  // scale 0 -> safe 1 -> v = 0 -> code 0 (quant.py:101-106)
    } else if (!(rng >= 1e-21f && rng <= 1e30f && fabsf(lo) <= 1e30f && fabsf(hi) <= 1e30f)) {
        // (range >= 1e-21: also keeps err_fast's +-0 / subnormal stand-ins
        // below 1e-14 of the row's error)
        r.mode = 2;
    } else {
        r.mode = 0;
        // inv = L/rng via the hardware reciprocal (MUFU.RCP, rel. error <=
        // 2^-23 = 2u) and one product: rel. error <= 4u (rng, rcp, mul); with
        // c-lo and v = t*inv that is |v_fast - v_ref| <= 6u*L, covered by the
        // 8u*L guard band (DS_RCP_RN=1: the correctly rounded reciprocal, 5u*L)
#if DS_RCP_RN
        r.inv = __fmul_rn(__frcp_rn(rng), (float)L);
#else
        float rc;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(rng));
        r.inv = __fmul_rn(rc, (float)L);
#endif
        r.eps = 8.f * kU * (float)L;
    }
    return r;
}

// The rare exact recomputation stays out of line so the fast path keeps its
// registers (an inlined f64 division per element doubles the kernel's count).
static __device__ __noinline__ int code_exact_slow(float x, float lo, float hi, double s, int L) {
    return code_exact(x, lo, hi, s, L);
}

// Returns the reference code of x.  `nexact` counts exact recomputations.
__device__ __forceinline__ int code_of(float x, const RowQ &r, unsigned &nexact) {
    if (r.mode == 1) return 0;
    if (r.mode == 0) {
        float c = fminf(fmaxf(x, r.lo), r.hi);
        float v = __fmul_rn(__fsub_rn(c, r.lo), r.inv);
        float q = rintf(v);
        if (fabsf(__fsub_rn(v, q)) <= 0.5f - r.eps) return (int)q;
    }
    nexact++;
    return code_exact_slow(x, r.lo, r.hi, r.s, r.L);
}

// ---------------------------------------------------------------------------
// numpy pairwise summation on shared memory (loops_utils.h.src; the order of
// np.linalg.norm at quant.py:138).  Single-thread forms.
// ---------------------------------------------------------------------------
static __device__ double pw_block(const double *a, int n) {
    if (n < 8) {
        double res = -0.0;
        for (int i = 0; i < n; i++) res = __dadd_rn(res, a[i]);
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = a[j];
    int i;
    for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[i + j]);
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; i++) res = __dadd_rn(res, a[i]);
    return res;
}

static __device__ double pw_sum(const double *a, int n) {
    // explicit stack instead of recursion: leaves of <= 128 elements combined
    // in the same binary-tree order numpy's recursion uses.
    if (n <= 128) return pw_block(a, n);
    struct Frame {
        int off, n, state;
        double left;
    };
    Frame st[24];
    int sp = 0;
    st[0] = {0, n, 0, 0.0};
    double ret = 0.0;
    while (true) {
        Frame &f = st[sp];
        if (f.n <= 128) {
            ret = pw_block(a + f.off, f.n);
            if (sp == 0) return ret;
            sp--;
            continue;
        }
        int n2 = f.n / 2;
        n2 -= n2 % 8;
        if (f.state == 0) {  // descend left
            f.state = 1;
            st[sp + 1] = {f.off, n2, 0, 0.0};
            sp++;
        } else if (f.state == 1) {  // left done -> descend right
            f.left = ret;
            f.state = 2;
            st[sp + 1] = {f.off + n2, f.n - n2, 0, 0.0};
            sp++;
        } else {  // both done
            ret = __dadd_rn(f.left, ret);
            if (sp == 0) return ret;
            sp--;
        }
    }
}

// ---------------------------------------------------------------------------
// exact ME of one candidate for every group of a warp (warp-collective).
// `buf` points at this group's scratch of >= d doubles (+8 for r[]).
// Lanes whose group has want == false still take part in the syncs.
// ---------------------------------------------------------------------------
template <int G, int C, int VEC>
__device__ __forceinline__ double exact_me_impl(const float (&x)[C * VEC], int d, int lig,
                                                float lo, float hi, int L, bool want,
                                                double *buf, unsigned &nexact_codes) {
    using Lay = Layout<G, C, VEC>;
    constexpr int EPL = C * VEC;
    if (want) {
        RowQ rq = make_rowq(lo, hi, L);
#pragma unroll
        for (int k = 0; k < EPL; k++) {
            int e = Lay::elem(lig, k);
            if (e < d) {
                int q = code_of(x[k], rq, nexact_codes);
                float dq = deq_exact(q, lo, rq.s);
                double err = __dsub_rn((double)x[k], (double)dq);
                buf[e] = __dmul_rn(err, err);
            }
        }
    }
    __syncwarp();
    double res = 0.0;
    if (d <= 128 && d >= 8) {
        // accumulator j (< 8) handled by lane j % G of the group
        if (want) {
            for (int j = lig; j < 8; j += G) {
                double r = buf[j];
                for (int i = 8; i < d - (d % 8); i += 8) r = __dadd_rn(r, buf[i + j]);
                buf[d + j] = r;
            }
        }
        __syncwarp();
        if (want && lig == 0) {
            const double *r = buf + d;
            res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                            __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
            for (int i = d - (d % 8); i < d; i++) res = __dadd_rn(res, buf[i]);
        }
    } else {
        if (want && lig == 0) res = pw_sum(buf, d);
        __syncwarp();
    }
    __syncwarp();
    // broadcast from the group leader
    int lane = threadIdx.x & 31;
    res = __shfl_sync(DS_FULL_MASK, res, lane & ~(G - 1));
    return __dsqrt_rn(res);
}

template <int G, int C, int VEC>
__device__ __noinline__ double exact_me_group(const float (&x)[C * VEC], int d, int lig,
                                              float lo, float hi, int L, bool want,
                                              double *buf, unsigned &nexact_codes) {
    return exact_me_impl<G, C, VEC>(x, d, lig, lo, hi, L, want, buf, nexact_codes);
}

// the same from the group's row in shared memory (Layout order at `row`)
template <int G, int C, int VEC>
__device__ __noinline__ double exact_me_row(const float *row, int d, int lig, float lo, float hi,
                                            int L, bool want, double *buf, unsigned &nexact_codes) {
    using Lay = Layout<G, C, VEC>;
    float x[C * VEC];
#pragma unroll
    for (int k = 0; k < C * VEC; k++) {
        const int e = Lay::elem(lig, k);
        x[k] = e < d ? row[e] : 0.f;
    }
    return exact_me_impl<G, C, VEC>(x, d, lig, lo, hi, L, want, buf, nexact_codes);
}

// ---------------------------------------------------------------------------
// packed fp32 pairs (sm_100a FADD2 / FMUL2 / FFMA2: two lanes of fp32 per
// instruction, IEEE round-to-nearest like the scalar ops)
// ---------------------------------------------------------------------------
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float a, float b) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void up2(f32x2 v, float &a, float &b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// ---------------------------------------------------------------------------
// certified fast ME^2 of one candidate (fp32), see DESIGN.md "numerics".
// Returns S (sum of squares, fp32 accumulation) and B with |S - S_ref| <= B,
// where S_ref is the reference's float64 sum for the same candidate.
// ---------------------------------------------------------------------------
template <int G, int C, int VEC, bool PAD>
__device__ __forceinline__ void eval_fast(const float (&x)[C * VEC], int d, int lig, float lo,
                                          float hi, int L, float &S, float &B) {
    using Lay = Layout<G, C, VEC>;
    constexpr int EPL = C * VEC;
    float rng = __fsub_rn(hi, lo);
    float M = fmaxf(fabsf(lo), fabsf(hi));
    bool ok = rng >= 1e-30f && rng <= 1e30f && M <= 1e30f;
    float inv = ok ? __fdividef((float)L, rng) : 0.f;
    float s32 = __fmul_rn(rng, 1.0f / (float)L);
    float sse = 0.f, rmax = 0.f;
#pragma unroll
    for (int k = 0; k < EPL; k++) {
        float c = fminf(fmaxf(x[k], lo), hi);
        float v = __fmul_rn(__fsub_rn(c, lo), inv);
        float q = rintf(v);
        rmax = fmaxf(rmax, fabsf(__fsub_rn(v, q)));
        float dq = __fmaf_rn(q, s32, lo);
        float e = __fsub_rn(x[k], dq);
        if (PAD) e = Lay::elem(lig, k) < d ? e : 0.f;
        sse = __fmaf_rn(e, e, sse);
    }
    S = grp_sum<G>(sse);
    rmax = grp_max<G>(rmax);
    if (!ok) {
        B = INFINITY;
        return;
    }
    float fd = (float)d;
    float delta = 16.f * kU * M + 1e-44f;                // |deq_fast - deq_ref|
    float epsw = 10.f * kU * (float)L;                   // |v_fast - v_ref|
    float b = 2.f * delta * sqrtf(fd * S) + 2.f * fd * delta * delta +
              (float)(EPL + log2i<G>() + 4) * kU * S;
    if (rmax > 0.5f - epsw) b += fd * 4.f * s32 * (epsw * s32 + 2.f * delta);  // code ties
    B = 1.5f * b + 1e-37f;
}

// Both candidates of a greedy step in one pass over the row: two independent
// accumulation chains per element (ILP), one loop over the registers.  Same
// arithmetic and bounds as two eval_fast calls.
#ifndef DS_GREEDY_NO_TIES
#define DS_GREEDY_NO_TIES 0
#endif
#ifndef DS_GREEDY_PACKED
#define DS_GREEDY_PACKED 1  // both candidates in packed fp32 pairs (FADD2/FMUL2/FFMA2)
#endif
template <int G, int C, int VEC, bool PAD>
__device__ __forceinline__ void eval_fast2(const float (&x)[C * VEC], int d, int lig, float loA,
                                           float hiA, float loB, float hiB, int L, float &SA,
                                           float &BA, float &SB, float &BB) {
    using Lay = Layout<G, C, VEC>;
    constexpr int EPL = C * VEC;
    const float rngA = __fsub_rn(hiA, loA), rngB = __fsub_rn(hiB, loB);
    const float MA = fmaxf(fabsf(loA), fabsf(hiA)), MB = fmaxf(fabsf(loB), fabsf(hiB));
    const bool okA = rngA >= 1e-30f && rngA <= 1e30f && MA <= 1e30f;
    const bool okB = rngB >= 1e-30f && rngB <= 1e30f && MB <= 1e30f;
    const float invA = okA ? __fdividef((float)L, rngA) : 0.f;
    const float invB = okB ? __fdividef((float)L, rngB) : 0.f;
    const float sA = __fmul_rn(rngA, 1.0f / (float)L), sB = __fmul_rn(rngB, 1.0f / (float)L);
    float sseA = 0.f, sseB = 0.f, rmA = 0.f, rmB = 0.f;
#if DS_GREEDY_PACKED
    // both candidates in the two halves of packed fp32 pairs (rint as the
    // 1.5*2^23 magic add: round half to even for v in [0, L(1+5u)])
    {
        const f32x2 LO = pk2(loA, loB), INV = pk2(invA, invB), S2 = pk2(sA, sB);
        const f32x2 MAG = pk2(12582912.0f, 12582912.0f);
        f32x2 sse = pk2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < EPL; k++) {
            const float cA = fminf(fmaxf(x[k], loA), hiA);
            const float cB = fminf(fmaxf(x[k], loB), hiB);
            // the product fused into the rounding and the distance (ptxas
            // contracts f32x2 mul+add anyway; explicit FMAs make it defined):
            // |t*inv - v_ref| is within the bound's epsw like the rounded v
            const f32x2 t = sub2(pk2(cA, cB), LO);
            const f32x2 qm = fma2(t, INV, MAG);
            const f32x2 q = sub2(qm, MAG);
            float rA, rB;
            up2(fma2(t, INV, sub2(MAG, qm)), rA, rB);
            if (!DS_GREEDY_NO_TIES) {
                rmA = fmaxf(rmA, fabsf(rA));
                rmB = fmaxf(rmB, fabsf(rB));
            } else {
                rmA = rmB = 1.f;
            }
            f32x2 e = sub2(pk2(x[k], x[k]), fma2(q, S2, LO));
            if (PAD && !(Lay::elem(lig, k) < d)) e = pk2(0.f, 0.f);
            sse = fma2(e, e, sse);
        }
        // group sums of both candidates in one packed add per level (the
        // scalar path's order: each value plus its xor partner)
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            float a, b;
            up2(sse, a, b);
            sse = add2(sse, pk2(__shfl_xor_sync(DS_FULL_MASK, a, o, G), __shfl_xor_sync(DS_FULL_MASK, b, o, G)));
        }
        up2(sse, sseA, sseB);
    }
    // a code tie anywhere in the group: one ballot per candidate
    const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
    const bool tieA = (__ballot_sync(DS_FULL_MASK, rmA > 0.5f - 10.f * kU * (float)L) & gmask) != 0u;
    const bool tieB = (__ballot_sync(DS_FULL_MASK, rmB > 0.5f - 10.f * kU * (float)L) & gmask) != 0u;
#else
#pragma unroll
    for (int k = 0; k < EPL; k++) {
        const float cA = fminf(fmaxf(x[k], loA), hiA);
        const float cB = fminf(fmaxf(x[k], loB), hiB);
        const float vA = __fmul_rn(__fsub_rn(cA, loA), invA);
        const float vB = __fmul_rn(__fsub_rn(cB, loB), invB);
        const float qA = rintf(vA), qB = rintf(vB);
        if (!DS_GREEDY_NO_TIES) {
            rmA = fmaxf(rmA, fabsf(__fsub_rn(vA, qA)));
            rmB = fmaxf(rmB, fabsf(__fsub_rn(vB, qB)));
        } else {
            rmA = rmB = 1.f;  // always budget for code ties (no per-element tracking)
        }
        float eA = __fsub_rn(x[k], __fmaf_rn(qA, sA, loA));
        float eB = __fsub_rn(x[k], __fmaf_rn(qB, sB, loB));
        if (PAD) {
            const bool in = Lay::elem(lig, k) < d;
            eA = in ? eA : 0.f;
            eB = in ? eB : 0.f;
        }
        sseA = __fmaf_rn(eA, eA, sseA);
        sseB = __fmaf_rn(eB, eB, sseB);
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
        sseA += __shfl_xor_sync(DS_FULL_MASK, sseA, o, G);
        sseB += __shfl_xor_sync(DS_FULL_MASK, sseB, o, G);
        rmA = fmaxf(rmA, __shfl_xor_sync(DS_FULL_MASK, rmA, o, G));
        rmB = fmaxf(rmB, __shfl_xor_sync(DS_FULL_MASK, rmB, o, G));
    }
    const bool tieA = rmA > 0.5f - 10.f * kU * (float)L, tieB = rmB > 0.5f - 10.f * kU * (float)L;
#endif
    SA = sseA;
    SB = sseB;
    const float fd = (float)d;
    const float epsw = 10.f * kU * (float)L;  // |v_fast - v_ref|
    auto bound = [&](float S, float M, float s32, bool tie, bool ok) -> float {
        if (!ok) return INFINITY;
        const float delta = 16.f * kU * M + 1e-44f;  // |deq_fast - deq_ref|
        float b = 2.f * delta * sqrtf(fd * S) + 2.f * fd * delta * delta +
                  (float)(EPL + log2i<G>() + 4) * kU * S;
        if (tie) b += fd * 4.f * s32 * (epsw * s32 + 2.f * delta);  // code ties
        return 1.5f * b + 1e-37f;
    };
    BA = bound(SA, MA, sA, tieA, okA);
    BB = bound(SB, MB, sB, tieB, okB);
}

// ---------------------------------------------------------------------------
// greedy range search of one row per group (quant.py:160-209), certified.
// All lanes of the warp must call it (exact re-evaluation is warp-collective).
// ---------------------------------------------------------------------------
struct Cand {
    float lo, hi, S, B;
    double me;    // exact ME when has_me
    bool has_me;
};

#ifndef DS_GREEDY_LEAN
#define DS_GREEDY_LEAN 1  // decisions: certified fast path, exact bookkeeping behind one warp vote
#endif
template <int G, int C, int VEC, bool PAD>
__device__ __forceinline__ void greedy_row(const float (&x)[C * VEC], int d, int lig, bool row_ok,
                                           float lo0, float hi0, int L, int bins, int steps,
                                           double *buf, float &out_lo, float &out_hi,
                                           unsigned &n_exact_dec, unsigned &n_exact_codes) {
#if DS_GREEDY_LEAN
    // the reference's decisions (take_a = me_a <= me_b, quant.py:198;
    // improved = me_cur < best_me, :204) from certified fp32 intervals; a
    // comparison whose intervals overlap is re-taken with exact MEs
    // (exact_me_group), the cached exact ME of `best` reused while it stands
    const double full = __dsub_rn((double)hi0, (double)lo0);
    const double step = __ddiv_rn(full, (double)bins);
    float best_lo = lo0, best_hi = hi0, best_S, best_B;
    double best_me = 0.0;
    bool best_has_me = false;
    eval_fast<G, C, VEC, PAD>(x, d, lig, lo0, hi0, L, best_S, best_B);
    double cur_lo = (double)lo0, cur_hi = (double)hi0;
    bool active = row_ok && step > 0.0;
    for (int it = 0; it < steps; it++) {
        active = active && (__dsub_rn(__dsub_rn(cur_hi, cur_lo), step) > 0.0);
        if (!__any_sync(DS_FULL_MASK, active)) break;
        const float a_lo = __double2float_rn(__dadd_rn(cur_lo, step)), a_hi = __double2float_rn(cur_hi);
        const float b_lo = __double2float_rn(cur_lo), b_hi = __double2float_rn(__dsub_rn(cur_hi, step));
        float SA, BA, SB, BB;
        eval_fast2<G, C, VEC, PAD>(x, d, lig, a_lo, a_hi, b_lo, b_hi, L, SA, BA, SB, BB);
        const bool ta_yes = SA + BA < SB - BB, ta_no = SA - BA > SB + BB;
        bool take_a = !ta_no;
        float Sc = take_a ? SA : SB, Bc = take_a ? BA : BB;
        const bool imp_yes = Sc + Bc < best_S - best_B, imp_no = Sc - Bc > best_S + best_B;
        bool improved = imp_yes;
        double me_c = 0.0;
        bool c_has = false;
        if (__any_sync(DS_FULL_MASK, active && !((ta_yes || ta_no) && (imp_yes || imp_no)))) {
            const bool need_t = active && !(ta_yes || ta_no);
            if (__any_sync(DS_FULL_MASK, need_t)) {
                const double ma = exact_me_group<G, C, VEC>(x, d, lig, a_lo, a_hi, L, need_t, buf, n_exact_codes);
                const double mb = exact_me_group<G, C, VEC>(x, d, lig, b_lo, b_hi, L, need_t, buf, n_exact_codes);
                if (need_t) {
                    take_a = ma <= mb;
                    me_c = take_a ? ma : mb;
                    c_has = true;
                    if (lig == 0) n_exact_dec++;
                }
            }
            Sc = take_a ? SA : SB;
            Bc = take_a ? BA : BB;
            const bool iy = Sc + Bc < best_S - best_B, in_ = Sc - Bc > best_S + best_B;
            improved = iy;
            const bool undecided = active && !(iy || in_);
            const float c_lo = take_a ? a_lo : b_lo, c_hi = take_a ? a_hi : b_hi;
            const bool need_c = undecided && !c_has, need_b = undecided && !best_has_me;
            if (__any_sync(DS_FULL_MASK, need_c)) {
                const double m = exact_me_group<G, C, VEC>(x, d, lig, c_lo, c_hi, L, need_c, buf, n_exact_codes);
                if (need_c) {
                    me_c = m;
                    c_has = true;
                }
            }
            if (__any_sync(DS_FULL_MASK, need_b)) {
                const double m = exact_me_group<G, C, VEC>(x, d, lig, best_lo, best_hi, L, need_b, buf, n_exact_codes);
                if (need_b) {
                    best_me = m;
                    best_has_me = true;
                }
            }
            if (undecided) {
                improved = me_c < best_me;
                if (lig == 0) n_exact_dec++;
            }
        }
        if (active) {
            if (take_a) cur_lo = __dadd_rn(cur_lo, step);
            else cur_hi = __dsub_rn(cur_hi, step);
            if (improved) {
                best_lo = take_a ? a_lo : b_lo;
                best_hi = take_a ? a_hi : b_hi;
                best_S = Sc;
                best_B = Bc;
                best_me = me_c;
                best_has_me = c_has;
            }
        }
    }
    out_lo = best_lo;
    out_hi = best_hi;
#else

    double full = __dsub_rn((double)hi0, (double)lo0);
    double step = __ddiv_rn(full, (double)bins);
    Cand best;
    best.lo = lo0;
    best.hi = hi0;
    best.has_me = false;
    best.me = 0.0;
    eval_fast<G, C, VEC, PAD>(x, d, lig, lo0, hi0, L, best.S, best.B);
    double cur_lo = (double)lo0, cur_hi = (double)hi0;
    bool active = row_ok && step > 0.0;
    for (int it = 0; it < steps; it++) {
        active = active && (__dsub_rn(__dsub_rn(cur_hi, cur_lo), step) > 0.0);
        if (!__any_sync(DS_FULL_MASK, active)) break;
        Cand a, b;
        a.lo = __double2float_rn(__dadd_rn(cur_lo, step));
        a.hi = __double2float_rn(cur_hi);
        b.lo = __double2float_rn(cur_lo);
        b.hi = __double2float_rn(__dsub_rn(cur_hi, step));
        a.has_me = b.has_me = false;
        a.me = b.me = 0.0;
        eval_fast2<G, C, VEC, PAD>(x, d, lig, a.lo, a.hi, b.lo, b.hi, L, a.S, a.B, b.S, b.B);
        // take_a = me_a <= me_b (quant.py:198)
        bool take_a = true;
        bool sure = true;
        if (a.S + a.B < b.S - b.B) take_a = true;
        else if (a.S - a.B > b.S + b.B) take_a = false;
        else sure = false;
        bool need = active && !sure;
        if (__any_sync(DS_FULL_MASK, need)) {
            double ma = exact_me_group<G, C, VEC>(x, d, lig, a.lo, a.hi, L, need, buf,
                                                  n_exact_codes);
            double mb = exact_me_group<G, C, VEC>(x, d, lig, b.lo, b.hi, L, need, buf,
                                                  n_exact_codes);
            if (need) {
                a.me = ma;
                b.me = mb;
                a.has_me = b.has_me = true;
                take_a = ma <= mb;
                if (lig == 0) n_exact_dec++;
            }
        }
        // no `continue` for inactive rows: the exact paths below are
        // warp-collective, so every lane walks the same control flow.
        if (active) {
            if (take_a) cur_lo = __dadd_rn(cur_lo, step);
            else cur_hi = __dsub_rn(cur_hi, step);
        }
        Cand c = take_a ? a : b;
        // improved = active & (me_cur < best_me) (quant.py:204)
        bool improved = false;
        sure = true;
        if (!active) improved = false;
        else if (c.has_me && best.has_me) improved = c.me < best.me;
        else if (c.S + c.B < best.S - best.B) improved = true;
        else if (c.S - c.B > best.S + best.B) improved = false;
        else sure = false;
        need = !sure;
        // exact evaluation of whichever side lacks an exact value
        bool need_c = need && !c.has_me, need_b = need && !best.has_me;
        if (__any_sync(DS_FULL_MASK, need_c)) {
            double m = exact_me_group<G, C, VEC>(x, d, lig, c.lo, c.hi, L, need_c, buf,
                                                 n_exact_codes);
            if (need_c) { c.me = m; c.has_me = true; }
        }
        if (__any_sync(DS_FULL_MASK, need_b)) {
            double m = exact_me_group<G, C, VEC>(x, d, lig, best.lo, best.hi, L, need_b, buf,
                                                 n_exact_codes);
            if (need_b) { best.me = m; best.has_me = true; }
        }
        if (need) {
            improved = c.me < best.me;
            if (lig == 0) n_exact_dec++;
        }
        if (improved) best = c;
    }
    out_lo = best.lo;
    out_hi = best.hi;
#endif
}

}  // namespace ds
