// ds_greedy.cuh -- the adaptive greedy range search (quant.py:160-209) by
// bucket sums instead of per-element candidate passes.
//
// The reference evaluates every candidate range with a full pass over the
// row (reconstruction_errors, quant.py:134-138): 2*floor(bins*ratio)+1
// passes of d elements.  Here a row is sorted once, and a candidate's error
// comes from its L code boundaries alone.  With the row sorted ascending,
// y_i = x_i - lo0 (lo0 = row min, so y >= 0), prefix sums P[i] = sum_{j<i} y_j,
// Q = sum y^2, and d_k = D_k - lo0 for the candidate's L+1 dequantized levels
// D_k = f32(RN(RN(s*k) + lo)) (quant.py:114-115, exact), the codes are a step
// function of the sorted index: code k for i in [idx_k, idx_{k+1}), idx_k =
// #{x < t_k}, t_k = lo + (k - 1/2) s the k-th code transition
// (floor((c - lo)/s + 1/2), quant.py:103-105; clipping puts every x < lo in
// code 0 and every x > hi in code L, which the same step function does).
// Telescoping the bucket sums,
//   SSE = sum_i (y_i - d_{q_i})^2
//       = Q - 2 d_L P[d] + d d_L^2
//         + sum_{k=1..L} (d_{k-1} - d_k) ((d_{k-1} + d_k) idx_k - 2 P[idx_k]),
// one term per boundary: O(L log) per candidate instead of O(d).
//
// Certification (the decisions must equal the reference's):
//   * SSE is computed in f64 with an absolute bound B = gamma * A, A a bound
//     on the magnitudes of every term (prefix sums of nonnegative y, Q, the
//     per-boundary products), gamma = (2d + 2L + 64) 2^-53 -- covering the
//     prefix-sum, level and product roundings and the reference's own
//     pairwise-summation error -- plus 2^-48 |SSE| so that a certified strict
//     order of two SSEs survives the reference's sqrt (quant.py:138).
//   * idx_k is exact unless an element lies within eps_k of t_k, where the
//     reference's f64 code arithmetic (3 roundings) could put it on either
//     side: eps_k = 2^-50 ((L+1) s + |t_k|).  In the sorted row the nearest
//     elements to t_k are xs[idx_k - 1] and xs[idx_k]; if either is within
//     eps_k (plus |t_k - f32(t_k)|), the candidate is uncertain.
//   * an uncertain candidate, or two candidates whose SSE intervals overlap,
//     are re-evaluated exactly (exact_me_group: the reference's per-element
//     f64 arithmetic and numpy's pairwise order), as in the fp32 path.
//
// Sorting: a bitonic network over the group's registers (no data-dependent
// control flow); beside it a histogram of the values over F = 2*DP cells of
// the row's range (a monotone cell function) gives each cell's end index, so
// a boundary's index is its cell's start plus a binary search inside the cell
// (about half an element per cell).  The bound A uses the row constant
// Q + (8L + 3) d Rm^2 >= every term's magnitude (y, d_k <= Rm = range + slack).
#pragma once

#include <type_traits>

#include "ds_common.cuh"

#ifndef DS_GREEDY_BUCKET
#define DS_GREEDY_BUCKET 0  // 1: bucketed search (measured slower); 0: fp32 candidate passes
#endif

namespace ds {

__host__ __device__ constexpr int bk_align16(int v) { return (v + 15) & ~15; }

// per-row scratch of the bucketed search, DP = padded dim of the layout
template <int DP>
struct BucketLayout {
    static constexpr int F = 2 * DP;  // cells
    using Tab = typename std::conditional<(DP <= 255), uint8_t, uint16_t>::type;
    static constexpr int XS_OFF = 0;                                  // float[DP] sorted row
    static constexpr int P_OFF = bk_align16(4 * DP);                  // double[DP+1] prefix sums
    static constexpr int TAB_OFF = bk_align16(P_OFF + 8 * (DP + 1));  // Tab[F+1]: 0, cell ends
    static constexpr int RAW = bk_align16(TAB_OFF + (F + 1) * (int)sizeof(Tab));
    // the exact re-evaluation (exact_me_group) borrows the scratch: d + 8 doubles
    static constexpr int BYTES = RAW > 8 * (DP + 8) ? RAW : bk_align16(8 * (DP + 8));
    static_assert(4 * F <= 8 * (DP + 1), "the build's u32 cell counts live in the prefix-sum area");
};

__host__ __device__ constexpr int bucket_bytes(int dp) {
    return (bk_align16(bk_align16(bk_align16(4 * dp) + 8 * (dp + 1)) + (2 * dp + 1) * (dp <= 255 ? 1 : 2)) >
            8 * (dp + 8))
               ? bk_align16(bk_align16(bk_align16(4 * dp) + 8 * (dp + 1)) + (2 * dp + 1) * (dp <= 255 ? 1 : 2))
               : bk_align16(8 * (dp + 8));
}

// per-row greedy scratch of the writers: the bucketed search's layout, or
// the exact evaluation's d + 8 doubles (numpy pairwise order)
__host__ __device__ constexpr int greedy_scratch_bytes(int dp, int d) {
    return DS_GREEDY_BUCKET ? bucket_bytes(dp) : (d + 8) * 8;
}

// monotone cell of a value: x1 <= x2 -> cell(x1) <= cell(x2) (RN subtraction
// and product by invw >= 0 are monotone, so are the clamp and truncation)
__device__ __forceinline__ int bk_cell(float x, float lo0, float invw, int F) {
    float p = __fmul_rn(__fsub_rn(x, lo0), invw);
    p = fminf(fmaxf(p, 0.f), (float)(F - 1));  // NaN (0 * inf) -> 0
    return __float2int_rz(p);
}

// Bitonic sort of the group's row (DP values, padding as +inf) in registers:
// value i = lig*EPL + j lives in lane lig, register j.  Every merge of size k
// starts by comparing i with its mirror i ^ (k-1), then half-cleans with
// strides k/4 .. 1, so every compare keeps the minimum at the lower index
// (no per-lane sort direction).  Strides >= EPL pair lanes (shuffles),
// smaller ones registers.  No data-dependent control flow.
template <int G, int EPL>
__device__ __forceinline__ void bitonic_group(float (&v)[EPL], int lig) {
    constexpr int DP = G * EPL;
#pragma unroll
    for (int k = 2; k <= DP; k <<= 1) {
        // mirror stage
        if (k <= EPL) {
#pragma unroll
            for (int j = 0; j < EPL; j++) {
                const int p = j ^ (k - 1);
                if (p > j) {
                    const float a = v[j], b = v[p];
                    v[j] = fminf(a, b);
                    v[p] = fmaxf(a, b);
                }
            }
        } else {
            const int m = k / EPL - 1;              // partner lane = lig ^ m
            const bool low = !(lig & (k / EPL / 2));  // this lane holds the lower indices
#pragma unroll
            for (int j = 0; j < EPL / 2; j++) {
                const int p = EPL - 1 - j;
                const float oj = __shfl_xor_sync(DS_FULL_MASK, v[p], m, G);  // partner's EPL-1-j
                const float op = __shfl_xor_sync(DS_FULL_MASK, v[j], m, G);
                v[j] = low ? fminf(v[j], oj) : fmaxf(v[j], oj);
                v[p] = low ? fminf(v[p], op) : fmaxf(v[p], op);
            }
        }
        // half-cleaners
#pragma unroll
        for (int s = k / 4; s >= 1; s >>= 1) {
            if (s >= EPL) {
                const int m = s / EPL;
                const bool low = !(lig & m);
#pragma unroll
                for (int j = 0; j < EPL; j++) {
                    const float o = __shfl_xor_sync(DS_FULL_MASK, v[j], m, G);
                    v[j] = low ? fminf(v[j], o) : fmaxf(v[j], o);
                }
            } else {
#pragma unroll
                for (int j = 0; j < EPL; j++) {
                    const int p = j ^ s;
                    if (p > j) {
                        const float a = v[j], b = v[p];
                        v[j] = fminf(a, b);
                        v[p] = fmaxf(a, b);
                    }
                }
            }
        }
    }
}

// Sort the group's row into the scratch, build the cell table, the prefix
// sums, Q and P[d].  Warp-collective; groups with want == false write nothing.
template <int G, int C, int VEC, bool PAD>
__device__ __forceinline__ void bucket_build(const float *row, int d, int lig, bool want,
                                             float lo0, float invw, uint8_t *scr, double &Q,
                                             double &Ptot) {
    using Lay = Layout<G, C, VEC>;
    constexpr int EPL = C * VEC;
    constexpr int DP = G * EPL;
    using BL = BucketLayout<DP>;
    constexpr int F = BL::F;
    constexpr int CPL = F / G;  // cells per lane = 2 * EPL
    float *xs = reinterpret_cast<float *>(scr + BL::XS_OFF);
    double *P = reinterpret_cast<double *>(scr + BL::P_OFF);
    uint32_t *cnt = reinterpret_cast<uint32_t *>(scr + BL::P_OFF);  // u32[F] during the build
    typename BL::Tab *tab = reinterpret_cast<typename BL::Tab *>(scr + BL::TAB_OFF);
    const double lo0d = (double)lo0;
    auto in = [&](int k) -> bool { return !PAD || Lay::elem(lig, k) < d; };

    // 1. zero the cell counts (the lane's CPL cells); sort the row
    if (want) {
        if (CPL % 4 == 0) {
#pragma unroll
            for (int i = 0; i < CPL / 4; i++)
                reinterpret_cast<uint4 *>(cnt + lig * CPL)[i] = make_uint4(0u, 0u, 0u, 0u);
        } else {
#pragma unroll
            for (int i = 0; i < CPL; i++) cnt[lig * CPL + i] = 0u;
        }
    }
    float v[EPL];
#pragma unroll
    for (int k = 0; k < EPL; k++) v[k] = in(k) ? row[Lay::elem(lig, k)] : INFINITY;
    // 2. cell histogram (of the values in any order)
    __syncwarp();  // (zeroed counts before the increments)
    if (want) {
#pragma unroll
        for (int k = 0; k < EPL; k++)
            if (in(k)) atomicAdd(cnt + bk_cell(v[k], lo0, invw, F), 1u);
    }
    bitonic_group<G, EPL>(v, lig);
    if (want) {
        if (EPL % 4 == 0) {
#pragma unroll
            for (int j = 0; j < EPL; j += 4)
                *reinterpret_cast<float4 *>(xs + lig * EPL + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < EPL; j++) xs[lig * EPL + j] = v[j];
        }
    }
    __syncwarp();
    // 3. inclusive scan of the counts over the group -> cell ends
    uint32_t run = 0;
    if (want) {
#pragma unroll
        for (int i = 0; i < CPL; i++) run += cnt[lig * CPL + i];
    }
    uint32_t incl = run;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
        const uint32_t u = __shfl_up_sync(DS_FULL_MASK, incl, o, G);
        if (lig >= o) incl += u;
    }
    uint32_t base = incl - run;
    if (want) {
#pragma unroll
        for (int i = 0; i < CPL; i++) {
            base += cnt[lig * CPL + i];
            tab[lig * CPL + i + 1] = (typename BL::Tab)base;
        }
        if (lig == 0) tab[0] = 0;
    }
    __syncwarp();  // (the counts are dead: P overwrites them)
    // 4. prefix sums of y = x - lo0 (>= 0) over the sorted row, and Q
    double srun = 0.0, q = 0.0;
#pragma unroll
    for (int i = 0; i < EPL; i++) {
        if (lig * EPL + i < d) {
            const double y = __dsub_rn((double)v[i], lo0d);
            srun = __dadd_rn(srun, y);
            q = __fma_rn(y, y, q);
        }
    }
    double sincl = srun;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
        const double u = __shfl_up_sync(DS_FULL_MASK, sincl, o, G);
        if (lig >= o) sincl = __dadd_rn(sincl, u);
    }
    double pb = __shfl_up_sync(DS_FULL_MASK, sincl, 1, G);  // the lanes before this one
    if (lig == 0) pb = 0.0;
    if (want) {
        if (lig == 0) P[0] = 0.0;
#pragma unroll
        for (int i = 0; i < EPL; i++) {
            const int j = lig * EPL + i;
            if (j < d) {
                pb = __dadd_rn(pb, __dsub_rn((double)v[i], lo0d));
                P[j + 1] = pb;
            }
        }
    }
    Q = grp_sumd<G>(q);
    Ptot = __shfl_sync(DS_FULL_MASK, sincl, (threadIdx.x & 31) | (G - 1), 32);
    __syncwarp();
}

// the row state the candidate evaluations share
struct BkRow {
    float lo0, invw;
    double lo0d, Q, Ptot;
    double Abound;  // gamma * (sum of the magnitudes of every SSE term), any candidate
    float es_c;     // RU(2^-50 (L+1)/L): the undecided band's floor per unit of range
    int d;
};

// One candidate's boundaries k0..k1 (this lane's share): the partial sum of
// (d_{k-1} - d_k)((d_{k-1} + d_k) idx_k - 2 P[idx_k]); NaN when an element
// sits within the reference's rounding of a boundary (undecided: NaN makes
// every comparison false, so the decision goes to the exact path).
template <int DP>
__device__ __forceinline__ double bk_boundaries(const uint8_t *scr, const BkRow &R, int k0, int k1,
                                                float lo, double s, float es32) {
    using BL = BucketLayout<DP>;
    const float *xs = reinterpret_cast<const float *>(scr + BL::XS_OFF);
    const double *P = reinterpret_cast<const double *>(scr + BL::P_OFF);
    const typename BL::Tab *tab = reinterpret_cast<const typename BL::Tab *>(scr + BL::TAB_OFF);
    double Sp = 0.0;
    if (k0 > k1) return Sp;
    const double lod = (double)lo;
    double dprev = __dsub_rn((double)deq_exact(k0 - 1, lo, s), R.lo0d);
    bool unc = false;
#pragma unroll 1
    for (int k = k0; k <= k1; k++) {
        // code transition t_k = lo + (k - 1/2) s (quant.py:103-105)
        const double t = __fma_rn((double)k - 0.5, s, lod);
        const float tf = __double2float_rn(t);
        // |x - t| <= 2^-50((L+1)s + |t|) is undecided; |t - tf| <= 2^-24|tf|
        const float epsf = __fmaf_rn(fabsf(tf), 0x1p-22f, es32);
        // idx = #{x < t}: the cell's start + a binary search inside the cell
        const int ct = bk_cell(tf, R.lo0, R.invw, BL::F);
        int i0 = tab[ct], i1 = tab[ct + 1];
        while (i0 < i1) {
            const int mid = (i0 + i1) >> 1;
            if (xs[mid] < tf) i0 = mid + 1;
            else i1 = mid;
        }
        const int idx = i0;
        // the nearest elements below and above t decide whether idx is certain
        const float xb = xs[max(idx - 1, 0)], xa = xs[min(idx, R.d - 1)];
        unc |= fabsf(__fsub_rn(xb, tf)) <= epsf || fabsf(__fsub_rn(xa, tf)) <= epsf;
        const double dk = __dsub_rn((double)deq_exact(k, lo, s), R.lo0d);
        Sp = __fma_rn(dprev - dk, __fma_rn(dprev + dk, (double)idx, -2.0 * P[idx]), Sp);
        dprev = dk;
    }
    return unc ? __longlong_as_double(0x7ff8000000000000ll) : Sp;
}

// a candidate's SSE from its reduced boundary sum (NaN: undecided)
__device__ __forceinline__ double bk_finish(const BkRow &R, int L, float lo, double s, double pS) {
    const double dL = __dsub_rn((double)deq_exact(L, lo, s), R.lo0d);
    const double S = pS + (R.Q + dL * ((double)R.d * dL - 2.0 * R.Ptot));
    return s > 0.0 ? S : __longlong_as_double(0x7ff8000000000000ll);
}
// its bound: the row's gamma*A plus a relative margin that keeps a certified
// strict order through the reference's sqrt (NaN stays NaN)
__device__ __forceinline__ double bk_bound(const BkRow &R, double S) {
    return R.Abound + 0x1p-48 * fabs(S);
}

// SSE of two candidates of one row (bounds: bk_bound).  G >= 2: the lanes
// of the group's lower half take candidate A's L boundaries, the upper half
// B's, consecutive boundaries per lane [k0, k1] (each level computed once);
// G == 1: one lane takes both.  Warp-collective.
template <int G, int C, int VEC>
__device__ __forceinline__ void bucket_eval2(const uint8_t *scr, const BkRow &R, bool on, int lig, int L,
                                             double invL, int k0, int k1, float loA, float hiA,
                                             float loB, float hiB, double &SA, double &SB) {
    constexpr int DP = G * C * VEC;
    const float es_c = R.es_c;
    if constexpr (G == 1) {
        const double sA = scale64_y(loA, hiA, (double)L, invL), sB = scale64_y(loB, hiB, (double)L, invL);
        const float eA = fmaxf(__fmul_ru(__fsub_ru(hiA, loA), es_c), 0x1p-126f);
        const float eB = fmaxf(__fmul_ru(__fsub_ru(hiB, loB), es_c), 0x1p-126f);
        const double pA = on ? bk_boundaries<DP>(scr, R, 1, L, loA, sA, eA) : 0.0;
        const double pB = on ? bk_boundaries<DP>(scr, R, 1, L, loB, sB, eB) : 0.0;
        SA = bk_finish(R, L, loA, sA, pA);
        SB = bk_finish(R, L, loB, sB, pB);
    } else {
        constexpr int H = G / 2;
        const bool hb = lig >= H;  // this lane works on candidate B
        const float lo = hb ? loB : loA, hi = hb ? hiB : hiA;
        const double s = scale64_y(lo, hi, (double)L, invL);
        // the undecided band's floor 2^-50 (L+1) s, rounded up, from hi - lo
        const float es32 = fmaxf(__fmul_ru(__fsub_ru(hi, lo), es_c), 0x1p-126f);
        double p = on ? bk_boundaries<DP>(scr, R, k0, k1, lo, s, es32) : 0.0;
#pragma unroll
        for (int o = H / 2; o > 0; o >>= 1) p += __shfl_xor_sync(DS_FULL_MASK, p, o, G);
        const double S = bk_finish(R, L, lo, s, p);
        const double So = __shfl_xor_sync(DS_FULL_MASK, S, H, G);
        SA = hb ? So : S;
        SB = hb ? S : So;
    }
}

// greedy range search of one row per group (quant.py:160-209) over bucket
// sums.  The row is read from shared memory (`row`, Layout order), so no
// element registers stay live across the search.  Same decisions as the reference: a comparison whose bounds overlap
// (or an undecided SSE, NaN) is re-taken with exact_me_group (the
// reference's arithmetic and summation order).  `scr` is the group's
// BucketLayout scratch, which the exact evaluation borrows (the group then
// rebuilds its buckets before the next evaluation).
template <int G, int C, int VEC, bool PAD>
__device__ __forceinline__ void greedy_row_bucket(const float *row, int d, int lig,
                                                  bool row_ok, float lo0, float hi0, int L,
                                                  double invL, int bins, int steps, uint8_t *scr,
                                                  float &out_lo, float &out_hi,
                                                  unsigned &n_exact_dec, unsigned &n_exact_codes) {
    constexpr int DP = G * C * VEC;
    constexpr int F = BucketLayout<DP>::F;
    out_lo = lo0;
    out_hi = hi0;
    const double full = __dsub_rn((double)hi0, (double)lo0);
    const double step = __ddiv_rn(full, (double)bins);
    bool active = row_ok && step > 0.0;
    if (!__any_sync(DS_FULL_MASK, active)) return;
    double *buf = reinterpret_cast<double *>(scr);
    BkRow R;
    R.lo0 = lo0;
    R.lo0d = (double)lo0;
    R.d = d;
    const float rng0 = __fsub_rn(hi0, lo0);
    R.invw = rng0 > 0.f ? __fdiv_rn((float)F, rng0) : 0.f;  // inf range -> 0: one cell
    // es32 = RU(hi - lo) * RU(2^-50 (L+1)/L (1 + 2^-20)) >= 2^-50 (L+1) s
    R.es_c = __double2float_ru(0x1p-50 * (double)(L + 1) / (double)L * (1.0 + 0x1p-20));
    bucket_build<G, C, VEC, PAD>(row, d, lig, active, lo0, R.invw, scr, R.Q, R.Ptot);
    {
        // every SSE term's magnitude, for any candidate inside [lo0, hi0]:
        // y, d_k <= Rm, so Q + |tail| + sum_k |term_k| <= Q + (8L + 3) d Rm^2
        const double Rm = full + 0x1p-23 * fmax(fabs((double)lo0), fabs((double)hi0));
        const double fd = (double)d, fL = (double)L;
        R.Abound = (2.0 * fd + 2.0 * fL + 64.0) * 0x1p-53 *
                   (R.Q + (8.0 * fL + 3.0) * fd * Rm * Rm) * (1.0 + 0x1p-40);
    }
    // this lane's boundaries of its half's candidate
    int k0 = 1, k1 = L;
    if (G >= 2) {
        const int H = G / 2, kpl = (L + H - 1) / H;
        k0 = 1 + (lig & (H - 1)) * kpl;
        k1 = min(L, k0 + kpl - 1);
    }
    bool clob = false;  // this group's scratch holds an exact evaluation
    auto exact = [&](float lo, float hi, bool want) -> double {
        clob |= want;
        return exact_me_row<G, C, VEC>(row, d, lig, lo, hi, L, want, buf, n_exact_codes);
    };
    float best_lo = lo0, best_hi = hi0;
    double best_S, best_me = 0.0;
    bool best_has_me = false;
    {
        double s2;
        bucket_eval2<G, C, VEC>(scr, R, active, lig, L, invL, k0, k1, lo0, hi0, lo0, hi0, best_S, s2);
    }
    double cur_lo = (double)lo0, cur_hi = (double)hi0;
    for (int it = 0; it < steps; it++) {
        active = active && (__dsub_rn(__dsub_rn(cur_hi, cur_lo), step) > 0.0);
        if (!__any_sync(DS_FULL_MASK, active)) break;
        if (__any_sync(DS_FULL_MASK, clob)) {  // rebuild what an exact evaluation overwrote
            double q, p;
            bucket_build<G, C, VEC, PAD>(row, d, lig, clob && active, lo0, R.invw, scr, q, p);
            clob = false;
        }
        const float a_lo = __double2float_rn(__dadd_rn(cur_lo, step)), a_hi = __double2float_rn(cur_hi);
        const float b_lo = __double2float_rn(cur_lo), b_hi = __double2float_rn(__dsub_rn(cur_hi, step));
        double SA, SB;
        bucket_eval2<G, C, VEC>(scr, R, active, lig, L, invL, k0, k1, a_lo, a_hi, b_lo, b_hi, SA, SB);
        const double BA = bk_bound(R, SA), BB = bk_bound(R, SB), Bb = bk_bound(R, best_S);
        // take_a = me_a <= me_b (quant.py:198); improved = me_cur < best_me (:204)
        const bool ta_yes = SA + BA < SB - BB, ta_no = SA - BA > SB + BB;
        bool take_a = !ta_no;
        double Sc = take_a ? SA : SB;
        double Bc = take_a ? BA : BB;
        const bool imp_yes = Sc + Bc < best_S - Bb, imp_no = Sc - Bc > best_S + Bb;
        bool improved = imp_yes;
        const bool sure = (ta_yes || ta_no) && (imp_yes || imp_no);
        if (__any_sync(DS_FULL_MASK, active && !sure)) {
            // exact re-decisions (rare): take_a, then improved (the reference's
            // order), with exact MEs of whichever candidates they need
            const bool need_t = active && !(ta_yes || ta_no);
            double me_c = 0.0;
            bool c_has = false;
            if (__any_sync(DS_FULL_MASK, need_t)) {
                const double ma = exact(a_lo, a_hi, need_t);
                const double mb = exact(b_lo, b_hi, need_t);
                if (need_t) {
                    take_a = ma <= mb;
                    me_c = take_a ? ma : mb;
                    c_has = true;
                    if (lig == 0) n_exact_dec++;
                }
            }
            Sc = take_a ? SA : SB;
            Bc = take_a ? BA : BB;
            const bool iy = Sc + Bc < best_S - Bb, in_ = Sc - Bc > best_S + Bb;
            const bool need_i = active && !(c_has && best_has_me) && !(iy || in_);
            improved = iy;
            const float c_lo = take_a ? a_lo : b_lo, c_hi = take_a ? a_hi : b_hi;
            const bool need_c = need_i && !c_has, need_b = need_i && !best_has_me;
            if (__any_sync(DS_FULL_MASK, need_c)) {
                const double m = exact(c_lo, c_hi, need_c);
                if (need_c) {
                    me_c = m;
                    c_has = true;
                }
            }
            if (__any_sync(DS_FULL_MASK, need_b)) {
                const double m = exact(best_lo, best_hi, need_b);
                if (need_b) {
                    best_me = m;
                    best_has_me = true;
                }
            }
            if (active && c_has && best_has_me && !(iy || in_)) {
                improved = me_c < best_me;
                if (lig == 0) n_exact_dec++;
            }
            if (active && improved) {
                best_me = me_c;
                best_has_me = c_has;
            }
        } else if (active && improved) {
            best_has_me = false;
        }
        if (active) {
            if (take_a) cur_lo = __dadd_rn(cur_lo, step);
            else cur_hi = __dsub_rn(cur_hi, step);
            if (improved) {
                best_lo = take_a ? a_lo : b_lo;
                best_hi = take_a ? a_hi : b_hi;
                best_S = Sc;
            }
        }
    }
    out_lo = best_lo;
    out_hi = best_hi;
}

}  // namespace ds
