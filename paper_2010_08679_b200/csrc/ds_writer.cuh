// ds_writer.cuh -- the K3 writer kernel template, shared by the per-mode TUs.
#pragma once
//
// Replaces build_shard_payload's chunk loop (deltasnap/engine.py:139-187) with
// quantize_rows / adaptive_params_rows / pack_code_rows (quant.py:93-209,
// 372-382) and serialize_section (payload.py:84-104).
//
// Shape of the work: the shard payload is [hdr t0][records t0][hdr t1]... .
// A layout kernel turns per-table row counts into section offsets, writes the
// 24-byte headers and a tile schedule.  The writer is a persistent grid over
// tiles of TR consecutive records of one table: each group of G lanes codes
// one row into a shared-memory stage laid out exactly like the wire bytes,
// then the CTA streams the stage to HBM with aligned 32-bit stores (the
// records of a tile are one contiguous byte range, whatever the record size).
#include <cuda_runtime.h>
#include <stdint.h>

#include "ds_common.cuh"
#include "ds_greedy.cuh"
#include "ds_host.h"

#ifndef DS_ERR_DEFER
// 1: code_row_m1 leaves its row's sum of squares to the warp writer, which
// takes each tile row's root on its own lane (one root per 32 rows instead of
// one per group per chunk); only the G > 1 warp writer calls code_row_m1
#define DS_ERR_DEFER 1
#endif
#ifndef DS_M1_LEVELS
#define DS_M1_LEVELS 0  // 1: 2/4-bit rows take the exact levels by shuffles (A/B r02: T 6.79 vs 6.64 ms, off)
#endif
#ifndef DS_M1_PACKED
#define DS_M1_PACKED 1  // naive rows: codes and the tie check in packed fp32 pairs
#endif
#ifndef DS_ERR_F2F
#define DS_ERR_F2F 1  // 1: the err_sum term through the conversion unit; 0: err_fast (integer bits)
#endif
#ifndef DS_M1_ERR
#define DS_M1_ERR 1  // naive rows' err term: 0 F2F for q and the level, 1 q by the 2^52 magic
                     // (DADD; T shard 6.98 -> 6.61 ms), 2 also the level rounded by integer bits
#endif
#ifndef DS_TT_BALLOT
#define DS_TT_BALLOT 0  // 1: strided tiles find their table by ballot (measured 2 us slower at C2)
#endif
#ifndef DS_M1_FUSED
#define DS_M1_FUSED 1  // naive 2/4/8-bit rows: codes packed as produced (code_row_m1)
#endif

namespace ds {

constexpr int WT = 256;  // threads per writer CTA

struct WriterArgs {
    ds_table_desc t[DS_MAX_TABLES];
    int ntables;
    int bitwidth;  // 0 = fp32 section
    int L;
    int incremental;
    int bins, steps;
    int aux;
    int write_headers;
    int dim;
    int rec;        // record bytes
    int par_off;    // params (mode 1) or values (mode 0) offset in the record
    int code_off;   // packed codes offset (mode 1)
    int packed;     // packed code bytes (mode 1)
    int aux_off;    // aux offset in the record
    int tile_rows;  // TR
    double invL;    // RN(1/L) for the division-free scale
    int ids_packed;
    int ids_local;
    const int64_t *ids;
    const int64_t *counts;  // device per-table counts (incremental) or null
    int64_t *sec_off;       // [nt+1] section offsets + total (written by CTA 0)
    uint8_t *payload;
    int64_t capacity;
    double *partials;       // per-CTA error partials
    double *err_out;        // final error sum (may be null)
    unsigned *done;         // CTAs finished (last one reduces; zero between calls)
    uint32_t *fix_mask;    // MODE 1: per warp-tile mask of rows for the fixup pass
    uint32_t *flags;
    unsigned long long *stats;
    const float *staged;  // rows gathered by ds_stage_rows (read record i of the packed order)
    int64_t staged_rows;  // capacity of staged in rows (a larger dirty total: flagged, nothing written)
    int has_x;            // the row-sharded count exchange runs in this launch
    ds_peer_exchange x;
};

// ---------------------------------------------------------------------------
// the row-sharded count exchange (include/deltasnap_cuda.h, ds_peer.cu)
// ---------------------------------------------------------------------------
__host__ __device__ inline size_t peer_flags_bytes(int world) {
    return ((size_t)2 * world * sizeof(uint32_t) + 255) & ~(size_t)255;
}
__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// one warp: this rank's counts (per table from the layout, then the total)
// into slot [e & 1][rank] of every peer's buffer, then the slot's flag
__device__ __forceinline__ void peer_publish(const WriterArgs &a, const int64_t *s_sched) {
    const int lane = threadIdx.x & 31, nt = a.ntables, n = nt + 1;
    const ds_peer_exchange &x = a.x;
    const int par = x.epoch & 1;
    int64_t tot = 0;
    for (int t = lane; t < nt; t += 32) tot += s_sched[nt + 1 + t];
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(DS_FULL_MASK, tot, o);
    for (int p = 0; p < x.world; p++) {
        uint8_t *base = static_cast<uint8_t *>(x.peers[p]);
        int64_t *slot = reinterpret_cast<int64_t *>(base + peer_flags_bytes(x.world)) +
                        ((size_t)par * x.world + x.rank) * n;
        for (int t = lane; t < n; t += 32) slot[t] = t < nt ? s_sched[nt + 1 + t] : tot;
    }
    __syncwarp();
    __threadfence_system();  // every slot before any flag, for every observer
    if (lane < x.world)
        st_release_sys(reinterpret_cast<uint32_t *>(x.peers[lane]) + par * x.world + x.rank, x.epoch);
}

// one warp (the last CTA): until every rank's flag of the epoch is up, then
// the slots -> x.out; DS_FLAG_TIMEOUT if a rank stays missing
__device__ __forceinline__ void peer_wait(const WriterArgs &a) {
    const int lane = threadIdx.x & 31, n = a.ntables + 1;
    const ds_peer_exchange &x = a.x;
    const int par = x.epoch & 1;
    const uint8_t *local = static_cast<const uint8_t *>(x.peers[x.rank]);
    const uint32_t *flags = reinterpret_cast<const uint32_t *>(local) + par * x.world;
    bool late = false;
    const uint64_t t0 = globaltimer_ns();
    for (int r = lane; r < x.world; r += 32)
        while (ld_acquire_sys(flags + r) != x.epoch) {
            if ((int64_t)(globaltimer_ns() - t0) > x.timeout_ns) {
                late = true;
                break;
            }
            __nanosleep(64);
        }
    if (__any_sync(DS_FULL_MASK, late)) {
        if (lane == 0) atomicOr(x.flags, DS_FLAG_TIMEOUT);
        return;
    }
    // lane r's acquire orders only lane r's later loads: a system-scope
    // acquire fence makes every rank's slot writes visible to every lane
    __syncwarp();
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    const volatile int64_t *slots =
        reinterpret_cast<const int64_t *>(local + peer_flags_bytes(x.world)) + (size_t)par * x.world * n;
    for (int i = lane; i < x.world * n; i += 32) x.out[i] = slots[i];
}

// ---------------------------------------------------------------------------
// shared-memory byte helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ void st_bytes(uint8_t *p, uint64_t v, int n) {
    for (int i = 0; i < n; i++) p[i] = (uint8_t)(v >> (8 * i));
}
// misaligned record layouts only (odd record sizes): out of line, so the
// aligned stores of the common layouts stay real branches, not predicated
// byte-store sequences
static __device__ __noinline__ void st_bytes_slow(uint8_t *p, uint64_t v, int n) {
    for (int i = 0; i < n; i++) p[i] = (uint8_t)(v >> (8 * i));
}
__device__ __forceinline__ void st_u32(uint8_t *p, uint32_t v) {
    if ((reinterpret_cast<uintptr_t>(p) & 3) == 0) *reinterpret_cast<uint32_t *>(p) = v;
    else st_bytes(p, v, 4);
}
__device__ __forceinline__ uint32_t ld_u32_unaligned(const uint8_t *base, int o) {
    const uint32_t *w = reinterpret_cast<const uint32_t *>(base + (o & ~3));
    int sh = (o & 3) * 8;
    if (sh == 0) return w[0];
    return __funnelshift_r(w[0], w[1], sh);
}

// stream nbytes of the stage to dst (any alignment) with aligned 32-bit stores
__device__ __forceinline__ void copy_out(uint8_t *__restrict__ dst, const uint8_t *stage,
                                         int64_t nbytes, int tid, int nthr) {
    // the stage is 16-byte aligned: an 8/16-byte aligned destination copies
    // with 64/128-bit moves (records of a tile are contiguous)
    const uintptr_t al = reinterpret_cast<uintptr_t>(dst);
    if ((al & 7) == 0) {
        // (a tile stage is < 2^31 bytes: 32-bit induction variables)
        const int nb = (int)nbytes;
        if ((al & 15) == 0) {
            const int n16 = nb >> 4;
            for (int k = tid; k < n16; k += nthr)
                __stcs(reinterpret_cast<int4 *>(dst) + k, reinterpret_cast<const int4 *>(stage)[k]);
            for (int b = (n16 << 4) + tid; b < nb; b += nthr) dst[b] = stage[b];
        } else {
            const int n8 = nb >> 3;
            for (int k = tid; k < n8; k += nthr)
                __stcs(reinterpret_cast<unsigned long long *>(dst) + k,
                       reinterpret_cast<const unsigned long long *>(stage)[k]);
            for (int b = (n8 << 3) + tid; b < nb; b += nthr) dst[b] = stage[b];
        }
        return;
    }
    int head = (int)((4 - (reinterpret_cast<uintptr_t>(dst) & 3)) & 3);
    if (head > nbytes) head = (int)nbytes;
    if ((int)tid < head) dst[tid] = stage[tid];
    int64_t nw = (nbytes - head) >> 2;
    uint32_t *dw = reinterpret_cast<uint32_t *>(dst + head);
    for (int64_t k = tid; k < nw; k += nthr)
        __stcs(dw + k, ld_u32_unaligned(stage, head + 4 * (int)k));  // streamed, not re-read
    int64_t done = head + 4 * nw;
    int tail = (int)(nbytes - done);
    if ((int)tid < tail) dst[done + tid] = stage[done + tid];
}

// ---------------------------------------------------------------------------
// async copies (cp.async / LDGSTS): the gather lands in shared memory without
// holding registers, so a CTA keeps a whole tile of rows in flight
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------
// the writer
// ---------------------------------------------------------------------------
// MODE 0: fp32 section (payload.py:101), 1: naive ranges (engine.py:163-164),
// 2: greedy ranges (engine.py:166 -> quant.py:160-209).

// per-thread accumulators of the writer
struct WAcc {
    double err = 0.0;  // sum of row L2 errors (engine.py:171-173)
    double row_sse = 0.0;  // DS_ERR_DEFER: the last code_row_m1 row's sum of squares (group-reduced)
    unsigned n_exact_dec = 0, n_exact_codes = 0, n_rows = 0;
    bool bad_data = false, bad_ids = false;
};

// MODE 1 at 8/4/2 bits with 128-bit element chunks: codes, the certified
// tie check, the err_sum term and the packed bytes in ONE pass over the
// registers -- a chunk's 4 codes are packed as they are produced, so no
// per-element code array stays live (register pressure is the limit of
// this kernel: 128 per thread at two CTAs per SM).
template <int G, int C, bool PAD, bool CONTIG, int N>
__device__ __forceinline__ bool code_row_m1(const WriterArgs &a, const float (&x)[C * 4], bool valid,
                                            bool row_ok, const RowQ &rq, uint8_t *rec, int lig,
                                            int d, WAcc &acc, bool al8) {
    using Lay = Layout<G, C, 4>;
    constexpr int EPL = C * 4;
    auto el = [&](int k) -> int { return CONTIG ? EPL * lig + k : Lay::elem(lig, k); };
    const double lod = (double)rq.lo;
    // 2/4-bit rows on enough lanes: the row's 2^N exact levels f32(RN(RN(s*q)
    // + lo)) (quant.py:114-115) computed once, two per lane, for the err_sum term
    constexpr bool LEVELS = DS_M1_LEVELS && DS_ERR_F2F && G >= 2 && (1 << N) <= 2 * G;
    float lv0 = 0.f, lv1 = 0.f;
    if constexpr (LEVELS) {
        lv0 = deq_exact(2 * lig, rq.lo, rq.s);
        lv1 = deq_exact(2 * lig + 1, rq.lo, rq.s);
    }
    float dev = 0.f;
    double sse = 0.0;
    uint32_t w[C];  // chunk c's 4 codes, N bits each, LSB first (quant.py:376-382)
#pragma unroll
    for (int c = 0; c < C; c++) {
        uint32_t pk = 0;
#if DS_M1_PACKED
        // the chunk's codes two at a time in packed fp32 pairs, the product
        // fused (ptxas contracts f32x2 mul+add even with .rn, so it is written
        // as FMAs and fix_tile mirrors exactly these): qm = RN(t*inv + 1.5*2^23)
        // rounds the exact product t*inv half-to-even to the code, r =
        // RN(t*inv - q) its distance; |t*inv - v_ref| <= 5u*L as for the
        // rounded product, so the 8u*L guard band still certifies the code
        float qms[4];
        {
            const f32x2 LO = pk2(rq.lo, rq.lo), INV = pk2(rq.inv, rq.inv);
            const f32x2 MAG = pk2(12582912.0f, 12582912.0f);
#pragma unroll
            for (int j = 0; j < 4; j += 2) {
                const f32x2 t = sub2(pk2(x[4 * c + j], x[4 * c + j + 1]), LO);
                const f32x2 qm = fma2(t, INV, MAG);
                float r0, r1;
                up2(fma2(t, INV, sub2(MAG, qm)), r0, r1);  // MAG - qm = -q exactly
                up2(qm, qms[j], qms[j + 1]);
                dev = fmaxf(dev, fmaxf(fabsf(r0), fabsf(r1)));
            }
        }
#endif
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int k = 4 * c + j;
            // min/max ranges hold every element: no clip, v in [0, L(1+5u)];
            // round half to even through the 1.5*2^23 magic (low mantissa
            // bits = the code); |v - q| near 1/2 -> the exact fixup (RowQ)
#if DS_M1_PACKED
            const float qm = qms[j];
#else
            const float v = __fmul_rn(__fsub_rn(x[k], rq.lo), rq.inv);
            const float qm = __fadd_rn(v, 12582912.0f);
            dev = fmaxf(dev, fabsf(__fsub_rn(v, __fsub_rn(qm, 12582912.0f))));
#endif
            const uint32_t qi = __float_as_uint(qm) & 0x3fffffu;
            const bool in = !PAD || el(k) < d;
#if DS_ERR_F2F
            double er;
            if constexpr (LEVELS) {
                // the level from the lane that holds it: two shuffles, a select
                const int src = (threadIdx.x & 31 & ~(G - 1)) | (int)(qi >> 1);
                const float la = __shfl_sync(DS_FULL_MASK, lv0, src);
                const float lb = __shfl_sync(DS_FULL_MASK, lv1, src);
                er = __dsub_rn((double)x[k], (double)((qi & 1u) ? lb : la));
            } else {
                // x - f32(RN(RN(s*q) + lo)), exact in f64 (DS_M1_ERR: how q enters
                // f64 and how the level is rounded to f32 -- same value)
                const double qd = DS_M1_ERR >= 1 ? code_to_f64(qi)
                                                 : (double)__fsub_rn(qm, 12582912.0f);
                const double wv = __dadd_rn(__dmul_rn(rq.s, qd), lod);
                const double dq = DS_M1_ERR >= 2 ? round_f32_in_f64(wv) : (double)__double2float_rn(wv);
                er = __dsub_rn((double)x[k], dq);
            }
#else
            const double er = err_fast(x[k], qi, rq.s, lod);  // engine.py:171-173
#endif
            if (in) sse = fma(er, er, sse);
            pk |= (in ? qi : 0u) << (N * j);
        }
        w[c] = row_ok ? pk : 0u;
    }
    dev = grp_max<G>(dev);  // every lane shuffles (no short-circuit)
    const bool fix = row_ok && (rq.mode == 2 || dev > 0.5f - rq.eps);
    if (rq.mode == 2 || !row_ok) sse = 0.0;  // mode 2: the fixup adds the exact error
    sse = grp_sumd<G>(sse);
    if (DS_ERR_DEFER) acc.row_sse = sse;  // the warp takes the root once per tile row (one lane each)
    if (row_ok && lig == 0) {
        if (!DS_ERR_DEFER) acc.err += DS_ERR_F2F ? (sse > 0.0 ? sse * rsqrt(sse) : 0.0) : row_err(sse);
        acc.n_rows++;
        if (al8)
            *reinterpret_cast<uint2 *>(rec + a.par_off) = make_uint2(__float_as_uint(rq.lo), __float_as_uint(rq.hi));
        else
            st_bytes_slow(rec + a.par_off, ((uint64_t)__float_as_uint(rq.hi) << 32) | __float_as_uint(rq.lo), 8);
    }
    if (!valid) return fix;
    uint8_t *pk = rec + a.code_off;
    if (CONTIG && !PAD && C == 4 && al8) {
        // the lane's 16 contiguous codes -> one 16 / 8 / 4-byte store
        if (N == 8) {
            if ((a.code_off & 15) == 0 && (a.rec & 15) == 0)
                *reinterpret_cast<uint4 *>(pk + 16 * lig) = make_uint4(w[0], w[1], w[2], w[3]);
            else {
                *reinterpret_cast<uint2 *>(pk + 16 * lig) = make_uint2(w[0], w[1]);
                *reinterpret_cast<uint2 *>(pk + 16 * lig + 8) = make_uint2(w[2], w[3]);
            }
        } else if (N == 4) {
            *reinterpret_cast<uint2 *>(pk + 8 * lig) = make_uint2(w[0] | (w[1] << 16), w[2] | (w[3] << 16));
        } else {
            *reinterpret_cast<uint32_t *>(pk + 4 * lig) = w[0] | (w[1] << 8) | (w[2] << 16) | (w[3] << 24);
        }
        return fix;
    }
#pragma unroll
    for (int c = 0; c < C; c++) {
        const int m = CONTIG ? C * lig + c : lig + c * G;  // chunk: elements 4m..4m+3
        if (4 * m < d) {
            if (N == 8) {
                if (al8) *reinterpret_cast<uint32_t *>(pk + 4 * m) = w[c];
                else st_bytes_slow(pk + 4 * m, w[c], 4);
            } else if (N == 4) {
                if (al8) *reinterpret_cast<uint16_t *>(pk + 2 * m) = (uint16_t)w[c];
                else st_bytes_slow(pk + 2 * m, w[c], 2);
            } else {
                pk[m] = (uint8_t)w[c];
            }
        }
    }
    return fix;
}

// Code one row held by the G lanes of a group into its record in `rec`
// (wire layout of payload.py:84-104): [u64 row] [f32 lo, f32 hi, codes] |
// [dim f32] [dim f32 aux].  `cs` is the group's dim-byte code scratch,
// `buf` its exact-evaluation scratch (MODE 2).
// CONTIG: lane lig holds elements [EPL*lig, EPL*lig + EPL) (the warp writer's
// shared-memory row chunks); else the interleaved Layout<G, C, VEC> order.
template <int G, int C, int VEC, int MODE, bool PAD, bool CONTIG = false>
__device__ __forceinline__ bool code_row(const WriterArgs &a, const ds_table_desc &td,
                                         float (&x)[C * VEC], const float *xs, bool valid, int64_t local,
                                         uint8_t *rec, uint8_t *cs, double *buf, int lig, int d,
                                         WAcc &acc) {
    using Lay = Layout<G, C, VEC>;
    constexpr int EPL = C * VEC;
    auto el = [&](int k) -> int { return CONTIG ? EPL * lig + k : Lay::elem(lig, k); };
    const int L = a.L;
    const int64_t gid = td.row_base + local;
    bool fix = false;  // MODE 1: row left to the exact fixup pass (fix_tile)
    // record fields 8-byte aligned (stages are 16-byte aligned, so every
    // record of a stage then is): warp-uniform
    const bool al8 = (((unsigned)a.rec | (unsigned)a.par_off | (unsigned)a.code_off) & 7u) == 0u;
    if (valid && a.incremental && lig == 0) {
        if (al8) *reinterpret_cast<uint64_t *>(rec) = (uint64_t)gid;
        else st_bytes_slow(rec, (uint64_t)gid, 8);
    }
    if (MODE == 0) {
        if (valid) {
#pragma unroll
            for (int k = 0; k < EPL; k++) {
                int e = el(k);
                if (e < d) st_u32(rec + a.par_off + 4 * e, __float_as_uint(x[k]));
            }
        }
    } else {
        // finiteness (quant.py:70-72,173): x*0 is NaN exactly for NaN/Inf;
        // naive range: row min / max (engine.py:163-164)
        // (NaN-propagating min/max: a NaN or Inf element leaves lo or hi
        // non-finite, so the range doubles as the finiteness test)
        float mn = INFINITY, mx = -INFINITY;
#pragma unroll
        for (int k = 0; k < EPL; k++) {
            if (!PAD || el(k) < d) {
                mn = fmin_nan(mn, x[k]);
                mx = fmax_nan(mx, x[k]);
            }
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            mn = fmin_nan(mn, __shfl_xor_sync(DS_FULL_MASK, mn, o, G));
            mx = fmax_nan(mx, __shfl_xor_sync(DS_FULL_MASK, mx, o, G));
        }
        const bool fin = isfinite(mn) && isfinite(mx);
        if (valid && !fin) acc.bad_data = true;
        const bool row_ok = valid && fin;
        float lo = mn, hi = mx;
        if (!row_ok) { lo = 0.f; hi = 0.f; }
        if (MODE == 2) {
            if constexpr (DS_GREEDY_BUCKET) {
                // the row stays in the ring stage (xs): re-read after the search
                greedy_row_bucket<G, C, VEC, PAD>(xs, d, lig, row_ok, lo, hi, L, a.invL, a.bins, a.steps,
                                                  reinterpret_cast<uint8_t *>(buf), lo, hi,
                                                  acc.n_exact_dec, acc.n_exact_codes);
#pragma unroll
                for (int k = 0; k < EPL; k++) x[k] = (valid && el(k) < d) ? xs[el(k)] : 0.f;
            } else
                greedy_row<G, C, VEC, PAD>(x, d, lig, row_ok, lo, hi, L, a.bins, a.steps, buf, lo, hi,
                                           acc.n_exact_dec, acc.n_exact_codes);
        }
        const RowQ rq = make_rowq(lo, hi, L, a.invL);
        bool fused = false;
        if constexpr (MODE == 1 && VEC == 4 && DS_M1_FUSED && G > 1) {  // one-lane rows: measured slower
            if (a.bitwidth == 8) {
                fix = code_row_m1<G, C, PAD, CONTIG, 8>(a, x, valid, row_ok, rq, rec, lig, d, acc, al8);
                fused = true;
            } else if (a.bitwidth == 4) {
                fix = code_row_m1<G, C, PAD, CONTIG, 4>(a, x, valid, row_ok, rq, rec, lig, d, acc, al8);
                fused = true;
            } else if (a.bitwidth == 2) {
                fix = code_row_m1<G, C, PAD, CONTIG, 2>(a, x, valid, row_ok, rq, rec, lig, d, acc, al8);
                fused = true;
            }
        }
        if (!fused) {
        int q[EPL];
        double sse = 0.0;
        if (MODE == 1) {
            // min/max ranges hold every element: no clip, v in [0, L(1+5u)].
            // Round half to even through the 1.5*2^23 magic: the sum's low
            // mantissa bits are the integer code, the difference its float.
            // A row with a code inside the guard band of a tie (~0.3% of rows)
            // or a range outside fp32's comfort zone is left to
            // the fixup pass (fix_tile), which re-codes it in exact f64: no f64 code
            // path here, so the hot loop keeps its registers.
            float dev = 0.f;
            const double lod = (double)lo;
#pragma unroll
            for (int k = 0; k < EPL; k++) {
                const float v = __fmul_rn(__fsub_rn(x[k], rq.lo), rq.inv);
                const float qm = __fadd_rn(v, 12582912.0f);
                q[k] = __float_as_int(qm) & 0x3fffff;
                const float qf = __fsub_rn(qm, 12582912.0f);
                dev = fmaxf(dev, fabsf(__fsub_rn(v, qf)));
                // err_sum term (engine.py:171-173): exact dequantized value
#if DS_ERR_F2F
                const double qd = DS_M1_ERR >= 1 ? code_to_f64((uint32_t)q[k]) : (double)qf;
                const float dq = __double2float_rn(__dadd_rn(__dmul_rn(rq.s, qd), lod));
                const double er = __dsub_rn((double)x[k], (double)dq);
#else
                const double er = err_fast(x[k], (uint32_t)q[k], rq.s, lod);
#endif
                if (!PAD || el(k) < d) sse = fma(er, er, sse);
            }
            dev = grp_max<G>(dev);  // every lane shuffles (no short-circuit)
            fix = row_ok && (rq.mode == 2 || dev > 0.5f - rq.eps);
            if (rq.mode == 2) sse = 0.0;  // fix_tile adds this row's exact error
        } else {
            const double lod = (double)lo;
            const bool exact_err = DS_ERR_F2F || rq.mode == 2;  // err_fast's range (RowQ)
#pragma unroll
            for (int k = 0; k < EPL; k++) {
                q[k] = code_of(x[k], rq, acc.n_exact_codes);
                double er;
                if (exact_err) {
                    const float dq = __double2float_rn(__dadd_rn(__dmul_rn(rq.s, (double)q[k]), lod));
                    er = __dsub_rn((double)x[k], (double)dq);
                } else {
                    er = err_fast(x[k], (uint32_t)q[k], rq.s, lod);
                }
                if (!PAD || el(k) < d) sse = fma(er, er, sse);
            }
        }
#pragma unroll
        for (int k = 0; k < EPL; k++)
            if (!row_ok || (PAD && el(k) >= d)) q[k] = 0;  // padding codes are 0
        if (!row_ok) sse = 0.0;  // rejected rows add no error
        sse = grp_sumd<G>(sse);
        if (row_ok && lig == 0) {
            // row L2 norm: sqrt as sse * rsqrt(sse) (within an ulp; err_sum is a
            // diagnostic sum whose low bits depend on summation order anyway)
            acc.err += DS_ERR_F2F ? (sse > 0.0 ? sse * rsqrt(sse) : 0.0) : row_err(sse);
            acc.n_rows++;
            if (al8)
                *reinterpret_cast<uint2 *>(rec + a.par_off) = make_uint2(__float_as_uint(lo), __float_as_uint(hi));
            else
                st_bytes_slow(rec + a.par_off,
                              ((uint64_t)__float_as_uint(hi) << 32) | __float_as_uint(lo), 8);
        }
        // ---- pack (quant.py:376-382): LSB-first bitstream ----
        uint8_t *pk = rec + a.code_off;
        if (CONTIG && VEC == 4 && !PAD && C == 4 && al8 &&
            (a.bitwidth == 8 || a.bitwidth == 4 || a.bitwidth == 2)) {
            // the lane's 16 contiguous codes -> one 16 / 8 / 4-byte store
            if (valid) {
                if (a.bitwidth == 8) {
                    uint32_t w[4];
#pragma unroll
                    for (int c = 0; c < 4; c++)
                        w[c] = q[4 * c] + (q[4 * c + 1] << 8) + (q[4 * c + 2] << 16) + ((uint32_t)q[4 * c + 3] << 24);
                    if ((a.code_off & 15) == 0 && (a.rec & 15) == 0)
                        *reinterpret_cast<uint4 *>(pk + 16 * lig) = make_uint4(w[0], w[1], w[2], w[3]);
                    else {
                        *reinterpret_cast<uint2 *>(pk + 16 * lig) = make_uint2(w[0], w[1]);
                        *reinterpret_cast<uint2 *>(pk + 16 * lig + 8) = make_uint2(w[2], w[3]);
                    }
                } else if (a.bitwidth == 4) {
                    uint32_t w[2];
#pragma unroll
                    for (int h = 0; h < 2; h++) {
                        uint32_t v = 0;
#pragma unroll
                        for (int j = 7; j >= 0; j--) v = (v << 4) + (uint32_t)q[8 * h + j];
                        w[h] = v;
                    }
                    *reinterpret_cast<uint2 *>(pk + 8 * lig) = make_uint2(w[0], w[1]);
                } else {
                    uint32_t v = 0;
#pragma unroll
                    for (int j = 15; j >= 0; j--) v = (v << 2) + (uint32_t)q[j];
                    *reinterpret_cast<uint32_t *>(pk + 4 * lig) = v;
                }
            }
        } else if (VEC == 4 && (a.bitwidth == 8 || a.bitwidth == 4 || a.bitwidth == 2)) {
            if (valid) {
#pragma unroll
                for (int c = 0; c < C; c++) {
                    const int m = CONTIG ? C * lig + c : lig + c * G;  // chunk: elements 4m..4m+3
                    if (4 * m < d) {
                        uint32_t v;
                        if (a.bitwidth == 8) {
                            v = q[4 * c] | (q[4 * c + 1] << 8) | (q[4 * c + 2] << 16) |
                                ((uint32_t)q[4 * c + 3] << 24);
                            if (al8) *reinterpret_cast<uint32_t *>(pk + 4 * m) = v;
                            else st_bytes_slow(pk + 4 * m, v, 4);
                        } else if (a.bitwidth == 4) {
                            v = q[4 * c] | (q[4 * c + 1] << 4) | (q[4 * c + 2] << 8) |
                                (q[4 * c + 3] << 12);
                            if (al8) *reinterpret_cast<uint16_t *>(pk + 2 * m) = (uint16_t)v;
                            else st_bytes_slow(pk + 2 * m, v, 2);
                        } else {
                            v = q[4 * c] | (q[4 * c + 1] << 2) | (q[4 * c + 2] << 4) |
                                (q[4 * c + 3] << 6);
                            pk[m] = (uint8_t)v;
                        }
                    }
                }
            }
        } else {
            // generic: codes through shared memory, each lane builds bytes
            if (valid) {
#pragma unroll
                for (int k = 0; k < EPL; k++) {
                    int e = el(k);
                    if (e < d) cs[e] = (uint8_t)q[k];
                }
            }
            __syncwarp();
            if (valid) {
                const int N = a.bitwidth;
                for (int b = lig; b < a.packed; b += G) {
                    int bit0 = 8 * b;
                    int j0 = bit0 / N, j1 = min(d - 1, (bit0 + 7) / N);
                    uint32_t v = 0;
                    for (int j = j0; j <= j1; j++) {
                        int pos = j * N - bit0;
                        uint32_t cv = cs[j];
                        v |= pos >= 0 ? (cv << pos) : (cv >> (-pos));
                    }
                    pk[b] = (uint8_t)v;
                }
            }
            __syncwarp();
        }
        }  // !fused
    }
    if (a.aux && valid) {
        float xa[EPL];
        load_row<G, C, VEC>(td.aux + local * td.ld, d, lig, xa, 0.f);
#pragma unroll
        for (int k = 0; k < EPL; k++) {
            int e = Lay::elem(lig, k);
            if (e < d) st_u32(rec + a.aux_off + 4 * e, __float_as_uint(xa[k]));
        }
    }
    return fix;
}

// ---------------------------------------------------------------------------
// layout (payload.py:84-104): every CTA derives the section offsets and the
// tile schedule from the device counts with one warp scan (no layout launch);
// CTA 0 publishes sec_off, the 24-byte headers (payload.py:88-91) and the
// capacity flag.  s_sched: [0..nt] tile prefix, [nt+1..2nt] row counts,
// [2nt+1..3nt] ids offsets; s_sec: [0..nt] section offsets + total.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void writer_layout(const WriterArgs &a, int64_t *s_sched, int64_t *s_sec) {
    const int nt = a.ntables;
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        int64_t tiles0 = 0, ids0 = 0, off0 = 0;  // carried across 32-table blocks
        for (int b = 0; b < nt; b += 32) {
            const int t = b + lane;
            int64_t n = 0, tl = 0, by = 0;
            if (t < nt) {
                n = a.counts ? a.counts[t] : a.t[t].rows;
                tl = (n + a.tile_rows - 1) / a.tile_rows;
                by = (a.write_headers ? DS_HEADER_SIZE : 0) + n * (int64_t)a.rec;
            }
            int64_t it = tl, ii = n, io = by;  // inclusive scans
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t u = __shfl_up_sync(DS_FULL_MASK, it, o);
                const int64_t v = __shfl_up_sync(DS_FULL_MASK, ii, o);
                const int64_t w = __shfl_up_sync(DS_FULL_MASK, io, o);
                if (lane >= o) { it += u; ii += v; io += w; }
            }
            if (t < nt) {
                s_sched[t] = tiles0 + it - tl;
                s_sched[nt + 1 + t] = n;
                s_sched[2 * nt + 1 + t] = a.ids_packed ? ids0 + ii - n : a.t[t].ids_off;
                s_sec[t] = off0 + io - by;
            }
            tiles0 += __shfl_sync(DS_FULL_MASK, it, 31);
            ids0 += __shfl_sync(DS_FULL_MASK, ii, 31);
            off0 += __shfl_sync(DS_FULL_MASK, io, 31);
        }
        if (lane == 0) {
            s_sched[nt] = tiles0;
            s_sched[3 * nt + 1] = ids0;  // records of the call
            s_sec[nt] = off0;
        }
    }
    __syncthreads();
    if (blockIdx.x == 0) {
        const int64_t total = s_sec[nt];
        // a staged write whose dirty total exceeds the staging buffer would
        // read rows stage_rows never wrote: flagged, no records written
        if (threadIdx.x == 0 && a.staged && s_sched[3 * nt + 1] > a.staged_rows)
            atomicOr(a.flags, DS_FLAG_CAPACITY);
        // the last warp publishes this rank's counts to the peers (its fence
        // delays only that warp)
        if (a.has_x && (threadIdx.x >> 5) == (int)(blockDim.x >> 5) - 1) peer_publish(a, s_sched);
        for (int t = threadIdx.x; t <= nt; t += blockDim.x) a.sec_off[t] = s_sec[t];
        if (threadIdx.x == 0 && total > a.capacity) atomicOr(a.flags, DS_FLAG_CAPACITY);
        if (a.write_headers && total <= a.capacity) {
            for (int t = threadIdx.x; t < nt; t += blockDim.x) {
                uint8_t *h = a.payload + s_sec[t];
                const uint32_t tid = a.t[t].table_id, dim = a.t[t].dim;
                const uint64_t n = (uint64_t)s_sched[nt + 1 + t];
                h[0] = 'C'; h[1] = 'N'; h[2] = 'R'; h[3] = '1';
                for (int k = 0; k < 4; k++) h[4 + k] = (uint8_t)(tid >> (8 * k));
                for (int k = 0; k < 8; k++) h[8 + k] = (uint8_t)(n >> (8 * k));
                for (int k = 0; k < 4; k++) h[16 + k] = (uint8_t)(dim >> (8 * k));
                h[20] = (uint8_t)(a.bitwidth ? a.bitwidth : DS_FP32_TAG);
                h[21] = (uint8_t)(a.bitwidth ? 1 : 0);
                h[22] = (uint8_t)(a.aux ? 1 : 0);
                h[23] = 0;
            }
        }
    }
}

// the records fit the payload (and, staged, the staging buffer); else flagged
// by CTA 0 and nothing but the headers is written
__device__ __forceinline__ bool writer_fits(const WriterArgs &a, const int64_t *s_sched,
                                            const int64_t *s_sec) {
    const int nt = a.ntables;
    return s_sec[nt] <= a.capacity && (!a.staged || s_sched[3 * nt + 1] <= a.staged_rows);
}

// block-level epilogue: error partial, flags, diagnostics; the last CTA to
// finish sums the partials in CTA order (deterministic) into err_out
__device__ __forceinline__ void writer_epilogue(const WriterArgs &a, WAcc &acc, double *s_red) {
    const int lane = threadIdx.x & 31;
    for (int o = 16; o > 0; o >>= 1) acc.err += __shfl_xor_sync(DS_FULL_MASK, acc.err, o);
    if (lane == 0) s_red[threadIdx.x >> 5] = acc.err;
    if (__any_sync(DS_FULL_MASK, acc.bad_data) && lane == 0) atomicOr(a.flags, DS_FLAG_DATA);
    if (__any_sync(DS_FULL_MASK, acc.bad_ids) && lane == 0) atomicOr(a.flags, DS_FLAG_BOUNDS);
    if (a.stats) {
        unsigned v0 = acc.n_exact_dec, v1 = acc.n_exact_codes, v2 = acc.n_rows;
        for (int o = 16; o > 0; o >>= 1) {
            v0 += __shfl_xor_sync(DS_FULL_MASK, v0, o);
            v1 += __shfl_xor_sync(DS_FULL_MASK, v1, o);
            v2 += __shfl_xor_sync(DS_FULL_MASK, v2, o);
        }
        if (lane == 0) {
            if (v0) atomicAdd(a.stats + DS_STAT_EXACT_DECISIONS, (unsigned long long)v0);
            if (v1) atomicAdd(a.stats + DS_STAT_EXACT_CODES, (unsigned long long)v1);
            if (v2) atomicAdd(a.stats + DS_STAT_ROWS, (unsigned long long)v2);
        }
    }
    __syncthreads();
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += s_red[w];
        a.partials[blockIdx.x] = s;
        __threadfence();
        s_last = atomicAdd(a.done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x < 32) {
        __threadfence();
        // lane l sums partials l, l+32, ... in order; then a fixed shuffle tree
        double s = 0.0;
        for (int i = lane; i < (int)gridDim.x; i += 32) s += __ldcg(a.partials + i);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(DS_FULL_MASK, s, o);
        if (lane == 0) {
            if (a.err_out) *a.err_out = s;
            *a.done = 0u;  // ready for the next call on this workspace
        }
        if (a.has_x) peer_wait(a);
    }
}

// table of a tile: the last table whose first tile is <= tile (one ballot
// per 32 tables; warp-uniform)
__device__ __forceinline__ int tile_table(const int64_t *s_sched, int nt, int64_t tile, int lane) {
    int t = 0;
    for (int b = 0; b < nt; b += 32) {
        unsigned m = __ballot_sync(DS_FULL_MASK, b + lane < nt && s_sched[b + lane] <= tile);
        if (m) t = b + 31 - __clz(m);
    }
    return t;
}

// ---------------------------------------------------------------------------
// MODE 1 exact fixup, in place: for the rows of a chunk whose codes the hot
// loop could not certify (a code within the fp32 guard band of a tie, or a
// range outside fp32's comfort zone; ~0.3% of rows), re-check the ambiguous
// elements in exact f64 from the row still in registers, rewrite the
// record's packed codes in the stage if any code changes, and swap the row's
// error term.  Warp-collective (every lane calls it when any row needs it).
// ---------------------------------------------------------------------------
template <int G, int C, int VEC, bool PAD, bool CONTIG>
__device__ __forceinline__ void fix_rows_inline(const WriterArgs &a, const float (&x)[C * VEC],
                                                int lig, int d, bool mine, uint8_t *rec,
                                                uint8_t *cs, WAcc &acc) {
    using Lay = Layout<G, C, VEC>;
    constexpr int EPL = C * VEC;
    auto el = [&](int k) -> int { return CONTIG ? EPL * lig + k : Lay::elem(lig, k); };
    float mn = INFINITY, mx = -INFINITY;
#pragma unroll
    for (int k = 0; k < EPL; k++)
        if (!PAD || el(k) < d) {
            mn = fminf(mn, x[k]);
            mx = fmaxf(mx, x[k]);
        }
    const float lo = grp_min<G>(mn), hi = grp_max<G>(mx);
    const RowQ rq = make_rowq(lo, hi, a.L, a.invL);
    int qfast[EPL], qex[EPL];
    bool changed = false;
#pragma unroll
    for (int k = 0; k < EPL; k++) {
        const float v = __fmul_rn(__fsub_rn(x[k], rq.lo), rq.inv);
        const float qm = __fadd_rn(v, 12582912.0f);
        qfast[k] = __float_as_int(qm) & 0x3fffff;
        qex[k] = qfast[k];
        const bool in = mine && (!PAD || el(k) < d);
        if (in && (rq.mode == 2 || fabsf(__fsub_rn(v, __fsub_rn(qm, 12582912.0f))) > 0.5f - rq.eps)) {
            qex[k] = code_exact_slow(x[k], lo, hi, rq.s, a.L);
            acc.n_exact_codes++;
            changed |= qex[k] != qfast[k];
        }
    }
    // a fast code was wrong (exact ties; rare), or the range is outside
    // fp32's comfort zone (the hot loop left the row's error out)
    const int any_changed = grp_or<G>(changed ? 1 : 0);  // every lane shuffles
    const bool row_changed = mine && (rq.mode == 2 || any_changed != 0);
    if (__any_sync(DS_FULL_MASK, row_changed)) {
        double sf = 0.0, se = 0.0;
#pragma unroll
        for (int k = 0; k < EPL; k++) {
            const int e = el(k);
            if (row_changed && e < d) {
#if DS_ERR_F2F
                const double ef = __dsub_rn((double)x[k], (double)deq_exact(qfast[k], lo, rq.s));
#else
                const double ef = err_fast(x[k], (uint32_t)qfast[k], rq.s, (double)lo);  // as the hot loop
#endif
                const double ee = __dsub_rn((double)x[k], (double)deq_exact(qex[k], lo, rq.s));
                sf = fma(ef, ef, sf);
                se = fma(ee, ee, se);
                cs[e] = (uint8_t)qex[k];
            }
        }
        sf = grp_sumd<G>(sf);
        se = grp_sumd<G>(se);
        if (row_changed && lig == 0)
            acc.err += (se > 0.0 ? se * rsqrt(se) : 0.0) -
                       (rq.mode == 2 ? 0.0 : (DS_ERR_F2F ? (sf > 0.0 ? sf * rsqrt(sf) : 0.0) : row_err(sf)));
        __syncwarp();
        if (row_changed) {  // rewrite the record's packed codes (LSB-first bitstream)
            uint8_t *pk = rec + a.code_off;
            const int N = a.bitwidth;
            for (int b = lig; b < a.packed; b += G) {
                const int bit0 = 8 * b;
                const int j0 = bit0 / N, j1 = min(d - 1, (bit0 + 7) / N);
                uint32_t v = 0;
                for (int j = j0; j <= j1; j++) {
                    const int pos = j * N - bit0;
                    const uint32_t cv = cs[j];
                    v |= pos >= 0 ? (cv << pos) : (cv >> (-pos));
                }
                pk[b] = (uint8_t)v;
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// MODE 1 fixup: re-code, in exact f64, the rows of one warp-tile that the
// hot loop flagged (a code within the fp32 guard band of a tie, or a range
// outside fp32's comfort zone; ~0.3% of rows on realistic data).  Called by
// each warp after its tile loop for its own flagged tiles, so the f64 code
// shares no live range with the hot loop and the error sum stays in a fixed
// order.  The packed codes of each flagged record are overwritten in the
// payload; the rows' exact errors are added (the hot loop left them out).
// ---------------------------------------------------------------------------
template <int G, int C, int VEC, bool PAD>
__device__ __forceinline__ void fix_tile(const WriterArgs &a, const int64_t *s_sched,
                                         const int64_t *s_sec, int t, int64_t i0,
                                         unsigned m, uint8_t *cs_warp, int d, WAcc &acc) {
    // rows i0 + slot of table t whose bit slot is set in m
    using Lay = Layout<G, C, VEC>;
    constexpr int EPL = C * VEC;
    const int lane = threadIdx.x & 31;
    const int lig = lane & (G - 1), slot = lane / G;
    const int nt = a.ntables;
    const ds_table_desc &td = a.t[t];
    const bool mine = (m >> slot) & 1u;
    uint8_t *cs = cs_warp + slot * d;
    int64_t local = 0;
    if (mine) {
        local = i0 + slot;
        if (a.incremental) {
            const int64_t raw = a.ids[s_sched[2 * nt + 1 + t] + i0 + slot];
            local = a.ids_local ? raw : raw - td.row_base;  // validated by the hot loop
        }
    }
    float x[EPL];
    if (mine)
        load_row<G, C, VEC>(a.staged ? a.staged + (s_sched[2 * nt + 1 + t] + i0 + slot) * (int64_t)d
                                     : td.values + local * td.ld,
                            d, lig, x, 0.f);
    else
#pragma unroll
        for (int k = 0; k < EPL; k++) x[k] = 0.f;
    float mn = INFINITY, mx = -INFINITY;
#pragma unroll
    for (int k = 0; k < EPL; k++)
        if (!PAD || Lay::elem(lig, k) < d) {
            mn = fminf(mn, x[k]);
            mx = fmaxf(mx, x[k]);
        }
    const float lo = grp_min<G>(mn), hi = grp_max<G>(mx);
    const RowQ rq = make_rowq(lo, hi, a.L, a.invL);
    // the hot loop's codes (the packed code_row_m1 fuses the product, the
    // generic path rounds it), exact codes for the ambiguous elements only
    const bool fused = DS_M1_PACKED && DS_M1_FUSED && VEC == 4 && G > 1 &&
                       (a.bitwidth == 8 || a.bitwidth == 4 || a.bitwidth == 2);
    int qfast[EPL], qex[EPL];
    bool changed = false;
#pragma unroll
    for (int k = 0; k < EPL; k++) {
        const float t = __fsub_rn(x[k], rq.lo);
        float qm, r;
        if (fused) {
            qm = __fmaf_rn(t, rq.inv, 12582912.0f);
            r = __fmaf_rn(t, rq.inv, __fsub_rn(12582912.0f, qm));
        } else {
            const float v = __fmul_rn(t, rq.inv);
            qm = __fadd_rn(v, 12582912.0f);
            r = __fsub_rn(v, __fsub_rn(qm, 12582912.0f));
        }
        qfast[k] = __float_as_int(qm) & 0x3fffff;
        qex[k] = qfast[k];
        const bool in = mine && (!PAD || Lay::elem(lig, k) < d);
        if (in && (rq.mode == 2 || fabsf(r) > 0.5f - rq.eps)) {
            qex[k] = code_exact(x[k], lo, hi, rq.s, a.L);
            acc.n_exact_codes++;
            changed |= qex[k] != qfast[k];
        }
    }
    // a fast code was wrong (exact ties; rare): replace the record's codes and
    // swap the row's error contribution
    // (range outside fp32's comfort zone: the hot loop left the error out)
    const int any_changed = grp_or<G>(changed ? 1 : 0);  // every lane shuffles
    const bool row_changed = mine && (rq.mode == 2 || any_changed != 0);
    if (__any_sync(DS_FULL_MASK, row_changed)) {
        double sf = 0.0, se = 0.0;
#pragma unroll
        for (int k = 0; k < EPL; k++) {
            const int e = Lay::elem(lig, k);
            if (row_changed && e < d) {
#if DS_ERR_F2F
                const double ef = __dsub_rn((double)x[k], (double)deq_exact(qfast[k], lo, rq.s));
#else
                const double ef = err_fast(x[k], (uint32_t)qfast[k], rq.s, (double)lo);  // as the hot loop
#endif
                const double ee = __dsub_rn((double)x[k], (double)deq_exact(qex[k], lo, rq.s));
                sf = fma(ef, ef, sf);
                se = fma(ee, ee, se);
                cs[e] = (uint8_t)qex[k];
            }
        }
        sf = grp_sumd<G>(sf);
        se = grp_sumd<G>(se);
        if (row_changed && lig == 0)
            acc.err += (se > 0.0 ? se * rsqrt(se) : 0.0) -
                       (rq.mode == 2 ? 0.0 : (DS_ERR_F2F ? (sf > 0.0 ? sf * rsqrt(sf) : 0.0) : row_err(sf)));
        __syncwarp();
        if (row_changed) {  // overwrite the record's packed codes (LSB-first bitstream)
            uint8_t *pk = a.payload + s_sec[t] + (a.write_headers ? DS_HEADER_SIZE : 0) +
                          (i0 + slot) * a.rec + a.code_off;
            const int N = a.bitwidth;
            for (int b = lig; b < a.packed; b += G) {
                const int bit0 = 8 * b;
                const int j0 = bit0 / N, j1 = min(d - 1, (bit0 + 7) / N);
                uint32_t v = 0;
                for (int j = j0; j <= j1; j++) {
                    const int pos = j * N - bit0;
                    const uint32_t cv = cs[j];
                    v |= pos >= 0 ? (cv << pos) : (cv >> (-pos));
                }
                pk[b] = (uint8_t)v;
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// MODE 0/1: HBM-bound gather.  Every warp runs its own pipeline (no CTA
// barriers) over tiles of 32 records: one dirty-row id per lane, loaded two
// tiles ahead into registers; the tile's rows move in G chunks of 32/G rows
// (a chunk = one row per group of G lanes) through a ring of NS cp.async
// stages in the warp's shared memory, NS-1 chunks ahead of the chunk being
// coded into the tile's record stage; the 32 records then stream to HBM as
// one contiguous run.  Per-tile bookkeeping is amortised over 32 rows at
// every dim.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int align16(int v) { return (v + 15) & ~15; }

// 16-byte chunk g of a row-chunk stage lives at slot g ^ ((g >> 3) & 3): the
// 8 lanes of a quarter-warp then hit 8 distinct bank groups both when lane
// lig reads chunks C*lig..C*lig+C-1 of its row and when consecutive lanes
// write consecutive chunks (a permutation inside each aligned group of 4)
__device__ __forceinline__ int chunk_swz(int g) { return g ^ ((g >> 3) & 3); }

#ifndef DS_WRITER_MINB
#define DS_WRITER_MINB 2
#endif

#ifndef DS_FIX_INLINE
#define DS_FIX_INLINE 1  // 0: flagged rows always re-coded in a pass after the warp's tiles
#endif
#ifndef DS_WRITER_NS
#define DS_WRITER_NS 3
#endif
#ifndef DS_WRITER_NS1
#define DS_WRITER_NS1 2
#endif
template <int G>
__host__ __device__ constexpr int writer_stages() { return G == 1 ? DS_WRITER_NS1 : DS_WRITER_NS; }

// the greedy writer's CTA: 256 threads at 2 CTAs/SM (128 registers) for the
// fp32 candidate passes; the bucketed search (DS_GREEDY_BUCKET=1) needs 4 KB
// more shared memory per row: 128 threads at 3 CTAs/SM, a 2-stage ring
#ifndef DS_WRITER_MINB_GREEDY
#define DS_WRITER_MINB_GREEDY (DS_GREEDY_BUCKET ? 3 : 2)
#endif
#ifndef DS_WT_GREEDY
#define DS_WT_GREEDY (DS_GREEDY_BUCKET ? 128 : 256)
#endif
#ifndef DS_WRITER_NS_GREEDY
#define DS_WRITER_NS_GREEDY (DS_GREEDY_BUCKET ? 2 : 3)
#endif
#ifndef DS_WT_WARP
#define DS_WT_WARP WT  // threads per CTA of the warp-pipelined writer
#endif
template <int G, int C, int VEC, int MODE, bool PAD>
__global__ void __launch_bounds__(MODE == 2 ? DS_WT_GREEDY : DS_WT_WARP,
                                  MODE == 2 ? DS_WRITER_MINB_GREEDY : DS_WRITER_MINB)
    writer_warp_kernel(const WriterArgs a) {
    pdl_wait();  // K2's ids and counts (PDL launch after the emit pass)
    constexpr int EPL = C * VEC;
    constexpr int RPC = 32 / G;  // rows per chunk
    constexpr int NS = MODE == 2 ? DS_WRITER_NS_GREEDY : writer_stages<G>();
    // one-lane rows re-code flagged rows in place (measured faster); wider
    // groups keep the after-loop pass (fewer live registers in the hot loop)
    constexpr bool FIXIN = DS_FIX_INLINE && G == 1;
    const int TR = a.tile_rows;  // records per tile: 32, fewer for huge records (host)
    const int NCH = TR / RPC;    // chunks per tile (the host keeps NCH >= NS - 1)
    extern __shared__ __align__(16) uint8_t smem[];
    const int d = PAD ? a.dim : (VEC == 4 ? 4 * G * C : G * C);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int lig = lane & (G - 1);
    const int slot = lane / G;  // row of the chunk this group codes
    // per-warp shared memory (the host computes the same sizes)
    const int stage_b = align16(TR * a.rec) + 16;
    const int codes_b = align16(RPC * d);
    const int chunk_b = (RPC * d * 4 + 63) & ~63;  // whole 4-chunk swizzle groups
    // greedy scratch per row: the bucket sort + prefix sums (ds_greedy.cuh),
    // which the exact re-evaluation also borrows
    static_assert(bucket_bytes(G * EPL) == BucketLayout<G * EPL>::BYTES, "host and device scratch sizes");
    const int gscr = greedy_scratch_bytes(G * EPL, d);
    const int exact_b = MODE == 2 ? align16(RPC * gscr) : 0;
    const int warp_b = stage_b + codes_b + NS * chunk_b + exact_b;
    uint8_t *smem_al = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem) + 15) & ~(uintptr_t)15);
    uint8_t *wbase = smem_al + (size_t)wid * warp_b;
    uint8_t *stage = wbase;
    uint8_t *codes = wbase + stage_b;
    float *ring = reinterpret_cast<float *>(codes + codes_b);
    double *exact = reinterpret_cast<double *>(codes + codes_b + NS * chunk_b);
    // 16-byte chunk g of a stage: swizzled when each lane reads its own row
    // (G == 1: rows 64 B apart would put 4 lanes on one bank group), natural
    // otherwise (consecutive lanes already read consecutive chunks, and the
    // cp.async writes stay contiguous)
    auto slot_of = [](int g) -> int { return G == 1 ? chunk_swz(g) : g; };

    __shared__ int64_t s_sched[3 * DS_MAX_TABLES + 2];
    __shared__ double s_red[WT / 32];
    __shared__ int64_t s_sec[DS_MAX_TABLES + 1];
    writer_layout(a, s_sched, s_sec);
    const int nt = a.ntables;
    WAcc acc;
    if (writer_fits(a, s_sched, s_sec)) {  // else flagged (DS_FLAG_CAPACITY) by CTA 0
        const int64_t total_tiles = s_sched[nt];
        const int nwc = blockDim.x >> 5;  // warps per CTA (fewer for huge records)
        const int64_t gw = (int64_t)blockIdx.x * nwc + wid;
        const int64_t nwarps = (int64_t)gridDim.x * nwc;
        // multi-lane rows: each warp codes one contiguous run of tiles (ids and
        // records contiguous); one-lane rows: tiles strided over the warps
        // (measured faster there).  Either way a warp's tiles only move
        // forward, so the table search is incremental.
        constexpr bool RUN = G > 1;
        const int64_t tpw = (total_tiles + nwarps - 1) / nwarps;
        const int64_t tbeg = RUN ? min(total_tiles, gw * tpw) : gw;
        const int64_t tend = RUN ? min(total_tiles, tbeg + tpw) : total_tiles;
        const int64_t tstep = RUN ? 1 : nwarps;
        int tcur = tbeg < tend ? tile_table(s_sched, nt, tbeg, lane) : 0;  // table of the newest tinfo
        // tile j of this warp: table, first record, records, and lane's row id
        struct TI {
            int t, nrow;
            int64_t i0, loc;  // loc: table-local row of record `lane` (-1: none / invalid)
            bool ok;
        };
        auto tinfo = [&](int j) -> TI {  // called for j = 0, 1, 2, ... in order
            TI r;
            const int64_t tile = tbeg + (int64_t)j * tstep;
            r.ok = tile < tend;
            if (r.ok) {
                // warp-uniform: runs of tiles step table by table; strided
                // tiles can jump many small tables -- one ballot per 32 tables
                if (RUN || !DS_TT_BALLOT) while (tcur + 1 < nt && s_sched[tcur + 1] <= tile) tcur++;
                else tcur = tile_table(s_sched, nt, tile, lane);
            }
            r.t = r.ok ? tcur : 0;
            r.i0 = r.ok ? (tile - s_sched[r.t]) * TR : 0;
            r.nrow = r.ok ? (int)min((int64_t)TR, s_sched[nt + 1 + r.t] - r.i0) : 0;
            r.loc = -1;
            // the raw id only: nothing here may consume the load, or the warp
            // waits for it now instead of a tile later (resolve())
            if (lane < r.nrow)
                r.loc = a.incremental ? a.ids[s_sched[2 * nt + 1 + r.t] + r.i0 + lane] : r.i0 + lane;
            return r;
        };
        // raw id -> table-local row, validated (-2: out of range); once per tile,
        // a tile after its load was issued
        auto resolve = [&](TI &r) {
            if (lane < r.nrow) {
                const ds_table_desc &td = a.t[r.t];
                // ids from capture are table-local; plan ids are global
                const int64_t loc = (a.incremental && !a.ids_local) ? r.loc - td.row_base : r.loc;
                r.loc = (loc < 0 || loc >= td.rows) ? -2 : loc;
            }
        };
        // chunk `sub` of tile T into ring stage st (one row per lane group)
        auto issue = [&](const TI &T, int sub, int st) {
            const int r = sub * RPC + slot;
            const int64_t loc = __shfl_sync(DS_FULL_MASK, T.loc, r);
            if (T.ok && r < T.nrow && loc >= 0) {
                const ds_table_desc &td = a.t[T.t];
                // staged: record i0 + r of table t sits at its packed position
                const float *src = a.staged ? a.staged + (s_sched[2 * nt + 1 + T.t] + T.i0 + r) * (int64_t)d
                                            : td.values + loc * td.ld;
                float *dst = ring + st * (chunk_b / 4) + slot * d;
                float *sbase = ring + st * (chunk_b / 4);
#pragma unroll
                for (int c = 0; c < C; c++) {
                    if (VEC == 4) {
                        // global: consecutive lanes, consecutive 16 bytes; shared:
                        // 16-byte chunk g of the stage at swizzled slot chunk_swz(g)
                        const int q = lig + c * G;
                        if (4 * q < d) cp_async16(sbase + 4 * slot_of(slot * (d >> 2) + q), src + 4 * q);
                    } else {
                        const int e = lig + c * G;
                        if (e < d) cp_async4(dst + e, src + e);
                    }
                }
            }
            cp_async_commit();
        };
        TI cur = tinfo(0), nxt = tinfo(1);
        resolve(cur);
        resolve(nxt);
        // prologue: the first NS-1 chunks of the warp's chunk stream
        int isub = 0, irel = 0, ist = 0;  // next chunk to issue: sub-chunk, tile (0 cur, 1 nxt), stage
#pragma unroll
        for (int cc = 0; cc < NS - 1; cc++) {
            issue(irel == 0 ? cur : nxt, isub, ist);
            ist++;
            if (++isub == NCH) { isub = 0; irel++; }
        }
        int cst = 0;  // ring stage of the chunk being coded
        for (int j = 0; cur.ok; j++) {
            const TI far = tinfo(j + 2);  // ids two tiles ahead (plain loads, consumed a tile later)
            const ds_table_desc &td = a.t[cur.t];
            bool row_fix = false;  // lane r: record r of the tile goes to the fixup pass
            double tile_sse = 0.0;  // lane r: record r's sum of squares (DS_ERR_DEFER)
#pragma unroll 1
            for (int sub = 0; sub < NCH; sub++) {
                // keep NS-1 chunks in flight
                issue(irel == 0 ? cur : nxt, isub, ist);
                ist = ist + 1 == NS ? 0 : ist + 1;
                if (++isub == NCH) { isub = 0; irel++; }
                cp_async_wait<NS - 1>();  // this lane's copies of the chunk landed (it reads only those)
                const int r = sub * RPC + slot;
                const int64_t loc = __shfl_sync(DS_FULL_MASK, cur.loc, r);
                bool valid = r < cur.nrow;
                if (valid && loc < 0) {
                    acc.bad_ids = true;
                    valid = false;
                }
                float x[EPL];
                const float *row = ring + cst * (chunk_b / 4) + slot * d;
                if (VEC == 4) {
                    // G == 1: the lane's own row, through the swizzle (conflict-free);
                    // G > 1: chunk lig + cv*G (consecutive lanes, consecutive chunks)
                    const float *sb = ring + cst * (chunk_b / 4);
#pragma unroll
                    for (int cv = 0; cv < C; cv++) {
                        const int q = G == 1 ? cv : lig + cv * G;
                        const float4 v = (valid && 4 * q < d)
                                             ? *reinterpret_cast<const float4 *>(sb + 4 * slot_of(slot * (d >> 2) + q))
                                             : make_float4(0.f, 0.f, 0.f, 0.f);
                        x[4 * cv] = v.x; x[4 * cv + 1] = v.y; x[4 * cv + 2] = v.z; x[4 * cv + 3] = v.w;
                    }
                } else {
#pragma unroll
                    for (int kk = 0; kk < C; kk++) {
                        const int e = lig + kk * G;
                        x[kk] = (valid && e < d) ? row[e] : 0.f;
                    }
                }
                const bool fix = code_row<G, C, VEC, MODE, PAD, VEC == 4 && G == 1>(a, td, x, row, valid, valid ? loc : 0,
                                                                stage + r * a.rec, codes + slot * d,
                                                                exact + slot * (gscr / 8), lig, d, acc);
                if (MODE == 1 && FIXIN) {
                    // exact fixup now, from the registers (no second pass)
                    if (__any_sync(DS_FULL_MASK, fix))
                        fix_rows_inline<G, C, VEC, PAD, VEC == 4 && G == 1>(a, x, lig, d, fix, stage + r * a.rec,
                                                                            codes + slot * d, acc);
                } else if (MODE == 1) {  // record r's flag (and sum of squares) to lane r
                    const int from = ((lane - sub * RPC) & (RPC - 1)) * G;
                    const bool mine = lane >= sub * RPC && lane < (sub + 1) * RPC;
                    const bool f = __shfl_sync(DS_FULL_MASK, fix, from);
                    if (mine) row_fix |= f;
                    if (DS_ERR_DEFER) {
                        const double rs = __shfl_sync(DS_FULL_MASK, acc.row_sse, from);
                        if (mine) tile_sse = rs;
                        acc.row_sse = 0.0;
                    }
                }
                __syncwarp();  // every lane is done with ring stage cst before it is refilled
                cst = cst + 1 == NS ? 0 : cst + 1;
            }
            irel--;  // the next tile becomes the current one
            if (MODE == 1 && !FIXIN && DS_ERR_DEFER)  // the tile's row errors, 32 roots at once
                acc.err += DS_ERR_F2F ? (tile_sse > 0.0 ? tile_sse * rsqrt(tile_sse) : 0.0) : row_err(tile_sse);
            if (MODE == 1 && !FIXIN) {
                const unsigned fm = __ballot_sync(DS_FULL_MASK, row_fix);
                if (lane == 0) a.fix_mask[tbeg + (int64_t)j * tstep] = fm;
            }
            const int64_t dst = s_sec[cur.t] + (a.write_headers ? DS_HEADER_SIZE : 0) + cur.i0 * a.rec;
            copy_out(a.payload + dst, stage, (int64_t)cur.nrow * a.rec, lane, 32);
            __syncwarp();  // the stage is rewritten by the next tile
            cur = nxt;
            nxt = far;
            resolve(nxt);
        }
        cp_async_wait<0>();  // nothing may land after the warp exits
        if (MODE == 1 && !FIXIN) {
            // exact re-coding of this warp's flagged records (its tiles, in order)
            __syncwarp();
            for (int64_t tile = tbeg; tile < tend; tile += tstep) {
                const unsigned m = a.fix_mask[tile];
                if (!m) continue;
                const int t = tile_table(s_sched, nt, tile, lane);
                const int64_t i0 = (tile - s_sched[t]) * TR;
                for (int sub = 0; sub < NCH; sub++) {
                    const unsigned ms = (m >> (sub * RPC)) & (RPC == 32 ? 0xffffffffu : ((1u << RPC) - 1u));
                    if (ms) fix_tile<G, C, VEC, PAD>(a, s_sched, s_sec, t, i0 + sub * RPC, ms, codes, d, acc);
                }
            }
        }
    }
    writer_epilogue(a, acc, s_red);
}

// ---------------------------------------------------------------------------
// MODE 2 (greedy ranges): compute-bound (~20 candidate evaluations per row);
// rows load straight into registers, one pass of WT/G rows per tile.
// ---------------------------------------------------------------------------
template <int G, int C, int VEC, int MODE, bool PAD>
__global__ void __launch_bounds__(WT, 1) writer_kernel(const WriterArgs a) {
    static_assert(!(MODE == 2 && DS_GREEDY_BUCKET), "the bucketed search reads rows from the warp writer's ring");
    pdl_wait();
    constexpr int EPL = C * VEC;
    constexpr int RPP = WT / G;  // rows per pass
    extern __shared__ __align__(16) uint8_t smem[];
    const int TR = a.tile_rows;
    const int d = PAD ? a.dim : (VEC == 4 ? 4 * G * C : G * C);
    const int stage_bytes = align16(TR * a.rec) + 16;
    uint8_t *stage = smem;
    uint8_t *codes_sh = smem + stage_bytes;                                 // RPP * d bytes
    const int gscr = greedy_scratch_bytes(G * EPL, d);  // per row: the greedy scratch
    double *exact_sh = reinterpret_cast<double *>(codes_sh + align16(RPP * d));

    __shared__ int64_t s_sched[3 * DS_MAX_TABLES + 2];
    __shared__ double s_red[WT / 32];
    const int nt = a.ntables;
    __shared__ int64_t s_sec[DS_MAX_TABLES + 1];
    writer_layout(a, s_sched, s_sec);
    WAcc acc;
    const int lane = threadIdx.x & 31;
    const int lig = lane & (G - 1);
    const int slot = threadIdx.x / G;
    if (writer_fits(a, s_sched, s_sec)) {  // else flagged (DS_FLAG_CAPACITY) by CTA 0
        const int64_t total_tiles = s_sched[nt];
        for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
            const int t = tile_table(s_sched, nt, tile, lane);
            const ds_table_desc &td = a.t[t];
            const int64_t i0 = (tile - s_sched[t]) * TR;
            const int nrow = (int)min((int64_t)TR, s_sched[nt + 1 + t] - i0);
            const int64_t ids_base = s_sched[2 * nt + 1 + t];
            for (int p = 0; p < TR; p += RPP) {
                const int r = p + slot;
                bool valid = r < nrow;
                if (!__any_sync(DS_FULL_MASK, valid)) continue;
                int64_t local = 0;
                if (valid) {
                    local = i0 + r;
                    if (a.incremental) {
                        int64_t id = __ldg(a.ids + ids_base + i0 + r);
                        local = a.ids_local ? id : id - td.row_base;
                        if (local < 0 || local >= td.rows) {
                            acc.bad_ids = true;
                            valid = false;
                            local = 0;
                        }
                    }
                }
                float x[EPL];
                if (valid) load_row<G, C, VEC>(td.values + local * td.ld, d, lig, x, 0.f);
                else
#pragma unroll
                    for (int k = 0; k < EPL; k++) x[k] = 0.f;
                code_row<G, C, VEC, MODE, PAD>(a, td, x, nullptr, valid, local, stage + r * a.rec,
                                               codes_sh + slot * d, exact_sh + slot * (gscr / 8), lig,
                                               d, acc);
            }
            __syncthreads();
            const int64_t dst = s_sec[t] + (a.write_headers ? DS_HEADER_SIZE : 0) + i0 * a.rec;
            copy_out(a.payload + dst, stage, (int64_t)nrow * a.rec, threadIdx.x, WT);
            __syncthreads();
        }
    }
    writer_epilogue(a, acc, s_red);
}

// ---------------------------------------------------------------------------
// host dispatch
// ---------------------------------------------------------------------------
typedef void (*writer_fn)(const WriterArgs);
#ifndef DS_GREEDY_CTA
#define DS_GREEDY_CTA 0  // 1: the greedy ranges run in the CTA-tiled writer_kernel
#endif

struct Cfg {
    int G, C, VEC;
};

// ~16 elements per lane: per-row work (range, scale, record fields) is then
// amortised over enough elements, and small dims need no cross-lane shuffles
// (dim 16 -> one thread per row, four 128-bit chunks).
static int next_pow2(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

#ifndef DS_EPL_NAIVE
#define DS_EPL_NAIVE 16
#endif
// mode 2 (greedy search) keeps ~16 elements per lane (register-bound); the
// HBM-bound naive/fp32 writer amortises per-row work over DS_EPL_NAIVE
#ifndef DS_EPL_GREEDY
#define DS_EPL_GREEDY 16
#endif
static Cfg pick_cfg(int d, bool vec4, int mode = 2) {
    Cfg c;
    const int epl = mode == 2 ? DS_EPL_GREEDY : DS_EPL_NAIVE;
    if (vec4) {
        int chunks = d / 4;
        c.VEC = 4;
        c.G = next_pow2((chunks + epl / 4 - 1) / (epl / 4));
        if (c.G > 32) c.G = 32;
        c.C = next_pow2((chunks + c.G - 1) / c.G);
    } else {
        c.VEC = 1;
        c.G = next_pow2((d + 15) / 16);
        if (c.G > 32) c.G = 32;
        c.C = next_pow2((d + c.G - 1) / c.G);
    }
    return c;
}

template <int MODE, bool PAD>
static writer_fn select_writer(const Cfg &c) {
#define DS_W(G_, C_, V_) \
    if (c.G == G_ && c.C == C_ && c.VEC == V_)                                                  \
    {                                                                                            \
        if constexpr (MODE == 2 && DS_GREEDY_CTA) return writer_kernel<G_, C_, V_, MODE, PAD>;   \
        else return writer_warp_kernel<G_, C_, V_, MODE, PAD>;                                   \
    }
    DS_W(1, 1, 4) DS_W(1, 2, 4) DS_W(1, 4, 4) DS_W(2, 4, 4) DS_W(4, 4, 4) DS_W(8, 4, 4)
    DS_W(16, 4, 4) DS_W(32, 4, 4) DS_W(32, 8, 4)
    if constexpr (MODE != 2) {
        DS_W(1, 8, 4) DS_W(2, 8, 4) DS_W(4, 8, 4) DS_W(8, 8, 4) DS_W(16, 8, 4)
    }
#if DS_EPL_GREEDY == 32
    if constexpr (MODE == 2) {
        DS_W(1, 8, 4) DS_W(2, 8, 4) DS_W(4, 8, 4) DS_W(8, 8, 4) DS_W(16, 8, 4)
        DS_W(1, 32, 1) DS_W(2, 32, 1) DS_W(4, 32, 1) DS_W(8, 32, 1) DS_W(16, 32, 1)
    }
#endif
#if DS_EPL_GREEDY == 8
    if constexpr (MODE == 2) {
        DS_W(2, 2, 4) DS_W(4, 2, 4) DS_W(8, 2, 4) DS_W(16, 2, 4) DS_W(32, 2, 4)
        DS_W(1, 8, 1) DS_W(2, 8, 1) DS_W(4, 8, 1) DS_W(8, 8, 1) DS_W(16, 8, 1) DS_W(32, 8, 1)
    }
#endif
    DS_W(1, 1, 1) DS_W(1, 2, 1) DS_W(1, 4, 1) DS_W(1, 8, 1) DS_W(1, 16, 1) DS_W(2, 16, 1)
    DS_W(4, 16, 1) DS_W(8, 16, 1) DS_W(16, 16, 1) DS_W(32, 16, 1) DS_W(32, 32, 1)
#undef DS_W
    return nullptr;
}


// per-mode instantiation units (ds_writer_m0.cu / _m1.cu / _m2.cu)
writer_fn select_writer_mode0(const Cfg &c, bool pad);
writer_fn select_writer_mode1(const Cfg &c, bool pad);
writer_fn select_writer_mode2(const Cfg &c, bool pad);
// one row per lane group (ds_writer_row.cu): d in {64, 128, 256}, naive 2/4/8-bit
writer_fn select_writer_row(int d, int g, int n);
size_t row_writer_smem_bytes(int d, int g, int64_t rec);

}  // namespace ds
