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
#include "ds_host.h"

#define DS_FLAG_CAPACITY 0x10u

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
    int64_t *sched;         // [0..nt] tile prefix, [nt+1..2nt] row counts, [2nt+1..3nt] ids offsets
    int64_t *sec_off;       // [nt+1] section offsets + total
    uint8_t *payload;
    int64_t capacity;
    double *partials;
    uint32_t *flags;
    unsigned long long *stats;
};

// ---------------------------------------------------------------------------
// shared-memory byte helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ void st_bytes(uint8_t *p, uint64_t v, int n) {
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
                                         int64_t nbytes) {
    // the stage is 16-byte aligned: an 8/16-byte aligned destination copies
    // with 64/128-bit moves (records of a tile are contiguous)
    const uintptr_t al = reinterpret_cast<uintptr_t>(dst);
    if ((al & 7) == 0) {
        if ((al & 15) == 0) {
            const int64_t n16 = nbytes >> 4;
            for (int64_t k = threadIdx.x; k < n16; k += blockDim.x)
                __stcs(reinterpret_cast<int4 *>(dst) + k, reinterpret_cast<const int4 *>(stage)[k]);
            for (int64_t b = (n16 << 4) + threadIdx.x; b < nbytes; b += blockDim.x) dst[b] = stage[b];
        } else {
            const int64_t n8 = nbytes >> 3;
            for (int64_t k = threadIdx.x; k < n8; k += blockDim.x)
                __stcs(reinterpret_cast<unsigned long long *>(dst) + k,
                       reinterpret_cast<const unsigned long long *>(stage)[k]);
            for (int64_t b = (n8 << 3) + threadIdx.x; b < nbytes; b += blockDim.x) dst[b] = stage[b];
        }
        return;
    }
    int head = (int)((4 - (reinterpret_cast<uintptr_t>(dst) & 3)) & 3);
    if (head > nbytes) head = (int)nbytes;
    if ((int)threadIdx.x < head) dst[threadIdx.x] = stage[threadIdx.x];
    int64_t nw = (nbytes - head) >> 2;
    uint32_t *dw = reinterpret_cast<uint32_t *>(dst + head);
    for (int64_t k = threadIdx.x; k < nw; k += blockDim.x)
        __stcs(dw + k, ld_u32_unaligned(stage, head + 4 * (int)k));  // streamed, not re-read
    int64_t done = head + 4 * nw;
    int tail = (int)(nbytes - done);
    if ((int)threadIdx.x < tail) dst[done + threadIdx.x] = stage[done + threadIdx.x];
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
//
// MODE 0/1 are HBM-bound gathers: per tile, (A) the tile's row ids go to
// shared memory with coalesced loads, (B) every row of the tile is requested
// with cp.async into shared memory (each lane copies the chunks it will later
// code), (C) rows are coded from shared memory into the record stage, (D) the
// stage streams out.  MODE 2 is compute-bound (~20 candidate evaluations per
// row) and loads each row straight into registers.
template <int G, int C, int VEC, int MODE, bool PAD>
__global__ void __launch_bounds__(WT, MODE == 2 ? 1 : 4) writer_kernel(const WriterArgs a) {
    using Lay = Layout<G, C, VEC>;
    constexpr int EPL = C * VEC;
    constexpr int RPP = WT / G;  // rows per pass
    extern __shared__ __align__(16) uint8_t smem[];
    const int TR = a.tile_rows;
    // without padding the layout covers the row exactly: dim is a constant
    const int d = PAD ? a.dim : (VEC == 4 ? 4 * G * C : G * C);
    // shared memory carve-up (host computes the same sizes)
    const int stage_bytes = ((TR * a.rec + 15) & ~15) + 16;
    uint8_t *stage = smem;
    uint8_t *codes_sh = smem + stage_bytes;                        // RPP * d bytes
    uint8_t *after_codes = codes_sh + ((RPP * d + 15) & ~15);
    double *exact_sh = reinterpret_cast<double *>(after_codes);    // MODE 2: RPP*(d+8)
    float *rows_sh = reinterpret_cast<float *>(after_codes);       // MODE 0/1: 2 x TR*d
    int64_t *ids_sh =                                               // MODE 0/1: 3 x TR
        reinterpret_cast<int64_t *>(after_codes + 2 * (((size_t)TR * d * 4 + 15) & ~(size_t)15));

    __shared__ int64_t s_sched[3 * DS_MAX_TABLES + 2];
    __shared__ double s_red[WT / 32];
    const int nt = a.ntables;
    for (int k = threadIdx.x; k < 3 * nt + 1; k += WT) s_sched[k] = a.sched[k];
    __syncthreads();
    if (a.sec_off[nt] > a.capacity) return;  // flagged by the layout kernel

    const int lane = threadIdx.x & 31;
    const int lig = lane & (G - 1);
    const int slot = threadIdx.x / G;
    const int L = a.L;
    const int64_t total_tiles = s_sched[nt];
    double err_acc = 0.0;
    unsigned n_exact_dec = 0, n_exact_codes = 0, n_rows = 0;
    bool bad_data = false, bad_ids = false;

    // tile k of this CTA -> (table, first record, records).  The table is the
    // last one whose first tile is <= tile: one ballot per 32 tables.
    auto tile_info = [&](int k, int &t, int64_t &i0, int &nrow) -> bool {
        const int64_t tile = blockIdx.x + (int64_t)k * gridDim.x;
        if (tile >= total_tiles) return false;
        t = 0;
        for (int b = 0; b < nt; b += 32) {
            unsigned m = __ballot_sync(DS_FULL_MASK, b + lane < nt && s_sched[b + lane] <= tile);
            if (m) t = b + 31 - __clz(m);
        }
        i0 = (tile - s_sched[t]) * TR;
        nrow = (int)min((int64_t)TR, s_sched[nt + 1 + t] - i0);
        return true;
    };
    // table-local row of a record (-1: outside the table -> BoundsError)
    auto local_of = [&](const ds_table_desc &td, int64_t raw) -> int64_t {
        // ids from capture are table-local; plan ids are global
        int64_t local = a.ids_local ? raw : raw - td.row_base;
        return (local < 0 || local >= td.rows) ? -1 : local;
    };
    // MODE 0/1 pipeline: ids of tile k+2 and rows of tile k+1 are in flight
    // (cp.async groups) while tile k is coded
    auto issue_ids = [&](int k) {
        int t, nrow;
        int64_t i0;
        if (a.incremental && tile_info(k, t, i0, nrow)) {
            const int64_t *src = a.ids + s_sched[2 * nt + 1 + t] + i0;
            int64_t *dst = ids_sh + (size_t)(k % 3) * TR;
            for (int j = threadIdx.x; j < nrow; j += WT) cp_async8(dst + j, src + j);
        }
        cp_async_commit();
    };
    auto issue_rows = [&](int k) {
        int t, nrow;
        int64_t i0;
        if (tile_info(k, t, i0, nrow)) {
            const ds_table_desc &td = a.t[t];
            const int64_t *ids = ids_sh + (size_t)(k % 3) * TR;
            float *rows = rows_sh + (size_t)(k & 1) * TR * d;
            for (int r = slot; r < nrow; r += RPP) {
                const int64_t local = a.incremental ? local_of(td, ids[r]) : i0 + r;
                if (local < 0) continue;
                const float *src = td.values + local * td.ld;
                float *dst = rows + r * d;
                // each lane requests exactly the chunks it will code
#pragma unroll
                for (int c = 0; c < C; c++) {
                    if (VEC == 4) {
                        int e = 4 * (lig + c * G);
                        if (e < d) cp_async16(dst + e, src + e);
                    } else {
                        int e = lig + c * G;
                        if (e < d) cp_async4(dst + e, src + e);
                    }
                }
            }
        }
        cp_async_commit();
    };
    if (MODE != 2) {  // prologue: ids(0) landed, then ids(1) and rows(0) in flight
        issue_ids(0);
        cp_async_wait<0>();
        __syncthreads();
        issue_ids(1);
        issue_rows(0);
    }

    for (int kt = 0;; kt++) {
        int t, nrow;
        int64_t i0;
        if (!tile_info(kt, t, i0, nrow)) break;
        const ds_table_desc &td = a.t[t];
        const int64_t ids_base = s_sched[2 * nt + 1 + t];
        const int64_t *tile_ids = ids_sh + (size_t)(kt % 3) * TR;
        const float *tile_rows = rows_sh + (size_t)(kt & 1) * TR * d;

        if (MODE != 2) {
            cp_async_wait<1>();  // ids(kt+1) landed (rows(kt) may still be in flight)
            __syncthreads();
            issue_ids(kt + 2);
            issue_rows(kt + 1);
            cp_async_wait<2>();  // rows(kt) landed: own copies only, no CTA barrier
        }

        for (int p = 0; p < TR; p += RPP) {
            const int r = p + slot;
            bool valid = r < nrow;
            if (!__any_sync(DS_FULL_MASK, valid)) continue;
            int64_t local = 0;
            float x[EPL];
            if (MODE != 2) {
                if (valid) {
                    local = a.incremental ? local_of(td, tile_ids[r]) : i0 + r;
                    if (local < 0) {
                        bad_ids = true;
                        valid = false;
                        local = 0;
                    }
                }
                if (valid) {
                    const float *row = tile_rows + r * d;
                    if (VEC == 4) {
#pragma unroll
                        for (int c = 0; c < C; c++) {
                            int e = 4 * (lig + c * G);
                            float4 v = e < d ? *reinterpret_cast<const float4 *>(row + e)
                                             : make_float4(0.f, 0.f, 0.f, 0.f);
                            x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < C; k++) {
                            int e = lig + k * G;
                            x[k] = e < d ? row[e] : 0.f;
                        }
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < EPL; k++) x[k] = 0.f;
                }
            } else {
                if (valid) {
                    const int64_t i = i0 + r;
                    local = i;
                    if (a.incremental) {
                        int64_t id = __ldg(a.ids + ids_base + i);
                        local = a.ids_local ? id : id - td.row_base;
                        if (local < 0 || local >= td.rows) {
                            bad_ids = true;
                            valid = false;
                            local = 0;
                        }
                    }
                }
                if (valid) load_row<G, C, VEC>(td.values + local * td.ld, d, lig, x, 0.f);
                else
#pragma unroll
                    for (int k = 0; k < EPL; k++) x[k] = 0.f;
            }
            const int64_t gid = td.row_base + local;
            uint8_t *rec = stage + r * a.rec;
            if (valid && a.incremental && lig == 0) {
                if ((reinterpret_cast<uintptr_t>(rec) & 7) == 0)
                    *reinterpret_cast<uint64_t *>(rec) = (uint64_t)gid;
                else
                    st_bytes(rec, (uint64_t)gid, 8);
            }

            if (MODE == 0) {
                if (valid) {
#pragma unroll
                    for (int k = 0; k < EPL; k++) {
                        int e = Lay::elem(lig, k);
                        if (e < d) st_u32(rec + a.par_off + 4 * e, __float_as_uint(x[k]));
                    }
                }
            } else {
                // finiteness (quant.py:70-72,173): x*0 is NaN exactly for NaN/Inf;
                // naive range: row min / max (engine.py:163-164)
                float nz = 0.f, mn = INFINITY, mx = -INFINITY;
#pragma unroll
                for (int k = 0; k < EPL; k++) {
                    if (!PAD || Lay::elem(lig, k) < d) {
                        nz = __fmaf_rn(x[k], 0.f, nz);
                        mn = fminf(mn, x[k]);
                        mx = fmaxf(mx, x[k]);
                    }
                }
                const bool fin = grp_sum<G>(nz) == 0.f;
                if (valid && !fin) bad_data = true;
                const bool row_ok = valid && fin;
                float lo = grp_min<G>(mn), hi = grp_max<G>(mx);
                if (!row_ok) { lo = 0.f; hi = 0.f; }
                if (MODE == 2) {
                    double *buf = exact_sh + slot * (d + 8);
                    greedy_row<G, C, VEC, PAD>(x, d, lig, row_ok, lo, hi, L, a.bins, a.steps, buf,
                                               lo, hi, n_exact_dec, n_exact_codes);
                }
                const RowQ rq = make_rowq(lo, hi, L, a.invL);
                float qf[EPL];
                if (MODE == 1) {
                    // min/max ranges hold every element: no clip, v in [0, L(1+5u)];
                    // one deviation test per row replaces per-element branches
                    float dev = 0.f;
#pragma unroll
                    for (int k = 0; k < EPL; k++) {
                        float v = __fmul_rn(__fsub_rn(x[k], rq.lo), rq.inv);
                        qf[k] = rintf(v);
                        dev = fmaxf(dev, fabsf(__fsub_rn(v, qf[k])));
                    }
                    dev = grp_max<G>(dev);
                    if (row_ok && (rq.mode == 2 || dev > 0.5f - rq.eps)) {
                        // rare: a code within the guard band of a tie -> exact f64
#pragma unroll
                        for (int k = 0; k < EPL; k++) {
                            if (!PAD || Lay::elem(lig, k) < d) {
                                qf[k] = (float)code_exact_slow(x[k], lo, hi, rq.s, L);
                                n_exact_codes++;
                            }
                        }
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < EPL; k++) qf[k] = (float)code_of(x[k], rq, n_exact_codes);
                }
                int q[EPL];
                double sse = 0.0;
#pragma unroll
                for (int k = 0; k < EPL; k++) {
                    const bool in = row_ok && (!PAD || Lay::elem(lig, k) < d);
                    if (!in) qf[k] = 0.f;
                    // code as an integer from the float bits (q < 2^22): 1.5*2^23 + q
                    q[k] = __float_as_int(__fadd_rn(qf[k], 12582912.0f)) & 0x3fffff;
                    // err_sum term (engine.py:171-173): exact dequantized value
                    float dq = __double2float_rn(__dadd_rn(__dmul_rn(rq.s, (double)qf[k]), (double)lo));
                    double er = __dsub_rn((double)x[k], (double)dq);
                    sse = in ? fma(er, er, sse) : sse;
                }
                sse = grp_sumd<G>(sse);
                if (row_ok && lig == 0) {
                    err_acc += sqrt(sse);
                    n_rows++;
                    st_u32(rec + a.par_off, __float_as_uint(lo));
                    st_u32(rec + a.par_off + 4, __float_as_uint(hi));
                }
                // ---- pack (quant.py:376-382): LSB-first bitstream ----
                uint8_t *pk = rec + a.code_off;
                if (VEC == 4 && (a.bitwidth == 8 || a.bitwidth == 4 || a.bitwidth == 2)) {
                    if (valid) {
#pragma unroll
                        for (int c = 0; c < C; c++) {
                            int m = lig + c * G;  // chunk index: elements 4m..4m+3
                            if (4 * m < d) {
                                uint32_t v;
                                if (a.bitwidth == 8) {
                                    v = q[4 * c] | (q[4 * c + 1] << 8) | (q[4 * c + 2] << 16) |
                                        ((uint32_t)q[4 * c + 3] << 24);
                                    st_u32(pk + 4 * m, v);
                                } else if (a.bitwidth == 4) {
                                    v = q[4 * c] | (q[4 * c + 1] << 4) | (q[4 * c + 2] << 8) |
                                        (q[4 * c + 3] << 12);
                                    st_bytes(pk + 2 * m, v, 2);
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
                    uint8_t *cs = codes_sh + slot * d;
                    if (valid) {
#pragma unroll
                        for (int k = 0; k < EPL; k++) {
                            int e = Lay::elem(lig, k);
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
        }
        __syncthreads();
        int64_t dst = a.sec_off[t] + (a.write_headers ? DS_HEADER_SIZE : 0) + i0 * a.rec;
        copy_out(a.payload + dst, stage, (int64_t)nrow * a.rec);
        __syncthreads();
    }
    if (MODE != 2) cp_async_wait<0>();  // nothing may land after the CTA exits

    // per-CTA error partial (deterministic final sum in err_reduce_kernel)
    for (int o = 16; o > 0; o >>= 1) err_acc += __shfl_xor_sync(DS_FULL_MASK, err_acc, o);
    if (lane == 0) s_red[threadIdx.x >> 5] = err_acc;
    if (__any_sync(DS_FULL_MASK, bad_data) && lane == 0) atomicOr(a.flags, DS_FLAG_DATA);
    if (__any_sync(DS_FULL_MASK, bad_ids) && lane == 0) atomicOr(a.flags, DS_FLAG_BOUNDS);
    if (a.stats) {
        unsigned v0 = n_exact_dec, v1 = n_exact_codes, v2 = n_rows;
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
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < WT / 32; w++) s += s_red[w];
        a.partials[blockIdx.x] = s;
    }
}

// ---------------------------------------------------------------------------
// host dispatch
// ---------------------------------------------------------------------------
typedef void (*writer_fn)(const WriterArgs);

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

static Cfg pick_cfg(int d, bool vec4) {
    Cfg c;
    if (vec4) {
        int chunks = d / 4;
        c.VEC = 4;
        c.G = next_pow2((chunks + 3) / 4);
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
    if (c.G == G_ && c.C == C_ && c.VEC == V_) return writer_kernel<G_, C_, V_, MODE, PAD>;
    DS_W(1, 1, 4) DS_W(1, 2, 4) DS_W(1, 4, 4) DS_W(2, 4, 4) DS_W(4, 4, 4) DS_W(8, 4, 4)
    DS_W(16, 4, 4) DS_W(32, 4, 4) DS_W(32, 8, 4)
    DS_W(1, 1, 1) DS_W(1, 2, 1) DS_W(1, 4, 1) DS_W(1, 8, 1) DS_W(1, 16, 1) DS_W(2, 16, 1)
    DS_W(4, 16, 1) DS_W(8, 16, 1) DS_W(16, 16, 1) DS_W(32, 16, 1) DS_W(32, 32, 1)
#undef DS_W
    return nullptr;
}


// per-mode instantiation units (ds_writer_m0.cu / _m1.cu / _m2.cu)
writer_fn select_writer_mode0(const Cfg &c, bool pad);
writer_fn select_writer_mode1(const Cfg &c, bool pad);
writer_fn select_writer_mode2(const Cfg &c, bool pad);

}  // namespace ds
