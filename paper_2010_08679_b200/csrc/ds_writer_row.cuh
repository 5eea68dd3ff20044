// ds_writer_row.cuh -- K3 for wide rows (d = 64 / 128 / 256, naive ranges at
// 2 / 4 / 8 bits): build_shard_payload's chunk loop (engine.py:139-187) with
// quantize_rows / pack_code_rows (quant.py:93-106, 372-382) and
// serialize_section (payload.py:84-104), one row per group of G lanes.
//
// Why a second writer: the warp-pipelined writer (ds_writer.cuh) spreads a
// 128-wide row over 8 lanes with 16 elements each, so every per-row step --
// the range reduction, the f64 scale, the guard band, the error norm, the
// record fields -- runs on all 8 lanes, and 16 warps x 128 registers leave no
// room to amortise it (ncu, T shard: 5.0-6.1 G warp instructions per step,
// ~47 per element, issue-bound at 41% of HBM).  Here G = 1..2 lanes own a
// row: per-row work is paid once per 64..128 elements, the row streams from
// shared memory in two passes (range, then codes), and registers are not the
// limit (one warp per CTA, ~150 registers).
//
// Per element the expensive part is the err_sum term (engine.py:171-173),
// x - deq(q) in f64 with deq(q) = f32(RN(RN(s*q) + lo)).  At 2 and 4 bits a
// row has only 4 / 16 levels: they are computed once per row, exactly, into a
// per-row table in shared memory (as doubles), so an element's term is one
// table load, one conversion of x, one subtraction and one FMA.  At 8 bits
// (256 levels) the level is computed per element without the conversion
// unit (err_fast: two rounded f64 ops, then integer rounding to f32).
//
// Data movement: a tile is RPC = 32/G rows (records).  Each row arrives by
// ONE TMA bulk copy (cp.async.bulk, issued by the row's first lane) into a
// ring of DS_ROW_NS stages whose mbarriers count the bytes, so the next tile
// lands while this one is coded.  Rows sit contiguous; within every aligned
// group of 8 chunks a lane starts at chunk (lane & 7), so the 8 lanes of a
// 128-byte wavefront read 8 different 16-byte bank groups.  Records of a tile
// are built in a stage laid out like the wire bytes and leave as one
// contiguous run (copy_out).
#pragma once

#include "ds_writer.cuh"

#ifndef DS_ROW_NS
#define DS_ROW_NS 2  // tile stages per warp
#endif
#ifndef DS_ROW_RND
#define DS_ROW_RND 1  // f64 -> f32 rounding of a level: 1 conversion unit, 0 integer bits
#endif
#ifndef DS_ROW_LEVELS
#define DS_ROW_LEVELS 0  // 1: 2/4-bit level table in shared memory (measured slower: bank conflicts)
#endif

namespace ds {

__device__ __forceinline__ unsigned rw_smem(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void rw_mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(rw_smem(bar)), "r"(count));
}
__device__ __forceinline__ void rw_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(rw_smem(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void rw_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "RW_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra RW_WAIT_%=;\n"
        "}\n" ::"r"(rw_smem(bar)),
        "r"(parity)
        : "memory");
}
// one row (or row part) global -> shared through the TMA engine
__device__ __forceinline__ void rw_bulk_load(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            rw_smem(dst)),
        "l"(src), "r"(bytes), "r"(rw_smem(bar))
        : "memory");
}

template <int D, int G>
struct RowWriterShape {
    static constexpr int CH = D / 4;    // 16-byte chunks per row
    static constexpr int RPC = 32 / G;  // rows (records) per tile
    static constexpr int CPL = CH / G;  // chunks per lane
    static_assert(CPL >= 8 && (CPL & 7) == 0, "the swizzle needs >= 8 chunks per lane");
    static constexpr int TAB = 16;      // level-table slots per row (128 bytes)
};

// shared memory of one (one-warp) CTA: NS row stages, the record stage, the
// level tables, alignment slack
__host__ __device__ constexpr size_t row_writer_smem(int d, int g, int64_t rec) {
    return (size_t)DS_ROW_NS * (32 / g) * d * 4 + (((32 / g) * (size_t)rec + 15) & ~(size_t)15) +
           (size_t)(32 / g) * 16 * 8 + 16 + 128;
}

// CTAs (warps) per SM the shared memory allows: the register cap follows
// from it (no point in keeping registers that no extra warp could use)
__host__ __device__ constexpr int rw_min_blocks(int d, int g) {
    return (int)(232448 / ((size_t)DS_ROW_NS * (32 / g) * d * 4 + 4096)) < 1
               ? 1
               : ((int)(232448 / ((size_t)DS_ROW_NS * (32 / g) * d * 4 + 4096)) > 16
                      ? 16
                      : (int)(232448 / ((size_t)DS_ROW_NS * (32 / g) * d * 4 + 4096)));
}

template <int N>
__device__ __forceinline__ void rw_store_codes(uint8_t *pk, int cc, uint32_t v) {
    if (N == 8) *reinterpret_cast<uint32_t *>(pk + 4 * cc) = v;
    else if (N == 4) *reinterpret_cast<uint16_t *>(pk + 2 * cc) = (uint16_t)v;
    else pk[cc] = (uint8_t)v;
}

// Exact re-check of a flagged row (a code within the fp32 guard band of a tie,
// or a range outside fp32's comfort zone; ~0.3% of rows): the ambiguous
// elements' codes in exact f64 (quant.py:99-106), the packed chunk rewritten
// where a code changes, and the row's error from the exact dequantized values
// (the hot loop leaves flagged rows' errors out).  Warp-collective for G > 1.
struct RwFix {
    double err;
    unsigned nexact;
};
template <int D, int G, int N>
__device__ __noinline__ RwFix rw_fix_row(const float *row, const RowQ rq, bool mine, uint8_t *pk, int lig,
                                         int lane) {
    using S = RowWriterShape<D, G>;
    double se = 0.0;
    unsigned nexact = 0;
    if (mine) {
        for (int cl = 0; cl < S::CPL; cl++) {
            const int c = lig * S::CPL + cl;
            const float4 v4 = *reinterpret_cast<const float4 *>(row + 4 * c);
            const float xs[4] = {v4.x, v4.y, v4.z, v4.w};
            uint32_t packed = 0;
            bool changed = false;
            for (int j = 0; j < 4; j++) {
                const float v = __fmul_rn(__fsub_rn(xs[j], rq.lo), rq.inv);
                const float qm = __fadd_rn(v, 12582912.0f);
                int q = (int)(__float_as_uint(qm) & 0x3fffffu);
                if (rq.mode == 2 || fabsf(__fsub_rn(v, __fsub_rn(qm, 12582912.0f))) > 0.5f - rq.eps) {
                    const int qx = code_exact(xs[j], rq.lo, rq.hi, rq.s, rq.L);
                    nexact++;
                    changed |= qx != q;
                    q = qx;
                }
                packed |= (uint32_t)q << (N * j);
                const double e = __dsub_rn((double)xs[j], (double)deq_exact(q, rq.lo, rq.s));
                se = fma(e, e, se);
            }
            if (changed) rw_store_codes<N>(pk, c, packed);
        }
    }
    se = grp_sumd<G>(se);
    return {mine && lig == 0 && se > 0.0 ? se * rsqrt(se) : 0.0, nexact};
}

template <int D, int G, int N>
__global__ void __launch_bounds__(32, rw_min_blocks(D, G)) writer_row_kernel(const WriterArgs a) {
    pdl_wait();  // K2's ids and counts (PDL launch after the emit pass)
    using S = RowWriterShape<D, G>;
    constexpr int RPC = S::RPC, CPL = S::CPL, CH = S::CH, NS = DS_ROW_NS;
    constexpr bool LEVELS = DS_ROW_LEVELS && N <= 4;
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int64_t s_sched[3 * DS_MAX_TABLES + 2];
    __shared__ int64_t s_sec[DS_MAX_TABLES + 1];
    __shared__ double s_red[1];
    __shared__ __align__(8) uint64_t s_bar[DS_ROW_NS];
    writer_layout(a, s_sched, s_sec);
    const int nt = a.ntables;
    const int lane = threadIdx.x & 31, slot = lane / G, lig = lane & (G - 1);
    float *ring = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(smem) + 127) & ~(uintptr_t)127);
    uint8_t *stage = reinterpret_cast<uint8_t *>(ring + NS * RPC * D);
    double *tab = reinterpret_cast<double *>(stage + ((RPC * a.rec + 15) & ~15));
    if (lane == 0) {
        for (int st = 0; st < NS; st++) rw_mbar_init(&s_bar[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    WAcc acc;
    if (writer_fits(a, s_sched, s_sec)) {
        const int64_t total_tiles = s_sched[nt];
        int tcur = 0;
        struct TI {
            int t, nrow;
            int64_t i0, loc;  // loc: raw id of record `slot`, then table-local row (-2 invalid)
            const float *src;  // the row of record `slot` (after resolve)
            bool ok;
        };
        auto tinfo = [&](int j) -> TI {  // j = 0, 1, 2, ... in order; loads the id only
            TI r;
            const int64_t tile = (int64_t)blockIdx.x + (int64_t)j * gridDim.x;
            r.ok = tile < total_tiles;
            if (r.ok)
                while (tcur + 1 < nt && s_sched[tcur + 1] <= tile) tcur++;
            r.t = r.ok ? tcur : 0;
            r.i0 = r.ok ? (tile - s_sched[r.t]) * RPC : 0;
            r.nrow = r.ok ? (int)min((int64_t)RPC, s_sched[nt + 1 + r.t] - r.i0) : 0;
            r.loc = -1;
            r.src = nullptr;
            if (slot < r.nrow)
                r.loc = a.incremental ? a.ids[s_sched[2 * nt + 1 + r.t] + r.i0 + slot] : r.i0 + slot;
            return r;
        };
        auto resolve = [&](TI &r) {  // a tile after the id load was issued
            if (slot < r.nrow) {
                const ds_table_desc &td = a.t[r.t];
                const int64_t loc = (a.incremental && !a.ids_local) ? r.loc - td.row_base : r.loc;
                r.loc = (loc < 0 || loc >= td.rows) ? -2 : loc;
                if (r.loc >= 0 && lig == 0)
                    r.src = a.staged ? a.staged + (s_sched[2 * nt + 1 + r.t] + r.i0 + slot) * (int64_t)D
                                     : td.values + r.loc * td.ld;
            }
        };
        // the tile's rows -> stage st: one TMA bulk copy per row (lane 0 of
        // the row's group), the stage's mbarrier counting the bytes
        auto issue = [&](const TI &T, int st) {
            const bool mine = T.src != nullptr;
            const unsigned m = __ballot_sync(DS_FULL_MASK, mine);
            if (lane == 0) rw_expect_tx(&s_bar[st], (unsigned)__popc(m) * (unsigned)(D * 4));
            __syncwarp();
            if (mine) rw_bulk_load(ring + (st * RPC + slot) * D, T.src, D * 4, &s_bar[st]);
        };
        TI ti[NS + 1];  // ti[0] = current tile, ti[k] = k tiles ahead (ti[NS] raw id only)
#pragma unroll
        for (int k = 0; k <= NS; k++) ti[k] = tinfo(k);
#pragma unroll
        for (int k = 0; k < NS; k++) resolve(ti[k]);
#pragma unroll
        for (int k = 0; k < NS - 1; k++)
            if (ti[k].ok) issue(ti[k], k);
        const int L = a.L;
        unsigned phase = 0;  // parity bit per stage
        for (int j = 0; ti[0].ok; j++) {
            const int st = j % NS;
            // keep NS-1 tiles in flight: tile j+NS-1 into the stage tile j-1 freed
            if (ti[NS - 1].ok) issue(ti[NS - 1], (j + NS - 1) % NS);
            const TI cur = ti[0];
            rw_wait(&s_bar[st], (phase >> st) & 1u);
            phase ^= 1u << st;
            const ds_table_desc &td = a.t[cur.t];
            bool valid = slot < cur.nrow;
            if (valid && cur.loc < 0) {
                acc.bad_ids = true;
                valid = false;
            }
            const float *row = ring + (st * RPC + slot) * D;
            // within each aligned group of 8 chunks a lane starts at chunk
            // (lane & 7): the 8 lanes of a wavefront read 8 different 16-byte
            // bank groups.  rot[k] = the k-th chunk of the group this lane reads.
            int rot[8];
#pragma unroll
            for (int k = 0; k < 8; k++) rot[k] = (k + lane) & 7;
            auto ld = [&](int cb, int k) -> float4 {
                return *reinterpret_cast<const float4 *>(row + 4 * (lig * CPL + cb + rot[k]));
            };
            uint8_t *rec = stage + slot * a.rec;
            // ---- pass 1: the row's range, NaN-propagating (engine.py:163-164;
            // a NaN / Inf element leaves lo or hi non-finite: DataError) ----
            float mn0 = INFINITY, mn1 = INFINITY, mx0 = -INFINITY, mx1 = -INFINITY;
            if (valid) {
#pragma unroll 2
                for (int cb = 0; cb < CPL; cb += 8) {
#pragma unroll
                    for (int k = 0; k < 8; k++) {
                        const float4 v = ld(cb, k);
                        mn0 = fmin_nan(mn0, fmin_nan(v.x, v.y));
                        mn1 = fmin_nan(mn1, fmin_nan(v.z, v.w));
                        mx0 = fmax_nan(mx0, fmax_nan(v.x, v.y));
                        mx1 = fmax_nan(mx1, fmax_nan(v.z, v.w));
                    }
                }
            }
            float mn = fmin_nan(mn0, mn1), mx = fmax_nan(mx0, mx1);
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) {
                mn = fmin_nan(mn, __shfl_xor_sync(DS_FULL_MASK, mn, o, G));
                mx = fmax_nan(mx, __shfl_xor_sync(DS_FULL_MASK, mx, o, G));
            }
            const bool fin = isfinite(mn) && isfinite(mx);
            if (valid && !fin) acc.bad_data = true;
            const bool row_ok = valid && fin;
            const RowQ rq = make_rowq(row_ok ? mn : 0.f, row_ok ? mx : 0.f, L, a.invL);
            const double lod = (double)rq.lo;
            // ---- the row's 2^N levels, exactly (quant.py:114-115), as doubles:
            // slot (q + slot) & 15 of the row's 128-byte table ----
            double *mytab = tab + slot * S::TAB;
            if (LEVELS) {
#pragma unroll
                for (int q = lig; q < (1 << N); q += G) {
                    const double w = __dadd_rn(__dmul_rn(rq.s, (double)q), lod);
                    mytab[(q + slot) & 15] = round_f32_in_f64(w);
                }
                __syncwarp();
            }
            // ---- pass 2: codes (certified fp32), err_sum terms, packed bytes ----
            uint8_t *pk = rec + a.code_off;
            float dev0 = 0.f, dev1 = 0.f;
            double s0 = 0.0, s1 = 0.0;
            if (valid) {
#pragma unroll 1
                for (int cb = 0; cb < CPL; cb += 8) {
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const int cl = cb + rot[k];
                    const float4 v4 = ld(cb, k);
                    const float xs[4] = {v4.x, v4.y, v4.z, v4.w};
                    uint32_t packed = 0;
#pragma unroll
                    for (int jj = 0; jj < 4; jj++) {
                        // min/max ranges hold every element: no clip, v in [0, L(1+5u)];
                        // round half to even through the 1.5*2^23 magic
                        const float v = __fmul_rn(__fsub_rn(xs[jj], rq.lo), rq.inv);
                        const float qm = __fadd_rn(v, 12582912.0f);
                        const uint32_t qi = __float_as_uint(qm) & 0x3fffffu;
                        const float dv = fabsf(__fsub_rn(v, __fsub_rn(qm, 12582912.0f)));
                        if (jj & 1) dev1 = fmaxf(dev1, dv); else dev0 = fmaxf(dev0, dv);
                        // engine.py:171-173: x - deq(q)
                        double er;
                        if (LEVELS) {
                            er = __dsub_rn((double)xs[jj], mytab[(qi + slot) & 15]);
                        } else {
                            // w = RN(RN(s*q) + lo); deq = f32(w) -- rounded by the
                            // conversion unit (DS_ROW_RND 1) or integer bits (0)
                            const double w = __dadd_rn(__dmul_rn(rq.s, code_to_f64(qi)), lod);
                            const double dq = DS_ROW_RND ? (double)__double2float_rn(w) : round_f32_in_f64(w);
                            er = __dsub_rn((double)xs[jj], dq);
                        }
                        if (jj & 1) s1 = fma(er, er, s1); else s0 = fma(er, er, s0);
                        packed |= qi << (N * jj);
                    }
                    rw_store_codes<N>(pk, lig * CPL + cl, row_ok ? packed : 0u);
                }
                }
            }
            const float dev = grp_max<G>(fmaxf(dev0, dev1));
            const bool fix = row_ok && (rq.mode == 2 || dev > 0.5f - rq.eps);
            const double sse = grp_sumd<G>(__dadd_rn(s0, s1));
            if (valid && lig == 0) {
                if (a.incremental) *reinterpret_cast<uint64_t *>(rec) = (uint64_t)(td.row_base + cur.loc);
                if (row_ok) {
                    if (!fix) acc.err += row_err(sse);  // flagged rows: the exact pass adds it
                    acc.n_rows++;
                    *reinterpret_cast<uint2 *>(rec + a.par_off) =
                        make_uint2(__float_as_uint(rq.lo), __float_as_uint(rq.hi));
                }
            }
            if (__any_sync(DS_FULL_MASK, fix)) {
                const RwFix f = rw_fix_row<D, G, N>(row, rq, fix, pk, lig, lane);
                acc.err += f.err;
                acc.n_exact_codes += f.nexact;
            }
            __syncwarp();
            const int64_t dst = s_sec[cur.t] + (a.write_headers ? DS_HEADER_SIZE : 0) + cur.i0 * a.rec;
            copy_out(a.payload + dst, stage, (int64_t)cur.nrow * a.rec, lane, 32);
            __syncwarp();  // stage st, the record stage and the tables are free again
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before the next bulk copies
#pragma unroll
            for (int k = 0; k < NS; k++) ti[k] = ti[k + 1];
            resolve(ti[NS - 1]);
            ti[NS] = tinfo(j + NS + 1);
        }
    }
    writer_epilogue(a, acc, s_red);
}

// d in {64, 128, 256}, G lanes per row -> the kernel for bitwidth N (2, 4, 8)
template <int D, int G>
static writer_fn select_row_writer_n(int n) {
    if (n == 8) return writer_row_kernel<D, G, 8>;
    if (n == 4) return writer_row_kernel<D, G, 4>;
    if (n == 2) return writer_row_kernel<D, G, 2>;
    return nullptr;
}

}  // namespace ds
