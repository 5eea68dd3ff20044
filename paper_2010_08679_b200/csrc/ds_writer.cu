// ds_writer.cu -- K3: gather + range search + quantize + bit-pack + CNR1 records.
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
    const int64_t *ids;
    const int64_t *counts;  // device per-table counts (incremental) or null
    int64_t *sched;         // [0..nt] tile prefix, [nt+1..2nt+1] row counts
    int64_t *sec_off;       // [nt+1] section offsets + total
    uint8_t *payload;
    int64_t capacity;
    double *partials;
    uint32_t *flags;
    unsigned long long *stats;
};

// ---------------------------------------------------------------------------
// layout: section offsets, headers (payload.py:88-91), tile schedule
// ---------------------------------------------------------------------------
__global__ void layout_kernel(const WriterArgs a) {
    if (threadIdx.x != 0) return;
    int64_t off = 0, tiles = 0;
    int nt = a.ntables;
    for (int t = 0; t < nt; t++) {
        int64_t n = a.counts ? a.counts[t] : a.t[t].rows;
        a.sched[t] = tiles;
        a.sched[nt + 1 + t] = n;
        a.sec_off[t] = off;
        if (a.write_headers) {
            if (off + DS_HEADER_SIZE <= a.capacity) {
                uint8_t *h = a.payload + off;
                h[0] = 'C'; h[1] = 'N'; h[2] = 'R'; h[3] = '1';
                uint32_t tid = a.t[t].table_id, dim = a.t[t].dim;
                for (int k = 0; k < 4; k++) h[4 + k] = (uint8_t)(tid >> (8 * k));
                for (int k = 0; k < 8; k++) h[8 + k] = (uint8_t)((uint64_t)n >> (8 * k));
                for (int k = 0; k < 4; k++) h[16 + k] = (uint8_t)(dim >> (8 * k));
                h[20] = (uint8_t)(a.bitwidth ? a.bitwidth : DS_FP32_TAG);
                h[21] = (uint8_t)(a.bitwidth ? 1 : 0);
                h[22] = (uint8_t)(a.aux ? 1 : 0);
                h[23] = 0;
            }
            off += DS_HEADER_SIZE;
        }
        off += n * (int64_t)a.rec;
        tiles += (n + a.tile_rows - 1) / a.tile_rows;
    }
    a.sched[nt] = tiles;
    a.sec_off[nt] = off;
    if (off > a.capacity) atomicOr(a.flags, DS_FLAG_CAPACITY);
}

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
// the writer
// ---------------------------------------------------------------------------
// MODE 0: fp32 section (payload.py:101), 1: naive ranges (engine.py:163-164),
// 2: greedy ranges (engine.py:166 -> quant.py:160-209).
template <int G, int C, int VEC, int MODE, bool PAD>
__global__ void __launch_bounds__(WT) writer_kernel(const WriterArgs a) {
    using Lay = Layout<G, C, VEC>;
    constexpr int EPL = C * VEC;
    constexpr int RPP = WT / G;  // rows per pass
    extern __shared__ __align__(16) uint8_t smem[];
    const int TR = a.tile_rows;
    const int stage_bytes = ((TR * a.rec + 15) & ~15) + 16;
    uint8_t *stage = smem;
    uint8_t *codes_sh = smem + stage_bytes;                       // RPP * dim bytes
    double *exact_sh = reinterpret_cast<double *>(codes_sh + ((RPP * a.dim + 15) & ~15));

    __shared__ int64_t s_sched[2 * DS_MAX_TABLES + 2];
    __shared__ double s_red[WT / 32];
    const int nt = a.ntables;
    for (int k = threadIdx.x; k < 2 * nt + 1; k += WT) s_sched[k] = a.sched[k];
    __syncthreads();
    if (a.sec_off[nt] > a.capacity) return;  // flagged by the layout kernel

    const int lane = threadIdx.x & 31;
    const int lig = lane & (G - 1);
    const int slot = threadIdx.x / G;
    const int d = a.dim;
    const int L = a.L;
    const int64_t total_tiles = s_sched[nt];
    double err_acc = 0.0;
    unsigned n_exact_dec = 0, n_exact_codes = 0, n_rows = 0;
    bool bad_data = false, bad_ids = false;

    for (int64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        int t = 0;
        {
            int lo = 0, hi = nt - 1;
            while (lo < hi) {
                int mid = (lo + hi + 1) >> 1;
                if (s_sched[mid] <= tile) lo = mid;
                else hi = mid - 1;
            }
            t = lo;
        }
        const ds_table_desc &td = a.t[t];
        const int64_t n_t = s_sched[nt + 1 + t];
        const int64_t i0 = (tile - s_sched[t]) * TR;
        const int nrow = (int)min((int64_t)TR, n_t - i0);

        for (int p = 0; p < TR; p += RPP) {
            const int r = p + slot;
            const bool valid = r < nrow;
            if (!__any_sync(DS_FULL_MASK, valid)) continue;
            const int64_t i = i0 + r;
            int64_t gid = 0, local = 0;
            if (valid) {
                if (a.incremental) {
                    gid = __ldg(a.ids + td.ids_off + i);
                    local = gid - td.row_base;
                    if (local < 0 || local >= td.rows) {
                        bad_ids = true;
                        local = 0;
                    }
                } else {
                    local = i;
                    gid = td.row_base + i;
                }
            }
            float x[EPL];
            const float *row = td.values + local * td.ld;
            if (valid) load_row<G, C, VEC>(row, d, lig, x, 0.f);
            else
#pragma unroll
                for (int k = 0; k < EPL; k++) x[k] = 0.f;

            uint8_t *rec = stage + r * a.rec;
            if (valid && a.incremental && lig == 0) st_bytes(rec, (uint64_t)gid, 8);

            if (MODE == 0) {
                if (valid) {
#pragma unroll
                    for (int k = 0; k < EPL; k++) {
                        int e = Lay::elem(lig, k);
                        if (e < d) st_u32(rec + a.par_off + 4 * e, __float_as_uint(x[k]));
                    }
                }
            } else {
                // finiteness (quant.py:70-72,173); padding lanes hold 0
                bool fin = true;
#pragma unroll
                for (int k = 0; k < EPL; k++) fin = fin && isfinite(x[k]);
                fin = grp_or<G>(fin ? 0 : 1) == 0;
                if (valid && !fin) bad_data = true;
                bool row_ok = valid && fin;
                // naive range: row min / max (engine.py:163-164)
                float mn = INFINITY, mx = -INFINITY;
#pragma unroll
                for (int k = 0; k < EPL; k++) {
                    if (Lay::elem(lig, k) < d) {
                        mn = fminf(mn, x[k]);
                        mx = fmaxf(mx, x[k]);
                    }
                }
                float lo = grp_min<G>(mn), hi = grp_max<G>(mx);
                if (!row_ok) { lo = 0.f; hi = 0.f; }
                if (MODE == 2) {
                    double *buf = exact_sh + slot * (d + 8);
                    greedy_row<G, C, VEC, PAD>(x, d, lig, row_ok, lo, hi, L, a.bins, a.steps, buf,
                                               lo, hi, n_exact_dec, n_exact_codes);
                }
                RowQ rq = make_rowq(lo, hi, L);
                int q[EPL];
                double sse = 0.0;
#pragma unroll
                for (int k = 0; k < EPL; k++) {
                    int e = Lay::elem(lig, k);
                    q[k] = 0;
                    if (row_ok && e < d) {
                        q[k] = code_of(x[k], rq, n_exact_codes);
                        float dq = deq_exact(q[k], lo, rq.s);
                        double er = __dsub_rn((double)x[k], (double)dq);
                        sse = fma(er, er, sse);
                    }
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

__global__ void err_reduce_kernel(const double *partials, int n, double *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < n; i++) s += partials[i];
        *out = s;
    }
}

// ---------------------------------------------------------------------------
// host dispatch
// ---------------------------------------------------------------------------
typedef void (*writer_fn)(const WriterArgs);

struct Cfg {
    int G, C, VEC;
};

static Cfg pick_cfg(int d, bool vec4) {
    Cfg c;
    if (vec4) {
        int chunks = d / 4;
        c.VEC = 4;
        c.G = 1;
        while (c.G < chunks && c.G < 32) c.G <<= 1;
        c.C = (chunks + c.G - 1) / c.G;
        int cc = 1;
        while (cc < c.C) cc <<= 1;
        c.C = cc;
    } else {
        c.VEC = 1;
        c.G = 1;
        while (c.G < d && c.G < 32) c.G <<= 1;
        c.C = (d + c.G - 1) / c.G;
        int cc = 1;
        while (cc < c.C) cc <<= 1;
        c.C = cc;
    }
    return c;
}

template <int MODE, bool PAD>
static writer_fn select_writer(const Cfg &c) {
#define DS_W(G_, C_, V_) \
    if (c.G == G_ && c.C == C_ && c.VEC == V_) return writer_kernel<G_, C_, V_, MODE, PAD>;
    DS_W(1, 1, 4) DS_W(2, 1, 4) DS_W(4, 1, 4) DS_W(8, 1, 4) DS_W(16, 1, 4) DS_W(32, 1, 4)
    DS_W(32, 2, 4) DS_W(32, 4, 4) DS_W(32, 8, 4)
    DS_W(1, 1, 1) DS_W(2, 1, 1) DS_W(4, 1, 1) DS_W(8, 1, 1) DS_W(16, 1, 1) DS_W(32, 1, 1)
    DS_W(32, 2, 1) DS_W(32, 4, 1) DS_W(32, 8, 1) DS_W(32, 16, 1) DS_W(32, 32, 1)
#undef DS_W
    return nullptr;
}

}  // namespace ds

using namespace ds;

extern "C" int64_t ds_record_size(int64_t dim, int bitwidth, int aux, int incremental) {
    int64_t s = incremental ? 8 : 0;
    if (bitwidth > 0) s += 8 + (dim * bitwidth + 7) / 8;
    else s += dim * 4;
    if (aux) s += dim * 4;
    return s;
}

extern "C" size_t ds_writer_workspace_size(int ntables, int64_t max_rows) {
    (void)max_rows;
    return (size_t)(2 * DS_MAX_TABLES + 4) * sizeof(int64_t) + (size_t)4096 * sizeof(double) + 256;
}

extern "C" int ds_write_payload(const ds_table_desc *tables_host, int ntables,
                                const ds_ckpt_params *p, const int64_t *ids,
                                const int64_t *counts, uint8_t *payload, int64_t capacity,
                                int64_t *sec_off, double *err_sum, uint32_t *flags,
                                void *workspace, size_t workspace_bytes, void *stream) {
    if (ntables < 1 || ntables > DS_MAX_TABLES)
        return host::fail(DS_ERR_ARG, "ds_write_payload: ntables out of range (1..64)");
    if (!p || !tables_host || !sec_off || !flags || !workspace || !payload)
        return host::fail(DS_ERR_ARG, "ds_write_payload: null pointer");
    if (workspace_bytes < ds_writer_workspace_size(ntables, 0))
        return host::fail(DS_ERR_ARG, "ds_write_payload: workspace too small");
    const int bw = p->bitwidth;
    if (!(bw == 0 || bw == 2 || bw == 3 || bw == 4 || bw == 8))
        return host::fail(DS_ERR_CONFIG, "bitwidth must be one of (2, 3, 4, 8) or 0 (fp32)");
    if (p->incremental && (!ids || !counts))
        return host::fail(DS_ERR_ARG, "ds_write_payload: incremental needs ids and counts");
    WriterArgs a;
    a.ntables = ntables;
    int d = (int)tables_host[0].dim;
    bool vec4 = d % 4 == 0;
    for (int t = 0; t < ntables; t++) {
        a.t[t] = tables_host[t];
        if ((int)tables_host[t].dim != d)
            return host::fail(DS_ERR_SHAPE, "ds_write_payload: tables of one call must share dim");
        if (!tables_host[t].values) return host::fail(DS_ERR_ARG, "ds_write_payload: null values");
        if (p->aux && !tables_host[t].aux) return host::fail(DS_ERR_ARG, "ds_write_payload: null aux");
        if (tables_host[t].ld % 4 || (reinterpret_cast<uintptr_t>(tables_host[t].values) & 15) ||
            (p->aux && (reinterpret_cast<uintptr_t>(tables_host[t].aux) & 15)))
            vec4 = false;
    }
    if (d < 1 || d > 1024)
        return host::fail(DS_ERR_CONFIG, "ds_write_payload: dim must be in 1..1024");
    a.bitwidth = bw;
    a.L = bw ? (1 << bw) - 1 : 0;
    a.incremental = p->incremental;
    a.bins = p->adaptive_bins;
    a.steps = p->adaptive_steps;
    a.aux = p->aux;
    a.write_headers = p->write_headers;
    a.dim = d;
    a.rec = (int)ds_record_size(d, bw, p->aux, p->incremental);
    a.par_off = p->incremental ? 8 : 0;
    a.code_off = a.par_off + 8;
    a.packed = bw ? (d * bw + 7) / 8 : 0;
    a.aux_off = bw ? a.code_off + a.packed : a.par_off + 4 * d;
    a.ids = ids;
    a.counts = p->incremental ? counts : nullptr;
    a.sched = reinterpret_cast<int64_t *>(workspace);
    a.partials = reinterpret_cast<double *>(a.sched + 2 * DS_MAX_TABLES + 4);
    a.sec_off = sec_off;
    a.payload = payload;
    a.capacity = capacity;
    a.flags = flags;
    a.stats = p->stats;

    Cfg c = pick_cfg(d, vec4);
    const int mode = bw == 0 ? 0 : (p->adaptive_bins > 0 ? 2 : 1);
    const bool pad = (c.VEC == 4 ? 4 * c.G * c.C : c.G * c.C) != d;
    writer_fn fn = nullptr;
    if (mode == 0) fn = select_writer<0, false>(c);
    else if (mode == 1) fn = select_writer<1, false>(c);
    else fn = pad ? select_writer<2, true>(c) : select_writer<2, false>(c);
    if (!fn) return host::fail(DS_ERR_CONFIG, "ds_write_payload: no kernel for this dim");

    const int rpp = WT / c.G;
    const int epl = c.C * c.VEC;
    int passes = mode == 2 ? 1 : (epl >= 16 ? 1 : (epl >= 8 ? 2 : 4));
    int tr = rpp * passes;
    // keep the stage within 48 KB
    while (tr > rpp && (int64_t)tr * a.rec > 48 * 1024) tr -= rpp;
    a.tile_rows = tr;
    size_t stage_bytes = (((size_t)tr * a.rec + 15) & ~(size_t)15) + 16;
    size_t codes_bytes = ((size_t)rpp * d + 15) & ~(size_t)15;
    size_t exact_bytes = mode == 2 ? (size_t)rpp * (d + 8) * sizeof(double) : 0;
    size_t smem = stage_bytes + codes_bytes + exact_bytes;
    if (smem > 200 * 1024) return host::fail(DS_ERR_CONFIG, "ds_write_payload: record too large");

    // grid: persistent over an upper bound of the tile count
    int64_t max_tiles = 0;
    for (int t = 0; t < ntables; t++) {
        // incremental counts live on the device; bound by table rows
        max_tiles += (tables_host[t].rows + tr - 1) / tr;
    }
    int per_sm = mode == 2 ? 4 : 8;
    int64_t grid = max_tiles < (int64_t)host::sm_count() * per_sm ? max_tiles
                                                                 : (int64_t)host::sm_count() * per_sm;
    if (grid < 1) grid = 1;
    if (grid > 4096) grid = 4096;

    cudaStream_t s = (cudaStream_t)stream;
    layout_kernel<<<1, 32, 0, s>>>(a);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
    fn<<<(unsigned)grid, WT, smem, s>>>(a);
    int st = host::check_launch("ds_write_payload");
    if (st) return st;
    if (err_sum) err_reduce_kernel<<<1, 32, 0, s>>>(a.partials, (int)grid, err_sum);
    return host::check_launch("ds_write_payload(err)");
}
