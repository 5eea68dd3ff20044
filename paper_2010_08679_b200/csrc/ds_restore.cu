// ds_restore.cu -- K4: unpack + dequantize + scatter of one CNR1 section body.
//
// Replaces the _restore_at apply loop (deltasnap/engine.py:459-485):
// parse_shard_payload's column split (payload.py:142-162), decode_values
// (payload.py:60-65 -> unpack_code_rows quant.py:385-395 + dequantize_rows
// quant.py:109-115), `table.values[idx] = values` and mark_baseline (:476).
// Section headers are parsed and validated on the host (payload.py:116-137).
#include <cuda_runtime.h>
#include <stdint.h>

#include "ds_common.cuh"
#include "ds_host.h"

namespace ds {

constexpr int RT = 256;

struct RestoreArgs {
    const uint8_t *body;
    int64_t rec_begin, rec_end;  // records to visit
    int64_t table_rows;
    int64_t row_lo, row_hi;      // rows held by this table (global ids)
    float *values;
    float *aux_values;
    uint32_t *baseline;
    uint32_t *flags;
    int64_t ld;
    int dim, bitwidth, L, aux, incremental;
    int rec, par_off, code_off, packed, aux_off;
    int tile_rows;
    double invL;
};

__device__ __forceinline__ uint32_t ld4_unaligned_g(const uint8_t *p) {
    uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uint32_t *w = reinterpret_cast<const uint32_t *>(a & ~(uintptr_t)3);
    int sh = (int)(a & 3) * 8;
    uint32_t lo = __ldg(w);
    if (sh == 0) return lo;
    return __funnelshift_r(lo, __ldg(w + 1), sh);
}

template <int G>
__global__ void __launch_bounds__(RT) restore_kernel(const RestoreArgs a) {
    extern __shared__ __align__(16) uint8_t stage[];
    constexpr int RPP = RT / G;
    const int lane = threadIdx.x & 31, lig = lane & (G - 1), slot = threadIdx.x / G;
    const int d = a.dim, TR = a.tile_rows;
    const int64_t nrec = a.rec_end - a.rec_begin;
    const int64_t ntiles = (nrec + TR - 1) / TR;
    bool bad_fmt = false, bad_row = false;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t r0 = a.rec_begin + tile * TR;
        const int nr = (int)min((int64_t)TR, a.rec_end - r0);
        // stage the tile's bytes with aligned 32-bit loads (the source is a
        // contiguous run of records at any byte alignment)
        const uint8_t *src = a.body + r0 * a.rec;
        const int nbytes = nr * a.rec;
        const int nw = (nbytes + 3) >> 2;
        // the last word may read up to 3 bytes past the run: bounded by the
        // host, which keeps 16 bytes of slack after every staged payload
        for (int k = threadIdx.x; k < nw; k += RT)
            reinterpret_cast<uint32_t *>(stage)[k] = ld4_unaligned_g(src + 4 * k);
        __syncthreads();
        for (int p = 0; p < TR; p += RPP) {
            const int r = p + slot;
            if (r >= nr) continue;
            const uint8_t *rec = stage + r * a.rec;
            int64_t gid;
            if (a.incremental) {
                uint64_t u = 0;
                for (int k = 0; k < 8; k++) u |= (uint64_t)rec[k] << (8 * k);
                gid = (int64_t)u;
                if (gid < 0 || gid >= a.table_rows) {  // engine.py:470-472
                    bad_row = true;
                    continue;
                }
            } else {
                gid = r0 + r;
            }
            if (gid < a.row_lo || gid >= a.row_hi) continue;  // another rank's rows
            const int64_t local = gid - a.row_lo;
            float *dst = a.values + local * a.ld;
            if (a.bitwidth == 0) {
                for (int e = lig; e < d; e += G) {
                    uint32_t u = rec[a.par_off + 4 * e] | (rec[a.par_off + 4 * e + 1] << 8) |
                                 (rec[a.par_off + 4 * e + 2] << 16) |
                                 ((uint32_t)rec[a.par_off + 4 * e + 3] << 24);
                    dst[e] = __uint_as_float(u);
                }
            } else {
                uint32_t ulo = 0, uhi = 0;
                for (int k = 0; k < 4; k++) {
                    ulo |= (uint32_t)rec[a.par_off + k] << (8 * k);
                    uhi |= (uint32_t)rec[a.par_off + 4 + k] << (8 * k);
                }
                const float lo = __uint_as_float(ulo), hi = __uint_as_float(uhi);
                const double s = scale64_y(lo, hi, (double)a.L, a.invL);
                const uint8_t *pk = rec + a.code_off;
                const int N = a.bitwidth;
                for (int e = lig; e < d; e += G) {
                    int bit = e * N;
                    uint32_t w = pk[bit >> 3] | ((uint32_t)pk[(bit >> 3) + 1] << 8);
                    int q = (int)((w >> (bit & 7)) & (uint32_t)a.L);
                    dst[e] = deq_exact(q, lo, s);
                }
                // padding bits must be zero (quant.py:390-392)
                if (lig == 0) {
                    int padbits = 8 * a.packed - d * N;
                    if (padbits > 0 && (pk[a.packed - 1] >> (8 - padbits)) != 0) bad_fmt = true;
                }
            }
            if (a.aux && a.aux_values) {
                float *adst = a.aux_values + local * a.ld;
                for (int e = lig; e < d; e += G) {
                    const uint8_t *q = rec + a.aux_off + 4 * e;
                    uint32_t u = q[0] | (q[1] << 8) | (q[2] << 16) | ((uint32_t)q[3] << 24);
                    adst[e] = __uint_as_float(u);
                }
            }
            if (a.incremental && a.baseline && lig == 0)  // mark_baseline, engine.py:476
                atomicOr(a.baseline + (local >> 5), 1u << (local & 31));
        }
        __syncthreads();
    }
    if (bad_fmt) atomicOr(a.flags, DS_FLAG_FORMAT);
    if (bad_row) atomicOr(a.flags, DS_FLAG_INTEGRITY);
}

// ---------------------------------------------------------------------------
// Every section of a payload in one launch: tiles of records across sections,
// staged into shared memory with aligned 32-bit loads; G lanes per record,
// each lane 4 consecutive elements at a time (one 32-bit code read, 4 exact
// dequantizations, one 16-byte store when the table rows allow it).
// ---------------------------------------------------------------------------
struct RestorePArgs {
    const uint8_t *payload;
    ds_restore_sec s[DS_MAX_TABLES];
    int64_t rec_begin[DS_MAX_TABLES], rec_end[DS_MAX_TABLES];
    int64_t tile_off[DS_MAX_TABLES + 1];
    uint32_t *flags;
    int nsec, dim, bitwidth, L, aux, incremental, rec, par_off, code_off, packed, aux_off;
    int tile_rows, vec;
    double invL;
};

__device__ __forceinline__ uint32_t lds32u(const uint8_t *base, int o) {
    const uint32_t *w = reinterpret_cast<const uint32_t *>(base + (o & ~3));
    const int sh = (o & 3) * 8;
    return sh ? __funnelshift_r(w[0], w[1], sh) : w[0];
}

template <int G>
__global__ void __launch_bounds__(RT) restore_payload_kernel(const RestorePArgs a) {
    extern __shared__ __align__(16) uint8_t stage[];
    // chained payloads (PDL): the next one launches into this one's tail and
    // waits here until it is complete (later payloads override earlier rows)
    pdl_trigger();
    pdl_wait();
    constexpr int RPP = RT / G;
    const int lane = threadIdx.x & 31, lig = lane & (G - 1), slot = threadIdx.x / G;
    const int d = a.dim, TR = a.tile_rows, N = a.bitwidth;
    const int64_t ntiles = a.tile_off[a.nsec];
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int sec = 0;  // last section whose first tile <= tile (binary search, uniform)
        for (int lo = 0, hi = a.nsec - 1; lo <= hi;) {
            const int mid = (lo + hi) >> 1;
            if (a.tile_off[mid] <= tile) { sec = mid; lo = mid + 1; }
            else hi = mid - 1;
        }
        const ds_restore_sec &S = a.s[sec];
        const int64_t r0 = a.rec_begin[sec] + (tile - a.tile_off[sec]) * TR;
        const int nr = (int)min((int64_t)TR, a.rec_end[sec] - r0);
        const uint8_t *src = a.payload + S.body_off + r0 * a.rec;
        const int nw = (nr * a.rec + 3) >> 2;
        // the last word may read up to 3 bytes past the run: the host keeps
        // 16 bytes of slack after every staged payload
        for (int k = threadIdx.x; k < nw; k += RT)
            reinterpret_cast<uint32_t *>(stage)[k] = ld4_unaligned_g(src + 4 * k);
        __syncthreads();
        bool bad_fmt = false, bad_row = false;
        for (int p = 0; p < nr; p += RPP) {
            const int r = p + slot;
            if (r >= nr) continue;
            const int ro = r * a.rec;
            int64_t gid = r0 + r;
            if (a.incremental) {
                gid = (int64_t)(((uint64_t)lds32u(stage, ro + 4) << 32) | lds32u(stage, ro));
                if (gid < 0 || gid >= S.table_rows) {  // engine.py:470-472
                    bad_row = true;
                    continue;
                }
            }
            if (gid < S.row_lo || gid >= S.row_hi) continue;  // another rank's rows
            const int64_t local = gid - S.row_lo;
            float *dst = S.values + local * S.ld;
            if (N == 0) {
                for (int e = lig; e < d; e += G) dst[e] = __uint_as_float(lds32u(stage, ro + a.par_off + 4 * e));
            } else {
                const float lo = __uint_as_float(lds32u(stage, ro + a.par_off));
                const float hi = __uint_as_float(lds32u(stage, ro + a.par_off + 4));
                const double s = scale64_y(lo, hi, (double)a.L, a.invL);
                for (int m = lig; 4 * m < d; m += G) {
                    const int bit = 4 * m * N;
                    const uint32_t w = lds32u(stage, ro + a.code_off + (bit >> 3)) >> (bit & 7);
                    float v[4];
#pragma unroll
                    for (int j = 0; j < 4; j++) v[j] = deq_exact((int)((w >> (j * N)) & (uint32_t)a.L), lo, s);
                    if (a.vec && 4 * m + 4 <= d)
                        *reinterpret_cast<float4 *>(dst + 4 * m) = make_float4(v[0], v[1], v[2], v[3]);
                    else
#pragma unroll
                        for (int j = 0; j < 4; j++)
                            if (4 * m + j < d) dst[4 * m + j] = v[j];
                }
                // padding bits must be zero (quant.py:390-392)
                if (lig == 0) {
                    const int padbits = 8 * a.packed - d * N;
                    if (padbits > 0 && (stage[ro + a.code_off + a.packed - 1] >> (8 - padbits)) != 0)
                        bad_fmt = true;
                }
            }
            if (a.aux && S.aux_values) {
                float *adst = S.aux_values + local * S.ld;
                for (int e = lig; e < d; e += G) adst[e] = __uint_as_float(lds32u(stage, ro + a.aux_off + 4 * e));
            }
            if (a.incremental && S.baseline && lig == 0)  // mark_baseline, engine.py:476
                atomicOr(S.baseline + (local >> 5), 1u << (local & 31));
        }
        if (bad_fmt) atomicOr(a.flags + sec, DS_FLAG_FORMAT);
        if (bad_row) atomicOr(a.flags + sec, DS_FLAG_INTEGRITY);
        __syncthreads();
    }
}

}  // namespace ds

using namespace ds;

extern "C" int ds_restore_section(const uint8_t *body, int64_t nrec, int64_t dim, int bitwidth,
                                  int aux, int incremental, int64_t table_rows, int64_t row_lo,
                                  int64_t row_hi, float *values, int64_t ld, float *aux_values,
                                  uint32_t *baseline_words, uint32_t *flags, void *stream) {
    if (!(bitwidth == 0 || bitwidth == 2 || bitwidth == 3 || bitwidth == 4 || bitwidth == 8))
        return host::fail(DS_ERR_FORMAT, "ds_restore_section: invalid bitwidth");
    if (dim < 1 || dim > 65536) return host::fail(DS_ERR_ARG, "ds_restore_section: dim");
    if (!values || !flags) return host::fail(DS_ERR_ARG, "ds_restore_section: null pointer");
    if (nrec <= 0) return DS_OK;
    if (!body) return host::fail(DS_ERR_ARG, "ds_restore_section: null body");
    RestoreArgs a;
    a.body = body;
    a.table_rows = table_rows;
    a.row_lo = row_lo;
    a.row_hi = row_hi;
    a.values = values;
    a.aux_values = aux_values;
    a.baseline = baseline_words;
    a.flags = flags;
    a.ld = ld;
    a.dim = (int)dim;
    a.bitwidth = bitwidth;
    a.L = bitwidth ? (1 << bitwidth) - 1 : 0;
    a.invL = bitwidth ? 1.0 / (double)a.L : 0.0;
    a.aux = aux;
    a.incremental = incremental;
    a.rec = (int)ds_record_size(dim, bitwidth, aux, incremental);
    a.par_off = incremental ? 8 : 0;
    a.code_off = a.par_off + 8;
    a.packed = bitwidth ? (int)((dim * bitwidth + 7) / 8) : 0;
    a.aux_off = bitwidth ? a.code_off + a.packed : a.par_off + 4 * (int)dim;
    if (incremental) {
        a.rec_begin = 0;
        a.rec_end = nrec;
    } else {  // record i is row i: visit only this table's rows
        a.rec_begin = row_lo > 0 ? row_lo : 0;
        a.rec_end = row_hi < nrec ? row_hi : nrec;
        if (a.rec_end <= a.rec_begin) return DS_OK;
    }
    int G = 1;
    while (G < dim && G < 32) G <<= 1;
    int rpp = RT / G;
    int tr = rpp;
    while (tr * 2 * a.rec <= 32 * 1024 && tr < 1024) tr *= 2;
    while (tr > rpp && tr * a.rec > 32 * 1024) tr /= 2;
    a.tile_rows = tr;
    size_t smem = ((size_t)tr * a.rec + 15) / 16 * 16 + 16;
    if (smem > 200 * 1024) return host::fail(DS_ERR_CONFIG, "ds_restore_section: record too large");
    int64_t ntiles = (a.rec_end - a.rec_begin + tr - 1) / tr;
    int64_t grid = ntiles < (int64_t)host::sm_count() * 8 ? ntiles : (int64_t)host::sm_count() * 8;
    cudaStream_t s = (cudaStream_t)stream;
    void (*fn)(const RestoreArgs) = nullptr;
    switch (G) {
        case 1: fn = restore_kernel<1>; break;
        case 2: fn = restore_kernel<2>; break;
        case 4: fn = restore_kernel<4>; break;
        case 8: fn = restore_kernel<8>; break;
        case 16: fn = restore_kernel<16>; break;
        default: fn = restore_kernel<32>; break;
    }
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
    fn<<<(unsigned)grid, RT, smem, s>>>(a);
    return host::check_launch("ds_restore_section");
}

extern "C" int ds_restore_payload(const uint8_t *payload, const ds_restore_sec *secs, int nsec,
                                  int64_t dim, int bitwidth, int aux, int incremental,
                                  uint32_t *flags, void *stream) {
    if (!(bitwidth == 0 || bitwidth == 2 || bitwidth == 3 || bitwidth == 4 || bitwidth == 8))
        return host::fail(DS_ERR_FORMAT, "ds_restore_payload: invalid bitwidth");
    if (nsec < 1 || nsec > DS_MAX_TABLES) return host::fail(DS_ERR_ARG, "ds_restore_payload: nsec (1..64)");
    if (dim < 1 || dim > 65536) return host::fail(DS_ERR_ARG, "ds_restore_payload: dim");
    if (!payload || !secs || !flags) return host::fail(DS_ERR_ARG, "ds_restore_payload: null pointer");
    RestorePArgs a;
    a.payload = payload;
    a.flags = flags;
    a.nsec = nsec;
    a.dim = (int)dim;
    a.bitwidth = bitwidth;
    a.L = bitwidth ? (1 << bitwidth) - 1 : 0;
    a.invL = bitwidth ? 1.0 / (double)a.L : 0.0;
    a.aux = aux;
    a.incremental = incremental;
    a.rec = (int)ds_record_size(dim, bitwidth, aux, incremental);
    a.par_off = incremental ? 8 : 0;
    a.code_off = a.par_off + 8;
    a.packed = bitwidth ? (int)((dim * bitwidth + 7) / 8) : 0;
    a.aux_off = bitwidth ? a.code_off + a.packed : a.par_off + 4 * (int)dim;
    // lanes per record: one per 4-element group, up to a warp
    int G = 1;
    while (G * 4 < dim && G < 32) G <<= 1;
    const int rpp = RT / G;
    int tr = rpp;
    while (tr * 2 * a.rec <= 32 * 1024 && tr < 1024) tr *= 2;
    while (tr > rpp && tr * a.rec > 32 * 1024) tr /= 2;
    a.tile_rows = tr;
    a.vec = 1;
    int64_t tiles = 0;
    for (int k = 0; k < nsec; k++) {
        a.s[k] = secs[k];
        if (!secs[k].values) return host::fail(DS_ERR_ARG, "ds_restore_payload: null values");
        if (secs[k].ld % 4 || reinterpret_cast<uintptr_t>(secs[k].values) % 16) a.vec = 0;
        int64_t b = 0, e = secs[k].nrec;
        if (!incremental) {  // record i is row i: visit only this table's rows
            b = secs[k].row_lo > 0 ? secs[k].row_lo : 0;
            e = secs[k].row_hi < e ? secs[k].row_hi : e;
            if (e < b) e = b;
        }
        a.rec_begin[k] = b;
        a.rec_end[k] = e;
        a.tile_off[k] = tiles;
        tiles += (e - b + tr - 1) / tr;
    }
    a.tile_off[nsec] = tiles;
    if (tiles == 0) return DS_OK;
    size_t smem = ((size_t)tr * a.rec + 15) / 16 * 16 + 16;
    if (smem > 200 * 1024) return host::fail(DS_ERR_CONFIG, "ds_restore_payload: record too large");
    void (*fn)(const RestorePArgs) = nullptr;
    switch (G) {
        case 1: fn = restore_payload_kernel<1>; break;
        case 2: fn = restore_payload_kernel<2>; break;
        case 4: fn = restore_payload_kernel<4>; break;
        case 8: fn = restore_payload_kernel<8>; break;
        case 16: fn = restore_payload_kernel<16>; break;
        default: fn = restore_payload_kernel<32>; break;
    }
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, RT, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t cap = (int64_t)host::sm_count() * per_sm;
    const int64_t grid = tiles < cap ? tiles : cap;
    e = host::launch_pdl(fn, (unsigned)grid, (unsigned)RT, smem, (cudaStream_t)stream, a);
    if (e != cudaSuccess) return host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
    return host::check_launch("ds_restore_payload");
}
