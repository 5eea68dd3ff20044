// ds_writer.cu -- K3 host side: launch configuration and the C ABI entry.
//
// The writer kernel itself is ds_writer.cuh (instantiated per mode in
// ds_writer_m0.cu / ds_writer_m1.cu / ds_writer_m2.cu).
#include "ds_writer.cuh"

namespace ds {

// MODE 0/1 writer tiles: 32 records, fewer for huge records (keeping at
// least ns-1 chunks of 32/G rows per tile); then fewer warps per CTA
struct WarpPlan {
    int tr, threads;
    size_t smem;
};
static WarpPlan warp_plan(int d, int64_t rec, const Cfg &c, int mode = 1) {
    const int rpc = 32 / c.G;
    const int ns = mode == 2 ? DS_WRITER_NS_GREEDY : (c.G == 1 ? DS_WRITER_NS1 : DS_WRITER_NS);
    auto warp_bytes = [&](int trr) {
        return (size_t)align16((int)(trr * rec)) + 16 + align16(rpc * d) +
               (size_t)ns * ((rpc * d * 4 + 63) & ~63) +
               (mode == 2 ? (size_t)align16(rpc * greedy_scratch_bytes(c.G * c.C * c.VEC, d)) : 0);
    };
    WarpPlan p;
    p.tr = 32;
    const int wt = mode == 2 ? DS_WT_GREEDY : DS_WT_WARP;
    while (warp_bytes(p.tr) * (wt / 32) > 200 * 1024 && p.tr / 2 >= rpc * (ns - 1) && p.tr > 1)
        p.tr /= 2;
    p.threads = wt;
    while (warp_bytes(p.tr) * (p.threads / 32) > 200 * 1024 && p.threads > 32) p.threads /= 2;
    p.smem = warp_bytes(p.tr) * (p.threads / 32) + 16;  // + alignment slack
    return p;
}

// tiles of the MODE 0/1 writer for `rows` records of dim `dim` (any record
// layout of that dim: sized with the largest, fp32 + aux + row ids)
static int64_t warp_tiles(int64_t rows, int ntables, int64_t dim) {
    int tr = 32;
    for (int v = 0; v < 2; v++) {  // float4 or scalar layout, whichever the call picks
        if (v == 1 && dim % 4) continue;
        for (int m = 1; m <= 2; m++) {
            const WarpPlan p = warp_plan((int)dim, 8 + 8 * dim, pick_cfg((int)dim, v == 1, m), m);
            tr = p.tr < tr ? p.tr : tr;
        }
    }
    return rows / tr + ntables + 1;
}

// ---------------------------------------------------------------------------
// stall-window staging: staged[k] = values_t[ids[k]] for the packed ids
// ---------------------------------------------------------------------------
struct StageArgs {
    ds_table_desc t[DS_MAX_TABLES];
    const int64_t *ids;
    const int64_t *counts;
    float *staged;
    uint32_t *flags;
    int64_t max_rows;
    int ntables, dim, vec;
};

__global__ void __launch_bounds__(256) stage_rows_kernel(const StageArgs a) {
    __shared__ int64_t s_off[DS_MAX_TABLES + 1];
    const int nt = a.ntables;
    if (threadIdx.x < 32) {  // packed id offsets: one warp scan over the counts
        const int lane = threadIdx.x;
        int64_t base = 0;
        for (int b = 0; b < nt; b += 32) {
            const int64_t n = b + lane < nt ? a.counts[b + lane] : 0;
            int64_t x = n;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(DS_FULL_MASK, x, o);
                if (lane >= o) x += y;
            }
            if (b + lane < nt) s_off[b + lane] = base + x - n;
            base += __shfl_sync(DS_FULL_MASK, x, 31);
        }
        if (lane == 0) s_off[nt] = base;
    }
    __syncthreads();
    int64_t total = s_off[nt];
    if (total > a.max_rows) {  // the staging buffer is too small: flagged, capped
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(a.flags, DS_FLAG_CAPACITY);
        total = a.max_rows;
    }
    const int d = a.dim;
    // lanes per row: one float4 each (or one float) up to a warp
    const int per = a.vec ? (d >> 2) : d;
    const int gl = per >= 32 ? 32 : (per >= 16 ? 16 : (per >= 8 ? 8 : (per >= 4 ? 4 : (per >= 2 ? 2 : 1))));
    const int lane = threadIdx.x & 31, lig = lane % gl;
    const int64_t rows_per_step = ((int64_t)gridDim.x * blockDim.x) / gl;
    bool bad = false;
    constexpr int U = 4;  // rows in flight per lane group
    for (int64_t k0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / gl; k0 < total;
         k0 += U * rows_per_step) {
        const float *src[U];
        int64_t kk[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t k = k0 + u * rows_per_step;
            kk[u] = k;
            src[u] = nullptr;
            if (k < total) {
                int lo = 0, hi = nt - 1;  // table of packed position k
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (s_off[mid] <= k) lo = mid;
                    else hi = mid - 1;
                }
                const ds_table_desc &td = a.t[lo];
                const int64_t id = a.ids[k];
                if (id < 0 || id >= td.rows) bad = true;
                else src[u] = td.values + id * td.ld;
            }
        }
        if (a.vec) {
            for (int c = lig; c < per; c += gl) {
                float4 v[U];
#pragma unroll
                for (int u = 0; u < U; u++)
                    if (src[u]) v[u] = __ldg(reinterpret_cast<const float4 *>(src[u]) + c);
#pragma unroll
                for (int u = 0; u < U; u++)
                    if (src[u]) __stcs(reinterpret_cast<float4 *>(a.staged + kk[u] * (int64_t)d) + c, v[u]);
            }
        } else {
#pragma unroll
            for (int u = 0; u < U; u++)
                if (src[u])
                    for (int e = lig; e < d; e += gl) a.staged[kk[u] * (int64_t)d + e] = __ldg(src[u] + e);
        }
    }
    if (__any_sync(DS_FULL_MASK, bad) && (threadIdx.x & 31) == 0) atomicOr(a.flags, DS_FLAG_BOUNDS);
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

// workspace: [done counter, 16 B] [4096 error partials] [fixup masks]
static size_t ws_head_bytes() { return 16 + (size_t)4096 * sizeof(double); }

extern "C" size_t ds_writer_workspace_size(int ntables, int64_t max_rows, int64_t dim) {
    // done counter + 4096 error partials + one fixup mask word per warp-tile
    int64_t tiles = warp_tiles(max_rows > 0 ? max_rows : 0, ntables, dim > 0 ? dim : 1);
    return ws_head_bytes() + (size_t)tiles * sizeof(uint32_t) + 256;
}

static int mode_of(const ds_ckpt_params *p) {
    return p->bitwidth == 0 ? 0 : (p->adaptive_bins > 0 ? 2 : 1);
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
    int64_t rows_bound = 0;
    for (int t = 0; t < ntables; t++) rows_bound += tables_host[t].rows;
    if (workspace_bytes < ds_writer_workspace_size(ntables, rows_bound, tables_host[0].dim))
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
    a.invL = bw ? 1.0 / (double)a.L : 0.0;
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
    a.done = reinterpret_cast<unsigned *>(workspace);
    a.partials = reinterpret_cast<double *>(static_cast<uint8_t *>(workspace) + 16);
    a.fix_mask = reinterpret_cast<uint32_t *>(a.partials + 4096);
    a.err_out = err_sum;
    a.ids_packed = p->ids_packed;
    a.ids_local = p->ids_local;
    a.sec_off = sec_off;
    a.payload = payload;
    a.capacity = capacity;
    a.flags = flags;
    a.stats = p->stats;
    a.staged = p->staged;
    a.staged_rows = p->staged ? p->staged_rows : 0;
    if (p->staged && (!p->incremental || !p->ids_packed || p->aux || (mode_of(p) == 2 && DS_GREEDY_CTA)))
        return host::fail(DS_ERR_ARG, "ds_write_payload: staged rows need an incremental "
                                      "checkpoint with packed ids and no aux");
    if (p->staged && p->staged_rows < 0)
        return host::fail(DS_ERR_ARG, "ds_write_payload: negative staged_rows");

    a.has_x = p->exchange != nullptr;
    if (a.has_x) {
        const ds_peer_exchange &x = *p->exchange;
        if (x.world < 1 || x.world > DS_PEER_MAX || x.rank < 0 || x.rank >= x.world || x.epoch == 0 ||
            !x.out || !x.flags)
            return host::fail(DS_ERR_ARG, "ds_write_payload: bad count exchange");
        for (int r = 0; r < x.world; r++)
            if (!x.peers[r]) return host::fail(DS_ERR_ARG, "ds_write_payload: null peer buffer");
        a.x = x;
    }

    const int mode = bw == 0 ? 0 : (p->adaptive_bins > 0 ? 2 : 1);
    Cfg c = pick_cfg(d, vec4, mode);
    const bool pad = (c.VEC == 4 ? 4 * c.G * c.C : c.G * c.C) != d;
    writer_fn fn = nullptr;
    if (mode == 0) fn = select_writer_mode0(c, pad);
    else if (mode == 1) fn = select_writer_mode1(c, pad);
    else fn = select_writer_mode2(c, pad);
    if (!fn) return host::fail(DS_ERR_CONFIG, "ds_write_payload: no kernel for this dim");

    int tr;
    int threads = WT;
    size_t smem;
    // wide rows at 2/4/8 bits with naive ranges: one row per lane group
    // (ds_writer_row.cuh); DS_ROW_G=0 keeps the warp-pipelined writer
    // (A/B r02, T shard: 7.07 ms at G = 4 vs 6.95 ms for the warp-pipelined
    // writer with fused packing: off by default, DS_ROW_G=4 selects it)
    static const int row_g = (int)host::env_int("DS_ROW_G", 0);
    bool row_kernel = false;
    if (mode == 1 && c.VEC == 4 && vec4 && !p->aux && a.rec % 8 == 0 && row_g > 0 &&
        (bw == 8 || bw == 4 || bw == 2)) {
        writer_fn rf = select_writer_row(d, row_g, bw);
        if (rf) {
            fn = rf;
            row_kernel = true;
        }
    }
    if (row_kernel) {
        tr = 32 / row_g;
        threads = 32;
        smem = row_writer_smem_bytes(d, row_g, a.rec);
    } else if (mode != 2 || !DS_GREEDY_CTA) {
        // warp pipeline: tiles of 32 records, per-warp record stage + codes
        // scratch + a ring of NS row chunks of 32/G rows (+ the greedy exact
        // scratch; writer_warp_kernel computes the same layout)
        const WarpPlan wp = warp_plan(d, a.rec, c, mode);
        tr = wp.tr;
        threads = wp.threads;
        smem = wp.smem;
    } else {
        const int rpp = WT / c.G;  // one pass of rows per tile (compute-bound)
        tr = rpp;
        smem = (size_t)align16(tr * a.rec) + 16 + align16(rpp * d) +
               (size_t)rpp * greedy_scratch_bytes(c.G * c.C * c.VEC, d);
    }
    a.tile_rows = tr;
    if (smem > 200 * 1024) return host::fail(DS_ERR_CONFIG, "ds_write_payload: record too large");

    // grid: persistent over an upper bound of the tile count
    int64_t max_tiles = 0;
    for (int t = 0; t < ntables; t++) {
        // incremental counts live on the device; bound by table rows
        max_tiles += (tables_host[t].rows + tr - 1) / tr;
    }
    if (!row_kernel && (mode != 2 || !DS_GREEDY_CTA))
        max_tiles = (max_tiles + threads / 32 - 1) / (threads / 32);  // warps -> CTAs
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
    if (per_sm < 1) per_sm = 1;
    int64_t grid = max_tiles < (int64_t)host::sm_count() * per_sm ? max_tiles
                                                                 : (int64_t)host::sm_count() * per_sm;
    if (grid < 1) grid = 1;
    if (grid > 4096) grid = 4096;

    // one launch: layout, records, exact fixups and the error sum
    e = host::launch_pdl(fn, (unsigned)grid, (unsigned)threads, smem, (cudaStream_t)stream, a);
    if (e != cudaSuccess) return host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
    return host::check_launch("ds_write_payload");
}

extern "C" int ds_stage_rows(const ds_table_desc *tables_host, int ntables, const int64_t *ids,
                             const int64_t *counts, int64_t max_rows, float *staged, uint32_t *flags,
                             void *stream) {
    if (ntables < 1 || ntables > DS_MAX_TABLES) return host::fail(DS_ERR_ARG, "ds_stage_rows: ntables");
    if (!tables_host || !counts || !flags) return host::fail(DS_ERR_ARG, "ds_stage_rows: null pointer");
    if (max_rows <= 0) return DS_OK;
    if (!ids || !staged) return host::fail(DS_ERR_ARG, "ds_stage_rows: null ids / staged");
    StageArgs a;
    a.ntables = ntables;
    a.ids = ids;
    a.counts = counts;
    a.staged = staged;
    a.flags = flags;
    a.max_rows = max_rows;
    a.dim = (int)tables_host[0].dim;
    a.vec = a.dim % 4 == 0 && (reinterpret_cast<uintptr_t>(staged) & 15) == 0;
    for (int t = 0; t < ntables; t++) {
        if ((int)tables_host[t].dim != a.dim)
            return host::fail(DS_ERR_SHAPE, "ds_stage_rows: tables of one call share dim");
        a.t[t] = tables_host[t];
        if (tables_host[t].ld % 4 || (reinterpret_cast<uintptr_t>(tables_host[t].values) & 15)) a.vec = 0;
    }
    const int per = a.vec ? a.dim / 4 : a.dim;
    const int gl = per >= 32 ? 32 : (per >= 16 ? 16 : (per >= 8 ? 8 : (per >= 4 ? 4 : (per >= 2 ? 2 : 1))));
    int64_t blocks = (max_rows * gl + 255) / 256;
    const int64_t cap = (int64_t)host::sm_count() * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    stage_rows_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(a);
    return host::check_launch("ds_stage_rows");
}
