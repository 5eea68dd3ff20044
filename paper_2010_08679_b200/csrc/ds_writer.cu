// ds_writer.cu -- K3 host side: layout kernel, error reduction, C ABI entry.
//
// The writer kernel itself is ds_writer.cuh (instantiated per mode in
// ds_writer_m0.cu / ds_writer_m1.cu / ds_writer_m2.cu).
#include "ds_writer.cuh"

namespace ds {

// ---------------------------------------------------------------------------
// layout: section offsets, headers (payload.py:88-91), tile schedule
// ---------------------------------------------------------------------------
__global__ void layout_kernel(const WriterArgs a) {
    if (threadIdx.x != 0) return;
    int64_t off = 0, tiles = 0, ids = 0;
    int nt = a.ntables;
    for (int t = 0; t < nt; t++) {
        int64_t n = a.counts ? a.counts[t] : a.t[t].rows;
        a.sched[t] = tiles;
        a.sched[nt + 1 + t] = n;
        a.sched[2 * nt + 1 + t] = a.ids_packed ? ids : a.t[t].ids_off;
        ids += n;
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

__global__ void err_reduce_kernel(const double *partials, int n, double *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < n; i++) s += partials[i];
        *out = s;
    }
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
    return (size_t)(3 * DS_MAX_TABLES + 4) * sizeof(int64_t) + (size_t)4096 * sizeof(double) + 256;
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
    a.sched = reinterpret_cast<int64_t *>(workspace);
    a.partials = reinterpret_cast<double *>(a.sched + 3 * DS_MAX_TABLES + 4);
    a.ids_packed = p->ids_packed;
    a.ids_local = p->ids_local;
    a.sec_off = sec_off;
    a.payload = payload;
    a.capacity = capacity;
    a.flags = flags;
    a.stats = p->stats;

    Cfg c = pick_cfg(d, vec4);
    const int mode = bw == 0 ? 0 : (p->adaptive_bins > 0 ? 2 : 1);
    const bool pad = (c.VEC == 4 ? 4 * c.G * c.C : c.G * c.C) != d;
    writer_fn fn = nullptr;
    if (mode == 0) fn = select_writer_mode0(c, pad);
    else if (mode == 1) fn = select_writer_mode1(c, pad);
    else fn = select_writer_mode2(c, pad);
    if (!fn) return host::fail(DS_ERR_CONFIG, "ds_write_payload: no kernel for this dim");

    const int rpp = WT / c.G;
    // MODE 0/1: a tile is ~32 KB of gathered rows (a multiple of the rows per
    // pass); MODE 2: one pass per tile (compute-bound)
    int tr = rpp;
    if (mode != 2) {
        tr = (int)((16 * 1024) / ((int64_t)d * 4));  // 16 KB of rows per buffer (x2)
        tr = tr / rpp * rpp;
        if (tr < rpp) tr = rpp;
        if (tr > 1024) tr = 1024;
    }
    // keep the record stage within 48 KB
    while (tr > rpp && (int64_t)tr * a.rec > 48 * 1024) tr -= rpp;
    a.tile_rows = tr;
    size_t stage_bytes = (((size_t)tr * a.rec + 15) & ~(size_t)15) + 16;
    size_t codes_bytes = ((size_t)rpp * d + 15) & ~(size_t)15;
    size_t tail_bytes = mode == 2 ? (size_t)rpp * (d + 8) * sizeof(double)
                                  : 2 * (((size_t)tr * d * 4 + 15) & ~(size_t)15) + 3 * (size_t)tr * 8;
    size_t smem = stage_bytes + codes_bytes + tail_bytes;
    if (smem > 200 * 1024) return host::fail(DS_ERR_CONFIG, "ds_write_payload: record too large");

    // grid: persistent over an upper bound of the tile count
    int64_t max_tiles = 0;
    for (int t = 0; t < ntables; t++) {
        // incremental counts live on the device; bound by table rows
        max_tiles += (tables_host[t].rows + tr - 1) / tr;
    }
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, WT, smem);
    if (per_sm < 1) per_sm = 1;
    int64_t grid = max_tiles < (int64_t)host::sm_count() * per_sm ? max_tiles
                                                                 : (int64_t)host::sm_count() * per_sm;
    if (grid < 1) grid = 1;
    if (grid > 4096) grid = 4096;

    cudaStream_t s = (cudaStream_t)stream;
    layout_kernel<<<1, 32, 0, s>>>(a);
    fn<<<(unsigned)grid, WT, smem, s>>>(a);
    int st = host::check_launch("ds_write_payload");
    if (st) return st;
    if (err_sum) err_reduce_kernel<<<1, 32, 0, s>>>(a.partials, (int)grid, err_sum);
    return host::check_launch("ds_write_payload(err)");
}
