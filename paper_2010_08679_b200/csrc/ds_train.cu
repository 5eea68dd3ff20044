// ds_train.cu -- the synthetic training step with tracking folded in
// (SURVEY.md 8(f) row 1).
//
// Reference: deltasnap/sim.py:140-155 apply_batch: for every table,
// np.add.at(values, idx, delta); np.add.at(aux, idx, delta * delta);
// tracker.mark(tid, idx).  np.add.at applies the updates one index at a time
// in array order, so a row hit twice gets (v + d1) + d2: float addition order
// matters.  Here each table's batch is sorted by (row, position) in shared
// memory (bitonic), every distinct row is then updated by one thread group
// that adds its deltas in the original order -- bit-identical to np.add.at --
// and the same group sets the row's dirty bit (RED.OR), so tracking costs one
// atomic per distinct row and no second pass over the lookups.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ds_common.cuh"
#include "ds_host.h"

namespace ds {

constexpr int TS_THREADS = 1024;
constexpr int TS_MAX = 4096;  // lookups per table per batch (one shared-memory sort)

struct TrainArgs {
    ds_train_table t[DS_MAX_TABLES];
    const int64_t *idx;      // every batch's ids, table-major: batch b of table t at seg(t, b)
    const float *delta;      // [ids, dim] deltas in the same order
    const int64_t *seg_off;  // device [(ntables * nbatches) + 1]: table t, batch b -> t * nb + b
    uint32_t *flags;
    int ntables, nbatches, dim;
};

__global__ void __launch_bounds__(TS_THREADS) train_apply_kernel(const TrainArgs a) {
    __shared__ unsigned long long keys[TS_MAX];
    const int t = blockIdx.x;
    const ds_train_table &tb = a.t[t];
    const int d = a.dim;
    bool bad = false;
    for (int b = 0; b < a.nbatches; b++) {  // batches in order: row updates stay sequential
        const int64_t s0 = a.seg_off[t * a.nbatches + b], s1 = a.seg_off[t * a.nbatches + b + 1];
        const int n = (int)(s1 - s0);
        if (n <= 0) continue;
        int np2 = 1;
        while (np2 < n) np2 <<= 1;
        // key = row << 12 | position; out-of-range ids sort last and are skipped
        for (int i = threadIdx.x; i < np2; i += TS_THREADS) {
            unsigned long long k = ~0ull;
            if (i < n) {
                const int64_t r = a.idx[s0 + i];
                if (r < 0 || r >= tb.rows) bad = true;
                else k = ((unsigned long long)r << 12) | (unsigned long long)i;
            }
            keys[i] = k;
        }
        __syncthreads();
        for (int k = 2; k <= np2; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < np2; i += TS_THREADS) {
                    const int l = i ^ j;
                    if (l > i) {
                        const unsigned long long x = keys[i], y = keys[l];
                        if (((i & k) == 0) == (x > y)) {
                            keys[i] = y;
                            keys[l] = x;
                        }
                    }
                }
                __syncthreads();
            }
        // every run of equal rows is applied by the thread at its head, in
        // position order (np.add.at), 4 elements at a time
        for (int i = threadIdx.x; i < n; i += TS_THREADS) {
            const unsigned long long k = keys[i];
            if (k == ~0ull) continue;
            const int64_t row = (int64_t)(k >> 12);
            if (i > 0 && (int64_t)(keys[i - 1] >> 12) == row && keys[i - 1] != ~0ull) continue;
            float *v = tb.values + row * tb.ld;
            float *x = tb.aux ? tb.aux + row * tb.ld : nullptr;
            for (int e = 0; e < d; e += 4) {
                const int w = min(4, d - e);
                float acc[4], aac[4];
                for (int q = 0; q < w; q++) {
                    acc[q] = v[e + q];
                    if (x) aac[q] = x[e + q];
                }
                for (int m = i; m < n && keys[m] != ~0ull && (int64_t)(keys[m] >> 12) == row; m++) {
                    const float *dl = a.delta + (s0 + (int64_t)(keys[m] & 0xFFF)) * d + e;
                    for (int q = 0; q < w; q++) {
                        acc[q] = __fadd_rn(acc[q], dl[q]);
                        if (x) aac[q] = __fadd_rn(aac[q], __fmul_rn(dl[q], dl[q]));
                    }
                }
                for (int q = 0; q < w; q++) {
                    v[e + q] = acc[q];
                    if (x) x[e + q] = aac[q];
                }
            }
            if (tb.words) atomicOr(tb.words + (row >> 5), 1u << (row & 31));  // tracker.mark
        }
        __syncthreads();  // the keys are rewritten by the next batch
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(a.flags, DS_FLAG_BOUNDS);
}

// ---------------------------------------------------------------------------
// The same update over an interval whose ids are stably sorted by row (host
// side: one stable sort per table), so every row's updates from all batches
// are one contiguous run in np.add.at order.  A warp owns each run that
// starts in its slice of the sorted positions: lane e adds element e's
// deltas in order (loads of the next 8 occurrences in flight), then one lane
// sets the row's dirty bit.  Hot rows no longer serialise a whole batch.
// ---------------------------------------------------------------------------
struct TrainSArgs {
    ds_train_table t[DS_MAX_TABLES];
    int64_t off[DS_MAX_TABLES + 1];  // sorted positions of table t: [off[t], off[t+1])
    const int64_t *rows;             // sorted row ids
    const int64_t *order;            // position of each sorted id in delta
    const float *delta;              // [n, dim]
    uint32_t *flags;
    int ntables, dim;
    int64_t per_warp;                // sorted positions per warp slice
};

__global__ void __launch_bounds__(256) train_sorted_kernel(const TrainSArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t n = a.off[a.ntables];
    const int64_t p0 = gw * a.per_warp, p1 = min(n, p0 + a.per_warp);
    const int d = a.dim;
    bool bad = false;
    int t = 0;
    for (int64_t b = p0; b < p1; b += 32) {
        const int64_t p = b + lane;
        int64_t row = -1, prev = -1;
        if (p < p1) {
            row = a.rows[p];
            prev = p > 0 ? a.rows[p - 1] : -1;
        }
        // heads: first occurrence of a row within its table (tables are
        // contiguous, so a table boundary is also a head)
        bool head = false;
        if (p < p1) {
            int tt = 0;
            while (tt + 1 < a.ntables && a.off[tt + 1] <= p) tt++;
            head = p == a.off[tt] || row != prev;
        }
        unsigned hm = __ballot_sync(DS_FULL_MASK, head);
        while (hm) {
            const int src = __ffs(hm) - 1;
            hm &= hm - 1;
            const int64_t hp = b + src;
            const int64_t r = __shfl_sync(DS_FULL_MASK, row, src);
            while (t + 1 < a.ntables && a.off[t + 1] <= hp) t++;  // warp-uniform
            const ds_train_table &tb = a.t[t];
            const int64_t tend = a.off[t + 1];
            if (r < 0 || r >= tb.rows) {  // out-of-range ids sort first or last: skip the run
                bad = true;
                continue;
            }
            for (int e0 = 0; e0 < d; e0 += 32) {
                const int e = e0 + lane;
                const bool on = e < d;
                float acc = 0.f, aac = 0.f;
                if (on) {
                    acc = tb.values[r * tb.ld + e];
                    if (tb.aux) aac = tb.aux[r * tb.ld + e];
                }
                int64_t m = hp;
                while (m < tend) {
                    // the next up to 8 occurrences of row r: order + delta in flight
                    int64_t pos[8];
                    float dl[8];
                    int k = 0;
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        const bool in = m + q < tend && a.rows[m + q] == r;
                        pos[q] = in ? a.order[m + q] : -1;
                    }
#pragma unroll
                    for (int q = 0; q < 8; q++) dl[q] = (pos[q] >= 0 && on) ? a.delta[pos[q] * d + e] : 0.f;
#pragma unroll
                    for (int q = 0; q < 8; q++)
                        if (pos[q] >= 0) {
                            acc = __fadd_rn(acc, dl[q]);
                            aac = __fadd_rn(aac, __fmul_rn(dl[q], dl[q]));
                            k++;
                        }
                    m += k;
                    if (k < 8) break;
                }
                if (on) {
                    tb.values[r * tb.ld + e] = acc;
                    if (tb.aux) tb.aux[r * tb.ld + e] = aac;
                }
            }
            if (lane == 0 && tb.words) atomicOr(tb.words + (r >> 5), 1u << (r & 31));
        }
    }
    if (__any_sync(DS_FULL_MASK, bad) && lane == 0) atomicOr(a.flags, DS_FLAG_BOUNDS);
}

}  // namespace ds

using namespace ds;

extern "C" int ds_train_apply(const ds_train_table *tables_host, int ntables, int nbatches,
                              int64_t dim, const int64_t *idx, const float *delta,
                              const int64_t *seg_off, uint32_t *flags, void *stream) {
    if (ntables < 1 || ntables > DS_MAX_TABLES) return host::fail(DS_ERR_ARG, "ds_train_apply: ntables");
    if (nbatches < 1 || dim < 1) return host::fail(DS_ERR_ARG, "ds_train_apply: nbatches / dim");
    if (!tables_host || !idx || !delta || !seg_off || !flags)
        return host::fail(DS_ERR_ARG, "ds_train_apply: null pointer");
    TrainArgs a;
    a.ntables = ntables;
    a.nbatches = nbatches;
    a.dim = (int)dim;
    a.idx = idx;
    a.delta = delta;
    a.seg_off = seg_off;
    a.flags = flags;
    for (int t = 0; t < ntables; t++) {
        if (!tables_host[t].values) return host::fail(DS_ERR_ARG, "ds_train_apply: null values");
        a.t[t] = tables_host[t];
    }
    train_apply_kernel<<<ntables, TS_THREADS, 0, (cudaStream_t)stream>>>(a);
    return host::check_launch("ds_train_apply");
}

extern "C" int ds_train_apply_sorted(const ds_train_table *tables_host, int ntables,
                                     const int64_t *table_off_host, int64_t dim,
                                     const int64_t *rows, const int64_t *order, const float *delta,
                                     uint32_t *flags, void *stream) {
    if (ntables < 1 || ntables > DS_MAX_TABLES)
        return host::fail(DS_ERR_ARG, "ds_train_apply_sorted: ntables");
    if (dim < 1 || !tables_host || !table_off_host || !flags)
        return host::fail(DS_ERR_ARG, "ds_train_apply_sorted: bad argument");
    TrainSArgs a;
    a.ntables = ntables;
    a.dim = (int)dim;
    a.rows = rows;
    a.order = order;
    a.delta = delta;
    a.flags = flags;
    for (int t = 0; t < ntables; t++) {
        if (!tables_host[t].values) return host::fail(DS_ERR_ARG, "ds_train_apply_sorted: null values");
        a.t[t] = tables_host[t];
    }
    for (int t = 0; t <= ntables; t++) a.off[t] = table_off_host[t];
    const int64_t n = a.off[ntables];
    if (n <= 0) return DS_OK;
    if (!rows || !order || !delta) return host::fail(DS_ERR_ARG, "ds_train_apply_sorted: null ids");
    const int64_t warps = (int64_t)host::sm_count() * 64;
    a.per_warp = ((n + warps - 1) / warps + 31) / 32 * 32;
    const int64_t nw = (n + a.per_warp - 1) / a.per_warp;
    train_sorted_kernel<<<(unsigned)((nw + 7) / 8), 256, 0, (cudaStream_t)stream>>>(a);
    return host::check_launch("ds_train_apply_sorted");
}
