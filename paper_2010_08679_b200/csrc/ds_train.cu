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


// ---------------------------------------------------------------------------
// A whole interval with the in-tree stable sort (ds_sort.cu): every lookup
// becomes a (table << row_bits | row, position) pair, one stable radix sort
// groups each row's updates in array order, and a warp applies each run.
// Hot rows (Zipf heads: ~80k updates of one row per C2 interval) are a
// sequential chain of float adds whatever the hardware; what must not be
// serial is the memory: 32 occurrences' positions arrive with one coalesced
// load, and every lane has 32 independent delta loads in flight before it
// adds them in order.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) train_keys_kernel(const int64_t *idx, int64_t n, const int64_t *off,
                                                         const int64_t *rows, int ntables, int row_bits,
                                                         uint32_t *keys, uint32_t *vals, uint32_t *flags) {
    bool bad = false;
    const uint32_t sentinel = (1u << row_bits) - 1u;  // > every valid row: out-of-range ids sort last
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int t = 0;
        for (int lo = 0, hi = ntables - 1; lo <= hi;) {  // last table with off[t] <= i
            const int mid = (lo + hi) >> 1;
            if (off[mid] <= i) { t = mid; lo = mid + 1; }
            else hi = mid - 1;
        }
        const int64_t r = idx[i];
        const bool ok = r >= 0 && r < rows[t];
        bad |= !ok;
        keys[i] = ((uint32_t)t << row_bits) | (ok ? (uint32_t)r : sentinel);
        vals[i] = (uint32_t)i;
    }
    if (__any_sync(DS_FULL_MASK, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, DS_FLAG_BOUNDS);
}

// the interval's deltas in sorted order: dsorted[m] = delta[order[m]] (one
// fully parallel gather, so the sequential per-row pass streams contiguous rows)
__global__ void __launch_bounds__(256) train_gather_kernel(const float *delta, const uint32_t *order,
                                                           int64_t n, int dim, float *dsorted) {
    if ((dim & 3) == 0) {
        const int c4 = dim >> 2;
        const int64_t total = n * c4;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
             i += (int64_t)gridDim.x * blockDim.x) {
            const int64_t m = i / c4;
            const int c = (int)(i - m * c4);
            reinterpret_cast<float4 *>(dsorted)[i] =
                __ldg(reinterpret_cast<const float4 *>(delta + (int64_t)order[m] * dim) + c);
        }
    } else {
        const int64_t total = n * dim;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
             i += (int64_t)gridDim.x * blockDim.x) {
            const int64_t m = i / dim;
            dsorted[i] = __ldg(delta + (int64_t)order[m] * dim + (i - m * dim));
        }
    }
}

constexpr int TRAIN_LONG_RUN = 4096;  // runs at least this long go to train_long_kernel

struct TrainIArgs {
    ds_train_table t[DS_MAX_TABLES];
    int64_t off[DS_MAX_TABLES + 1];  // sorted positions of table t: [off[t], off[t+1])
    const uint32_t *keys;            // sorted (table, row) keys
    const float *dsorted;            // [n, dim] deltas in sorted order
    uint32_t row_mask;
    int ntables, dim;
    int64_t per_warp;
    unsigned *nlong;                 // long runs found (device counter)
    int4 *longs;                     // (table, head lo, head hi... ) see train_interval_kernel
};

// first position in (hp, end) whose key differs from k (sorted keys): one
// probe of the next 32 positions, then (long runs) an exponential probe and
// 32-way bisection -- a handful of dependent loads for any run length
__device__ __forceinline__ int64_t run_end(const uint32_t *keys, int64_t hp, int64_t end, uint32_t k, int lane) {
    int64_t p = hp + 1 + lane;
    unsigned diff = __ballot_sync(DS_FULL_MASK, p >= end || keys[p] != k);
    if (diff) return hp + 1 + (__ffs(diff) - 1);
    // keys[hp .. hp+32] all k: exponential probe at hp + 32 * 2^lane
    int64_t lo = hp + 32;  // known equal
    p = lane < 31 ? hp + ((int64_t)32 << lane) : end;
    diff = __ballot_sync(DS_FULL_MASK, p >= end || keys[p] != k);
    const int j = __ffs(diff) - 1;  // first probe past the run (diff != 0: the last probe is end)
    int64_t hi = min(end, hp + ((int64_t)32 << j));
    if (j > 0) lo = hp + ((int64_t)32 << (j - 1));
    // run end in (lo, hi]: bisect 32 ways until the gap closes
    while (hi - lo > 1) {
        const int64_t step = (hi - lo + 31) / 32;
        const int64_t q = lo + step * (lane + 1);
        const unsigned dm = __ballot_sync(DS_FULL_MASK, q >= hi || keys[q] != k);
        const int f = __ffs(dm) - 1;
        const int64_t nlo = lo + step * f, nhi = min(hi, lo + step * (f + 1));
        lo = nlo;
        hi = nhi;
    }
    return hi;
}

__global__ void __launch_bounds__(256) train_interval_kernel(const TrainIArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t n = a.off[a.ntables];
    const int64_t p0 = gw * a.per_warp, p1 = min(n, p0 + a.per_warp);
    const int d = a.dim;
    int t = 0;
    for (int64_t b = p0; b < p1; b += 32) {
        const int64_t p = b + lane;
        uint32_t key = 0xFFFFFFFFu;
        bool head = false;
        if (p < p1) {
            key = a.keys[p];
            head = p == 0 || a.keys[p - 1] != key;  // the table is in the key: a new table is a head
        }
        unsigned hm = __ballot_sync(DS_FULL_MASK, head);
        while (hm) {
            const int src = __ffs(hm) - 1;
            hm &= hm - 1;
            const int64_t hp = b + src;
            const uint32_t k = __shfl_sync(DS_FULL_MASK, key, src);
            while (t + 1 < a.ntables && a.off[t + 1] <= hp) t++;  // warp-uniform
            const ds_train_table &tb = a.t[t];
            const int64_t r = (int64_t)(k & a.row_mask);
            if (r >= tb.rows) continue;  // out-of-range ids (flagged by the key pass)
            const int64_t re = run_end(a.keys, hp, a.off[t + 1], k, lane);
            if (d <= 32 && re - hp >= TRAIN_LONG_RUN) {  // a hot row: a whole CTA streams it (train_long_kernel)
                if (lane == 0) {
                    const unsigned slot = atomicAdd(a.nlong, 1u);
                    a.longs[slot] = make_int4(t, (int)(hp & 0xFFFFFFFF), (int)(hp >> 32), (int)(re - hp));
                }
                continue;
            }
            // lanes over elements; a d <= 16 row uses lanes 16.. for the aux chain
            const bool split = d <= 16 && tb.aux != nullptr;
            for (int e0 = 0; e0 < d; e0 += split ? 16 : 32) {
                const int e = e0 + (split ? (lane & 15) : lane);
                const bool on = e < d && (!split || e0 == 0);
                const bool do_aux = split ? lane >= 16 : tb.aux != nullptr;
                const bool do_val = split ? lane < 16 : true;
                float acc = 0.f, aac = 0.f;
                if (on) {
                    if (do_val) acc = tb.values[r * tb.ld + e];
                    if (do_aux) aac = tb.aux[r * tb.ld + e];
                }
                const float *ds = a.dsorted + (int64_t)e;
                int64_t m = hp;
                for (; m + 32 <= re; m += 32) {  // full chunks: 32 loads in flight per lane
                    float dl[32];
#pragma unroll
                    for (int j = 0; j < 32; j++) dl[j] = on ? __ldg(ds + (m + j) * d) : 0.f;
#pragma unroll
                    for (int j = 0; j < 32; j++) {  // np.add.at order
                        if (do_val) acc = __fadd_rn(acc, dl[j]);
                        if (do_aux) aac = __fadd_rn(aac, __fmul_rn(dl[j], dl[j]));
                    }
                }
                // the tail (most runs are 1-3 updates long): 4 at a time
                for (; m < re; m += 4) {
                    const int cnt = (int)min((int64_t)4, re - m);
                    float dl[4];
#pragma unroll
                    for (int j = 0; j < 4; j++) dl[j] = (j < cnt && on) ? __ldg(ds + (m + j) * d) : 0.f;
#pragma unroll
                    for (int j = 0; j < 4; j++)
                        if (j < cnt) {
                            if (do_val) acc = __fadd_rn(acc, dl[j]);
                            if (do_aux) aac = __fadd_rn(aac, __fmul_rn(dl[j], dl[j]));
                        }
                }
                if (on) {
                    if (do_val) tb.values[r * tb.ld + e] = acc;
                    if (do_aux) tb.aux[r * tb.ld + e] = aac;
                }
                if (split) break;
            }
            if (lane == 0 && tb.words) atomicOr(tb.words + (r >> 5), 1u << (r & 31));
        }
    }
}

// One CTA per hot row (a run >= TRAIN_LONG_RUN updates): warps 1..7 stream
// the run's sorted deltas through a shared-memory ring with coalesced 16-byte
// loads; warp 0 walks the ring in order, one lane per element (lanes 16..31
// carry the aux chain of a d <= 16 row), so the sequential float chain -- the
// only part np.add.at order forbids to parallelise -- is fed from shared
// memory instead of waiting on HBM.
constexpr int TL_THREADS = 256;
constexpr int TL_STAGES = 8;
constexpr int TL_OCC = 64;  // occurrences per stage

__global__ void __launch_bounds__(TL_THREADS) train_long_kernel(const TrainIArgs a) {
    extern __shared__ __align__(16) float ring[];  // TL_STAGES x TL_OCC x dim
    __shared__ volatile int filled[TL_STAGES];      // chunk index held by each stage (+1)
    __shared__ volatile int consumed;               // chunks the consumer has finished
    if ((int)blockIdx.x >= (int)*a.nlong) return;
    const int4 info = a.longs[blockIdx.x];
    const int t = info.x;
    const int64_t hp = (int64_t)(uint32_t)info.y | ((int64_t)info.z << 32);
    const int64_t len = info.w;
    const ds_train_table &tb = a.t[t];
    const int d = a.dim;
    const int64_t r = (int64_t)(a.keys[hp] & a.row_mask);
    const int64_t nchunks = (len + TL_OCC - 1) / TL_OCC;
    if (threadIdx.x < TL_STAGES) filled[threadIdx.x] = 0;
    if (threadIdx.x == 0) consumed = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp > 0) {
        // producers: warp w fills chunks w-1, w-1+7, ... (one chunk in flight
        // per warp, no CTA barrier), each into stage c % TL_STAGES once the
        // consumer released that stage's previous chunk
        const int npw = TL_THREADS / 32 - 1;
        for (int64_t c = warp - 1; c < nchunks; c += npw) {
            const int st = (int)(c % TL_STAGES);
            if (lane == 0)
                while (consumed + TL_STAGES <= c) __nanosleep(32);
            __syncwarp();
            const int64_t m0 = hp + c * TL_OCC;
            const int cnt = (int)min((int64_t)TL_OCC, hp + len - m0);
            const int nf = cnt * d;
            float *dst = ring + (size_t)st * TL_OCC * d;
            const float *src = a.dsorted + m0 * d;
            if ((d & 3) == 0) {
                constexpr int U = TL_OCC * 32 / 4 / 32;  // float4 per lane of a full d32 chunk
                float4 v[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int i = lane + 32 * u;
                    if (i < (nf >> 2)) v[u] = __ldg(reinterpret_cast<const float4 *>(src) + i);
                }
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int i = lane + 32 * u;
                    if (i < (nf >> 2)) reinterpret_cast<float4 *>(dst)[i] = v[u];
                }
            } else {
                for (int i = lane; i < nf; i += 32) dst[i] = __ldg(src + i);
            }
            __threadfence_block();
            __syncwarp();
            if (lane == 0) filled[st] = (int)(c + 1);
        }
        return;
    }
    // consumer (warp 0)
    const bool split = d <= 16 && tb.aux != nullptr;
    for (int e0 = 0; e0 < (split ? 16 : d); e0 += split ? 16 : 32) {
        // (d > 32: the ring is walked once per 32 elements -- the producers
        // only run once, so stream all chunks per pass is not possible; such
        // rows take several passes over a re-filled ring)
        const int e = e0 + (split ? (lane & 15) : lane);
        const bool on = e < d;
        const bool do_aux = split ? lane >= 16 : tb.aux != nullptr;
        const bool do_val = split ? lane < 16 : true;
        float acc = 0.f, aac = 0.f;
        if (on) {
            if (do_val) acc = tb.values[r * tb.ld + e];
            if (do_aux) aac = tb.aux[r * tb.ld + e];
        }
        for (int64_t c = 0; c < nchunks; c++) {
            const int st = (int)(c % TL_STAGES);
            while (filled[st] != (int)(c + 1)) __nanosleep(16);
            __threadfence_block();
            __syncwarp();
            const int cnt = (int)min((int64_t)TL_OCC, len - c * TL_OCC);
            const float *src = ring + (size_t)st * TL_OCC * d + e;
            if (on) {
                if (cnt == TL_OCC) {
#pragma unroll 16
                    for (int j = 0; j < TL_OCC; j++) {  // np.add.at order
                        const float dl = src[j * d];
                        if (do_val) acc = __fadd_rn(acc, dl);
                        if (do_aux) aac = __fadd_rn(aac, __fmul_rn(dl, dl));
                    }
                } else {
                    for (int j = 0; j < cnt; j++) {
                        const float dl = src[j * d];
                        if (do_val) acc = __fadd_rn(acc, dl);
                        if (do_aux) aac = __fadd_rn(aac, __fmul_rn(dl, dl));
                    }
                }
            }
            __syncwarp();
            if (lane == 0) consumed = (int)(c + 1);
        }
        if (on) {
            if (do_val) tb.values[r * tb.ld + e] = acc;
            if (do_aux) tb.aux[r * tb.ld + e] = aac;
        }
    }
    if (lane == 0 && tb.words) atomicOr(tb.words + (r >> 5), 1u << (r & 31));
}

}  // namespace ds

using namespace ds;

extern "C" size_t ds_sort_workspace_size(int64_t n);
extern "C" int ds_sort_pairs_u32(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                                 uint32_t *vals_out, int64_t n, int key_bits, void *workspace,
                                 size_t workspace_bytes, void *stream);

static int bits_for(int64_t v) {  // smallest b with 2^b > v
    int b = 0;
    while (b < 62 && ((int64_t)1 << b) <= v) b++;
    return b;
}

extern "C" size_t ds_train_interval_workspace_size(int64_t n) {
    return (size_t)4 * 4 * (n > 0 ? n : 0) + 256 + ds_sort_workspace_size(n) + (size_t)2 * 520 + 1024;
}

// deltas in sorted order ([n, dim] floats) are a second workspace
extern "C" size_t ds_train_interval_delta_bytes(int64_t n, int64_t dim) {
    // + the hot-row list: a counter and one int4 per possible long run
    return (size_t)(n > 0 ? n : 0) * (size_t)(dim > 0 ? dim : 0) * 4 + 64 +
           (size_t)((n > 0 ? n : 0) / 4096 + 1) * 16;
}

extern "C" int ds_train_apply_interval(const ds_train_table *tables_host, int ntables,
                                       const int64_t *table_off_host, int64_t dim, const int64_t *idx,
                                       const float *delta, void *workspace, size_t workspace_bytes,
                                       uint32_t *flags, void *stream) {
    if (ntables < 1 || ntables > DS_MAX_TABLES) return host::fail(DS_ERR_ARG, "ds_train_apply_interval: ntables");
    if (dim < 1 || !tables_host || !table_off_host || !flags || !workspace)
        return host::fail(DS_ERR_ARG, "ds_train_apply_interval: bad argument");
    const int64_t n = table_off_host[ntables];
    if (n <= 0) return DS_OK;
    if (!idx || !delta) return host::fail(DS_ERR_ARG, "ds_train_apply_interval: null ids");
    if (workspace_bytes < ds_train_interval_workspace_size(n) + ds_train_interval_delta_bytes(n, dim))
        return host::fail(DS_ERR_ARG, "ds_train_apply_interval: workspace too small");
    int64_t max_rows = 0;
    for (int t = 0; t < ntables; t++) {
        if (!tables_host[t].values) return host::fail(DS_ERR_ARG, "ds_train_apply_interval: null values");
        if (tables_host[t].rows > max_rows) max_rows = tables_host[t].rows;
    }
    const int row_bits = bits_for(max_rows);       // 2^row_bits - 1 >= max_rows: the sentinel
    const int table_bits = bits_for(ntables - 1);
    if (row_bits + table_bits > 32 || n > 0xFFFFFFFFll)
        return host::fail(DS_ERR_CONFIG, "ds_train_apply_interval: (table, row) keys need > 32 bits");
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t *ws = static_cast<uint8_t *>(workspace);
    uint32_t *k0 = reinterpret_cast<uint32_t *>(ws);
    uint32_t *v0 = k0 + n, *k1 = v0 + n, *v1 = k1 + n;
    ws += ((size_t)16 * n + 255) & ~(size_t)255;
    int64_t *dev_off = reinterpret_cast<int64_t *>(ws);
    int64_t *dev_rows = dev_off + (DS_MAX_TABLES + 1);
    ws += 2 * 520 + 8;
    ws = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(ws) + 255) & ~(uintptr_t)255);
    const size_t sort_ws = ds_sort_workspace_size(n);
    int64_t host_small[2 * (DS_MAX_TABLES + 1)];
    for (int t = 0; t <= ntables; t++) host_small[t] = table_off_host[t];
    for (int t = 0; t < ntables; t++) host_small[DS_MAX_TABLES + 1 + t] = tables_host[t].rows;
    cudaError_t e = cudaMemcpyAsync(dev_off, host_small, sizeof(host_small), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)host::sm_count() * 16) blocks = (int64_t)host::sm_count() * 16;
    train_keys_kernel<<<(unsigned)blocks, 256, 0, s>>>(idx, n, dev_off, dev_rows, ntables, row_bits, k0, v0, flags);
    int st = ds_sort_pairs_u32(k0, v0, k1, v1, n, row_bits + table_bits, ws, sort_ws, stream);
    if (st != DS_OK) return st;
    float *dsorted = reinterpret_cast<float *>(ws + ((sort_ws + 255) & ~(size_t)255));
    int64_t gblocks = (n * (dim % 4 == 0 ? dim / 4 : dim) + 255) / 256;
    if (gblocks > (int64_t)host::sm_count() * 16) gblocks = (int64_t)host::sm_count() * 16;
    train_gather_kernel<<<(unsigned)gblocks, 256, 0, s>>>(delta, v1, n, (int)dim, dsorted);
    TrainIArgs a;
    a.ntables = ntables;
    a.dim = (int)dim;
    a.keys = k1;
    a.dsorted = dsorted;
    a.row_mask = (uint32_t)(((uint64_t)1 << row_bits) - 1);
    for (int t = 0; t < ntables; t++) a.t[t] = tables_host[t];
    for (int t = 0; t <= ntables; t++) a.off[t] = table_off_host[t];
    const int64_t warps = (int64_t)host::sm_count() * 64;
    a.per_warp = ((n + warps - 1) / warps + 31) / 32 * 32;
    const int64_t nw = (n + a.per_warp - 1) / a.per_warp;
    unsigned *nlong = reinterpret_cast<unsigned *>(dsorted + n * dim + 4);
    nlong = reinterpret_cast<unsigned *>((reinterpret_cast<uintptr_t>(nlong) + 15) & ~(uintptr_t)15);
    a.nlong = nlong;
    a.longs = reinterpret_cast<int4 *>(nlong + 4);
    e = cudaMemsetAsync(nlong, 0, 16, s);
    if (e != cudaSuccess) return host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
    train_interval_kernel<<<(unsigned)((nw + 7) / 8), 256, 0, s>>>(a);
    // hot rows: at most n / TRAIN_LONG_RUN of them, one CTA each (the kernel
    // reads the count on the device: no host sync); rows wider than 32
    // elements keep the warp path (the ring is filled once)
    const int64_t maxlong = n / TRAIN_LONG_RUN;
    if (maxlong > 0 && (dim <= 32)) {
        const size_t smem = (size_t)TL_STAGES * TL_OCC * dim * 4;
        cudaFuncSetAttribute(train_long_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        train_long_kernel<<<(unsigned)maxlong, TL_THREADS, smem, s>>>(a);
    }
    return host::check_launch("ds_train_apply_interval");
}

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
