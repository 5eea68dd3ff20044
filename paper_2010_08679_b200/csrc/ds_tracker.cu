// ds_tracker.cu -- K0 bitmap maintenance, K1 mark, K2 capture/compaction.
//
// Reference: deltasnap/tracker.py:19-139.  The bitmap of a table is a run of
// uint32 little-endian words (bit r -> word r>>5, bit r&31), byte-identical to
// the reference's uint8 bitset (tracker.py:25,36).
#include <cuda_runtime.h>
#include <stdint.h>

#include "ds_common.cuh"
#include "ds_host.h"

namespace ds {

// ---------------------------------------------------------------------------
// K1: mark.  Test-before-set: a bit that is already set (the common case for
// Zipf-hot rows) costs one L2 read instead of a contended atomic; a stale read
// only costs a redundant atomicOr, never a lost mark (bits are only set here).
// ---------------------------------------------------------------------------
struct MarkArgs {
    uint32_t *words;
    const int64_t *idx;
    uint32_t *flags;
    int64_t word_off[DS_MAX_TABLES];
    int64_t rows[DS_MAX_TABLES];
    int64_t seg_off[DS_MAX_TABLES + 1];
    int32_t seg_table[DS_MAX_TABLES];
    int nseg;
};

__global__ void __launch_bounds__(256) mark_kernel(const MarkArgs a) {
    __shared__ int64_t s_seg_off[DS_MAX_TABLES + 1];
    __shared__ int64_t s_base[DS_MAX_TABLES];
    __shared__ int64_t s_rows[DS_MAX_TABLES];
    for (int s = threadIdx.x; s <= a.nseg; s += blockDim.x) {
        s_seg_off[s] = a.seg_off[s];
        if (s < a.nseg) {
            s_base[s] = a.word_off[a.seg_table[s]];
            s_rows[s] = a.rows[a.seg_table[s]];
        }
    }
    __syncthreads();
    const int64_t total = s_seg_off[a.nseg];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        int64_t r = __ldcs(a.idx + i);  // streamed once: do not keep in L2
        int lo = 0, hi = a.nseg - 1;     // segment of i: largest s with seg_off[s] <= i
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (s_seg_off[mid] <= i) lo = mid;
            else hi = mid - 1;
        }
        if (r < 0 || r >= s_rows[lo]) {
            bad = true;
            continue;
        }
        uint32_t *w = a.words + s_base[lo] + (r >> 5);
        uint32_t bit = 1u << (r & 31);
        if (!(__ldcg(w) & bit)) atomicOr(w, bit);
    }
    if (__any_sync(DS_FULL_MASK, bad) && (threadIdx.x & 31) == 0) atomicOr(a.flags, DS_FLAG_BOUNDS);
}

// ---------------------------------------------------------------------------
// K0: bitmap ops and popcount
// ---------------------------------------------------------------------------
__global__ void bitmap_op_kernel(uint32_t *dst, uint32_t *a, uint32_t *b, int64_t n, int op) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        switch (op) {
            case 0: dst[i] = a[i] | b[i]; break;         // merge_or   tracker.py:38-44
            case 1: dst[i] |= a[i]; break;               // merge_in   tracker.py:46-49
            case 2: b[i] |= a[i]; a[i] = 0u; break;      // reset_interval :120-124
            case 3: a[i] = 0u; b[i] = 0u; break;         // reset_baseline :126-130
        }
    }
}

__global__ void popcount_kernel(const uint32_t *w, int64_t n, unsigned long long *out) {
    unsigned long long c = 0;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        c += __popc(w[i]);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(DS_FULL_MASK, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// ---------------------------------------------------------------------------
// K2: capture.  Three launches over "chunks" of WPB words that never straddle
// a table: count -> scan -> write (+ optional fold).  Ids are written through
// a shared-memory stage so global stores are coalesced int64 runs.
// ---------------------------------------------------------------------------
constexpr int CAP_THREADS = 256;
constexpr int CAP_ROUNDS = 8;
constexpr int CAP_WPB = CAP_THREADS * CAP_ROUNDS;  // 2048 words = 65536 rows per chunk

struct CapArgs {
    const uint32_t *interval;
    const uint32_t *baseline;  // may be null
    uint32_t *interval_w;      // fold targets
    uint32_t *baseline_w;
    int64_t *ids_int;
    int64_t *ids_uni;
    int64_t *counts;           // [2*ntables+2]
    unsigned long long *chunk_cnt;  // [2*nchunks]
    unsigned long long *chunk_base; // [2*nchunks]
    int64_t word_off[DS_MAX_TABLES + 1];
    int64_t chunk_off[DS_MAX_TABLES + 1];
    int ntables;
    int64_t nchunks;
    int fold;
};

__device__ __forceinline__ int chunk_table(const CapArgs &a, int64_t c) {
    int lo = 0, hi = a.ntables - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (a.chunk_off[mid] <= c) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long v, unsigned long long *sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(DS_FULL_MASK, v, o);
    int w = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[w] = v;
    __syncthreads();
    unsigned long long t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); i++) t += sh[i];
    return t;
}

__global__ void __launch_bounds__(CAP_THREADS) capture_count_kernel(const CapArgs a) {
    __shared__ unsigned long long sh[2][CAP_THREADS / 32];
    int64_t c = blockIdx.x;
    int t = chunk_table(a, c);
    int64_t w0 = a.word_off[t] + (c - a.chunk_off[t]) * CAP_WPB;
    int64_t w1 = min(w0 + CAP_WPB, a.word_off[t + 1]);
    unsigned long long ci = 0, cu = 0;
    for (int64_t w = w0 + threadIdx.x; w < w1; w += CAP_THREADS) {
        uint32_t iv = a.interval[w];
        uint32_t bv = a.baseline ? a.baseline[w] : 0u;
        ci += __popc(iv);
        cu += __popc(iv | bv);
    }
    ci = block_sum_u64(ci, sh[0]);
    cu = block_sum_u64(cu, sh[1]);
    if (threadIdx.x == 0) {
        a.chunk_cnt[c] = ci;
        a.chunk_cnt[a.nchunks + c] = cu;
    }
}

// single block: exclusive scan of chunk counts (both scopes) + per-table totals
__global__ void __launch_bounds__(1024) capture_scan_kernel(const CapArgs a) {
    __shared__ unsigned long long warp_tot[32];
    __shared__ unsigned long long carry;
    for (int scope = 0; scope < 2; scope++) {
        const unsigned long long *cnt = a.chunk_cnt + scope * a.nchunks;
        unsigned long long *base = a.chunk_base + scope * a.nchunks;
        if (threadIdx.x == 0) carry = 0;
        __syncthreads();
        for (int64_t s = 0; s < a.nchunks; s += blockDim.x) {
            int64_t i = s + threadIdx.x;
            unsigned long long v = i < a.nchunks ? cnt[i] : 0ull;
            unsigned long long x = v;  // inclusive warp scan
            for (int o = 1; o < 32; o <<= 1) {
                unsigned long long y = __shfl_up_sync(DS_FULL_MASK, x, o);
                if ((threadIdx.x & 31) >= o) x += y;
            }
            if ((threadIdx.x & 31) == 31) warp_tot[threadIdx.x >> 5] = x;
            __syncthreads();
            if (threadIdx.x < 32) {
                unsigned long long wv = threadIdx.x < (blockDim.x >> 5) ? warp_tot[threadIdx.x] : 0ull;
                unsigned long long wx = wv;
                for (int o = 1; o < 32; o <<= 1) {
                    unsigned long long y = __shfl_up_sync(DS_FULL_MASK, wx, o);
                    if (threadIdx.x >= o) wx += y;
                }
                warp_tot[threadIdx.x] = wx - wv;  // exclusive
            }
            __syncthreads();
            unsigned long long excl = carry + warp_tot[threadIdx.x >> 5] + x - v;
            if (i < a.nchunks) base[i] = excl;
            __syncthreads();
            if (threadIdx.x == blockDim.x - 1) carry = excl + v;
            __syncthreads();
        }
        // per-table counts from the chunk bases
        for (int t = threadIdx.x; t < a.ntables; t += blockDim.x) {
            int64_t c0 = a.chunk_off[t], c1 = a.chunk_off[t + 1];
            unsigned long long b0 = c0 < a.nchunks ? base[c0] : carry;
            unsigned long long b1 = c1 < a.nchunks ? base[c1] : carry;
            a.counts[scope * (a.ntables + 1) + t] = (int64_t)(b1 - b0);
        }
        if (threadIdx.x == 0) a.counts[scope * (a.ntables + 1) + a.ntables] = (int64_t)carry;
        __syncthreads();
    }
}

// block-wide exclusive scan of one int per thread (CAP_THREADS threads)
__device__ __forceinline__ int block_excl_scan(int v, int *sh, int &total) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(DS_FULL_MASK, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[w] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
        int wv = threadIdx.x < CAP_THREADS / 32 ? sh[threadIdx.x] : 0;
        int wx = wv;
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(DS_FULL_MASK, wx, o);
            if (threadIdx.x >= o) wx += y;
        }
        sh[32 + threadIdx.x] = wx - wv;
        if (threadIdx.x == 31) sh[64] = wx;
    }
    __syncthreads();
    int r = sh[32 + w] + x - v;
    total = sh[64];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(CAP_THREADS) capture_write_kernel(const CapArgs a) {
    __shared__ uint16_t stage[2][CAP_THREADS * 32];
    __shared__ int scan_sh[2][72];
    int64_t c = blockIdx.x;
    int t = chunk_table(a, c);
    int64_t wt0 = a.word_off[t];
    int64_t w0 = wt0 + (c - a.chunk_off[t]) * CAP_WPB;
    int64_t w1 = min(w0 + CAP_WPB, a.word_off[t + 1]);
    int64_t row0 = (w0 - wt0) * 32;  // table row of bit 0 of word w0
    // output positions: table section of the concatenated id list
    int64_t out_i = (int64_t)a.chunk_base[c];
    int64_t out_u = (int64_t)a.chunk_base[a.nchunks + c];
    for (int rnd = 0; rnd < CAP_ROUNDS; rnd++) {
        int64_t w = w0 + rnd * CAP_THREADS + threadIdx.x;
        uint32_t iv = 0, bv = 0;
        if (w < w1) {
            iv = a.interval[w];
            bv = a.baseline ? a.baseline[w] : 0u;
        }
        uint32_t uv = iv | bv;
        int tot_i, tot_u;
        int off_i = block_excl_scan(__popc(iv), scan_sh[0], tot_i);
        int off_u = block_excl_scan(__popc(uv), scan_sh[1], tot_u);
        uint16_t local = (uint16_t)((rnd * CAP_THREADS + threadIdx.x) * 32);
        if (a.ids_int) {
            uint32_t m = iv;
            while (m) {
                int b = __ffs(m) - 1;
                stage[0][off_i++] = (uint16_t)(local + b);
                m &= m - 1;
            }
        }
        if (a.ids_uni) {
            uint32_t m = uv;
            while (m) {
                int b = __ffs(m) - 1;
                stage[1][off_u++] = (uint16_t)(local + b);
                m &= m - 1;
            }
        }
        __syncthreads();
        if (a.ids_int)
            for (int k = threadIdx.x; k < tot_i; k += CAP_THREADS)
                a.ids_int[out_i + k] = row0 + stage[0][k];
        if (a.ids_uni)
            for (int k = threadIdx.x; k < tot_u; k += CAP_THREADS)
                a.ids_uni[out_u + k] = row0 + stage[1][k];
        out_i += tot_i;
        out_u += tot_u;
        if (w < w1) {
            if (a.fold == 1) {
                if (a.baseline_w) a.baseline_w[w] = uv;
                a.interval_w[w] = 0u;
            } else if (a.fold == 2) {
                if (a.baseline_w) a.baseline_w[w] = 0u;
                a.interval_w[w] = 0u;
            }
        }
        __syncthreads();
    }
}

}  // namespace ds

using namespace ds;

extern "C" int ds_mark(uint32_t *words, const int64_t *word_off, const int64_t *rows,
                       const int64_t *idx, const int64_t *seg_off_host,
                       const int32_t *seg_table_host, int nseg, uint32_t *flags, void *stream) {
    if (nseg < 1 || nseg > DS_MAX_TABLES) return host::fail(DS_ERR_ARG, "ds_mark: nseg out of range");
    if (!words || !word_off || !rows || !flags) return host::fail(DS_ERR_ARG, "ds_mark: null pointer");
    MarkArgs a;
    a.words = words;
    a.idx = idx;
    a.flags = flags;
    a.nseg = nseg;
    for (int s = 0; s < nseg; s++) {
        int t = seg_table_host ? seg_table_host[s] : 0;
        if (t < 0 || t >= DS_MAX_TABLES) return host::fail(DS_ERR_ARG, "ds_mark: table index");
        a.seg_table[s] = s;  // resolved below: per-segment base/rows
        a.word_off[s] = word_off[t];
        a.rows[s] = rows[t];
        a.seg_off[s] = seg_off_host[s];
    }
    a.seg_off[nseg] = seg_off_host[nseg];
    int64_t total = a.seg_off[nseg] - a.seg_off[0];
    if (total <= 0) return DS_OK;
    if (!idx) return host::fail(DS_ERR_ARG, "ds_mark: null idx");
    int64_t blocks = host::grid_for(total, 256, 8);
    mark_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(a);
    return host::check_launch("ds_mark");
}

extern "C" int ds_mark_table(uint32_t *words, int64_t rows, const int64_t *idx, int64_t n,
                             uint32_t *flags, void *stream) {
    int64_t wo = 0, so[2] = {0, n};
    return ds_mark(words, &wo, &rows, idx, so, nullptr, 1, flags, stream);
}

extern "C" int ds_bitmap_op(uint32_t *dst, uint32_t *a, uint32_t *b, int64_t nwords, int op,
                            void *stream) {
    if (op < 0 || op > 3) return host::fail(DS_ERR_ARG, "ds_bitmap_op: op");
    if (nwords <= 0) return DS_OK;
    bitmap_op_kernel<<<(unsigned)host::grid_for(nwords, 256, 4), 256, 0, (cudaStream_t)stream>>>(
        dst, a, b, nwords, op);
    return host::check_launch("ds_bitmap_op");
}

extern "C" int ds_popcount(const uint32_t *words, int64_t nwords, int64_t *out, void *stream) {
    cudaMemsetAsync(out, 0, sizeof(int64_t), (cudaStream_t)stream);
    if (nwords > 0)
        popcount_kernel<<<(unsigned)host::grid_for(nwords, 256, 4), 256, 0, (cudaStream_t)stream>>>(
            words, nwords, reinterpret_cast<unsigned long long *>(out));
    return host::check_launch("ds_popcount");
}

static int64_t capture_nchunks(const int64_t *word_off_host, int ntables) {
    int64_t n = 0;
    for (int t = 0; t < ntables; t++) {
        int64_t w = word_off_host[t + 1] - word_off_host[t];
        n += w > 0 ? (w + CAP_WPB - 1) / CAP_WPB : 1;
    }
    return n;
}

extern "C" size_t ds_capture_workspace_size(int64_t total_words, int ntables) {
    // 4 arrays of nchunks u64; nchunks <= total_words/CAP_WPB + ntables
    int64_t nchunks = total_words / CAP_WPB + 2 * (int64_t)ntables + 1;
    return (size_t)(4 * nchunks) * sizeof(unsigned long long) + 256;
}

extern "C" int ds_capture(uint32_t *interval, uint32_t *baseline, const int64_t *word_off_host,
                          const int64_t *rows_host, int ntables, int64_t *ids_int,
                          int64_t *ids_union, int64_t *counts, int fold, void *workspace,
                          size_t workspace_bytes, void *stream) {
    (void)rows_host;
    if (ntables < 1 || ntables > DS_MAX_TABLES) return host::fail(DS_ERR_ARG, "ds_capture: ntables");
    if (!interval || !counts || !workspace) return host::fail(DS_ERR_ARG, "ds_capture: null pointer");
    CapArgs a;
    a.interval = interval;
    a.baseline = baseline;
    a.interval_w = interval;
    a.baseline_w = baseline;
    a.ids_int = ids_int;
    a.ids_uni = ids_union;
    a.counts = counts;
    a.ntables = ntables;
    a.fold = fold;
    int64_t nch = 0;
    for (int t = 0; t <= ntables; t++) a.word_off[t] = word_off_host[t];
    for (int t = 0; t < ntables; t++) {
        a.chunk_off[t] = nch;
        int64_t w = word_off_host[t + 1] - word_off_host[t];
        nch += w > 0 ? (w + CAP_WPB - 1) / CAP_WPB : 1;
    }
    a.chunk_off[ntables] = nch;
    a.nchunks = nch;
    size_t need = (size_t)(4 * nch) * sizeof(unsigned long long);
    if (workspace_bytes < need) return host::fail(DS_ERR_ARG, "ds_capture: workspace too small");
    a.chunk_cnt = reinterpret_cast<unsigned long long *>(workspace);
    a.chunk_base = a.chunk_cnt + 2 * nch;
    cudaStream_t s = (cudaStream_t)stream;
    capture_count_kernel<<<(unsigned)nch, CAP_THREADS, 0, s>>>(a);
    capture_scan_kernel<<<1, 1024, 0, s>>>(a);
    capture_write_kernel<<<(unsigned)nch, CAP_THREADS, 0, s>>>(a);
    (void)capture_nchunks;
    return host::check_launch("ds_capture");
}
