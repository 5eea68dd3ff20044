// ds_sort.cu -- stable LSD radix sort of (u32 key, u32 value) pairs.
//
// The training step (sim.py:140-155) groups an interval's
// lookups by (table, row) so each row's updates can be applied in np.add.at
// order by one warp; the grouping must be STABLE (array order within a row).
// This replaces the library sort (torch.sort) the round-1 path called.
//
// Per 8-bit digit (ceil(key_bits / 8) passes):
//   sort_hist_kernel     per tile of 2048 pairs: digit counts -> hist[digit][tile]
//   scan (3 launches)    exclusive prefix of hist in digit-major order: each
//                        (digit, tile)'s first output position
//   sort_scatter_kernel  per tile, 8 rounds of 256 pairs in array order: a
//                        pair's rank among equal digits of its warp comes from
//                        __match_any_sync, warps of a round are prefixed per
//                        digit in shared memory, rounds accumulate -- so equal
//                        digits keep their input order (stability).
#include <cuda_runtime.h>
#include <stdint.h>

#include "ds_common.cuh"
#include "ds_host.h"

namespace ds {

constexpr int SR_THREADS = 256;
constexpr int SR_ROUNDS = 8;
constexpr int SR_TILE = SR_THREADS * SR_ROUNDS;  // 2048 pairs
constexpr int SR_SCAN_CHUNK = 4096;              // hist entries per scan block

__global__ void __launch_bounds__(SR_THREADS) sort_hist_kernel(const uint32_t *keys, int64_t n, int shift,
                                                               uint32_t *hist, int64_t ntiles) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * SR_TILE;
#pragma unroll
    for (int r = 0; r < SR_ROUNDS; r++) {
        const int64_t i = base + r * SR_THREADS + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255u], 1u);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// block sums of SR_SCAN_CHUNK-entry chunks
__global__ void __launch_bounds__(SR_THREADS) sort_scan_reduce(const uint32_t *hist, int64_t m, uint32_t *part) {
    __shared__ uint32_t s[SR_THREADS / 32];
    const int64_t c0 = (int64_t)blockIdx.x * SR_SCAN_CHUNK;
    uint32_t v = 0;
    for (int k = threadIdx.x; k < SR_SCAN_CHUNK; k += SR_THREADS)
        if (c0 + k < m) v += hist[c0 + k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(DS_FULL_MASK, v, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < SR_THREADS / 32; w++) t += s[w];
        part[blockIdx.x] = t;
    }
}

// exclusive scan of the block sums (one block; nparts <= a few thousand)
__global__ void __launch_bounds__(SR_THREADS) sort_scan_parts(uint32_t *part, int nparts) {
    __shared__ uint32_t carry;
    __shared__ uint32_t ws[SR_THREADS / 32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int b = 0; b < nparts; b += SR_THREADS) {
        const int i = b + threadIdx.x;
        const uint32_t v = i < nparts ? part[i] : 0;
        uint32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(DS_FULL_MASK, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) ws[w] = x;
        __syncthreads();
        uint32_t wp = 0;
        for (int k = 0; k < w; k++) wp += ws[k];
        const uint32_t c = carry;
        if (i < nparts) part[i] = c + wp + x - v;
        __syncthreads();
        if (threadIdx.x == SR_THREADS - 1) carry = c + wp + x;
        __syncthreads();
    }
}

// exclusive scan inside each chunk, offset by the chunk's prefix
__global__ void __launch_bounds__(SR_THREADS) sort_scan_apply(uint32_t *hist, int64_t m, const uint32_t *part) {
    __shared__ uint32_t ws[SR_THREADS / 32];
    __shared__ uint32_t carry;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t c0 = (int64_t)blockIdx.x * SR_SCAN_CHUNK;
    if (threadIdx.x == 0) carry = part[blockIdx.x];
    __syncthreads();
    for (int b = 0; b < SR_SCAN_CHUNK; b += SR_THREADS) {
        const int64_t i = c0 + b + threadIdx.x;
        const uint32_t v = i < m ? hist[i] : 0;
        uint32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(DS_FULL_MASK, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) ws[w] = x;
        __syncthreads();
        uint32_t wp = 0;
        for (int k = 0; k < w; k++) wp += ws[k];
        const uint32_t c = carry;
        if (i < m) hist[i] = c + wp + x - v;
        __syncthreads();
        if (threadIdx.x == SR_THREADS - 1) carry = c + wp + x;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(SR_THREADS) sort_scatter_kernel(const uint32_t *kin, const uint32_t *vin,
                                                                  uint32_t *kout, uint32_t *vout, int64_t n,
                                                                  int shift, const uint32_t *offs,
                                                                  int64_t ntiles) {
    __shared__ uint32_t run[256];                  // next output position per digit
    __shared__ uint32_t wc[SR_THREADS / 32][257];  // per-warp digit counts -> warp prefixes
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    run[tid] = offs[(int64_t)tid * ntiles + blockIdx.x];
    const unsigned lt = (1u << lane) - 1u;
    const int64_t base = (int64_t)blockIdx.x * SR_TILE;
    for (int r = 0; r < SR_ROUNDS; r++) {
#pragma unroll
        for (int k = 0; k < SR_THREADS / 32; k++) wc[k][tid] = 0;
        __syncthreads();
        const int64_t i = base + r * SR_THREADS + tid;
        const bool valid = i < n;
        const uint32_t key = valid ? kin[i] : 0u;
        const uint32_t val = valid ? vin[i] : 0u;
        const int digit = valid ? (int)((key >> shift) & 255u) : 256;  // 256: out of range
        const unsigned peers = __match_any_sync(DS_FULL_MASK, digit);
        const int rank = __popc(peers & lt);
        if (valid && rank == 0) wc[w][digit] = __popc(peers);
        __syncthreads();
        {  // thread d: warps' counts of digit d -> their first positions
            uint32_t acc = run[tid];
#pragma unroll
            for (int k = 0; k < SR_THREADS / 32; k++) {
                const uint32_t c = wc[k][tid];
                wc[k][tid] = acc;
                acc += c;
            }
            run[tid] = acc;
        }
        __syncthreads();
        if (valid) {
            const uint32_t pos = wc[w][digit] + (uint32_t)rank;
            kout[pos] = key;
            vout[pos] = val;
        }
        __syncthreads();
    }
}

static int64_t sort_tiles(int64_t n) { return (n + SR_TILE - 1) / SR_TILE; }
static int64_t sort_scan_blocks(int64_t n) { return (256 * sort_tiles(n) + SR_SCAN_CHUNK - 1) / SR_SCAN_CHUNK; }

}  // namespace ds

using namespace ds;

extern "C" size_t ds_sort_workspace_size(int64_t n) {
    if (n < 0) n = 0;
    const size_t hist = (size_t)256 * sort_tiles(n) * 4;
    const size_t part = (size_t)sort_scan_blocks(n) * 4;
    return ((hist + 255) & ~(size_t)255) + ((part + 255) & ~(size_t)255) + (size_t)2 * n * 4 + 512;
}

// Stable sort of n (key, value) pairs by the low key_bits bits of the key.
// Input arrays are left intact; the result lands in keys_out / vals_out.
extern "C" int ds_sort_pairs_u32(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                                 uint32_t *vals_out, int64_t n, int key_bits, void *workspace,
                                 size_t workspace_bytes, void *stream) {
    if (n < 0 || key_bits < 1 || key_bits > 32) return host::fail(DS_ERR_ARG, "ds_sort_pairs_u32: bad n / key_bits");
    if (n == 0) return DS_OK;
    if (n > 0xFFFFFFFFll) return host::fail(DS_ERR_ARG, "ds_sort_pairs_u32: at most 2^32 - 1 pairs");
    if (!keys_in || !vals_in || !keys_out || !vals_out || !workspace)
        return host::fail(DS_ERR_ARG, "ds_sort_pairs_u32: null pointer");
    if (workspace_bytes < ds_sort_workspace_size(n)) return host::fail(DS_ERR_ARG, "ds_sort_pairs_u32: workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t ntiles = sort_tiles(n), m = 256 * ntiles, nscan = sort_scan_blocks(n);
    uint8_t *ws = static_cast<uint8_t *>(workspace);
    uint32_t *hist = reinterpret_cast<uint32_t *>(ws);
    ws += ((size_t)m * 4 + 255) & ~(size_t)255;
    uint32_t *part = reinterpret_cast<uint32_t *>(ws);
    ws += ((size_t)nscan * 4 + 255) & ~(size_t)255;
    uint32_t *tk = reinterpret_cast<uint32_t *>(ws);
    uint32_t *tv = tk + n;
    const int passes = (key_bits + 7) / 8;
    // ping-pong so the last pass writes keys_out / vals_out
    const uint32_t *ck = keys_in, *cv = vals_in;
    for (int p = 0; p < passes; p++) {
        const bool last = p == passes - 1;
        uint32_t *ok = ((passes - 1 - p) & 1) == 0 ? keys_out : tk;
        uint32_t *ov = ((passes - 1 - p) & 1) == 0 ? vals_out : tv;
        (void)last;
        sort_hist_kernel<<<(unsigned)ntiles, SR_THREADS, 0, s>>>(ck, n, 8 * p, hist, ntiles);
        sort_scan_reduce<<<(unsigned)nscan, SR_THREADS, 0, s>>>(hist, m, part);
        sort_scan_parts<<<1, SR_THREADS, 0, s>>>(part, (int)nscan);
        sort_scan_apply<<<(unsigned)nscan, SR_THREADS, 0, s>>>(hist, m, part);
        sort_scatter_kernel<<<(unsigned)ntiles, SR_THREADS, 0, s>>>(ck, cv, ok, ov, n, 8 * p, hist, ntiles);
        ck = ok;
        cv = ov;
    }
    return host::check_launch("ds_sort_pairs_u32");
}
