// ds_crc.cu -- CRC-32 (IEEE 802.3, zlib.crc32) of a device buffer.
//
// The reference checksums every shard payload on the host before it goes to
// the store and again on read-back (deltasnap/store.py:46-47, :362, :500;
// SURVEY.md 8(f) row 3).  Here the payload never has to be re-read on the
// host: CTAs take 32 KB chunks, each thread the CRC of its own 128 bytes
// (slicing-by-4 tables in shared memory), and CRCs of consecutive pieces
// combine linearly, crc(A|B) = x^(8|B|) * crc(A) xor crc(B) (zlib's
// crc32_combine), with the multiply-by-x^(8n) operators precomputed as
// 32x32 GF(2) matrices: each chunk shifts its CRC by the bytes after it
// (binary powers of the 32 KB operator) and xors it into the result.
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "ds_common.cuh"
#include "ds_host.h"

namespace ds {

constexpr int CRC_THREADS = 256;
constexpr int CRC_PIECE = 128;                         // bytes per thread
constexpr int CRC_CHUNK = CRC_THREADS * CRC_PIECE;     // 32 KB per CTA
constexpr uint32_t CRC_POLY = 0xEDB88320u;             // reflected IEEE polynomial

// operators (columns: image of bit i): shift by 128*k bytes (k = 0..256) and
// by r bytes (r = 0..128); slicing-by-4 tables
__device__ uint32_t g_op128[257][32];
__device__ uint32_t g_opr[CRC_PIECE + 1][32];
__device__ uint32_t g_pow[32][32];  // shift by 32 KB * 2^b
__device__ uint32_t g_tab[4][256];

// warp-parallel GF(2) mat-vec: lane i holds column i (every lane gets M v)
__device__ __forceinline__ uint32_t gf2_times_warp(const uint32_t *mat, uint32_t v, int lane) {
    uint32_t s = (v >> lane & 1u) ? __ldg(mat + lane) : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s ^= __shfl_xor_sync(DS_FULL_MASK, s, o);
    return s;
}

__device__ __forceinline__ uint32_t gf2_times(const uint32_t *mat, uint32_t v) {
    uint32_t s = 0;
#pragma unroll 8
    for (int i = 0; i < 32; i++)
        if (v >> i & 1u) s ^= __ldg(mat + i);
    return s;
}

// conditioned CRC (zlib.crc32) of each 32 KB chunk
__global__ void __launch_bounds__(CRC_THREADS) crc_chunk_kernel(const uint8_t *data, int64_t n,
                                                               uint32_t *out) {
    __shared__ uint32_t tab[4][256];
    __shared__ uint32_t s_red[CRC_THREADS / 32];
    for (int i = threadIdx.x; i < 4 * 256; i += CRC_THREADS) tab[i >> 8][i & 255] = g_tab[i >> 8][i & 255];
    __syncthreads();
    const int64_t c0 = (int64_t)blockIdx.x * CRC_CHUNK;
    const int clen = (int)min((int64_t)CRC_CHUNK, n - c0);
    const int npieces = (clen + CRC_PIECE - 1) / CRC_PIECE;
    const int t = threadIdx.x;
    const int plen = t < npieces ? min(CRC_PIECE, clen - t * CRC_PIECE) : 0;
    const uint8_t *p = data + c0 + (int64_t)t * CRC_PIECE;
    uint32_t crc = 0xFFFFFFFFu;
    int i = 0;
    if ((reinterpret_cast<uintptr_t>(p) & 3) == 0) {
        for (; i + 4 <= plen; i += 4) {
            crc ^= *reinterpret_cast<const uint32_t *>(p + i);
            crc = tab[3][crc & 255] ^ tab[2][(crc >> 8) & 255] ^ tab[1][(crc >> 16) & 255] ^ tab[0][crc >> 24];
        }
    }
    for (; i < plen; i++) crc = tab[0][(crc ^ p[i]) & 255] ^ (crc >> 8);
    crc = plen ? ~crc : 0u;  // crc32(b"") == 0
    // shift by the bytes after this piece: 128 * (npieces - 2 - t) + last piece length
    if (plen && t < npieces - 1) {
        const int rlast = clen - (npieces - 1) * CRC_PIECE;
        crc = gf2_times(g_opr[rlast], gf2_times(g_op128[npieces - 2 - t], crc));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) crc ^= __shfl_xor_sync(DS_FULL_MASK, crc, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = crc;
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        uint32_t v = 0;
#pragma unroll
        for (int w = 0; w < CRC_THREADS / 32; w++) v ^= s_red[w];
        // this chunk's term of the whole CRC: shift by the bytes after it,
        // 32 KB * j (binary powers) + the last chunk's length
        const int64_t nchunks = (n + CRC_CHUNK - 1) / CRC_CHUNK;
        if ((int64_t)blockIdx.x < nchunks - 1) {
            const int64_t j = nchunks - 2 - (int64_t)blockIdx.x;
            for (int b = 0; (j >> b) != 0; b++)
                if (j >> b & 1) v = gf2_times_warp(g_pow[b], v, lane);
            const int64_t llen = n - (nchunks - 1) * (int64_t)CRC_CHUNK;
            v = gf2_times_warp(g_op128[llen / CRC_PIECE], v, lane);
            v = gf2_times_warp(g_opr[llen % CRC_PIECE], v, lane);
        }
        if (lane == 0) atomicXor(out, v);  // xor: order-independent, deterministic
    }
}

}  // namespace ds

using namespace ds;

namespace {

void gf2_square(uint32_t *dst, const uint32_t *m) {
    for (int i = 0; i < 32; i++) {
        uint32_t s = 0, v = m[i];
        for (int j = 0; v; j++, v >>= 1)
            if (v & 1u) s ^= m[j];
        dst[i] = s;
    }
}

// c = a o b (apply b, then a)
void gf2_mul(uint32_t *c, const uint32_t *a, const uint32_t *b) {
    uint32_t t[32];
    for (int i = 0; i < 32; i++) {
        uint32_t s = 0, v = b[i];
        for (int j = 0; v; j++, v >>= 1)
            if (v & 1u) s ^= a[j];
        t[i] = s;
    }
    for (int i = 0; i < 32; i++) c[i] = t[i];
}

// per-device one-time upload of the operator and slicing tables
int crc_init(int dev) {
    static std::once_flag flags[DS_MAX_TABLES];
    static int status[DS_MAX_TABLES];
    if (dev < 0 || dev >= DS_MAX_TABLES) return host::fail(DS_ERR_ARG, "ds_crc32: device ordinal");
    std::call_once(flags[dev], [dev] {
        static uint32_t op128[257][32], opr[129][32], pw[32][32], tab[4][256];
        uint32_t one[32], two[32], byte1[32];
        one[0] = CRC_POLY;  // multiply by x: one zero bit
        for (int i = 1; i < 32; i++) one[i] = 1u << (i - 1);
        gf2_square(two, one);     // 2 bits
        gf2_square(one, two);     // 4 bits
        gf2_square(byte1, one);   // 8 bits = 1 byte
        for (int i = 0; i < 32; i++) opr[0][i] = 1u << i;
        for (int r = 1; r <= 128; r++) gf2_mul(opr[r], byte1, opr[r - 1]);
        for (int i = 0; i < 32; i++) op128[0][i] = 1u << i;
        for (int k = 1; k <= 256; k++) gf2_mul(op128[k], opr[128], op128[k - 1]);
        for (int i = 0; i < 32; i++) pw[0][i] = op128[256][i];  // 32 KB
        for (int b = 1; b < 32; b++) gf2_square(pw[b], pw[b - 1]);
        for (int b = 0; b < 256; b++) {
            uint32_t c = (uint32_t)b;
            for (int k = 0; k < 8; k++) c = c & 1u ? (c >> 1) ^ CRC_POLY : c >> 1;
            tab[0][b] = c;
        }
        for (int b = 0; b < 256; b++)
            for (int s = 1; s < 4; s++) tab[s][b] = (tab[s - 1][b] >> 8) ^ tab[0][tab[s - 1][b] & 255];
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(dev);
        cudaError_t e = cudaMemcpyToSymbol(g_op128, op128, sizeof(op128));
        if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_opr, opr, sizeof(opr));
        if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_pow, pw, sizeof(pw));
        if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_tab, tab, sizeof(tab));
        cudaSetDevice(cur);
        status[dev] = e == cudaSuccess ? DS_OK : host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
    });
    return status[dev];
}

}  // namespace

extern "C" size_t ds_crc32_workspace_size(int64_t n) {
    (void)n;
    return 256;  // reserved
}

extern "C" int ds_crc32(const uint8_t *data, int64_t n, uint32_t *out, void *workspace,
                        size_t workspace_bytes, void *stream) {
    if (!out || (n > 0 && !data)) return host::fail(DS_ERR_ARG, "ds_crc32: null pointer");
    if (n < 0) return host::fail(DS_ERR_ARG, "ds_crc32: negative length");
    cudaStream_t s = (cudaStream_t)stream;
    if (n == 0) {
        cudaMemsetAsync(out, 0, sizeof(uint32_t), s);  // crc32(b"") == 0
        return host::check_launch("ds_crc32");
    }
    (void)workspace_bytes;
    int dev = 0;
    cudaGetDevice(&dev);
    int st = crc_init(dev);
    if (st) return st;
    const int64_t nchunks = (n + CRC_CHUNK - 1) / CRC_CHUNK;
    (void)workspace;
    // every chunk xors its shifted term into *out
    cudaMemsetAsync(out, 0, sizeof(uint32_t), s);
    crc_chunk_kernel<<<(unsigned)nchunks, CRC_THREADS, 0, s>>>(data, n, out);
    return host::check_launch("ds_crc32");
}
