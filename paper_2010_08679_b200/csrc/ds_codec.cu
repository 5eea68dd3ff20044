// ds_codec.cu -- row-matrix codec entry points (the quant.py API mirror).
//
// quantize_rows / dequantize_rows / reconstruction_errors (quant.py:93-138),
// adaptive_params_rows (quant.py:160-209), pack_code_rows / unpack_code_rows
// (quant.py:376-395) and the naive row min/max (engine.py:163-164).  The
// checkpoint writer (ds_writer.cu) fuses these; these stand-alone kernels
// serve callers of the reference's quant module directly.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ds_common.cuh"
#include "ds_host.h"

namespace ds {

// one warp per row, VEC1 layout; d <= 1024
__global__ void minmax_kernel(const float *x, int64_t n, int d, float *mins, float *maxs) {
    int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (row >= n) return;
    const float *r = x + row * d;
    float mn = INFINITY, mx = -INFINITY;
    for (int e = lane; e < d; e += 32) {
        float v = r[e];
        mn = fminf(mn, v);
        mx = fmaxf(mx, v);
    }
    mn = grp_min<32>(mn);
    mx = grp_max<32>(mx);
    if (lane == 0) {
        mins[row] = mn;
        maxs[row] = mx;
    }
}

// element-wise quantize with per-row RowQ (certified fast path + exact fallback)
__global__ void quantize_kernel(const float *x, int64_t n, int d, const float *mins,
                                const float *maxs, int L, uint8_t *codes) {
    int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (row >= n) return;
    RowQ rq = make_rowq(mins[row], maxs[row], L);
    unsigned nex = 0;
    for (int e = lane; e < d; e += 32) codes[row * d + e] = (uint8_t)code_of(x[row * d + e], rq, nex);
}

__global__ void dequantize_kernel(const uint8_t *codes, int64_t n, int d, const float *mins,
                                  const float *maxs, int L, float *out, uint32_t *flags) {
    int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (row >= n) return;
    float lo = mins[row];
    double s = scale64(lo, maxs[row], L);
    bool bad = false;
    for (int e = lane; e < d; e += 32) {
        int q = codes[row * d + e];
        if (q > L) bad = true;  // quant.py:111-112
        out[row * d + e] = deq_exact(q, lo, s);
    }
    if (bad) atomicOr(flags, DS_FLAG_FORMAT);
}

// exact reconstruction error in numpy order; one warp per row, scratch in smem
constexpr int RE_WARPS = 4;
__global__ void recon_kernel(const float *x, int64_t n, int d, const float *mins,
                             const float *maxs, int L, double *out) {
    extern __shared__ double sh[];
    int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t row = (int64_t)blockIdx.x * RE_WARPS + w;
    double *buf = sh + (size_t)w * d;
    if (row < n) {
        float lo = mins[row], hi = maxs[row];
        RowQ rq = make_rowq(lo, hi, L);
        unsigned nex = 0;
        for (int e = lane; e < d; e += 32) {
            float xv = x[row * d + e];
            int q = code_of(xv, rq, nex);
            double err = __dsub_rn((double)xv, (double)deq_exact(q, lo, rq.s));
            buf[e] = __dmul_rn(err, err);
        }
    }
    __syncwarp();
    if (row < n && lane == 0) out[row] = __dsqrt_rn(pw_sum(buf, d));
}

template <int G, int C, int VEC, bool PAD>
__global__ void __launch_bounds__(256) adaptive_kernel(const float *x, int64_t n, int d, int L,
                                                       int bins, int steps, float *mins,
                                                       float *maxs, uint32_t *flags,
                                                       unsigned long long *stats) {
    using Lay = Layout<G, C, VEC>;
    constexpr int EPL = C * VEC;
    extern __shared__ double scratch[];
    const int lane = threadIdx.x & 31, lig = lane & (G - 1), slot = threadIdx.x / G;
    int64_t row = (int64_t)blockIdx.x * (256 / G) + slot;
    bool valid = row < n;
    float xv[EPL];
    if (valid) load_row<G, C, VEC>(x + row * d, d, lig, xv, 0.f);
    else
        for (int k = 0; k < EPL; k++) xv[k] = 0.f;
    bool fin = true;
    for (int k = 0; k < EPL; k++) fin = fin && isfinite(xv[k]);
    fin = grp_or<G>(fin ? 0 : 1) == 0;
    if (valid && !fin && lig == 0) atomicOr(flags, DS_FLAG_DATA);
    float mn = INFINITY, mx = -INFINITY;
    for (int k = 0; k < EPL; k++)
        if (Lay::elem(lig, k) < d) {
            mn = fminf(mn, xv[k]);
            mx = fmaxf(mx, xv[k]);
        }
    float lo = grp_min<G>(mn), hi = grp_max<G>(mx);
    bool ok = valid && fin;
    if (!ok) lo = hi = 0.f;
    unsigned nd = 0, nc = 0;
    greedy_row<G, C, VEC, PAD>(xv, d, lig, ok, lo, hi, L, bins, steps, scratch + slot * (d + 8), lo,
                               hi, nd, nc);
    if (valid && lig == 0) {
        mins[row] = lo;
        maxs[row] = hi;
    }
    if (stats && lig == 0 && (nd | nc)) {
        atomicAdd(stats + DS_STAT_EXACT_DECISIONS, (unsigned long long)nd);
        atomicAdd(stats + DS_STAT_EXACT_CODES, (unsigned long long)nc);
    }
}

// pack: one thread per output byte
__global__ void pack_kernel(const uint8_t *codes, int64_t n, int d, int N, int packed,
                            uint8_t *out, uint32_t *flags) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * packed) return;
    int64_t row = i / packed;
    int b = (int)(i - row * packed);
    const uint8_t *c = codes + row * d;
    int bit0 = 8 * b;
    int j0 = bit0 / N, j1 = min(d - 1, (bit0 + 7) / N);
    uint32_t v = 0;
    bool bad = false;
    for (int j = j0; j <= j1; j++) {
        uint32_t cv = c[j];
        if (cv >= (1u << N)) bad = true;  // quant.py:378-379
        int pos = j * N - bit0;
        v |= pos >= 0 ? (cv << pos) : (cv >> (-pos));
    }
    out[i] = (uint8_t)v;
    if (bad) atomicOr(flags, DS_FLAG_DATA);
}

// unpack: one thread per code; the last byte of a row checks the padding
__global__ void unpack_kernel(const uint8_t *packed_in, int64_t n, int d, int N, int packed,
                              uint8_t *out, uint32_t *flags) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * d) return;
    int64_t row = i / d;
    int e = (int)(i - row * d);
    const uint8_t *p = packed_in + row * packed;
    int bit = e * N;
    uint32_t w = p[bit >> 3];
    if ((bit >> 3) + 1 < packed) w |= (uint32_t)p[(bit >> 3) + 1] << 8;
    out[i] = (uint8_t)((w >> (bit & 7)) & ((1u << N) - 1));
    if (e == d - 1) {
        int padbits = 8 * packed - d * N;
        if (padbits > 0 && (p[packed - 1] >> (8 - padbits)) != 0) atomicOr(flags, DS_FLAG_FORMAT);
    }
}

}  // namespace ds

using namespace ds;

static bool valid_bw(int bw) { return bw == 2 || bw == 3 || bw == 4 || bw == 8; }

extern "C" int ds_row_minmax(const float *x, int64_t n, int64_t d, float *mins, float *maxs,
                             void *stream) {
    if (n <= 0) return DS_OK;
    if (d < 1) return host::fail(DS_ERR_DATA, "vector must be non-empty");
    int64_t blocks = (n * 32 + 255) / 256;
    minmax_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(x, n, (int)d, mins, maxs);
    return host::check_launch("ds_row_minmax");
}

extern "C" int ds_quantize_rows(const float *x, int64_t n, int64_t d, const float *mins,
                                const float *maxs, int bitwidth, uint8_t *codes, void *stream) {
    if (!valid_bw(bitwidth)) return host::fail(DS_ERR_CONFIG, "bitwidth must be one of (2, 3, 4, 8)");
    if (n <= 0 || d <= 0) return DS_OK;
    int64_t blocks = (n * 32 + 255) / 256;
    quantize_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(x, n, (int)d, mins, maxs,
                                                                      (1 << bitwidth) - 1, codes);
    return host::check_launch("ds_quantize_rows");
}

extern "C" int ds_dequantize_rows(const uint8_t *codes, int64_t n, int64_t d, const float *mins,
                                  const float *maxs, int bitwidth, float *out, uint32_t *flags,
                                  void *stream) {
    if (!valid_bw(bitwidth)) return host::fail(DS_ERR_CONFIG, "bitwidth must be one of (2, 3, 4, 8)");
    if (n <= 0 || d <= 0) return DS_OK;
    int64_t blocks = (n * 32 + 255) / 256;
    dequantize_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        codes, n, (int)d, mins, maxs, (1 << bitwidth) - 1, out, flags);
    return host::check_launch("ds_dequantize_rows");
}

extern "C" int ds_reconstruction_errors(const float *x, int64_t n, int64_t d, const float *mins,
                                        const float *maxs, int bitwidth, double *out,
                                        void *stream) {
    if (!valid_bw(bitwidth)) return host::fail(DS_ERR_CONFIG, "bitwidth must be one of (2, 3, 4, 8)");
    if (n <= 0) return DS_OK;
    if (d < 1 || d > 4096) return host::fail(DS_ERR_CONFIG, "reconstruction_errors: dim 1..4096");
    size_t smem = (size_t)RE_WARPS * d * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(recon_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
    int64_t blocks = (n + RE_WARPS - 1) / RE_WARPS;
    recon_kernel<<<(unsigned)blocks, 32 * RE_WARPS, smem, (cudaStream_t)stream>>>(
        x, n, (int)d, mins, maxs, (1 << bitwidth) - 1, out);
    return host::check_launch("ds_reconstruction_errors");
}

typedef void (*adaptive_fn)(const float *, int64_t, int, int, int, int, float *, float *,
                            uint32_t *, unsigned long long *);

template <bool PAD>
static adaptive_fn pick_adaptive(int G, int C, int VEC) {
#define DS_A(G_, C_, V_) \
    if (G == G_ && C == C_ && VEC == V_) return adaptive_kernel<G_, C_, V_, PAD>;
    DS_A(1, 1, 4) DS_A(2, 1, 4) DS_A(4, 1, 4) DS_A(8, 1, 4) DS_A(16, 1, 4) DS_A(32, 1, 4)
    DS_A(32, 2, 4) DS_A(32, 4, 4) DS_A(32, 8, 4)
    DS_A(1, 1, 1) DS_A(2, 1, 1) DS_A(4, 1, 1) DS_A(8, 1, 1) DS_A(16, 1, 1) DS_A(32, 1, 1)
    DS_A(32, 2, 1) DS_A(32, 4, 1) DS_A(32, 8, 1) DS_A(32, 16, 1) DS_A(32, 32, 1)
#undef DS_A
    return nullptr;
}

extern "C" int ds_adaptive_params_rows(const float *x, int64_t n, int64_t d, int bitwidth,
                                       int num_bins, int steps, float *mins, float *maxs,
                                       uint32_t *flags, unsigned long long *stats, void *stream) {
    if (!valid_bw(bitwidth)) return host::fail(DS_ERR_CONFIG, "bitwidth must be one of (2, 3, 4, 8)");
    if (num_bins < 1) return host::fail(DS_ERR_CONFIG, "num_bins must be >= 1");
    if (n <= 0) return DS_OK;
    if (d < 1 || d > 1024) return host::fail(DS_ERR_CONFIG, "adaptive_params_rows: dim 1..1024");
    bool vec4 = d % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    int G = 1, C, VEC;
    if (vec4) {
        int chunks = (int)d / 4;
        VEC = 4;
        while (G < chunks && G < 32) G <<= 1;
        C = (chunks + G - 1) / G;
    } else {
        VEC = 1;
        while (G < d && G < 32) G <<= 1;
        C = ((int)d + G - 1) / G;
    }
    int cc = 1;
    while (cc < C) cc <<= 1;
    C = cc;
    bool pad = (VEC == 4 ? 4 * G * C : G * C) != d;
    adaptive_fn fn = pad ? pick_adaptive<true>(G, C, VEC) : pick_adaptive<false>(G, C, VEC);
    if (!fn) return host::fail(DS_ERR_CONFIG, "adaptive_params_rows: no kernel for this dim");
    int rpb = 256 / G;
    size_t smem = (size_t)rpb * (d + 8) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
    int64_t blocks = (n + rpb - 1) / rpb;
    fn<<<(unsigned)blocks, 256, smem, (cudaStream_t)stream>>>(x, n, (int)d, (1 << bitwidth) - 1,
                                                               num_bins, steps, mins, maxs, flags,
                                                               stats);
    return host::check_launch("ds_adaptive_params_rows");
}

extern "C" int ds_pack_code_rows(const uint8_t *codes, int64_t n, int64_t d, int bitwidth,
                                 uint8_t *out, uint32_t *flags, void *stream) {
    if (!valid_bw(bitwidth)) return host::fail(DS_ERR_CONFIG, "bitwidth must be one of (2, 3, 4, 8)");
    int packed = (int)((d * bitwidth + 7) / 8);
    int64_t tot = n * packed;
    if (tot <= 0) return DS_OK;
    pack_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        codes, n, (int)d, bitwidth, packed, out, flags);
    return host::check_launch("ds_pack_code_rows");
}

extern "C" int ds_unpack_code_rows(const uint8_t *packed_in, int64_t n, int64_t d, int bitwidth,
                                   uint8_t *out, uint32_t *flags, void *stream) {
    if (!valid_bw(bitwidth)) return host::fail(DS_ERR_CONFIG, "bitwidth must be one of (2, 3, 4, 8)");
    int packed = (int)((d * bitwidth + 7) / 8);
    int64_t tot = n * d;
    if (tot <= 0) return DS_OK;
    unpack_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        packed_in, n, (int)d, bitwidth, packed, out, flags);
    return host::check_launch("ds_unpack_code_rows");
}
