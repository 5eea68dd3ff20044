// ds_tracker.cu -- K0 bitmap maintenance, K1 mark, K2 capture/compaction.
//
// Reference: deltasnap/tracker.py:19-139.  The bitmap of a table is a run of
// uint32 little-endian words (bit r -> word r>>5, bit r&31), byte-identical to
// the reference's uint8 bitset (tracker.py:25,36).
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

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
    const void *idx;
    int idx32;  // 1: int32 ids, 0: int64 ids
    uint32_t *flags;
    int64_t word_off[DS_MAX_TABLES];
    int64_t rows[DS_MAX_TABLES];
    int64_t seg_off[DS_MAX_TABLES + 1];
    int32_t seg_table[DS_MAX_TABLES];
    int blk_off[DS_MAX_TABLES + 1];  // TMA kernel: first CTA of the j-th segment of seg_order
    int32_t seg_order[DS_MAX_TABLES];  // TMA kernel: segments, most expensive kind first
    int64_t seg_pb[DS_MAX_TABLES];     // TMA kernel: lookups per CTA of each segment
    const uint8_t *ibytes;             // TMA kernel: packed lookup stream
    int64_t seg_boff[DS_MAX_TABLES];   // TMA kernel: byte offset of each segment (16-aligned)
    int64_t seg_n[DS_MAX_TABLES];      // TMA kernel: ids in each segment
    int32_t seg_width[DS_MAX_TABLES];  // TMA kernel: bits per id (4..28 packed, 8/16 unsigned; 32/64 signed)
    int nseg;
};

// Each CTA marks one contiguous range of the lookup stream (so it sees a
// table's Zipf head over and over), 8 ids per thread per iteration from
// 128-bit loads.  A direct-mapped shared-memory cache remembers bitmap words
// whose bits this CTA already knows to be set: a repeat of a hot row costs a
// shared-memory probe instead of an L2 round trip to one contended word.
// Cache entries are (word+1) << 32 | known_bits written with one 64-bit store,
// so a racing update can only lose knowledge, never invent a set bit.
constexpr int MARK_THREADS = 256;
constexpr int MARK_PER_THREAD = 8;
constexpr int MARK_CACHE = 1024;  // entries (8 KB)

template <typename IdxT>
__device__ __forceinline__ void load8(const IdxT *p, int64_t i, int64_t end, bool vec,
                                      int64_t (&r)[MARK_PER_THREAD]) {
    if (vec && i + MARK_PER_THREAD <= end) {
        if (sizeof(IdxT) == 4) {
            const int4 *q = reinterpret_cast<const int4 *>(p + i);
            int4 u = __ldcs(q), v = __ldcs(q + 1);  // streamed once
            r[0] = u.x; r[1] = u.y; r[2] = u.z; r[3] = u.w;
            r[4] = v.x; r[5] = v.y; r[6] = v.z; r[7] = v.w;
        } else {
            const longlong2 *q = reinterpret_cast<const longlong2 *>(p + i);
#pragma unroll
            for (int k = 0; k < 4; k++) {
                longlong2 u = __ldcs(q + k);
                r[2 * k] = u.x;
                r[2 * k + 1] = u.y;
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < MARK_PER_THREAD; k++)
            r[k] = i + k < end ? (int64_t)__ldcs(p + i + k) : -1;
    }
}

template <typename IdxT>
__global__ void __launch_bounds__(MARK_THREADS) mark_kernel(const MarkArgs a, int64_t per_block,
                                                           int vec, int use_cache) {
    __shared__ int64_t s_seg_off[DS_MAX_TABLES + 1];
    __shared__ int64_t s_base[DS_MAX_TABLES];
    __shared__ int64_t s_rows[DS_MAX_TABLES];
    __shared__ unsigned long long cache[MARK_CACHE];
    for (int s = threadIdx.x; s <= a.nseg; s += blockDim.x) {
        s_seg_off[s] = a.seg_off[s];
        if (s < a.nseg) {
            s_base[s] = a.word_off[a.seg_table[s]];
            s_rows[s] = a.rows[a.seg_table[s]];
        }
    }
    for (int k = threadIdx.x; k < MARK_CACHE; k += blockDim.x) cache[k] = 0ull;
    __syncthreads();
    const IdxT *idx = static_cast<const IdxT *>(a.idx);
    const int64_t total = s_seg_off[a.nseg];
    const int64_t start = s_seg_off[0] + (int64_t)blockIdx.x * per_block;
    const int64_t end = min(total, start + per_block);
    bool bad = false;
    int seg = 0;
    for (int64_t i = start + (int64_t)threadIdx.x * MARK_PER_THREAD; i < end;
         i += (int64_t)MARK_THREADS * MARK_PER_THREAD) {
        int64_t r[MARK_PER_THREAD];
        load8<IdxT>(idx, i, end, vec, r);
        while (i >= s_seg_off[seg + 1]) seg++;  // ranges only move forward
        // word ids fit 32 bits (checked on the host); the 8 ids usually share
        // one segment, else fall back to a per-id segment walk
        const bool one_seg = i + MARK_PER_THREAD <= s_seg_off[seg + 1] && i + MARK_PER_THREAD <= end;
        uint32_t w[MARK_PER_THREAD], bit[MARK_PER_THREAD], old[MARK_PER_THREAD];
        uint32_t slot[MARK_PER_THREAD];
        bool need[MARK_PER_THREAD];
        if (one_seg) {
            const uint32_t base = (uint32_t)s_base[seg];
            const uint64_t rows = (uint64_t)s_rows[seg];
#pragma unroll
            for (int k = 0; k < MARK_PER_THREAD; k++) {
                need[k] = (uint64_t)r[k] < rows;  // negative ids wrap to huge
                bad |= !need[k];
                uint32_t u = (uint32_t)r[k];
                w[k] = base + (u >> 5);
                bit[k] = 1u << (u & 31);
                slot[k] = (w[k] * 2654435761u) >> (32 - 10);
            }
        } else {
            int sg = seg;
#pragma unroll
            for (int k = 0; k < MARK_PER_THREAD; k++) {
                need[k] = false;
                w[k] = bit[k] = slot[k] = 0;
                if (i + k >= end) continue;
                while (i + k >= s_seg_off[sg + 1]) sg++;
                if ((uint64_t)r[k] >= (uint64_t)s_rows[sg]) {
                    bad = true;
                    continue;
                }
                uint32_t u = (uint32_t)r[k];
                w[k] = (uint32_t)s_base[sg] + (u >> 5);
                bit[k] = 1u << (u & 31);
                slot[k] = (w[k] * 2654435761u) >> (32 - 10);
                need[k] = true;
            }
        }
        if (use_cache) {
#pragma unroll
            for (int k = 0; k < MARK_PER_THREAD; k++) {
                unsigned long long e = cache[slot[k]];
                // this CTA already knows the bit is set
                if ((uint32_t)(e >> 32) == w[k] + 1 && ((uint32_t)e & bit[k])) need[k] = false;
            }
        }
        // all L2 probes in flight together, then the atomics
#pragma unroll
        for (int k = 0; k < MARK_PER_THREAD; k++) old[k] = need[k] ? __ldcg(a.words + w[k]) : 0u;
#pragma unroll
        for (int k = 0; k < MARK_PER_THREAD; k++) {
            if (!need[k]) continue;
            if (!(old[k] & bit[k])) atomicOr(a.words + w[k], bit[k]);
            if (use_cache)
                cache[slot[k]] = ((unsigned long long)(w[k] + 1) << 32) | (old[k] | bit[k]);
        }
    }
    if (__any_sync(DS_FULL_MASK, bad) && (threadIdx.x & 31) == 0) atomicOr(a.flags, DS_FLAG_BOUNDS);
}

// ---------------------------------------------------------------------------
// K1, TMA form: the lookup stream is pulled into shared memory by the Tensor
// Memory Accelerator (cp.async.bulk, 16 KB per stage, 4 stages, mbarrier
// completion), so the HBM stream needs no registers and no issue slots.
// Threads probe a direct-mapped shared cache of (word, bits known set); a miss
// issues a fire-and-forget RED.OR (no dependent L2 round trip) and records the
// bit.  Correct for any interleaving: bits are only ever set, and a cache
// entry only claims bits this CTA has itself OR-ed (or seen OR-ed) into HBM.
// ---------------------------------------------------------------------------
#ifndef DS_MK_CACHE_BITS
#define DS_MK_CACHE_BITS 13
#endif
#ifndef DS_MK_GRP_ROLLED
#define DS_MK_GRP_ROLLED 0  // 1: packed id groups in a rolled loop (smaller code, A/B)
#endif
#ifndef DS_MK_WIN_SEQ
#define DS_MK_WIN_SEQ 0  // 1: bit-window ids tested one at a time (A/B)
#endif
#ifndef DS_MK_PG
// cache probes batched per lane (mode 2).  1 measured best (C2 K1 60 -> 48
// µs): a batch reads its slots before updating them, so a repeated hot row
// inside a batch sees a stale entry and issues a redundant RED
#define DS_MK_PG 1
#endif
constexpr int MK_CACHE_BITS = DS_MK_CACHE_BITS;  // 2^13 entries = 64 KB (A/B: DS_MK_CACHE_BITS)

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, unsigned bytes,
                                            unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Every CTA works inside ONE segment (one table's slice of the lookup
// stream) and each of its warps runs its own TMA ring over every 8th chunk of
// the CTA's range (no CTA barrier in the loop).  Per table size, in a 64 KB
// shared region:
//  * rows <= MK_BYTE_ROWS (65,504; all 18 small Criteo-Kaggle tables): a
//    shared byte per row; a lookup is one plain byte store (racing stores all
//    write 1, so no atomics and no read), folded into bitmap words and OR-ed
//    into HBM once per CTA at the end;
//  * rows <= 32 * MK_WIN_WORDS (524,288): a shared copy of the bitmap words
//    (read-before-ATOMS: hot words are already set and same-address reads
//    broadcast), flushed with one RED per touched word;
//  * larger: a shared cache of (word, bits known set) with second-chance
//    replacement (8,192 entries); a miss issues one fire-and-forget RED.OR.
// Correct for any interleaving: bits are only ever set, and a cache entry
// only claims bits this CTA itself OR-ed into HBM.
constexpr int MK_CACHE_BYTES = (1 << MK_CACHE_BITS) * 8;
constexpr int MK_WIN_WORDS = MK_CACHE_BYTES / 8 < 2048 ? MK_CACHE_BYTES / 8 : MK_CACHE_BYTES / 4;  // window words
constexpr int MK_BYTE_ROWS = MK_CACHE_BYTES - 32;  // byte map + one dummy byte in the cache region
constexpr int MK_WSTAGES = 4;        // per-warp ring depth
constexpr int MK_WSTAGE_BYTES = 1024;  // per-warp stage: 256 int32 / 128 int64 ids
constexpr int MK_WARPS = MARK_THREADS / 32;

// ids bit-packed at a segment-specific width (LSB-first bitstream)
struct BitPacked {};

// One CTA's range [start, end) of segment `seg`: typed ids (uint8_t,
// uint16_t, int32_t, int64_t) or BitPacked ids of a.seg_width[seg] bits.
template <typename IdxT, int WB = 0>
__device__ __forceinline__ void mark_range(const MarkArgs &a, int seg, int64_t start, int64_t end,
                                           unsigned long long *cache,
                                           unsigned long long (*bars)[MK_WSTAGES], uint8_t *mk_smem) {
    constexpr bool BITS = std::is_same<IdxT, BitPacked>::value;
    static_assert(!BITS || (WB >= 4 && WB <= 28 && WB % 4 == 0), "packed widths: 4..28 bits, step 4");
    using T = typename std::conditional<BITS, uint32_t, IdxT>::type;  // element type of a lane's ids
    // ids per warp stage: 32 B of typed ids per lane, 8 bit-packed ids per lane
    // (packed: 16 ids per lane while a stage of 512 fits the 1 KB ring slot)
    constexpr int IDS = BITS ? (WB <= 16 ? 512 : 256) : MK_WSTAGE_BYTES / (int)sizeof(T);
    constexpr int PER_LANE = IDS / 32;
    constexpr int wbits = BITS ? WB : 8 * (int)sizeof(T);  // bits per id
    constexpr uint32_t wmask = wbits >= 32 ? 0xffffffffu : (1u << wbits) - 1u;
    uint32_t *win = reinterpret_cast<uint32_t *>(cache);  // bit window (aliases the cache)
    uint8_t *bytes = reinterpret_cast<uint8_t *>(cache);  // byte map (aliases the cache)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t base = (uint32_t)a.word_off[seg];
    const uint64_t rows = (uint64_t)a.rows[seg];
    const uint32_t nwords = (uint32_t)((rows + 31) / 32);
    // 32-bit bound for the byte map (int32 ids never exceed 2^31 - 1)
    const uint32_t rows32 = (uint32_t)min(rows, (uint64_t)0x80000000ull);
    auto in_range = [&](T v) -> bool {  // negatives wrap high
        if (sizeof(T) <= 4) return (uint32_t)v < rows32;
        return (uint64_t)(int64_t)v < rows;
    };
    const int mode = rows <= (uint64_t)MK_BYTE_ROWS ? 0 : (nwords <= (uint32_t)MK_WIN_WORDS ? 1 : 2);
    for (int k = threadIdx.x; k < (1 << MK_CACHE_BITS); k += MARK_THREADS) cache[k] = 0ull;
    const uint8_t *sbytes = a.ibytes + a.seg_boff[seg];
    const T *idx = reinterpret_cast<const T *>(sbytes);
    // a stage holds IDS ids: sizeof(T) * IDS bytes, or 32 * wbits bytes packed
    uint8_t *ring = mk_smem + (size_t)wid * MK_WSTAGES * MK_WSTAGE_BYTES;
    unsigned long long *wb = bars[wid];
    // TMA moves whole 16-byte units: typed ids leave a ragged tail (< 16 B)
    // read directly; packed segments are padded to 16 bytes, so their last
    // chunk is copied whole
    const int64_t bulk_end =
        BITS ? end : start + ((end - start) * (int64_t)sizeof(T) / 16) * 16 / (int64_t)sizeof(T);
    const int nch = (int)((bulk_end - start + IDS - 1) / IDS);
    if (lane == 0) {
        for (int s = 0; s < MK_WSTAGES; s++) mbar_init(&wb[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();  // cache/map zeroed, barriers initialised
    auto issue = [&](int k) {  // lane 0: chunk wid + 8k into stage k % STAGES
        const int c = wid + k * MK_WARPS;
        if (c < nch) {
            const int64_t c0 = start + (int64_t)c * IDS;
            const int64_t n = min((int64_t)IDS, bulk_end - c0);
            const uint8_t *src;
            unsigned nb;
            if (BITS) {  // c0 is a multiple of 256 ids: a whole number of 16-byte units
                src = sbytes + ((uint64_t)c0 >> 3) * wbits;
                nb = (((unsigned)n * wbits + 7u) >> 3) + 15u & ~15u;
            } else {
                src = reinterpret_cast<const uint8_t *>(idx + c0);
                nb = (unsigned)(n * sizeof(T));
            }
            mbar_expect_tx(&wb[k % MK_WSTAGES], nb);
            tma_load_1d(ring + (size_t)(k % MK_WSTAGES) * MK_WSTAGE_BYTES, src, nb, &wb[k % MK_WSTAGES]);
        }
    };
    if (lane == 0)
        for (int k = 0; k < MK_WSTAGES; k++) issue(k);
    bool bad = false;
    // Cache entry: key (word+1, 31 bits) << 33 | referenced << 32 | bits known
    // set.  Second-chance replacement keeps the Zipf head cached.
    auto cache_mark = [&](uint32_t w, uint32_t bit, uint32_t slot, unsigned long long e) {
        const bool match = (uint32_t)(e >> 33) == w + 1;
        const uint32_t known = match ? (uint32_t)e : 0u;
        if (known & bit) {
            if (!(e & (1ull << 32))) cache[slot] = e | (1ull << 32);  // referenced
            return;
        }
        atomicOr(a.words + w, bit);  // result unused -> RED, no round trip
        if (match) cache[slot] = e | bit | (1ull << 32);
        else if (e & (1ull << 32)) cache[slot] = e & ~(1ull << 32);  // second chance
        else cache[slot] = ((unsigned long long)(w + 1) << 33) | bit;
    };
    auto mark_row = [&](uint32_t u) {
        if (mode == 0) {
            bytes[u] = 1;
        } else if (mode == 1) {
            atomicOr(win + (u >> 5), 1u << (u & 31));  // shared-memory OR
        } else {
            const uint32_t w = base + (u >> 5);
            const uint32_t slot = (w * 2654435761u) >> (32 - MK_CACHE_BITS);
            cache_mark(w, 1u << (u & 31), slot, cache[slot]);
        }
    };
    // id q of a bit-packed stage (words of the stage; may read one word past)
    auto unpack = [&](const uint32_t *wds, int q) -> uint32_t {
        const int p = q * wbits;
        return __funnelshift_r(wds[p >> 5], wds[(p >> 5) + 1], p & 31) & wmask;
    };
    // the lane's 8 ids: the width is a multiple of 4 bits, so the lane's
    // 8*w bits are w/4 whole words; every shift is a compile-time constant
    auto unpack8 = [&](const uint32_t *wds, int grp, uint32_t (&v)[8]) {
        constexpr int NW = wbits / 4;  // words per 8 ids
        const uint32_t *lw = wds + (lane * (PER_LANE / 8) + grp) * NW;
        uint32_t wd[NW + 1];
#pragma unroll
        for (int k = 0; k < NW; k++) wd[k] = lw[k];
        wd[NW] = 0u;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int bit = q * wbits;  // constant after unrolling
            v[q] = __funnelshift_r(wd[bit >> 5], wd[(bit >> 5) + 1], bit & 31) & wmask;
        }
    };
    // a group of NQ ids of this lane, all of the current segment
    auto mark_group = [&](auto &v) {
        constexpr int NQ = sizeof(v) / sizeof(v[0]);
        if (mode == 0) {
            // out-of-range ids store to the dummy byte at index `rows`
            // (masked off by the flush) instead of branching
            const uint32_t sb = smem_u32(bytes);
            if (sizeof(T) <= 4) {
                uint32_t umax = 0;  // negatives wrap high
#pragma unroll
                for (int q = 0; q < NQ; q++) {
                    const uint32_t u = (uint32_t)v[q];
                    umax = max(umax, u);
                    asm volatile("st.shared.u8 [%0], %1;" ::"r"(sb + min(u, rows32)), "r"(1) : "memory");
                }
                bad |= umax >= rows32;
            } else {
#pragma unroll
                for (int q = 0; q < NQ; q++) {
                    const bool ok = in_range(v[q]);
                    bad |= !ok;
                    asm volatile("st.shared.u8 [%0], %1;" ::"r"(sb + (ok ? (uint32_t)v[q] : rows32)),
                                 "r"(1) : "memory");
                }
            }
        } else if (mode == 1 && DS_MK_WIN_SEQ) {
            // one id at a time: each test sees the bits the previous ids set
#pragma unroll
            for (int q = 0; q < NQ; q++) {
                const bool ok = in_range(v[q]);
                bad |= !ok;
                const uint32_t bit = 1u << ((uint32_t)v[q] & 31);
                if (ok && !(win[(uint32_t)v[q] >> 5] & bit)) atomicOr(win + ((uint32_t)v[q] >> 5), bit);
            }
        } else if (mode == 1) {
            uint32_t cur[NQ];
            bool ok[NQ];
#pragma unroll
            for (int q = 0; q < NQ; q++) {
                ok[q] = in_range(v[q]);
                bad |= !ok[q];
                cur[q] = ok[q] ? win[(uint32_t)v[q] >> 5] : ~0u;
            }
#pragma unroll
            for (int q = 0; q < NQ; q++) {
                const uint32_t bit = 1u << ((uint32_t)v[q] & 31);
                if (!(cur[q] & bit)) atomicOr(win + ((uint32_t)v[q] >> 5), bit);
            }
        } else {
            // probes in groups of DS_MK_PG (1: each probe sees the previous update)
            constexpr int PG = NQ < DS_MK_PG ? NQ : DS_MK_PG;
#pragma unroll
            for (int g = 0; g < NQ; g += PG) {
                uint32_t w[PG], slot[PG];
                unsigned long long e[PG];
                bool ok[PG];
#pragma unroll
                for (int q = 0; q < PG; q++) {
                    ok[q] = in_range(v[g + q]);
                    bad |= !ok[q];
                    w[q] = base + ((uint32_t)v[g + q] >> 5);
                    slot[q] = (w[q] * 2654435761u) >> (32 - MK_CACHE_BITS);
                    e[q] = cache[slot[q]];
                }
#pragma unroll
                for (int q = 0; q < PG; q++)
                    if (ok[q]) cache_mark(w[q], 1u << ((uint32_t)v[g + q] & 31), slot[q], e[q]);
            }
        }
    };
    for (int k = 0;; k++) {
        const int c = wid + k * MK_WARPS;
        if (c >= nch) break;
        const int s = k % MK_WSTAGES;
        mbar_wait(&wb[s], (unsigned)(k / MK_WSTAGES) & 1u);
        const int64_t c0 = start + (int64_t)c * IDS;
        const int cnt = (int)min((int64_t)IDS, bulk_end - c0);
        const uint8_t *stg = ring + (size_t)s * MK_WSTAGE_BYTES;
        const int j0 = lane * PER_LANE;
        if (j0 + PER_LANE <= cnt) {
            if constexpr (BITS) {
                static_assert(PER_LANE % 8 == 0, "groups of 8 packed ids per lane");
#if DS_MK_GRP_ROLLED
#pragma unroll 1
#else
#pragma unroll
#endif
                for (int grp = 0; grp < PER_LANE / 8; grp++) {
                    uint32_t v[8];
                    unpack8(reinterpret_cast<const uint32_t *>(stg), grp, v);
                    mark_group(v);
                }
            } else {
                // two 16-byte halves per lane (keeps the live ids few)
                constexpr int PH = PER_LANE / 2;
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    T v[PH];
                    *reinterpret_cast<int4 *>(v) =
                        reinterpret_cast<const int4 *>(reinterpret_cast<const T *>(stg) + j0)[h];
                    mark_group(v);
                }
            }
        } else {
            for (int q = j0; q < cnt && q < j0 + PER_LANE; q++) {
                int64_t r;
                if constexpr (BITS) r = unpack(reinterpret_cast<const uint32_t *>(stg), q);
                else r = (int64_t)reinterpret_cast<const T *>(stg)[q];
                if ((uint64_t)r >= rows) bad = true;
                else mark_row((uint32_t)r);
            }
        }
        __syncwarp();  // every lane is done with stage s
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(k + MK_WSTAGES);
        }
    }
    // ragged tail (typed ids only)
    if constexpr (!BITS) {
        for (int64_t i = bulk_end + threadIdx.x; i < end; i += MARK_THREADS) {
            const int64_t r = (int64_t)idx[i];
            if ((uint64_t)r >= rows) bad = true;
            else mark_row((uint32_t)r);
        }
    }
    if (mode != 2) {
        __syncthreads();
        if (mode == 0) {  // byte map -> bitmap words: 32 bytes (0/1) per word
            for (uint32_t k = threadIdx.x; k < nwords; k += MARK_THREADS) {
                const uint4 *p = reinterpret_cast<const uint4 *>(bytes + 32 * k);
                const uint4 u0 = p[0], u1 = p[1];
                const uint32_t c8[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
                uint32_t v = 0;
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const uint32_t c = c8[q];
                    v |= ((c & 1u) | ((c >> 7) & 2u) | ((c >> 14) & 4u) | ((c >> 21) & 8u)) << (4 * q);
                }
                if (k == nwords - 1 && (rows & 31)) v &= (1u << (rows & 31)) - 1u;  // dummy byte
                if (v) atomicOr(a.words + base + k, v);
            }
        } else {
            for (uint32_t k = threadIdx.x; k < nwords; k += MARK_THREADS) {
                const uint32_t v = win[k];
                if (v) atomicOr(a.words + base + k, v);
            }
        }
    }
    if (__any_sync(DS_FULL_MASK, bad) && lane == 0) atomicOr(a.flags, DS_FLAG_BOUNDS);
}

// Segments of ids bit-packed at 4..28 bits (8 and 16: plain u8 / u16) or
// 32 / 64-bit signed ids: the host sends each table's lookups at the width
// its row count needs, which is what bounds the end-to-end H2D of the lookup
// stream.
__global__ void __launch_bounds__(MARK_THREADS) mark_tma_kernel(const MarkArgs a) {
    pdl_trigger();  // K2 may launch once every K1 CTA is resident
    extern __shared__ __align__(128) uint8_t mk_smem[];
    __shared__ __align__(8) unsigned long long bars[MK_WARPS][MK_WSTAGES];
    // dynamic shared memory: [per-warp TMA rings][cache | bit window | byte map]
    unsigned long long *cache = reinterpret_cast<unsigned long long *>(
        mk_smem + (size_t)MK_WARPS * MK_WSTAGES * MK_WSTAGE_BYTES);
    static_assert(MK_WIN_WORDS * 4 <= MK_CACHE_BYTES, "window must fit the cache");
    static_assert(MK_BYTE_ROWS + 32 <= MK_CACHE_BYTES, "byte map must fit the cache");
    int j = 0;  // position in seg_order: last j with blk_off[j] <= blockIdx.x
    while (j + 1 < a.nseg && a.blk_off[j + 1] <= (int)blockIdx.x) j++;
    const int seg = a.seg_order[j];
    const int64_t start = (int64_t)(blockIdx.x - a.blk_off[j]) * a.seg_pb[seg];
    const int64_t end = min(a.seg_n[seg], start + a.seg_pb[seg]);
    switch (a.seg_width[seg]) {
    case 8: mark_range<uint8_t>(a, seg, start, end, cache, bars, mk_smem); break;
    case 16: mark_range<uint16_t>(a, seg, start, end, cache, bars, mk_smem); break;
    case 32: mark_range<int32_t>(a, seg, start, end, cache, bars, mk_smem); break;
    case 64: mark_range<int64_t>(a, seg, start, end, cache, bars, mk_smem); break;
    case 4: mark_range<BitPacked, 4>(a, seg, start, end, cache, bars, mk_smem); break;
    case 12: mark_range<BitPacked, 12>(a, seg, start, end, cache, bars, mk_smem); break;
    case 20: mark_range<BitPacked, 20>(a, seg, start, end, cache, bars, mk_smem); break;
    case 24: mark_range<BitPacked, 24>(a, seg, start, end, cache, bars, mk_smem); break;
    default: mark_range<BitPacked, 28>(a, seg, start, end, cache, bars, mk_smem); break;
    }
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

constexpr int CF_THREADS = 256;
#ifndef DS_C3_WPT
#define DS_C3_WPT 1
#endif

// ---------------------------------------------------------------------------
// K2 as count (+ scan by the last CTA) -> emit over chunks of 1024 words (4
// consecutive words per thread, 32768 rows: short, balanced CTAs).  The emit
// pass knows every chunk's base, so no CTA waits on another (a decoupled
// look-back single pass serialises through chunk order and measured slower).
// ---------------------------------------------------------------------------
constexpr int C3_WPT = DS_C3_WPT;
constexpr int C3_WPB = CF_THREADS * C3_WPT;

struct Cap3Args {
    uint32_t *interval;
    uint32_t *baseline;  // may be null
    int64_t *ids_int;
    int64_t *ids_uni;
    int64_t *counts;
    unsigned long long *cnt;    // [nchunks] packed (union << 32 | interval)
    unsigned long long *super;  // [nchunks / 256 + 1] sums of 256 chunks (left at 0)
    unsigned *ticket;           // emit CTAs done (the last one clears super; left at 0)
    int64_t word_off[DS_MAX_TABLES + 1];
    int64_t chunk_off[DS_MAX_TABLES + 1];
    int ntables;
    int nchunks;
    int fold;
};

// table of chunk c: binary search over the kernel parameters (every thread,
// no barrier)
__device__ __forceinline__ int cap3_table(const Cap3Args &a, int c) {
    int lo = 0, hi = a.ntables - 1;  // last t with chunk_off[t] <= c
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.chunk_off[mid] <= c) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// the thread's C3_WPT words of chunk c: one 16-byte load when the table's
// words start 16-byte aligned (ModelTracker pads every table to 4 words)
__device__ __forceinline__ void cap3_load(const Cap3Args &a, int c, int t, uint32_t (&iv)[C3_WPT],
                                          uint32_t (&uv)[C3_WPT], int64_t &w0, int64_t &wend) {
    w0 = a.word_off[t] + (int64_t)(c - a.chunk_off[t]) * C3_WPB + threadIdx.x * C3_WPT;
    wend = a.word_off[t + 1];
    if constexpr (C3_WPT == 4) {
        if ((w0 & 3) == 0 && w0 + 4 <= wend) {
            const uint4 i4 = __ldcg(reinterpret_cast<const uint4 *>(a.interval + w0));
            uint4 b4 = make_uint4(0u, 0u, 0u, 0u);
            if (a.baseline) b4 = __ldcg(reinterpret_cast<const uint4 *>(a.baseline + w0));
            iv[0] = i4.x; iv[1] = i4.y; iv[2] = i4.z; iv[3] = i4.w;
            uv[0] = i4.x | b4.x; uv[1] = i4.y | b4.y; uv[2] = i4.z | b4.z; uv[3] = i4.w | b4.w;
            return;
        }
    }
#pragma unroll
    for (int k = 0; k < C3_WPT; k++) {
        const int64_t w = w0 + k;
        iv[k] = w < wend ? __ldcg(a.interval + w) : 0u;
        const uint32_t bv = (w < wend && a.baseline) ? __ldcg(a.baseline + w) : 0u;
        uv[k] = iv[k] | bv;
    }
}

// CTA-wide sum (every thread gets it); s_red holds CF_THREADS/32 values
__device__ __forceinline__ unsigned long long cap3_block_sum(unsigned long long v,
                                                             unsigned long long *s_red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(DS_FULL_MASK, v, o);
    __syncthreads();  // s_red may still be read by a previous call
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
    __syncthreads();
    unsigned long long s = 0;
#pragma unroll
    for (int k = 0; k < CF_THREADS / 32; k++) s += s_red[k];
    return s;
}

// pass 1: per-chunk popcounts, and their 256-chunk group sums
__global__ void __launch_bounds__(CF_THREADS) cap3_count_kernel(const Cap3Args a) {
    pdl_trigger();
    pdl_wait();  // K1's bits
    __shared__ unsigned long long s_red[CF_THREADS / 32];
    const int c = blockIdx.x, t = cap3_table(a, c);
    uint32_t iv[C3_WPT], uv[C3_WPT];
    int64_t w0, wend;
    cap3_load(a, c, t, iv, uv, w0, wend);
    unsigned long long v = 0;
#pragma unroll
    for (int k = 0; k < C3_WPT; k++)
        v += (unsigned long long)__popc(iv[k]) | ((unsigned long long)__popc(uv[k]) << 32);
    const unsigned long long s = cap3_block_sum(v, s_red);
    if (threadIdx.x == 0) {
        a.cnt[c] = s;
        atomicAdd(a.super + (c >> 8), s);
    }
}

constexpr unsigned CAP3_STAGE = C3_WPB * 32;  // every id of a chunk fits the stage
static_assert(CAP3_STAGE * 4 <= 48 * 1024, "stage must fit static shared memory");

// pass 2: the chunk's base from the group sums, its sorted ids (staged in
// shared memory, coalesced int64 stores), the per-table counts (by each
// table's last chunk), then the fold.  Two CTA barriers: one reduction that
// yields the thread's scan offset, the chunk's base and (last chunks) the
// table's start together, and one before the staged ids leave.
__global__ void __launch_bounds__(CF_THREADS) cap3_emit_kernel(const Cap3Args a) {
    pdl_trigger();
    pdl_wait();  // the count pass's chunk and group sums
    constexpr int NWP = CF_THREADS / 32;
    __shared__ unsigned long long s_cnt[NWP], s_base[NWP], s_start[NWP];
    __shared__ uint32_t s_ids[CAP3_STAGE];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = blockIdx.x;
    const int t = __shfl_sync(DS_FULL_MASK, lane == 0 ? cap3_table(a, c) : 0, 0);  // one search per warp
    const bool last = c == a.chunk_off[t + 1] - 1;  // this table's last chunk
    uint32_t iv[C3_WPT], uv[C3_WPT];
    int64_t w0, wend;
    cap3_load(a, c, t, iv, uv, w0, wend);
    unsigned ci = 0, cu = 0;
#pragma unroll
    for (int k = 0; k < C3_WPT; k++) {
        ci += __popc(iv[k]);
        cu += __popc(uv[k]);
    }
    // packed (union << 32 | interval) ids before chunk x: the 256-chunk group
    // sums before it plus its own group's chunks before it (one load each)
    auto part = [&](int x) -> unsigned long long {
        unsigned long long v = 0;
        const int g = x >> 8, g0 = g << 8;
        for (int i = threadIdx.x; i < g; i += CF_THREADS) v += __ldcg(a.super + i);
        if (g0 + (int)threadIdx.x < x) v += __ldcg(a.cnt + g0 + threadIdx.x);
        return v;
    };
    const unsigned long long p = (unsigned long long)ci | ((unsigned long long)cu << 32);
    unsigned long long x = p, pb = part(c), ps = last ? part((int)a.chunk_off[t]) : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(DS_FULL_MASK, x, o);
        if (lane >= o) x += y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        pb += __shfl_xor_sync(DS_FULL_MASK, pb, o);
        ps += __shfl_xor_sync(DS_FULL_MASK, ps, o);
    }
    if (lane == 31) s_cnt[wid] = x;
    if (lane == 0) {
        s_base[wid] = pb;
        s_start[wid] = ps;
    }
    __syncthreads();  // (1): every read of super/cnt of this CTA is done
    if (threadIdx.x == 0) {
        // the last CTA past this point clears the group sums for the next call
        if (atomicAdd(a.ticket, 1u) == gridDim.x - 1) {
            for (int i = 0; i <= (a.nchunks >> 8); i++) a.super[i] = 0ull;
            *a.ticket = 0u;
        }
    }
    // lane k < NWP holds warp k's values; shuffles give every lane the
    // exclusive prefix of its warp and the CTA totals
    const unsigned long long mc = lane < NWP ? s_cnt[lane] : 0ull;
    unsigned long long b = lane < NWP ? s_base[lane] : 0ull;
    unsigned long long start = lane < NWP ? s_start[lane] : 0ull;
    unsigned long long incl = mc;
#pragma unroll
    for (int o = 1; o < NWP; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(DS_FULL_MASK, incl, o);
        if (lane >= o) incl += y;
    }
#pragma unroll
    for (int o = NWP / 2; o > 0; o >>= 1) {
        b += __shfl_xor_sync(DS_FULL_MASK, b, o);
        start += __shfl_xor_sync(DS_FULL_MASK, start, o);
    }
    b = __shfl_sync(DS_FULL_MASK, b, 0);  // lanes >= NWP reduced zeros
    start = __shfl_sync(DS_FULL_MASK, start, 0);
    const unsigned long long tot = __shfl_sync(DS_FULL_MASK, incl, NWP - 1);
    const unsigned long long wbase = __shfl_sync(DS_FULL_MASK, incl - mc, wid);
    const unsigned long long excl = wbase + x - p;
    const int64_t crow0 = (w0 - threadIdx.x * C3_WPT - a.word_off[t]) * 32;  // chunk's first row
    const unsigned lrow0 = threadIdx.x * C3_WPT * 32;                         // thread's first row
    // one scope is emitted per call (capture_into); both share the stage in
    // two rounds when both are asked for
    for (int scope = 0; scope < 2; scope++) {
        int64_t *out = scope ? a.ids_uni : a.ids_int;
        if (!out) continue;
        const unsigned n = (unsigned)(scope ? tot >> 32 : tot & 0xffffffffu);
        unsigned o = (unsigned)(scope ? excl >> 32 : excl & 0xffffffffu);
        const int64_t gbase = scope ? (int64_t)(b >> 32) : (int64_t)(uint32_t)b;
        if (scope == 1 && a.ids_int) __syncthreads();  // the interval round left the stage
#pragma unroll
        for (int k = 0; k < C3_WPT; k++) {
            uint32_t m = scope ? uv[k] : iv[k];
            while (m) {
                s_ids[o++] = lrow0 + 32 * k + __ffs(m) - 1;
                m &= m - 1;
            }
        }
        __syncthreads();  // (2)
        for (unsigned j = threadIdx.x; j < n; j += CF_THREADS)
            __stcs(out + gbase + j, crow0 + s_ids[j]);
    }
    // per-table counts: written by the table's last chunk
    if (last && threadIdx.x == 0) {
        const unsigned long long end = b + tot;
        const int nt = a.ntables;
        a.counts[t] = (int64_t)((uint32_t)end - (uint32_t)start);
        a.counts[nt + 1 + t] = (int64_t)((end >> 32) - (start >> 32));
        if (t == nt - 1) {
            a.counts[nt] = (int64_t)(uint32_t)end;
            a.counts[2 * nt + 1] = (int64_t)(end >> 32);
        }
    }
    if (a.fold) {  // reset_interval (1) / reset_baseline (2)
        bool done = false;
        if constexpr (C3_WPT == 4) {
            if ((w0 & 3) == 0 && w0 + 4 <= wend) {
                if (a.baseline)
                    *reinterpret_cast<uint4 *>(a.baseline + w0) =
                        a.fold == 1 ? make_uint4(uv[0], uv[1], uv[2], uv[3]) : make_uint4(0u, 0u, 0u, 0u);
                *reinterpret_cast<uint4 *>(a.interval + w0) = make_uint4(0u, 0u, 0u, 0u);
                done = true;
            }
        }
        if (!done) {
#pragma unroll
            for (int k = 0; k < C3_WPT; k++) {
                const int64_t w = w0 + k;
                if (w < wend) {
                    if (a.baseline) a.baseline[w] = a.fold == 1 ? uv[k] : 0u;
                    a.interval[w] = 0u;
                }
            }
        }
    }
}

}  // namespace ds

using namespace ds;

// TMA form over a packed stream of segments (16-byte aligned, any width).
// Lookups are weighted by the per-lookup cost of their table's kind (byte map
// 1, bit window 2, cache + RED 2, measured on B200) and cut into CTAs of
// about equal cost, expensive kinds first; every CTA range is a multiple of a
// warp stage so every bulk copy starts 16-byte aligned.
static int mark_packed_impl(uint32_t *words, const int64_t *word_off, const int64_t *rows,
                            const void *lookups, const int64_t *seg_boff, const int64_t *seg_n,
                            const int32_t *seg_width, const int32_t *seg_table_host, int nseg,
                            uint32_t *flags, void *stream) {
    if (nseg < 1 || nseg > DS_MAX_TABLES)
        return host::fail(DS_ERR_ARG, "ds_mark_packed: nseg out of range");
    if (!words || !word_off || !rows || !flags || !seg_boff || !seg_n || !seg_width)
        return host::fail(DS_ERR_ARG, "ds_mark_packed: null pointer");
    MarkArgs a;
    a.words = words;
    a.idx = lookups;
    a.ibytes = static_cast<const uint8_t *>(lookups);
    a.flags = flags;
    a.nseg = nseg;
    int64_t total = 0, max_word = 0;
    for (int s = 0; s < nseg; s++) {
        const int t = seg_table_host ? seg_table_host[s] : 0;
        if (t < 0 || t >= DS_MAX_TABLES) return host::fail(DS_ERR_ARG, "ds_mark_packed: table index");
        const int w = seg_width[s];
        if (!((w >= 4 && w <= 28 && w % 4 == 0) || w == 32 || w == 64))
            return host::fail(DS_ERR_ARG, "ds_mark_packed: id width must be 4..28 (step 4), 32 or 64 bits");
        if (seg_boff[s] % 16 || seg_n[s] < 0)
            return host::fail(DS_ERR_ARG, "ds_mark_packed: segments must start 16-byte aligned");
        a.word_off[s] = word_off[t];
        a.rows[s] = rows[t];
        a.seg_boff[s] = seg_boff[s];
        a.seg_n[s] = seg_n[s];
        a.seg_width[s] = w;
        total += seg_n[s];
        const int64_t mw = word_off[t] + (rows[t] + 31) / 32;
        max_word = mw > max_word ? mw : max_word;
    }
    if (total == 0) return DS_OK;
    if (!lookups || reinterpret_cast<uintptr_t>(lookups) % 16)
        return host::fail(DS_ERR_ARG, "ds_mark_packed: lookups must be 16-byte aligned");
    // the cache keys are 31-bit word ids
    if (max_word >= (int64_t)0x7fffffffLL)
        return host::fail(DS_ERR_CONFIG, "ds_mark: a table set holds at most 2^31-1 bitmap words");
    const size_t smem = (size_t)MK_WARPS * MK_WSTAGES * MK_WSTAGE_BYTES + MK_CACHE_BYTES;
    auto fn = mark_tma_kernel;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
    int tper = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tper, fn, MARK_THREADS, smem);
    if (tper < 1) tper = 1;
    static const int64_t kCost[3] = {1, 2, 2};
    const int64_t cost_cache = host::env_int("DS_MARK_COST_CACHE", kCost[2]);
    int kind[DS_MAX_TABLES];
    double total_cost = 0.0;
    for (int s = 0; s < nseg; s++) {
        const int64_t r = a.rows[s];
        kind[s] = r <= MK_BYTE_ROWS ? 0 : ((r + 31) / 32 <= MK_WIN_WORDS ? 1 : 2);
        const int64_t w = kind[s] == 2 ? cost_cache : kCost[kind[s]];
        total_cost += (double)a.seg_n[s] * (double)w;
    }
    const double waves = (double)host::env_int("DS_MARK_WAVES", 2);
    const double target = total_cost / ((double)host::sm_count() * tper * waves);
    int64_t nb = 0;
    int j = 0;
    for (int kd = 2; kd >= 0; kd--) {
        for (int s = 0; s < nseg; s++) {
            if (kind[s] != kd) continue;
            const int64_t w = kd == 2 ? cost_cache : kCost[kd];
            const int wb = a.seg_width[s];  // bits
            const int64_t ids_per_stage =
                (wb == 8 || wb == 16 || wb == 32 || wb == 64) ? MK_WSTAGE_BYTES * 8 / wb
                                                              : (wb <= 16 ? 512 : 256);  // mark_range IDS
            int64_t pb = (int64_t)(target / (double)w) + 1;
            pb = (pb + ids_per_stage - 1) / ids_per_stage * ids_per_stage;
            a.seg_pb[s] = pb;
            a.seg_order[j] = s;
            a.blk_off[j] = (int)nb;
            nb += (a.seg_n[s] + pb - 1) / pb;
            j++;
        }
    }
    a.blk_off[nseg] = (int)nb;
    if (nb == 0) return DS_OK;
    fn<<<(unsigned)nb, MARK_THREADS, smem, (cudaStream_t)stream>>>(a);
    return host::check_launch("ds_mark");
}

static int mark_impl(uint32_t *words, const int64_t *word_off, const int64_t *rows,
                     const void *idx, int idx32, const int64_t *seg_off_host,
                     const int32_t *seg_table_host, int nseg, uint32_t *flags, void *stream) {
    if (nseg < 1 || nseg > DS_MAX_TABLES) return host::fail(DS_ERR_ARG, "ds_mark: nseg out of range");
    if (!words || !word_off || !rows || !flags) return host::fail(DS_ERR_ARG, "ds_mark: null pointer");
    const int64_t isz = idx32 ? 4 : 8;
    int64_t total = seg_off_host[nseg] - seg_off_host[0];
    if (total <= 0) return DS_OK;
    if (!idx) return host::fail(DS_ERR_ARG, "ds_mark: null idx");
    // TMA form when every segment starts 16-byte aligned
    bool aligned = reinterpret_cast<uintptr_t>(idx) % 16 == 0;
    for (int s = 0; s <= nseg; s++) aligned &= (seg_off_host[s] * isz) % 16 == 0;
    int64_t max_word = 0;
    for (int s = 0; s < nseg; s++) {
        const int t = seg_table_host ? seg_table_host[s] : 0;
        if (t < 0 || t >= DS_MAX_TABLES) return host::fail(DS_ERR_ARG, "ds_mark: table index");
        const int64_t mw = word_off[t] + (rows[t] + 31) / 32;
        max_word = mw > max_word ? mw : max_word;
    }
    if (aligned && max_word < (int64_t)0x7fffffffLL && !host::env_flag("DS_MARK_NO_TMA")) {
        int64_t boff[DS_MAX_TABLES], n[DS_MAX_TABLES];
        int32_t wd[DS_MAX_TABLES];
        for (int s = 0; s < nseg; s++) {
            boff[s] = seg_off_host[s] * isz;
            n[s] = seg_off_host[s + 1] - seg_off_host[s];
            wd[s] = (int32_t)(8 * isz);
        }
        return mark_packed_impl(words, word_off, rows, idx, boff, n, wd, seg_table_host, nseg, flags,
                                stream);
    }
    // grid-stride form for unaligned streams
    MarkArgs a;
    a.words = words;
    a.idx = idx;
    a.idx32 = idx32;
    a.flags = flags;
    a.nseg = nseg;
    for (int s = 0; s < nseg; s++) {
        const int t = seg_table_host ? seg_table_host[s] : 0;
        a.seg_table[s] = s;  // per-segment base/rows resolved here
        a.word_off[s] = word_off[t];
        a.rows[s] = rows[t];
        a.seg_off[s] = seg_off_host[s];
    }
    a.seg_off[nseg] = seg_off_host[nseg];
    // word ids are 32-bit inside the kernel (and the cache keys are word+1)
    if (max_word >= (int64_t)0xffffffffLL)
        return host::fail(DS_ERR_CONFIG, "ds_mark: a table set holds at most 2^32-1 bitmap words");
    const int64_t quantum = (int64_t)MARK_THREADS * MARK_PER_THREAD;
    int per_sm = 0;
    if (idx32)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mark_kernel<int32_t>, MARK_THREADS, 0);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mark_kernel<int64_t>, MARK_THREADS, 0);
    if (per_sm < 1) per_sm = 1;
    int64_t blocks = host::grid_for((total + MARK_PER_THREAD - 1) / MARK_PER_THREAD, MARK_THREADS,
                                    per_sm);
    int64_t per_block = (total + blocks - 1) / blocks;
    per_block = (per_block + quantum - 1) / quantum * quantum;
    blocks = (total + per_block - 1) / per_block;
    const int vec = (reinterpret_cast<uintptr_t>(idx) % 16 == 0) && ((a.seg_off[0] * isz) % 16 == 0);
    if (idx32)
        mark_kernel<int32_t><<<(unsigned)blocks, MARK_THREADS, 0, (cudaStream_t)stream>>>(
            a, per_block, vec, 1);
    else
        mark_kernel<int64_t><<<(unsigned)blocks, MARK_THREADS, 0, (cudaStream_t)stream>>>(
            a, per_block, vec, 1);
    return host::check_launch("ds_mark");
}

extern "C" int ds_mark_packed(uint32_t *words, const int64_t *word_off_host, const int64_t *rows_host,
                              const void *lookups, const int64_t *seg_byte_off_host,
                              const int64_t *seg_count_host, const int32_t *seg_width_host,
                              const int32_t *seg_table_host, int nseg, uint32_t *flags,
                              void *stream) {
    return mark_packed_impl(words, word_off_host, rows_host, lookups, seg_byte_off_host,
                            seg_count_host, seg_width_host, seg_table_host, nseg, flags, stream);
}

extern "C" int ds_mark(uint32_t *words, const int64_t *word_off_host, const int64_t *rows_host,
                       const int64_t *idx, const int64_t *seg_off_host,
                       const int32_t *seg_table_host, int nseg, uint32_t *flags, void *stream) {
    return mark_impl(words, word_off_host, rows_host, idx, 0, seg_off_host, seg_table_host, nseg,
                     flags, stream);
}

extern "C" int ds_mark_i32(uint32_t *words, const int64_t *word_off_host, const int64_t *rows_host,
                           const int32_t *idx, const int64_t *seg_off_host,
                           const int32_t *seg_table_host, int nseg, uint32_t *flags,
                           void *stream) {
    return mark_impl(words, word_off_host, rows_host, idx, 1, seg_off_host, seg_table_host, nseg,
                     flags, stream);
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
    // count/emit form: ticket + 2 arrays of nchunks u64 (chunks of C3_WPB words);
    // the > 2^32-row form: 4 arrays of nchunks u64 (chunks of CAP_WPB words)
    const int64_t n3 = total_words / C3_WPB + 2 * (int64_t)ntables + 1;
    const int64_t n1 = total_words / CAP_WPB + 2 * (int64_t)ntables + 1;
    const size_t b3 = 16 + (size_t)(2 * n3) * sizeof(unsigned long long);
    const size_t b1 = (size_t)(4 * n1) * sizeof(unsigned long long);
    return (b3 > b1 ? b3 : b1) + 256;
}

extern "C" int ds_capture(uint32_t *interval, uint32_t *baseline, const int64_t *word_off_host,
                          const int64_t *rows_host, int ntables, int64_t *ids_int,
                          int64_t *ids_union, int64_t *counts, int fold, void *workspace,
                          size_t workspace_bytes, void *stream) {
    (void)rows_host;
    if (ntables < 1 || ntables > DS_MAX_TABLES) return host::fail(DS_ERR_ARG, "ds_capture: ntables");
    if (!interval || !counts || !workspace) return host::fail(DS_ERR_ARG, "ds_capture: null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    int64_t total_rows = 0;
    for (int t = 0; t < ntables; t++) total_rows += (word_off_host[t + 1] - word_off_host[t]) * 32;
    if (total_rows < (int64_t)0xffffffffLL) {
        // count -> scan -> emit (ids per scope fit the 32-bit packed counts)
        Cap3Args f;
        f.interval = interval;
        f.baseline = baseline;
        f.ids_int = ids_int;
        f.ids_uni = ids_union;
        f.counts = counts;
        f.ntables = ntables;
        f.fold = fold;
        int64_t nch = 0;
        for (int t = 0; t <= ntables; t++) f.word_off[t] = word_off_host[t];
        for (int t = 0; t < ntables; t++) {
            f.chunk_off[t] = nch;
            int64_t w = word_off_host[t + 1] - word_off_host[t];
            nch += w > 0 ? (w + C3_WPB - 1) / C3_WPB : 1;
        }
        f.chunk_off[ntables] = nch;
        f.nchunks = (int)nch;
        size_t need = 16 + (size_t)(nch + nch / 256 + 1) * sizeof(unsigned long long);
        if (workspace_bytes < need) return host::fail(DS_ERR_ARG, "ds_capture: workspace too small");
        f.ticket = reinterpret_cast<unsigned *>(workspace);
        f.cnt = reinterpret_cast<unsigned long long *>(static_cast<uint8_t *>(workspace) + 16);
        f.super = f.cnt + nch;
        cudaError_t e = host::launch_pdl(cap3_count_kernel, (unsigned)nch, CF_THREADS, 0, s, f);
        if (e == cudaSuccess) e = host::launch_pdl(cap3_emit_kernel, (unsigned)nch, CF_THREADS, 0, s, f);
        if (e != cudaSuccess) return host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
        return host::check_launch("ds_capture");
    }
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
    capture_count_kernel<<<(unsigned)nch, CAP_THREADS, 0, s>>>(a);
    capture_scan_kernel<<<1, 1024, 0, s>>>(a);
    capture_write_kernel<<<(unsigned)nch, CAP_THREADS, 0, s>>>(a);
    (void)capture_nchunks;
    return host::check_launch("ds_capture");
}
