// ds_peer.cu -- the row-sharded count exchange over NVLink peer memory
// (include/deltasnap_cuda.h documents the protocol).
//
// The sharded checkpoint exchanges only every rank's per-table dirty counts
// (sharded.py: where each rank's records land in a CNR1 section).  A NCCL
// all_gather beside the writer costs more than its bytes: its kernel sits on
// SMs until the peers arrive, so some of the writer's CTAs (two per SM, the
// register file full) wait a whole wave.  Here the capture stream stores the
// counts into every peer's exchange buffer itself (P2P stores over NVLink
// through CUDA IPC mappings, then a system-scope release of the slot's epoch
// flag); by the time the writer has run, the peers' counts are there and the
// wait is one warp reading local memory.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ds_common.cuh"
#include "ds_host.h"

namespace ds {

constexpr int PEER_MAX = 64;  // ranks of one exchange (one box: <= 8 GPUs)

struct PublishArgs {
    void *peers[PEER_MAX];
    const int64_t *counts;
    int n, world, rank;
    uint32_t epoch;
};

__host__ __device__ inline size_t peer_flags_bytes(int world) {
    return ((size_t)2 * world * sizeof(uint32_t) + 255) & ~(size_t)255;
}

__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// warp w writes this rank's counts into peer w's slot, then releases the flag
__global__ void counts_publish_kernel(const PublishArgs a) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int par = a.epoch & 1;
    for (int p = w; p < a.world; p += blockDim.x >> 5) {
        uint8_t *base = static_cast<uint8_t *>(a.peers[p]);
        uint32_t *flags = reinterpret_cast<uint32_t *>(base);
        int64_t *slot = reinterpret_cast<int64_t *>(base + peer_flags_bytes(a.world)) +
                        ((size_t)par * a.world + a.rank) * a.n;
        for (int i = lane; i < a.n; i += 32) slot[i] = __ldcg(a.counts + i);
        __syncwarp();
        if (lane == 0) {
            __threadfence_system();  // the slot before its flag, for every observer
            st_release_sys(flags + par * a.world + a.rank, a.epoch);
        }
    }
}

// lane r spins on rank r's flag; then the warp copies the slots out
__global__ void counts_wait_kernel(const uint8_t *local, int n, int world, uint32_t epoch,
                                   int64_t *out, uint32_t *err, int64_t timeout_ns) {
    const int lane = threadIdx.x;
    const int par = epoch & 1;
    const uint32_t *flags = reinterpret_cast<const uint32_t *>(local) + par * world;
    bool late = false;
    const uint64_t t0 = globaltimer();
    for (int r = lane; r < world; r += 32) {
        while (ld_acquire_sys(flags + r) != epoch) {
            if ((int64_t)(globaltimer() - t0) > timeout_ns) {
                late = true;
                break;
            }
            __nanosleep(100);
        }
    }
    if (__any_sync(DS_FULL_MASK, late)) {
        if (lane == 0) atomicOr(err, DS_FLAG_TIMEOUT);
        return;
    }
    const int64_t *slots = reinterpret_cast<const int64_t *>(local + peer_flags_bytes(world)) +
                           (size_t)par * world * n;
    for (int i = lane; i < world * n; i += 32) out[i] = *(volatile const int64_t *)(slots + i);
}

}  // namespace ds

using namespace ds;

extern "C" size_t ds_peer_buffer_size(int world, int n) {
    if (world < 1 || n < 1) return 0;
    return peer_flags_bytes(world) + (size_t)2 * world * n * sizeof(int64_t);
}

extern "C" int ds_peer_alloc(size_t bytes, void **ptr, uint8_t *handle64) {
    if (!ptr || !handle64 || bytes == 0) return host::fail(DS_ERR_ARG, "ds_peer_alloc: bad argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) e = cudaMemset(p, 0, bytes);
    cudaIpcMemHandle_t h;
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
        if (p) cudaFree(p);
        return host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
    }
    memcpy(handle64, &h, 64);
    *ptr = p;
    return DS_OK;
}

extern "C" int ds_peer_open(const uint8_t *handle64, void **ptr) {
    if (!ptr || !handle64) return host::fail(DS_ERR_ARG, "ds_peer_open: bad argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
    return e == cudaSuccess ? DS_OK : host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
}

extern "C" int ds_peer_close(void *ptr) {
    cudaError_t e = cudaIpcCloseMemHandle(ptr);
    return e == cudaSuccess ? DS_OK : host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
}

extern "C" int ds_peer_free(void *ptr) {
    cudaError_t e = cudaFree(ptr);
    return e == cudaSuccess ? DS_OK : host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
}

extern "C" int ds_counts_publish(const int64_t *counts, int n, void *const *peers_host, int world,
                                 int rank, uint32_t epoch, void *stream) {
    if (world < 1 || world > PEER_MAX || rank < 0 || rank >= world || n < 1 || !counts || !peers_host)
        return host::fail(DS_ERR_ARG, "ds_counts_publish: bad argument");
    PublishArgs a;
    for (int p = 0; p < world; p++) {
        if (!peers_host[p]) return host::fail(DS_ERR_ARG, "ds_counts_publish: null peer buffer");
        a.peers[p] = peers_host[p];
    }
    a.counts = counts;
    a.n = n;
    a.world = world;
    a.rank = rank;
    a.epoch = epoch;
    const int warps = world < 8 ? world : 8;
    counts_publish_kernel<<<1, 32 * warps, 0, (cudaStream_t)stream>>>(a);
    return host::check_launch("ds_counts_publish");
}

extern "C" int ds_counts_wait(const void *local, int n, int world, uint32_t epoch, int64_t *out,
                              uint32_t *flags, int64_t timeout_ns, void *stream) {
    if (world < 1 || world > PEER_MAX || n < 1 || !local || !out || !flags || epoch == 0)
        return host::fail(DS_ERR_ARG, "ds_counts_wait: bad argument");
    counts_wait_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(static_cast<const uint8_t *>(local), n, world,
                                                           epoch, out, flags, timeout_ns);
    return host::check_launch("ds_counts_wait");
}
