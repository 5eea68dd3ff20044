// ds_peer.cu -- exchange buffers of the row-sharded count exchange over NVLink
// peer memory (include/deltasnap_cuda.h documents the
// protocol, ds_writer.cuh peer_publish / peer_wait run it inside K3).
//
// The sharded checkpoint exchanges only every rank's per-table dirty counts
// (sharded.py: where each rank's records land in a CNR1 section).  A NCCL
// all_gather beside the writer costs more than its bytes: its kernel sits on
// SMs until the peers arrive, so some of the writer's CTAs (two per SM, the
// register file full) wait a whole wave.  Here the writer's CTA 0 stores the
// counts into every peer's exchange buffer itself (P2P stores over NVLink
// through CUDA IPC mappings, then a system-scope release of the slot's epoch
// flag); by the time the writer has run, the peers' counts are there and the
// last CTA's wait is one warp reading local memory.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "ds_common.cuh"
#include "ds_host.h"

#include "ds_writer.cuh"  // peer_flags_bytes (the kernels' side is in writer_layout / _epilogue)

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
