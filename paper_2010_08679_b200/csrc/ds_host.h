// ds_host.h -- host-side helpers of the C ABI (status text, launch checks, grid sizing).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "../../include/deltasnap_cuda.h"

namespace ds {
namespace host {

// Thread-local text of the last failure (ds_last_error); no shared state.
inline char *err_buf() {
    static thread_local char buf[512];
    return buf;
}

inline int fail(int status, const char *msg) {
    snprintf(err_buf(), 512, "%s", msg);
    return status;
}

inline int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        snprintf(err_buf(), 512, "%s: %s", what, cudaGetErrorString(e));
        return DS_ERR_CUDA;
    }
    return DS_OK;
}

// SM count of the current device, cached per device (read-only after init).
int sm_count();

// Diagnostic switches (A/B measurements), read from the environment.
inline bool env_flag(const char *name) {
    const char *v = getenv(name);
    return v && v[0] && v[0] != '0';
}
inline int64_t env_int(const char *name, int64_t dflt) {
    const char *v = getenv(name);
    return v && v[0] ? strtoll(v, nullptr, 10) : dflt;
}

// Launch with programmatic stream serialization (see ds_common.cuh pdl_*);
// DS_PDL=0 launches normally (A/B).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                              cudaStream_t s, Args... args) {
    static const bool on = env_int("DS_PDL", 1) != 0;
    if (!on) {
        kern<<<grid, block, smem, s>>>(args...);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Grid for a grid-stride kernel: enough blocks to cover n, capped at
// `per_sm` resident blocks per SM.
inline int64_t grid_for(int64_t n, int threads, int per_sm) {
    int64_t need = (n + threads - 1) / threads;
    int64_t cap = (int64_t)sm_count() * per_sm;
    if (need < 1) need = 1;
    return need < cap ? need : cap;
}

}  // namespace host
}  // namespace ds
