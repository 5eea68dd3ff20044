// ds_capi.cu -- library identity and diagnostics of the C ABI.
#include <cuda_runtime.h>

#include "ds_host.h"

namespace ds {
namespace host {

int sm_count() {
    // per-device cached attribute (read-only after the first query)
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (cache[dev] == 0) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = n > 0 ? n : 148;
    }
    return cache[dev];
}

}  // namespace host
}  // namespace ds

extern "C" const char *ds_version(void) { return "deltasnap-b200 0.1.0 (sm_100a)"; }

extern "C" const char *ds_last_error(void) { return ds::host::err_buf(); }

extern "C" int ds_device_sm_count(int device) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
    return n;
}

extern "C" int ds_set_l2_fetch_granularity(int bytes) {
    // Process-wide hint for the current device: how many bytes an L2 miss
    // pulls from HBM.  Random 64-byte row gathers (dim 16 fp32) waste half of
    // every 128-byte fetch; 64 fetches only what the row needs.
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)bytes);
    if (e != cudaSuccess) return ds::host::fail(DS_ERR_CUDA, cudaGetErrorString(e));
    return DS_OK;
}

extern "C" int ds_get_l2_fetch_granularity(void) {
    size_t v = 0;
    if (cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity) != cudaSuccess) return -1;
    return (int)v;
}
