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
