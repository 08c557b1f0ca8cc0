// Host-side error state and small C-ABI utilities of femasm_b200.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "fa_common.cuh"

namespace fa {
static thread_local char g_error[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_error, sizeof(g_error), fmt, ap);
    va_end(ap);
}

int pdl_mask() {
    static const int mask = [] {
        const char* env = getenv("FEMASM_B200_PDL_MASK");
        return env ? int(strtol(env, nullptr, 0)) : 0x1bf;
    }();
    return mask;
}

int num_sms() {
    // per device (cached): grids are sized in multiples of the SM count
    static thread_local int cached_dev = -1, cached_n = 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (dev != cached_dev) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
        cached_dev = dev;
        cached_n = n;
    }
    return cached_n;
}

int cuda_status(cudaError_t e, const char* what) {
    set_error("%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
    return FA_ERR_CUDA;
}
}  // namespace fa

extern "C" const char* fa_last_error(void) { return fa::g_error; }

extern "C" const char* fa_version(void) { return "femasm_b200 0.1.0 sm_100a"; }

extern "C" int fa_result_status(const fa_result* r) {
    if (!r) return FA_ERR_ARGUMENT;
    if (r->index_error_pos != INT64_MAX || r->col_error_pos != INT64_MAX || r->repeat_error_pos != INT64_MAX)
        return FA_ERR_INDEX;
    if (r->degenerate_index != INT64_MAX) return FA_ERR_DEGENERATE;
    return FA_OK;
}
