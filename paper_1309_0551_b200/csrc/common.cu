// libsu3g: error reporting and cached device properties.
#include <cstdio>
#include <atomic>
#include <mutex>

#include "su3g_common.cuh"

namespace su3g {

static thread_local std::string g_last_error;
static thread_local std::string g_last_kernel;

void note_kernel(const std::string& name) { g_last_kernel = name; }
static std::atomic<int> g_sm_reserve{0};

int sm_reserve() { return g_sm_reserve.load(); }
void set_sm_reserve(int n) { g_sm_reserve.store(n); }

void set_error(const std::string& msg) { g_last_error = msg; }

int fail_invalid(const std::string& msg) {
    set_error(msg);
    return SU3G_EINVAL;
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string(what) + ": " + cudaGetErrorString(e));
        return static_cast<int>(e);
    }
    return SU3G_OK;
}

const DeviceInfo& device_info() {
    static DeviceInfo cache[64];
    static std::mutex mu;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    DeviceInfo& d = cache[dev];
    if (d.device != dev) {
        std::lock_guard<std::mutex> lock(mu);
        if (d.device != dev) {
            DeviceInfo n;
            n.device = dev;
            cudaDeviceGetAttribute(&n.num_sms, cudaDevAttrMultiProcessorCount, dev);
            cudaDeviceGetAttribute(&n.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
            cudaDeviceGetAttribute(&n.l2_bytes, cudaDevAttrL2CacheSize, dev);
            d = n;
        }
    }
    return d;
}

}  // namespace su3g

extern "C" {

int su3g_abi_version(void) { return SU3G_ABI_VERSION; }

const char* su3g_last_error(void) { return su3g::g_last_error.c_str(); }

const char* su3g_last_kernel(void) { return su3g::g_last_kernel.c_str(); }

int su3g_device_sm_count(void) { return su3g::device_info().num_sms; }

int64_t su3g_device_l2_bytes(void) { return su3g::device_info().l2_bytes; }

}  // extern "C"
