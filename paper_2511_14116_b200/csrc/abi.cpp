// Status / error plumbing of the C ABI (thread-local last-error message).
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <string>

#include "common.cuh"

namespace fs {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

int cuda_status(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return FS_OK;
    return fail(FS_ECUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

int sm_count(int device) {
    static int cache[64] = {0};
    static std::mutex mu;
    if (device < 0 || device >= 64) return -1;
    std::lock_guard<std::mutex> lock(mu);
    if (cache[device] == 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
            cudaGetLastError();
            return -1;
        }
        cache[device] = v;
    }
    return cache[device];
}

}  // namespace fs

extern "C" int fs_abi_version(void) { return FS_ABI_VERSION; }

extern "C" const char *fs_last_error(void) { return fs::g_last_error.c_str(); }

extern "C" int fs_device_sms(int device) { return fs::sm_count(device); }
