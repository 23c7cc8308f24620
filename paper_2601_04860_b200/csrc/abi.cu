// abi.cu -- error reporting and version entry points of the C ABI.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace divas {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return DIVAS_ECUDA;
    }
    return DIVAS_OK;
}

}  // namespace divas

extern "C" const char *divas_last_error(void) { return divas::g_err; }
extern "C" int divas_abi_version(void) { return DIVAS_ABI_VERSION; }

// Host -> device copy of a pitched sub-rectangle (rows of `width_bytes` bytes):
// windowed uploads of view planes (refine_and_fuse).
extern "C" int divas_copy2d_h2d(void *dst, size_t dpitch, const void *src, size_t spitch,
                                size_t width_bytes, size_t height, void *stream) {
    if (!dst || !src || width_bytes > dpitch || width_bytes > spitch) {
        divas::set_error("divas_copy2d_h2d: bad arguments");
        return DIVAS_EINVAL;
    }
    if (width_bytes == 0 || height == 0) return DIVAS_OK;
    if (cudaMemcpy2DAsync(dst, dpitch, src, spitch, width_bytes, height, cudaMemcpyHostToDevice,
                          (cudaStream_t)stream) != cudaSuccess)
        return divas::check_launch("divas_copy2d_h2d");
    return DIVAS_OK;
}
