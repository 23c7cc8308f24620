// abi.cu -- error reporting and version entry points of the C ABI.
#include <algorithm>
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

// Store `bytes` of src into every peer buffer at `offset` (NVLink stores into
// symmetric-memory peer mappings): a rank's block of an all-gather, one launch.
namespace divas {
__global__ void peer_put_kernel(const uint8_t *__restrict__ src, size_t bytes,
                                uint8_t *const *__restrict__ peers, int n_peers, size_t offset) {
    const int p = blockIdx.y;
    uint8_t *dst = peers[p] + offset;
    const size_t n16 = bytes / 16;
    const bool vec = ((((uintptr_t)src) | ((uintptr_t)dst)) & 15) == 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < (vec ? n16 : 0);
         i += (size_t)gridDim.x * blockDim.x)
        reinterpret_cast<uint4 *>(dst)[i] = __ldg(reinterpret_cast<const uint4 *>(src) + i);
    for (size_t i = (vec ? n16 * 16 : 0) + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < bytes;
         i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}
}  // namespace divas

extern "C" int divas_peer_put(const void *src, size_t bytes, uint8_t *const *peers,
                              int32_t n_peers, size_t offset, void *stream) {
    if (!src || !peers || n_peers < 1 || n_peers > 65535) {
        divas::set_error("divas_peer_put: bad arguments");
        return DIVAS_EINVAL;
    }
    if (bytes == 0) return DIVAS_OK;
    const size_t blocks = std::min<size_t>((bytes / 16 + 255) / 256 + 1, 1024);
    divas::peer_put_kernel<<<dim3((unsigned)blocks, (unsigned)n_peers), 256, 0,
                             (cudaStream_t)stream>>>((const uint8_t *)src, bytes, peers, n_peers,
                                                     offset);
    return divas::check_launch("divas_peer_put");
}
