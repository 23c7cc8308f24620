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

// Batched window upload read by the SMs from mapped page-locked host memory.
// One warp per row (rows of a job spread over blockIdx.x, jobs over
// blockIdx.y); 16-byte loads where the source and destination share their
// alignment (the plane windows: both pitches are multiples of 16), byte
// copies for the ragged ends.  Each warp keeps kGatherUnroll 16-byte loads
// per lane (2 KB) in flight; about one 8-warp CTA per SM (~2.4 MB in flight)
// covers the link's bandwidth-delay product with room to spare, and leaves
// the SMs to the fusion kernels running beside it.
namespace divas {
constexpr int kGatherJobs = 96;
constexpr int kGatherUnroll = 4;

struct GatherJobs {
    divas_copy2d j[kGatherJobs];
};
__global__ void __launch_bounds__(256) gather2d_kernel(GatherJobs J) {
    const divas_copy2d &c = J.j[blockIdx.y];
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < c.rows;
         r += warps) {
        const uint8_t *s = (const uint8_t *)c.src + r * c.spitch;
        uint8_t *d = (uint8_t *)c.dst + r * c.dpitch;
        const int64_t w = c.width_bytes;
        int64_t head = 0, nvec = 0;
        if ((((uintptr_t)s ^ (uintptr_t)d) & 15) == 0) {
            head = min((int64_t)((16 - ((uintptr_t)s & 15)) & 15), w);
            nvec = (w - head) >> 4;
        }
        for (int64_t i = lane; i < head; i += 32) d[i] = s[i];
        const uint4 *sv = reinterpret_cast<const uint4 *>(s + head);
        uint4 *dv = reinterpret_cast<uint4 *>(d + head);
        int64_t i = lane;
        for (; i + 32 * (kGatherUnroll - 1) < nvec; i += 32 * kGatherUnroll) {
            uint4 t[kGatherUnroll];
#pragma unroll
            for (int u = 0; u < kGatherUnroll; ++u) t[u] = sv[i + 32 * u];
#pragma unroll
            for (int u = 0; u < kGatherUnroll; ++u) dv[i + 32 * u] = t[u];
        }
        for (; i < nvec; i += 32) dv[i] = sv[i];
        for (int64_t k = head + (nvec << 4) + lane; k < w; k += 32) d[k] = s[k];
    }
}
}  // namespace divas

extern "C" int divas_gather2d_h2d(const divas_copy2d *jobs, int32_t n, void *stream) {
    if (n < 0 || (n > 0 && !jobs)) {
        divas::set_error("divas_gather2d_h2d: bad arguments");
        return DIVAS_EINVAL;
    }
    int sms = 148;
    {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    for (int32_t j0 = 0; j0 < n; j0 += divas::kGatherJobs) {
        divas::GatherJobs J;
        const int m = std::min<int32_t>(divas::kGatherJobs, n - j0);
        int64_t rows = 0;
        for (int k = 0; k < m; ++k) {
            divas_copy2d c = jobs[j0 + k];
            if (!c.dst || !c.src || c.width_bytes < 0 || c.rows < 0 ||
                c.width_bytes > c.spitch || c.width_bytes > c.dpitch) {
                divas::set_error("divas_gather2d_h2d: bad job %d", j0 + k);
                return DIVAS_EINVAL;
            }
            void *dp = nullptr;                      // the source's device mapping
            if (c.rows > 0 && c.width_bytes > 0 &&
                cudaHostGetDevicePointer(&dp, const_cast<void *>(c.src), 0) != cudaSuccess) {
                cudaGetLastError();
                divas::set_error("divas_gather2d_h2d: job %d source is not page-locked", j0 + k);
                return DIVAS_EINVAL;
            }
            if (dp) c.src = dp;
            J.j[k] = c;
            rows = std::max<int64_t>(rows, c.rows);
        }
        for (int k = m; k < divas::kGatherJobs; ++k) J.j[k] = divas_copy2d{nullptr, nullptr, 0, 0, 0, 0};
        if (rows == 0) continue;
        // about one CTA of 8 warps per SM in total, spread over the jobs (more
        // CTAs measured slower: they crowd out the fusion kernels beside them)
        const int64_t per_job = std::max<int64_t>(1, (sms + m - 1) / m);
        const unsigned bx = (unsigned)std::min<int64_t>(per_job, (rows + 7) / 8);
        divas::gather2d_kernel<<<dim3(bx, (unsigned)m), 256, 0, (cudaStream_t)stream>>>(J);
        if (int rc = divas::check_launch("divas_gather2d_h2d")) return rc;
    }
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
