// threshold.cu -- kernel (c): occupancy threshold and C-order compaction.
//
// Reference: `pred = ogrid.probs >= threshold` (/root/reference/pkg/src/divas/
// ablation.py:109) and the occupied-voxel list np.argwhere(pred) (C order).
//
//   thr_mark   p -> occ (u8) and one count per 4096-voxel tile (warp ballots)
//   thr_scan   exclusive scan of the tile counts (one CTA), total -> *count
//   thr_emit   occ -> indices: per-row ballots + a 128-entry CTA scan give each
//              set voxel its C-order rank, so the output order is exactly
//              np.argwhere's regardless of scheduling (no atomics).
// HBM bytes: 8 B/voxel (p) + 1 B (occ write) + 1 B (occ re-read) + 24 B per hit.
#include <algorithm>

#include "common.cuh"

namespace divas {

constexpr int kThrThreads = 256;
constexpr int kThrRows = 16;
constexpr int kThrTile = kThrThreads * kThrRows;   // 4096 voxels per CTA
constexpr int kThrWarps = kThrThreads / 32;

__global__ void __launch_bounds__(kThrThreads)
thr_mark(const double *__restrict__ p, int64_t n, double thr, uint8_t *__restrict__ occ,
         int64_t *__restrict__ tile_counts) {
    __shared__ int s_total;
    if (threadIdx.x == 0) s_total = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kThrTile;
    int mine = 0;
#pragma unroll 4
    for (int r = 0; r < kThrRows; ++r) {
        const int64_t e = base + (int64_t)r * kThrThreads + threadIdx.x;
        uint8_t pred = 0;
        if (e < n) {
            pred = (__ldcs(p + e) >= thr) ? 1 : 0;
            occ[e] = pred;
        }
        mine += pred;
    }
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&s_total, mine);
    __syncthreads();
    if (threadIdx.x == 0) tile_counts[blockIdx.x] = s_total;
}

// single CTA: exclusive scan in place, total -> *count
__global__ void __launch_bounds__(1024)
thr_scan(int64_t *__restrict__ tile_counts, int64_t ntiles, int64_t *__restrict__ count) {
    __shared__ int64_t s_warp[32];
    __shared__ int64_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t base = 0; base < ntiles; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const int64_t v = i < ntiles ? tile_counts[i] : 0;
        int64_t incl = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            int64_t w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
            int64_t wi = w;
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += y;
            }
            s_warp[lane] = wi - w;   // exclusive warp offsets
        }
        __syncthreads();
        const int64_t carry = s_carry;
        if (i < ntiles) tile_counts[i] = carry + s_warp[warp] + incl - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry = carry + s_warp[warp] + incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) *count = s_carry;
}

__global__ void __launch_bounds__(kThrThreads)
thr_emit(const uint8_t *__restrict__ occ, int64_t n, int64_t g,
         const int64_t *__restrict__ tile_offsets, int64_t *__restrict__ idx) {
    __shared__ int s_cnt[kThrRows * kThrWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t base = (int64_t)blockIdx.x * kThrTile;
    unsigned ball[kThrRows];
#pragma unroll
    for (int r = 0; r < kThrRows; ++r) {
        const int64_t e = base + (int64_t)r * kThrThreads + threadIdx.x;
        const bool pred = e < n && occ[e] != 0;
        ball[r] = __ballot_sync(0xffffffffu, pred);
        if (lane == 0) s_cnt[r * kThrWarps + warp] = __popc(ball[r]);
    }
    __syncthreads();
    if (warp == 0) {   // exclusive scan of the 128 (row, warp) counts in C order
        constexpr int per = kThrRows * kThrWarps / 32;
        int v[per], sum = 0;
#pragma unroll
        for (int k = 0; k < per; ++k) { v[k] = s_cnt[lane * per + k]; sum += v[k]; }
        int incl = sum;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        int run = incl - sum;
#pragma unroll
        for (int k = 0; k < per; ++k) { s_cnt[lane * per + k] = run; run += v[k]; }
    }
    __syncthreads();
    const int64_t tile_off = tile_offsets[blockIdx.x];
    const unsigned lt = (1u << lane) - 1u;
    const int64_t gg = g * g;
#pragma unroll
    for (int r = 0; r < kThrRows; ++r) {
        if (ball[r] & (1u << lane)) {
            const int64_t e = base + (int64_t)r * kThrThreads + threadIdx.x;
            const int64_t pos = tile_off + s_cnt[r * kThrWarps + warp] + __popc(ball[r] & lt);
            if (g > 0) {
                const int64_t ix = e / gg;
                const int64_t rem = e - ix * gg;
                const int64_t iy = rem / g;
                idx[3 * pos + 0] = ix;
                idx[3 * pos + 1] = iy;
                idx[3 * pos + 2] = rem - iy * g;
            } else {
                idx[pos] = e;
            }
        }
    }
}

static int64_t ntiles_for(int64_t n) { return (n + kThrTile - 1) / kThrTile; }

}  // namespace divas

using namespace divas;

extern "C" size_t divas_threshold_workspace_size(int64_t n) {
    const int64_t nt = ntiles_for(n > 0 ? n : 0);
    // tile counts + an occupancy scratch plane when the caller passes occ == NULL
    return 256 + (size_t)nt * sizeof(int64_t) + (size_t)((n + 255) / 256) * 256;
}

extern "C" int divas_threshold(const double *p, int64_t n, double thr, int64_t g, uint8_t *occ,
                               int64_t *idx, int64_t *count, void *workspace,
                               size_t workspace_bytes, void *stream) {
    if (n < 0 || !p || !workspace) { set_error("divas_threshold: bad arguments"); return DIVAS_EINVAL; }
    if (g > 0 && g * g * g != n) { set_error("divas_threshold: n != g^3"); return DIVAS_EINVAL; }
    if (workspace_bytes < divas_threshold_workspace_size(n)) {
        set_error("divas_threshold: workspace too small");
        return DIVAS_EWORKSPACE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nt = ntiles_for(n);
    int64_t *tiles = (int64_t *)((char *)workspace + 256);
    uint8_t *occ_buf = occ ? occ : (uint8_t *)(tiles + nt);
    if (n == 0) {
        if (count && cudaMemsetAsync(count, 0, sizeof(int64_t), s) != cudaSuccess)
            return check_launch("divas_threshold(memset)");
        return DIVAS_OK;
    }
    if (nt > 0x7fffffffLL) { set_error("divas_threshold: too many tiles"); return DIVAS_EINVAL; }
    thr_mark<<<(unsigned)nt, kThrThreads, 0, s>>>(p, n, thr, occ_buf, tiles);
    int rc = check_launch("divas_threshold(mark)");
    if (rc) return rc;
    if (!idx && !count) return DIVAS_OK;
    int64_t *cnt = count ? count : (int64_t *)workspace;
    thr_scan<<<1, 1024, 0, s>>>(tiles, nt, cnt);
    rc = check_launch("divas_threshold(scan)");
    if (rc || !idx) return rc;
    thr_emit<<<(unsigned)nt, kThrThreads, 0, s>>>(occ_buf, n, g, tiles, idx);
    return check_launch("divas_threshold(emit)");
}

// ---------------------------------------------------------------------------
// .vgrid payload: p [ix][iy][iz] f64 -> f32 in x-fastest order [iz][iy][ix]
// (io.write_vgrid, /root/reference/pkg/src/divas/io.py:59-69).  32x32 tiles of
// the (ix, iz) plane of one iy through shared memory: coalesced both ways.
// ---------------------------------------------------------------------------
namespace divas {
__global__ void vgrid_transpose(const double *__restrict__ p, float *__restrict__ out, int64_t g) {
    __shared__ float tile[32][33];
    const int64_t iy = blockIdx.z;
    const int64_t ix0 = (int64_t)blockIdx.y * 32, iz0 = (int64_t)blockIdx.x * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {      // read rows ix, columns iz
        const int64_t ix = ix0 + r, iz = iz0 + threadIdx.x;
        if (ix < g && iz < g) tile[r][threadIdx.x] = (float)p[(ix * g + iy) * g + iz];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {      // write rows iz, columns ix
        const int64_t iz = iz0 + r, ix = ix0 + threadIdx.x;
        if (ix < g && iz < g) out[(iz * g + iy) * g + ix] = tile[threadIdx.x][r];
    }
}
}  // namespace divas

extern "C" int divas_vgrid_payload(const double *p, int64_t g, float *out, void *stream) {
    if (!p || !out || g < 1 || g > 65535) { set_error("divas_vgrid_payload: bad arguments"); return DIVAS_EINVAL; }
    dim3 grid((unsigned)((g + 31) / 32), (unsigned)((g + 31) / 32), (unsigned)g);
    divas::vgrid_transpose<<<grid, dim3(32, 8), 0, (cudaStream_t)stream>>>(p, out, g);
    return check_launch("divas_vgrid_payload");
}
