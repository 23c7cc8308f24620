// fuse.cu -- kernel (b): multi-view voxel fusion.
//
// Reference: fusion._fuse_kernel -> _voxel_views (/root/reference/pkg/src/divas/
// fusion.py:493-509, :410-490) with its helpers _project_px (:170-184),
// _pixel_index (:187-192), _grad_at (:195-229, padded-plane semantics of
// _gradient_maps :684-689), _contract_pt (:243-254), _thick_pair (:257-303),
// _thin_pair (:306-370) and the value-sorted sums (:373-407).
//
// Three launches on the caller's stream, no host synchronisation:
//
//   fuse_gate    dense stream over the slab [lo, hi): 16-byte rho loads, 32-byte
//                zero stores of p (and optional votes / occupancy) and a
//                warp-aggregated append of every voxel that clears the exact
//                density gate  rho >= rho_thr || (enable_thin && rho >= rho_thin)
//                to the slot list.  Below both gates no pair can vote, so p = 0
//                exactly ("exact shortcuts").
//   fuse_pairs   one thread per (view, gated voxel) pair; grid (slots, views),
//                so a CTA works on one view and its 256 threads on adjacent
//                voxels: their centre pixels and footprints are neighbours in
//                the same view plane (L1/L2 locality).  Decisions that hinge on
//                a floor / compare of a projected coordinate are CERTIFIED with
//                a cheap reciprocal-based projection plus a rigorous error
//                margin; only pairs within the margin of a boundary (or that
//                reach the thick spatial test, which needs the exact u, v)
//                evaluate the reference's exact IEEE division chain.  Every
//                vote-deciding quantity is therefore bit-identical to numba's.
//                Contributions land in [view][slot] arrays with one bit per
//                (slot, view) set by atomicOr.
//   fuse_reduce  one thread per gated voxel: gathers its flagged contributions,
//                sorts them (w, then m*w; t) and sums in the reference's
//                value-sorted order -> p bit-identical under view permutation,
//                writes p, votes, sums and the fused occupancy.
//
// Arithmetic: IEEE f64 in the reference's evaluation order, no FMA contraction
// (the TU is compiled with -fmad=false; explicit fma() appears only inside the
// certified approximations), binary32 exactly at the 8 numba f32 sites.
#include <algorithm>
#include <cstring>

#include <cstdio>

#include "bands.cuh"
#include "exp_cr.cuh"

namespace divas {

struct FuseConst {
    int64_t g, lo, hi;
    double origin0, origin1, origin2, dx;
    int nv, hm, wm, w32;
    int64_t cap;   // slot capacity of the workspace (max gated voxels)
    int view0;     // first view of the pair launch (incremental updates)
    double gamma, beta, bmax, lam, rho_thr, rho_thin, thin_pct, alpha1, thin_accept, eps,
        mask_thr, thin_floor, kappa;
    int enable_thin;
    int band_ok;         // thin_percent_cover > 0: zero support can never vote
    int ntx, nty;        // depth-band tiles per view
    double cube_r;       // circumradius of a voxel, padded
    double tau_max;      // (2 gamma + bmax) dx >= tau_d(n) for every n
    double bc0, bc1, bc2, bh0, bh1, bh2;
    int unbounded;
    double occ_thr;
    int gshift;          // log2(g) when g is a power of two, else -1
    unsigned long long *fallbacks;   // exact-chain counters (DIVAS_FB_*), or NULL
    int cull;            // tile-level band rejection allowed (tile_culled)
};

// Count one exact-chain evaluation (rare sites only; no-op without counters).
__device__ __forceinline__ void fallback(const FuseConst &C, int i) {
    if (C.fallbacks) atomicAdd(C.fallbacks + i, 1ull);
}

// (ix, iy, iz) of a flat voxel index: shifts for power-of-two grids
__device__ __forceinline__ void voxel_coords(const FuseConst &C, uint32_t vi, uint32_t &ix,
                                             uint32_t &iy, uint32_t &iz) {
    if (C.gshift >= 0) {
        const uint32_t m = (1u << C.gshift) - 1u;
        ix = vi >> (2 * C.gshift);
        iy = (vi >> C.gshift) & m;
        iz = vi & m;
    } else {
        const uint32_t g = (uint32_t)C.g, gg = g * g;
        ix = vi / gg;
        const uint32_t rem = vi - ix * gg;
        iy = rem / g;
        iz = rem - iy * g;
    }
}

struct FuseOut {
    double *probs;
    int32_t *n_thick, *n_thin;
    double *sw, *smw, *st;
    uint8_t *occ;
    uint8_t *const *occ_peers;   // fused slab all-gather: every rank's buffer
    int n_peers;
};

struct FuseMaps {
    const float *masks, *dmins, *dmaxs, *dexps;
    const int32_t *nsamps;
    const double2 *bands;   // [nv][nty][ntx] depth bands (bands.cuh)
    const float2 *rec;      // [nv][2][hm][wm] scan record planes A, B (bands.cuh)
};

struct Contrib {                 // all [view or word][cap]
    uint32_t *bits_thick, *bits_thin;
    double *w, *mw, *t;
};

struct WsHeader {
    unsigned long long count;    // gated voxels found
    unsigned int overflow;       // count > cap
    unsigned int pad;
    unsigned long long reserved;
};

// ---------------------------------------------------------------------------
// dense gate pass
// ---------------------------------------------------------------------------
constexpr int kGateThreads = 256;

__device__ __forceinline__ bool density_gate(float rho, const FuseConst &C) {
    const double r = (double)rho;
    return r >= C.rho_thr || (C.enable_thin && r >= C.rho_thin);
}

// One quad = up to 4 consecutive voxels base + [k0, k1) (k0 > 0 or k1 < 4 where
// the range or the grid row ends): loads rho (one float4 when the whole quad
// is valid and aligned), zeroes the outputs (unless count_only) and returns
// the density-gate bits of the valid voxels.
__device__ __forceinline__ unsigned gate_quad(const float *__restrict__ dens, const FuseConst &C,
                                              const FuseOut &O, int64_t base, int k0, int k1,
                                              bool vec_ok, bool count_only) {
    if (k1 <= k0) return 0u;
    const bool full = vec_ok && k0 == 0 && k1 == 4;
    const uint8_t occ0 = (0.0 >= C.occ_thr) ? 1 : 0;
    float r[4] = {0.f, 0.f, 0.f, 0.f};
    if (full) {
        const float4 v = __ldg(reinterpret_cast<const float4 *>(dens + base));
        r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w;
    } else {
        for (int k = k0; k < k1; ++k) r[k] = __ldg(dens + base + k);
    }
    if (!count_only) {
        if (full) {
            const double2 z2 = make_double2(0.0, 0.0);
            if (O.probs) {
                __stcs(reinterpret_cast<double2 *>(O.probs + base), z2);
                __stcs(reinterpret_cast<double2 *>(O.probs + base) + 1, z2);
            }
            if (O.n_thick) *reinterpret_cast<int4 *>(O.n_thick + base) = make_int4(0, 0, 0, 0);
            if (O.n_thin) *reinterpret_cast<int4 *>(O.n_thin + base) = make_int4(0, 0, 0, 0);
            double *sums[3] = {O.sw, O.smw, O.st};
            for (int s = 0; s < 3; ++s)
                if (sums[s]) {
                    reinterpret_cast<double2 *>(sums[s] + base)[0] = z2;
                    reinterpret_cast<double2 *>(sums[s] + base)[1] = z2;
                }
            if (O.occ) *reinterpret_cast<uchar4 *>(O.occ + base) = make_uchar4(occ0, occ0, occ0, occ0);
            for (int p = 0; p < O.n_peers; ++p)           // NVLink stores to every rank
                *reinterpret_cast<uchar4 *>(O.occ_peers[p] + base) =
                    make_uchar4(occ0, occ0, occ0, occ0);
        } else {
            for (int k = k0; k < k1; ++k) {
                if (O.probs) O.probs[base + k] = 0.0;
                if (O.n_thick) O.n_thick[base + k] = 0;
                if (O.n_thin) O.n_thin[base + k] = 0;
                if (O.sw) O.sw[base + k] = 0.0;
                if (O.smw) O.smw[base + k] = 0.0;
                if (O.st) O.st[base + k] = 0.0;
                if (O.occ) O.occ[base + k] = occ0;
                for (int p = 0; p < O.n_peers; ++p) O.occ_peers[p][base + k] = occ0;
            }
        }
    }
    unsigned bits = 0;
    for (int k = k0; k < k1; ++k)
        if (density_gate(r[k], C)) bits |= 1u << k;
    return bits;
}

// A flat-range quad (the counting pass): voxels [base, base + 4) cut to [lo, hi)
__device__ __forceinline__ unsigned gate_flat_quad(const float *__restrict__ dens,
                                                   const FuseConst &C, const FuseOut &O,
                                                   int64_t base, bool count_only) {
    const int64_t left = C.hi - base;
    const int k1 = left < 4 ? (int)left : 4;
    return gate_quad(dens, C, O, base, 0, k1, (C.lo & 3) == 0, count_only);
}

// Brick tiles for the ordered gate: 16 x 16 x 16 voxels; quad j of a brick
// is (ix, iy) = (j / 64, (j / 4) % 16) and iz = 4 (j % 4) .. +3 locally.
constexpr int kBrick = 16;
struct BrickGrid {
    int64_t ix0;      // first ix of the range
    int nbx, nby, nbz;
};

// A brick's origin voxel, once per CTA (tile = blockIdx.x)
struct BrickOrigin {
    int64_t ix, iy, iz;
};

__device__ __forceinline__ BrickOrigin brick_origin(const BrickGrid &G, uint32_t tile) {
    const uint32_t bz = tile % (uint32_t)G.nbz;
    const uint32_t t1 = tile / (uint32_t)G.nbz;
    const uint32_t by = t1 % (uint32_t)G.nby;
    const uint32_t bx = t1 / (uint32_t)G.nby;
    return BrickOrigin{G.ix0 + (int64_t)bx * kBrick, (int64_t)by * kBrick, (int64_t)bz * kBrick};
}

// Slot order inside a brick (the order gate_emit lists gated voxels in):
// quad j (0..1023; a quad = 4 voxels along iz) -> brick-local quad coordinates
// (qx, qy, qz) in 0..15 x 0..15 x 0..3.  Consecutive runs are compact blocks:
// 8 quads (a warp's 32 slots when all are gated) = 2 x 4 x 4 voxels, 64 quads
// (a pair CTA's 256 slots) = 8 x 8 x 4 voxels, consecutive 64-quad tiles step
// along iz.  Compact blocks keep a pair CTA's footprints overlapping (L1
// reuse) and its bounding box small (tile_cull).
__device__ __forceinline__ void brick_quad_xyz(int j, int &qx, int &qy, int &qz) {
    const int T = j >> 6, u = j & 63;                 // 8x8x1-quad tile, quad in tile
    const int w8 = u >> 3, v = u & 7;                 // 2x4-quad chunk, quad in chunk
    qx = 8 * (T >> 3) + 2 * (w8 >> 1) + (v >> 2);
    qy = 8 * ((T >> 2) & 1) + 4 * (w8 & 1) + (v & 3);
    qz = T & 3;
}

__device__ __forceinline__ unsigned gate_brick_quad(const float *__restrict__ dens,
                                                    const FuseConst &C, const FuseOut &O,
                                                    const BrickOrigin &Bo, int j,
                                                    bool count_only, int64_t &base_out) {
    int qx, qy, qz;
    brick_quad_xyz(j, qx, qy, qz);
    const int64_t ix = Bo.ix + qx;
    const int64_t iy = Bo.iy + qy;
    const int64_t iz = Bo.iz + 4 * qz;
    const int64_t g = C.g;
    base_out = (ix * g + iy) * g + iz;
    if (ix >= g || iy >= g || iz >= g) return 0u;
    // valid part of the quad: inside the row and inside [lo, hi)
    const int64_t rowleft = g - iz, before = C.lo - base_out, after = C.hi - base_out;
    int k0 = 0, k1 = rowleft < 4 ? (int)rowleft : 4;
    if (before > 0) k0 = before < 4 ? (int)before : 4;
    if (after < k1) k1 = after > 0 ? (int)after : 0;
    return gate_quad(dens, C, O, base_out, k0, k1, (g & 3) == 0, count_only);
}
// Counting pass (divas_gate_count): grid-stride over quads, one atomic per
// warp that found gated voxels.
__global__ void __launch_bounds__(kGateThreads)
fuse_gate_count(const float *__restrict__ dens, FuseConst C, WsHeader *__restrict__ hdr) {
    const int64_t nquads = (C.hi - C.lo + 3) / 4;
    const FuseOut none{};
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
         q - (threadIdx.x & 31) < nquads; q += (int64_t)gridDim.x * blockDim.x) {
        const unsigned bits = q < nquads ? gate_flat_quad(dens, C, none, C.lo + 4 * q, true) : 0u;
        int cnt = __popc(bits);
        if (__ballot_sync(0xffffffffu, cnt != 0) == 0) continue;
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if ((threadIdx.x & 31) == 0) atomicAdd(&hdr->count, (unsigned long long)cnt);
    }
}

// Ordered gate, pass 1: tiles of kGateTile voxels; zero the outputs and count
// each tile's gated voxels.  Quad j of a tile is handled by thread j % 256 in
// round j / 256, so the rounds walk the tile in C order.
constexpr int kGateRounds = 4;                     // quads per thread per 16^3 brick
constexpr int kGateTile = 4 * kGateRounds * kGateThreads;   // 4096 = 16^3
constexpr int64_t kGateTileMax = (1LL << 32) / kGateTile;   // tiles of any u32 voxel range

template <bool ZERO>
__global__ void __launch_bounds__(kGateThreads)
gate_tiles(const float *__restrict__ dens, FuseConst C, FuseOut O, BrickGrid G,
           uint32_t *__restrict__ tiles) {
    griddep_wait();                     // PDL: after the previous kernel completes
    __shared__ int s_w[kGateThreads / 32];
    int cnt = 0;
    int64_t base;
    const BrickOrigin Bo = brick_origin(G, blockIdx.x);
    const int64_t g = C.g, gg = g * g;
    // interior brick (the common case): inside the grid, inside [lo, hi),
    // quads aligned -- one float4 per quad, no per-quad bounds logic; round r
    // of thread t is quad t + 256 r, i.e. 4 ix planes further
    if ((g & 3) == 0 && Bo.ix + kBrick <= g && Bo.iy + kBrick <= g && Bo.iz + kBrick <= g &&
        C.lo <= Bo.ix * gg && C.hi >= (Bo.ix + kBrick) * gg) {
        const int t = (int)threadIdx.x;
        base = ((Bo.ix + (t >> 6)) * g + Bo.iy + ((t >> 2) & 15)) * g + Bo.iz + 4 * (t & 3);
        const uint8_t occ0 = (0.0 >= C.occ_thr) ? 1 : 0;
        const double2 z2 = make_double2(0.0, 0.0);
#pragma unroll
        for (int r = 0; r < kGateRounds; ++r, base += (kGateThreads / 64) * gg) {
            // (DIVAS_GATE_STREAM=1: evict-first rho loads / occupancy stores,
            // measured +2.5 us on the overlapped step: off)
#ifndef DIVAS_GATE_STREAM
#define DIVAS_GATE_STREAM 0
#endif
            const float4 v = DIVAS_GATE_STREAM ? __ldcs(reinterpret_cast<const float4 *>(dens + base))
                                               : __ldg(reinterpret_cast<const float4 *>(dens + base));
            if (ZERO && O.probs) {
                __stcs(reinterpret_cast<double2 *>(O.probs + base), z2);
                __stcs(reinterpret_cast<double2 *>(O.probs + base) + 1, z2);
            }
            if (ZERO && (O.n_thick || O.n_thin || O.sw || O.smw || O.st)) {   // stats (rare)
                if (O.n_thick) *reinterpret_cast<int4 *>(O.n_thick + base) = make_int4(0, 0, 0, 0);
                if (O.n_thin) *reinterpret_cast<int4 *>(O.n_thin + base) = make_int4(0, 0, 0, 0);
                double *sums[3] = {O.sw, O.smw, O.st};
                for (int q = 0; q < 3; ++q)
                    if (sums[q]) {
                        reinterpret_cast<double2 *>(sums[q] + base)[0] = z2;
                        reinterpret_cast<double2 *>(sums[q] + base)[1] = z2;
                    }
            }
            const uchar4 o4 = make_uchar4(occ0, occ0, occ0, occ0);
            if (ZERO && O.occ) {
                if (DIVAS_GATE_STREAM) __stcs(reinterpret_cast<char4 *>(O.occ + base),
                                              *reinterpret_cast<const char4 *>(&o4));
                else *reinterpret_cast<uchar4 *>(O.occ + base) = o4;
            }
            if (ZERO)
                for (int p = 0; p < O.n_peers; ++p)
                    *reinterpret_cast<uchar4 *>(O.occ_peers[p] + base) = o4;
            cnt += (int)density_gate(v.x, C) + (int)density_gate(v.y, C) +
                   (int)density_gate(v.z, C) + (int)density_gate(v.w, C);
        }
    } else {
#pragma unroll
        for (int r = 0; r < kGateRounds; ++r)
            cnt += __popc(gate_brick_quad(dens, C, O, Bo, r * kGateThreads + (int)threadIdx.x,
                                          !ZERO, base));
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < kGateThreads / 32; ++w) t += s_w[w];
        tiles[blockIdx.x] = (uint32_t)t;
    }
}

// pass 2 (one CTA): exclusive scan of the tile counts in place; the total is
// the gated count, beyond `cap` the overflow flag.  Each thread scans 4
// consecutive counts per round (a 16^3-brick grid of 256^3 is one round).
__global__ void __launch_bounds__(1024)
gate_scan(uint32_t *__restrict__ tiles, int64_t ntiles, int64_t cap, WsHeader *__restrict__ hdr) {
    griddep_wait();                     // PDL: after the previous kernel completes
    __shared__ unsigned long long s_w[32];
    __shared__ unsigned long long s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t b = 0; b < ntiles; b += 4 * (int64_t)blockDim.x) {
        const int64_t i0 = b + 4 * (int64_t)threadIdx.x;
        unsigned long long v[4], t = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[k] = i0 + k < ntiles ? tiles[i0 + k] : 0ull;
            t += v[k];
        }
        unsigned long long incl = t;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_w[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const unsigned long long w = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0ull;
            unsigned long long wi = w;
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += y;
            }
            s_w[lane] = wi - w;
        }
        __syncthreads();
        const unsigned long long carry = s_carry;
        unsigned long long run = carry + s_w[warp] + incl - t;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (i0 + k < ntiles) tiles[i0 + k] = (uint32_t)run;
            run += v[k];
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry = run;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        hdr->count = s_carry;
        hdr->overflow = s_carry > (unsigned long long)cap ? 1u : 0u;
    }
}

// pass 3: each gated voxel's C-order rank -> its slot (deterministic order);
// tiles without a gated voxel (most of the grid) return at once
__global__ void __launch_bounds__(kGateThreads)
gate_emit(const float *__restrict__ dens, FuseConst C, BrickGrid G,
          const uint32_t *__restrict__ tiles, int64_t ntiles, const WsHeader *__restrict__ hdr,
          uint32_t *__restrict__ work) {
    griddep_wait();                     // PDL: after the previous kernel completes
    constexpr int NW = kGateThreads / 32;
    constexpr int NC = kGateRounds * NW;               // (round, warp) chunks, C order
    static_assert(NC % 32 == 0, "chunk scan");
    __shared__ int s_pre[NC];
    const int64_t off = tiles[blockIdx.x];
    const int64_t end = (int64_t)blockIdx.x + 1 < ntiles ? (int64_t)tiles[blockIdx.x + 1]
                                                          : (int64_t)hdr->count;
    if (end == off) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const FuseOut none{};
    unsigned bits[kGateRounds];
    int lp[kGateRounds];
    int64_t qbase[kGateRounds];
    const BrickOrigin Bo = brick_origin(G, blockIdx.x);
    const int64_t g = C.g, gg = g * g;
    // interior brick: the lean quad walk of gate_tiles
    const bool interior = (g & 3) == 0 && Bo.ix + kBrick <= g && Bo.iy + kBrick <= g &&
                          Bo.iz + kBrick <= g && C.lo <= Bo.ix * gg &&
                          C.hi >= (Bo.ix + kBrick) * gg;
    const int t = (int)threadIdx.x;
#pragma unroll
    for (int r = 0; r < kGateRounds; ++r) {
        if (interior) {
            int qx, qy, qz;
            brick_quad_xyz(r * kGateThreads + t, qx, qy, qz);
            qbase[r] = ((Bo.ix + qx) * g + Bo.iy + qy) * g + Bo.iz + 4 * qz;
            const float4 v = __ldg(reinterpret_cast<const float4 *>(dens + qbase[r]));
            bits[r] = (density_gate(v.x, C) ? 1u : 0u) | (density_gate(v.y, C) ? 2u : 0u) |
                      (density_gate(v.z, C) ? 4u : 0u) | (density_gate(v.w, C) ? 8u : 0u);
        } else {
            bits[r] = gate_brick_quad(dens, C, none, Bo, r * kGateThreads + t, true, qbase[r]);
        }
        const int c = __popc(bits[r]);
        int incl = c;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        lp[r] = incl - c;
        if (lane == 31) s_pre[r * NW + warp] = incl;
    }
    __syncthreads();
    if (warp == 0) {   // exclusive scan of the chunk totals, NC / 32 per lane
        constexpr int PER = NC / 32;
        int v[PER], sum = 0;
#pragma unroll
        for (int k = 0; k < PER; ++k) { v[k] = s_pre[lane * PER + k]; sum += v[k]; }
        int incl = sum;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        int run = incl - sum;
#pragma unroll
        for (int k = 0; k < PER; ++k) { s_pre[lane * PER + k] = run; run += v[k]; }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kGateRounds; ++r) {
        unsigned b = bits[r];
        int64_t pos = off + s_pre[r * NW + warp] + lp[r];
        const int64_t base = qbase[r];
        while (b) {
            const int k = __ffs(b) - 1;
            b &= b - 1;
            if (pos < C.cap) work[pos] = (uint32_t)(base + k);
            ++pos;
        }
    }
}

// Zero fill of the outputs on [lo, hi) alone (DIVAS_STEP_ZERO): p (f64) and
// the optional votes / sums / occupancy / peer buffers, 16-byte streaming
// stores over aligned 16-voxel groups, scalar stores at the range ends.  The
// exact value every voxel outside the density gate keeps (p = 0, occupancy
// 0 >= occ_thr).
__global__ void __launch_bounds__(256)
fuse_zero(FuseConst C, FuseOut O) {
    const uint8_t occ0 = (0.0 >= C.occ_thr) ? 1 : 0;
    const int64_t a = (C.lo + 15) & ~(int64_t)15, b = C.hi & ~(int64_t)15;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    auto scalar = [&](int64_t i) {
        if (O.probs) O.probs[i] = 0.0;
        if (O.n_thick) O.n_thick[i] = 0;
        if (O.n_thin) O.n_thin[i] = 0;
        if (O.sw) O.sw[i] = 0.0;
        if (O.smw) O.smw[i] = 0.0;
        if (O.st) O.st[i] = 0.0;
        if (O.occ) O.occ[i] = occ0;
        for (int p = 0; p < O.n_peers; ++p) O.occ_peers[p][i] = occ0;
    };
    if (b <= a) {                                   // tiny range: scalar only
        for (int64_t i = C.lo + tid; i < C.hi; i += nth) scalar(i);
        return;
    }
    for (int64_t i = C.lo + tid; i < a; i += nth) scalar(i);
    for (int64_t i = b + tid; i < C.hi; i += nth) scalar(i);
    const double2 z2 = make_double2(0.0, 0.0);
    const int4 zi = make_int4(0, 0, 0, 0);
    const uint32_t o1 = occ0 * 0x01010101u;
    const uint4 o16 = make_uint4(o1, o1, o1, o1);
    for (int64_t g = a / 16 + tid; g < b / 16; g += nth) {      // 16 voxels per thread
        const int64_t i = g * 16;
        if (O.probs) {
            double2 *q = reinterpret_cast<double2 *>(O.probs + i);
#pragma unroll
            for (int k = 0; k < 8; ++k) __stcs(q + k, z2);
        }
        if (O.n_thick || O.n_thin || O.sw || O.smw || O.st) {
            int32_t *iv[2] = {O.n_thick, O.n_thin};
            for (int s = 0; s < 2; ++s)
                if (iv[s])
                    for (int k = 0; k < 4; ++k) reinterpret_cast<int4 *>(iv[s] + i)[k] = zi;
            double *dv[3] = {O.sw, O.smw, O.st};
            for (int s = 0; s < 3; ++s)
                if (dv[s])
                    for (int k = 0; k < 8; ++k) reinterpret_cast<double2 *>(dv[s] + i)[k] = z2;
        }
        if (O.occ) *reinterpret_cast<uint4 *>(O.occ + i) = o16;
        for (int p = 0; p < O.n_peers; ++p) *reinterpret_cast<uint4 *>(O.occ_peers[p] + i) = o16;
    }
}

// ---------------------------------------------------------------------------
// exact restatement of the reference helpers
// ---------------------------------------------------------------------------
struct Cam {
    double r[9];   // row-major: r[row*3 + col]
    double p0, p1, p2, fx, fy, cx, cy, w, h;
};

__device__ __forceinline__ void load_cam(const double *__restrict__ c, Cam &k) {
#pragma unroll
    for (int i = 0; i < 9; ++i) k.r[i] = __ldg(c + i);
    k.p0 = __ldg(c + 9); k.p1 = __ldg(c + 10); k.p2 = __ldg(c + 11);
    k.fx = __ldg(c + 12); k.fy = __ldg(c + 13); k.cx = __ldg(c + 14); k.cy = __ldg(c + 15);
    k.w = __ldg(c + 16); k.h = __ldg(c + 17);
}

// _project_px (fusion.py:170-184); returns in_front, writes u, v, d
__device__ __forceinline__ bool project_px(const Cam &k, double px, double py, double pz,
                                           double &u, double &v, double &d) {
    const double relx = px - k.p0;
    const double rely = py - k.p1;
    const double relz = pz - k.p2;
    const double zc = k.r[2] * relx + k.r[5] * rely + k.r[8] * relz;
    d = -zc;
    if (d <= 0.0) { u = -1.0; v = -1.0; return false; }
    const double xc = k.r[0] * relx + k.r[3] * rely + k.r[6] * relz;
    const double yc = k.r[1] * relx + k.r[4] * rely + k.r[7] * relz;
    u = (k.fx * (xc / d) + k.cx) / k.w;
    v = (k.cy - k.fy * (yc / d)) / k.h;
    return true;
}

// _pixel_index (fusion.py:187-192)
__device__ __forceinline__ long long pixel_index(double u, long long n) {
    long long i = nb_floor_int(u * (double)n);
    if (i > n - 1) i = n - 1;
    return i;
}

// _grad_at over the padded (hm, wm) plane (fusion.py:195-229, :684-689)
__device__ __forceinline__ double grad_at(const float *__restrict__ dexp,
                                          const float *__restrict__ dmin,
                                          const float *__restrict__ dmax, int hm, int wm, int ix,
                                          int iy, double eps, double kappa) {
    const int64_t c = (int64_t)iy * wm + ix;
    const float center = __ldg(dexp + c);
    const float r32 = __ldg(dmax + c) - __ldg(dmin + c);            // f32 site
    const double rng = (double)r32 + eps;
    double gmax = 0.0, s;
    if (ix > 0) {
        s = (double)fabsf(__ldg(dexp + c - 1) - center) / rng;      // f32 site
        if (s > gmax) gmax = s;
    }
    if (ix < wm - 1) {
        s = (double)fabsf(__ldg(dexp + c + 1) - center) / rng;
        if (s > gmax) gmax = s;
    }
    if (iy > 0) {
        s = (double)fabsf(__ldg(dexp + c - wm) - center) / rng;
        if (s > gmax) gmax = s;
    }
    if (iy < hm - 1) {
        s = (double)fabsf(__ldg(dexp + c + wm) - center) / rng;
        if (s > gmax) gmax = s;
    }
    double g = 1.0 / (1.0 + kappa * gmax);
    const double hi = 1.0 - eps;
    if (g > hi) g = hi;
    if (g < 0.0) g = 0.0;
    return g;
}

// _grad_at from pre-loaded centre / neighbour values with one division:
// fl(a / rng) is monotone in a for rng > 0, so the max over neighbours
// commutes with the division (NaN differences never win in either form);
// the 4-division form (grad_at) otherwise.  f32 sites: fl(|nb - centre|).
__device__ __forceinline__ double grad_from(float center, float dmin, float dmax, float nl,
                                            float nr, float nu, float nd, const float *dexp,
                                            const float *dmins, const float *dmaxs,
                                            const FuseConst &C, int ix, int iy) {
    const float r32 = dmax - dmin;                                  // f32 site
    const double rng = (double)r32 + C.eps;
    if (!(rng > 0.0)) return grad_at(dexp, dmins, dmaxs, C.hm, C.wm, ix, iy, C.eps, C.kappa);
    float amax = 0.0f;
    amax = fmaxf(amax, fabsf(nl - center));                         // f32 sites
    amax = fmaxf(amax, fabsf(nr - center));
    amax = fmaxf(amax, fabsf(nu - center));
    amax = fmaxf(amax, fabsf(nd - center));
    const double gmax = amax > 0.0f ? (double)amax / rng : 0.0;
    double g = 1.0 / (1.0 + C.kappa * gmax);
    const double hi = 1.0 - C.eps;
    if (g > hi) g = hi;
    if (g < 0.0) g = 0.0;
    return g;
}

// _thick_pair's spatial half and weight (fusion.py:268-303).  The depth test
// |x_d - dexp| <= tau_dp is evaluated by the caller first: both are pure, so
// the conjunction's value is unchanged.
__device__ __forceinline__ bool thick_spatial(const FuseConst &C, const Cam &k, double xc0,
                                           double xc1, double xc2, double u, double v,
                                           float dmin, float dmax, double g, double &wd) {
    const double *R = k.r;
    const double rx = (u * k.w - k.cx) / k.fx;
    const double ry = (k.cy - v * k.h) / k.fy;
    double ddx = R[0] * rx + R[1] * ry - R[2];
    double ddy = R[3] * rx + R[4] * ry - R[5];
    double ddz = R[6] * rx + R[7] * ry - R[8];
    const double norm = sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
    ddx /= norm;
    ddy /= norm;
    ddz /= norm;
    const double t_proj = ((xc0 - k.p0) * ddx + (xc1 - k.p1) * ddy + (xc2 - k.p2) * ddz);
    double t_c = t_proj;
    if (t_c < (double)dmin) t_c = (double)dmin;
    else if (t_c > (double)dmax) t_c = (double)dmax;
    double pcx = k.p0 + ddx * t_c;
    double pcy = k.p1 + ddy * t_c;
    double pcz = k.p2 + ddz * t_c;
    if (C.unbounded != 0) {   // _contract_pt (fusion.py:243-254)
        const double nx = (pcx - C.bc0) / C.bh0;
        const double ny = (pcy - C.bc1) / C.bh1;
        const double nz = (pcz - C.bc2) / C.bh2;
        const double r = sqrt(nx * nx + ny * ny + nz * nz);
        if (r > 1.0) {
            const double s = (2.0 - 1.0 / r) / r;
            pcx = C.bc0 + nx * s * C.bh0;
            pcy = C.bc1 + ny * s * C.bh1;
            pcz = C.bc2 + nz * s * C.bh2;
        }
    }
    const double dx = xc0 - pcx;
    const double dy = xc1 - pcy;
    const double dz = xc2 - pcz;
    const double delta = sqrt(dx * dx + dy * dy + dz * dz);
    const float span = dmax - dmin;                                   // f32 site
    const double tau_sp = C.dx * g + C.lam * (double)span;
    if (!(delta <= tau_sp)) return false;
    const float msum = dmin + dmax;                                   // f32 site
    const double mu = 0.5 * (double)msum;
    double hd = 0.5 * (double)span;                                   // f32 site
    if (hd < C.eps) hd = C.eps;
    const double r = fabs(t_c - mu) / hd;
    wd = exp_ref(-C.alpha1 * r * r);
    return true;
}

// ---------------------------------------------------------------------------
// certified fast projection
// ---------------------------------------------------------------------------
// f32 reciprocal seed on the MUFU (rcp.approx: relative error < 2^-22 after
// the f64 -> f32 rounding of the argument); subnormal / overflowing arguments
// give inf / 0, which the callers' range guards keep out of every decision.
__device__ __forceinline__ double rcp_seed(double d) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"((float)d));
    return (double)r;
}

// Reciprocal accurate to ~1 ulp: seed + two Newton steps in f64.  Only used
// inside certified approximations (never for an output bit); callers pass
// 1e-30 < d < 1e30.
__device__ __forceinline__ double rcp_fast(double d) {
    double r = rcp_seed(d);
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}

// Relative error bound of the certified projections.  The exact chain
// (fl(fl(fl(fx * fl(x/d)) + cx) / w) * w, 5 roundings) and the approximation
// (rcp_fast, 3 roundings) each deviate from the real value by < 1e-15 times
// the magnitudes involved; 1e-11 leaves four orders of magnitude of slack.
constexpr double kCertRel = 1e-11;

// floor(U) certified for |U - exact| <= E; returns false when undecidable.
__device__ __forceinline__ bool cert_floor(double U, double E, long long &out) {
    // (|f| < 2^30: a 32-bit conversion; larger coordinates -- far outside any
    // image -- take the exact chain)
    const double f = floor(U);
    if (U - f > E && (f + 1.0) - U > E && fabs(f) < 1073741824.0) {
        out = (long long)__double2int_rz(f);
        return true;
    }
    return false;
}

// Classify one image axis of the centre projection from the approximation
// Ua ~= fl(u * n) (== numerator of u).  0: certainly outside [0, 1);
// 1: certainly inside with pixel idx; 2: undecided.
__device__ __forceinline__ int cert_axis(double Ua, double E, double n, long long &idx) {
    if (Ua < -E || Ua >= n + E) return 0;
    if (Ua > E && Ua < n - E && cert_floor(Ua, E, idx)) return 1;
    return 2;
}

// ---------------------------------------------------------------------------
// pair kernel
// ---------------------------------------------------------------------------
constexpr int kPairThreads = 256;

// Debug builds (-DDIVAS_CHECK=1, tests only): trap on any out-of-range read.
#if DIVAS_CHECK
#define DIVAS_BOUND(ptr, base, n)                                                          \
    do {                                                                                   \
        if ((ptr) < (base) || (ptr) >= (base) + (n)) {                                     \
            printf("divas bound check failed at %s:%d\n", __FILE__, __LINE__);              \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define DIVAS_BOUND(ptr, base, n) ((void)0)
#endif

#if DIVAS_STATS
// experiment builds only: per-stage pair counters (tools/pair_stats.py)
__device__ unsigned long long g_pair_stats[24];
#define PSTAT(i, v) atomicAdd(&g_pair_stats[i], (unsigned long long)(v))
#else
#define PSTAT(i, v) ((void)0)
#endif

// (2 gamma + min(beta * n, bmax)) * dx, the reference's ops (fusion.py:362-365)
__device__ __forceinline__ double tau_thin(const FuseConst &C, int32_t n) {
    double b = C.beta * (double)n;
    if (b > C.bmax) b = C.bmax;
    return (2.0 * C.gamma + b) * C.dx;
}

// Reciprocal for certified bounds: seed + one Newton step (rel. error
// < 2^-43, far inside kCertRel); 1e-30 < d < 1e30.
__device__ __forceinline__ double rcp_fast1(double d) {
    const double r = rcp_seed(d);
    return fma(r, fma(-d, r, 1.0), r);
}

// 1/sqrt(x) to ~1 ulp: the MUFU seed + two Newton steps in f64 (certified
// approximations only; 1e-300 < x < 1e300)
__device__ __forceinline__ double rsqrt_fast(double x) {
    double y = (double)rsqrtf((float)x);
    const double h = 0.5 * x;
    y = y * fma(-h * y, y, 1.5);
    y = y * fma(-h * y, y, 1.5);
    return y;
}

// branch-free min / max of finite doubles (fmin / fmax carry NaN handling)
__device__ __forceinline__ double dmin2(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double dmax2(double a, double b) { return b > a ? b : a; }

// _thin_pair (fusion.py:306-370): footprint bounds from the 8 projected
// corners.  floor(fl(umin * w)) = min_j floor(fl(u_j * w)) (floor and
// rounding are monotone), and |min_j a_j - min_j b_j| <= max_j |a_j - b_j|, so
// it suffices to certify the floors of the approximate min / max with a bound
// valid for every corner.  Corner camera coordinates are the centre's plus
// +-half * rotation offsets; their distance to the reference's exact chain
// is below eabs.  Undecided cases (and corners near the camera plane) run
// the reference's exact corner chain.
__device__ __forceinline__ bool thin_bounds(const FuseConst &C, const Cam &k, double xc0,
                                            double xc1, double xc2, double d_c, double x_c,
                                            double y_c, long long &xs, long long &xe,
                                            long long &ys, long long &ye) {
    const double half = 0.5 * C.dx;
    const double *R = k.r;
    const double S = fabs(xc0) + fabs(xc1) + fabs(xc2) + fabs(k.p0) + fabs(k.p1) + fabs(k.p2) +
                     3.0 * half;
    const double eabs = 4e-15 * S;
    const double rho = C.cube_r;
    const double dmn = d_c - rho;                  // every corner is at least this deep
    if (dmn > 2.0 * eabs && dmn > 1e-30 && d_c < 1e30) {
        // corner j = (sx, sy, sz) of half * (+-R col) offsets; corners j and
        // 7 - j are opposite (negated offsets), so four offset triples give
        // all eight: with p = a + b, m = a - b the sz = -1 corners are
        // -p - c, m - c, -m - c, p - c
        const double az = half * R[2], bz = half * R[5], cz_ = half * R[8];
        const double fax = k.fx * (half * R[0]), fbx = k.fx * (half * R[3]), fcx = k.fx * (half * R[6]);
        const double fay = k.fy * (half * R[1]), fby = k.fy * (half * R[4]), fcy = k.fy * (half * R[7]);
        const double pz = az + bz, mz = az - bz, pu = fax + fbx, mu = fax - fbx;
        const double pv = fay + fby, mv = fay - fby;
        const double Z[4] = {-pz - cz_, mz - cz_, -mz - cz_, pz - cz_};
        const double Uo[4] = {-pu - fcx, mu - fcx, -mu - fcx, pu - fcx};
        const double Vo[4] = {-pv - fcy, mv - fcy, -mv - fcy, pv - fcy};
        const double FX = k.fx * x_c, FY = k.fy * y_c;
        double umin = 0.0, umax = 0.0, vmin = 0.0, vmax = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const double r1 = rcp_fast1(d_c - Z[j]), r2 = rcp_fast1(d_c + Z[j]);
            const double U1 = (FX + Uo[j]) * r1, U2 = (FX - Uo[j]) * r2;
            const double V1 = (FY + Vo[j]) * r1, V2 = (FY - Vo[j]) * r2;
            const bool uu = U1 < U2, vv = V1 < V2;
            const double ulo = uu ? U1 : U2, uhi = uu ? U2 : U1;
            const double vlo = vv ? V1 : V2, vhi = vv ? V2 : V1;
            umin = j ? dmin2(umin, ulo) : ulo;
            umax = j ? dmax2(umax, uhi) : uhi;
            vmin = j ? dmin2(vmin, vlo) : vlo;
            vmax = j ? dmax2(vmax, vhi) : vhi;
        }
        const double idm = rcp_fast1(dmn) * (1.0 + 1e-9);
        const double mx = fabs(x_c) + rho, my = fabs(y_c) + rho;
        const double EU = kCertRel * (k.fx * mx * idm + fabs(k.cx) + 1.0) +
                          4.0 * k.fx * eabs * (d_c + rho + mx) * idm * idm;
        const double EV = kCertRel * (k.fy * my * idm + fabs(k.cy) + 1.0) +
                          4.0 * k.fy * eabs * (d_c + rho + my) * idm * idm;
        if (cert_floor(umin + k.cx, EU, xs) && cert_floor(umax + k.cx, EU, xe) &&
            cert_floor(k.cy - vmax, EV, ys) && cert_floor(k.cy - vmin, EV, ye))
            return true;
    }
    PSTAT(13, 1);
    fallback(C, DIVAS_FB_CORNERS);
    // exact corner chain (fusion.py:315-341)
    double umn = 1e30, umx = -1e30, vmn = 1e30, vmx = -1e30;
#pragma unroll 1
    for (int j = 0; j < 8; ++j) {
        const double sx = ((j & 1) == 0) ? -1.0 : 1.0;
        const double sy = ((j & 2) == 0) ? -1.0 : 1.0;
        const double sz = ((j & 4) == 0) ? -1.0 : 1.0;
        double cu, cv, cd;
        if (!project_px(k, xc0 + sx * half, xc1 + sy * half, xc2 + sz * half, cu, cv, cd))
            return false;
        if (cu < umn) umn = cu;
        if (cu > umx) umx = cu;
        if (cv < vmn) vmn = cv;
        if (cv > vmx) vmx = cv;
    }
    xs = nb_floor_int(umn * k.w);
    xe = nb_floor_int(umx * k.w);
    ys = nb_floor_int(vmn * k.h);
    ye = nb_floor_int(vmx * k.h);
    return true;
}

// Exact rejection through the depth bands (bands.cuh): the footprint box lies
// within +-R pixels of the centre projection, R bounding the projected
// circumsphere of the voxel.  Returns true when no box pixel can support x_d.
__device__ __forceinline__ bool band_reject(const FuseConst &C, const FuseMaps &M, const Cam &k,
                                            int view, double x_d, double xcam, double ycam,
                                            double Uc, double Vc) {
#ifndef DIVAS_BANDR
#define DIVAS_BANDR 1
#endif
#if DIVAS_BANDR
    // per-axis extent of the cube in camera coordinates: the corners are
    // (xcam, ycam, x_d) + h (+-R0 +-R1 +-R2) along the camera axes, so
    // |dx| <= h (|r0| + |r3| + |r6|), |dy| <= h (|r1| + |r4| + |r7|),
    // |dz| <= h (|r2| + |r5| + |r8|); the projected offset of a corner from
    // the centre is fx (dx x_d - xcam dz) / (x_d (x_d + dz)), bounded below
    // with dz = -Dz.  A margin far above every rounding (0.01 px) keeps the
    // footprint box inside [Uc - Ru, Uc + Ru].
    const double h = 0.5 * C.dx;
    const double Dx = h * (fabs(k.r[0]) + fabs(k.r[3]) + fabs(k.r[6]));
    const double Dy = h * (fabs(k.r[1]) + fabs(k.r[4]) + fabs(k.r[7]));
    const double Dz = h * (fabs(k.r[2]) + fabs(k.r[5]) + fabs(k.r[8]));
    const double den = x_d * (x_d - Dz);
    if (!(x_d > 2.0 * Dz && den > 1e-30 && den < 1e30)) return false;
    const double inv = rcp_fast1(den) * (1.0 + 1e-9);
    const double Ru = k.fx * (Dx * x_d + fabs(xcam) * Dz) * inv * (1.0 + 1e-9) + 0.01;
    const double Rv = k.fy * (Dy * x_d + fabs(ycam) * Dz) * inv * (1.0 + 1e-9) + 0.01;
#else
    const double rho = C.cube_r;
    const double den = x_d * (x_d - rho);
    if (!(x_d > 2.0 * rho && den > 1e-30 && den < 1e30)) return false;
    const double inv = rcp_fast1(den) * (1.0 + 1e-9);
    const double Ru = k.fx * rho * (x_d + fabs(xcam)) * inv + 2.0;
    const double Rv = k.fy * rho * (x_d + fabs(ycam)) * inv + 2.0;
#endif
    const double fx0 = floor((Uc - Ru) * (1.0 / kBandTile)), fx1 = floor((Uc + Ru) * (1.0 / kBandTile));
    const double fy0 = floor((Vc - Rv) * (1.0 / kBandTile)), fy1 = floor((Vc + Rv) * (1.0 / kBandTile));
    const int tx0 = (int)fmax(fx0, 0.0), tx1 = (int)fmin(fx1, (double)(C.ntx - 1));
    const int ty0 = (int)fmax(fy0, 0.0), ty1 = (int)fmin(fy1, (double)(C.nty - 1));
    if (tx1 < tx0 || ty1 < ty0) return false;
    if ((tx1 - tx0 + 1) * (ty1 - ty0 + 1) > kBandMaxTiles) {
        PSTAT(15, 1);
        fallback(C, DIVAS_FB_BAND_WIDE);
        return false;
    }
    const double2 *bv = M.bands + (int64_t)view * band_view_stride(C.nty, C.ntx);
    // tiles in row-major order, four loads in flight per round trip (indices
    // past the last tile repeat it: always in range, never changes the answer)
    const int nx = tx1 - tx0 + 1;
    const int nt = nx * (ty1 - ty0 + 1);
    PSTAT(7, nt);
    const int skip = C.ntx - nx;
    const double2 *__restrict__ bp = bv + ty0 * C.ntx + tx0;
    int left = nx;
    for (int i0 = 0; i0 < nt; i0 += 4) {
        double2 b[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            DIVAS_BOUND(bp, bv, (int64_t)C.nty * C.ntx);
            b[j] = __ldg(bp);
            if (i0 + j + 1 < nt) {
                ++bp;
                if (--left == 0) { left = nx; bp += skip; }
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (x_d >= b[j].x && x_d <= b[j].y) return false;   // this tile may support
    }
    return true;
}

// Certified thick spatial test (fusion.py:268-296).  u, v are the projection
// of the voxel centre X, so the reference's ray through (u, v) passes through X
// up to rounding: dd ~ rel / |rel|, t_proj ~ |rel|, and the closest point of
// the clamped segment is pos + dd * clamp(t_proj).  The approximations below
// are within E of the exact chain's values; decisions farther than E from a
// boundary are certain.  Returns 1 = ok, 0 = not ok, 2 = undecided (run the
// exact chain).  On ok, `tc` is the clamped parameter when the clamp is
// certain (then equal to dmin or dmax exactly) and `need_exact_t` tells
// whether the weight needs the exact t_proj.
__device__ __forceinline__ int thick_certified(const FuseConst &C, const Cam &k, double xc0,
                                               double xc1, double xc2, double relx, double rely,
                                               double relz, float dmin, float dmax, double g,
                                               double &tc, bool &need_exact_t) {
    const double L2 = relx * relx + rely * rely + relz * relz;
    if (!(L2 > 1e-300 && L2 < 1e300)) return 2;
    const double rL = rsqrt_fast(L2);                 // ~1 ulp: certified below
    const double L = L2 * rL;
    const double scale = fabs(xc0) + fabs(xc1) + fabs(xc2) + fabs(k.p0) + fabs(k.p1) +
                         fabs(k.p2) + L + fabs((double)dmin) + fabs((double)dmax) + 1.0;
    double E = 1e-10 * scale;
    if (C.unbounded)
        E *= 16.0 * fmax(fmax(C.bh0, C.bh1), C.bh2) /
             fmin(fmin(C.bh0, C.bh1), C.bh2);
    const double lo = (double)dmin, hi = (double)dmax;
    int clamp;                       // -1: t = dmin, +1: t = dmax, 0: t = t_proj
    if (L < lo - E) clamp = -1;
    else if (L > hi + E && L > lo + E) clamp = 1;
    else if (L > lo + E && L < hi - E) clamp = 0;
    else return 2;
    const double t_c = clamp < 0 ? lo : (clamp > 0 ? hi : L);
    double pcx, pcy, pcz;
    if (clamp == 0) {
        pcx = xc0; pcy = xc1; pcz = xc2;          // the ray point at t_proj is X
    } else {
        const double s = t_c * rL;
        pcx = k.p0 + relx * s;
        pcy = k.p1 + rely * s;
        pcz = k.p2 + relz * s;
    }
    if (C.unbounded != 0) {
        const double nx = (pcx - C.bc0) / C.bh0;
        const double ny = (pcy - C.bc1) / C.bh1;
        const double nz = (pcz - C.bc2) / C.bh2;
        const double r = sqrt(nx * nx + ny * ny + nz * nz);
        if (fabs(r - 1.0) < 1e-9) return 2;       // contraction branch undecided
        if (r > 1.0) {
            const double sc = (2.0 - 1.0 / r) / r;
            pcx = C.bc0 + nx * sc * C.bh0;
            pcy = C.bc1 + ny * sc * C.bh1;
            pcz = C.bc2 + nz * sc * C.bh2;
        }
    }
    const double ex = xc0 - pcx, ey = xc1 - pcy, ez = xc2 - pcz;
    const double d2 = ex * ex + ey * ey + ez * ez;    // delta^2: no sqrt needed
    const float span = dmax - dmin;                                   // f32 site
    const double tau_sp = C.dx * g + C.lam * (double)span;
    const double thi = tau_sp + E, tlo = tau_sp - E;
    if (d2 > thi * thi) return 0;
    if (tlo > 0.0 && d2 < tlo * tlo) {
        tc = t_c;
        need_exact_t = clamp == 0;
        return 1;
    }
    return 2;
}

// Depth weight from the clamped parameter (fusion.py:297-302).
__device__ __forceinline__ double depth_weight(const FuseConst &C, double t_c, float dmin,
                                               float dmax) {
    const float span = dmax - dmin;                                   // f32 site
    const float msum = dmin + dmax;                                   // f32 site
    const double mu = 0.5 * (double)msum;
    double hd = 0.5 * (double)span;
    if (hd < C.eps) hd = C.eps;
    const double r = fabs(t_c - mu) / hd;
    return exp_ref(-C.alpha1 * r * r);
}

// The exact t_proj of the reference's chain (fusion.py:268-277).
__device__ __forceinline__ double exact_tproj(const Cam &k, double xc0, double xc1, double xc2,
                                              double u, double v) {
    const double *R = k.r;
    const double rx = (u * k.w - k.cx) / k.fx;
    const double ry = (k.cy - v * k.h) / k.fy;
    double ddx = R[0] * rx + R[1] * ry - R[2];
    double ddy = R[3] * rx + R[4] * ry - R[5];
    double ddz = R[6] * rx + R[7] * ry - R[8];
    const double norm = sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
    ddx /= norm;
    ddy /= norm;
    ddz /= norm;
    return ((xc0 - k.p0) * ddx + (xc1 - k.p1) * ddy + (xc2 - k.p2) * ddz);
}

#ifndef DIVAS_QSMALL
#define DIVAS_QSMALL 1
#endif
struct QItem {                  // a thin candidate that survived the band test
    uint32_t slot, vi;
#if !DIVAS_QSMALL
    double x_d, xcam, ycam;
#endif
};

constexpr int kQueue = kPairThreads;
#ifndef DIVAS_CARVEOUT
#define DIVAS_CARVEOUT (DIVAS_QSMALL ? 7 : 25)
#endif
constexpr int kPairCarveout = DIVAS_CARVEOUT;      // % of the unified L1 / shared memory

// Per-lane part of one (view, voxel) pair: centre projection, routing, the
// thick path, the thin gates and the band test.  Returns true when the pair
// needs corner projections + a footprint scan.
__device__ __forceinline__ bool pair_route(const FuseConst &C, const Cam &k, const float *dens,
                                           const FuseMaps &M, const Contrib &K, uint32_t vi,
                                           int view, int64_t kidx, int64_t bidx, uint32_t bit,
                                           double &x_d_out, double &xcam_out, double &ycam_out) {
    uint32_t ix, iy, iz;
    voxel_coords(C, vi, ix, iy, iz);
    const double rho = (double)__ldg(dens + vi);
    const double xc0 = C.origin0 + ((double)ix + 0.5) * C.dx;
    const double xc1 = C.origin1 + ((double)iy + 0.5) * C.dx;
    const double xc2 = C.origin2 + ((double)iz + 0.5) * C.dx;

    // centre projection: exact camera-frame coordinates (no division)
    const double relx = xc0 - k.p0;
    const double rely = xc1 - k.p1;
    const double relz = xc2 - k.p2;
    const double zc = k.r[2] * relx + k.r[5] * rely + k.r[8] * relz;
    const double x_d = -zc;
    PSTAT(0, 1);
    if (!(x_d > 0.0)) return false;                            // behind the camera
    const double xcam = k.r[0] * relx + k.r[3] * rely + k.r[6] * relz;
    const double ycam = k.r[1] * relx + k.r[4] * rely + k.r[7] * relz;

    // frustum + pixel: certified from one reciprocal, exact chain otherwise
    double A, B;
    long long px, py;
    int cu = 2, cv = 2;
    if (x_d > 1e-30 && x_d < 1e30) {
        const double r = rcp_fast(x_d);
        A = k.fx * xcam * r;
        B = k.fy * ycam * r;
        cu = cert_axis(A + k.cx, kCertRel * (fabs(A) + fabs(k.cx) + 1.0), k.w, px);
        cv = cert_axis(k.cy - B, kCertRel * (fabs(B) + fabs(k.cy) + 1.0), k.h, py);
        if (cu == 0 || cv == 0) return false;
    }
    if (cu == 2 || cv == 2) {
        A = k.fx * (xcam / x_d);
        B = k.fy * (ycam / x_d);
        const double u = (A + k.cx) / k.w;
        const double v = (k.cy - B) / k.h;
        if (u < 0.0 || u >= 1.0 || v < 0.0 || v >= 1.0) return false;
        px = pixel_index(u, (long long)k.w);
        py = pixel_index(v, (long long)k.h);
    }
    PSTAT(1, 1);
    if (cu == 2 || cv == 2) {
        PSTAT(14, 1);
        fallback(C, DIVAS_FB_CENTRE);
    }
    const int64_t plane = (int64_t)C.hm * C.wm;
    const int64_t vplane = (int64_t)view * plane;
    const int64_t q = py * (int64_t)C.wm + px;
    const int64_t pix = vplane + q;
    const float2 *recA = M.rec + 2 * vplane;                   // this view's record planes
    DIVAS_BOUND(recA + q, recA, plane);
    const float2 ra = __ldg(recA + q);                         // {m, d_exp or NaN}
    const int32_t ns = __ldg(M.nsamps + pix);
    const float m = fabsf(ra.x);                              // sign: the tau flag
    // neither path can take a centre mask below both gates, whatever the
    // pixel's validity: return without waiting for n_samples
    if (!((double)m >= C.mask_thr) && !((double)m > C.thin_floor)) return false;
    if (ns <= 0) return false;                                 // valids[view, py, px] == 0
    PSTAT(2, 1);
#if defined(DIVAS_ABL) && DIVAS_ABL >= 3
    K.t[kidx] = (double)m;
    return false;
#endif

    if ((double)m >= C.mask_thr && rho >= C.rho_thr) {
        // plane A holds d_exp only where a thin candidate could be supported
        const float dexp = (ra.y == ra.y) ? ra.y : __ldg(M.dexps + pix);
        PSTAT(3, 1);
        double b = C.beta * (double)ns;
        if (b > C.bmax) b = C.bmax;
        const double tau_dp = (C.gamma + b) * C.dx;
        if (fabs(x_d - (double)dexp) <= tau_dp) {
            PSTAT(4, 1);
            // dmin, dmax and the four neighbour depths in one round trip; a
            // missing neighbour reads the centre itself (|d - d| = 0 never
            // raises the max, exactly like skipping it)
            const float *de = M.dexps + pix;
            DIVAS_BOUND(de - (px > 0 ? 1 : 0), M.dexps + vplane, (int64_t)C.hm * C.wm);
            DIVAS_BOUND(de + (py < C.hm - 1 ? C.wm : 0), M.dexps + vplane, (int64_t)C.hm * C.wm);
            const float dmin = __ldg(M.dmins + pix), dmax = __ldg(M.dmaxs + pix);
            const float nl = __ldg(de - (px > 0 ? 1 : 0));
            const float nr = __ldg(de + (px < C.wm - 1 ? 1 : 0));
            const float nu = __ldg(de - (py > 0 ? C.wm : 0));
            const float nd = __ldg(de + (py < C.hm - 1 ? C.wm : 0));
            const double gr = grad_from(dexp, dmin, dmax, nl, nr, nu, nd, M.dexps + vplane,
                                        M.dmins + vplane, M.dmaxs + vplane, C, (int)px, (int)py);
            double t_c = 0.0;
            bool need_t = false;
            int ok = thick_certified(C, k, xc0, xc1, xc2, relx, rely, relz, dmin, dmax, gr, t_c,
                                     need_t);
            double wd = 0.0;
            if (ok == 1) {
                if (need_t) {
                    fallback(C, DIVAS_FB_THICK_T);
                    const double u = (k.fx * (xcam / x_d) + k.cx) / k.w;
                    const double v = (k.cy - k.fy * (ycam / x_d)) / k.h;
                    t_c = exact_tproj(k, xc0, xc1, xc2, u, v);
                    if (t_c < (double)dmin) t_c = (double)dmin;
                    else if (t_c > (double)dmax) t_c = (double)dmax;
                }
                wd = depth_weight(C, t_c, dmin, dmax);
            } else if (ok == 2) {                  // exact reference chain
                PSTAT(12, 1);
                fallback(C, DIVAS_FB_THICK);
                const double u = (k.fx * (xcam / x_d) + k.cx) / k.w;
                const double v = (k.cy - k.fy * (ycam / x_d)) / k.h;
                ok = thick_spatial(C, k, xc0, xc1, xc2, u, v, dmin, dmax, gr, wd) ? 1 : 0;
            }
            if (ok == 1) {
                K.w[kidx] = wd;
                K.mw[kidx] = (double)m * wd;
                atomicOr(K.bits_thick + bidx, bit);
                PSTAT(5, 1);
                return false;                                  // routed thick
            }
        }
    }
#if defined(DIVAS_ABL) && DIVAS_ABL >= 2
    return false;
#endif
    if (!C.enable_thin) return false;
    if (!((double)m > C.thin_floor && rho >= C.rho_thin)) return false;
    {   // dx_vox * fmax / x_d >= 1.0, certified (division monotone and correctly rounded)
        const double fmax = k.fx > k.fy ? k.fx : k.fy;
        const double a = C.dx * fmax;
        if (a < x_d * (1.0 - 1e-12)) return false;
        if (!(a > x_d * (1.0 + 1e-12))) {
            fallback(C, DIVAS_FB_THIN_GATE);
            if (!(a / x_d >= 1.0)) return false;
        }
    }
    PSTAT(6, 1);
    if (C.band_ok && band_reject(C, M, k, view, x_d, xcam, ycam, A + k.cx, k.cy - B))
        return false;                                          // support is exactly 0
    PSTAT(8, 1);
    x_d_out = x_d;
    xcam_out = xcam;
    ycam_out = ycam;
    return true;
}

// Footprint scan of one box, row by row (groups of four records at constant
// offsets, then a pair and a single for the row's remainder).  Per record
// {m, D}: m_max in f32 (widening is exact and monotone: fmaxf equals the
// reference's f64 `if mv > m_max`; NaN never wins), e = |f32(x_d) - D| - tau
// decides support when |e| >= Mg (see thin_item), and the smallest |e| tells
// whether any record fell inside the margin.  MODE 0: one tau per view
// (plane A alone); 1: the base tau, a flagged record (negative m) also makes
// the item unsure; 2: per-record tau from plane B.  Returns "unsure".
// -1 when a <= b, else 0 (NaN compares false): one FSET, so a count is one
// add per record instead of a compare, an increment and a select
__device__ __forceinline__ int le_mask(float a, float b) {
    int m;
    asm("set.le.s32.f32 %0, %1, %2;" : "=r"(m) : "f"(a), "f"(b));
    return m;
}

template <int MODE>
__device__ __forceinline__ bool scan_box(const float2 *__restrict__ rp, int wm, int64_t plane,
                                         int bw, int bh, float xd32, float tau, float Mg,
                                         int &sup, float &mmax) {
    float emin = __int_as_float(0x7f800000);   // +inf
    float fmin_ = 0.0f;                         // most negative m (MODE 1 flags)
    const float nMg = -Mg;
    auto pix = [&](float2 r, float t) {
        mmax = fmaxf(mmax, fabsf(r.x));
        const float e = fabsf(xd32 - r.y) - (MODE == 2 ? t : tau);
        sup -= le_mask(e, nMg);                  // e <= -Mg (NaN: no)
        emin = fminf(emin, fabsf(e));
        if (MODE == 1) fmin_ = fminf(fmin_, r.x);
    };
    const int rem = bw & 3;
    const int full = bw - rem;
    for (int y = 0; y < bh; ++y, rp += wm) {
        int c = 0;
        for (; c < full; c += 4) {
            const float2 *q = rp + c;
            float2 r[4];
            float t[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                r[j] = __ldg(q + j);
                t[j] = MODE == 2 ? __ldg(q + j + plane).x : 0.0f;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) pix(r[j], t[j]);
        }
        const float2 *q = rp + c;
        if (rem & 2) {
            const float2 r0 = __ldg(q), r1 = __ldg(q + 1);
            const float t0 = MODE == 2 ? __ldg(q + plane).x : 0.0f;
            const float t1 = MODE == 2 ? __ldg(q + 1 + plane).x : 0.0f;
            pix(r0, t0);
            pix(r1, t1);
            q += 2;
        }
        if (rem & 1) pix(__ldg(q), MODE == 2 ? __ldg(q + plane).x : 0.0f);
    }
    return emin < Mg || (MODE == 1 && fmin_ < 0.0f);
}

// Exact f32 support interval of a thin candidate with one tau (MODE 0 / 1):
// a record depth D (f32, widened exactly) supports x_d iff the reference's
// f64 test |x_d - D| <= tau holds (fusion.py:361-367).  fl(x_d - D) is
// monotone in D, so the f32 depths that pass form one interval [lo, hi]; its
// ends lie within an ulp of fl32(x_d -+ tau) and are found by evaluating the
// reference's own test on the neighbouring f32 values.  The scan then decides
// each pixel with two f32 compares, exactly (NaN depth -- an ineligible
// pixel -- fails both).  Returns false (the caller recounts in f64) when the
// interval reaches non-positive depths or an end does not settle.
__device__ __forceinline__ float f32_up(float f) {      // next f32 above f > 0
    return __int_as_float(__float_as_int(f) + 1);
}
__device__ __forceinline__ float f32_down(float f) {    // next f32 below f > 0
    return __int_as_float(__float_as_int(f) - 1);
}
__device__ __forceinline__ bool support_interval(double xd, double tau, float &lo, float &hi) {
    // straight-line (no data-dependent loop: lanes must enter the scan
    // together): fl32(x_d +- tau) is within an ulp of each end, so the end is
    // one of its neighbours; the next neighbour outward must fail the test
    auto ok = [&](float D) { return fabs(xd - (double)D) <= tau; };
    const double a = xd - tau, b = xd + tau;
    const float h0 = __double2float_rn(b), l0 = __double2float_rn(a);
    const float hm = f32_down(h0), hp = f32_up(h0), hq = f32_up(hp);
    const float lp = f32_up(l0), lm = f32_down(l0), lq = f32_down(lm);
    const bool okhm = ok(hm), okh0 = ok(h0), okhp = ok(hp), okhq = ok(hq);
    const bool oklp = ok(lp), okl0 = ok(l0), oklm = ok(lm), oklq = ok(lq);
    hi = okhp ? hp : (okh0 ? h0 : hm);
    lo = oklm ? lm : (okl0 ? l0 : lp);
    // each side's candidates lie on its own side of x_d (there the test is
    // monotone in D), the inner ones pass, the outer ones fail
    return a > 1e-30 && b < 1e30 && lq > 0.0f && (double)hm > xd && (double)lp < xd && okhm &&
           oklp && !okhq && !oklq;
}

// -1 when lo <= D <= hi, else 0 (NaN: 0), branch-free: one FSETP + one FSET
__device__ __forceinline__ int in_mask(float D, float lo, float hi) {
    int m;
    asm("{\n\t.reg .pred p;\n\tsetp.ge.f32 p, %1, %2;\n\tset.le.and.s32.f32 %0, %1, %3, p;\n\t}"
        : "=r"(m) : "f"(D), "f"(lo), "f"(hi));
    return m;
}

// Footprint scan with an exact interval (MODE 0: one tau per view; MODE 1:
// the base tau, and a flagged record -- negative m, its tau differs -- makes
// the item unsure).  Same row walk as scan_box.  Returns "unsure" (MODE 1
// flags only).
template <int MODE>
__device__ __forceinline__ bool scan_exact(const float2 *__restrict__ rp, int wm, int bw, int bh,
                                           float lo, float hi, int &sup, float &mmax) {
    float fmin_ = 0.0f;
    auto pix = [&](float2 r) {
        mmax = fmaxf(mmax, fabsf(r.x));
        sup -= in_mask(r.y, lo, hi);
        if (MODE == 1) fmin_ = fminf(fmin_, r.x);
    };
    const int rem = bw & 3;
    const int full = bw - rem;
#ifndef DIVAS_SCAN_2ROWS
#define DIVAS_SCAN_2ROWS 1
#endif
    int y = 0;
    if (DIVAS_SCAN_2ROWS) {
        // two rows per pass: eight loads in flight per group, the loop
        // bookkeeping shared by both rows
#pragma unroll 1
        for (; y + 1 < bh; y += 2, rp += 2 * wm) {
            const float2 *rq = rp + wm;
            int c = 0;
#pragma unroll 1
            for (; c < full; c += 4) {
                float2 r[8];
#pragma unroll
                for (int j = 0; j < 4; ++j) { r[j] = __ldg(rp + c + j); r[4 + j] = __ldg(rq + c + j); }
#pragma unroll
                for (int j = 0; j < 8; ++j) pix(r[j]);
            }
            if (rem & 2) {
                const float2 a0 = __ldg(rp + c), a1 = __ldg(rp + c + 1);
                const float2 b0 = __ldg(rq + c), b1 = __ldg(rq + c + 1);
                pix(a0); pix(a1); pix(b0); pix(b1);
                c += 2;
            }
            if (rem & 1) { const float2 a0 = __ldg(rp + c), b0 = __ldg(rq + c); pix(a0); pix(b0); }
        }
    }
#pragma unroll 1
    for (; y < bh; ++y, rp += wm) {
        int c = 0;
#pragma unroll 1
        for (; c < full; c += 4) {
            const float2 *q = rp + c;
            float2 r[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) r[j] = __ldg(q + j);
#pragma unroll
            for (int j = 0; j < 4; ++j) pix(r[j]);
        }
        const float2 *q = rp + c;
        if (rem & 2) {
            const float2 r0 = __ldg(q), r1 = __ldg(q + 1);
            pix(r0);
            pix(r1);
            q += 2;
        }
        if (rem & 1) pix(__ldg(q));
    }
    return MODE == 1 && fmin_ < 0.0f;
}

// Corner projections + footprint scan of one queued thin candidate.
__device__ __forceinline__ void thin_item(const FuseConst &C, const Cam &k, const FuseMaps &M,
                                          const Contrib &K, int view,
                                          const QItem &q) {
    uint32_t ix, iy, iz;
    voxel_coords(C, q.vi, ix, iy, iz);
    const double xc0 = C.origin0 + ((double)ix + 0.5) * C.dx;
    const double xc1 = C.origin1 + ((double)iy + 0.5) * C.dx;
    const double xc2 = C.origin2 + ((double)iz + 0.5) * C.dx;
#if DIVAS_QSMALL
    // the camera-frame centre again, the very operations of pair_route (so
    // bit-identical): a queue item is 8 bytes, which leaves the pair kernel
    // a 16 KB shared-memory carve-out and 240 KB of L1 for the scans
    const double relx = xc0 - k.p0, rely = xc1 - k.p1, relz = xc2 - k.p2;
    const double q_x_d = -(k.r[2] * relx + k.r[5] * rely + k.r[8] * relz);
    const double q_xcam = k.r[0] * relx + k.r[3] * rely + k.r[6] * relz;
    const double q_ycam = k.r[1] * relx + k.r[4] * rely + k.r[7] * relz;
#else
    const double q_x_d = q.x_d, q_xcam = q.xcam, q_ycam = q.ycam;
#endif
    long long xs, xe, ys, ye;
    if (!thin_bounds(C, k, xc0, xc1, xc2, q_x_d, q_xcam, q_ycam, xs, xe, ys, ye)) return;
    const long long wi = (long long)k.w, hi = (long long)k.h;
    if (xe < 0 || xs > wi - 1 || ye < 0 || ys > hi - 1) return;
    if (xs < 0) xs = 0;
    if (ys < 0) ys = 0;
    if (xe > wi - 1) xe = wi - 1;
    if (ye > hi - 1) ye = hi - 1;
#if defined(DIVAS_ABL) && DIVAS_ABL >= 1
    K.t[(int64_t)view * C.cap + q.slot] = q_x_d + (double)(xe - xs);
    return;
#endif
    // Footprint scan over record plane A {m, D (NaN: cannot support)} and,
    // for views whose supporting pixels do not share one tau, plane B {tau32,
    // n}.  m_max: f32 widening is exact and monotone, so fmaxf in f32 equals
    // the reference's f64 `if mv > m_max` (NaN never wins).  Support: the f32
    // margin test e = |f32(x_d) - D| - tau32 has |error| < 2^-22 (|x_d| +
    // tau_max); beyond M = 2^-20 (|x_d| + tau_max) from 0 it decides the
    // reference's f64 test |x_d - f64(D)| <= tau(n) exactly, inside M the f64
    // test runs.  NaN D (mask <= 0.5 or n == 0) never counts, never is unsure.
    const int64_t plane = (int64_t)C.hm * C.wm;
    const float2 *__restrict__ recA = M.rec + 2 * (int64_t)view * plane;
    const float2 *__restrict__ rp = recA + ys * (int64_t)C.wm + xs;
    const uint32_t *te = reinterpret_cast<const uint32_t *>(
        M.bands + (int64_t)view * band_view_stride(C.nty, C.ntx) + (int64_t)C.nty * C.ntx);
    const uint32_t tk0 = __ldg(te), tk1 = __ldg(te + 1);
    const uint32_t nflag = __ldg(te + 2), nsup = __ldg(te + 3);
    const double xd = q_x_d;
    const float xd32 = (float)xd;
    const float Mg = (float)(9.5367431640625e-07 * (fabs(xd) + C.tau_max));   // 2^-20
    const int bw = (int)(xe - xs) + 1;
    const int npix = bw * ((int)(ye - ys) + 1);
    PSTAT(9, npix);
    const int bh = (int)(ye - ys) + 1;
    int sup = 0;
    float mmax = 0.0f;
    bool unsure;
    const bool one_tau = tk0 >= tk1;                  // one tau for every supporting pixel
    const bool few_flags = !one_tau && (uint64_t)nflag * 32u <= nsup;
    float ilo = 0.0f, ihi = 0.0f;
    bool exact_ok = false;
    // the exact interval needs the f64 tau the reference uses: tau_thin(n)
    // from the n range of the view's supporting pixels (one f64 tau when its
    // ends agree), or the base n whose f64 tau every unflagged pixel shares
    const uint32_t nlo = __ldg(te + 5), nhi = __ldg(te + 6), nbase = __ldg(te + 7);
#ifndef DIVAS_EXACT_SCAN
#define DIVAS_EXACT_SCAN 1
#endif
    const bool single = DIVAS_EXACT_SCAN &&
                        (nlo > nhi || tau_thin(C, (int32_t)nlo) == tau_thin(C, (int32_t)nhi));
    if (!DIVAS_EXACT_SCAN) {
    } else if (single) {                                      // (no supporting pixel: any tau)
        exact_ok = support_interval(xd, tau_thin(C, nlo > nhi ? 1 : (int32_t)nlo), ilo, ihi);
    } else if (few_flags && nbase > 0) {
        exact_ok = support_interval(xd, tau_thin(C, (int32_t)nbase), ilo, ihi);
    }
    if (exact_ok && single) {
        unsure = scan_exact<0>(rp, C.wm, bw, bh, ilo, ihi, sup, mmax);
    } else if (exact_ok) {
        // few supporting pixels differ from the base tau: scan with the base
        // tau, a flagged pixel (negative mask) sends the item to the recount
        unsure = scan_exact<1>(rp, C.wm, bw, bh, ilo, ihi, sup, mmax);
    } else if (one_tau) {
        unsure = scan_box<0>(rp, C.wm, plane, bw, bh, xd32, __uint_as_float(tk0), Mg,
                             sup, mmax);
    } else if (few_flags) {
        unsure = scan_box<1>(rp, C.wm, plane, bw, bh, xd32, __uint_as_float(__ldg(te + 4)),
                             Mg, sup, mmax);
    } else {
        unsure = scan_box<2>(rp, C.wm, plane, bw, bh, xd32, 0.0f, Mg, sup, mmax);
    }
    if (unsure) {
        PSTAT(10, 1);
        fallback(C, DIVAS_FB_RECOUNT);
    }
    if (unsure) {   // some pixel within the margin: recount with the reference's f64 test
        sup = 0;
        const int32_t *np = M.nsamps + (int64_t)view * plane + ys * (int64_t)C.wm + xs;
        const float2 *__restrict__ pp = rp;
        for (int y = 0; y < bh; ++y, pp += C.wm, np += C.wm)
            for (int c = 0; c < bw; ++c) {
                const float2 r = __ldg(pp + c);
                sup += (r.y == r.y && fabs(xd - (double)r.y) <= tau_thin(C, __ldg(np + c))) ? 1 : 0;
            }
    }
    const double m_max = (double)mmax;
    const double p_cov = sup == 0 ? 0.0 : (double)sup / (double)npix;
    const double t = (p_cov >= C.thin_pct) ? m_max : p_cov;
    if (m_max < C.thin_accept) { PSTAT(16, 1); PSTAT(17, npix); }   // no vote possible
    if (sup == 0) { PSTAT(18, 1); PSTAT(19, npix); }
    if (sup == npix) { PSTAT(20, 1); PSTAT(21, npix); }
    if (npix >= 64) { PSTAT(22, 1); PSTAT(23, npix); }
    if (npix > 0 && t >= C.thin_accept) {
        K.t[(int64_t)view * C.cap + q.slot] = t;
        PSTAT(11, 1);
        atomicOr(K.bits_thin + (int64_t)(view >> 5) * C.cap + q.slot, 1u << (view & 31));
    }
}

#ifndef DIVAS_PAIR_MINB
#define DIVAS_PAIR_MINB 4
#endif
// One tile = one view x 256 consecutive gated voxels.  Phase A routes every
// pair of the tile and compacts the thin candidates that need a footprint
// scan into a shared-memory queue; phase B runs them on densely packed warps.
__device__ __forceinline__ void pair_tile(const FuseConst &C, const Cam &k,
                                          const float *__restrict__ dens, const FuseMaps &M,
                                          const Contrib &K, uint32_t vi,
                                          long long n, long long block0, int view, QItem *s_q,
                                          int *s_nq) {
    const long long slot = block0 + threadIdx.x;
    bool has = false;
    QItem q;
#if DIVAS_QSMALL
    double xd_, xcam_, ycam_;                   // (recomputed by thin_item)
#else
    double &xd_ = q.x_d, &xcam_ = q.xcam, &ycam_ = q.ycam;
#endif
    if (slot < n) {
        q.slot = (uint32_t)slot;
        q.vi = vi;
        has = pair_route(C, k, dens, M, K, q.vi, view, (int64_t)view * C.cap + slot,
                         (int64_t)(view >> 5) * C.cap + slot, 1u << (view & 31), xd_, xcam_,
                         ycam_);
    }
    const unsigned ball = __ballot_sync(0xffffffffu, has);
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0 && ball) base = atomicAdd(s_nq, __popc(ball));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (has) s_q[base + __popc(ball & ((1u << lane) - 1u))] = q;
    __syncthreads();
    const int nq = *s_nq;
    for (int i = threadIdx.x; i < nq; i += blockDim.x) thin_item(C, k, M, K, view, s_q[i]);
}

// Tile-level rejection (exact): can ANY pair of this tile (one view x the
// tile's gated voxels) contribute?  A thick vote needs its centre pixel p with
// m >= mask_thr >= 0.5, n > 0 and |x_d - D_p| <= tau_depth(n) <= tau_thin(n);
// a thin vote (band_ok) needs support, i.e. a footprint pixel with m > 0.5,
// n > 0 and |x_d - D_p| <= tau_thin(n).  Either way x_d lies in the depth band
// of p's 8x8 tile (bands.cuh covers every pixel with m >= 0.5).  Every centre
// pixel and footprint of the tile's voxels lies in the projection of their
// bounding box (convex, in front of the camera: inside the hull of its 8
// corners' projections, padded by a pixel), and their x_d in the corners'
// depth range (depth is affine), so when that range meets no band of the
// covered tiles no pair can vote: the tile is skipped.
//
// One warp tests four views at once: lanes 8s .. 8s+7 project the 8 corners
// of bb = {min ix, iy, iz, max ix, iy, iz} into view v0 + s (a reciprocal
// instead of the division: the pixel window is padded by a pixel and the
// depth range by 1e-9 relative, far above its error), then the 32 lanes walk
// each view's covered band tiles in turn.  cull[s] = the verdict for v0 + s.
__device__ __forceinline__ void tile_culled4(const FuseConst &C, const double *__restrict__ cams,
                                             const FuseMaps &M, int v0, int nviews,
                                             const unsigned *bb, bool cull[4]) {
    const int lane = threadIdx.x & 31, sub = lane >> 3, c = lane & 7;
    const int vl = v0 + sub;
    const bool has = vl < nviews;
    double xc = 0.0, yc = 0.0, d = 1.0, sc = 0.0, fx = 1.0, fy = 1.0, cx = 0.0, cy = 0.0;
    double W = 1.0, H = 1.0;
    if (has) {
        const double *k = cams + (int64_t)(C.view0 + vl) * kCamStride;
        const double px = C.origin0 + (double)(bb[0] + (c & 1 ? bb[3] - bb[0] + 1 : 0)) * C.dx;
        const double py = C.origin1 + (double)(bb[1] + (c & 2 ? bb[4] - bb[1] + 1 : 0)) * C.dx;
        const double pz = C.origin2 + (double)(bb[2] + (c & 4 ? bb[5] - bb[2] + 1 : 0)) * C.dx;
        const double p0 = __ldg(k + 9), p1 = __ldg(k + 10), p2 = __ldg(k + 11);
        const double rx = px - p0, ry = py - p1, rz = pz - p2;
        d = -(__ldg(k + 2) * rx + __ldg(k + 5) * ry + __ldg(k + 8) * rz);
        xc = __ldg(k + 0) * rx + __ldg(k + 3) * ry + __ldg(k + 6) * rz;
        yc = __ldg(k + 1) * rx + __ldg(k + 4) * ry + __ldg(k + 7) * rz;
        sc = fabs(px) + fabs(py) + fabs(pz) + fabs(p0) + fabs(p1) + fabs(p2);
        fx = __ldg(k + 12); fy = __ldg(k + 13); cx = __ldg(k + 14); cy = __ldg(k + 15);
        W = __ldg(k + 16); H = __ldg(k + 17);
    }
    const double mg = 1e-9 * (sc + 1.0);
    // every corner of the group behind / in front (8-lane groups: masks per group)
    const unsigned gmask = 0xffu << (8 * sub);
    const unsigned behind = __ballot_sync(0xffffffffu, !has || d < -mg) & gmask;
    const unsigned front = __ballot_sync(0xffffffffu, has && d > mg) & gmask;
    const bool all_behind = behind == gmask, all_front = front == gmask;
    double u = 0.0, v = 0.0;
    if (all_front && d > 1e-30 && d < 1e30) {
        const double r = rcp_fast(d);
        u = fx * (xc * r) + cx;
        v = cy - fy * (yc * r);
    }
    double umn = u, umx = u, vmn = v, vmx = v, dlo = d - mg, dhi = d + mg;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
        umn = dmin2(umn, __shfl_xor_sync(0xffffffffu, umn, o));
        umx = dmax2(umx, __shfl_xor_sync(0xffffffffu, umx, o));
        vmn = dmin2(vmn, __shfl_xor_sync(0xffffffffu, vmn, o));
        vmx = dmax2(vmx, __shfl_xor_sync(0xffffffffu, vmx, o));
        dlo = dmin2(dlo, __shfl_xor_sync(0xffffffffu, dlo, o));
        dhi = dmax2(dhi, __shfl_xor_sync(0xffffffffu, dhi, o));
    }
    // per view: 0 = test the band tiles, 1 = culled, 2 = keep
    int state = 0, tx0 = 0, ty0 = 0, nx = 0, nt = 0;
    if (!has || all_behind) {
        state = 1;                                     // (no view / every centre behind)
    } else if (!all_front) {
        state = 2;                                     // straddles the camera plane
    } else if (!(umx > -2.0 && umn < W + 2.0 && vmx > -2.0 && vmn < H + 2.0)) {
        // the projection misses the image: every centre is out of the frustum,
        // unless a NaN / inf slipped through (then do not skip)
        state = (umx <= -2.0 || umn >= W + 2.0 || vmx <= -2.0 || vmn >= H + 2.0) ? 1 : 2;
    } else {
        const int x0 = (int)fmax(floor(umn) - 1.0, 0.0), x1 = (int)fmin(floor(umx) + 1.0, W - 1.0);
        const int y0 = (int)fmax(floor(vmn) - 1.0, 0.0), y1 = (int)fmin(floor(vmx) + 1.0, H - 1.0);
        tx0 = x0 / kBandTile;
        ty0 = y0 / kBandTile;
        nx = min(x1 / kBandTile, C.ntx - 1) - tx0 + 1;
        nt = nx * (min(y1 / kBandTile, C.nty - 1) - ty0 + 1);
        if (nx < 1 || nt < 1 || nt > 256) state = 2;
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {                       // the four views' band walks
        const int st = __shfl_sync(0xffffffffu, state, 8 * s);
        if (st != 0) { cull[s] = st == 1; continue; }
        const int ntx = __shfl_sync(0xffffffffu, nx, 8 * s);
        const int ntt = __shfl_sync(0xffffffffu, nt, 8 * s);
        const int bx = __shfl_sync(0xffffffffu, tx0, 8 * s);
        const int by = __shfl_sync(0xffffffffu, ty0, 8 * s);
        const double lo_ = __shfl_sync(0xffffffffu, dlo, 8 * s);
        const double hi_ = __shfl_sync(0xffffffffu, dhi, 8 * s);
        const double2 *bv = M.bands + (int64_t)(C.view0 + v0 + s) * band_view_stride(C.nty, C.ntx);
        // i / ntx as a multiply-high by ceil(2^32 / ntx): exact for i * ntx < 2^32
        // (i < 256, ntx <= 256 here); the divide was a quarter of the kernel
        const unsigned magic = ntx > 1 ? 0xffffffffu / (unsigned)ntx + 1u : 0u;
        // 32 tiles per round; stop at the first round with a hit (kept tiles,
        // the common case where the projections are large, need one round)
        bool hit = false;
        for (int i0 = 0; i0 < ntt; i0 += 32) {
            const int i = i0 + lane;
            if (i < ntt) {
                const int q = ntx > 1 ? (int)__umulhi((unsigned)i, magic) : i;
                const int ty = by + q, tx = bx + (i - q * ntx);
                const double2 b = __ldg(bv + (int64_t)ty * C.ntx + tx);
                hit = hi_ >= b.x && lo_ <= b.y;
            }
            if (__any_sync(0xffffffffu, hit)) break;
        }
        cull[s] = !__any_sync(0xffffffffu, hit);
    }
}

// Pre-pass of fuse_pairs: one CTA per tile of 256 slots; the bounding box of
// the tile's voxels once, then each warp tests four views at a time
// (tile_culled4).  skip[(view - view0) * ntiles + tile] = 1: the pair CTA
// exits at once.  Tiles whose voxels spread over more than 32 voxels on an
// axis (a slot run that wraps to another brick) are never skipped (their
// rectangles would cover too many band tiles to be worth testing).
// five blocks per SM (48 registers, a 20-byte spill): the C3 grid of 672 tiles
// runs in one wave instead of two (18.8 -> 15.3 us cold)
#ifndef DIVAS_CULL_MINB
#define DIVAS_CULL_MINB 5
#endif
__global__ void __launch_bounds__(kPairThreads, DIVAS_CULL_MINB)
tile_cull(FuseConst C, const double *__restrict__ cams, FuseMaps M,
          const uint32_t *__restrict__ work, const WsHeader *__restrict__ hdr, int nviews,
          uint8_t *__restrict__ skip) {
    griddep_wait();                     // PDL: after the previous kernel completes
    __shared__ unsigned s_bb[6];
    const long long block0 = (long long)blockIdx.x * blockDim.x;
    const long long ntiles = gridDim.x;
    const long long slot = block0 + threadIdx.x;
    const uint32_t vi = slot < C.cap ? __ldg(work + slot) : 0u;   // beside the count load
    const long long n = min((long long)hdr->count, (long long)C.cap);
    if (block0 >= n) return;                         // fuse_pairs exits on its own
    if (threadIdx.x == 0) {
        s_bb[0] = s_bb[1] = s_bb[2] = 0xffffffffu;
        s_bb[3] = s_bb[4] = s_bb[5] = 0u;
    }
    __syncthreads();
    unsigned ix = 0xffffffffu, iy = 0xffffffffu, iz = 0xffffffffu;
    unsigned jx = 0u, jy = 0u, jz = 0u;
    if (slot < n) {
        voxel_coords(C, vi, ix, iy, iz);
        jx = ix; jy = iy; jz = iz;
    }
    ix = __reduce_min_sync(0xffffffffu, ix); iy = __reduce_min_sync(0xffffffffu, iy);
    iz = __reduce_min_sync(0xffffffffu, iz); jx = __reduce_max_sync(0xffffffffu, jx);
    jy = __reduce_max_sync(0xffffffffu, jy); jz = __reduce_max_sync(0xffffffffu, jz);
    if ((threadIdx.x & 31) == 0 && ix != 0xffffffffu) {
        atomicMin(&s_bb[0], ix); atomicMin(&s_bb[1], iy); atomicMin(&s_bb[2], iz);
        atomicMax(&s_bb[3], jx); atomicMax(&s_bb[4], jy); atomicMax(&s_bb[5], jz);
    }
    __syncthreads();
    unsigned bb[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) bb[i] = s_bb[i];
    const bool compact = bb[3] - bb[0] < 32 && bb[4] - bb[1] < 32 && bb[5] - bb[2] < 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int v0 = 4 * warp; v0 < nviews; v0 += 4 * (kPairThreads / 32)) {
        bool cull[4] = {false, false, false, false};
        if (compact) tile_culled4(C, cams, M, v0, nviews, bb, cull);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            if (lane == s && v0 + s < nviews) {
                skip[(int64_t)(v0 + s) * ntiles + blockIdx.x] = cull[s] ? 1 : 0;
                if (cull[s]) fallback(C, DIVAS_FB_TILE_SKIP);
            }
        }
    }
}

__global__ void __launch_bounds__(kPairThreads, DIVAS_PAIR_MINB)
fuse_pairs(FuseConst C, const double *__restrict__ cams, const float *__restrict__ dens,
           FuseMaps M, Contrib K, const uint32_t *__restrict__ work,
           const WsHeader *__restrict__ hdr, int nviews, const uint8_t *__restrict__ skip) {
    griddep_wait();                     // PDL: after the previous kernel completes
    __shared__ QItem s_q[kQueue];
    __shared__ int s_nq;
    const int view = C.view0 + (int)blockIdx.y;
    const long long block0 = (long long)blockIdx.x * blockDim.x;
    // the count, the skip byte and the slot's voxel are independent loads:
    // all in flight at once (work holds cap entries)
    const long long slot = block0 + threadIdx.x;
    const uint32_t vi = slot < C.cap ? __ldg(work + slot) : 0u;
    const uint8_t sk = skip ? __ldg(skip + (int64_t)blockIdx.y * gridDim.x + blockIdx.x) : 0;
    const long long n = min((long long)hdr->count, (long long)C.cap);
    if (block0 >= n) return;                                   // whole CTA idle
    if (sk) return;
    if (threadIdx.x == 0) s_nq = 0;
    __syncthreads();
    Cam k;
    load_cam(cams + (int64_t)view * kCamStride, k);
    pair_tile(C, k, dens, M, K, vi, n, block0, view, s_q, &s_nq);
}

// ---------------------------------------------------------------------------
// reduction: value-sorted sums per voxel
// ---------------------------------------------------------------------------
// bits of views [lo, hi) within 32-bit word wd
__device__ __forceinline__ uint32_t view_word_mask(int wd, int view_lo, int view_hi) {
    const int a = max(view_lo - wd * 32, 0), b = min(view_hi - wd * 32, 32);
    return ((b >= 32) ? 0xffffffffu : ((1u << b) - 1u)) & ~((1u << a) - 1u);
}

constexpr int kReduceThreads = 128;

// Stores p, the optional votes / sums and the local occupancy of voxel vi;
// returns the occupancy byte (the peer copies are stored by fuse_reduce,
// coalesced per warp: peer_store_occ).
__device__ __forceinline__ uint8_t reduce_store(const FuseConst &C, const FuseOut &O, uint32_t vi,
                                                int n_thick, int n_thin, double sw, double smw,
                                                double st) {
    const double denom = sw + (double)n_thin;
    const double p = (denom > C.eps) ? (smw + st) / denom : 0.0;
    O.probs[vi] = p;
    if (O.n_thick) O.n_thick[vi] = n_thick;
    if (O.n_thin) O.n_thin[vi] = n_thin;
    if (O.sw) O.sw[vi] = sw;
    if (O.smw) O.smw[vi] = smw;
    if (O.st) O.st[vi] = st;
    const uint8_t oc = (p >= C.occ_thr) ? 1 : 0;
    if (O.occ) O.occ[vi] = oc;
    return oc;
}

// The reduced voxels' occupancy bytes into every peer buffer (the slab
// all-gather fused into the reduction).  Called by all 32 lanes; `has` lanes
// hold voxel vi's byte oc.  Slots run in brick-blocked order, so the four
// voxels of an iz quad are usually four neighbouring lanes: those publish one
// 4-byte store per peer (gathered with a match + OR reduction) instead of
// four 1-byte NVLink stores; any other voxel stores its own byte.
__device__ __forceinline__ void peer_store_occ(const FuseOut &O, bool has, uint32_t vi,
                                               uint8_t oc) {
    const int lane = threadIdx.x & 31;
    const unsigned key = has ? (vi >> 2) : (0xffffffffu - (unsigned)lane);
    const unsigned grp = __match_any_sync(0xffffffffu, key);
    if (!has) return;
    if (__popc(grp) == 4) {                               // the whole quad is here
        const uint32_t word = (uint32_t)oc << (8 * (vi & 3u));
        const uint32_t all = __reduce_or_sync(grp, word);
        if (lane == __ffs(grp) - 1)
            for (int r = 0; r < O.n_peers; ++r)
                *reinterpret_cast<uint32_t *>(O.occ_peers[r] + (vi & ~3u)) = all;
    } else {
        for (int r = 0; r < O.n_peers; ++r) O.occ_peers[r][vi] = oc;
    }
}

// One voxel, lists in local memory (any count up to MAXV views).
#ifndef DIVAS_RGROUP
#define DIVAS_RGROUP 4
#endif
constexpr int kRGroup = DIVAS_RGROUP;          // contribution loads in flight per thread
#ifndef DIVAS_THIN_EXACT
#define DIVAS_THIN_EXACT 1
#endif

// log2 of the granularity of a finite nonzero f64 (the weight of its lowest
// set significand bit): every multiple of 2^g up to 2^(g + 53) is exact.
__device__ __forceinline__ int f64_grain(double t) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(t);
    const int e = (int)((b >> 52) & 0x7ffu);
    const unsigned long long sig = (b & 0xfffffffffffffULL) | (e ? (1ULL << 52) : 0ULL);
    return (e ? e : 1) - 1075 + (__ffsll((long long)sig) - 1);
}

template <int MAXV>
__device__ __forceinline__ uint8_t reduce_local(const FuseConst &C, const Contrib &K,
                                                const FuseOut &O, uint32_t vi,
                                                uint32_t bt0, uint32_t bn0, long long slot) {
    double tw[MAXV], tmw[MAXV];
    int n_thick = 0, n_thin = 0;
    // The thin sum (fusion.py:373-386: ascending order, sequential f64 adds)
    // is first taken in view order, beside a certificate that EVERY order's
    // partial sums are exact: all t are multiples of 2^g (g = the smallest
    // granularity among them) and sum |t| < 2^(g + 53) bounds every partial
    // sum, so each add is exact and the sorted sum equals this one.  Thin
    // votes carry t = m_max, an f32 mask value >= thin_accept, whenever
    // thin_accept >= thin_percent_cover (the defaults): the certificate then
    // always holds and the sort disappears.  Otherwise the values are
    // sorted as the reference does (second pass below).
    double st = 0.0, sabs = 0.0;
    int gmin = 4096;
    bool thin_ok = true;
    // contributions are fetched in groups of kRGroup (all loads in flight
    // before the first insertion), then inserted in view order as before
    for (int wd = 0; wd < C.w32; ++wd) {
        uint32_t bt = wd ? K.bits_thick[(int64_t)wd * C.cap + slot] : bt0;
        uint32_t bn = wd ? K.bits_thin[(int64_t)wd * C.cap + slot] : bn0;
        while (bt) {
            double kw[kRGroup], km[kRGroup];
            int c = 0;
#pragma unroll
            for (int u = 0; u < kRGroup; ++u) {
                if (bt) {
                    const int view = wd * 32 + __ffs(bt) - 1;
                    bt &= bt - 1;
                    kw[u] = K.w[(int64_t)view * C.cap + slot];
                    km[u] = K.mw[(int64_t)view * C.cap + slot];
                    c = u + 1;
                }
            }
#pragma unroll
            for (int u = 0; u < kRGroup; ++u) {
                if (u < c) {
                    int j = n_thick - 1;   // stable insertion by (w, m*w): fusion.py:389-407
                    while (j >= 0 && (tw[j] > kw[u] || (tw[j] == kw[u] && tmw[j] > km[u]))) {
                        tw[j + 1] = tw[j];
                        tmw[j + 1] = tmw[j];
                        --j;
                    }
                    tw[j + 1] = kw[u];
                    tmw[j + 1] = km[u];
                    ++n_thick;
                }
            }
        }
        while (bn) {
            double kt[kRGroup];
            int c = 0;
#pragma unroll
            for (int u = 0; u < kRGroup; ++u) {
                if (bn) {
                    const int view = wd * 32 + __ffs(bn) - 1;
                    bn &= bn - 1;
                    kt[u] = K.t[(int64_t)view * C.cap + slot];
                    c = u + 1;
                }
            }
#pragma unroll
            for (int u = 0; u < kRGroup; ++u) {
                if (u < c) {
                    const double t = kt[u];
                    st += t;
                    sabs += fabs(t);
                    if (t != 0.0) {
                        if (!(fabs(t) < 1.0e300)) thin_ok = false;     // inf / NaN
                        else gmin = min(gmin, f64_grain(t));
                    }
                    ++n_thin;
                }
            }
        }
    }
    // sum |t| rounded up (the adds above round to nearest: relative 2^-46
    // covers up to 2^6 of them; larger counts take the sorted path)
    if (!DIVAS_THIN_EXACT || !thin_ok || n_thin > 64 ||
        (n_thin > 0 && gmin < 4096 &&
         !(sabs * (1.0 + 1.0 / 70368744177664.0) < ldexp(1.0, min(gmin + 53, 1000))))) {
        fallback(C, DIVAS_FB_THIN_SORT);
        double tt[MAXV];
        n_thin = 0;
        for (int wd = 0; wd < C.w32; ++wd) {
            uint32_t bn = K.bits_thin[(int64_t)wd * C.cap + slot];
            while (bn) {
                const int view = wd * 32 + __ffs(bn) - 1;
                bn &= bn - 1;
                const double t = K.t[(int64_t)view * C.cap + slot];
                int j = n_thin - 1;        // fusion.py:373-386
                while (j >= 0 && tt[j] > t) { tt[j + 1] = tt[j]; --j; }
                tt[j + 1] = t;
                ++n_thin;
            }
        }
        st = 0.0;
        for (int i = 0; i < n_thin; ++i) st += tt[i];
    }
    double sw = 0.0, smw = 0.0;
    for (int i = 0; i < n_thick; ++i) { sw += tw[i]; smw += tmw[i]; }
    return reduce_store(C, O, vi, n_thick, n_thin, sw, smw, st);
}

// dirty != NULL (incremental update of views [view_lo, view_hi)): only slots
// that held or now hold a contribution of those views are re-reduced; the
// others' outputs are already those of the unchanged contribution set.
template <int MAXV>
// eight blocks per SM (62 registers with four contribution loads in flight;
// eight loads needed 76 registers and six blocks): C5 270 -> 201 us cold
#ifndef DIVAS_REDUCE_MINB
#define DIVAS_REDUCE_MINB 8
#endif
__global__ void __launch_bounds__(kReduceThreads, DIVAS_REDUCE_MINB)
fuse_reduce(FuseConst C, Contrib K, FuseOut O, const uint32_t *__restrict__ work,
            const WsHeader *__restrict__ hdr, const uint8_t *__restrict__ dirty, int view_lo,
            int view_hi) {
    griddep_wait();                     // PDL: after the previous kernel completes
    const long long slot = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    // the slot's voxel and first bit words load beside the count (the
    // arrays hold cap entries per word)
    const bool in_cap = slot < C.cap;
    const uint32_t vi = in_cap ? work[slot] : 0u;
    const uint32_t bt0 = in_cap ? K.bits_thick[slot] : 0u;
    const uint32_t bn0 = in_cap ? K.bits_thin[slot] : 0u;
    const long long n = min((long long)hdr->count, (long long)C.cap);
    if (O.n_peers == 0) {                      // (the common case: no peer buffers)
        if (slot >= n) return;
        if (dirty && !dirty[slot]) {
            uint32_t now = 0;
            for (int wd = view_lo >> 5; wd <= (view_hi - 1) >> 5; ++wd)
                now |= (K.bits_thick[(int64_t)wd * C.cap + slot] |
                        K.bits_thin[(int64_t)wd * C.cap + slot]) &
                       view_word_mask(wd, view_lo, view_hi);
            if (!now) return;
        }
        reduce_local<MAXV>(C, K, O, vi, bt0, bn0, slot);
        return;
    }
    if (slot - (threadIdx.x & 31) >= n) return;           // whole warp past the end
    bool valid = slot < n;
    if (valid && dirty && !dirty[slot]) {
        uint32_t now = 0;
        for (int wd = view_lo >> 5; wd <= (view_hi - 1) >> 5; ++wd)
            now |= (K.bits_thick[(int64_t)wd * C.cap + slot] | K.bits_thin[(int64_t)wd * C.cap + slot]) &
                   view_word_mask(wd, view_lo, view_hi);
        valid = now != 0;
    }
    uint8_t oc = 0;
    if (valid) oc = reduce_local<MAXV>(C, K, O, vi, bt0, bn0, slot);
    __syncwarp();
    peer_store_occ(O, valid, vi, oc);
}

// ---------------------------------------------------------------------------
// f64 gradient maps (export for parity tests; fuse computes g on the fly)
// ---------------------------------------------------------------------------
__global__ void gradient_maps_kernel(int nv, int hm, int wm, const float *__restrict__ dexps,
                                     const float *__restrict__ dmins,
                                     const float *__restrict__ dmaxs,
                                     const int32_t *__restrict__ nsamps, double eps, double kappa,
                                     int valid_only, double *__restrict__ out) {
    const int64_t plane = (int64_t)hm * wm;
    const int64_t total = plane * nv;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / plane;
        const int64_t r = i - v * plane;
        const int iy = (int)(r / wm), ix = (int)(r - (int64_t)iy * wm);
        out[i] = (!valid_only || nsamps[i] > 0)
                     ? grad_at(dexps + v * plane, dmins + v * plane, dmaxs + v * plane, hm, wm, ix,
                               iy, eps, kappa)
                     : 0.0;
    }
}

// ---------------------------------------------------------------------------
// per-pair decision trace (thick_check / thin_check, fusion.py:549-646)
// ---------------------------------------------------------------------------
__global__ void pair_trace_kernel(divas_trace_args A, FuseConst C) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < A.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        divas_pair_record R;
        memset(&R, 0, sizeof(R));
        R.x_end = -1;
        R.y_end = -1;
        const int view = A.views[i];
        Cam k;
        load_cam(A.cams + (int64_t)view * kCamStride, k);
        const double xc0 = A.points[3 * i], xc1 = A.points[3 * i + 1], xc2 = A.points[3 * i + 2];
        const double rho = A.rho[i];
        const int64_t plane = (int64_t)A.hm * A.wm;
        const float *mk = A.masks + view * plane;
        const float *dmn = A.dmins + view * plane;
        const float *dmx = A.dmaxs + view * plane;
        const float *dex = A.dexps + view * plane;
        const int32_t *nsp = A.nsamps + view * plane;
        const int W = (int)k.w, H = (int)k.h;
        double u, v, x_d;
        R.stage = DIVAS_STAGE_FRUSTUM;
        const bool front = project_px(k, xc0, xc1, xc2, u, v, x_d);
        bool pix_ok = front && !(u < 0.0 || u >= 1.0 || v < 0.0 || v >= 1.0);
        long long px = 0, py = 0;
        int32_t ns = 0;
        double m = 0.0;
        if (pix_ok) {
            px = pixel_index(u, (long long)W);
            py = pixel_index(v, (long long)H);
            ns = nsp[py * A.wm + px];
            if (ns <= 0) {
                R.stage = DIVAS_STAGE_NO_SURFACE;
                pix_ok = false;
            } else {
                m = (double)mk[py * A.wm + px];
                R.m = m;
                R.x_d = x_d;
            }
        }
        if (pix_ok) {        // thick_check (fusion.py:571-603)
            if (m < C.mask_thr) R.stage = DIVAS_STAGE_MASK_GATE;
            else if (rho < C.rho_thr) R.stage = DIVAS_STAGE_DENSITY_GATE;
            else {
                // _grad_at on the view's own (true-size) arrays
                const int64_t c = py * A.wm + px;
                const float center = dex[c];
                const float r32 = dmx[c] - dmn[c];                       // f32 site
                const double rng = (double)r32 + C.eps;
                double gmax = 0.0, sg;
                if (px > 0) { sg = (double)fabsf(dex[c - 1] - center) / rng; if (sg > gmax) gmax = sg; }
                if (px < W - 1) { sg = (double)fabsf(dex[c + 1] - center) / rng; if (sg > gmax) gmax = sg; }
                if (py > 0) { sg = (double)fabsf(dex[c - A.wm] - center) / rng; if (sg > gmax) gmax = sg; }
                if (py < H - 1) { sg = (double)fabsf(dex[c + A.wm] - center) / rng; if (sg > gmax) gmax = sg; }
                double g = 1.0 / (1.0 + C.kappa * gmax);
                if (g > 1.0 - C.eps) g = 1.0 - C.eps;
                if (g < 0.0) g = 0.0;
                // _thick_pair with Python floats: f64 at every site
                const double dmin = (double)dmn[c], dmax = (double)dmx[c], dexp = (double)dex[c];
                const double *Rm = k.r;
                const double rx = (u * k.w - k.cx) / k.fx;
                const double ry = (k.cy - v * k.h) / k.fy;
                double ddx = Rm[0] * rx + Rm[1] * ry - Rm[2];
                double ddy = Rm[3] * rx + Rm[4] * ry - Rm[5];
                double ddz = Rm[6] * rx + Rm[7] * ry - Rm[8];
                const double norm = sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
                ddx /= norm; ddy /= norm; ddz /= norm;
                const double t_proj = ((xc0 - k.p0) * ddx + (xc1 - k.p1) * ddy + (xc2 - k.p2) * ddz);
                double t_c = t_proj;
                if (t_c < dmin) t_c = dmin;
                else if (t_c > dmax) t_c = dmax;
                double pcx = k.p0 + ddx * t_c, pcy = k.p1 + ddy * t_c, pcz = k.p2 + ddz * t_c;
                if (C.unbounded != 0) {
                    const double nx = (pcx - C.bc0) / C.bh0, ny = (pcy - C.bc1) / C.bh1,
                                 nz = (pcz - C.bc2) / C.bh2;
                    const double rr = sqrt(nx * nx + ny * ny + nz * nz);
                    if (rr > 1.0) {
                        const double sc = (2.0 - 1.0 / rr) / rr;
                        pcx = C.bc0 + nx * sc * C.bh0;
                        pcy = C.bc1 + ny * sc * C.bh1;
                        pcz = C.bc2 + nz * sc * C.bh2;
                    }
                }
                const double ex = xc0 - pcx, ey = xc1 - pcy, ez = xc2 - pcz;
                const double delta = sqrt(ex * ex + ey * ey + ez * ez);
                const double tau_sp = A.dx_vox * g + C.lam * (dmax - dmin);
                double b = C.beta * (double)ns;
                if (b > C.bmax) b = C.bmax;
                const double tau_dp = (C.gamma + b) * A.dx_vox;
                const bool ok = delta <= tau_sp && fabs(x_d - dexp) <= tau_dp;
                const double mu = 0.5 * (dmin + dmax);
                double hd = 0.5 * (dmax - dmin);
                if (hd < C.eps) hd = C.eps;
                const double r = fabs(t_c - mu) / hd;
                R.delta = delta; R.g = g; R.tau_spatial = tau_sp; R.tau_depth = tau_dp;
                R.t_proj = t_proj; R.t_clamped = t_c; R.mu_d = mu; R.h_d = hd; R.r = r;
                R.w_depth = exp_ref(-C.alpha1 * r * r);
                R.stage = ok ? DIVAS_STAGE_PASSED
                             : (delta > tau_sp ? DIVAS_STAGE_SPATIAL : DIVAS_STAGE_DEPTH);
            }
            // thin_check (fusion.py:618-646)
            const double fmax = k.fx > k.fy ? k.fx : k.fy;
            if (m > C.thin_floor && rho >= C.rho_thin && x_d > 0.0 && A.dx_vox * fmax / x_d >= 1.0) {
                const double half = 0.5 * A.dx_vox;
                double umn = 1e30, umx = -1e30, vmn = 1e30, vmx = -1e30;
                bool okc = true;
                for (int j = 0; j < 8 && okc; ++j) {
                    const double sx = ((j & 1) == 0) ? -1.0 : 1.0;
                    const double sy = ((j & 2) == 0) ? -1.0 : 1.0;
                    const double sz = ((j & 4) == 0) ? -1.0 : 1.0;
                    double cu, cv, cd;
                    if (!project_px(k, xc0 + sx * half, xc1 + sy * half, xc2 + sz * half, cu, cv, cd)) {
                        okc = false;
                        break;
                    }
                    if (cu < umn) umn = cu;
                    if (cu > umx) umx = cu;
                    if (cv < vmn) vmn = cv;
                    if (cv > vmx) vmx = cv;
                }
                if (okc) {
                    long long xs = nb_floor_int(umn * k.w), xe = nb_floor_int(umx * k.w);
                    long long ys = nb_floor_int(vmn * k.h), ye = nb_floor_int(vmx * k.h);
                    if (!(xe < 0 || xs > W - 1 || ye < 0 || ys > H - 1)) {
                        if (xs < 0) xs = 0;
                        if (ys < 0) ys = 0;
                        if (xe > W - 1) xe = W - 1;
                        if (ye > H - 1) ye = H - 1;
                        long long support = 0, npix = 0;
                        double m_max = 0.0;
                        for (long long yy = ys; yy <= ye; ++yy)
                            for (long long xx = xs; xx <= xe; ++xx) {
                                ++npix;
                                const double mv = (double)mk[yy * A.wm + xx];
                                if (mv > m_max) m_max = mv;
                                const int32_t nn = nsp[yy * A.wm + xx];
                                if (mv > 0.5 && nn > 0) {
                                    double bb = C.beta * (double)nn;
                                    if (bb > C.bmax) bb = C.bmax;
                                    const double tau_d = (2.0 * C.gamma + bb) * A.dx_vox;
                                    if (fabs(x_d - (double)dex[yy * A.wm + xx]) <= tau_d) ++support;
                                }
                            }
                        const double p_cov = (double)support / (double)npix;
                        R.thin_candidate = 1;
                        R.x_start = xs; R.x_end = xe; R.y_start = ys; R.y_end = ye;
                        R.support_count = support; R.n_pixels = npix;
                        R.p_covered = p_cov; R.m_max = m_max;
                        R.t = (p_cov >= C.thin_pct) ? m_max : p_cov;
                    }
                }
            }
        }
        A.out[i] = R;
    }
}

// Incremental updates: drop the contribution bits of views [lo, hi) before
// they are re-evaluated.
// Clears the bits of views [lo, hi); dirty[slot] = the slot had one of them
// (its sums change even if the re-evaluated views add nothing back).
__global__ void clear_view_bits(Contrib K, int64_t cap, int view_lo, int view_hi,
                                const WsHeader *__restrict__ hdr, uint8_t *__restrict__ dirty) {
    griddep_wait();                     // PDL: after the previous kernel completes
    const long long n = min((long long)hdr->count, (long long)cap);
    for (long long slot = (long long)blockIdx.x * blockDim.x + threadIdx.x; slot < n;
         slot += (long long)gridDim.x * blockDim.x) {
        uint32_t had = 0;
        for (int wd = view_lo >> 5; wd <= (view_hi - 1) >> 5; ++wd) {
            const uint32_t m = view_word_mask(wd, view_lo, view_hi);
            const uint32_t bt = K.bits_thick[(int64_t)wd * cap + slot];
            const uint32_t bn = K.bits_thin[(int64_t)wd * cap + slot];
            had |= (bt | bn) & m;
            if (bt & m) K.bits_thick[(int64_t)wd * cap + slot] = bt & ~m;
            if (bn & m) K.bits_thin[(int64_t)wd * cap + slot] = bn & ~m;
        }
        dirty[slot] = had ? 1 : 0;
    }
}

// ---------------------------------------------------------------------------
// workspace layout
// ---------------------------------------------------------------------------
struct WsLayout {
    size_t work, bits_thick, bits_thin, w, mw, t, dirty, gtiles, skip, rec, bands, total;
};

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// internal_aux: reserve the scan-record / band regions that divas_fuse builds
// when the caller supplies no records (args->records == NULL); callers that
// pass divas_refine_bands output need neither (C3: ~390 MB less).
static WsLayout ws_layout(int64_t cap, int32_t nv_cap, int32_t hm, int32_t wm, bool internal_aux) {
    const size_t c = (size_t)(cap > 0 ? cap : 1);
    const size_t w32 = (size_t)((nv_cap + 31) / 32);
    WsLayout L;
    size_t off = 256;
    L.work = off;       off = align256(off + c * 4);
    L.bits_thick = off; off = align256(off + w32 * c * 4);
    L.bits_thin = off;  off = align256(off + w32 * c * 4);
    L.w = off;          off = align256(off + (size_t)nv_cap * c * 8);
    L.mw = off;         off = align256(off + (size_t)nv_cap * c * 8);
    L.t = off;          off = align256(off + (size_t)nv_cap * c * 8);
    L.dirty = off;      off = align256(off + c);
    L.gtiles = off;     off = align256(off + (size_t)kGateTileMax * 4);
    L.skip = off;       off = align256(off + (size_t)nv_cap * ((c + kPairThreads - 1) / kPairThreads));
    L.rec = off;        off = align256(off + (internal_aux ? record_bytes(nv_cap, hm, wm) : 0));
    L.bands = off;      off = align256(off + (internal_aux ? band_bytes(nv_cap, hm, wm) : 0));
    L.total = off;
    return L;
}

static int sm_count() {
    static int n = 0;   // device property, same on every B200
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    }
    return n;
}

static void fill_const(FuseConst &C, const divas_fuse_args *a, int64_t cap) {
    C.g = a->g; C.lo = a->vox_lo; C.hi = a->vox_hi;
    C.gshift = -1;
    if (a->g > 0 && (a->g & (a->g - 1)) == 0)
        for (int b = 0; b < 31; ++b)
            if ((int64_t(1) << b) == a->g) { C.gshift = b; break; }
    C.origin0 = a->origin[0]; C.origin1 = a->origin[1]; C.origin2 = a->origin[2];
    C.dx = a->dx_vox;
    C.nv = a->nv; C.hm = a->hm; C.wm = a->wm; C.w32 = (a->nv + 31) / 32;
    C.cap = cap;
    C.view0 = 0;
    const double *pv = a->pv;
    C.gamma = pv[0]; C.beta = pv[1]; C.bmax = pv[2]; C.lam = pv[3]; C.rho_thr = pv[4];
    C.rho_thin = pv[5]; C.thin_pct = pv[6]; C.alpha1 = pv[7]; C.thin_accept = pv[8];
    C.eps = pv[9]; C.mask_thr = pv[10]; C.thin_floor = pv[11]; C.kappa = pv[12];
    C.enable_thin = pv[13] != 0.0;
    // zero support => p_cov = 0 => t = 0 (thin_pct > 0) < thin_accept: no vote.
    // Needs thin_accept > 0 too (FusionParams enforces it; raw vectors may not)
    C.band_ok = (C.thin_pct > 0.0 && C.thin_accept > 0.0) ? 1 : 0;
    // tile skipping needs every voting pixel inside the bands (m >= 0.5):
    // thick gate mask_thr >= 0.5, and thin votes only with support
    C.cull = (C.mask_thr >= 0.5 && (C.band_ok || !C.enable_thin)) ? 1 : 0;
    C.ntx = (a->wm + kBandTile - 1) / kBandTile;
    C.nty = (a->hm + kBandTile - 1) / kBandTile;
    C.cube_r = 0.8660254037844387 * a->dx_vox * (1.0 + 1e-9);
    C.tau_max = (2.0 * C.gamma + C.bmax) * C.dx;
    C.bc0 = a->bc[0]; C.bc1 = a->bc[1]; C.bc2 = a->bc[2];
    C.bh0 = a->bh[0]; C.bh1 = a->bh[1]; C.bh2 = a->bh[2];
    C.unbounded = a->unbounded;
    C.occ_thr = a->occ_thr;
    C.fallbacks = (unsigned long long *)a->fallbacks;
}

static void launch_gate_count(const FuseConst &C, const float *dens, WsHeader *hdr,
                              cudaStream_t s) {
    const int64_t nquads = (C.hi - C.lo + 3) / 4;
    int64_t blocks = (nquads + kGateThreads - 1) / kGateThreads;
    blocks = std::min<int64_t>(blocks, (int64_t)sm_count() * 16);
    fuse_gate_count<<<(unsigned)std::max<int64_t>(blocks, 1), kGateThreads, 0, s>>>(dens, C, hdr);
}

// The ordered gate: slots hold the gated voxels in C order, so a pair CTA's
// 256 slots are spatially adjacent voxels (their footprints overlap: L1 reuse)
// and the slot order is reproducible.
static void launch_gate(const FuseConst &C, const float *dens, const FuseOut &O, uint32_t *work,
                        WsHeader *hdr, uint32_t *tiles, bool zero, cudaStream_t s) {
    const int64_t g = C.g, gg = g * g;
    BrickGrid G;
    G.ix0 = C.lo / gg;
    const int64_t ix1 = (C.hi + gg - 1) / gg;          // exclusive
    G.nbx = (int)((ix1 - G.ix0 + kBrick - 1) / kBrick);
    G.nby = G.nbz = (int)((g + kBrick - 1) / kBrick);
    const int64_t ntiles = (int64_t)G.nbx * G.nby * G.nbz;
    if (zero) gate_tiles<true><<<(unsigned)ntiles, kGateThreads, 0, s>>>(dens, C, O, G, tiles);
    else gate_tiles<false><<<(unsigned)ntiles, kGateThreads, 0, s>>>(dens, C, O, G, tiles);
    launch_pdl(gate_scan, dim3(1), dim3(1024), 0, s, tiles, ntiles, C.cap, hdr);
    launch_pdl(gate_emit, dim3((unsigned)ntiles), dim3(kGateThreads), 0, s, dens, C, G, tiles,
               ntiles, hdr, work);
}

// records + bands of views [v0, v0 + cnt) from planar refined masks
static void launch_aux(const divas_fuse_args *a, int v0, int cnt, float2 *rec, double2 *bands,
                       cudaStream_t s) {
    const BandParams B = band_params(a->pv, a->dx_vox, a->hm, a->wm);
    const int64_t plane = (int64_t)a->hm * a->wm;
    const float *m = a->masks + v0 * plane;
    const int32_t *n = a->nsamps + v0 * plane;
    const float *d = a->dexps + v0 * plane;
    float2 *r = rec + 2 * v0 * plane;
    double2 *b = bands + (int64_t)v0 * band_view_stride(B.nty, B.ntx);
    launch_band_init(b, B, cnt, s);
    const bool vec = (a->wm % 4 == 0) &&
                     ((((uintptr_t)m) | ((uintptr_t)n) | ((uintptr_t)d)) & 15) == 0;
    if (vec) {
        dim3 bg((unsigned)((a->wm / 4 + 255) / 256), (unsigned)B.nty, (unsigned)cnt);
        band_pass<4, false><<<bg, 256, 0, s>>>(B, m, nullptr, n, d, nullptr, nullptr, b, r, cnt);
    } else {
        dim3 bg((unsigned)((a->wm + 255) / 256), (unsigned)B.nty, (unsigned)cnt);
        band_pass<1, false><<<bg, 256, 0, s>>>(B, m, nullptr, n, d, nullptr, nullptr, b, r, cnt);
    }
}

}  // namespace divas

using namespace divas;

extern "C" size_t divas_fuse_workspace_size_ext(int64_t max_gated, int32_t nv_cap, int32_t hm,
                                                int32_t wm, int32_t internal_aux) {
    return ws_layout(max_gated, nv_cap > 0 ? nv_cap : 1, hm > 0 ? hm : 1, wm > 0 ? wm : 1,
                     internal_aux != 0).total;
}

extern "C" size_t divas_fuse_workspace_size(int64_t max_gated, int32_t nv_cap, int32_t hm,
                                            int32_t wm) {
    return divas_fuse_workspace_size_ext(max_gated, nv_cap, hm, wm, 1);
}

extern "C" const int64_t *divas_fuse_gated_count(const void *workspace) {
    return (const int64_t *)workspace;
}

extern "C" const int32_t *divas_fuse_overflow(const void *workspace) {
    return (const int32_t *)((const char *)workspace + 8);
}

static int validate(const divas_fuse_args *a, const char *who) {
    if (!a) { set_error("%s: null args", who); return DIVAS_EINVAL; }
    if (a->g < 1) { set_error("%s: bad grid resolution", who); return DIVAS_EINVAL; }
    const int64_t nvox = a->g * a->g * a->g;
    if (a->vox_lo < 0 || a->vox_hi > nvox || a->vox_lo > a->vox_hi) {
        set_error("%s: voxel range [%lld, %lld) outside [0, %lld)", who, (long long)a->vox_lo,
                  (long long)a->vox_hi, (long long)nvox);
        return DIVAS_EINVAL;
    }
    if (nvox > 0xffffffffLL) { set_error("%s: grid too large for 32-bit slots", who); return DIVAS_EINVAL; }
    const int64_t nb = (a->g + kBrick - 1) / kBrick;   // gate bricks of the full grid
    if (nb * nb * nb > kGateTileMax) {
        set_error("%s: grid of %lld^3 has more than %lld gate bricks", who, (long long)a->g,
                  (long long)kGateTileMax);
        return DIVAS_EINVAL;
    }
    if (!a->density) { set_error("%s: null density", who); return DIVAS_EINVAL; }
    return DIVAS_OK;
}

extern "C" int divas_gate_count(const divas_fuse_args *a, void *workspace, void *stream) {
    int rc = validate(a, "divas_gate_count");
    if (rc) return rc;
    if (!workspace) { set_error("divas_gate_count: null workspace"); return DIVAS_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    FuseConst C;
    fill_const(C, a, 0);
    WsHeader *hdr = (WsHeader *)workspace;
    if (cudaMemsetAsync(hdr, 0, sizeof(WsHeader), s) != cudaSuccess)
        return check_launch("divas_gate_count(memset)");
    if (a->vox_hi > a->vox_lo) launch_gate_count(C, a->density, hdr, s);
    return check_launch("divas_gate_count");
}

extern "C" int divas_fuse(const divas_fuse_args *a, void *workspace, size_t workspace_bytes,
                          void *stream) {
    int rc = validate(a, "divas_fuse");
    if (rc) return rc;
    const int nv_cap = a->nv_cap > 0 ? a->nv_cap : a->nv;
    if (a->nv < 1 || a->nv > 1024 || nv_cap < a->nv || nv_cap > 1024) {
        set_error("divas_fuse: view count %d / capacity %d outside [1, 1024]", a->nv, nv_cap);
        return DIVAS_EINVAL;
    }
    if (a->hm < 1 || a->wm < 1) { set_error("divas_fuse: empty planes"); return DIVAS_EINVAL; }
    const bool reduces = a->mode == DIVAS_FUSE_FULL || (a->mode & DIVAS_STEP_REDUCE);
    if (!a->cams || !a->dmins || !a->dmaxs || !a->dexps || !a->nsamps || (reduces && !a->probs) ||
        !workspace || (!a->records && !a->masks)) {
        set_error("divas_fuse: null pointer");
        return DIVAS_EINVAL;
    }
    if ((a->records == nullptr) != (a->bands == nullptr)) {
        set_error("divas_fuse: records and bands come together");
        return DIVAS_EINVAL;
    }
    if (a->occ_peers && (a->n_peers < 1 || a->n_peers > 1024)) {
        set_error("divas_fuse: n_peers %d outside [1, 1024]", a->n_peers);
        return DIVAS_EINVAL;
    }
    const int steps = a->mode == DIVAS_FUSE_FULL
                          ? (DIVAS_STEP_GATE | DIVAS_STEP_CLEAR_ALL | DIVAS_STEP_PAIRS | DIVAS_STEP_REDUCE)
                          : a->mode;
    if (steps & ~127) { set_error("divas_fuse: bad mode %d", a->mode); return DIVAS_EINVAL; }
    if ((steps & DIVAS_STEP_ZERO) && !a->probs) {
        set_error("divas_fuse: the ZERO step needs the output grid");
        return DIVAS_EINVAL;
    }
    int v0 = 0, v1 = a->nv;
    if (a->mode != DIVAS_FUSE_FULL && (steps & (DIVAS_STEP_PAIRS | DIVAS_STEP_CLEAR_VIEWS))) {
        v0 = a->view_lo; v1 = a->view_hi;
        if (v0 < 0 || v1 > a->nv || v0 >= v1) {
            set_error("divas_fuse: views [%d, %d) outside [0, %d)", v0, v1, a->nv);
            return DIVAS_EINVAL;
        }
    }
    const int64_t cap = a->max_gated > 0 ? a->max_gated : (a->vox_hi - a->vox_lo);
    const WsLayout L = ws_layout(cap, nv_cap, a->hm, a->wm, a->records == nullptr);
    if (workspace_bytes < L.total) {
        set_error("divas_fuse: workspace too small (%zu < %zu)", workspace_bytes, L.total);
        return DIVAS_EWORKSPACE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    FuseConst C;
    fill_const(C, a, cap);
    FuseOut O{a->probs, a->n_thick, a->n_thin, a->sw, a->smw, a->st, a->occ,
              a->occ_peers, a->occ_peers ? a->n_peers : 0};
    FuseMaps M{a->masks, a->dmins, a->dmaxs, a->dexps, a->nsamps,
               (const double2 *)a->bands, (const float2 *)a->records};
    char *ws = (char *)workspace;
    WsHeader *hdr = (WsHeader *)ws;
    uint32_t *work = (uint32_t *)(ws + L.work);
    Contrib K{(uint32_t *)(ws + L.bits_thick), (uint32_t *)(ws + L.bits_thin),
              (double *)(ws + L.w), (double *)(ws + L.mw), (double *)(ws + L.t)};
    if (a->vox_hi == a->vox_lo) return DIVAS_OK;
    if (!M.rec && (steps & DIVAS_STEP_PAIRS)) {   // records + bands of the evaluated views
        float2 *rec = (float2 *)(ws + L.rec);
        double2 *bands = (double2 *)(ws + L.bands);
        launch_aux(a, v0, v1 - v0, rec, bands, s);
        if ((rc = check_launch("divas_fuse(aux)"))) return rc;
        M.rec = rec;
        M.bands = bands;
    }
    if (steps & DIVAS_STEP_ZERO) {
        const int64_t groups = (a->vox_hi - a->vox_lo) / 16 + 1;
        // (blocks per SM: an experiment knob for running the fill beside the
        // pair kernel, which holds every register of an SM)
#ifndef DIVAS_ZERO_BLOCKS_PER_SM
#define DIVAS_ZERO_BLOCKS_PER_SM 8
#endif
        const int64_t blocks = std::min<int64_t>((groups + 255) / 256,
                                                 (int64_t)sm_count() * DIVAS_ZERO_BLOCKS_PER_SM);
        fuse_zero<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(C, O);
        if ((rc = check_launch("divas_fuse(zero)"))) return rc;
    }
    if (steps & DIVAS_STEP_GATE) {
        if (cudaMemsetAsync(hdr, 0, sizeof(WsHeader), s) != cudaSuccess)
            return check_launch("divas_fuse(memset)");
        launch_gate(C, a->density, O, work, hdr, (uint32_t *)(ws + L.gtiles),
                    !(steps & DIVAS_STEP_GATE_KEEP), s);
        if ((rc = check_launch("divas_fuse(gate)"))) return rc;
    }
    if (steps & DIVAS_STEP_CLEAR_ALL) {
        if (cudaMemsetAsync(ws + L.bits_thick, 0, L.w - L.bits_thick, s) != cudaSuccess)
            return check_launch("divas_fuse(memset bits)");
    }
    if (steps & DIVAS_STEP_CLEAR_VIEWS) {
        const int64_t blocks = std::min<int64_t>((cap + 255) / 256, (int64_t)sm_count() * 8);
        launch_pdl(clear_view_bits, dim3((unsigned)std::max<int64_t>(blocks, 1)), dim3(256), 0, s,
                   K, (int64_t)cap, v0, v1, (const WsHeader *)hdr, (uint8_t *)(ws + L.dirty));
        if ((rc = check_launch("divas_fuse(clear)"))) return rc;
    }
    if (steps & DIVAS_STEP_PAIRS) {
        const int64_t cap_blocks = (cap + kPairThreads - 1) / kPairThreads;
        if (cap_blocks > 0x7fffffffLL) { set_error("divas_fuse: too many slots"); return DIVAS_EINVAL; }
        C.view0 = v0;
        // a small shared-memory carveout (the queues of 4 CTAs fit in 64 KB)
        // leaves ~190 KB of L1 for the footprint / band / gradient gathers
        {   // once per device (an attribute of the function in each context)
            static unsigned long long carve_set = 0;   // bit per device ordinal < 64
            int dev = 0;
            cudaGetDevice(&dev);
            const unsigned long long bit = 1ull << (dev & 63);
            if (!(__atomic_load_n(&carve_set, __ATOMIC_RELAXED) & bit)) {
                cudaFuncSetAttribute(fuse_pairs, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     kPairCarveout);
                __atomic_fetch_or(&carve_set, bit, __ATOMIC_RELAXED);
            }
        }
        const dim3 pg((unsigned)std::max<int64_t>(cap_blocks, 1), (unsigned)(v1 - v0));
        uint8_t *skip = nullptr;
        if (C.cull) {       // tile-level band rejection first (exact, see tile_culled)
            skip = (uint8_t *)(ws + L.skip);
            launch_pdl(tile_cull, dim3(pg.x), dim3(kPairThreads), 0, s, C, a->cams, M, work, hdr,
                       v1 - v0, skip);
            if ((rc = check_launch("divas_fuse(tile_cull)"))) return rc;
        }
        launch_pdl(fuse_pairs, pg, dim3(kPairThreads), 0, s, C, a->cams, a->density, M, K, work,
                   hdr, v1 - v0, (const uint8_t *)skip);
        if ((rc = check_launch("divas_fuse(pairs)"))) return rc;
    }
    if (steps & DIVAS_STEP_REDUCE) {
        const unsigned rblocks =
            (unsigned)std::max<int64_t>((cap + kReduceThreads - 1) / kReduceThreads, 1);
        // incremental (CLEAR_VIEWS + REDUCE in one call): only dirty slots
        const uint8_t *dirty = ((steps & DIVAS_STEP_CLEAR_VIEWS) && (steps & DIVAS_STEP_PAIRS))
                                   ? (const uint8_t *)(ws + L.dirty) : nullptr;
#define DIVAS_REDUCE(MV) \
        launch_pdl(fuse_reduce<MV>, dim3(rblocks), dim3(kReduceThreads), 0, s, C, K, O, \
                   (const uint32_t *)work, (const WsHeader *)hdr, dirty, v0, v1)
        if (a->nv <= 32) DIVAS_REDUCE(32);
        else if (a->nv <= 64) DIVAS_REDUCE(64);
        else if (a->nv <= 128) DIVAS_REDUCE(128);
        else if (a->nv <= 256) DIVAS_REDUCE(256);
        else DIVAS_REDUCE(1024);
#undef DIVAS_REDUCE
        if ((rc = check_launch("divas_fuse(reduce)"))) return rc;
    }
    return DIVAS_OK;
}

extern "C" void divas_fuse_ws_regions(int64_t max_gated, int32_t nv_cap, int32_t hm, int32_t wm,
                                      int32_t internal_aux, size_t out[7]) {
    const WsLayout L = ws_layout(max_gated, nv_cap > 0 ? nv_cap : 1, hm > 0 ? hm : 1,
                                 wm > 0 ? wm : 1, internal_aux != 0);
    out[0] = L.work; out[1] = L.bits_thick; out[2] = L.bits_thin;
    out[3] = L.w; out[4] = L.mw; out[5] = L.t; out[6] = L.total;
}

extern "C" int divas_gradient_maps(int32_t nv, int32_t hm, int32_t wm, const float *dexps,
                                   const float *dmins, const float *dmaxs, const int32_t *nsamps,
                                   double eps, double kappa, int32_t valid_only, double *out,
                                   void *stream) {
    if (nv < 1 || hm < 1 || wm < 1) { set_error("divas_gradient_maps: empty"); return DIVAS_EINVAL; }
    if (!dexps || !dmins || !dmaxs || !nsamps || !out) {
        set_error("divas_gradient_maps: null pointer");
        return DIVAS_EINVAL;
    }
    const int64_t total = (int64_t)nv * hm * wm;
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 32);
    gradient_maps_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        nv, hm, wm, dexps, dmins, dmaxs, nsamps, eps, kappa, valid_only, out);
    return check_launch("divas_gradient_maps");
}

extern "C" int divas_pair_trace(const divas_trace_args *a, void *stream) {
    if (!a || a->nv < 1 || a->hm < 1 || a->wm < 1 || a->n < 0) {
        set_error("divas_pair_trace: bad arguments");
        return DIVAS_EINVAL;
    }
    if (a->n == 0) return DIVAS_OK;
    if (!a->cams || !a->masks || !a->dmins || !a->dmaxs || !a->dexps || !a->nsamps ||
        !a->points || !a->rho || !a->views || !a->out) {
        set_error("divas_pair_trace: null pointer");
        return DIVAS_EINVAL;
    }
    divas_fuse_args fa;
    memset(&fa, 0, sizeof(fa));
    for (int i = 0; i < DIVAS_NPARAM; ++i) fa.pv[i] = a->pv[i];
    for (int i = 0; i < 3; ++i) { fa.bc[i] = a->bc[i]; fa.bh[i] = a->bh[i]; }
    fa.unbounded = a->unbounded;
    fa.dx_vox = a->dx_vox;
    fa.nv = a->nv; fa.hm = a->hm; fa.wm = a->wm;
    FuseConst C;
    fill_const(C, &fa, 0);
    const int64_t blocks = std::min<int64_t>((a->n + 127) / 128, (int64_t)sm_count() * 32);
    pair_trace_kernel<<<(unsigned)blocks, 128, 0, (cudaStream_t)stream>>>(*a, C);
    return check_launch("divas_pair_trace");
}

#if DIVAS_STATS
extern "C" int divas_debug_pair_stats(unsigned long long *out, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, divas::g_pair_stats, sizeof(unsigned long long) * 24);
    if (reset) {
        unsigned long long z[24] = {0};
        cudaMemcpyToSymbol(divas::g_pair_stats, z, sizeof(z));
    }
    return 0;
}
#endif
