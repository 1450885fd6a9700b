// kernels_fill.cu — materialised point fills (configs C1-C4) for sm_100a.
//
// HBM-write-bound design: the only algorithmic traffic is the
// 4 B written per (index, dimension) sample, so each kernel is built around
// full-line 128-bit streaming stores and a per-sample instruction budget of
// ~22 issue slots (6.5 TB/s / 4 B / 148 SMs / 1.9 GHz = 5.8 samples per SM
// clock at 128 lanes/clk). Fast paths:
//   * lane -> (point, 4 consecutive dims); one warp store covers 512
//     contiguous bytes (dims | 128, dims >= 4);
//   * each warp owns a contiguous run of 32-step tiles; inside a tile the
//     index advances by a compile-time stride, so the Sobol' update is one
//     XOR with a register mask selected by a compile-time ctz, and the
//     lattice update is one IMAD with a compile-time brev constant;
//   * the float map is 9 full-rate ops (device.cuh map_u32).
#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <type_traits>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "device.cuh"
#include "internal.hpp"


namespace qmcgpu {

namespace {

constexpr int kBlock = 256;

__host__ __device__ constexpr uint32_t ctz_const(uint32_t v)
{
    uint32_t c = 0;
    while (!(v & 1u)) {
        v >>= 1;
        ++c;
    }
    return c;
}


// element e of a row-major [points][dims] chunk -> point (dims == 1 needs no
// division; div32 requires a divisor >= 2)
__device__ __forceinline__ uint32_t point_of(uint32_t e, uint32_t dims, const Div32& d)
{
    return dims == 1 ? e : div32(e, d);
}

// Block-wide copy of rows [r0, r0 + rows) of a padded shared tile (row
// stride ld >= dims words) to the consecutive global words o[0, rows*dims).
// Each thread walks its (row, col) position by a fixed stride (no division
// per word) and writes one 16-B streaming store per step. With dims % 4 == 0
// and o 16-B aligned, quads never straddle a row; otherwise scalar stores run
// up to the first 16-B boundary of o, the quads check the row wrap per word,
// and the tail is scalar.
__device__ __noinline__ void tile_store_rows_any(const uint32_t* src, uint32_t ld, uint32_t dims,
                                                 Div32 div_dims, uint32_t words, uint32_t* o)
{
    const uint32_t mis = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(o) & 15u);
    const uint32_t head = min(words, (mis & 3u) ? words : ((16u - mis) & 15u) >> 2);
    const uint32_t quads = (words - head) >> 2;
    const uint32_t adv = blockDim.x * 4 - 4; // end of one quad -> start of the thread's next
    const uint32_t padv = adv / dims, cadv = adv - padv * dims;
    const uint32_t e = head + threadIdx.x * 4;
    uint32_t p = point_of(e, dims, div_dims), c = e - p * dims;
    for (uint32_t qd = threadIdx.x; qd < quads; qd += blockDim.x) {
        uint32_t v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[k] = src[p * ld + c];
            if (++c == dims) {
                c = 0;
                ++p;
            }
        }
        __stcs(reinterpret_cast<uint4*>(o + head + qd * 4), make_uint4(v[0], v[1], v[2], v[3]));
        p += padv;
        c += cadv;
        if (c >= dims) {
            c -= dims;
            ++p;
        }
    }
    const uint32_t tail0 = head + quads * 4; // head and tail: < 4 + 4 words
    for (uint32_t w = threadIdx.x; w < head + (words - tail0); w += blockDim.x) {
        const uint32_t ew = w < head ? w : tail0 + (w - head);
        const uint32_t pw = point_of(ew, dims, div_dims);
        o[ew] = src[pw * ld + (ew - pw * dims)];
    }
}

__device__ __forceinline__ void tile_store_rows(const uint32_t* tile, uint32_t ld, uint32_t dims,
                                                const Div32& div_dims, uint32_t r0, uint32_t rows,
                                                uint32_t* o)
{
    const uint32_t words = rows * dims;
    const uint32_t* src = tile + r0 * ld;
    if ((dims & 3u) != 0 || (reinterpret_cast<uintptr_t>(o) & 15u) != 0) {
        tile_store_rows_any(src, ld, dims, div_dims, words, o);
        return;
    }
    const uint32_t stride = blockDim.x * 4;
    const uint32_t pstep = stride / dims, cstep = stride - pstep * dims;
    uint32_t e = threadIdx.x * 4;
    uint32_t p = point_of(e, dims, div_dims), c = e - p * dims;
    for (; e < words; e += stride) {
        const uint32_t* s4 = src + p * ld + c;
        __stcs(reinterpret_cast<uint4*>(o + e), make_uint4(s4[0], s4[1], s4[2], s4[3]));
        p += pstep;
        c += cstep;
        if (c >= dims) {
            c -= dims;
            ++p;
        }
    }
}

// Warp tiles [t, tend) owned by the calling warp: contiguous runs, so the
// tile-to-tile update is incremental.
__device__ __forceinline__ bool warp_tiles(uint64_t tile0, uint64_t ntiles, uint64_t per_warp,
                                           uint64_t& t, uint64_t& tend)
{
    const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    t = tile0 + warp * per_warp;
    tend = t + per_warp;
    if (tend > tile0 + ntiles)
        tend = tile0 + ntiles;
    return t < tend;
}

// ------------------------------------------------------------ map / check

__global__ void k_map(const uint32_t* __restrict__ in, float* __restrict__ out, uint64_t n)
{
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
         k += stride)
        out[k] = map_u32(in[k]);
}

__global__ void k_map_selfcheck(unsigned long long* count)
{
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    unsigned long long bad = 0;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
         k < (1ull << 32); k += stride) {
        const uint32_t u = static_cast<uint32_t>(k);
        bad += map_bits(u) != map_bits_reference(u);
    }
    for (int o = 16; o; o >>= 1)
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
    if ((threadIdx.x & 31) == 0 && bad)
        atomicAdd(count, bad);
}

// ------------------------------------------------------------------ Sobol'

// DPL consecutive dimensions per lane (8 -> one 256-bit store per lane,
// 1 KiB contiguous per warp store; 4 -> 128-bit stores, 512 B per warp).
template <int DPL>
__device__ __forceinline__ void load_cols(const uint32_t* p, uint32_t (&v)[DPL])
{
    if constexpr (DPL < 4) { // the slab kernels' narrow lanes
#pragma unroll
        for (int e = 0; e < DPL; ++e)
            v[e] = __ldg(p + e);
        return;
    }
#pragma unroll
    for (int q = 0; q < DPL / 4; ++q) {
        const uint4 t = __ldg(reinterpret_cast<const uint4*>(p) + q);
        v[4 * q] = t.x;
        v[4 * q + 1] = t.y;
        v[4 * q + 2] = t.z;
        v[4 * q + 3] = t.w;
    }
}

// Array `a` / `b` of the by-value SmallArgs (param space) or its device copy.
__device__ __forceinline__ const uint32_t* small_a(const SmallArgs& g)
{
    return g.dev_a ? g.dev_a : (g.has_a ? g.a : nullptr);
}
__device__ __forceinline__ const uint32_t* small_b(const SmallArgs& g)
{
    return g.dev_b ? g.dev_b : (g.has_b ? g.b : nullptr);
}

template <int DPL>
__device__ __forceinline__ void load_small(const uint32_t* p, uint32_t (&v)[DPL])
{
#pragma unroll
    for (int e = 0; e < DPL; ++e)
        v[e] = p[e];
}

template <int DPL>
__device__ __forceinline__ void store_vec(uint32_t* p, const uint32_t (&v)[DPL])
{
    if constexpr (DPL == 8) {
        asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]),
                     "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                     : "memory");
    } else if constexpr (DPL == 2) {
        __stcs(reinterpret_cast<uint2*>(p), make_uint2(v[0], v[1]));
    } else if constexpr (DPL == 1) {
        __stcs(p, v[0]);
    } else {
        __stcs(reinterpret_cast<uint4*>(p), make_uint4(v[0], v[1], v[2], v[3]));
    }
}

// MODE 0: plain / XOR-scrambled (words = XOR words, folded into the start
// value since the scramble is linear). MODE 2: hash-Owen, columns and the
// running value live in the bit-reversed domain; words = per-dim seeds.
template <int DPL, int LOG_PPS, int MODE, bool U32OUT>
__global__ void __launch_bounds__(kBlock)
    k_sobol_fast(const uint32_t* __restrict__ colsT, const __grid_constant__ SmallArgs args,
                 uint64_t first, uint64_t n, uint64_t tile0, uint64_t ntiles, uint64_t per_warp,
                 uint32_t* __restrict__ out)
{
    constexpr int PPS = 1 << LOG_PPS;  // points per warp store
    constexpr int LPP = 32 >> LOG_PPS; // lanes per point
    constexpr int DIMS = DPL * LPP;
    constexpr int LOG_TP = LOG_PPS + 5; // 32 steps per tile
    uint64_t t, tend;
    if (!warp_tiles(tile0, ntiles, per_warp, t, tend))
        return;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t r = lane / LPP;  // point within a step
    const uint32_t dq = lane % LPP; // dims DPL*dq .. DPL*dq + DPL-1
    const uint32_t* cols = colsT + dq * DPL; // column k of my dims at cols + k * DIMS

    // Step masks: index += PPS flips bits LOG_PPS .. LOG_PPS + ctz(u+1).
    uint32_t D[5][DPL];
    {
        uint32_t c[DPL];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            load_cols<DPL>(cols + (LOG_PPS + k) * DIMS, c);
#pragma unroll
            for (int e = 0; e < DPL; ++e)
                D[k][e] = k ? D[k - 1][e] ^ c[e] : c[e];
        }
    }
    uint32_t seed[DPL], xr[DPL], xp[DPL], c[DPL];
#pragma unroll
    for (int e = 0; e < DPL; ++e)
        seed[e] = xr[e] = xp[e] = 0;
    if (const uint32_t* words = small_a(args)) {
        if (MODE == 2)
            load_small<DPL>(words + dq * DPL, seed);
        else
            load_small<DPL>(words + dq * DPL, xr);
    }
    uint32_t omul[DPL], oadd[DPL]; // Owen seed terms, folded (owen_lk_folded)
#pragma unroll
    for (int e = 0; e < DPL; ++e) {
        omul[e] = (seed[e] >> 16) | 1u;
        oadd[e] = seed[e] * omul[e];
    }
#pragma unroll
    for (int k = 0; k < LOG_PPS; ++k)
        if ((r >> k) & 1u) {
            load_cols<DPL>(cols + k * DIMS, c);
#pragma unroll
            for (int e = 0; e < DPL; ++e)
                xr[e] ^= c[e];
        }
    // Value of the tile base t << LOG_TP (bits >= LOG_TP).
    for (uint64_t b = t; b; b &= b - 1) {
        load_cols<DPL>(cols + (LOG_TP + __ffsll(static_cast<long long>(b)) - 1) * DIMS, c);
#pragma unroll
        for (int e = 0; e < DPL; ++e)
            xp[e] ^= c[e];
    }

    for (;;) {
        const uint64_t p0 = (t << LOG_TP) + r; // this thread's point at step 0
        uint32_t x[DPL], y[DPL];
#pragma unroll
        for (int e = 0; e < DPL; ++e)
            x[e] = xp[e] ^ xr[e];
        const uint64_t lo = t << LOG_TP, hi = (t + 1) << LOG_TP;
        const bool full = lo >= first && hi <= first + n;
        uint32_t* o = out + (p0 - first) * DIMS + dq * DPL;
        // 32 steps as 4 x 8: the inner 8 are unrolled with compile-time
        // masks (ctz(w+1), w < 7); the step between groups flips bits up to
        // 3 + ctz(v+1) (v = 0,1,2 -> D[3], D[4], D[3]). Keeps the loop body
        // ~12 KB of SASS (inside the 32 KB L1.5 I-cache).
        auto group = [&](uint32_t v, auto check) {
#pragma unroll
            for (uint32_t w = 0; w < 8; ++w) {
                const uint32_t u = 8 * v + w;
#pragma unroll
                for (int e = 0; e < DPL; ++e) {
                    uint32_t val = x[e];
                    if (MODE == 2)
                        val = brev32(owen_lk_folded(val, omul[e], oadd[e]));
                    y[e] = U32OUT ? val : map_bits(val);
                }
                if (!decltype(check)::value || (p0 + u * PPS) - first < n)
                    store_vec<DPL>(o + u * 32 * DPL, y);
                if (w < 7) {
#pragma unroll
                    for (int e = 0; e < DPL; ++e)
                        x[e] ^= D[ctz_const(w + 1)][e];
                }
            }
#pragma unroll
            for (int e = 0; e < DPL; ++e)
                x[e] ^= (v == 1) ? D[4][e] : D[3][e];
        };
        if (full) { // interior tile: no per-store predicate
#pragma unroll 1
            for (uint32_t v = 0; v < 4; ++v)
                group(v, std::false_type{});
        } else {
#pragma unroll 1
            for (uint32_t v = 0; v < 4; ++v)
                group(v, std::true_type{});
        }
        if (++t >= tend)
            break;
        // tile t-1 -> t flips bits LOG_TP .. LOG_TP + ctz(t)
        const int cz = __ffsll(static_cast<long long>(t)) - 1;
        for (int k = 0; k <= cz; ++k) {
            load_cols<DPL>(cols + (LOG_TP + k) * DIMS, c);
#pragma unroll
            for (int e = 0; e < DPL; ++e)
                xp[e] ^= c[e];
        }
    }
}

// Work split of the slab kernels: warps come in groups of nslab, one per
// slab, and a group walks one contiguous range of 32-point tiles. The
// slabs of a row are thus written by sibling warps at about the same time,
// so a 128-B line that a slab boundary splits (row pitches that are no
// multiple of 128 B) is completed in L2 before it is evicted.
__device__ __forceinline__ bool slab_tiles(uint32_t nslab, uint64_t tile0, uint64_t ntp,
                                           uint64_t per_group, uint32_t& slab, uint64_t& t,
                                           uint64_t& tend)
{
    const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t group = warp / nslab;
    slab = static_cast<uint32_t>(warp - group * nslab);
    t = tile0 + group * per_group;
    tend = t + per_group < tile0 + ntp ? t + per_group : tile0 + ntp;
    return t < tend;
}

// Wide rows (dims a multiple of DPL whose rows the fast kernels cannot
// tile: dims > 256, or dims up to 256 not dividing 256 / 128): the row is
// cut into slabs of 32 * DPL dims, and a warp walks one slab, one point per
// step, each lane DPL consecutive dims, with k_sobol_fast's step-mask
// recurrence (32 steps per tile, the step from point i to i + 1 flips the
// columns 0 .. ctz(i + 1)). Every warp store is one 32 * DPL-word row
// segment (256-bit or 128-bit per lane), so the stream is as dense as the
// fast kernels' whatever the row length (work split: slab_tiles).
template <int DPL, int MODE, bool U32OUT>
__global__ void __launch_bounds__(kBlock)
    k_sobol_slab(const uint32_t* __restrict__ colsT, const __grid_constant__ SmallArgs args,
                 uint32_t dims, uint64_t first, uint64_t n, uint64_t tile0, uint64_t ntp,
                 uint32_t nslab, uint64_t per_group, uint32_t* __restrict__ out)
{
    constexpr uint32_t kSlab = 32 * DPL;
    const uint32_t lane = threadIdx.x & 31u;
    uint64_t t, tend;
    uint32_t slab;
    if (!slab_tiles(nslab, tile0, ntp, per_group, slab, t, tend))
        return;
    {
        const uint32_t j0 = slab * kSlab + lane * DPL; // this lane's first dimension
        const bool mine = j0 < dims;                    // dims % DPL == 0: all DPL or none
        const uint32_t* cols = colsT + (mine ? j0 : 0u);
        uint32_t D[5][DPL], c[DPL], seed[DPL], xr[DPL], xp[DPL];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            load_cols<DPL>(cols + k * dims, c);
#pragma unroll
            for (int e = 0; e < DPL; ++e)
                D[k][e] = k ? D[k - 1][e] ^ c[e] : c[e];
        }
#pragma unroll
        for (int e = 0; e < DPL; ++e)
            seed[e] = xr[e] = xp[e] = 0;
        if (const uint32_t* words = small_a(args)) {
            if (MODE == 2)
                load_small<DPL>(words + (mine ? j0 : 0u), seed);
            else
                load_small<DPL>(words + (mine ? j0 : 0u), xr);
        }
        uint32_t omul[DPL], oadd[DPL];
#pragma unroll
        for (int e = 0; e < DPL; ++e) {
            omul[e] = (seed[e] >> 16) | 1u;
            oadd[e] = seed[e] * omul[e];
        }
        for (uint64_t b = t; b; b &= b - 1) { // value of the tile base t << 5
            load_cols<DPL>(cols + (5 + __ffsll(static_cast<long long>(b)) - 1) * dims, c);
#pragma unroll
            for (int e = 0; e < DPL; ++e)
                xp[e] ^= c[e];
        }
        for (;;) {
            const uint64_t p0 = t << 5;
            uint32_t x[DPL], y[DPL];
#pragma unroll
            for (int e = 0; e < DPL; ++e)
                x[e] = xp[e] ^ xr[e];
            const bool full = p0 >= first && p0 + 32 <= first + n;
            uint32_t* o = out + (p0 - first) * dims + j0;
            auto group = [&](uint32_t v, auto check) {
#pragma unroll
                for (uint32_t w = 0; w < 8; ++w) {
                    const uint32_t k = 8 * v + w;
#pragma unroll
                    for (int e = 0; e < DPL; ++e) {
                        uint32_t val = x[e];
                        if (MODE == 2)
                            val = brev32(owen_lk_folded(val, omul[e], oadd[e]));
                        y[e] = U32OUT ? val : map_bits(val);
                    }
                    if (mine && (!decltype(check)::value || (p0 + k) - first < n))
                        store_vec<DPL>(o + static_cast<uint64_t>(k) * dims, y);
                    if (w < 7) {
#pragma unroll
                        for (int e = 0; e < DPL; ++e)
                            x[e] ^= D[ctz_const(w + 1)][e];
                    }
                }
#pragma unroll
                for (int e = 0; e < DPL; ++e)
                    x[e] ^= (v == 1) ? D[4][e] : D[3][e];
            };
            if (full) {
#pragma unroll 1
                for (uint32_t v = 0; v < 4; ++v)
                    group(v, std::false_type{});
            } else {
#pragma unroll 1
                for (uint32_t v = 0; v < 4; ++v)
                    group(v, std::true_type{});
            }
            if (++t >= tend)
                break;
            const int cz = __ffsll(static_cast<long long>(t)) - 1; // tile t-1 -> t
            for (int k = 0; k <= cz; ++k) {
                load_cols<DPL>(cols + (5 + k) * dims, c);
#pragma unroll
                for (int e = 0; e < DPL; ++e)
                    xp[e] ^= c[e];
            }
        }
    }
}

// Wide lattice rows, the slab layout of k_sobol_slab with k_lattice_fast's
// arithmetic at one point per step: brev(p0 + u) = brev(p0) + brev5(u) << 27
// for the 32 points u of a tile (disjoint bits), so each value is x0 plus a
// compile-time multiple of g << 27.
template <int DPL, bool U32OUT>
__global__ void __launch_bounds__(kBlock)
    k_lattice_slab(const __grid_constant__ SmallArgs args, uint32_t dims, uint64_t first,
                   uint64_t n, uint64_t tile0, uint64_t ntp, uint32_t nslab, uint64_t per_group,
                   uint32_t* __restrict__ out)
{
    constexpr uint32_t kSlab = 32 * DPL;
    const uint32_t lane = threadIdx.x & 31u;
    uint64_t t, tend;
    uint32_t slab;
    if (!slab_tiles(nslab, tile0, ntp, per_group, slab, t, tend))
        return;
    {
        const uint32_t j0 = slab * kSlab + lane * DPL;
        const bool mine = j0 < dims; // dims % DPL == 0: all DPL or none
        uint32_t gv[DPL], sv[DPL], G[DPL];
        load_small<DPL>(small_a(args) + (mine ? j0 : 0u), gv);
#pragma unroll
        for (int e = 0; e < DPL; ++e) {
            sv[e] = 0;
            G[e] = gv[e] << 27;
        }
        if (const uint32_t* shifts = small_b(args))
            load_small<DPL>(shifts + (mine ? j0 : 0u), sv);
        for (; t < tend; ++t) {
            const uint64_t p0 = t << 5;
            const uint32_t b = brev32(static_cast<uint32_t>(p0));
            uint32_t x0[DPL], y[DPL];
#pragma unroll
            for (int e = 0; e < DPL; ++e)
                x0[e] = b * gv[e] + sv[e];
            const bool full = p0 >= first && p0 + 32 <= first + n;
            uint32_t* o = out + (p0 - first) * dims + j0;
            auto group = [&](uint32_t v, auto check) {
                const uint32_t cv = ((v & 1u) << 1) | (v >> 1);
                uint32_t xv[DPL];
#pragma unroll
                for (int e = 0; e < DPL; ++e)
                    xv[e] = x0[e] + cv * G[e];
#pragma unroll
                for (uint32_t w = 0; w < 8; ++w) {
                    const uint32_t k = 8 * v + w;
                    const uint32_t cw = (((w & 1u) << 2) | (w & 2u) | (w >> 2)) << 2;
#pragma unroll
                    for (int e = 0; e < DPL; ++e) {
                        const uint32_t xx = xv[e] + cw * G[e];
                        y[e] = U32OUT ? xx : map_bits(xx);
                    }
                    if (mine && (!decltype(check)::value || (p0 + k) - first < n))
                        store_vec<DPL>(o + static_cast<uint64_t>(k) * dims, y);
                }
            };
            if (full) {
#pragma unroll 1
                for (uint32_t v = 0; v < 4; ++v)
                    group(v, std::false_type{});
            } else {
#pragma unroll 1
                for (uint32_t v = 0; v < 4; ++v)
                    group(v, std::true_type{});
            }
        }
    }
}

// Any dims whose tables fit shared memory (dims <= kElemMaxDims), element-
// wise with no transpose: a CTA owns a contiguous range of output words,
// walked in chunks of at most 1024 points. Word (p, j) is
// XP[tile][j] ^ T[j][(p >> 5) & 31] ^ L[j][p & 31] with 1024-point tiles
// (disjoint index bits): three shared loads and two XORs, then the map, and
// four consecutive words leave as one 16-B store. XP (X of the tile base,
// scramble included) advances by the index bits that change from one tile to
// the next; the chunk's points span the current tile and the next.
constexpr uint32_t kElemMaxDims = 128;

template <int MODE, bool U32OUT>
__global__ void __launch_bounds__(kBlock)
    k_sobol_elem(const uint32_t* __restrict__ colsT, const __grid_constant__ SmallArgs args,
                 uint32_t dims, Div32 div_dims, uint64_t first, uint64_t words_total,
                 uint64_t words_per_cta, uint32_t chunk_words, uint32_t* __restrict__ out)
{
    extern __shared__ uint32_t sm[];
    // [32][dims+1] rows: the lanes of a warp read consecutive dimensions of
    // one or a few points, so a padded row per index value keeps them on
    // distinct banks
    const uint32_t ld = dims + 1;
    uint32_t* L = sm;              // [32][ld]: X(l)
    uint32_t* T = L + 32 * ld;     // [32][ld]: X(32 m)
    uint32_t* XP = T + 32 * ld;    // [2][dims]: tiles tc, tc+1
    const uint32_t* words = small_a(args);
    auto col = [&](uint32_t k, uint32_t j) {
        return __ldg(colsT + static_cast<size_t>(k) * dims + j);
    };
    for (uint32_t e = threadIdx.x; e < dims * 32; e += blockDim.x) {
        const uint32_t j = e >> 5, l = e & 31u;
        uint32_t xl = 0, xt = 0;
        for (uint32_t k = 0; k < 5; ++k)
            if ((l >> k) & 1u) {
                xl ^= col(k, j);
                xt ^= col(5 + k, j);
            }
        L[l * ld + j] = xl;
        T[l * ld + j] = xt;
    }
    const uint64_t w0 = static_cast<uint64_t>(blockIdx.x) * words_per_cta;
    const uint64_t w1 = min(words_total, w0 + words_per_cta);
    if (w0 >= w1)
        return;
    // tile of the CTA's first point: XP = X(tile base) (^ XOR words)
    uint64_t tc = (first + w0 / dims) >> 10;
    for (uint32_t j = threadIdx.x; j < dims; j += blockDim.x) {
        uint32_t x0 = (MODE == 0 && words) ? words[j] : 0u;
        for (uint64_t b = tc << 10; b; b &= b - 1)
            x0 ^= col(__ffsll(static_cast<long long>(b)) - 1, j);
        uint32_t x1 = x0;
        for (uint64_t b = (tc << 10) ^ ((tc + 1) << 10); b; b &= b - 1)
            x1 ^= col(__ffsll(static_cast<long long>(b)) - 1, j);
        XP[j] = x0;
        XP[dims + j] = x1;
    }
    const bool vec = (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
    const uint32_t adv = blockDim.x * 4 - 4; // end of a thread's quad -> its next quad
    const uint32_t padv = adv / dims, cadv = adv - padv * dims;
    for (uint64_t c0 = w0; c0 < w1; c0 += chunk_words) {
        const uint32_t cw = static_cast<uint32_t>(w1 - c0 < chunk_words ? w1 - c0 : chunk_words);
        __syncthreads(); // tables / XP ready
        const uint64_t pa = c0 / dims; // chunk's first point (relative)
        const uint64_t ta = (first + pa) >> 10;
        if (ta != tc) { // the chunk starts in tile tc + 1: shift the pair
            for (uint32_t j = threadIdx.x; j < dims; j += blockDim.x) {
                const uint32_t x1 = XP[dims + j];
                uint32_t x2 = x1;
                for (uint64_t b = ((ta) << 10) ^ ((ta + 1) << 10); b; b &= b - 1)
                    x2 ^= col(__ffsll(static_cast<long long>(b)) - 1, j);
                XP[j] = x1;
                XP[dims + j] = x2;
            }
            tc = ta;
            __syncthreads();
        }
        const uint32_t rem = static_cast<uint32_t>(c0 - pa * dims); // column of word c0
        // shared-memory rows of point pr (relative to pa): its XP, T and L rows
        auto rows = [&](uint32_t pr, const uint32_t*& xr, const uint32_t*& tr,
                        const uint32_t*& lr) {
            const uint64_t i = first + pa + pr;
            xr = XP + (static_cast<uint32_t>(i >> 10) != static_cast<uint32_t>(tc)) * dims;
            tr = T + (static_cast<uint32_t>(i >> 5) & 31u) * ld;
            lr = L + (static_cast<uint32_t>(i) & 31u) * ld;
        };
        auto finish = [&](uint32_t v, uint32_t j) {
            if (MODE == 2)
                v = brev32(owen_lk(v, words ? words[j] : 0u));
            return U32OUT ? v : map_bits(v);
        };
        uint32_t* o = out + c0;
        uint32_t e0 = 0;
        if (vec) {
            const uint32_t quads = cw >> 2;
            e0 = quads << 2;
            const uint32_t e = threadIdx.x * 4 + rem;
            uint32_t p = point_of(e, dims, div_dims), c = e - p * dims;
            for (uint32_t qd = threadIdx.x; qd < quads; qd += blockDim.x) {
                uint32_t v[4];
                if (dims >= 8) { // a quad spans at most two points: rows per point
                    const uint32_t *xr, *tr, *lr;
                    rows(p, xr, tr, lr);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        v[k] = finish(xr[c] ^ tr[c] ^ lr[c], c);
                        if (++c == dims) {
                            c = 0;
                            ++p;
                            rows(p, xr, tr, lr);
                        }
                    }
                } else { // few dims: rows per word, no divergent re-fetch
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t *xr, *tr, *lr;
                        rows(p, xr, tr, lr);
                        v[k] = finish(xr[c] ^ tr[c] ^ lr[c], c);
                        if (++c == dims) {
                            c = 0;
                            ++p;
                        }
                    }
                }
                __stcs(reinterpret_cast<uint4*>(o) + qd, make_uint4(v[0], v[1], v[2], v[3]));
                p += padv;
                c += cadv;
                if (c >= dims) {
                    c -= dims;
                    ++p;
                }
            }
        }
        for (uint32_t e = e0 + threadIdx.x; e < cw; e += blockDim.x) {
            const uint32_t p = point_of(e + rem, dims, div_dims), c = e + rem - p * dims;
            const uint32_t *xr, *tr, *lr;
            rows(p, xr, tr, lr);
            o[e] = finish(xr[c] ^ tr[c] ^ lr[c], c);
        }
    }
}

// Any dims, shared-memory tiled: a CTA owns a contiguous range of tiles of
// tp = 2^k consecutive points; a warp computes one (dimension, run of m)
// item at a time: lane l holds points p0 + l + 32 m, whose value is
// X(p0) ^ X(l) ^ X(32 m) (disjoint index bits). X(32 m) for m < tp/32 is a
// per-CTA shared table T[j][m] built once, so the m loop has no dependency
// chain (one LDS + XOR per sample); X(p0) advances from tile to tile through
// the index bits that change. The padded [tp][dims+1] tile is then written
// out with tile_store_rows.
// Sobol' with more dimensions than any shared-memory tile holds (direction
// number files reach tens of thousands): element-wise over the output words,
// each point component the XOR of the columns of its index's set bits
// (digitalnet.cpp:96-110) — correct at any dims, not a fast path.
template <int MODE, bool U32OUT>
__global__ void __launch_bounds__(kBlock)
    k_sobol_huge(const uint32_t* __restrict__ colsT, const __grid_constant__ SmallArgs args,
                 uint32_t dims, Div32 div_dims, uint64_t first, uint64_t n,
                 uint32_t* __restrict__ out)
{
    const uint32_t* words = small_a(args);
    const uint64_t total = n * dims;
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t p = e / dims;
        const uint32_t j = static_cast<uint32_t>(e - p * dims);
        uint32_t x = (MODE == 0 && words) ? words[j] : 0u;
        for (uint64_t b = first + p; b; b &= b - 1)
            x ^= __ldg(colsT + static_cast<size_t>(__ffsll(static_cast<long long>(b)) - 1) * dims + j);
        if (MODE == 2)
            x = brev32(owen_lk(x, words ? words[j] : 0u));
        out[e] = U32OUT ? x : map_bits(x);
    }
    (void)div_dims;
}

template <int MODE, bool U32OUT, int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_sobol_tiled(const uint32_t* __restrict__ colsT, const __grid_constant__ SmallArgs args,
                  uint32_t dims, Div32 div_dims, uint32_t tp, uint64_t first, uint64_t n,
                  uint64_t tile0, uint64_t ntiles, uint32_t* __restrict__ out)
{
    extern __shared__ uint32_t smem[];
    const uint32_t ld = dims + 1;
    const uint32_t mt = tp / 32; // m steps per tile
    uint32_t* tile = smem;
    uint32_t* T = smem + static_cast<size_t>(tp) * ld; // [dims][mt]: X(32 m)
    uint32_t* XP = T + static_cast<size_t>(dims) * mt; // [dims]: words ^ X(p0)
    const uint32_t* words = small_a(args);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u, nwarps = blockDim.x >> 5;
    auto col = [&](uint32_t k, uint32_t j) {
        return __ldg(colsT + static_cast<size_t>(k) * dims + j);
    };
    for (uint32_t e = threadIdx.x; e < dims * mt; e += blockDim.x) {
        const uint32_t j = e / mt, m = e - j * mt;
        uint32_t x = 0;
        for (uint32_t k = 0; (m >> k) != 0; ++k)
            if ((m >> k) & 1u)
                x ^= col(5 + k, j);
        T[e] = x;
    }
    // a contiguous range of tiles per CTA: X(p0) advances incrementally
    // (only the index bits that change between consecutive tiles), and
    // several warps share a dimension when dims < warps per CTA
    const uint64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
    const uint64_t tb = tile0 + blockIdx.x * per;
    const uint64_t te = min(tile0 + ntiles, tb + per);
    const uint32_t runs = dims >= nwarps ? 1u : nwarps / dims;
    const uint32_t mchunk = (mt + runs - 1) / runs;
    uint64_t prev = 0;
    for (uint64_t t = tb; t < te; ++t) {
        const uint64_t p0 = t * tp; // absolute index of the tile's first point
        __syncthreads(); // T/L ready (first tile), XP and the tile free (later tiles)
        for (uint32_t j = threadIdx.x; j < dims; j += blockDim.x) {
            uint32_t x;
            uint64_t b;
            if (t == tb) {
                x = (MODE == 0 && words) ? words[j] : 0u;
                b = p0;
            } else {
                x = XP[j];
                b = p0 ^ prev;
            }
            for (; b; b &= b - 1)
                x ^= col(__ffsll(static_cast<long long>(b)) - 1, j);
            XP[j] = x;
        }
        prev = p0;
        __syncthreads();
        for (uint32_t item = warp; item < dims * runs; item += nwarps) {
            const uint32_t j = runs == 1 ? item : item % dims;
            const uint32_t mb = (runs == 1 ? 0u : item / dims) * mchunk;
            const uint32_t me = min(mt, mb + mchunk);
            uint32_t x = XP[j]; // ^ X(lane), from the columns (no table: dims can be large)
            for (uint32_t k = 0; k < 5; ++k)
                if ((lane >> k) & 1u)
                    x ^= col(k, j);
            const uint32_t seed = (MODE == 2 && words) ? words[j] : 0u;
            const uint32_t* Tj = T + j * mt;
            for (uint32_t m = mb; m < me; ++m) {
                const uint64_t i = p0 + lane + 32ull * m;
                uint32_t v = x ^ Tj[m];
                if (MODE == 2)
                    v = brev32(owen_lk(v, seed));
                if (i - first < n)
                    tile[(lane + 32 * m) * ld + j] = U32OUT ? v : map_bits(v);
            }
        }
        __syncthreads();
        // rows [lo, hi) of the tile that belong to [first, first + n)
        const uint64_t lo = p0 > first ? p0 : first;
        const uint64_t hi = (p0 + tp < first + n) ? p0 + tp : first + n;
        tile_store_rows(tile, ld, dims, div_dims, static_cast<uint32_t>(lo - p0),
                        static_cast<uint32_t>(hi - lo), out + (lo - first) * dims);
        __syncthreads();
    }
}

// dims 1 and 2: a lane owns Q = 8 / D consecutive points (8 words, one
// 256-bit store); a warp step covers PPS = 32 Q points. Point base + o of a
// lane has value X(P) ^ X(u PPS) ^ X(lane Q) ^ X(o) (disjoint index bits):
// X(o) are 7 register constants, the step update is the usual compile-time
// ctz mask. One XOR + the map per sample.
template <int D, int MODE, bool U32OUT>
__global__ void __launch_bounds__(kBlock)
    k_sobol_narrow(const uint32_t* __restrict__ colsT, const __grid_constant__ SmallArgs args,
                   uint64_t first, uint64_t n, uint64_t tile0, uint64_t ntiles, uint64_t per_warp,
                   uint32_t* __restrict__ out)
{
    constexpr int Q = 8 / D, LOG_Q = D == 1 ? 3 : 2;
    constexpr int LOG_PPS = LOG_Q + 5, PPS = 1 << LOG_PPS;
    constexpr int LOG_TP = LOG_PPS + 5;
    uint64_t t, tend;
    if (!warp_tiles(tile0, ntiles, per_warp, t, tend))
        return;
    const uint32_t lane = threadIdx.x & 31u;
    auto col = [&](uint32_t k, int d) { return __ldg(colsT + k * D + d); };
    uint32_t xo[Q][D], Dm[5][D], xl[D], xp[D], seed[D], omul[D], oadd[D];
    const uint32_t* words = small_a(args);
#pragma unroll
    for (int d = 0; d < D; ++d) {
        seed[d] = (MODE == 2 && words) ? words[d] : 0u;
        omul[d] = (seed[d] >> 16) | 1u;
        oadd[d] = seed[d] * omul[d];
        uint32_t acc = 0;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            acc ^= col(LOG_PPS + k, d);
            Dm[k][d] = acc;
        }
#pragma unroll
        for (int o = 0; o < Q; ++o) {
            uint32_t v = 0;
#pragma unroll
            for (int k = 0; k < LOG_Q; ++k)
                if ((o >> k) & 1)
                    v ^= col(k, d);
            xo[o][d] = v;
        }
        uint32_t v = (MODE == 0 && words) ? words[d] : 0u;
#pragma unroll
        for (int k = 0; k < 5; ++k)
            if ((lane >> k) & 1u)
                v ^= col(LOG_Q + k, d);
        xl[d] = v;
        xp[d] = 0;
        for (uint64_t b = t; b; b &= b - 1)
            xp[d] ^= col(LOG_TP + __ffsll(static_cast<long long>(b)) - 1, d);
    }
    for (;;) {
        const uint64_t p0 = (t << LOG_TP) + lane * Q; // lane's first point at step 0
        uint32_t x[D], y[8];
#pragma unroll
        for (int d = 0; d < D; ++d)
            x[d] = xp[d] ^ xl[d];
        const uint64_t lo = t << LOG_TP, hi = (t + 1) << LOG_TP;
        const bool full = lo >= first && hi <= first + n;
        uint32_t* o = out + (p0 - first) * D;
        auto group = [&](uint32_t v, auto check) {
#pragma unroll
            for (uint32_t w = 0; w < 8; ++w) {
                const uint32_t u = 8 * v + w;
#pragma unroll
                for (int q = 0; q < Q; ++q)
#pragma unroll
                    for (int d = 0; d < D; ++d) {
                        uint32_t val = x[d] ^ xo[q][d];
                        if (MODE == 2)
                            val = brev32(owen_lk_folded(val, omul[d], oadd[d]));
                        y[q * D + d] = U32OUT ? val : map_bits(val);
                    }
                if (!decltype(check)::value) {
                    store_vec<8>(o + u * 256, y);
                } else {
#pragma unroll
                    for (int q = 0; q < Q; ++q)
                        if ((p0 + u * PPS + q) - first < n)
#pragma unroll
                            for (int d = 0; d < D; ++d)
                                o[u * 256 + q * D + d] = y[q * D + d];
                }
                if (w < 7) {
#pragma unroll
                    for (int d = 0; d < D; ++d)
                        x[d] ^= Dm[ctz_const(w + 1)][d];
                }
            }
#pragma unroll
            for (int d = 0; d < D; ++d)
                x[d] ^= (v == 1) ? Dm[4][d] : Dm[3][d];
        };
        if (full) {
#pragma unroll 1
            for (uint32_t v = 0; v < 4; ++v)
                group(v, std::false_type{});
        } else {
#pragma unroll 1
            for (uint32_t v = 0; v < 4; ++v)
                group(v, std::true_type{});
        }
        if (++t >= tend)
            break;
        const int cz = __ffsll(static_cast<long long>(t)) - 1;
        for (int k = 0; k <= cz; ++k)
#pragma unroll
            for (int d = 0; d < D; ++d)
                xp[d] ^= col(LOG_TP + k, d);
    }
}

// Lattice, dims 1 and 2 (same lane layout as k_sobol_narrow):
// brev(i) = brev(P + lane Q) + brev(u PPS) + brev(o), disjoint bits.
template <int D, bool U32OUT>
__global__ void __launch_bounds__(kBlock)
    k_lattice_narrow(const uint32_t* __restrict__ unused, const __grid_constant__ SmallArgs args,
                     uint64_t first, uint64_t n, uint64_t tile0, uint64_t ntiles,
                     uint64_t per_warp, uint32_t* __restrict__ out)
{
    constexpr int Q = 8 / D, LOG_Q = D == 1 ? 3 : 2;
    constexpr int LOG_PPS = LOG_Q + 5, PPS = 1 << LOG_PPS;
    constexpr int LOG_TP = LOG_PPS + 5;
    uint64_t t, tend;
    if (!warp_tiles(tile0, ntiles, per_warp, t, tend))
        return;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t* g = small_a(args);
    const uint32_t* sh = small_b(args);
    uint32_t gv[D], sv[D], G[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
        gv[d] = g[d];
        sv[d] = sh ? sh[d] : 0u;
        G[d] = gv[d] << (27 - LOG_PPS);
    }
    for (; t < tend; ++t) {
        const uint64_t p0 = (t << LOG_TP) + lane * Q;
        const uint32_t b = brev32(static_cast<uint32_t>(p0));
        uint32_t x0[D], y[8];
#pragma unroll
        for (int d = 0; d < D; ++d)
            x0[d] = b * gv[d] + sv[d];
        const uint64_t lo = t << LOG_TP, hi = (t + 1) << LOG_TP;
        const bool full = lo >= first && hi <= first + n;
        uint32_t* o = out + (p0 - first) * D;
#pragma unroll 1
        for (uint32_t v = 0; v < 4; ++v) {
            const uint32_t cv = ((v & 1u) << 1) | (v >> 1);
#pragma unroll
            for (uint32_t w = 0; w < 8; ++w) {
                const uint32_t u = 8 * v + w;
                const uint32_t cw = (((w & 1u) << 2) | (w & 2u) | (w >> 2)) << 2;
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    // brev of the in-lane offset q (LOG_Q bits) at the top
                    const uint32_t cq = (D == 1 ? (((q & 1) << 2) | (q & 2) | (q >> 2))
                                                : (((q & 1) << 1) | (q >> 1)))
                                        << (32 - LOG_Q);
#pragma unroll
                    for (int d = 0; d < D; ++d) {
                        const uint32_t xx = x0[d] + (cw | cv) * G[d] + cq * gv[d];
                        y[q * D + d] = U32OUT ? xx : map_bits(xx);
                    }
                }
                if (full) {
                    store_vec<8>(o + u * 256, y);
                } else {
#pragma unroll
                    for (int q = 0; q < Q; ++q)
                        if ((p0 + u * PPS + q) - first < n)
#pragma unroll
                            for (int d = 0; d < D; ++d)
                                o[u * 256 + q * D + d] = y[q * D + d];
                }
            }
        }
    }
}

// x_j(i) = brev((uint32_t)i) * g_j + s_j (mod 2^32). Inside a tile the index
// is P | (u << LOG_PPS) | r with disjoint bits, so brev(i) = brev(P | r) +
// brev5(u) << (27 - LOG_PPS): one IMAD per sample with a compile-time
// multiplier.
template <int DPL, int LOG_PPS, bool U32OUT>
__global__ void __launch_bounds__(kBlock)
    k_lattice_fast(const uint32_t* __restrict__ unused, const __grid_constant__ SmallArgs args,
                   uint64_t first, uint64_t n, uint64_t tile0, uint64_t ntiles, uint64_t per_warp,
                   uint32_t* __restrict__ out)
{
    constexpr int PPS = 1 << LOG_PPS;
    constexpr int LPP = 32 >> LOG_PPS;
    constexpr int DIMS = DPL * LPP;
    constexpr int LOG_TP = LOG_PPS + 5;
    uint64_t t, tend;
    if (!warp_tiles(tile0, ntiles, per_warp, t, tend))
        return;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t r = lane / LPP, dq = lane % LPP;
    uint32_t gv[DPL], sv[DPL], G[DPL];
    load_small<DPL>(small_a(args) + dq * DPL, gv);
    const uint32_t* shifts = small_b(args);
#pragma unroll
    for (int e = 0; e < DPL; ++e) {
        sv[e] = 0;
        G[e] = gv[e] << (27 - LOG_PPS);
    }
    if (shifts)
        load_small<DPL>(shifts + dq * DPL, sv);
    for (; t < tend; ++t) {
        const uint64_t p0 = (t << LOG_TP) + r;
        const uint32_t b = brev32(static_cast<uint32_t>(p0));
        uint32_t x0[DPL], y[DPL];
#pragma unroll
        for (int e = 0; e < DPL; ++e)
            x0[e] = b * gv[e] + sv[e];
        const uint64_t lo = t << LOG_TP, hi = (t + 1) << LOG_TP;
        const bool full = lo >= first && hi <= first + n;
        uint32_t* o = out + (p0 - first) * DIMS + dq * DPL;
        // u = 8v + w: brev5(u) = brev3(w) << 2 | brev2(v); the v part is
        // added once per group of 8, the w part is a compile-time multiplier.
        auto group = [&](uint32_t v, auto check) {
            const uint32_t cv = ((v & 1u) << 1) | (v >> 1);
            uint32_t xv[DPL];
#pragma unroll
            for (int e = 0; e < DPL; ++e)
                xv[e] = x0[e] + cv * G[e];
#pragma unroll
            for (uint32_t w = 0; w < 8; ++w) {
                const uint32_t u = 8 * v + w;
                const uint32_t cw = (((w & 1u) << 2) | (w & 2u) | (w >> 2)) << 2;
#pragma unroll
                for (int e = 0; e < DPL; ++e) {
                    const uint32_t xx = xv[e] + cw * G[e];
                    y[e] = U32OUT ? xx : map_bits(xx);
                }
                if (!decltype(check)::value || (p0 + u * PPS) - first < n)
                    store_vec<DPL>(o + u * 32 * DPL, y);
            }
        };
        if (full) {
#pragma unroll 1
            for (uint32_t v = 0; v < 4; ++v)
                group(v, std::false_type{});
        } else {
#pragma unroll 1
            for (uint32_t v = 0; v < 4; ++v)
                group(v, std::true_type{});
        }
    }
}

__global__ void __launch_bounds__(kBlock)
    k_lattice_generic(const __grid_constant__ SmallArgs args, uint32_t dims, Div32 div_dims,
                      uint64_t first, uint32_t elems, bool u32out, uint32_t* __restrict__ out)
{
    const uint32_t* g = small_a(args);
    const uint32_t* shifts = small_b(args);
    const uint32_t stride = gridDim.x * blockDim.x;
    auto value = [&](uint32_t p, uint32_t j) {
        uint32_t x = brev32(static_cast<uint32_t>(first + p)) * g[j];
        if (shifts)
            x += shifts[j];
        return u32out ? x : map_bits(x);
    };
    const uint32_t t0 = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t e0 = 0;
    if ((reinterpret_cast<uintptr_t>(out) & 15u) == 0) {
        // four consecutive elements per thread, one 16-B streaming store;
        // (point, dim) walk with the row wrap checked per element
        const uint32_t quads = elems >> 2;
        e0 = quads << 2;
        for (uint32_t qd = t0; qd < quads; qd += stride) {
            uint32_t p = point_of(qd * 4, dims, div_dims), j = qd * 4 - p * dims;
            uint32_t v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                v[k] = value(p, j);
                if (++j == dims) {
                    j = 0;
                    ++p;
                }
            }
            __stcs(reinterpret_cast<uint4*>(out) + qd, make_uint4(v[0], v[1], v[2], v[3]));
        }
    }
    for (uint32_t e = e0 + t0; e < elems; e += stride) {
        const uint32_t p = point_of(e, dims, div_dims);
        out[e] = value(p, e - p * dims);
    }
}

// ----------------------------------------------------------------- Halton

// dims == 1, base 2 (config C1: van der Corput = brev(i mod 2^31)); four
// consecutive points per thread, one 128-bit store.
// dims == 1, base 2 from a first index that is a multiple of 8 into 32-B
// aligned output: eight points per thread (brev(i + c) = brev(i) + brev(c)
// for c < 8), one 256-bit streaming store — 64 MiB one-shot fills reach the
// write-only store kernel's rate under the same conditions (0.72 vs 0.63 of
// the copy peak with 128-bit stores)
template <bool U32OUT>
__global__ void __launch_bounds__(kBlock)
    k_vdc8(uint64_t first, uint64_t n, uint32_t* __restrict__ out)
{
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint64_t octs = (n + 7) / 8;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < octs;
         q += stride) {
        const uint64_t k = q * 8;
        uint32_t v[8];
        const uint32_t b = brev32(static_cast<uint32_t>(first + k) & 0x7fffffffu);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            // first + k is a multiple of 8 (launcher): brev(i + c) = brev(i) + brev(c)
            const uint32_t x = b + (c ? (__brev(static_cast<uint32_t>(c))) : 0u);
            v[c] = U32OUT ? x : map_bits(x);
        }
        if (k + 8 <= n) {
            uint32_t* p = out + k;
            asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]),
                         "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                         : "memory");
        } else {
            for (int c = 0; c < 8; ++c)
                if (k + c < n)
                    out[k + c] = v[c];
        }
    }
}

template <bool U32OUT>
__global__ void __launch_bounds__(kBlock)
    k_vdc(uint64_t first, uint64_t n, uint32_t* __restrict__ out)
{
    // programmatic dependent launch: let the next kernel in the stream start
    // its launch now, and wait for the previous grid (its stores) before ours
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint64_t quads = (n + 3) / 4;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const bool aligned = (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
    for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < quads;
         q += stride) {
        const uint64_t k = q * 4;
        uint32_t v[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t x = brev32(static_cast<uint32_t>(first + k + c) & 0x7fffffffu);
            v[c] = U32OUT ? x : map_bits(x);
        }
        if (aligned && k + 4 <= n) {
            __stcs(reinterpret_cast<uint4*>(out + k), make_uint4(v[0], v[1], v[2], v[3]));
        } else {
            for (int c = 0; c < 4; ++c)
                if (k + c < n)
                    out[k + c] = v[c];
        }
    }
}

// Continuation state of one dimension's incremental walk (shared memory or
// registers, 20 words): valid when `live` and the next run starts at index `next`.
struct HaltonState {
    uint32_t next, lob, h1, live;
    HiRecord r0, r1;
    uint32_t g0, mulg; // hi_advance state of r1
};
static_assert(sizeof(HaltonState) % 16 == 0, "HaltonState is whole 16-B units");

// No memory clobber: the tile is only read back after __syncthreads(), and
// leaving it out lets the table loads of later steps move ahead of the stores.
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v)
{
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v));
}

// One warp, one dimension, `cnt` consecutive indices from i0 into the
// padded tile column at shared address col (row stride ld words). `st` (or
// null) carries the incremental state from the previous contiguous run.
template <bool U32OUT>
__device__ __forceinline__ void halton_run(const RadicalDim& r, uint32_t i0, uint32_t cnt,
                                           uint32_t lane, uint32_t col, uint32_t ld,
                                           HaltonState* st)
{
    const uint32_t row = ld * 4;
    if (r.base == 2) {
        for (uint32_t p = lane; p < cnt; p += 32) {
            const uint32_t x = brev32((i0 + p) & 0x7fffffffu);
            sts32(col + p * row, U32OUT ? x : map_bits(x));
        }
    } else if (r.ftable && i0 <= 0xffffffffu - cnt) {
        // incremental split i = h * G + lo (G = fgroup > 32): the warp's 32
        // indices of a step span h, or h and h+1 on the step that crosses a
        // multiple of G; the records of h and h+1 are warp-uniform, so a lane
        // adds one table lookup, one IMAD and an integer division by magic.
        const uint32_t G = r.fgroup;
        uint32_t lob, h1, g0, mulg;
        HiRecord r0, r1;
        if (st && st->live && st->next == i0) {
            lob = st->lob;
            h1 = st->h1;
            r0 = st->r0;
            r1 = st->r1;
            g0 = st->g0;
            mulg = st->mulg;
        } else {
            const uint32_t ir = i0 - div32(i0, r.divmp) * r.maxpow; // i %= maxpow
            uint32_t h = div32(ir, r.fdivg);
            lob = ir - h * G;
            r0 = hi_record(h, r, g0, mulg);
            h1 = h;
            r1 = r0;
            hi_advance(h1, r1, g0, mulg, r);
        }
        // Rows up to the next multiple of 32 past cnt stay inside the tile
        // (tp is a multiple of 32), so every step stores unconditionally.
        const uint32_t stride = 32 * row;
        uint32_t addr = col + lane * row;
        const uint32_t steps = (cnt + 31) >> 5;
        for (uint32_t s = 0; s < steps;) {
            // steps whose 32 indices all lie in h's block: one record
            const uint32_t nf = min(steps - s, (G - lob) >> 5);
            // quotient-only table: the remainder rT = -qT * G mod 2^32 is
            // one IMAD, and the stream is 4 B per sample instead of 8
            // (+10 % at 32 dims: the L2 table stream is the bound)
            const uint32_t* tab = r.fqx + lob + lane;
            const uint32_t negG = 0u - G;
#pragma unroll 4
            for (uint32_t e = 0; e < nf; ++e) {
                const uint32_t v = __ldg(tab);
                const uint32_t x = v + r0.qa + (v * negG >= r0.thr ? 1u : 0u);
                sts32(addr, U32OUT ? x : map_bits(x));
                addr += stride;
                tab += 32;
            }
            lob += nf << 5;
            s += nf;
            if (lob < G && s < steps) { // the step crossing into h+1's block
                uint32_t lo = lob + lane;
                const bool up = lo >= G;
                lo = up ? lo - G : lo;
                const uint32_t v = __ldg(r.fqx + lo);
                const uint32_t x = v + (up ? r1.qa : r0.qa) + (v * (0u - G) >= (up ? r1.thr : r0.thr) ? 1u : 0u);
                sts32(addr, U32OUT ? x : map_bits(x));
                addr += stride;
                lob += 32;
                ++s;
            }
            if (lob >= G) {
                lob -= G;
                r0 = r1;
                hi_advance(h1, r1, g0, mulg, r);
            }
        }
        if (st) { // every lane: the state may live in registers (k_runs, k_tma)
            st->next = i0 + (steps << 5);
            st->lob = lob;
            st->h1 = h1;
            st->r0 = r0;
            st->r1 = r1;
            st->g0 = g0;
            st->mulg = mulg;
            st->live = 1;
        }
    } else {
        for (uint32_t p = lane; p < cnt; p += 32) {
            const uint32_t x = radical_fixed(i0 + p, r);
            sts32(col + p * row, U32OUT ? x : map_bits(x));
        }
    }
}

// Prime-base Halton (radical.cpp:240-269), shared-memory tiled: a CTA owns
// a contiguous range of tiles of tp consecutive points; a warp computes one
// (dimension, run of consecutive points) item at a time into a padded
// [tp][dims+1] shared tile (one base per warp -> uniform digit loops and
// records, halton_run), then the whole tile — tp*dims consecutive output
// words — is written out coalesced (tile_store_rows). With one run
// per dimension the same warp owns a dimension in every tile, so its
// incremental state carries over from tile to tile (HaltonState, after the
// tile in shared memory).
template <bool U32OUT, int BLOCK>
__global__ void __launch_bounds__(BLOCK)
    k_halton_tiled(const RadicalDim* __restrict__ rd, uint32_t dims, Div32 div_dims, uint32_t tp,
                   uint64_t first, uint64_t n, uint64_t ntiles, uint32_t* __restrict__ out)
{
    extern __shared__ __align__(16) uint32_t tile[];
    const uint32_t ld = dims | 1u; // odd row stride: a column store hits 32 banks
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u, nwarps = blockDim.x >> 5;
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(tile));
    // (dim, point run) work items: several warps share a dimension when
    // dims < warps per CTA (no carried state then)
    const bool carry = dims >= nwarps; // launch_halton sizes the state slots alike
    const uint32_t runs = carry ? 1u : nwarps / dims;
    HaltonState* states =
        carry ? reinterpret_cast<HaltonState*>(tile + ((tp * ld + 15u) & ~15u)) : nullptr;
    if (states)
        for (uint32_t j = threadIdx.x; j < dims; j += blockDim.x)
            states[j].live = 0;
    __syncthreads();
    const uint64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
    const uint64_t t1 = min(ntiles, (blockIdx.x + 1) * per);
    for (uint64_t t = blockIdx.x * per; t < t1; ++t) {
        const uint64_t p0 = t * tp;
        const uint32_t cnt = static_cast<uint32_t>(n - p0 < tp ? n - p0 : tp);
        const uint32_t chunk = ((cnt + runs - 1) / runs + 31u) & ~31u;
        for (uint32_t item = warp; item < dims * runs; item += nwarps) {
            const uint32_t j = runs == 1 ? item : item % dims;
            const uint32_t pb = (runs == 1 ? 0u : item / dims) * chunk;
            const uint32_t pe = min(cnt, pb + chunk);
            if (pb < pe)
                halton_run<U32OUT>(rd[j], static_cast<uint32_t>(first + p0 + pb), pe - pb, lane,
                                   sbase + (pb * ld + j) * 4, ld, states ? states + j : nullptr);
        }
        __syncthreads();
        tile_store_rows(tile, ld, dims, div_dims, 0, cnt, out + p0 * dims);
        __syncthreads();
    }
}

// Column walkers for the one-dimension-per-warp fills (k_runs, k_tma): a
// warp writes `cnt` consecutive points (from index i0) of dimension j into
// the shared column at address col, row stride ld words, carrying State from
// one call to the next (in registers); wsm is the warp's 32-word scratch.
template <bool U32OUT>
struct HaltonWalk {
    const RadicalDim* rd;
    using State = HaltonState;
    __device__ __forceinline__ void reset(State& st) const { st.live = 0; }
    __device__ __forceinline__ void run(uint32_t j, uint64_t i0, uint32_t cnt, uint32_t lane,
                                        uint32_t col, uint32_t ld, State& st, uint32_t*) const
    {
        halton_run<U32OUT>(rd[j], static_cast<uint32_t>(i0), cnt, lane, col, ld, &st);
    }
};

// Sobol' (digitalnet.cpp:96-110) from a 32-aligned i0: with i = 32 H + l and
// H = 32 b + t (disjoint index bits) the point is X(1024 b) ^ X(32 t) ^ X(l):
// X(l) stays in a register per lane, X(32 t) for t < 32 sits in the warp's
// scratch (one broadcast load per step) and X(1024 b) (with the XOR word)
// advances once per 32 steps by the columns of the bits that change.
// MODE 2: cols are bit-reversed, finished by brev(owen_lk(., seed)).
template <int MODE, bool U32OUT>
struct SobolWalk {
    const uint32_t* cols; // [52][dims]
    uint32_t dims;
    SmallArgs words;
    struct State {
        uint64_t next, h;
        uint32_t xq, xl, live, pad;
    };
    __device__ __forceinline__ void reset(State& st) const { st.live = 0; }
    __device__ __forceinline__ uint32_t col(uint32_t k, uint32_t j) const
    {
        return __ldg(cols + static_cast<size_t>(k) * dims + j);
    }
    __device__ __forceinline__ void run(uint32_t j, uint64_t i0, uint32_t cnt, uint32_t lane,
                                        uint32_t colad, uint32_t ld, State& st,
                                        uint32_t* wsm) const
    {
        const uint32_t* w = small_a(words);
        const uint32_t seed = MODE == 2 && w ? w[j] : 0u;
        if (!st.live || st.next != i0) {
            uint32_t xl = 0, xt = 0;
            for (uint32_t k = 0; k < 5; ++k)
                if ((lane >> k) & 1u) {
                    xl ^= col(k, j);
                    xt ^= col(5 + k, j);
                }
            __syncwarp();
            wsm[lane] = xt;
            uint32_t xb = MODE == 0 && w ? w[j] : 0u;
            for (uint64_t b = (i0 >> 10) << 10; b; b &= b - 1)
                xb ^= col(__ffsll(static_cast<long long>(b)) - 1, j);
            st.h = i0 >> 5;
            st.xl = xl;
            st.xq = xb ^ xl;
            st.live = 1;
        }
        __syncwarp();
        const uint32_t row = ld * 4, stride = 32 * row;
        uint32_t addr = colad + lane * row;
        uint64_t h = st.h;
        uint32_t xq = st.xq;
        const uint32_t steps = (cnt + 31) >> 5;
        for (uint32_t s = 0; s < steps;) {
            const uint32_t t0 = static_cast<uint32_t>(h) & 31u;
            const uint32_t m = min(steps - s, 32u - t0);
#pragma unroll 4
            for (uint32_t e = 0; e < m; ++e) {
                uint32_t v = xq ^ wsm[t0 + e];
                if (MODE == 2)
                    v = brev32(owen_lk(v, seed));
                sts32(addr, U32OUT ? v : map_bits(v));
                addr += stride;
            }
            s += m;
            h += m;
            if ((static_cast<uint32_t>(h) & 31u) == 0) { // next 1024-block: bits 10.. change
                const uint64_t b = h >> 5;
                const int cz = __ffsll(static_cast<long long>(b)) - 1;
                for (int k = 0; k <= cz; ++k)
                    xq ^= col(10 + k, j);
            }
        }
        st.h = h;
        st.xq = xq;
        st.next = i0 + (static_cast<uint64_t>(steps) << 5);
    }
};

__device__ __forceinline__ void bar_named(uint32_t id, uint32_t threads)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Prime-base Halton for dims <= 32, one dimension per warp for the whole
// launch: a CTA of runs x dims warps (runs = min(15, 32 / dims)) owns a
// contiguous range of sub-tiles of `chunk` points; run r walks its own
// contiguous part of that range, one sub-tile at a time, so every warp's
// incremental state (HaltonState) stays in registers from sub-tile to
// sub-tile and each warp step is just the table lookup, IMAD, magic division
// and map. A run's dims warps fill its padded [chunk][dims | 1] sub-tile,
// meet at their own named barrier, and write it out as consecutive words
// (each thread keeps a fixed column and a fixed shared-memory stride), so
// runs never wait for each other.
template <class W, int DPW>
__global__ void __launch_bounds__(1024, 1)
    k_runs(const __grid_constant__ W w, uint32_t dims, uint32_t runs, uint32_t chunk,
           uint64_t first, uint64_t n, uint64_t nsub, uint32_t* __restrict__ out)
{
    extern __shared__ __align__(16) uint32_t tile[];
    const uint32_t ld = dims | 1u; // odd row stride: a column store hits 32 banks
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    // DPW dimensions per warp (dims % DPW == 0): warp j of a run walks
    // dimensions j, j + wpr, ...
    const uint32_t wpr = dims / DPW;
    const uint32_t run = warp / wpr, j = warp - run * wpr;
    const uint32_t nthr = wpr * 32, tid = threadIdx.x - run * nthr;
    const uint32_t* sub = tile + static_cast<size_t>(run) * chunk * ld;
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(sub));
    // balanced split of the sub-tiles over the CTAs, then over the runs
    const uint64_t s0 = nsub * blockIdx.x / gridDim.x, s1 = nsub * (blockIdx.x + 1) / gridDim.x;
    const uint64_t q = (s1 - s0 + runs - 1) / runs;
    const uint64_t r0 = s0 + run * q, r1 = min(s1, r0 + q);
    // store mapping: thread tid owns the quads at words 4*tid + k*4*nthr of a
    // sub-tile, i.e. a fixed column and rows advancing by 128 / DPW (4*nthr =
    // 128*dims/DPW). Sub-tiles start on multiples of 32 points, so with out
    // 16-B aligned every quad is a 16-B store; its words sit at fixed offsets
    // from the row start (offk: +1 per row wrap when dims % 4 != 0).
    const bool vec = (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
    const uint32_t e0 = vec ? tid * 4 : tid, row0 = e0 / dims, col0 = e0 - row0 * dims;
    const uint32_t pad = ld - dims;
    const uint32_t off1 = 1 + (col0 + 1) / dims * pad, off2 = 2 + (col0 + 2) / dims * pad,
                   off3 = 3 + (col0 + 3) / dims * pad;
    uint32_t* wsm = tile + static_cast<size_t>(runs) * chunk * ld + warp * 32 * DPW;
    typename W::State st[DPW];
#pragma unroll
    for (int k = 0; k < DPW; ++k)
        w.reset(st[k]);
    for (uint64_t s = r0; s < r1; ++s) {
        const uint64_t p0 = s * chunk;
        const uint32_t cnt = static_cast<uint32_t>(n - p0 < chunk ? n - p0 : chunk);
#pragma unroll
        for (int k = 0; k < DPW; ++k)
            w.run(j + k * wpr, first + p0, cnt, lane, sbase + (j + k * wpr) * 4, ld, st[k],
                  wsm + 32 * k);
        bar_named(1 + run, nthr);
        const uint32_t words = cnt * dims;
        uint32_t* o = out + p0 * dims;
        const uint32_t* src = sub + row0 * ld + col0;
        uint32_t e = e0;
        if (!vec) {
#pragma unroll 4
            for (; e < words; e += nthr, src += 32 / DPW * ld)
                __stcs(o + e, *src);
        } else if ((dims & 3u) == 0) {
#pragma unroll 2
            for (; e < words; e += 4 * nthr, src += 128 / DPW * ld)
                __stcs(reinterpret_cast<uint4*>(o + e), make_uint4(src[0], src[1], src[2], src[3]));
        } else {
#pragma unroll 2
            for (; e + 4 <= words; e += 4 * nthr, src += 128 / DPW * ld)
                __stcs(reinterpret_cast<uint4*>(o + e),
                       make_uint4(src[0], src[off1], src[off2], src[off3]));
            if (e < words) { // the ragged end of the last sub-tile: < 4 words
                o[e] = src[0];
                if (e + 1 < words)
                    o[e + 1] = src[off1];
                if (e + 2 < words)
                    o[e + 2] = src[off2];
            }
        }
        bar_named(1 + run, nthr);
    }
}

// dims 33..32*DMAX with no exact per-warp split: one run of 32 warps per
// CTA, warp j walking dims j, j + 32, ... (< dims), the padded sub-tile
// written with the generic row copy (tile_store_rows, any dims).
template <class W, int DMAX>
__global__ void __launch_bounds__(1024, 1)
    k_runs_wide(const __grid_constant__ W w, uint32_t dims, Div32 div_dims, uint32_t chunk,
                uint64_t first, uint64_t n, uint64_t nsub, uint32_t* __restrict__ out)
{
    extern __shared__ __align__(16) uint32_t tile[];
    const uint32_t ld = dims | 1u;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(tile));
    uint32_t* wsm = tile + static_cast<size_t>(chunk) * ld + warp * 32 * DMAX;
    const uint64_t s0 = nsub * blockIdx.x / gridDim.x, s1 = nsub * (blockIdx.x + 1) / gridDim.x;
    typename W::State st[DMAX];
#pragma unroll
    for (int k = 0; k < DMAX; ++k)
        w.reset(st[k]);
    for (uint64_t s = s0; s < s1; ++s) {
        const uint64_t p0 = s * chunk;
        const uint32_t cnt = static_cast<uint32_t>(n - p0 < chunk ? n - p0 : chunk);
#pragma unroll
        for (int k = 0; k < DMAX; ++k) {
            const uint32_t j = warp + 32 * k;
            if (j < dims)
                w.run(j, first + p0, cnt, lane, sbase + j * 4, ld, st[k], wsm + 32 * k);
        }
        __syncthreads();
        tile_store_rows(tile, ld, dims, div_dims, 0, cnt, out + p0 * dims);
        __syncthreads();
    }
}

__device__ __forceinline__ void mbar_init(uint32_t addr, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t addr)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity)
{
    uint32_t ok;
    do {
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok)
                     : "r"(addr), "r"(parity)
                     : "memory");
    } while (!ok);
}

// Fills with dims % 32 == 0, stored by TMA: the k_runs walk
// (one dimension of a 32-dimension column block per warp, state in
// registers) into a ring of nbuf sub-tiles of `rows` points laid out exactly
// as the block's 128-B output row segments (whole cache lines) with the
// 128-B swizzle, so a column store by 32 lanes is a 4-way bank conflict
// instead of 32-way, and the tensor-map store (cp.async.bulk.tensor, boxes of
// 256 rows) runs asynchronously while the warps walk the next sub-tiles.
// full[b]: the 32 warps have written sub-tile b (count 32); empty[b]: its
// bulk store has finished reading shared memory (count 1, warp 0 lane 0,
// which also issues the stores; in block 0 it walks base 2, the cheapest).
template <class W>
__global__ void __launch_bounds__(1024, 1)
    k_tma(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ W w, uint32_t rows,
          uint32_t nbuf, uint32_t ncb, uint32_t dims, uint64_t first, uint64_t n, uint64_t nsub,
          uint32_t cb0)
{
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bars[16];
    __shared__ uint32_t scratch[32 * 32];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t base = (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) + 1023u) & ~1023u;
    const uint32_t bar0 = static_cast<uint32_t>(__cvta_generic_to_shared(bars));
    const uint32_t buf_bytes = rows * 128;
    if (threadIdx.x == 0) {
        for (uint32_t b = 0; b < nbuf; ++b) {
            mbar_init(bar0 + 8 * b, 32);             // full[b]
            mbar_init(bar0 + 8 * (8 + b), 1);        // empty[b]
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // lane l writes rows l + 32 s: row & 7 == l & 7, so the swizzled column
    // offset of dimension `warp` is fixed per lane
    const uint32_t col = (((warp >> 2) ^ (lane & 7u)) << 4) + (warp & 3u) * 4 - lane * 128;
    // work units (column block cb of 32 dimensions, sub-tile s), cb-major:
    // a CTA's contiguous range mostly stays in one column block
    const uint64_t units = nsub * ncb;
    const uint64_t u0 = units * blockIdx.x / gridDim.x, u1 = units * (blockIdx.x + 1) / gridDim.x;
    const bool issuer = threadIdx.x == 0;
    typename W::State st;
    w.reset(st);
    uint32_t b = 0, k = 0;
    // column blocks cb0 .. cb0 + ncb - 1 (the ones before cb0 went to the
    // level-table fill)
    uint32_t cb = static_cast<uint32_t>(u0 / nsub);
    uint64_t s = u0 - static_cast<uint64_t>(cb) * nsub;
    cb += cb0;
    for (uint64_t u = u0; u < u1; ++u, ++s) {
        if (s == nsub) { // next column block: other dimensions, fresh walk
            s = 0;
            ++cb;
            w.reset(st);
        }
        const uint64_t p0 = s * rows;
        const uint32_t cnt = static_cast<uint32_t>(n - p0 < rows ? n - p0 : rows);
        const uint32_t buf = base + b * buf_bytes;
        if (k > 0)
            mbar_wait(bar0 + 8 * (8 + b), (k - 1) & 1u);
        // the last column block may be partial (dims % 32 != 0): its
        // missing dimensions are not walked, and the tensor store clips them
        if (cb * 32 + warp < dims)
            w.run(cb * 32 + warp, first + p0, cnt, lane, buf + lane * 128 + col, 32, st,
                  scratch + warp * 32);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0)
            mbar_arrive(bar0 + 8 * b);
        if (issuer) {
            mbar_wait(bar0 + 8 * b, k & 1u);
            for (uint32_t r = 0; r < cnt; r += 256) {
                const int32_t y = static_cast<int32_t>(p0 + r);
                asm volatile(
                    "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                        reinterpret_cast<uint64_t>(&tmap)),
                    "r"(buf + r * 128), "r"(cb * 32), "r"(y)
                    : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            // the previous sub-tile's store has read its buffer: release it
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            if (u > u0)
                mbar_arrive(bar0 + 8 * (8 + (b == 0 ? nbuf - 1 : b - 1)));
        }
        __syncwarp();
        if (++b == nbuf) {
            b = 0;
            ++k;
        }
    }
    if (issuer)
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------------------
// Halton fill from on-chip level tables (dims % 32 == 0).
//
// The index i (mod prime_max_power) of a base-b dimension is split as
// i = (H * G1 + l1) * G0 + l0 with G0 = b^d0 >= 32 and G1 = b^d1 <= G0
// (lv_groups). With q0[l] = radical_inverse_fixed(l) for l < G0 (a
// d0-digit reversal over G0) and W1 = radical_inverse_fixed(H * G1 + l1)
// (the fixed-point inverse of the high part i / G0), the inverse of i is
// exactly
//     q0[l0] + floor(W1 / G0) + (r0 >= G0 - W1 mod G0),
// r0 = -q0[l0] * G0 mod 2^32 (q0's dropped remainder, < G0): i's low d0
// digits land on top of the reversal, 2^32 * RI(i) = 2^32 * T0 / G0 +
// 2^32 * RI(i / G0) / G0, and the two fractional parts add up to < 2.
// Every scramble maps digit 0 to 0 and uses one permutation for all digit
// positions (radical.cpp:130-181), so the split holds for plain, linear and
// Faure.
//
// Shared memory per dimension: the position table X[u] = {q0[u mod G0],
// 8 * floor(u / G0)} for u < G0 + kLvRows (a lane's position u relative to
// lane 0's G0-block runs past G0 within a sub-tile; the second word is the
// byte offset of its record), and per walker group a record table R[l1] =
// {floor(W1 / G0), 2^32 - (G0 - W1 mod G0)} for the G1 values of l1 of the
// current H plus the first kLvNext of the next H, rebuilt from q0 alone
// (lv_compose; the next block's inverse composes over a cached high part)
// when lane 0 enters the next H. A sample is two conflict-free shared loads (X at consecutive
// lanes, the record a broadcast), one address add, the carry add and the
// map: no table stream from L2 (the k_tma walk's bound).
//
// Layout: 32 / DPW walker warps per group (DPW = 4); warp k of a group owns
// the DPW consecutive dimensions DPW*k.. of the CTA's 32-dimension column block
// and lane l the point l of each 32-point step, so a step is one STS.128
// per lane into a sub-tile laid out as the output rows with the 128-B
// swizzle (conflict-free: 8 lanes cover the 8 swizzled chunks). GROUPS
// groups walk their own contiguous sub-tile ranges into their own rings;
// one extra warp per group issues its cp.async.bulk.tensor stores and
// releases each buffer as soon as its store has read it (a blocking
// wait_group.read stalls the whole warp, so the groups do not share one).
// One CTA per SM; a CTA stays in one column block (its tables).
__host__ __device__ inline void lv_groups(uint32_t b, uint32_t& G0, uint32_t& G1)
{
    G0 = b;
    while (G0 < 32)
        G0 *= b;
    G1 = b;
    while (G1 * b <= G0 && G0 * G1 < 1024)
        G1 *= b;
}

struct LvDim {
    uint32_t G0, G1, G0G1, hmod; // hmod = prime_max_power / (G0 * G1)
    uint32_t xoff, recoff;       // words: X in the table area, R in a group's area
    Div32 dG0, dG1;
};

constexpr uint32_t kLvMaxBufs = 4;
constexpr uint32_t kLvRows = 128; // points per sub-tile (4 warp steps)
// records of the next H: a lane's record index runs up to l1 + (G0 - 1 +
// 31 + 96) / G0 <= l1 + 4 within a sub-tile (G0 >= 32)
constexpr uint32_t kLvNext = 5;

__host__ __device__ inline uint32_t lv_xwords(uint32_t G0) { return 2 * (G0 + kLvRows); }
__host__ __device__ inline uint32_t lv_rwords(uint32_t G1) { return 2 * (G1 + kLvNext); }

__device__ __forceinline__ uint32_t lds32(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ uint2 lds64(uint32_t a)
{
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}

// Non-volatile shared load for tables that do not change while they are
// read (the walk's X and record loads between rebuilds): the scheduler may
// hoist the next step's loads above this step's math and store.
__device__ __forceinline__ uint2 lds64_ro(uint32_t a)
{
    uint2 v;
    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}

__device__ __forceinline__ void sts64(uint32_t a, uint32_t x, uint32_t y)
{
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y));
}

__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w)
{
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z),
                 "r"(w));
}

// radical_inverse_fixed(h * G + l) from Wc = radical_inverse_fixed(h), for
// l < G <= G0 (X at shared address xa)
__device__ __forceinline__ uint32_t lv_compose(uint32_t xa, uint32_t G, const Div32& dG,
                                               uint32_t l, uint32_t Wc)
{
    const uint32_t q = lds32(xa + 8 * l);
    const uint32_t r = q * (0u - G);
    const uint32_t t = div32(Wc, dG);
    return q + t + (r >= G - (Wc - t * G) ? 1u : 0u);
}

// Records of block H (l1 < G1) and of the first kLvNext values of l1 of the
// block after it; W2 = radical_inverse_fixed(H), W2n = that of the next
// block. Warp-collective.
__device__ __forceinline__ void lv_fill_records(const LvDim& D, uint32_t xa, uint32_t reca,
                                                uint32_t W2, uint32_t W2n, uint32_t lane)
{
    __syncwarp();
    for (uint32_t l = lane; l < D.G1 + kLvNext; l += 32) {
        const uint32_t W1 = l < D.G1 ? lv_compose(xa, D.G1, D.dG1, l, W2)
                                     : lv_compose(xa, D.G1, D.dG1, l - D.G1, W2n);
        const uint32_t qU = div32(W1, D.dG0);
        sts64(reca + 8 * l, qU, 0u - (D.G0 - (W1 - qU * D.G0)));
    }
    __syncwarp();
}

// Walk state of a dimension that is not touched per sub-tile: the current
// block H and radical_inverse_fixed of the next block (the next rebuild's W2).
struct LvSlot {
    // p0: lane 0's position in the block at the last check; W3 =
    // radical_inverse_fixed(Hn / G0), Hn the next block
    uint32_t H, W2n, p0, W3;
};

// Walk state in registers: a0 = X address of the lane's position, a1 = the
// record address of lane 0's l1 (warp-uniform), p0 = lane 0's position in
// its G0 * G1 block (warp-uniform).
struct LvWalk {
    uint32_t a0, a1, p0;
};

__device__ __noinline__ uint32_t lv_radical(uint32_t i, const RadicalDim& R)
{
    return radical_fixed(i, R);
}

// Start a walk at i0 (lane 0's index).
__device__ __forceinline__ LvWalk lv_init(const LvDim& D, const RadicalDim& R, uint32_t xa,
                                          uint32_t reca, LvSlot* slot, uint32_t i0, uint32_t lane)
{
    const uint32_t ir = i0 - div32(i0, R.divmp) * R.maxpow;
    const uint32_t H = ir / D.G0G1, pos = ir - H * D.G0G1;
    const uint32_t l1 = pos / D.G0;
    const LvWalk w{xa + 8 * (pos - l1 * D.G0 + lane), reca + 8 * l1, pos};
    const uint32_t Hn = H + 1 == D.hmod ? 0u : H + 1;
    const uint32_t W2 = radical_fixed(H, R), W2n = radical_fixed(Hn, R);
    lv_fill_records(D, xa, reca, W2, W2n, lane);
    if (lane == 0)
        *slot = LvSlot{H, W2n, 0u, radical_fixed(Hn / D.G0, R)};
    __syncwarp();
    return w;
}

// radical_inverse_fixed(h) for h < prime_max_power from the shared q0 table
// alone (no global loads): h's base-G0 groups, most significant first,
// composed with lv_compose.
__device__ __forceinline__ uint32_t lv_radical_q0(uint32_t h, const LvDim& D, uint32_t xa)
{
    uint32_t grp[6], m = 0; // G0 >= 32 and h < 2^32: at most 7 groups, the top one < 4
    while (h >= D.G0 && m < 6) {
        const uint32_t q = div32(h, D.dG0);
        grp[m++] = h - q * D.G0;
        h = q;
    }
    uint32_t W = lds32(xa + 8 * h); // q0[h], h < G0 (m < 6 always holds: G0^6 >= 2^30 * 32)
    while (m > 0)
        W = lv_compose(xa, D.G0, D.dG0, grp[--m], W);
    return W;
}

// Lane 0 entered block H + 1: rebuild the records; the record address moves
// back by G1 entries (the returned byte count).
__device__ __forceinline__ uint32_t lv_next_block(const LvDim& D, uint32_t xa, uint32_t reca,
                                                  LvSlot* slot, uint32_t lane)
{
    const LvSlot s = *slot;
    const uint32_t H = s.H + 1 == D.hmod ? 0u : s.H + 1;
    const uint32_t Hn = H + 1 == D.hmod ? 0u : H + 1;
    // radical_inverse_fixed(Hn) = compose of Hn mod G0 over that of Hn / G0
    // (cached; it changes once per G0 blocks)
    const uint32_t hq = div32(Hn, D.dG0), m = Hn - hq * D.G0;
    const uint32_t W3 = Hn == 0 ? 0u : (m == 0 ? lv_radical_q0(hq, D, xa) : s.W3);
    const uint32_t W2n = lv_compose(xa, D.G0, D.dG0, m, W3);
    lv_fill_records(D, xa, reca, s.W2n, W2n, lane);
    if (lane == 0)
        *slot = LvSlot{H, W2n, 0u, W3};
    __syncwarp();
    return 8 * D.G1;
}

template <bool U32OUT, int GROUPS, int DPW>
__global__ void __launch_bounds__(GROUPS * (32 / DPW + 1) * 32, 1)
    k_halton_lv(const __grid_constant__ CUtensorMap tmap, const RadicalDim* __restrict__ rd,
                uint32_t nbuf, uint32_t ctas_per_cb, uint32_t xw, uint32_t recw, uint64_t first,
                uint64_t n, uint64_t nsub)
{
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bars[2 * GROUPS * kLvMaxBufs];
    __shared__ LvDim desc[32];
    __shared__ LvSlot slots[GROUPS * 32];
    constexpr uint32_t WPG = 32 / DPW; // walker warps per group
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
    const uint32_t base = (raw + 1023u) & ~1023u;
    const uint32_t ring_bytes = GROUPS * nbuf * kLvRows * 128;
    const uint32_t xs = base + ring_bytes;
    const uint32_t recs = xs + xw * 4;
    uint32_t* xg = reinterpret_cast<uint32_t*>(smem_raw + (xs - raw));
    const uint32_t full0 = static_cast<uint32_t>(__cvta_generic_to_shared(bars));
    const uint32_t empty0 = full0 + 8 * GROUPS * kLvMaxBufs;
    const uint32_t cb = blockIdx.x / ctas_per_cb, cta = blockIdx.x - cb * ctas_per_cb;
    const RadicalDim* rdb = rd + cb * 32;
    if (warp == 0) {
        const RadicalDim& R = rdb[lane];
        uint32_t G0, G1;
        lv_groups(R.base, G0, G1);
        uint32_t a = lv_xwords(G0), c = lv_rwords(G1); // inclusive prefix sums over the lanes
        for (uint32_t o = 1; o < 32; o <<= 1) {
            const uint32_t ya = __shfl_up_sync(~0u, a, o), yc = __shfl_up_sync(~0u, c, o);
            if (lane >= o) {
                a += ya;
                c += yc;
            }
        }
        desc[lane] = LvDim{G0, G1, G0 * G1, R.maxpow / (G0 * G1), a - lv_xwords(G0),
                           c - lv_rwords(G1), make_div32(G0), make_div32(G1)};
    }
    if (threadIdx.x == 32) {
        for (uint32_t b = 0; b < GROUPS * kLvMaxBufs; ++b) {
            mbar_init(full0 + 8 * b, WPG);
            mbar_init(empty0 + 8 * b, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    for (uint32_t j = 0; j < 32; ++j) { // X[u] = {q0[u mod G0], 8 * (u / G0)}
        const uint32_t G0 = desc[j].G0, off = desc[j].xoff;
        for (uint32_t u = threadIdx.x; u < G0 + kLvRows; u += blockDim.x) {
            const uint32_t k = u / G0;
            xg[off + 2 * u] = lv_radical(u - k * G0, rdb[j]);
            xg[off + 2 * u + 1] = 8 * k;
        }
    }
    __syncthreads();
    const uint64_t s_beg = nsub * cta / ctas_per_cb, s_end = nsub * (cta + 1) / ctas_per_cb;
    if (warp >= GROUPS * WPG) { // warp WPG * GROUPS + g: lane 0 issues and releases group g's ring
        if (lane != 0)
            return;
        const uint32_t g = warp - GROUPS * WPG;
        const uint64_t gb = s_beg + (s_end - s_beg) * g / GROUPS;
        const uint64_t ge = s_beg + (s_end - s_beg) * (g + 1) / GROUPS;
        uint32_t b = 0, ph = 0;
        for (uint64_t s = gb; s < ge; ++s) {
            mbar_wait(full0 + 8 * (g * kLvMaxBufs + b), ph);
            const uint32_t buf = base + (g * nbuf + b) * kLvRows * 128;
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                             reinterpret_cast<uint64_t>(&tmap)),
                         "r"(buf), "r"(cb * 32), "r"(static_cast<int32_t>(s * kLvRows))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            // release the buffer as soon as the store has read it
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            mbar_arrive(empty0 + 8 * (g * kLvMaxBufs + b));
            if (++b == nbuf) {
                b = 0;
                ph ^= 1u;
            }
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        return;
    }
    const uint32_t g = warp / WPG, k = warp % WPG;
    const uint64_t gb = s_beg + (s_end - s_beg) * g / GROUPS;
    const uint64_t ge = s_beg + (s_end - s_beg) * (g + 1) / GROUPS;
    const uint32_t reca0 = recs + g * recw * 4;
    // row l of a sub-tile: row & 7 == lane & 7, so the swizzled 16-B chunk c
    // (dimensions 4c..4c+3; the warp's are DPW / 4 * k + cc) is fixed per lane
    const uint32_t stoff = lane * 128 + (((DPW / 4 * k) ^ (lane & 7u)) << 4);
    // lane 0's X entry one sub-tile ahead, relative to this lane's address
    const uint32_t ahead = 8 * kLvRows + 4 - 8 * lane;
    uint32_t a0[DPW], a1[DPW], ng[DPW];
    uint32_t nref = 0;  // sub-tiles until the first record rebuild of the 4 dims
    uint32_t since = 0; // sub-tiles since slots[].p0 was written
    bool live = false;
    uint32_t b = 0, ph = 0; // ring slot and the parity of its uses
    const uint32_t buf0 = base + g * nbuf * kLvRows * 128 + stoff;
    uint32_t buf = buf0;
    uint32_t i0 = static_cast<uint32_t>(first + gb * kLvRows);
    const uint32_t cnt = static_cast<uint32_t>(ge - gb);
    for (uint32_t u = 0; u < cnt; ++u, i0 += kLvRows) {
        if (u >= nbuf)
            mbar_wait(empty0 + 8 * (g * kLvMaxBufs + b), ph ^ 1u);
        if (i0 > 0xffffffffu - (kLvRows - 1)) { // the sub-tile crosses the u32 index wrap
            for (uint32_t st = 0; st < kLvRows; st += 32) {
                uint32_t v[DPW];
#pragma unroll
                for (int d = 0; d < DPW; ++d) {
                    const uint32_t x = lv_radical(i0 + st + lane, rdb[DPW * k + d]);
                    v[d] = U32OUT ? x : map_bits(x);
                }
#pragma unroll
                for (int cc = 0; cc < DPW / 4; ++cc)
                    sts128((buf ^ (cc << 4)) + st * 128, v[4 * cc], v[4 * cc + 1], v[4 * cc + 2],
                           v[4 * cc + 3]);
            }
            live = false;
        } else {
            if (!live || nref == 0) {
                nref = 0xffffffffu;
#pragma unroll
                for (int d = 0; d < DPW; ++d) {
                    const uint32_t j = DPW * k + d;
                    const LvDim& D = desc[j];
                    LvSlot* sl = &slots[g * 32 + j];
                    uint32_t p0;
                    if (!live) {
                        const LvWalk w =
                            lv_init(D, rdb[j], xs + 4 * D.xoff, reca0 + 4 * D.recoff, sl, i0, lane);
                        a0[d] = w.a0;
                        a1[d] = w.a1;
                        p0 = w.p0;
                        ng[d] = 0u - D.G0;
                    } else {
                        p0 = sl->p0 + since * kLvRows;
                        if (p0 >= D.G0G1) { // lane 0 is in the next block
                            p0 -= D.G0G1;
                            a1[d] -= lv_next_block(D, xs + 4 * D.xoff, reca0 + 4 * D.recoff, sl,
                                                   lane);
                        }
                    }
                    __syncwarp();
                    if (lane == 0)
                        sl->p0 = p0;
                    nref = min(nref, (D.G0G1 - p0 + kLvRows - 1) / kLvRows);
                }
                __syncwarp();
                since = 0;
                live = true;
            }
            // software-pipelined: step st + 1's table loads are issued before
            // step st's math and store (ptxas does not move shared loads above
            // the sub-tile stores, which it cannot tell apart from the tables)
            uint2 e[DPW], rc[DPW];
#pragma unroll
            for (int d = 0; d < DPW; ++d)
                e[d] = lds64_ro(a0[d]);
#pragma unroll
            for (int d = 0; d < DPW; ++d)
                rc[d] = lds64_ro(a1[d] + e[d].y);
#pragma unroll
            for (uint32_t st = 0; st < kLvRows / 32; ++st) {
                uint2 en[DPW], rn[DPW];
                if (st + 1 < kLvRows / 32) {
#pragma unroll
                    for (int d = 0; d < DPW; ++d)
                        en[d] = lds64_ro(a0[d] + 256 * (st + 1));
#pragma unroll
                    for (int d = 0; d < DPW; ++d)
                        rn[d] = lds64_ro(a1[d] + en[d].y);
                }
                uint32_t v[DPW];
#pragma unroll
                for (int d = 0; d < DPW; ++d) {
                    // q + qU + (r0 >= thr): the carry of r0 + (2^32 - thr)
                    uint32_t x, dummy;
                    asm("{\n\t"
                        "add.cc.u32 %1, %2, %3;\n\t"
                        "addc.u32 %0, %4, %5;\n\t}"
                        : "=r"(x), "=r"(dummy)
                        : "r"(e[d].x * ng[d]), "r"(rc[d].y), "r"(e[d].x), "r"(rc[d].x));
                    v[d] = U32OUT ? x : map_bits(x);
                }
#pragma unroll
                for (int cc = 0; cc < DPW / 4; ++cc)
                    sts128((buf ^ (cc << 4)) + st * 4096, v[4 * cc], v[4 * cc + 1], v[4 * cc + 2],
                           v[4 * cc + 3]);
                if (st + 1 < kLvRows / 32) {
#pragma unroll
                    for (int d = 0; d < DPW; ++d) {
                        e[d] = en[d];
                        rc[d] = rn[d];
                    }
                }
            }
            // next sub-tile: lane 0's position advances by kLvRows; fold the
            // G0-blocks it passed (k8 / 8 of them) into the record address
#pragma unroll
            for (int d = 0; d < DPW; ++d) {
                const uint32_t k8 = lds32(a0[d] + ahead);
                a0[d] += 8 * kLvRows;
                a0[d] += k8 * ng[d];
                a1[d] += k8;
            }
            --nref;
            ++since;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0)
            mbar_arrive(full0 + 8 * (g * kLvMaxBufs + b));
        buf += kLvRows * 128;
        if (++b == nbuf) {
            b = 0;
            ph ^= 1u;
            buf = buf0;
        }
    }
}

// Odd dims <= 31: the padded sub-tile of k_runs has an odd row stride, so
// with no padding at all (ld == dims) it is already conflict-free and laid
// out exactly as the output — so each run keeps a ring of nbuf dense
// sub-tiles and one bulk copy (cp.async.bulk, 16-B multiple; the < 16-B
// tail by plain stores) writes a sub-tile while the warps walk the next.
// Per run r: full[b] (count dims: every warp wrote sub-tile b), empty[b]
// (count 1: the copy has read it), signalled by warp 0 lane 0 of the run.
template <class W>
__global__ void __launch_bounds__(1024, 1)
    k_bulk(const __grid_constant__ W w, uint32_t dims, uint32_t runs, uint32_t rows,
           uint32_t nbuf, uint64_t first, uint64_t n, uint64_t nsub, uint32_t* __restrict__ out)
{
    extern __shared__ __align__(128) uint32_t ring[];
    __shared__ __align__(8) uint64_t bars[32][8];
    __shared__ uint32_t scratch[32 * 32];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t run = warp / dims, j = warp - run * dims;
    const uint32_t buf_words = rows * dims;
    const uint32_t ring0 = static_cast<uint32_t>(__cvta_generic_to_shared(ring)) +
                           run * nbuf * buf_words * 4;
    const uint32_t bar0 = static_cast<uint32_t>(__cvta_generic_to_shared(bars[run]));
    const bool issuer = j == 0 && lane == 0;
    if (issuer) {
        for (uint32_t b = 0; b < nbuf; ++b) {
            mbar_init(bar0 + 8 * b, dims);    // full[b]
            mbar_init(bar0 + 8 * (4 + b), 1); // empty[b]
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t s0 = nsub * blockIdx.x / gridDim.x, s1 = nsub * (blockIdx.x + 1) / gridDim.x;
    const uint64_t q = (s1 - s0 + runs - 1) / runs;
    const uint64_t r0 = s0 + run * q, r1 = min(s1, r0 + q);
    typename W::State st;
    w.reset(st);
    uint32_t b = 0, k = 0;
    for (uint64_t s = r0; s < r1; ++s) {
        const uint64_t p0 = s * rows;
        const uint32_t cnt = static_cast<uint32_t>(n - p0 < rows ? n - p0 : rows);
        const uint32_t buf = ring0 + b * buf_words * 4;
        if (k > 0)
            mbar_wait(bar0 + 8 * (4 + b), (k - 1) & 1u);
        w.run(j, first + p0, cnt, lane, buf + j * 4, dims, st, scratch + warp * 32);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0)
            mbar_arrive(bar0 + 8 * b);
        if (issuer) {
            mbar_wait(bar0 + 8 * b, k & 1u);
            const uint32_t words = cnt * dims, w16 = words & ~3u;
            uint32_t* o = out + p0 * dims;
            if (w16)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(o),
                             "r"(buf), "r"(w16 * 4)
                             : "memory");
            for (uint32_t e = w16; e < words; ++e) {
                uint32_t v;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(buf + e * 4));
                o[e] = v;
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            if (s > r0)
                mbar_arrive(bar0 + 8 * (4 + (b == 0 ? nbuf - 1 : b - 1)));
        }
        __syncwarp();
        if (++b == nbuf) {
            b = 0;
            ++k;
        }
    }
    if (issuer)
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------- launching

// Lets `kernel` launch with any dynamic shared memory size the device allows
// (the opt-in maximum less the kernel's static shared memory). The attribute
// is per function and process-wide, so it is set to one fixed value: setting
// it to each call's own size raced between host threads launching the same
// kernel with different sizes (one thread's smaller setting made another's
// launch fail with invalid argument).
template <typename K>
cudaError_t allow_dynamic_smem(K kernel)
{
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess)
        return e;
    cudaFuncAttributes fa{};
    e = cudaFuncGetAttributes(&fa, kernel);
    if (e != cudaSuccess)
        return e;
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                optin - static_cast<int>(fa.sharedSizeBytes));
}

template <typename K>
int blocks_per_sm(K kernel)
{
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kBlock, 0) != cudaSuccess || b < 1)
        b = 1;
    return b;
}

// Tiled launch for the fast paths: tiles of (32 << LOG_PPS) points aligned
// to the absolute index, contiguous tiles per warp, one wave of CTAs sized
// from the occupancy of the kernel (a multiple of the SM count).
template <typename K>
cudaError_t launch_tiled(K kernel, int log_tp, const FillRange& r, cudaStream_t s,
                         const uint32_t* a, const SmallArgs& b)
{
    const uint64_t tile0 = r.first >> log_tp;
    const uint64_t tile1 = (r.first + r.n + (1ull << log_tp) - 1) >> log_tp;
    const uint64_t ntiles = tile1 - tile0;
    const uint64_t max_warps =
        static_cast<uint64_t>(sm_count()) * blocks_per_sm(kernel) * (kBlock / 32);
    const uint64_t warps = ntiles < max_warps ? ntiles : max_warps;
    const uint64_t per_warp = (ntiles + warps - 1) / warps;
    const uint64_t used_warps = (ntiles + per_warp - 1) / per_warp;
    const unsigned grid = static_cast<unsigned>((used_warps * 32 + kBlock - 1) / kBlock);
    kernel<<<grid, kBlock, 0, s>>>(a, b, r.first, r.n, tile0, ntiles, per_warp,
                                   static_cast<uint32_t*>(r.out));
    return cudaGetLastError();
}

// Element-chunked launch for the generic paths (chunk elements < 2^31).
template <typename F>
cudaError_t launch_chunked(uint32_t dims, const FillRange& r, F&& f)
{
    const uint64_t max_pts = (1ull << 30) / dims;
    for (uint64_t done = 0; done < r.n; done += max_pts) {
        const uint64_t pts = r.n - done < max_pts ? r.n - done : max_pts;
        const uint32_t elems = static_cast<uint32_t>(pts * dims);
        const unsigned grid =
            static_cast<unsigned>(std::min<uint64_t>((elems + kBlock - 1) / kBlock,
                                                     static_cast<uint64_t>(sm_count()) * 16));
        f(grid, r.first + done, elems, static_cast<uint32_t*>(r.out) + done * dims);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess)
            return e;
    }
    return cudaSuccess;
}

// Fast-path lane width for `dims`: 8 dims per lane (256-bit stores) when
// dims is a multiple of 8 dividing 256 and the output is 32-B aligned; 4
// dims per lane (128-bit stores) when dims divides 128 and the output is
// 16-B aligned; 0 = generic path. The issue-bound Owen kernel keeps 4 dims
// per lane: at 8 its 128 registers halve occupancy (measured 4.3 vs 4.9
// TB/s), while the HBM-bound kernels gain ~1.5 % from 256-bit stores.
int fast_dpl(uint32_t dims, const FillRange& r, bool issue_bound = false)
{
    const uintptr_t a = reinterpret_cast<uintptr_t>(r.out);
    if (!issue_bound && dims >= 8 && dims <= 256 && (256 % dims) == 0 && (a & 31u) == 0)
        return 8;
    if (dims >= 4 && dims <= 128 && (128 % dims) == 0 && (a & 15u) == 0)
        return 4;
    return 0;
}

int log2u(uint32_t v)
{
    int l = 0;
    while ((1u << l) < v)
        ++l;
    return l;
}

template <int DPL, int LOG_PPS>
cudaError_t sobol_fast_dispatch(const uint32_t* colsT, const SmallArgs& words, int mode,
                                bool u32, const FillRange& r, cudaStream_t s)
{
    constexpr int LOG_TP = LOG_PPS + 5;
    if (mode == 2)
        return u32 ? launch_tiled(k_sobol_fast<DPL, LOG_PPS, 2, true>, LOG_TP, r, s, colsT, words)
                   : launch_tiled(k_sobol_fast<DPL, LOG_PPS, 2, false>, LOG_TP, r, s, colsT, words);
    return u32 ? launch_tiled(k_sobol_fast<DPL, LOG_PPS, 0, true>, LOG_TP, r, s, colsT, words)
               : launch_tiled(k_sobol_fast<DPL, LOG_PPS, 0, false>, LOG_TP, r, s, colsT, words);
}

template <int DPL, int LOG_PPS>
cudaError_t lattice_fast_dispatch(const SmallArgs& args, bool u32, const FillRange& r,
                                  cudaStream_t s)
{
    constexpr int LOG_TP = LOG_PPS + 5;
    return u32 ? launch_tiled(k_lattice_fast<DPL, LOG_PPS, true>, LOG_TP, r, s, nullptr, args)
               : launch_tiled(k_lattice_fast<DPL, LOG_PPS, false>, LOG_TP, r, s, nullptr, args);
}

// dims -> LOG_PPS = log2(32 * DPL / dims) dispatch for both fast kernels.
template <int DPL, typename F>
cudaError_t by_log_pps(uint32_t dims, F&& f)
{
    switch (log2u(32 * DPL / dims)) {
    case 0: return f(std::integral_constant<int, 0>{});
    case 1: return f(std::integral_constant<int, 1>{});
    case 2: return f(std::integral_constant<int, 2>{});
    case 3: return f(std::integral_constant<int, 3>{});
    case 4: return f(std::integral_constant<int, 4>{});
    case 5: return f(std::integral_constant<int, 5>{});
    }
    return cudaErrorInvalidValue;
}

// Write-only streaming probes: the ceiling pure store streams reach on this
// GPU (diagnostic for the roofline denominator, not part of any fill).
// mode 0: st.global.cs.v4 grid-stride; 1: st.global.v4 (write-back) grid-
// stride; 2: st.global.cs.v8 (256-bit) grid-stride; 3: st.global.cs.v4,
// contiguous chunk per warp (the fills' pattern).
template <int MODE>
__global__ void __launch_bounds__(kBlock) k_write_probe(uint4* __restrict__ out, uint64_t n16)
{
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint4 v = make_uint4(blockIdx.x, threadIdx.x, 0x3f000000u, 0u);
    if (MODE == 0) {
        for (uint64_t k = tid; k < n16; k += stride)
            __stcs(out + k, v);
    } else if (MODE == 1) {
        for (uint64_t k = tid; k < n16; k += stride)
            out[k] = v;
    } else if (MODE == 2) {
        const uint64_t n32 = n16 / 2;
        for (uint64_t k = tid; k < n32; k += stride) {
            uint4* p = out + 2 * k;
            asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                         "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(v.x), "r"(v.y), "r"(v.z),
                         "r"(v.w)
                         : "memory");
        }
    } else {
        const uint64_t warps = stride / 32, warp = tid / 32, lane = tid % 32;
        const uint64_t per = (n16 / 32 + warps - 1) / warps * 32;
        const uint64_t lo = warp * per, hi = lo + per < n16 ? lo + per : n16;
        for (uint64_t k = lo + lane; k < hi; k += 32)
            __stcs(out + k, v);
    }
}

// mode 5: TMA bulk stores — each warp fills a 2 KB shared-memory buffer
// (double-buffered) and one lane issues cp.async.bulk shared->global.
__global__ void __launch_bounds__(kBlock) k_write_probe_tma(uint4* __restrict__ out, uint64_t n16)
{
    __shared__ __align__(128) uint4 buf[kBlock / 32][2][128]; // 2 x 2 KB per warp
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    const uint64_t chunks = n16 / 128; // 2 KB chunks
    uint32_t k = 0;
    for (uint64_t c = gw; c < chunks; c += nw, k ^= 1u) {
        if (lane == 0)
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
        uint4* b = buf[warp][k];
        for (int e = lane; e < 128; e += 32)
            b[e] = make_uint4(static_cast<uint32_t>(c), e, 0x3f000000u, lane);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(b));
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 2048;" ::"l"(out + c * 128),
                         "r"(src)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (lane == 0)
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

} // namespace

cudaError_t launch_write_probe(void* out, uint64_t bytes, int mode, cudaStream_t s)
{
    const unsigned grid = static_cast<unsigned>(sm_count() * blocks_per_sm(k_write_probe<0>));
    uint4* o = static_cast<uint4*>(out);
    switch (mode) {
    case 1: k_write_probe<1><<<grid, kBlock, 0, s>>>(o, bytes / 16); break;
    case 2: k_write_probe<2><<<grid, kBlock, 0, s>>>(o, bytes / 16); break;
    case 3: k_write_probe<3><<<grid, kBlock, 0, s>>>(o, bytes / 16); break;
    case 4: return cudaMemsetAsync(out, 0, bytes, s);
    case 5:
        k_write_probe_tma<<<static_cast<unsigned>(sm_count() * 4), kBlock, 0, s>>>(o, bytes / 16);
        break;
    default: k_write_probe<0><<<grid, kBlock, 0, s>>>(o, bytes / 16); break;
    }
    return cudaGetLastError();
}

int sm_count()
{
    static thread_local int dev_cached = -1, sms = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != dev_cached) {
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        dev_cached = dev;
    }
    return sms > 0 ? sms : 148;
}

cudaError_t launch_map(const uint32_t* in, float* out, uint64_t n, cudaStream_t s)
{
    if (n == 0)
        return cudaSuccess;
    const unsigned grid = static_cast<unsigned>(
        std::min<uint64_t>((n + kBlock - 1) / kBlock, static_cast<uint64_t>(sm_count()) * 16));
    k_map<<<grid, kBlock, 0, s>>>(in, out, n);
    return cudaGetLastError();
}

cudaError_t launch_map_selfcheck(unsigned long long* count, cudaStream_t s)
{
    k_map_selfcheck<<<sm_count() * 8, kBlock, 0, s>>>(count);
    return cudaGetLastError();
}

// One-dimension-per-warp fills (k_tma / k_runs) over a column walker W.
// TMA: dims % 32 == 0, out 16-B aligned, n < 2^31; returns false otherwise.
template <class W>
bool launch_tma_fill(const W& w, uint32_t dims, const FillRange& r, cudaStream_t s,
                     cudaError_t* err, bool partial_blocks = false, uint32_t cb0 = 0)
{
    // partial_blocks: wide rows of whole 16-B units (dims > 256, dims % 4 ==
    // 0) also go here, the last 32-dim column block partial (the tensor
    // store clips it). A partial block's unit takes as long as a full one,
    // so narrower rows lose more to it than the per-dimension tiled path
    // (Halton 100 dims 0.27 -> 0.17 of the roofline, 1000 dims 0.08 -> 0.24)
    const bool shape = dims % 32 == 0 || (partial_blocks && dims > 256 && dims % 4 == 0);
    if (!shape || (reinterpret_cast<uintptr_t>(r.out) & 15u) != 0 || r.n >= (1ull << 31))
        return false;
    static PFN_cuTensorMapEncodeTiled encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
    }();
    if (!encode)
        return false;
    constexpr uint32_t kRows = 512, kBufs = 3; // 192 KB ring, 16 warp steps per sub-tile
    CUtensorMap tmap;
    const cuuint64_t gdim[2] = {dims, r.n};
    const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(dims) * 4};
    const cuuint32_t box[2] = {32, 256};
    const cuuint32_t estride[2] = {1, 1};
    if (encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, r.out, gdim, gstride, box, estride,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    const size_t smem = static_cast<size_t>(kRows) * 128 * kBufs + 1024;
    *err = allow_dynamic_smem(k_tma<W>);
    if (*err != cudaSuccess)
        return true;
    const uint64_t nsub = (r.n + kRows - 1) / kRows;
    const uint32_t ncb = (dims + 31) / 32 - cb0;
    const unsigned grid = static_cast<unsigned>(
        std::min<uint64_t>(nsub * ncb, static_cast<uint64_t>(sm_count())));
    k_tma<W><<<grid, 1024, smem, s>>>(tmap, w, kRows, kBufs, ncb, dims, r.first, r.n, nsub, cb0);
    *err = cudaGetLastError();
    return true;
}

// Halton fills with dims % 32 == 0 from on-chip level tables (k_halton_lv);
// false when the shape does not fit (the k_tma walk takes it then): out
// 16-B aligned, n < 2^31, and every column block's X tables plus the
// walker groups' record areas and rings within the opt-in shared memory.
template <bool U32OUT>
bool launch_halton_lv(const RadicalDim* rd, const RadicalDim* rd_host, uint32_t dims,
                      const FillRange& r, cudaStream_t s, cudaError_t* err, uint32_t* nblocks)
{
    if (!rd_host || dims % 32 != 0 || (reinterpret_cast<uintptr_t>(r.out) & 15u) != 0 ||
        r.n >= (1ull << 31))
        return false;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    constexpr uint32_t kRows = kLvRows;
    auto need_w = [&](int gr, uint32_t nb, uint32_t x, uint32_t rw) {
        return 1024 + static_cast<size_t>(gr) * nb * kRows * 128 + static_cast<size_t>(x) * 4 +
               static_cast<size_t>(gr) * rw * 4 + 2 * gr * kLvMaxBufs * 8 + 32 * sizeof(LvDim) +
               gr * 32 * sizeof(LvSlot);
    };
    // the leading column blocks whose tables fit (the small primes: at 32
    // dimensions the whole row; wider rows hand the rest to the k_tma walk)
    uint32_t xw = 0, recw = 0, nfit = 0;
    for (uint32_t cb = 0; cb < dims / 32; ++cb) {
        uint32_t a = 0, c = 0;
        bool ok = true;
        for (uint32_t j = 0; j < 32; ++j) {
            uint32_t G0, G1;
            lv_groups(rd_host[cb * 32 + j].base, G0, G1);
            ok = ok && rd_host[cb * 32 + j].maxpow % (G0 * G1) == 0;
            a += lv_xwords(G0);
            c += lv_rwords(G1);
        }
        const uint32_t nx = std::max(xw, a), nr = std::max(recw, c);
        if (!ok || need_w(3, 2, nx, nr) > static_cast<size_t>(optin))
            break;
        xw = nx;
        recw = nr;
        ++nfit;
    }
    if (nfit == 0)
        return false;
    // the most walker groups (latency hiding: the walk is issue / latency
    // bound), then the deepest ring, that fit: 3 groups x 2 buffers at 32
    // dimensions (measured: 2 groups x 3 buffers 1020, 3 x 2 1160 Gsamples/s)
    int kGroups = 0;
    uint32_t nbuf = 0;
    auto need = [&](int gr, uint32_t nb) { return need_w(gr, nb, xw, recw); };
    for (int gr = 3; gr >= 2 && !kGroups; --gr)
        for (uint32_t nb = 3; nb >= 2 && !kGroups; --nb)
            if (need(gr, nb) <= static_cast<size_t>(optin)) {
                kGroups = gr;
                nbuf = nb;
            }
    if (!kGroups)
        return false;
    static PFN_cuTensorMapEncodeTiled encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
    }();
    if (!encode)
        return false;
    CUtensorMap tmap;
    const cuuint64_t gdim[2] = {dims, r.n};
    const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(dims) * 4};
    const cuuint32_t box[2] = {32, kRows};
    const cuuint32_t estride[2] = {1, 1};
    if (encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, r.out, gdim, gstride, box, estride,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    // 4 dimensions per warp: 8 per warp (fewer, wider warps) measured 990 vs
    // 1154 Gsamples/s at 32 dims — the walk wants warps, not ILP
    constexpr int dpw = 4;
    auto kern = kGroups == 3 ? k_halton_lv<U32OUT, 3, dpw> : k_halton_lv<U32OUT, 2, dpw>;
    *err = allow_dynamic_smem(kern);
    if (*err != cudaSuccess)
        return true;
    const uint64_t nsub = (r.n + kRows - 1) / kRows;
    const uint32_t ncb = nfit;
    *nblocks = nfit;
    const uint32_t per = static_cast<uint32_t>(std::max<uint64_t>(
        1, std::min<uint64_t>(nsub, static_cast<uint64_t>(sm_count()) / ncb)));
    const size_t dyn = need(kGroups, nbuf) - (2 * kGroups * kLvMaxBufs * 8 + 32 * sizeof(LvDim) +
                                              kGroups * 32 * sizeof(LvSlot));
    kern<<<ncb * per, kGroups * (32 / dpw + 1) * 32, dyn, s>>>(
        tmap, rd, nbuf, per, xw, recw, r.first, r.n, nsub);
    *err = cudaGetLastError();
    return true;
}

// dims <= 32: one CTA per SM, runs x dims warps, sub-tiles sharing ~192 KB,
// plus a 32-word scratch per warp
template <class W, int DPW = 1>
cudaError_t launch_runs_fill(const W& w, uint32_t dims, const FillRange& r, cudaStream_t s)
{
    const uint32_t runs = std::min(15u, 32u * DPW / dims), ld = dims | 1u;
    constexpr uint32_t kRunsTileWords = 49152;
    uint32_t chunk = (kRunsTileWords / (runs * ld)) & ~31u;
    if (chunk < 32)
        chunk = 32;
    const size_t smem = (static_cast<size_t>(chunk) * ld * runs + runs * dims * 32) * 4;
    const cudaError_t e = allow_dynamic_smem(k_runs<W, DPW>);
    if (e != cudaSuccess)
        return e;
    const uint64_t nsub = (r.n + chunk - 1) / chunk;
    const unsigned grid =
        static_cast<unsigned>(std::min<uint64_t>(nsub, static_cast<uint64_t>(sm_count())));
    k_runs<W, DPW><<<grid, runs * dims / DPW * 32, smem, s>>>(w, dims, runs, chunk, r.first, r.n,
                                                               nsub, static_cast<uint32_t*>(r.out));
    return cudaGetLastError();
}

template <class W, int DMAX>
cudaError_t launch_runs_wide(const W& w, uint32_t dims, const FillRange& r, cudaStream_t s)
{
    const uint32_t ld = dims | 1u;
    uint32_t chunk = (49152u / ld) & ~31u;
    const size_t smem = (static_cast<size_t>(chunk) * ld + 32 * 32 * DMAX) * 4;
    const cudaError_t e = allow_dynamic_smem(k_runs_wide<W, DMAX>);
    if (e != cudaSuccess)
        return e;
    const uint64_t nsub = (r.n + chunk - 1) / chunk;
    const unsigned grid =
        static_cast<unsigned>(std::min<uint64_t>(nsub, static_cast<uint64_t>(sm_count())));
    k_runs_wide<W, DMAX><<<grid, 1024, smem, s>>>(w, dims, make_div32(dims), chunk, r.first, r.n,
                                                  nsub, static_cast<uint32_t*>(r.out));
    return cudaGetLastError();
}

// Odd dims <= 31 with out 16-B aligned: k_bulk; returns false otherwise.
template <class W>
bool launch_bulk_fill(const W& w, uint32_t dims, const FillRange& r, cudaStream_t s,
                      cudaError_t* err)
{
    if (dims > 31 || (dims & 1u) == 0 || (reinterpret_cast<uintptr_t>(r.out) & 15u) != 0)
        return false;
    // mbarriers, not named barriers, so a CTA may hold 32 one-warp runs
    const uint32_t runs = dims == 1 ? 32u : std::min(15u, 32u / dims), nbuf = 3;
    constexpr uint32_t kRingWords = 47104; // 184 KB over all runs
    uint32_t rows = (kRingWords / (runs * nbuf * dims)) & ~31u;
    if (rows < 32)
        rows = 32;
    const size_t smem = static_cast<size_t>(rows) * dims * runs * nbuf * 4;
    *err = allow_dynamic_smem(k_bulk<W>);
    if (*err != cudaSuccess)
        return true;
    const uint64_t nsub = (r.n + rows - 1) / rows;
    const unsigned grid =
        static_cast<unsigned>(std::min<uint64_t>(nsub, static_cast<uint64_t>(sm_count())));
    k_bulk<W><<<grid, runs * dims * 32, smem, s>>>(w, dims, runs, rows, nbuf, r.first, r.n, nsub,
                                                    static_cast<uint32_t*>(r.out));
    *err = cudaGetLastError();
    return true;
}

// Slab width per lane for the wide-row kernels: 8 dims (256-bit stores)
// unless 4 leaves fewer idle lanes; 0 when the rows are not 16-B multiples.
// narrow: also rows that are no multiple of 16 B (2 or 1 dims per lane).
// Their row segments start mid-sector, so L2 merges partial sectors; that
// measured 0.32-0.36 of the roofline at any width, better than the staged
// per-dimension paths only for wide Sobol' rows (255 / 1001 / 2999 dims:
// 0.13 / 0.15 / 0.05), worse at 65-127 dims (0.45 -> 0.27) and for the
// lattice (0.76 -> 0.30).
int slab_dpl(uint32_t dims, const FillRange& r, bool narrow = false)
{
    const uintptr_t a = reinterpret_cast<uintptr_t>(r.out);
    const bool ok8 = dims % 8 == 0 && (a & 31u) == 0, ok4 = dims % 4 == 0 && (a & 15u) == 0;
    if (ok8 && !(ok4 && (dims + 127) / 128 * 128 < (dims + 255) / 256 * 256))
        return 8;
    if (ok4)
        return 4;
    if (!narrow)
        return 0;
    return dims % 2 == 0 && (a & 7u) == 0 ? 2 : 1;
}

// Grid of a slab kernel: groups of nslab warps (slab_tiles), as many groups
// as the resident warps allow, each a contiguous range of 32-point tiles.
template <class K, class... A>
cudaError_t launch_slab(K kern, uint32_t dims, uint32_t slab, const FillRange& r, cudaStream_t s,
                        A... pre)
{
    const uint64_t tile0 = r.first >> 5, tile1 = (r.first + r.n + 31) >> 5;
    const uint64_t ntp = tile1 - tile0;
    const uint32_t nslab = (dims + slab - 1) / slab;
    const uint64_t max_warps =
        static_cast<uint64_t>(sm_count()) * blocks_per_sm(kern) * (kBlock / 32);
    uint64_t groups = max_warps / nslab;
    groups = groups < 1 ? 1 : (groups < ntp ? groups : ntp);
    const uint64_t per_group = (ntp + groups - 1) / groups;
    const uint64_t used = (ntp + per_group - 1) / per_group;
    const unsigned grid =
        static_cast<unsigned>((used * nslab * 32 + kBlock - 1) / kBlock);
    kern<<<grid, kBlock, 0, s>>>(pre..., dims, r.first, r.n, tile0, ntp, nslab, per_group,
                                 static_cast<uint32_t*>(r.out));
    return cudaGetLastError();
}

cudaError_t launch_sobol(const uint32_t* colsT, const uint32_t* colsT_rev, const SmallArgs& words,
                         uint32_t dims, int mode, bool u32, const FillRange& r, cudaStream_t s)
{
    if (r.n == 0)
        return cudaSuccess;
    const uint32_t* cols = mode == 2 ? colsT_rev : colsT;
    const int dpl = fast_dpl(dims, r, mode == 2);
    if (dpl == 8)
        return by_log_pps<8>(dims, [&](auto lp) {
            return sobol_fast_dispatch<8, decltype(lp)::value>(cols, words, mode, u32, r, s);
        });
    if (dpl == 4)
        return by_log_pps<4>(dims, [&](auto lp) {
            return sobol_fast_dispatch<4, decltype(lp)::value>(cols, words, mode, u32, r, s);
        });
    // the narrow kernels' interior tiles store 8 words (32 B) per lane at
    // out + (p - first) * dims with p a multiple of 8 / dims: first must be
    // too, or those stores are misaligned
    if ((dims == 1 || dims == 2) && (reinterpret_cast<uintptr_t>(r.out) & 31u) == 0 &&
        (r.first & (8u / dims - 1u)) == 0) {
        constexpr int kLogTp1 = 13, kLogTp2 = 12; // 8192 / D points per tile
        if (dims == 1)
            return mode == 2 ? (u32 ? launch_tiled(k_sobol_narrow<1, 2, true>, kLogTp1, r, s, cols, words)
                                    : launch_tiled(k_sobol_narrow<1, 2, false>, kLogTp1, r, s, cols, words))
                             : (u32 ? launch_tiled(k_sobol_narrow<1, 0, true>, kLogTp1, r, s, cols, words)
                                    : launch_tiled(k_sobol_narrow<1, 0, false>, kLogTp1, r, s, cols, words));
        return mode == 2 ? (u32 ? launch_tiled(k_sobol_narrow<2, 2, true>, kLogTp2, r, s, cols, words)
                                : launch_tiled(k_sobol_narrow<2, 2, false>, kLogTp2, r, s, cols, words))
                         : (u32 ? launch_tiled(k_sobol_narrow<2, 0, true>, kLogTp2, r, s, cols, words)
                                : launch_tiled(k_sobol_narrow<2, 0, false>, kLogTp2, r, s, cols, words));
    }
    // wide rows: slabs of 32 * DPL dims (k_sobol_slab)
    if (const int sdpl = dims > 64 ? slab_dpl(dims, r, dims > 128) : 0) {
        if (sdpl == 8)
            return mode == 2 ? (u32 ? launch_slab(k_sobol_slab<8, 2, true>, dims, 256, r, s, cols, words)
                                    : launch_slab(k_sobol_slab<8, 2, false>, dims, 256, r, s, cols, words))
                             : (u32 ? launch_slab(k_sobol_slab<8, 0, true>, dims, 256, r, s, cols, words)
                                    : launch_slab(k_sobol_slab<8, 0, false>, dims, 256, r, s, cols, words));
        if (sdpl == 4)
            return mode == 2 ? (u32 ? launch_slab(k_sobol_slab<4, 2, true>, dims, 128, r, s, cols, words)
                                    : launch_slab(k_sobol_slab<4, 2, false>, dims, 128, r, s, cols, words))
                             : (u32 ? launch_slab(k_sobol_slab<4, 0, true>, dims, 128, r, s, cols, words)
                                    : launch_slab(k_sobol_slab<4, 0, false>, dims, 128, r, s, cols, words));
        if (sdpl == 2)
            return mode == 2 ? (u32 ? launch_slab(k_sobol_slab<2, 2, true>, dims, 64, r, s, cols, words)
                                    : launch_slab(k_sobol_slab<2, 2, false>, dims, 64, r, s, cols, words))
                             : (u32 ? launch_slab(k_sobol_slab<2, 0, true>, dims, 64, r, s, cols, words)
                                    : launch_slab(k_sobol_slab<2, 0, false>, dims, 64, r, s, cols, words));
        return mode == 2 ? (u32 ? launch_slab(k_sobol_slab<1, 2, true>, dims, 32, r, s, cols, words)
                                : launch_slab(k_sobol_slab<1, 2, false>, dims, 32, r, s, cols, words))
                         : (u32 ? launch_slab(k_sobol_slab<1, 0, true>, dims, 32, r, s, cols, words)
                                : launch_slab(k_sobol_slab<1, 0, false>, dims, 32, r, s, cols, words));
    }
    // one dimension per warp (k_tma for dims % 32 == 0, else k_runs for dims
    // <= 32) from a 32-aligned index; the few points before it go through
    // the element-wise / tiled paths below
    // dimensions per warp: two for even dims 10-64 (more independent runs
    // per CTA for dims <= 32, measured +2-20 %), four for dims <= 128
    // divisible by 4
    // (-1: Owen at the other dims 33-128, k_runs_wide: +3-19 % over the
    // element-wise kernel, where plain Sobol' measured 1-13 % slower)
    const int dpw = (dims <= 8 || (dims <= 32 && dims % 2 != 0)) ? 1
                    : (dims <= 64 && dims % 2 == 0)              ? 2
                    : (dims <= 128 && dims % 4 == 0)             ? 4
                    : (dims <= 128 && mode == 2)                 ? -1
                                                                  : 0;
    if ((dpw || dims % 32 == 0) && r.n >= 64) {
        const uint64_t head = (32u - static_cast<uint32_t>(r.first & 31u)) & 31u;
        const FillRange main{r.first + head, r.n - head,
                             static_cast<uint32_t*>(r.out) + head * dims};
        const bool tma = dims % 32 == 0 && (reinterpret_cast<uintptr_t>(main.out) & 15u) == 0 &&
                         main.n < (1ull << 31);
        if (dpw || tma) {
            if (head) {
                const cudaError_t e = launch_sobol(colsT, colsT_rev, words, dims, mode, u32,
                                                   FillRange{r.first, head, r.out}, s);
                if (e != cudaSuccess)
                    return e;
            }
            auto go = [&](auto w) {
                cudaError_t err = cudaSuccess;
                if (tma && launch_tma_fill(w, dims, main, s, &err))
                    return err;
                if (dpw < 0)
                    return dims <= 64 ? launch_runs_wide<decltype(w), 2>(w, dims, main, s)
                                      : launch_runs_wide<decltype(w), 4>(w, dims, main, s);
                return dpw == 4 ? launch_runs_fill<decltype(w), 4>(w, dims, main, s)
                       : dpw == 2 ? launch_runs_fill<decltype(w), 2>(w, dims, main, s)
                                  : launch_runs_fill<decltype(w), 1>(w, dims, main, s);
            };
            if (mode == 2)
                return u32 ? go(SobolWalk<2, true>{cols, dims, words})
                           : go(SobolWalk<2, false>{cols, dims, words});
            return u32 ? go(SobolWalk<0, true>{cols, dims, words})
                       : go(SobolWalk<0, false>{cols, dims, words});
        }
    }
    if (dims <= kElemMaxDims) {
        // element-wise path: chunks of <= 1022 points (two 1024-point tiles)
        auto kern = mode == 2 ? (u32 ? k_sobol_elem<2, true> : k_sobol_elem<2, false>)
                              : (u32 ? k_sobol_elem<0, true> : k_sobol_elem<0, false>);
        const size_t smem = (static_cast<size_t>(dims + 1) * 64 + 2 * dims) * 4;
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, smem) !=
                cudaSuccess ||
            per_sm < 1)
            per_sm = 1;
        const uint32_t chunk = std::min<uint32_t>(4096u, (1022u * dims) & ~3u);
        const uint64_t total = r.n * dims;
        const uint64_t want = (total + chunk - 1) / chunk;
        const uint64_t cap = static_cast<uint64_t>(sm_count()) * per_sm;
        const unsigned grid = static_cast<unsigned>(want < cap ? want : cap);
        const uint64_t per = (((total + grid - 1) / grid) + 3) & ~3ull;
        const Div32 d = make_div32(dims);
        kern<<<grid, kBlock, smem, s>>>(cols, words, dims, d, r.first, total, per, chunk,
                                        static_cast<uint32_t*>(r.out));
        return cudaGetLastError();
    }
    // shared-memory tiled path: tp = 2^k points. dims > 128: one 1024-thread
    // CTA per SM with up to ~190 KB of tile + tables (longer runs per
    // dimension); else tp*(dims+1) <= 8192 words at several CTAs per SM
    const bool wide = dims > 128;
    const uint32_t block = wide ? 1024u : static_cast<uint32_t>(kBlock);
    auto words_for = [&](uint32_t t) {
        return static_cast<size_t>(t) * (dims + 1) + static_cast<size_t>(dims) * (t / 32 + 1);
    };
    if (words_for(32) > 56000u) { // thousands of dims: no tile fits, per-element path
        const unsigned grid = static_cast<unsigned>(sm_count()) * 8;
        const Div32 d = make_div32(dims);
        if (mode == 2)
            u32 ? k_sobol_huge<2, true><<<grid, kBlock, 0, s>>>(cols, words, dims, d, r.first, r.n,
                                                                static_cast<uint32_t*>(r.out))
                : k_sobol_huge<2, false><<<grid, kBlock, 0, s>>>(cols, words, dims, d, r.first, r.n,
                                                                 static_cast<uint32_t*>(r.out));
        else
            u32 ? k_sobol_huge<0, true><<<grid, kBlock, 0, s>>>(cols, words, dims, d, r.first, r.n,
                                                                static_cast<uint32_t*>(r.out))
                : k_sobol_huge<0, false><<<grid, kBlock, 0, s>>>(cols, words, dims, d, r.first, r.n,
                                                                 static_cast<uint32_t*>(r.out));
        return cudaGetLastError();
    }
    uint32_t tp = 32;
    if (wide) {
        while (words_for(tp * 2) <= 48000u)
            tp *= 2;
    } else {
        while (tp * 2 * (dims + 1) <= 8192u)
            tp *= 2;
    }
    const size_t smem = words_for(tp) * 4;
    auto kern = wide ? (mode == 2 ? (u32 ? k_sobol_tiled<2, true, 1024> : k_sobol_tiled<2, false, 1024>)
                                  : (u32 ? k_sobol_tiled<0, true, 1024> : k_sobol_tiled<0, false, 1024>))
                     : (mode == 2 ? (u32 ? k_sobol_tiled<2, true, kBlock> : k_sobol_tiled<2, false, kBlock>)
                                  : (u32 ? k_sobol_tiled<0, true, kBlock> : k_sobol_tiled<0, false, kBlock>));
    if (smem > 48 * 1024) {
        const cudaError_t e = allow_dynamic_smem(kern);
        if (e != cudaSuccess)
            return e;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem) != cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    const uint64_t tile0 = r.first / tp;
    const uint64_t ntiles = (r.first + r.n + tp - 1) / tp - tile0;
    const uint64_t cap = static_cast<uint64_t>(sm_count()) * per_sm;
    const unsigned grid = static_cast<unsigned>(ntiles < cap ? ntiles : cap);
    const Div32 d = dims >= 2 ? make_div32(dims) : Div32{0, 0};
    kern<<<grid, block, smem, s>>>(cols, words, dims, d, tp, r.first, r.n, tile0, ntiles,
                                   static_cast<uint32_t*>(r.out));
    return cudaGetLastError();
}

cudaError_t launch_lattice(const SmallArgs& args, uint32_t dims, bool u32, const FillRange& r,
                           cudaStream_t s)
{
    if (r.n == 0)
        return cudaSuccess;
    const int dpl = fast_dpl(dims, r);
    if (dpl == 8)
        return by_log_pps<8>(dims, [&](auto lp) {
            return lattice_fast_dispatch<8, decltype(lp)::value>(args, u32, r, s);
        });
    if (dpl == 4)
        return by_log_pps<4>(dims, [&](auto lp) {
            return lattice_fast_dispatch<4, decltype(lp)::value>(args, u32, r, s);
        });
    if ((dims == 1 || dims == 2) && (reinterpret_cast<uintptr_t>(r.out) & 31u) == 0 &&
        (r.first & (8u / dims - 1u)) == 0) { // see launch_sobol
        if (dims == 1)
            return u32 ? launch_tiled(k_lattice_narrow<1, true>, 13, r, s, nullptr, args)
                       : launch_tiled(k_lattice_narrow<1, false>, 13, r, s, nullptr, args);
        return u32 ? launch_tiled(k_lattice_narrow<2, true>, 12, r, s, nullptr, args)
                   : launch_tiled(k_lattice_narrow<2, false>, 12, r, s, nullptr, args);
    }
    if (const int sdpl = dims > 64 ? slab_dpl(dims, r) : 0) // wide rows (k_lattice_slab)
        return sdpl == 8   ? (u32 ? launch_slab(k_lattice_slab<8, true>, dims, 256, r, s, args)
                                  : launch_slab(k_lattice_slab<8, false>, dims, 256, r, s, args))
                           : (u32 ? launch_slab(k_lattice_slab<4, true>, dims, 128, r, s, args)
                                  : launch_slab(k_lattice_slab<4, false>, dims, 128, r, s, args));
    const Div32 d = dims >= 2 ? make_div32(dims) : Div32{0, 0};
    return launch_chunked(dims, r, [&](unsigned grid, uint64_t first, uint32_t elems, uint32_t* o) {
        k_lattice_generic<<<grid, kBlock, 0, s>>>(args, dims, d, first, elems, u32, o);
    });
}

cudaError_t launch_halton(const void* rd, uint32_t dims, bool u32, const FillRange& r,
                          cudaStream_t s, const void* rd_host)
{
    if (r.n == 0)
        return cudaSuccess;
    const RadicalDim* rdv = static_cast<const RadicalDim*>(rd);
    const RadicalDim* rdh = static_cast<const RadicalDim*>(rd_host);
    cudaError_t err = cudaSuccess;
    // QMC_HALTON_NO_LV=1: the k_tma walk instead (A/B, tools/exp_halton_lv.py)
    uint32_t lv_blocks = 0;
    if (std::getenv("QMC_HALTON_NO_LV") == nullptr &&
        (u32 ? launch_halton_lv<true>(rdv, rdh, dims, r, s, &err, &lv_blocks)
             : launch_halton_lv<false>(rdv, rdh, dims, r, s, &err, &lv_blocks))) {
        if (err != cudaSuccess || lv_blocks == dims / 32)
            return err;
        // the wider column blocks (larger primes) on the k_tma walk
        if (u32 ? launch_tma_fill(HaltonWalk<true>{rdv}, dims, r, s, &err, false, lv_blocks)
                : launch_tma_fill(HaltonWalk<false>{rdv}, dims, r, s, &err, false, lv_blocks))
            return err;
        return cudaErrorNotSupported;
    }
    if (u32 ? launch_tma_fill(HaltonWalk<true>{rdv}, dims, r, s, &err, true)
            : launch_tma_fill(HaltonWalk<false>{rdv}, dims, r, s, &err, true))
        return err;
    // odd dims >= 5: bulk-copy ring (the walk is the bottleneck and warp 0,
    // the issuer, walks base 2); the Sobol' walk is too cheap to spare the
    // issuer's waits, and 3 dims measured no better. dims == 1 (a single
    // radical inverse): 32 one-warp runs per CTA instead of k_runs' 15
    if ((dims >= 5 || dims == 1) && (u32 ? launch_bulk_fill(HaltonWalk<true>{rdv}, dims, r, s, &err)
                          : launch_bulk_fill(HaltonWalk<false>{rdv}, dims, r, s, &err)))
        return err;
    if (dims <= 32)
        return u32 ? launch_runs_fill(HaltonWalk<true>{rdv}, dims, r, s)
                   : launch_runs_fill(HaltonWalk<false>{rdv}, dims, r, s);
    // dims > 32 (not a multiple of 32): shared-memory walk state per
    // dimension. One CTA of 1024 threads per SM with a ~190 KB tile (minus
    // the states) makes each (tile, dimension) run 3-5x longer than 48 KB
    // tiles at 4 CTAs per SM, which pays for the per-run state load/store
    const bool wide = dims > 32;
    const uint32_t block = wide ? 1024u : static_cast<uint32_t>(kBlock);
    const size_t state_bytes =
        dims >= block / 32 ? static_cast<size_t>(dims) * sizeof(HaltonState) : 0;
    const uint32_t budget =
        wide ? static_cast<uint32_t>((196608 - std::min<size_t>(state_bytes, 98304)) / 4) : 12288u;
    uint32_t tp = (budget / (dims | 1u)) & ~31u;
    if (tp < 32)
        tp = 32;
    const size_t tile_words = (static_cast<size_t>(tp) * (dims | 1u) + 15) & ~size_t(15);
    const size_t smem = tile_words * 4 + state_bytes;
    auto kern = wide ? (u32 ? k_halton_tiled<true, 1024> : k_halton_tiled<false, 1024>)
                     : (u32 ? k_halton_tiled<true, kBlock> : k_halton_tiled<false, kBlock>);
    if (smem > 48 * 1024) {
        const cudaError_t e = allow_dynamic_smem(kern);
        if (e != cudaSuccess)
            return e;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem) != cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    const uint64_t ntiles = (r.n + tp - 1) / tp;
    const uint64_t cap = static_cast<uint64_t>(sm_count()) * per_sm;
    const unsigned grid = static_cast<unsigned>(ntiles < cap ? ntiles : cap);
    const Div32 dd = dims >= 2 ? make_div32(dims) : Div32{0, 0};
    kern<<<grid, block, smem, s>>>(static_cast<const RadicalDim*>(rd), dims, dd, tp, r.first, r.n,
                                   ntiles, static_cast<uint32_t*>(r.out));
    return cudaGetLastError();
}

cudaError_t launch_vdc(bool u32, const FillRange& r, cudaStream_t s)
{
    if (r.n == 0)
        return cudaSuccess;
    const uint64_t quads = (r.n + 3) / 4;
    const unsigned grid = static_cast<unsigned>(
        std::min<uint64_t>((quads + kBlock - 1) / kBlock, static_cast<uint64_t>(sm_count()) * 16));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kBlock);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    uint32_t* out = static_cast<uint32_t*>(r.out);
    if ((r.first & 7u) == 0 && (reinterpret_cast<uintptr_t>(out) & 31u) == 0) {
        const uint64_t octs = (r.n + 7) / 8;
        cfg.gridDim = dim3(static_cast<unsigned>(std::min<uint64_t>(
            (octs + kBlock - 1) / kBlock, static_cast<uint64_t>(sm_count()) * 8)));
        return u32 ? cudaLaunchKernelEx(&cfg, k_vdc8<true>, r.first, r.n, out)
                   : cudaLaunchKernelEx(&cfg, k_vdc8<false>, r.first, r.n, out);
    }
    return u32 ? cudaLaunchKernelEx(&cfg, k_vdc<true>, r.first, r.n, out)
               : cudaLaunchKernelEx(&cfg, k_vdc<false>, r.first, r.n, out);
}

} // namespace qmcgpu
