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
#include <cstdint>

#include "device.cuh"
#include "internal.hpp"

namespace qmcgpu {

namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ uint4 xor4(uint4 a, uint4 b)
{
    return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w);
}

__host__ __device__ constexpr uint32_t ctz_const(uint32_t v)
{
    uint32_t c = 0;
    while (!(v & 1u)) {
        v >>= 1;
        ++c;
    }
    return c;
}

__host__ __device__ constexpr uint32_t brev5(uint32_t u)
{
    return ((u & 1u) << 4) | ((u & 2u) << 2) | (u & 4u) | ((u & 8u) >> 2) | ((u & 16u) >> 4);
}

__device__ __forceinline__ uint4 map4(uint4 x)
{
    return make_uint4(map_bits(x.x), map_bits(x.y), map_bits(x.z), map_bits(x.w));
}

__device__ __forceinline__ void store4(uint4* p, uint4 v) { __stcs(p, v); }

// element e of a row-major [points][dims] chunk -> point (dims == 1 needs no
// division; div32 requires a divisor >= 2)
__device__ __forceinline__ uint32_t point_of(uint32_t e, uint32_t dims, const Div32& d)
{
    return dims == 1 ? e : div32(e, d);
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

// MODE 0: plain / XOR-scrambled (words = XOR words, folded into the start
// value since the scramble is linear). MODE 2: hash-Owen, columns and the
// running value live in the bit-reversed domain; words = per-dim seeds.
template <int LOG_PPS, int MODE, bool U32OUT>
__global__ void __launch_bounds__(kBlock)
    k_sobol_fast(const uint32_t* __restrict__ colsT, const uint32_t* __restrict__ words,
                 uint64_t first, uint64_t n, uint64_t tile0, uint64_t ntiles, uint64_t per_warp,
                 uint4* __restrict__ out)
{
    constexpr int PPS = 1 << LOG_PPS; // points per warp store
    constexpr int LPP = 32 >> LOG_PPS; // lanes per point
    constexpr int DIMS = 4 * LPP;
    constexpr int LOG_TP = LOG_PPS + 5; // 32 steps per tile
    uint64_t t, tend;
    if (!warp_tiles(tile0, ntiles, per_warp, t, tend))
        return;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t r = lane / LPP; // point within a step
    const uint32_t dq = lane % LPP; // dims 4*dq .. 4*dq+3
    const uint4* cols = reinterpret_cast<const uint4*>(colsT) + dq; // cols[k * LPP] = column k
    auto col = [&](uint32_t k) { return __ldg(cols + k * LPP); };

    // Step masks: index += PPS flips bits LOG_PPS .. LOG_PPS + ctz(u+1).
    uint4 D[5];
    {
        uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            acc = xor4(acc, col(LOG_PPS + k));
            D[k] = acc;
        }
    }
    uint4 seed = make_uint4(0, 0, 0, 0);
    uint4 xr = make_uint4(0, 0, 0, 0);
    if (words) {
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(words) + dq);
        if (MODE == 2)
            seed = w;
        else
            xr = w;
    }
#pragma unroll
    for (int k = 0; k < LOG_PPS; ++k)
        if ((r >> k) & 1u)
            xr = xor4(xr, col(k));
    // Value of the tile base t << LOG_TP (bits >= LOG_TP).
    uint4 xp = make_uint4(0, 0, 0, 0);
    for (uint64_t b = t; b; b &= b - 1)
        xp = xor4(xp, col(LOG_TP + __ffsll(static_cast<long long>(b)) - 1));

    auto emit = [&](uint4 x) -> uint4 {
        if (MODE == 2) {
            x = make_uint4(brev32(owen_lk(x.x, seed.x)), brev32(owen_lk(x.y, seed.y)),
                           brev32(owen_lk(x.z, seed.z)), brev32(owen_lk(x.w, seed.w)));
        }
        return U32OUT ? x : map4(x);
    };

    for (;;) {
        const uint64_t p0 = (t << LOG_TP) + r; // this thread's point at step 0
        uint4 x = xor4(xp, xr);
        const uint64_t lo = t << LOG_TP, hi = (t + 1) << LOG_TP;
        if (lo >= first && hi <= first + n) {
            uint4* o = out + (p0 - first) * LPP + dq;
#pragma unroll
            for (uint32_t u = 0; u < 32; ++u) {
                store4(o + u * 32, emit(x));
                if (u < 31)
                    x = xor4(x, D[ctz_const(u + 1)]);
            }
        } else {
#pragma unroll
            for (uint32_t u = 0; u < 32; ++u) {
                const uint64_t i = p0 + u * PPS;
                if (i - first < n)
                    store4(out + (i - first) * LPP + dq, emit(x));
                if (u < 31)
                    x = xor4(x, D[ctz_const(u + 1)]);
            }
        }
        if (++t >= tend)
            break;
        // tile t-1 -> t flips bits LOG_TP .. LOG_TP + ctz(t)
        const int c = __ffsll(static_cast<long long>(t)) - 1;
        for (int k = 0; k <= c; ++k)
            xp = xor4(xp, col(LOG_TP + k));
    }
    (void)DIMS;
}

// Any dims: one thread per (point, dim) element of a chunk whose element
// count fits 32 bits; direct per-set-bit evaluation (digitalnet.cpp:111-131).
template <int MODE, bool U32OUT>
__global__ void __launch_bounds__(kBlock)
    k_sobol_generic(const uint32_t* __restrict__ colsT, const uint32_t* __restrict__ words,
                    uint32_t dims, Div32 div_dims, uint64_t first, uint32_t elems,
                    uint32_t* __restrict__ out)
{
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < elems; e += stride) {
        const uint32_t p = point_of(e, dims, div_dims);
        const uint32_t j = e - p * dims;
        uint64_t i = first + p;
        uint32_t x = (MODE == 0 && words) ? __ldg(words + j) : 0u;
        for (uint32_t k = 0; i; ++k, i >>= 1)
            if (i & 1u)
                x ^= __ldg(colsT + k * dims + j);
        if (MODE == 2)
            x = brev32(owen_lk(brev32(x), words ? __ldg(words + j) : 0u));
        out[e] = U32OUT ? x : map_bits(x);
    }
}

// ---------------------------------------------------------------- lattice

// x_j(i) = brev((uint32_t)i) * g_j + s_j (mod 2^32). Inside a tile the index
// is P | (u << LOG_PPS) | r with disjoint bits, so brev(i) = brev(P | r) +
// brev5(u) << (27 - LOG_PPS): one IMAD per sample with a compile-time
// multiplier.
template <int LOG_PPS, bool U32OUT>
__global__ void __launch_bounds__(kBlock)
    k_lattice_fast(const uint32_t* __restrict__ g, const uint32_t* __restrict__ shifts,
                   uint64_t first, uint64_t n, uint64_t tile0, uint64_t ntiles, uint64_t per_warp,
                   uint4* __restrict__ out)
{
    constexpr int PPS = 1 << LOG_PPS;
    constexpr int LPP = 32 >> LOG_PPS;
    constexpr int LOG_TP = LOG_PPS + 5;
    uint64_t t, tend;
    if (!warp_tiles(tile0, ntiles, per_warp, t, tend))
        return;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t r = lane / LPP, dq = lane % LPP;
    const uint4 g4 = __ldg(reinterpret_cast<const uint4*>(g) + dq);
    const uint4 s4 = shifts ? __ldg(reinterpret_cast<const uint4*>(shifts) + dq)
                            : make_uint4(0, 0, 0, 0);
    const uint4 G = make_uint4(g4.x << (27 - LOG_PPS), g4.y << (27 - LOG_PPS),
                               g4.z << (27 - LOG_PPS), g4.w << (27 - LOG_PPS));
    for (; t < tend; ++t) {
        const uint64_t p0 = (t << LOG_TP) + r;
        const uint32_t b = brev32(static_cast<uint32_t>(p0));
        const uint4 x0 = make_uint4(b * g4.x + s4.x, b * g4.y + s4.y, b * g4.z + s4.z,
                                    b * g4.w + s4.w);
        const uint64_t lo = t << LOG_TP, hi = (t + 1) << LOG_TP;
        const bool full = lo >= first && hi <= first + n;
        uint4* o = out + (p0 - first) * LPP + dq;
#pragma unroll
        for (uint32_t u = 0; u < 32; ++u) {
            const uint32_t c = brev5(u);
            uint4 x = make_uint4(x0.x + c * G.x, x0.y + c * G.y, x0.z + c * G.z, x0.w + c * G.w);
            if (!U32OUT)
                x = map4(x);
            if (full || (p0 + u * PPS) - first < n)
                store4(o + u * 32, x);
        }
    }
}

__global__ void __launch_bounds__(kBlock)
    k_lattice_generic(const uint32_t* __restrict__ g, const uint32_t* __restrict__ shifts,
                      uint32_t dims, Div32 div_dims, uint64_t first, uint32_t elems, bool u32out,
                      uint32_t* __restrict__ out)
{
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < elems; e += stride) {
        const uint32_t p = point_of(e, dims, div_dims);
        const uint32_t j = e - p * dims;
        uint32_t x = brev32(static_cast<uint32_t>(first + p)) * __ldg(g + j);
        if (shifts)
            x += __ldg(shifts + j);
        out[e] = u32out ? x : map_bits(x);
    }
}

// ----------------------------------------------------------------- Halton

// dims == 1, base 2 (config C1: van der Corput = brev(i mod 2^31)); four
// consecutive points per thread, one 128-bit store.
template <bool U32OUT>
__global__ void __launch_bounds__(kBlock)
    k_vdc(uint64_t first, uint64_t n, uint32_t* __restrict__ out)
{
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

template <bool U32OUT>
__global__ void __launch_bounds__(kBlock)
    k_halton_generic(const RadicalDim* __restrict__ rd, uint32_t dims, Div32 div_dims,
                     uint64_t first, uint32_t elems, uint32_t* __restrict__ out)
{
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < elems; e += stride) {
        const uint32_t p = point_of(e, dims, div_dims);
        const uint32_t j = e - p * dims;
        const RadicalDim r = rd[j];
        const uint32_t x = radical_fixed(static_cast<uint32_t>(first + p), r);
        out[e] = U32OUT ? x : map_bits(x);
    }
}

// ------------------------------------------------------------- launching

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
                         const uint32_t* a, const uint32_t* b)
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
                                   static_cast<uint4*>(r.out));
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

bool fast_dims(uint32_t dims, const FillRange& r)
{
    return dims >= 4 && dims <= 128 && (128 % dims) == 0 &&
           (reinterpret_cast<uintptr_t>(r.out) & 15u) == 0;
}

int log2u(uint32_t v)
{
    int l = 0;
    while ((1u << l) < v)
        ++l;
    return l;
}

template <int LOG_PPS>
cudaError_t sobol_fast_dispatch(const uint32_t* colsT, const uint32_t* words, int mode,
                                bool u32, const FillRange& r, cudaStream_t s)
{
    constexpr int LOG_TP = LOG_PPS + 5;
    if (mode == 2)
        return u32 ? launch_tiled(k_sobol_fast<LOG_PPS, 2, true>, LOG_TP, r, s, colsT, words)
                   : launch_tiled(k_sobol_fast<LOG_PPS, 2, false>, LOG_TP, r, s, colsT, words);
    return u32 ? launch_tiled(k_sobol_fast<LOG_PPS, 0, true>, LOG_TP, r, s, colsT, words)
               : launch_tiled(k_sobol_fast<LOG_PPS, 0, false>, LOG_TP, r, s, colsT, words);
}

template <int LOG_PPS>
cudaError_t lattice_fast_dispatch(const uint32_t* g, const uint32_t* sh, bool u32,
                                  const FillRange& r, cudaStream_t s)
{
    constexpr int LOG_TP = LOG_PPS + 5;
    return u32 ? launch_tiled(k_lattice_fast<LOG_PPS, true>, LOG_TP, r, s, g, sh)
               : launch_tiled(k_lattice_fast<LOG_PPS, false>, LOG_TP, r, s, g, sh);
}

// Write-only streaming probe: the ceiling a pure 128-bit store stream reaches
// on this GPU (same grid shape and store hint as the fills). Diagnostic for
// the roofline denominator, not part of any fill.
__global__ void __launch_bounds__(kBlock) k_write_probe(uint4* __restrict__ out, uint64_t n16)
{
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint4 v = make_uint4(blockIdx.x, threadIdx.x, 0x3f000000u, 0u);
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n16;
         k += stride)
        store4(out + k, v);
}

} // namespace

cudaError_t launch_write_probe(void* out, uint64_t bytes, cudaStream_t s)
{
    const unsigned grid = static_cast<unsigned>(sm_count() * blocks_per_sm(k_write_probe));
    k_write_probe<<<grid, kBlock, 0, s>>>(static_cast<uint4*>(out), bytes / 16);
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

cudaError_t launch_sobol(const uint32_t* colsT, const uint32_t* colsT_rev, const uint32_t* words,
                         uint32_t dims, int mode, bool u32, const FillRange& r, cudaStream_t s)
{
    if (r.n == 0)
        return cudaSuccess;
    const uint32_t* cols = mode == 2 ? colsT_rev : colsT;
    if (fast_dims(dims, r)) {
        switch (log2u(128 / dims)) {
        case 0: return sobol_fast_dispatch<0>(cols, words, mode, u32, r, s);
        case 1: return sobol_fast_dispatch<1>(cols, words, mode, u32, r, s);
        case 2: return sobol_fast_dispatch<2>(cols, words, mode, u32, r, s);
        case 3: return sobol_fast_dispatch<3>(cols, words, mode, u32, r, s);
        case 4: return sobol_fast_dispatch<4>(cols, words, mode, u32, r, s);
        case 5: return sobol_fast_dispatch<5>(cols, words, mode, u32, r, s);
        }
    }
    // the generic kernel reads columns in the normal domain for both modes
    const Div32 d = dims >= 2 ? make_div32(dims) : Div32{0, 0};
    return launch_chunked(dims, r, [&](unsigned grid, uint64_t first, uint32_t elems, uint32_t* o) {
        if (mode == 2)
            u32 ? k_sobol_generic<2, true><<<grid, kBlock, 0, s>>>(colsT, words, dims, d, first, elems, o)
                : k_sobol_generic<2, false><<<grid, kBlock, 0, s>>>(colsT, words, dims, d, first, elems, o);
        else
            u32 ? k_sobol_generic<0, true><<<grid, kBlock, 0, s>>>(colsT, words, dims, d, first, elems, o)
                : k_sobol_generic<0, false><<<grid, kBlock, 0, s>>>(colsT, words, dims, d, first, elems, o);
    });
}

cudaError_t launch_lattice(const uint32_t* g, const uint32_t* shifts, uint32_t dims, bool u32,
                           const FillRange& r, cudaStream_t s)
{
    if (r.n == 0)
        return cudaSuccess;
    if (fast_dims(dims, r)) {
        switch (log2u(128 / dims)) {
        case 0: return lattice_fast_dispatch<0>(g, shifts, u32, r, s);
        case 1: return lattice_fast_dispatch<1>(g, shifts, u32, r, s);
        case 2: return lattice_fast_dispatch<2>(g, shifts, u32, r, s);
        case 3: return lattice_fast_dispatch<3>(g, shifts, u32, r, s);
        case 4: return lattice_fast_dispatch<4>(g, shifts, u32, r, s);
        case 5: return lattice_fast_dispatch<5>(g, shifts, u32, r, s);
        }
    }
    const Div32 d = dims >= 2 ? make_div32(dims) : Div32{0, 0};
    return launch_chunked(dims, r, [&](unsigned grid, uint64_t first, uint32_t elems, uint32_t* o) {
        k_lattice_generic<<<grid, kBlock, 0, s>>>(g, shifts, dims, d, first, elems, u32, o);
    });
}

cudaError_t launch_halton(const void* rd, uint32_t dims, bool u32, const FillRange& r,
                          cudaStream_t s)
{
    if (r.n == 0)
        return cudaSuccess;
    // rd[0].base == 2 is known to the caller; dims == 1 with base 2 is C1.
    const Div32 d = dims >= 2 ? make_div32(dims) : Div32{0, 0};
    return launch_chunked(dims, r, [&](unsigned grid, uint64_t first, uint32_t elems, uint32_t* o) {
        u32 ? k_halton_generic<true><<<grid, kBlock, 0, s>>>(
                  static_cast<const RadicalDim*>(rd), dims, d, first, elems, o)
            : k_halton_generic<false><<<grid, kBlock, 0, s>>>(
                  static_cast<const RadicalDim*>(rd), dims, d, first, elems, o);
    });
}

cudaError_t launch_vdc(bool u32, const FillRange& r, cudaStream_t s)
{
    if (r.n == 0)
        return cudaSuccess;
    const uint64_t quads = (r.n + 3) / 4;
    const unsigned grid = static_cast<unsigned>(
        std::min<uint64_t>((quads + kBlock - 1) / kBlock, static_cast<uint64_t>(sm_count()) * 16));
    if (u32)
        k_vdc<true><<<grid, kBlock, 0, s>>>(r.first, r.n, static_cast<uint32_t*>(r.out));
    else
        k_vdc<false><<<grid, kBlock, 0, s>>>(r.first, r.n, static_cast<uint32_t*>(r.out));
    return cudaGetLastError();
}

} // namespace qmcgpu
