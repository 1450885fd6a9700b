// kernels_integrate.cu — fused QMC integration (reference
// integrate(), quality.cpp:214-282, with builtin_integrands, :28-66).
//
// Fixed 4096-index chunks (quality.cpp:178), one CTA each: sample every
// integrand dimension at the integer stage -> bit-exact float map -> the
// integrand in FP64 with the reference's operation order (explicit _rn
// intrinsics, no FMA contraction) -> Neumaier in index order (kahan) or
// llround(v * 2^32) (int). Chunk partials are combined in chunk order on the
// host (Kahan: the reference's rank-ordered CompensatedSum,
// quality.cpp:262-267) or summed with exact 64-bit atomics (int, :268-272).
#include <cstdint>

#include "device.cuh"
#include "internal.hpp"

namespace qmcgpu {

namespace {

// Per-dimension incremental state (Sobol' register/local words, Halton
// quotient-table records) covers the first kStateDims integrand dimensions;
// dimensions beyond take the direct per-sample form (Sobol': XOR of the
// columns of the index's set bits; Halton: the digit loop), so any dims the
// stream allows integrate (quality.cpp:214-282 has no cap).
constexpr uint32_t kStateDims = 64;
// Threads per chunk CTA: 256 (16 samples per thread) for every kind but
// Sobol', whose per-thread state array (local memory) prefers 128 threads.
template <uint32_t KIND, bool SMALL = false>
struct ChunkShape {
    // Sobol' with more than kSmallDims dimensions (state in local memory): 128
    static constexpr uint32_t kLogBlock = KIND == 0 && !SMALL ? 7 : 8;
    static constexpr uint32_t kBlock = 1u << kLogBlock;
    static constexpr uint32_t kLogSteps = 12 - kLogBlock; // 4096 = block * steps
    static constexpr uint32_t kSteps = 1u << kLogSteps;
};
constexpr int kBlockMax = 256;

__device__ __forceinline__ uint32_t rad2(uint32_t i) { return brev32(i & 0x7fffffffu); }

// sobol_component_fixed (digitalnet.cpp:111-131) of dimension j at idx.
__device__ __forceinline__ uint32_t sobol_direct(uint64_t idx, uint32_t j, const IntegrateParams& p)
{
    uint32_t x = p.words ? __ldg(p.words + j) : 0u;
    for (uint32_t k = 0; idx; ++k, idx >>= 1)
        if (idx & 1u)
            x ^= __ldg(p.colsT + k * p.mdims + j);
    return x;
}

__device__ __forceinline__ uint64_t digit_reverse3(uint64_t v, uint32_t digits)
{
    uint64_t r = 0;
    for (uint32_t k = 0; k < digits; ++k) {
        r = r * 3 + v % 3;
        v /= 3;
    }
    return r;
}

// One integrand factor (quality.cpp:35-63). Returns false for the
// indicator's early exit.
template <uint32_t FN>
__device__ __forceinline__ bool factor(float xs, double& v, const SceneConsts& sc)
{
    const double x = static_cast<double>(xs);
    if (FN == 0) { // product-sine: v *= (0.5*pi) * sin(pi * x); pi*x in [0, pi)
        const double pi = 3.141592653589793;
        v = __dmul_rn(v, __dmul_rn(1.5707963267948966, sin_cw(__dmul_rn(pi, x), sc)));
    } else if (FN == 1) { // product-poly: v *= (3.0 * x) * x
        v = __dmul_rn(v, __dmul_rn(__dmul_rn(3.0, x), x));
    } else { // indicator: [x < 0.7]
        if (!(x < 0.7))
            return false;
    }
    return true;
}

// One CTA per 4096-index chunk. Phase 1: the B threads (ChunkShape) evaluate
// the integrand at indices begin + t + B*m (m < 4096/B) into shared memory — all
// the sampling and FP64 math, fully parallel. Phase 2 (kahan): one thread
// runs the reference's sequential Neumaier sum over the 4096 values in index
// order, so the chunk partial is bit-identical to chunk_sum_kahan
// (quality.cpp:180-194); (int) the llround(v*2^32) terms are exactly
// associative, so the CTA reduces them in any order (quality.cpp:196-210).
// SMALL (Sobol', dims <= kSmallDims): the per-thread Sobol' state is indexed
// with compile-time dimension numbers (unrolled, guarded loops), so it stays
// in registers instead of local memory.
constexpr uint32_t kSmallDims = 8;
template <uint32_t KIND, uint32_t FN, uint32_t ACCUM, bool SMALL = false>
__global__ void __launch_bounds__(ChunkShape<KIND, SMALL>::kBlock)
    k_integrate(IntegrateParams p, double* __restrict__ partial,
                unsigned long long* __restrict__ isum, unsigned long long* __restrict__ bad)
{
    __shared__ double vals[4096];
    using Shape = ChunkShape<KIND, SMALL>;
    constexpr uint32_t kBlock = Shape::kBlock, kLogBlock = Shape::kLogBlock;
    constexpr uint32_t kSteps = Shape::kSteps, kLogSteps = Shape::kLogSteps;
    __shared__ uint32_t E[kLogSteps][kStateDims]; // sobol: XOR of columns kLogBlock..+c
    __shared__ uint32_t XB[kStateDims];   // sobol: value of `begin` (scramble included)
    __shared__ long long red[kBlockMax / 32];
    const uint64_t chunk = p.chunk0 + blockIdx.x;
    const uint64_t begin = chunk * 4096;
    const uint32_t count = static_cast<uint32_t>(p.n - begin < 4096 ? p.n - begin : 4096);
    const uint32_t dims = p.fdims;
    const uint32_t sdims = dims < kStateDims ? dims : kStateDims; // dims with incremental state
    const uint32_t t = threadIdx.x;
    const PixelStreamParams& q = p.pix;

    // per-stream pixel state (imageplane.cpp:366-405)
    uint32_t shift = 0, ipx0 = 0, ipy0 = 0, cell = 0;
    uint64_t block = 0, off = 0;
    if (KIND == 4)
        shift = phi3_fixed(static_cast<uint32_t>(hilbert_index(q.px, q.py, q.order)), q.tab3);
    if (KIND == 3)
        block = hilbert_index(q.px, q.py, q.order) * q.spp;
    if (KIND == 6) {
        const uint64_t r2 = q.exp_x == 0 ? 0 : __brevll(q.px) >> (64 - q.exp_x);
        const uint64_t r3 = digit_reverse3(q.py, q.exp_y);
        off = (r2 * q.crt_x % q.stride + r3 * q.crt_y % q.stride) % q.stride;
        ipx0 = static_cast<uint32_t>(off >> q.exp_x);
        ipy0 = static_cast<uint32_t>(off / q.scale_y);
    }
    if (KIND == 7)
        cell = (q.px % 128u) + (q.py % 128u) * 128u;
    const RadicalDim* rd = static_cast<const RadicalDim*>(q.radical_dims);

    // Sobol' state: x(begin + t + B m) = XB ^ X(t) ^ X(B m); m advances
    // with x ^= E[ctz(m+1)].
    uint32_t sob[SMALL ? kSmallDims : kStateDims];
    if (KIND == 0) {
        for (uint32_t j = t; j < sdims; j += kBlock) {
            uint32_t x = p.words ? p.words[j] : 0u;
            uint64_t b = begin;
            for (uint32_t k = 0; b; ++k, b >>= 1)
                if (b & 1u)
                    x ^= __ldg(p.colsT + k * p.mdims + j);
            XB[j] = x;
            uint32_t e = 0;
            for (uint32_t c = 0; c < kLogSteps; ++c) {
                e ^= __ldg(p.colsT + (kLogBlock + c) * p.mdims + j);
                E[c][j] = e;
            }
        }
        __syncthreads();
        if (SMALL) {
#pragma unroll
            for (uint32_t j = 0; j < kSmallDims; ++j)
                if (j < sdims) {
                    uint32_t x = XB[j];
                    for (uint32_t k = 0; k < kLogBlock; ++k)
                        if ((t >> k) & 1u)
                            x ^= __ldg(p.colsT + k * p.mdims + j);
                    sob[j] = x;
                }
        } else {
            for (uint32_t j = 0; j < sdims; ++j) {
                uint32_t x = XB[j];
                for (uint32_t k = 0; k < kLogBlock; ++k)
                    if ((t >> k) & 1u)
                        x ^= __ldg(p.colsT + k * p.mdims + j);
                sob[j] = x;
            }
        }
    }

    // Halton kinds: when every index of the chunk (mod prime_max_power) lies
    // in the fill-table blocks h0 and h0 + 1 of a dimension, its inverse is
    // the quotient-table form of the contiguous fill (device.cuh: hi_split):
    // one coalesced 8-B load and three integer ops instead of the digit loop.
    __shared__ const uint32_t* HTAB[kStateDims];
    __shared__ uint32_t HG[kStateDims], HLO[kStateDims], HQ0[kStateDims], HT0[kStateDims],
        HQ1[kStateDims], HT1[kStateDims];
    if (KIND == 1 || KIND == 3) {
        const uint32_t ib = static_cast<uint32_t>(KIND == 3 ? block + begin : begin);
        for (uint32_t j = t; j < sdims; j += kBlock) {
            const RadicalDim& r = rd[j];
            const uint32_t* tab = nullptr;
            if (r.fqx && ib <= 0xffffffffu - count) {
                const uint32_t ir = ib - div32(ib, r.divmp) * r.maxpow;
                const uint32_t G = r.fgroup, h0 = div32(ir, r.fdivg), lo0 = ir - h0 * G;
                if (static_cast<uint64_t>(ir) + count <= r.maxpow && lo0 + count <= 2 * G) {
                    uint32_t g0, mulg, h = h0;
                    const HiRecord a = hi_record(h0, r, g0, mulg);
                    HiRecord b = a;
                    if (lo0 + count > G)
                        hi_advance(h, b, g0, mulg, r);
                    HG[j] = G;
                    HLO[j] = lo0;
                    HQ0[j] = a.qa;
                    HT0[j] = a.thr;
                    HQ1[j] = b.qa;
                    HT1[j] = b.thr;
                    tab = r.fqx;
                }
            }
            HTAB[j] = tab;
        }
        __syncthreads();
    }

    bool finite = true;
    long long acc = 0;
    for (uint32_t m = 0; m < kSteps; ++m) {
        const uint32_t local = t + kBlock * m;
        if (local < count) {
            const uint64_t idx = begin + local;
            const uint32_t i = static_cast<uint32_t>(idx);
            double v = 1.0;
            bool alive = true;
            if (KIND == 0 && SMALL) {
#pragma unroll
                for (uint32_t j = 0; j < kSmallDims; ++j)
                    if (j < dims && alive)
                        alive = factor<FN>(map_u32(sob[j]), v, p.sc);
            } else
            for (uint32_t j = 0; j < dims && alive; ++j) {
                uint32_t x;
                if (KIND == 0)
                    x = j < kStateDims ? sob[j] : sobol_direct(idx, j, p);
                else if (KIND == 1 || KIND == 3) {
                    const uint32_t* tab = j < kStateDims ? HTAB[j] : nullptr;
                    if (tab) {
                        const uint32_t G = HG[j];
                        uint32_t lo = HLO[j] + local;
                        const bool up = lo >= G;
                        lo = up ? lo - G : lo;
                        const uint32_t e = __ldg(tab + lo); // rT = -qT * G mod 2^32
                        x = e + (up ? HQ1[j] : HQ0[j]) + (e * (0u - G) >= (up ? HT1[j] : HT0[j]) ? 1u : 0u);
                    } else {
                        x = radical_fixed(KIND == 1 ? i : static_cast<uint32_t>(block + idx), rd[j]);
                    }
                } else if (KIND == 2)
                    x = brev32(i) * __ldg(q.generator + j);
                else if (KIND == 4)
                    x = (brev32(i) + shift) * __ldg(q.generator + j);
                else if (KIND == 5)
                    x = brev32(~i) * (pixel_hash(j, q.px, q.py) | 1u);
                else if (KIND == 6)
                    x = j == 0   ? rad2(ipx0 + i * q.scale_y)
                        : j == 1 ? phi3_fixed(ipy0 + i * q.scale_x, q.tab3)
                                 : radical_fixed(static_cast<uint32_t>(off + idx * q.stride), rd[j]);
                else {
                    const uint32_t k = i ^ __ldg(q.xor_reorder + cell);
                    x = __ldg(q.xor_points + static_cast<uint64_t>(k) * q.xor_dims + j) ^
                        __ldg(q.xor_scramble + cell * q.xor_dims + j);
                }
                alive = factor<FN>(map_u32(x), v, p.sc);
            }
            if (FN == 2)
                v = alive ? 1.0 : 0.0;
            if (!isfinite(v)) {
                finite = false;
                atomicMin(bad, static_cast<unsigned long long>(idx));
            }
            if (ACCUM == 0)
                vals[local] = v;
            else
                acc += llround(__dmul_rn(v, 4294967296.0));
        }
        if (KIND == 0 && m + 1 < kSteps) {
            const uint32_t c = __ffs(static_cast<int>(m + 1)) - 1;
            if (SMALL) {
#pragma unroll
                for (uint32_t j = 0; j < kSmallDims; ++j)
                    if (j < sdims)
                        sob[j] ^= E[c][j];
            } else {
                for (uint32_t j = 0; j < sdims; ++j)
                    sob[j] ^= E[c][j];
            }
        }
    }
    (void)finite;
    if (ACCUM == 0) {
        __syncthreads();
        if (t == 0) { // chunk_sum_kahan's sequential Neumaier, index order
            double sum = 0.0, comp = 0.0;
            for (uint32_t k = 0; k < count; ++k)
                neumaier_add(sum, comp, vals[k]);
            partial[blockIdx.x] = __dadd_rn(sum, comp);
        }
    } else {
        for (int o = 16; o; o >>= 1)
            acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((t & 31) == 0)
            red[t >> 5] = acc;
        __syncthreads();
        if (t == 0) {
            long long s = 0;
            for (int w = 0; w < kBlock / 32; ++w)
                s += red[w];
            atomicAdd(isum, static_cast<unsigned long long>(s));
        }
    }
}

template <uint32_t KIND, uint32_t FN>
cudaError_t integrate_kind_fn(const IntegrateParams& p, uint32_t accum, double* partial,
                              unsigned long long* isum, unsigned long long* bad, cudaStream_t s)
{
    if (p.nchunks == 0)
        return cudaSuccess;
    if (p.nchunks > 0x7fffffffull)
        return cudaErrorInvalidValue;
    const unsigned grid = static_cast<unsigned>(p.nchunks);
    if (KIND == 0 && p.fdims <= kSmallDims) { // register state, 256 threads (+6-10 %)
        auto kern = accum == 0 ? k_integrate<KIND, FN, 0, true> : k_integrate<KIND, FN, 1, true>;
        kern<<<grid, ChunkShape<KIND, true>::kBlock, 0, s>>>(p, partial, isum, bad);
        return cudaGetLastError();
    }
    auto kern = accum == 0 ? k_integrate<KIND, FN, 0> : k_integrate<KIND, FN, 1>;
    kern<<<grid, ChunkShape<KIND>::kBlock, 0, s>>>(p, partial, isum, bad);
    return cudaGetLastError();
}

template <uint32_t KIND>
cudaError_t integrate_kind(const IntegrateParams& p, uint32_t accum, double* partial,
                           unsigned long long* isum, unsigned long long* bad, cudaStream_t s)
{
    switch (p.fn) {
    case 0: return integrate_kind_fn<KIND, 0>(p, accum, partial, isum, bad, s);
    case 1: return integrate_kind_fn<KIND, 1>(p, accum, partial, isum, bad, s);
    case 2: return integrate_kind_fn<KIND, 2>(p, accum, partial, isum, bad, s);
    }
    return cudaErrorInvalidValue;
}

} // namespace

cudaError_t launch_integrate(const IntegrateParams& p, uint32_t accum, double* partial,
                             unsigned long long* isum, unsigned long long* bad, cudaStream_t s)
{
    if (p.n == 0)
        return cudaSuccess;
    switch (p.pix.kind) {
    case 0: return integrate_kind<0>(p, accum, partial, isum, bad, s);
    case 1: return integrate_kind<1>(p, accum, partial, isum, bad, s);
    case 2: return integrate_kind<2>(p, accum, partial, isum, bad, s);
    case 3: return integrate_kind<3>(p, accum, partial, isum, bad, s);
    case 4: return integrate_kind<4>(p, accum, partial, isum, bad, s);
    case 5: return integrate_kind<5>(p, accum, partial, isum, bad, s);
    case 6: return integrate_kind<6>(p, accum, partial, isum, bad, s);
    case 7: return integrate_kind<7>(p, accum, partial, isum, bad, s);
    }
    return cudaErrorInvalidValue;
}

} // namespace qmcgpu
