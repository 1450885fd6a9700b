// kernels_integrate.cu — fused QMC integration (reference
// integrate(), quality.cpp:214-282, with builtin_integrands, :28-66).
//
// One thread owns one fixed 4096-index chunk (quality.cpp:178) and walks it
// in index order: sample every integrand dimension at the integer stage ->
// bit-exact float map -> the integrand in FP64 with the reference's
// operation order (explicit _rn intrinsics, no FMA contraction) -> Neumaier
// (kahan) or llround(v * 2^32) (int) accumulation. Chunk partials are
// written per chunk and combined in chunk order on the host (Kahan: the
// reference's rank-ordered CompensatedSum, quality.cpp:262-267) or summed
// with exact 64-bit atomics on the device (int: associative, :268-272).
#include <cstdint>

#include "device.cuh"
#include "internal.hpp"

namespace qmcgpu {

namespace {

constexpr uint32_t kMaxDims = 64; // local sample-state capacity per thread
constexpr int kBlock = 128;

__device__ __forceinline__ uint32_t rad2(uint32_t i) { return brev32(i & 0x7fffffffu); }

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
__device__ __forceinline__ bool factor(float xs, double& v)
{
    const double x = static_cast<double>(xs);
    if (FN == 0) { // product-sine: v *= (0.5*pi) * sin(pi * x)
        const double pi = 3.141592653589793;
        v = __dmul_rn(v, __dmul_rn(1.5707963267948966, sin(__dmul_rn(pi, x))));
    } else if (FN == 1) { // product-poly: v *= (3.0 * x) * x
        v = __dmul_rn(v, __dmul_rn(__dmul_rn(3.0, x), x));
    } else { // indicator: [x < 0.7]
        if (!(x < 0.7))
            return false;
    }
    return true;
}

template <uint32_t KIND, uint32_t FN, uint32_t ACCUM>
__global__ void __launch_bounds__(kBlock)
    k_integrate(IntegrateParams p, double* __restrict__ partial,
                unsigned long long* __restrict__ isum, unsigned long long* __restrict__ bad)
{
    const uint64_t chunk = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t begin = chunk * 4096;
    if (begin >= p.n)
        return;
    const uint64_t end = begin + 4096 < p.n ? begin + 4096 : p.n;
    const uint32_t dims = p.fdims;
    const PixelStreamParams& q = p.pix;

    // per-stream pixel state (imageplane.cpp:366-405)
    uint32_t shift = 0, ipx0 = 0, ipy0 = 0, cell = 0;
    uint64_t block = 0, off = 0;
    if (KIND == 4)
        shift = phi3_fixed(static_cast<uint32_t>(hilbert_index(q.px, q.py, q.order)));
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

    // Sobol' state: value of index `begin`, then natural-order updates
    uint32_t sob[kMaxDims];
    if (KIND == 0) {
        for (uint32_t j = 0; j < dims; ++j) {
            uint32_t x = p.words ? p.words[j] : 0u;
            uint64_t b = begin;
            for (uint32_t k = 0; b; ++k, b >>= 1)
                if (b & 1u)
                    x ^= __ldg(p.colsT + k * p.mdims + j);
            sob[j] = x;
        }
    }

    double sum = 0.0, comp = 0.0;
    long long acc = 0;
    for (uint64_t idx = begin; idx < end; ++idx) {
        const uint32_t i = static_cast<uint32_t>(idx);
        double v = 1.0;
        bool alive = true;
        for (uint32_t j = 0; j < dims && alive; ++j) {
            uint32_t x;
            if (KIND == 0)
                x = sob[j];
            else if (KIND == 1)
                x = radical_fixed(i, rd[j]);
            else if (KIND == 2)
                x = brev32(i) * __ldg(q.generator + j);
            else if (KIND == 3)
                x = radical_fixed(static_cast<uint32_t>(block + idx), rd[j]);
            else if (KIND == 4)
                x = (brev32(i) + shift) * __ldg(q.generator + j);
            else if (KIND == 5)
                x = brev32(~i) * (pixel_hash(j, q.px, q.py) | 1u);
            else if (KIND == 6)
                x = j == 0   ? rad2(ipx0 + i * q.scale_y)
                    : j == 1 ? phi3_fixed(ipy0 + i * q.scale_x)
                             : radical_fixed(static_cast<uint32_t>(off + idx * q.stride), rd[j]);
            else {
                const uint32_t k = i ^ __ldg(q.xor_reorder + cell);
                x = __ldg(q.xor_points + static_cast<uint64_t>(k) * q.xor_dims + j) ^
                    __ldg(q.xor_scramble + cell * q.xor_dims + j);
            }
            alive = factor<FN>(map_u32(x), v);
        }
        if (FN == 2)
            v = alive ? 1.0 : 0.0;
        if (!isfinite(v))
            atomicMin(bad, static_cast<unsigned long long>(idx));
        if (ACCUM == 0)
            neumaier_add(sum, comp, v);
        else
            acc += llround(__dmul_rn(v, 4294967296.0));
        if (KIND == 0) { // x(i+1) = x(i) ^ C[0] ^ ... ^ C[ctz(i+1)]
            const uint64_t nx = idx + 1;
            const uint32_t c = static_cast<uint32_t>(__ffsll(static_cast<long long>(nx)) - 1);
            for (uint32_t k = 0; k <= c && k < 52; ++k)
                for (uint32_t j = 0; j < dims; ++j)
                    sob[j] ^= __ldg(p.colsT + k * p.mdims + j);
        }
    }
    if (ACCUM == 0)
        partial[chunk] = __dadd_rn(sum, comp);
    else
        atomicAdd(isum, static_cast<unsigned long long>(acc));
}

template <uint32_t KIND, uint32_t FN>
cudaError_t integrate_kind_fn(const IntegrateParams& p, uint32_t accum, double* partial,
                              unsigned long long* isum, unsigned long long* bad, cudaStream_t s)
{
    const uint64_t chunks = (p.n + 4095) / 4096;
    const unsigned grid = static_cast<unsigned>((chunks + kBlock - 1) / kBlock);
    if (accum == 0)
        k_integrate<KIND, FN, 0><<<grid, kBlock, 0, s>>>(p, partial, isum, bad);
    else
        k_integrate<KIND, FN, 1><<<grid, kBlock, 0, s>>>(p, partial, isum, bad);
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

uint32_t integrate_max_dims() { return kMaxDims; }

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
