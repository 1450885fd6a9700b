// kernels_bench.cu — the reference's component-generation benchmark
// (run_bench_kernel, bench.cpp:79-150) on the device, and the FP64 issue-rate
// probe that is the render's roofline denominator.
//
// run_bench_kernel walks a 128x128 tile (py wraps), 16 indices per pixel,
// `dims` components per index (bench.cpp:31-47), evaluates
// kernel(px, py, i, j) and folds every component into a Sink:
// value = rotl64(value, 7) ^ bits(x) (bench.cpp:23-25). rotl is linear over
// GF(2), so the fold of components x_0 .. x_{N-1} is
//     XOR_k rotl64(x_k, 7 * (N - 1 - k) mod 64),
// which every thread accumulates independently; warps XOR-reduce and one
// atomicXor per warp lands in the result — the same checksum as the
// reference's sequential walk.
#include "device.cuh"
#include "internal.hpp"

namespace qmcgpu {
namespace {

constexpr uint32_t kBenchTile = 128;     // bench.cpp:18
constexpr uint32_t kBenchPerPixel = 16;  // bench.cpp:19
constexpr uint32_t kBenchOrder = 7;      // bench.cpp:20 (Hilbert order of the tile)
constexpr int kBenchBlock = 256;

__device__ __forceinline__ uint64_t rotl64(uint64_t v, uint32_t s)
{
    return (v << s) | (v >> ((64u - s) & 63u)); // s = 0: v | v
}

// One row = one (pixel, index) pair: `dims` consecutive components.
template <int KIND>
__global__ void __launch_bounds__(kBenchBlock)
    k_bench(BenchParams p, unsigned long long* __restrict__ result)
{
    const uint64_t rows = (p.count + p.dims - 1) / p.dims;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t fold = 0;
    for (uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < rows;
         r += stride) {
        const uint32_t i = static_cast<uint32_t>(r % kBenchPerPixel);
        const uint64_t pix = r / kBenchPerPixel;
        const uint32_t px = static_cast<uint32_t>(pix % kBenchTile);
        const uint32_t py = static_cast<uint32_t>((pix / kBenchTile) % kBenchTile);
        const uint32_t gi = (py * kBenchTile + px) * kBenchPerPixel + i; // bench.cpp:74-77
        const uint64_t k0 = r * p.dims;
        const uint64_t left = p.count - k0;
        const uint32_t jn = left < p.dims ? static_cast<uint32_t>(left) : p.dims;
        // rotation of component k0: 7 * (count - 1 - k0) mod 64; -7 per step
        uint32_t rot = static_cast<uint32_t>((7u * ((p.count - 1 - k0) & 63u)) & 63u);
        uint32_t pre = 0; // per-row invariant of the kind
        if (KIND == QMC_BENCH_LATTICE)
            pre = brev32(gi);
        else if (KIND == QMC_BENCH_PIXEL_SHIFTED_LATTICE)
            pre = brev32(i) + phi3_fixed(static_cast<uint32_t>(hilbert_index(px, py, kBenchOrder)),
                                         p.tab3);
        else if (KIND == QMC_BENCH_PIXEL_RANDOM_LATTICE)
            pre = brev32(0xffffffffu - i);
        for (uint32_t j = 0; j < jn; ++j) {
            uint32_t x;
            if (KIND == QMC_BENCH_SOBOL) {
                x = 0; // sobol_component(gi, j, M), digitalnet.cpp:111-137
                for (uint32_t b = gi, k = 0; b; b >>= 1, ++k)
                    if (b & 1u)
                        x ^= __ldg(p.colsT + k * p.dims + j);
            } else if (KIND == QMC_BENCH_HALTON || KIND == QMC_BENCH_HALTON_TABLED) {
                x = radical_fixed(gi, static_cast<const RadicalDim*>(p.rd)[j]); // radical.cpp:130-208
            } else if (KIND == QMC_BENCH_PIXEL_RANDOM_LATTICE) {
                x = pre * (pixel_hash(j, px, py) | 1u); // lattice.hpp:51-56
            } else {
                x = pre * __ldg(p.g + j); // lattice.hpp:31-34, imageplane.hpp:26-31
            }
            fold ^= rotl64(map_bits(x), rot);
            rot = (rot - 7u) & 63u;
        }
    }
    for (int o = 16; o > 0; o >>= 1)
        fold ^= __shfl_xor_sync(0xffffffffu, fold, o);
    if ((threadIdx.x & 31u) == 0 && fold)
        atomicXor(result, static_cast<unsigned long long>(fold));
}

// FP64 issue-rate probe: 8 independent DFMA chains per thread.
constexpr int kProbeChains = 8;

__global__ void __launch_bounds__(kBenchBlock) k_fp64_probe(double* __restrict__ out, uint32_t iters)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    double a[kProbeChains];
#pragma unroll
    for (int c = 0; c < kProbeChains; ++c)
        a[c] = 1.0 + 1e-9 * (t + c);
    const double b = 0.999999999, d = 1e-7;
    for (uint32_t k = 0; k < iters; ++k) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int c = 0; c < kProbeChains; ++c)
                a[c] = __fma_rn(a[c], b, d);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kProbeChains; ++c)
        s += a[c];
    out[t] = s;
}

template <int KIND>
cudaError_t launch_bench_kind(const BenchParams& p, unsigned long long* result, cudaStream_t s)
{
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bench<KIND>, kBenchBlock, 0);
    const uint64_t rows = (p.count + p.dims - 1) / p.dims;
    const uint64_t want = (rows + kBenchBlock - 1) / kBenchBlock;
    const uint64_t grid = std::min<uint64_t>(want, static_cast<uint64_t>(sm_count()) *
                                                       std::max(per_sm, 1));
    k_bench<KIND><<<static_cast<unsigned>(std::max<uint64_t>(grid, 1)), kBenchBlock, 0, s>>>(
        p, result);
    return cudaGetLastError();
}

} // namespace

cudaError_t launch_bench(const BenchParams& p, unsigned long long* result, cudaStream_t s)
{
    switch (p.kind) {
    case QMC_BENCH_SOBOL: return launch_bench_kind<QMC_BENCH_SOBOL>(p, result, s);
    case QMC_BENCH_HALTON: return launch_bench_kind<QMC_BENCH_HALTON>(p, result, s);
    case QMC_BENCH_HALTON_TABLED: return launch_bench_kind<QMC_BENCH_HALTON_TABLED>(p, result, s);
    case QMC_BENCH_LATTICE: return launch_bench_kind<QMC_BENCH_LATTICE>(p, result, s);
    case QMC_BENCH_PIXEL_SHIFTED_LATTICE:
        return launch_bench_kind<QMC_BENCH_PIXEL_SHIFTED_LATTICE>(p, result, s);
    case QMC_BENCH_PIXEL_RANDOM_LATTICE:
        return launch_bench_kind<QMC_BENCH_PIXEL_RANDOM_LATTICE>(p, result, s);
    default: return cudaErrorInvalidValue;
    }
}

uint64_t fp64_probe_threads()
{
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fp64_probe, kBenchBlock, 0);
    return static_cast<uint64_t>(sm_count()) * std::max(per_sm, 1) * kBenchBlock;
}

cudaError_t launch_fp64_probe(double* out, uint64_t threads, uint32_t iters, cudaStream_t s)
{
    k_fp64_probe<<<static_cast<unsigned>(threads / kBenchBlock), kBenchBlock, 0, s>>>(out, iters);
    return cudaGetLastError();
}

uint64_t fp64_probe_flops(uint64_t threads, uint32_t iters)
{
    return 2ull * threads * kProbeChains * 4ull * iters; // one DFMA = 2 flops
}

} // namespace qmcgpu
