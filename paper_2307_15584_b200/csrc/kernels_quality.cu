// kernels_quality.cu — point-set quality metrics (the
// reference's quality.cpp:76-156), as O(N^2 s) pairwise GPU kernels.
//
//   l2_star_discrepancy  Warnock's closed form (quality.cpp:76-114). Every
//                        per-point / per-pair product is computed with the
//                        reference's operation order (explicit _rn FP64);
//                        only the summation order of the pair terms differs
//                        (per-row compensated tree sums, rows combined in row
//                        order), so the result agrees to ~1e-15 relative.
//                        The single-point sum is combined in index order:
//                        bit-identical to the reference's.
//   min_toroidal_distance min over pairs (quality.cpp:116-136): order-free,
//                        so bit-identical.
//   stratification       histogram of floor(v * 2^m) (quality.cpp:138-156).
#include <cstdint>

#include "device.cuh"
#include "internal.hpp"

namespace qmcgpu {

namespace {

constexpr int kBlock = 256;
constexpr uint32_t kMaxRowDims = 256;

// Neumaier-compensated pair (sum, comp) combine, for tree reductions.
struct KSum {
    double s, c;
};

__device__ __forceinline__ void kadd(KSum& a, double v) { neumaier_add(a.s, a.c, v); }

__device__ __forceinline__ void kmerge(KSum& a, const KSum& b)
{
    kadd(a, b.s);
    a.c = __dadd_rn(a.c, b.c);
}

// One CTA per row i: single_i, diag_i + sum_{k>i} 2 prod_j (1 - max(x_ij, x_kj)).
__global__ void __launch_bounds__(kBlock)
    k_l2star_rows(const float* __restrict__ pts, uint64_t n, uint32_t dims,
                  double* __restrict__ single, double* __restrict__ pair_row)
{
    __shared__ float xi[kMaxRowDims];
    __shared__ double red_s[kBlock], red_c[kBlock];
    const uint64_t i = blockIdx.x;
    for (uint32_t j = threadIdx.x; j < dims; j += blockDim.x)
        xi[j] = pts[i * dims + j];
    __syncthreads();
    KSum acc{0.0, 0.0};
    for (uint64_t k = i + 1 + threadIdx.x; k < n; k += blockDim.x) {
        double prod = 1.0;
        for (uint32_t j = 0; j < dims; ++j) {
            const float m = fmaxf(xi[j], pts[k * dims + j]);
            prod = __dmul_rn(prod, __dsub_rn(1.0, static_cast<double>(m)));
        }
        kadd(acc, __dmul_rn(2.0, prod));
    }
    red_s[threadIdx.x] = acc.s;
    red_c[threadIdx.x] = acc.c;
    __syncthreads();
    for (int w = kBlock / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            KSum a{red_s[threadIdx.x], red_c[threadIdx.x]};
            kmerge(a, KSum{red_s[threadIdx.x + w], red_c[threadIdx.x + w]});
            red_s[threadIdx.x] = a.s;
            red_c[threadIdx.x] = a.c;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double diag = 1.0, sp = 1.0;
        for (uint32_t j = 0; j < dims; ++j) {
            const double x = static_cast<double>(xi[j]);
            diag = __dmul_rn(diag, __dsub_rn(1.0, x));
            sp = __dmul_rn(sp, __dmul_rn(__dsub_rn(1.0, __dmul_rn(x, x)), 0.5));
        }
        KSum row{diag, 0.0};
        kmerge(row, KSum{red_s[0], red_c[0]});
        pair_row[i] = __dadd_rn(row.s, row.c);
        single[i] = sp;
    }
}

// One thread: the two compensated sums over rows in row order, then
// Warnock's formula (quality.cpp:110-113).
__global__ void k_l2star_final(const double* __restrict__ single,
                               const double* __restrict__ pair_row, uint64_t n, uint32_t dims,
                               double* __restrict__ out)
{
    double s1 = 0.0, c1 = 0.0, s2 = 0.0, c2 = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        neumaier_add(s1, c1, single[i]);
        neumaier_add(s2, c2, pair_row[i]);
    }
    const double nd = static_cast<double>(n);
    const double t2 = __dadd_rn(__dsub_rn(pow(3.0, -static_cast<double>(dims)),
                                          __dmul_rn(__ddiv_rn(2.0, nd), __dadd_rn(s1, c1))),
                                __ddiv_rn(__dadd_rn(s2, c2), __dmul_rn(nd, nd)));
    *out = sqrt(fmax(t2, 0.0));
}

// One CTA per row i: min_{k>i} sum_j min(|d|, 1-|d|)^2 (quality.cpp:124-133).
__global__ void __launch_bounds__(kBlock)
    k_mindist_rows(const float* __restrict__ pts, uint64_t n, uint32_t dims,
                   double* __restrict__ row_min)
{
    __shared__ float xi[kMaxRowDims];
    __shared__ double red[kBlock];
    const uint64_t i = blockIdx.x;
    for (uint32_t j = threadIdx.x; j < dims; j += blockDim.x)
        xi[j] = pts[i * dims + j];
    __syncthreads();
    double best = __longlong_as_double(0x7ff0000000000000ll); // +inf
    for (uint64_t k = i + 1 + threadIdx.x; k < n; k += blockDim.x) {
        double d2 = 0.0;
        for (uint32_t j = 0; j < dims; ++j) {
            double d = fabs(__dsub_rn(static_cast<double>(xi[j]),
                                      static_cast<double>(pts[k * dims + j])));
            d = fmin(d, __dsub_rn(1.0, d));
            d2 = __dadd_rn(d2, __dmul_rn(d, d));
        }
        best = fmin(best, d2);
    }
    red[threadIdx.x] = best;
    __syncthreads();
    for (int w = kBlock / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w)
            red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0)
        row_min[i] = red[0];
}

__global__ void k_min_final(const double* __restrict__ row_min, uint64_t n,
                            double* __restrict__ out)
{
    double best = __longlong_as_double(0x7ff0000000000000ll);
    for (uint64_t i = 0; i < n; ++i)
        best = fmin(best, row_min[i]);
    *out = sqrt(best);
}

// histogram of floor(v * 2^m) over column j of a row-major [2^m][dims]
// float array; `bad` counts buckets != 1 afterwards (second kernel).
__global__ void k_strat_hist(const float* __restrict__ v, uint32_t count, uint32_t dims,
                             uint32_t j, uint32_t m, uint32_t* __restrict__ hist)
{
    const uint32_t stride = gridDim.x * blockDim.x;
    const float scale = __uint_as_float((127u + m) << 23); // 2^m exactly
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const uint32_t b = static_cast<uint32_t>(__fmul_rn(v[static_cast<uint64_t>(i) * dims + j], scale));
        atomicAdd(hist + (b < count ? b : count - 1), 1u);
    }
}

__global__ void k_strat_check(const uint32_t* __restrict__ hist, uint32_t count,
                              unsigned int* __restrict__ bad)
{
    const uint32_t stride = gridDim.x * blockDim.x;
    unsigned int b = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
        b += hist[i] != 1u;
    if (b)
        atomicAdd(bad, b);
}

} // namespace

uint32_t quality_max_dims() { return kMaxRowDims; }

cudaError_t launch_l2star(const float* pts, uint64_t n, uint32_t dims, double* scratch,
                          double* out, cudaStream_t s)
{
    k_l2star_rows<<<static_cast<unsigned>(n), kBlock, 0, s>>>(pts, n, dims, scratch,
                                                            scratch + n);
    k_l2star_final<<<1, 1, 0, s>>>(scratch, scratch + n, n, dims, out);
    return cudaGetLastError();
}

cudaError_t launch_mindist(const float* pts, uint64_t n, uint32_t dims, double* scratch,
                           double* out, cudaStream_t s)
{
    k_mindist_rows<<<static_cast<unsigned>(n), kBlock, 0, s>>>(pts, n, dims, scratch);
    k_min_final<<<1, 1, 0, s>>>(scratch, n, out);
    return cudaGetLastError();
}

cudaError_t launch_stratification(const float* v, uint32_t m, uint32_t dims, uint32_t j,
                                  uint32_t* hist, unsigned int* bad, cudaStream_t s)
{
    const uint32_t count = 1u << m;
    const unsigned grid = (count + kBlock - 1) / kBlock < 1024 ? (count + kBlock - 1) / kBlock : 1024;
    k_strat_hist<<<grid, kBlock, 0, s>>>(v, count, dims, j, m, hist);
    k_strat_check<<<grid, kBlock, 0, s>>>(hist, count, bad);
    return cudaGetLastError();
}

} // namespace qmcgpu
