// internal.hpp — host<->kernel interface of libqmcgpu (not part of the ABI).
#pragma once

#include <cstdint>
#include <cstring>

#include <cuda_runtime.h>

namespace qmcgpu {

// Exact division by a runtime divisor d >= 2 (see div32 in device.cuh).
struct Div32 {
    uint32_t m, s;
};

#ifdef __CUDACC__
__host__ __device__
#endif
inline Div32 make_div32(uint32_t d)
{
    uint32_t l = 0;
    while (l < 32 && (1ull << l) < d)
        ++l; // l = ceil(log2 d)
    const uint64_t m = ((1ull << 32) * ((1ull << l) - d)) / d + 1;
    return Div32{static_cast<uint32_t>(m), l - 1};
}

// Per-launch placement of a fill: points [first, first + n) of the
// sequence land at out[(i - first) * dims + j] (device pointer).
struct FillRange {
    uint64_t first;
    uint64_t n;
    void* out;
};

// Render parameters resolved on the host (render.cpp:83-106 defaults).
// Constants of the render's sine (device.cuh sin_cw) and integrand, carried
// in the kernel parameters so the per-sample loop reads them from the
// constant bank instead of rematerialising 64-bit immediates every sample.
struct SceneConsts {
    double k8pi;                        // 8 * pi (render.hpp:24-27)
    double two_over_pi;                 // 0x3fe45f306dc9c883
    double pio2_hi, pio2_mid, pio2_lo;  // pi/2 in three parts, negated
    double disc_r2;                     // 0.3 * 0.3 rounded (render.cpp:23-24)
};

__host__ __device__ inline double bits_to_double(uint64_t b)
{
    double d;
    memcpy(&d, &b, 8);
    return d;
}

__host__ __device__ inline SceneConsts make_scene_consts()
{
    return {25.132741228718345, bits_to_double(0x3fe45f306dc9c883ull),
            -bits_to_double(0x3ff921fb54442d18ull), -bits_to_double(0x3c91a62633145c00ull),
            -bits_to_double(0x397b839a252049c0ull), bits_to_double(0x3fb70a3d70a3d70aull)};
}

struct RenderParams {
    SceneConsts sc;
    uint32_t width, height, spp, order;
    uint32_t row_begin, row_end;
    double inv_w, inv_h;
    uint32_t g0, g1;          // lattice kinds
    uint32_t scr0, scr1;      // sobol scrambles
    // image-plane Halton (imageplane.cpp:80-106)
    uint32_t scale_x, scale_y, exp_x, exp_y;
    uint64_t stride, crt_x, crt_y;
    uint64_t stride_magic;    // floor((2^64 - 1) / stride) when stride < 2^32, else 0
    const uint32_t* cols2;    // device, [2][52] MSB-aligned columns (sobol)
    const uint32_t* xor_reorder;  // device, 128*128 (sobol_xor_table)
    const uint32_t* xor_scramble; // device, 128*128*2
    const uint32_t* xor_points;   // device, point_count*xor_dims
    uint32_t xor_point_count, xor_dims;
    const uint32_t* tab3;         // device phi_3 7-digit table (or null)
    Div32 divw;                   // exact division by width (width >= 2)
    uint32_t small_band;          // rows * width < 2^32: 32-bit pixel indexing
    double inv_spp;               // 1 / spp when spp is a power of two (exact), else 0
    const uint32_t* colmap;       // device, k_render's column order at spp >= 8 (or null)
    const uint32_t* q3;           // device, phi3_q's quotient tables (2 x 3^7 words)
    uint32_t dlo3, dhi3;          // image-plane halton: scale_x = dhi3 * 3^7 + dlo3
    const uint32_t* t3q3;         // device, tab3 | 0 | q3 | 0 0 (render_t3q3, 16-B padded)
};

// Per-stream (one pixel context) parameters for qmc_stream_fill kinds that
// depend on the pixel.
struct PixelStreamParams {
    uint32_t kind, dims;
    uint32_t px, py, order, spp;
    uint32_t width, height;
    const uint32_t* generator;   // device (lattice kinds)
    const void* radical_dims;    // device RadicalDim[dims] (halton kinds)
    uint32_t scale_x, scale_y, exp_x, exp_y;
    uint64_t stride, crt_x, crt_y;
    const uint32_t* xor_reorder;
    const uint32_t* xor_scramble;
    const uint32_t* xor_points;
    uint32_t xor_point_count, xor_dims;
    const uint32_t* tab3;        // device phi_3 7-digit table (or null)
};

// Small per-call arrays (XOR words / Owen seeds, generator vector, CP
// shifts) passed BY VALUE in the kernel parameter space (read through a
// __grid_constant__ reference), so a fill is one launch with no per-call
// device allocation or H2D copy. Arrays longer than kSmall words go through
// dev_a / dev_b (device copies) instead.
constexpr uint32_t kSmall = 256;
struct SmallArgs {
    const uint32_t* dev_a;
    const uint32_t* dev_b;
    uint32_t has_a, has_b;
    uint32_t a[kSmall];
    uint32_t b[kSmall];
};

// Fused QMC integration (quality.cpp:214-282): the stream's pixel-context
// state plus the integrand and (sobol) matrices / scrambles on the device.
struct IntegrateParams {
    PixelStreamParams pix; // pix.kind = sampler kind, pix.dims = stream dims
    uint32_t fn, fdims;    // integrand id, integrand dims (<= stream dims)
    uint64_t n;
    const uint32_t* colsT; // sobol: device [52][mdims]
    uint32_t mdims;
    const uint32_t* words;    // sobol: device XOR scrambles or null
    SceneConsts sc;           // product-sine's sine (sin_cw)
    uint64_t chunk0, nchunks; // this launch: 4096-index chunks [chunk0, chunk0 + nchunks)
};

// run_bench_kernel (bench.cpp:79-150) on the device: kernel ids, and the
// tables the components read.
enum BenchKind : uint32_t {
    QMC_BENCH_SOBOL = 0,
    QMC_BENCH_HALTON = 1,
    QMC_BENCH_HALTON_TABLED = 2,
    QMC_BENCH_LATTICE = 3,
    QMC_BENCH_PIXEL_SHIFTED_LATTICE = 4,
    QMC_BENCH_PIXEL_RANDOM_LATTICE = 5,
};
struct BenchParams {
    uint64_t count;
    uint32_t dims, kind;
    const uint32_t* colsT; // sobol: device [52][dims]
    const void* rd;        // halton kinds: device RadicalDim[dims]
    const uint32_t* g;     // lattice kinds: device generator vector
    const uint32_t* tab3;  // phi_3 7-digit table (pixel shift)
};

// ------------------------------------------------------------ launchers
// All launchers write DEVICE memory and are asynchronous on `s`.
cudaError_t launch_map(const uint32_t* in, float* out, uint64_t n, cudaStream_t s);
cudaError_t launch_map_selfcheck(unsigned long long* dev_count, cudaStream_t s);

// colsT: device [52][dims] columns (k-major); args.a = per-dim words.
// mode 0 plain/xor (words = xor words), 2 owen (colsT bit-reversed, words =
// seeds). out_u32: write the integer stage instead of floats.
cudaError_t launch_sobol(const uint32_t* colsT, const uint32_t* colsT_rev, const SmallArgs& args,
                         uint32_t dims, int mode, bool out_u32, const FillRange& r,
                         cudaStream_t s);

// args.a = generator vector g, args.b = CP shifts (optional).
cudaError_t launch_lattice(const SmallArgs& args, uint32_t dims, bool out_u32,
                           const FillRange& r, cudaStream_t s);

// dims == 1, prime 2 (van der Corput, config C1).
cudaError_t launch_vdc(bool out_u32, const FillRange& r, cudaStream_t s);

// rd: device RadicalDim[dims].
// rd: device RadicalDim[dims]; rd_host: the same array on the host (or
// null: the level-table fill is then not taken)
cudaError_t launch_halton(const void* rd, uint32_t dims, bool out_u32, const FillRange& r,
                          cudaStream_t s, const void* rd_host = nullptr);

cudaError_t launch_pixel_stream(const PixelStreamParams& p, bool out_u32, const FillRange& r,
                                cudaStream_t s);

cudaError_t launch_render(const RenderParams& p, uint32_t kind, uint32_t accum, float* out,
                          cudaStream_t s);

// Int-mode partial render over samples first, first+step, ... (< spp):
// int64 per pixel of the band; finalize: float(sum / 2^32 / spp).
cudaError_t launch_render_partial(const RenderParams& p, uint32_t kind, uint32_t first,
                                  uint32_t step, long long* acc, cudaStream_t s,
                                  bool add = false);
cudaError_t launch_render_finalize(const long long* acc, uint64_t npix, uint32_t spp, float* out,
                                   cudaStream_t s);

// image.cpp:25-30 quantization to bytes, `channels` copies per pixel.
cudaError_t launch_quantize(const float* v, uint64_t npix, uint32_t channels, unsigned char* out,
                            cudaStream_t s);

cudaError_t launch_scene_value(const double* xy, double* out, uint64_t n, cudaStream_t s);

// Write-only 128-bit streaming store probe over `bytes` (diagnostic).
cudaError_t launch_write_probe(void* out, uint64_t bytes, int mode, cudaStream_t s);

// partial: device [ceil(n/4096)] chunk sums (kahan); isum: exact int64 sum
// (int); bad: first index with a non-finite integrand value (~0 if none).
cudaError_t launch_integrate(const IntegrateParams& p, uint32_t accum, double* partial,
                             unsigned long long* isum, unsigned long long* bad, cudaStream_t s);

// Quality metrics (quality.cpp:76-156). scratch: device, 2n doubles.
cudaError_t launch_l2star(const float* pts, uint64_t n, uint32_t dims, double* scratch,
                          double* out, cudaStream_t s);
cudaError_t launch_mindist(const float* pts, uint64_t n, uint32_t dims, double* scratch,
                           double* out, cudaStream_t s);
cudaError_t launch_stratification(const float* v, uint32_t m, uint32_t dims, uint32_t j,
                                  uint32_t* hist, unsigned int* bad, cudaStream_t s);
uint32_t quality_max_dims();

// result: device u64, zeroed by the caller; receives the Sink checksum.
cudaError_t launch_bench(const BenchParams& p, unsigned long long* result, cudaStream_t s);
// FP64 probe: threads = one full wave of resident CTAs; out has `threads` doubles.
uint64_t fp64_probe_threads();
cudaError_t launch_fp64_probe(double* out, uint64_t threads, uint32_t iters, cudaStream_t s);
uint64_t fp64_probe_flops(uint64_t threads, uint32_t iters);

// Number of SMs of the current device (cached).
int sm_count();

} // namespace qmcgpu
