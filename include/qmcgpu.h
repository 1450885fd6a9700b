/*
 * qmcgpu.h — C-ABI of the B200-native QMC sampling path.
 *
 * Drop-in boundary for the reference library's hot path (qmckit `qmc::`,
 * /root/reference/proj). The reference has no FFI; its callers use the
 * `qmc::` C++ headers. This header is what those callers (or a ctypes /
 * cgo-style binding) bind instead; include/qmcgpu.hpp
 * re-exposes `qmc::`-style names on top of it.
 *
 * Conventions
 *   - Plain pointers and sizes; no torch or CUDA types in signatures.
 *     `qmc_stream` is a cudaStream_t passed as void* (NULL = default stream).
 *   - Every call returns a qmc_status; qmc_last_error() gives the message
 *     (thread-local). Status classes mirror the reference exceptions
 *     (errors.hpp:13-15 ConfigError, std::invalid_argument, std::out_of_range,
 *     std::overflow_error). Preconditions are checked on the host with the
 *     reference's conditions before anything is launched.
 *   - Batched fills write row-major [n][dims] (the `qmckit points --format
 *     bin` layout, tools/qmckit.cpp:225-241), component (i, j) at
 *     out[(i - first_index) * dims + j]. `out` may be DEVICE memory (the call
 *     is asynchronous on `stream`) or HOST memory (pinned recommended; the
 *     call pipelines device chunks through D2H copies and returns when the
 *     host buffer is complete).
 *   - QMC_OUT_F32 writes map_u32_to_unifloat(x) (bit-exact, unitfloat.hpp:
 *     34-50); QMC_OUT_U32 writes the 32-bit fixed-point integer stage x
 *     (the reference `*_fixed` functions).
 *   - No CPU fallback: every per-sample computation runs on the GPU; without
 *     a usable CUDA device calls fail with QMC_CUDA.
 */
#ifndef QMCGPU_H
#define QMCGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QMCGPU_ABI_VERSION 1

typedef enum qmc_status {
    QMC_OK = 0,
    QMC_CONFIG = 1,           /* qmc::ConfigError (errors.hpp:13-15) */
    QMC_INVALID_ARGUMENT = 2, /* std::invalid_argument */
    QMC_OUT_OF_RANGE = 3,     /* std::out_of_range */
    QMC_OVERFLOW = 4,         /* std::overflow_error */
    QMC_CUDA = 5,             /* CUDA runtime error / no device */
    QMC_NCCL = 6,             /* collective failure (reserved for host drivers) */
    QMC_INTERNAL = 9
} qmc_status;

typedef void* qmc_stream; /* cudaStream_t */

typedef enum qmc_output { QMC_OUT_F32 = 0, QMC_OUT_U32 = 1 } qmc_output;

/* ------------------------------------------------------------------ misc */
const char* qmc_last_error(void);
const char* qmc_status_string(qmc_status s);
int qmc_abi_version(void);

/* ------------------------------------------------ L0 (unitfloat.hpp:13-50) */
/* Batched map_u32_to_unifloat (unitfloat.hpp:34-50); in/out device or host. */
qmc_status qmc_map_u32_to_unifloat(const uint32_t* in, float* out, uint64_t n, qmc_stream stream);
/* Exhaustive 2^32 self-check of the device map against a device restatement
 * of the reference formula (SPEC acceptance 1); *mismatches = count. */
qmc_status qmc_map_selfcheck(uint64_t* mismatches, qmc_stream stream);

/* Diagnostic: write-only store streams over a device buffer (the HBM write
 * ceiling the fills are compared against in bench.py). mode 0: 128-bit
 * streaming stores, grid-stride; 1: 128-bit write-back stores; 2: 256-bit
 * streaming stores; 3: 128-bit streaming, contiguous chunk per warp;
 * 4: cudaMemsetAsync. */
qmc_status qmc_write_probe(void* device_buffer, uint64_t bytes, int mode, qmc_stream stream);

/* --------------------------------------------- host setup (no per-sample work) */
/* primes.cpp:50-62 */
qmc_status qmc_prime(uint32_t index, uint32_t* out);
qmc_status qmc_prime_max_power(uint32_t index, uint32_t* out);
/* radical.cpp:50-74; out has `base` entries */
qmc_status qmc_faure_permutation(uint32_t base, uint32_t* out);
/* radical.cpp:271-279; out has `dims` entries (factor = prime - 1) */
qmc_status qmc_default_linear_factors(uint32_t dims, uint32_t* out);
/* lattice.cpp:81-104 */
qmc_status qmc_lfsr_generator_vector(uint32_t seed, uint32_t dims, uint32_t* out);
/* lattice.cpp:71-77 (seeds of the scrambles; the render kinds hash on device) */
uint32_t qmc_pixel_hash(uint32_t j, uint32_t px, uint32_t py);
/* render.cpp:28-34 */
uint32_t qmc_hilbert_order_for(uint32_t width, uint32_t height);
/* imageplane.cpp:114-130 */
qmc_status qmc_partition_by_extra_dimension(uint32_t part, uint32_t parts, uint32_t base,
                                            uint64_t* remainder, uint64_t* modulus);
/* hilbert.hpp:39-56: invalid_argument unless order in [1, 31], out_of_range
 * for a pixel outside the 2^order grid */
qmc_status qmc_hilbert_index(uint32_t x, uint32_t y, uint32_t order, uint64_t* out);
/* hilbert_phi3_fixed (imageplane.cpp:16-21): phi_3 of the pixel's Hilbert
 * index at the integer stage — the pixel-shifted lattice's shift */
qmc_status qmc_hilbert_phi3_fixed(uint32_t x, uint32_t y, uint32_t order, uint32_t* out);
/* hilbert.hpp:59-78: the inverse (same orientation) */
qmc_status qmc_hilbert_xy(uint64_t d, uint32_t order, uint32_t* x, uint32_t* y);
/* imageplane.cpp:43-51: the `digits` least significant base-b digits of v,
 * reversed */
uint64_t qmc_digit_reverse(uint64_t v, uint32_t base, uint32_t digits);
/* lattice_shift_fixed (lattice.cpp:157-170): delta_j = brev(k * 2^m) * g_j,
 * the integer shift that maps block 0 of 2^m lattice points onto block k
 * (pass it as qmc_lattice_fill's `shifts`); invalid_argument for m > 32,
 * overflow when k * 2^m does not fit 32 bits. out has `dims` entries. */
qmc_status qmc_lattice_shift_fixed(uint32_t k, uint32_t m, const uint32_t* g, uint32_t dims,
                                   uint32_t* out);
/* imageplane.cpp:80-106: scales, exponents, stride; offset of (px, py) */
typedef struct qmc_halton_enumeration {
    uint32_t scale_x, scale_y, exponent_x, exponent_y;
    uint64_t stride;
} qmc_halton_enumeration;
qmc_status qmc_halton_pixel_enumeration(uint32_t width, uint32_t height, uint32_t px, uint32_t py,
                                        qmc_halton_enumeration* e, uint64_t* offset);

/* ------------------------------- generator matrices (digitalnet.cpp:23-109) */
typedef struct qmc_matrices qmc_matrices; /* immutable; device copy per GPU */
/* build_matrices(builtin_direction_numbers(), dims) — digitalnet.cpp:73-109 */
qmc_status qmc_matrices_builtin(uint32_t dims, qmc_matrices** out);
/* parse_direction_numbers(text) + build_matrices — digitalnet.cpp:23-109 */
qmc_status qmc_matrices_from_text(const char* text, uint32_t dims, qmc_matrices** out);
/* caller-supplied MSB-aligned columns[dims][52] */
qmc_status qmc_matrices_from_columns(const uint32_t* columns, uint32_t dims, qmc_matrices** out);
uint32_t qmc_matrices_dims(const qmc_matrices* m);
qmc_status qmc_matrices_columns(const qmc_matrices* m, uint32_t* out /* dims*52 */);
void qmc_matrices_destroy(qmc_matrices* m);

/* ------------------------------------------------------------- batched fills */
typedef enum qmc_sobol_scramble {
    QMC_SOBOL_NONE = 0, /* digitalnet.cpp:111-131 with scramble 0 */
    QMC_SOBOL_XOR = 1,  /* per-dimension XOR word (the reference's scramble) */
    QMC_SOBOL_OWEN = 2  /* hash-based nested-uniform (Owen) scramble, per-dim seed */
} qmc_sobol_scramble;

/* sobol_component(_fixed) / sobol_point — digitalnet.cpp:111-151.
 * Requires dims <= qmc_matrices_dims(m) (else OUT_OF_RANGE) and
 * first_index + n <= 2^52 (else INVALID_ARGUMENT, digitalnet.cpp:114-115).
 * words: host array of dims entries (XOR words / Owen seeds), NULL = zeros. */
qmc_status qmc_sobol_fill(const qmc_matrices* m, uint64_t first_index, uint64_t n, uint32_t dims,
                          qmc_sobol_scramble scramble, const uint32_t* words, qmc_output kind,
                          void* out, qmc_stream stream);

typedef enum qmc_radical_scramble {
    QMC_RADICAL_PLAIN = 0,  /* radical.cpp:130-142 */
    QMC_RADICAL_LINEAR = 1, /* radical.cpp:144-164, factor per prime */
    QMC_RADICAL_FAURE = 2   /* radical.cpp:166-181 with faure_permutation */
} qmc_radical_scramble;

/* Halton points (radical.cpp:240-269): component j = radical inverse of
 * (uint32_t)i in prime(j). factors: host, dims entries, NULL = defaults.
 * dims <= 1000. With dims = 1 this is radical_inverse(i, 0) (config C1). */
qmc_status qmc_halton_fill(uint64_t first_index, uint64_t n, uint32_t dims,
                           qmc_radical_scramble scramble, const uint32_t* factors,
                           qmc_output kind, void* out, qmc_stream stream);
/* radical_inverse*(i, prime_index) for one prime: out[n]. */
qmc_status qmc_radical_inverse_fill(uint64_t first_index, uint64_t n, uint32_t prime_index,
                                    qmc_radical_scramble scramble, uint32_t factor,
                                    qmc_output kind, void* out, qmc_stream stream);

/* Rank-1 lattice (lattice.hpp:31-39, lattice.cpp:48-55) with optional
 * integer Cranley-Patterson rotation: x = brev((uint32_t)i) * g_j + s_j
 * (mod 2^32), like lattice_point (lattice.cpp:48-55, no parity check of g;
 * qmc_stream_fill's lattice kinds apply make_stream's odd-generator check).
 * g: host, dims entries; shifts: host, dims entries or NULL (= plain). */
qmc_status qmc_lattice_fill(const uint32_t* g, const uint32_t* shifts, uint32_t dims,
                            uint64_t first_index, uint64_t n, qmc_output kind, void* out,
                            qmc_stream stream);

/* ---------------------------------------- SampleStream façade (imageplane.hpp) */
typedef enum qmc_sampler_kind { /* imageplane.hpp:122-131 */
    QMC_KIND_SOBOL = 0,
    QMC_KIND_HALTON = 1,
    QMC_KIND_LATTICE = 2,
    QMC_KIND_HALTON_HILBERT = 3,
    QMC_KIND_PIXEL_SHIFTED_LATTICE = 4,
    QMC_KIND_PIXEL_RANDOM_LATTICE = 5,
    QMC_KIND_IMAGE_PLANE_HALTON = 6,
    QMC_KIND_SOBOL_XOR_TABLE = 7
} qmc_sampler_kind;

/* imageplane.cpp:250-292 (ConfigError for unknown names) */
qmc_status qmc_sampler_kind_from_name(const char* name, qmc_sampler_kind* out);
const char* qmc_sampler_kind_name(qmc_sampler_kind kind);

/* XOR-table sampler data (imageplane.hpp:92-120), immutable handle. */
typedef struct qmc_xor_tables qmc_xor_tables;
/* white_noise_xor_tables(dims, point_count, seed) (imageplane.cpp:197-229) */
qmc_status qmc_xor_tables_white_noise(uint32_t dims, uint32_t point_count, uint32_t seed,
                                      qmc_xor_tables** out);
/* load_xor_tables(file, dims, points, point_count) (imageplane.cpp:163-195):
 * `bytes` = an XQT1 file image; points = host [point_count][dims] words. */
qmc_status qmc_xor_tables_load(const void* bytes, size_t len, uint32_t dims,
                               const uint32_t* points, uint32_t point_count,
                               qmc_xor_tables** out);
/* write_xor_table_file (imageplane.cpp:154-161); call with bytes = NULL to
 * get the size in *len. */
qmc_status qmc_xor_tables_write(const qmc_xor_tables* t, void* bytes, size_t* len);
uint32_t qmc_xor_tables_dims(const qmc_xor_tables* t);
uint32_t qmc_xor_tables_point_count(const qmc_xor_tables* t);
void qmc_xor_tables_destroy(qmc_xor_tables* t);

/* StreamParams (imageplane.hpp:139-158). Unused fields are ignored per kind. */
typedef struct qmc_stream_params {
    uint32_t dims;              /* >= 1 */
    const uint32_t* generator;  /* lattice kinds: host, generator_dims odd words */
    uint32_t generator_dims;
    const qmc_matrices* matrices;     /* sobol: NULL = builtin for dims */
    const uint32_t* sobol_scrambles;  /* sobol: host words or NULL (plain) */
    uint32_t sobol_scrambles_len;     /* must be >= dims when given */
    uint32_t halton_scramble;         /* qmc_radical_scramble (halton kinds) */
    const uint32_t* linear_factors;   /* host or NULL (defaults) */
    uint32_t linear_factors_len;
    uint32_t px, py, order;           /* pixel context (PixelCoord) */
    uint32_t spp;                     /* halton_hilbert block size */
    uint32_t width, height;           /* image_plane_halton */
    uint32_t xor_seed;                /* sobol_xor_table: white-noise tables seed */
    uint32_t xor_point_count;         /* sobol_xor_table: power of two */
    const qmc_xor_tables* xor_tables; /* sobol_xor_table: given tables (NULL = white noise
                                         from xor_seed / xor_point_count) */
} qmc_stream_params;

/* make_stream(kind, params) validation + SampleStream::sample(i, j) for
 * i in [first_index, first_index + n), j < dims (imageplane.cpp:310-461). */
qmc_status qmc_stream_fill(qmc_sampler_kind kind, const qmc_stream_params* params,
                           uint64_t first_index, uint64_t n, qmc_output out_kind, void* out,
                           qmc_stream stream);

/* ------------------------------ integration (quality.cpp:28-66, :214-282) */
typedef enum qmc_accum { QMC_ACCUM_KAHAN = 0, QMC_ACCUM_INT = 1 } qmc_accum; /* quality.hpp:35 */

typedef enum qmc_integrand_kind {
    QMC_PRODUCT_SINE = 0, /* prod_j (pi/2) sin(pi x_j), integral 1 */
    QMC_PRODUCT_POLY = 1, /* prod_j 3 x_j^2, integral 1 */
    QMC_INDICATOR = 2     /* prod_j [x_j < 0.7], integral 0.7^s */
} qmc_integrand_kind;

/* builtin_integrand(name, dims) (quality.cpp:68-74): id and exact integral. */
qmc_status qmc_builtin_integrand(const char* name, uint32_t dims, qmc_integrand_kind* kind,
                                 double* exact_integral);

typedef struct qmc_integration_row { /* IntegrationRow, quality.hpp:90-95 */
    uint64_t n;
    double estimate, abs_error, seconds;
} qmc_integration_row;

/* integrate(stream, f, n, mode) (quality.cpp:214-282) over the stream made
 * from (kind, params): fixed 4096-index chunks, one GPU thread per chunk in
 * index order, chunk partials combined in chunk order — the reference's
 * worker-count-independent result. */
qmc_status qmc_integrate(qmc_sampler_kind kind, const qmc_stream_params* params,
                         qmc_integrand_kind f, uint32_t f_dims, uint64_t n, qmc_accum mode,
                         qmc_integration_row* row, qmc_stream stream);

/* The same integration over only the 4096-index chunks [chunk_begin,
 * chunk_end) of [0, n) — the per-rank share of a multi-GPU integration.
 * Kahan mode: partials[chunk - chunk_begin] = the chunk's compensated sum
 * (chunk_sum_kahan, quality.cpp:180-194). Int mode: *int_sum = the exact sum
 * of llround(f * 2^32) over the range (quality.cpp:196-210). Combining all
 * chunks' partials with qmc_reduce_deterministic (ranks = chunk indices), or
 * adding the int sums, gives exactly qmc_integrate's estimate * n. */
qmc_status qmc_integrate_partials(qmc_sampler_kind kind, const qmc_stream_params* params,
                                  qmc_integrand_kind f, uint32_t f_dims, uint64_t n,
                                  uint64_t chunk_begin, uint64_t chunk_end, qmc_accum mode,
                                  double* partials, int64_t* int_sum, qmc_stream stream);

/* reduce_deterministic (quality.cpp:158-166): the values sorted by rank
 * (stable), then one CompensatedSum in rank order. */
qmc_status qmc_reduce_deterministic(const uint64_t* ranks, const double* values, uint64_t count,
                                    double* out);

/* ------------------------------- quality metrics (quality.cpp:76-156) */
/* Warnock's L2-star discrepancy of a row-major [n][dims] float point set
 * (device or host). Per-term products follow the reference's operation order;
 * the pair terms are summed per row with compensated tree sums (result within
 * ~1e-15 relative of the reference's sequential sum). dims <= 256. */
qmc_status qmc_l2_star_discrepancy(const float* points, uint64_t n, uint32_t dims, double* out,
                                   qmc_stream stream);
/* Minimum pairwise toroidal distance (order-free: bit-identical). */
qmc_status qmc_min_toroidal_distance(const float* points, uint64_t n, uint32_t dims, double* out,
                                     qmc_stream stream);
/* check_1d_stratification(make_stream(kind, params), j, m): *ok = every one
 * of the 2^m dyadic intervals holds exactly one of the first 2^m values of
 * dimension j; histogram (host, 2^m words) optional. */
qmc_status qmc_check_1d_stratification(qmc_sampler_kind kind, const qmc_stream_params* params,
                                       uint32_t j, uint32_t m, int* ok, uint32_t* histogram,
                                       qmc_stream stream);

/* ------------------------------------------- file formats (host + device) */
/* load_generator_vector (lattice.cpp:21-46): decimal components, '#'
 * comments. *dims = count; out (capacity words) may be NULL to query. */
qmc_status qmc_load_generator_vector(const char* text, uint32_t* out, uint32_t capacity,
                                     uint32_t* dims);
/* load_linear_factors (radical.cpp:281-306): out[dims] = defaults (b-1)
 * overridden by the file's "base factor" lines. */
qmc_status qmc_load_linear_factors(const char* text, uint32_t dims, uint32_t* out);
/* `qmckit points --format csv` text (qmckit.cpp:225-235): "%.9f" values,
 * comma-separated rows; points device or host; bytes = NULL queries *len.
 * (--format bin is the fills' row-major little-endian fp32 output itself.) */
qmc_status qmc_write_points_csv(const float* points, uint64_t n, uint32_t dims, void* bytes,
                                size_t* len, qmc_stream stream);
/* fnv1a64 (image.cpp:54-63). */
uint64_t qmc_fnv1a64(const void* data, uint64_t size);
/* write_pgm (channels 1, P5) / write_ppm (channels 3, P6) (image.cpp:34-52)
 * of a row-major float image (device or host) into `bytes`; bytes = NULL
 * queries the size in *len. The quantization runs on the device. */
qmc_status qmc_write_pnm(const float* image, uint32_t width, uint32_t height, uint32_t channels,
                         void* bytes, size_t* len, qmc_stream stream);

/* --------------------------------------------------- render (render.cpp:83-143) */
typedef struct qmc_render_job { /* RenderJob, render.hpp:31-47 */
    uint32_t width, height, spp;
    qmc_sampler_kind kind;        /* default pixel_shifted_lattice */
    qmc_accum accum;
    uint32_t seed;                /* 0 = defaults (render.cpp:94-106) */
    const uint32_t* generator;    /* host, >= 2 odd words, NULL = lfsr default */
    uint32_t generator_dims;
    const qmc_matrices* matrices; /* NULL = builtin 2-dim */
    const qmc_xor_tables* tables; /* sobol_xor_table: NULL = white noise (render.cpp:102-104) */
} qmc_render_job;

/* Integrates scene_value over every pixel footprint of rows
 * [row_begin, row_end) (the full image: 0, height) and writes
 * float(estimate) row-major into out (device or host), out[0] = pixel
 * (0, row_begin). One GPU thread owns one pixel and sums its samples in the
 * reference order (bit-compatible accumulation). Multi-GPU: each rank
 * renders a band; the host driver gathers the bands (one collective). */
qmc_status qmc_render(const qmc_render_job* job, uint32_t row_begin, uint32_t row_end, float* out,
                      qmc_stream stream);

/* render(job) across several GPUs of one process (no collective): the rows
 * are split into n_devices bands, one host thread per device renders its
 * band with qmc_render and copies it into its rows of `out` (HOST memory,
 * pinned or pageable). Each pixel keeps the single-GPU summation order, so
 * the image is bit-identical to a one-device render. A device may repeat. */
qmc_status qmc_render_devices(const qmc_render_job* job, const int* devices, uint32_t n_devices,
                              float* out);

/* The paper's sample partition across several GPUs of one process, with
 * the reduction fused into the render: part k of n (a power of two; samples
 * i == rev_2(k) mod n, partition_by_extra_dimension) runs on devices[k] and
 * its kernel atomically adds the int64 partial sums straight into one
 * accumulator on devices[0] — through NVLink peer access when the devices
 * differ — so no separate collective runs. The finalized image goes to
 * `out` (HOST memory) and is bit-identical to the one-device int render.
 * Int accumulator only (job->accum == QMC_ACCUM_INT). A device may repeat. */
qmc_status qmc_render_samples_devices(const qmc_render_job* job, const int* devices,
                                      uint32_t n_devices, float* out);

/* Sample-partitioned render (the paper's parallelization by an extra
 * radical-inverse dimension; partition_by_extra_dimension,
 * imageplane.cpp:114-130): part `part` of `parts` (a power of two) owns the
 * samples i == rev_2(part) (mod parts). Int accumulator only: writes the
 * int64 sum of llround(f * 2^32) per pixel of rows [row_begin, row_end) into
 * `accum` (device). Summing the accumulators of all parts (e.g. one NCCL
 * all-reduce across GPUs) and qmc_render_finalize gives exactly the int
 * render (render.cpp:72-78). */
qmc_status qmc_render_partial(const qmc_render_job* job, uint32_t part, uint32_t parts,
                              uint32_t row_begin, uint32_t row_end, int64_t* accum,
                              qmc_stream stream);
/* float(sum / 2^32 / spp) per pixel (device buffers). */
qmc_status qmc_render_finalize(const int64_t* accum, uint64_t npix, uint32_t spp, float* out,
                               qmc_stream stream);

/* ------------------------------------- component-generation benchmark
 * run_bench_kernel (bench.cpp:79-150; `qmckit bench`, SPEC acceptance 9) on
 * the device: the same walk (128x128 tile, 16 indices per pixel, `dims`
 * components each), the same kernels ("sobol", "halton", "halton-tabled",
 * "lattice", "pixel-shifted-lattice", "pixel-random-lattice") and the same
 * Sink checksum (rotl 7 fold of the float bits), so `checksum` equals the
 * reference's for the same (kernel, count, dims). One warm-up walk of
 * count / 8, then the timed walk (CUDA events on `stream`); synchronous. */
typedef struct qmc_bench_result {
    uint64_t evaluations;
    double seconds;
    double components_per_second;
    uint64_t checksum;
} qmc_bench_result;
qmc_status qmc_run_bench_kernel(const char* kernel, uint64_t count, uint32_t dims,
                                qmc_bench_result* out, qmc_stream stream);

/* Diagnostic: dense FP64 FMA throughput of this GPU (one wave of CTAs, 8
 * independent DFMA chains per thread; 2 flops per DFMA), the roofline
 * denominator of the render's FP64 integrand. Synchronous. */
qmc_status qmc_fp64_probe(uint32_t iters, double* flops_per_second, qmc_stream stream);

/* ------------------------------------------ multi-GPU render over NCCL
 * The one collective of the path, inside the library. It
 * replaces the reference's host worker pool (render.cpp:114-139) across
 * GPUs. NCCL is loaded on first use (an already-loaded libnccl.so.2 is
 * preferred; QMC_NCCL_LIBRARY=<path> overrides); without it these calls fail
 * with QMC_NCCL. */
typedef struct qmc_comm qmc_comm; /* wraps an ncclComm_t */
#define QMC_COMM_UNIQUE_ID_BYTES 128

typedef enum qmc_partition {
    /* row bands of ceil(H / nranks) rows + one ncclAllGather of the fp32
     * bands: every pixel keeps the one-GPU order (bit-identical image) */
    QMC_PARTITION_ROWS = 0,
    /* the paper's sample partition (rank r owns samples i == rev_2(r) mod
     * nranks, imageplane.cpp:114-130) + one ncclAllReduce(sum) of the int64
     * accumulators + finalize: int accumulator, power-of-two rank count,
     * bit-identical to the one-GPU int render */
    QMC_PARTITION_SAMPLES = 1
} qmc_partition;

/* ncclGetVersion of the NCCL the library bound. */
qmc_status qmc_nccl_version(int* version);
/* ncclGetUniqueId into id[QMC_COMM_UNIQUE_ID_BYTES] (rank 0; the caller
 * ships it to the other ranks over its own transport). */
qmc_status qmc_comm_unique_id(void* id);
/* ncclCommInitRank on the calling thread's current device. */
qmc_status qmc_comm_init_rank(const void* id, int nranks, int rank, qmc_comm** out);
/* ncclCommInitAll: one communicator per device of this process, out[n]. */
qmc_status qmc_comm_init_all(const int* devices, int n, qmc_comm** out);
/* Borrows an existing ncclComm_t (not destroyed by qmc_comm_destroy). */
qmc_status qmc_comm_from_nccl(void* nccl_comm, qmc_comm** out);
qmc_status qmc_comm_info(const qmc_comm* comm, int* rank, int* nranks, int* device);
void qmc_comm_destroy(qmc_comm* comm);

/* render(job) by every rank of `comm` (collective: all ranks call it with
 * the same job): this rank's share, then the collective, on `stream`; the
 * whole [height][width] image lands in `out` (device memory of the
 * communicator's GPU) on every rank. Asynchronous like qmc_render. */
qmc_status qmc_render_nccl(const qmc_render_job* job, const qmc_comm* comm, qmc_partition mode,
                           float* out, qmc_stream stream);
/* The same across `devices` of one process (ncclCommInitAll, one NCCL group
 * call for the collectives); the image goes to `out` (HOST memory). Devices
 * must be distinct (an NCCL communicator holds each GPU once). */
qmc_status qmc_render_nccl_devices(const qmc_render_job* job, const int* devices,
                                   uint32_t n_devices, qmc_partition mode, float* out);

/* scene_value (render.cpp:17-26) evaluated on the device for n (x, y)
 * pairs (device or host arrays of doubles) — integrand parity probe. */
qmc_status qmc_scene_value(const double* xy, double* out, uint64_t n, qmc_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* QMCGPU_H */
