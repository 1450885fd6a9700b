// abi_core.cpp — the extern "C" boundary (include/qmcgpu.h) of libqmcgpu:
// status strings, L0 map, host setup, generator matrices, the fills, the
// SampleStream façade, integration, XOR tables, quality metrics and formats.
// (The fused render lives in abi_render.cpp.)
//
// Host responsibilities only: validate arguments with the reference's
// conditions (so callers see the same error classes), upload per-call
// parameters, place the output (device pointer: one asynchronous launch;
// host pointer: chunked device fill + D2H pipeline), and launch the kernels.
// No per-sample arithmetic happens here.
#include "objects.hpp"

#include <chrono>
#include <cmath>
#include <cstdio>
#include <random>
#include <sstream>

using namespace qmcgpu;
using namespace qmcgpu::host;

namespace qmcgpu {
namespace host {

// build_matrices(builtin_direction_numbers(), dims), built once per dims
// and kept for the process (the reference's builtin_direction_numbers() is
// likewise a function-local static, digitalnet.cpp:73-77).
qmc_matrices* builtin_matrices(uint32_t dims)
{
    static std::mutex mu;
    static std::map<uint32_t, std::unique_ptr<qmc_matrices>> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto& m = cache[dims];
    if (!m) {
        auto cols = build_columns(builtin_rows(), dims); // ConfigError beyond 64
        m = std::make_unique<qmc_matrices>();
        m->dims = dims;
        m->columns = std::move(cols);
    }
    return m.get();
}

void sobol_fill_impl(qmc_matrices* m, uint64_t first, uint64_t n, uint32_t dims,
                     qmc_sobol_scramble sc, const uint32_t* words, qmc_output kind, void* out,
                     cudaStream_t s)
{
    if (!m)
        fail(QMC_INVALID_ARGUMENT, "matrices handle is null");
    if (n == 0 || dims == 0)
        return;
    if (first >= (1ull << 52) || n > (1ull << 52) - first)
        fail(QMC_INVALID_ARGUMENT, "sobol_component: index must be below 2^52");
    if (dims > m->dims)
        fail(QMC_OUT_OF_RANGE, "sobol_component: dimension beyond the matrix set");
    if (sc != QMC_SOBOL_NONE && sc != QMC_SOBOL_XOR && sc != QMC_SOBOL_OWEN)
        fail(QMC_INVALID_ARGUMENT, "sobol_fill: unknown scramble kind");
    // the kernels read dims-strided columns: tables for this dims prefix
    const auto& dev = m->on_device(dims);
    const uint32_t* colsT = static_cast<const uint32_t*>(dev.colsT.get());
    const uint32_t* colsT_rev = static_cast<const uint32_t*>(dev.colsT_rev.get());
    CallArgs args(s);
    SmallArgs small{};
    SmallStage stage;
    if (words && sc != QMC_SOBOL_NONE)
        set_small(small, stage, 0, words, dims, args);
    args.upload();
    finish_small(small, stage, args);
    const int mode = sc == QMC_SOBOL_OWEN ? 2 : 0;
    const bool u32 = kind == QMC_OUT_U32;
    place_fill(out, first, n, dims, s, [&](const FillRange& r, cudaStream_t st) {
        return launch_sobol(colsT, colsT_rev, small, dims, mode, u32, r, st);
    });
}

// white_noise_xor_tables (imageplane.cpp:197-229): std::mt19937 words on the
// host, in the reference's draw order.
std::unique_ptr<qmc_xor_tables> make_white_noise(uint32_t dims, uint32_t point_count,
                                                 uint32_t seed)
{
    if (dims == 0)
        fail(QMC_CONFIG, "white_noise_xor_tables: dims must be >= 1");
    if (point_count == 0 || (point_count & (point_count - 1)) != 0)
        fail(QMC_CONFIG, "white_noise_xor_tables: point count must be a power of two");
    auto t = std::make_unique<qmc_xor_tables>();
    t->dims = dims;
    t->point_count = point_count;
    t->white_noise = true;
    std::mt19937 rng(seed);
    t->dim_scramble.assign(dims, 0u);
    if (seed != 0)
        for (auto& w : t->dim_scramble)
            w = rng();
    t->reorder.resize(kXorTile);
    t->scramble.resize(kXorTile * dims);
    for (auto& v : t->reorder)
        v = rng() & (point_count - 1);
    for (auto& v : t->scramble)
        v = rng();
    return t;
}

XorTablesDev xor_view(const qmc_xor_tables* given, uint32_t dims, uint32_t point_count,
                      uint32_t seed, cudaStream_t s)
{
    XorTablesDev v;
    qmc_xor_tables* t = const_cast<qmc_xor_tables*>(given);
    if (!t) {
        v.own = make_white_noise(dims, point_count, seed);
        t = v.own.get();
    }
    const auto& d = t->on_device(s);
    v.dims = t->dims;
    v.point_count = t->point_count;
    v.reorder = static_cast<const uint32_t*>(d.reorder.get());
    v.scramble = static_cast<const uint32_t*>(d.scramble.get());
    v.points = static_cast<const uint32_t*>(d.points.get());
    return v;
}

} // namespace host
} // namespace qmcgpu

const qmc_xor_tables::Dev& qmc_xor_tables::on_device(cudaStream_t s)
{
    const int d = current_device();
    std::lock_guard<std::mutex> lk(mu);
    auto& slot = dev[d];
    if (!slot) {
        auto e = std::make_unique<Dev>();
        e->reorder = dev_upload(reorder.data(), reorder.size() * 4);
        e->scramble = dev_upload(scramble.data(), scramble.size() * 4);
        if (white_noise) {
            // the first point_count Sobol' points at the integer stage,
            // XOR-scrambled per dimension when seeded (imageplane.cpp:224-227),
            // generated by the device fill
            void* pts = nullptr;
            cuda_ok(cudaMalloc(&pts, static_cast<size_t>(point_count) * dims * 4 + 32),
                    "cudaMalloc");
            e->points.reset(pts);
            const bool scr = std::any_of(dim_scramble.begin(), dim_scramble.end(),
                                         [](uint32_t w) { return w != 0; });
            sobol_fill_impl(builtin_matrices(dims), 0, point_count, dims,
                            scr ? QMC_SOBOL_XOR : QMC_SOBOL_NONE, dim_scramble.data(),
                            QMC_OUT_U32, pts, s);
            cuda_ok(cudaStreamSynchronize(s), "sync");
        } else {
            e->points = dev_upload(points.data(), points.size() * 4);
        }
        slot = std::move(e);
    }
    return *slot;
}

extern "C" {

const char* qmc_last_error(void) { return last_error().c_str(); }

const char* qmc_status_string(qmc_status s)
{
    switch (s) {
    case QMC_OK: return "ok";
    case QMC_CONFIG: return "config error";
    case QMC_INVALID_ARGUMENT: return "invalid argument";
    case QMC_OUT_OF_RANGE: return "out of range";
    case QMC_OVERFLOW: return "overflow";
    case QMC_CUDA: return "cuda error";
    case QMC_NCCL: return "nccl error";
    default: return "internal error";
    }
}

int qmc_abi_version(void) { return QMCGPU_ABI_VERSION; }

// ------------------------------------------------------------------ L0

qmc_status qmc_map_u32_to_unifloat(const uint32_t* in, float* out, uint64_t n, qmc_stream stream)
{
    return guard([&] {
        const NvtxRange nvtx("qmc_map_u32_to_unifloat");
        if (n == 0)
            return;
        const cudaStream_t s = as_stream(stream);
        if (is_device_pointer(in) && is_device_pointer(out)) {
            cuda_ok(launch_map(in, out, n, s), "launch_map");
            return;
        }
        // host arrays: stage through device memory
        uint32_t* din = nullptr;
        float* dout = nullptr;
        cuda_ok(cudaMallocAsync(&din, n * 4, s), "cudaMallocAsync");
        cuda_ok(cudaMallocAsync(&dout, n * 4, s), "cudaMallocAsync");
        cuda_ok(cudaMemcpyAsync(din, in, n * 4, cudaMemcpyDefault, s), "H2D");
        cuda_ok(launch_map(din, dout, n, s), "launch_map");
        cuda_ok(cudaMemcpyAsync(out, dout, n * 4, cudaMemcpyDefault, s), "D2H");
        cudaFreeAsync(din, s);
        cudaFreeAsync(dout, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
    });
}

qmc_status qmc_map_selfcheck(uint64_t* mismatches, qmc_stream stream)
{
    return guard([&] {
        const cudaStream_t s = as_stream(stream);
        unsigned long long* d = nullptr;
        cuda_ok(cudaMallocAsync(&d, 8, s), "cudaMallocAsync");
        cuda_ok(cudaMemsetAsync(d, 0, 8, s), "memset");
        cuda_ok(launch_map_selfcheck(d, s), "launch_map_selfcheck");
        unsigned long long h = 0;
        cuda_ok(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, s), "D2H");
        cudaFreeAsync(d, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
        *mismatches = h;
    });
}

qmc_status qmc_write_probe(void* device_buffer, uint64_t bytes, int mode, qmc_stream stream)
{
    return guard([&] {
        if (!is_device_pointer(device_buffer))
            fail(QMC_INVALID_ARGUMENT, "write probe needs a device buffer");
        cuda_ok(launch_write_probe(device_buffer, bytes & ~uint64_t(31), mode, as_stream(stream)),
                "launch_write_probe");
    });
}

// ------------------------------------------------------------ host setup

qmc_status qmc_prime(uint32_t index, uint32_t* out)
{
    return guard([&] { *out = prime_at(index); });
}

qmc_status qmc_prime_max_power(uint32_t index, uint32_t* out)
{
    return guard([&] {
        if (index >= kPrimes)
            fail(QMC_OUT_OF_RANGE, "prime_max_power: index beyond the bundled prime table");
        *out = primes().maxpow[index];
    });
}

qmc_status qmc_faure_permutation(uint32_t base, uint32_t* out)
{
    return guard([&] {
        const auto s = faure(base);
        std::memcpy(out, s.data(), s.size() * 4);
    });
}

qmc_status qmc_default_linear_factors(uint32_t dims, uint32_t* out)
{
    return guard([&] {
        if (dims > kPrimes)
            fail(QMC_INVALID_ARGUMENT, "default_linear_factors: dims beyond the prime table");
        for (uint32_t j = 0; j < dims; ++j)
            out[j] = primes().p[j] - 1;
    });
}

qmc_status qmc_lfsr_generator_vector(uint32_t seed, uint32_t dims, uint32_t* out)
{
    return guard([&] {
        const auto g = lfsr(seed, dims);
        std::memcpy(out, g.data(), g.size() * 4);
    });
}

uint32_t qmc_pixel_hash(uint32_t j, uint32_t px, uint32_t py) { return pixel_hash_host(j, px, py); }

qmc_status qmc_hilbert_index(uint32_t x, uint32_t y, uint32_t order, uint64_t* out)
{
    return guard([&] {
        if (!out)
            fail(QMC_INVALID_ARGUMENT, "output pointer is null");
        if (order == 0 || order > 31)
            fail(QMC_INVALID_ARGUMENT, "hilbert_index: order must be in [1, 31]");
        if (x >= (1u << order) || y >= (1u << order))
            fail(QMC_OUT_OF_RANGE, "hilbert_index: pixel outside the 2^order grid");
        *out = hilbert_index(x, y, order);
    });
}

qmc_status qmc_hilbert_phi3_fixed(uint32_t x, uint32_t y, uint32_t order, uint32_t* out)
{
    return guard([&] {
        uint64_t h = 0;
        const qmc_status st = qmc_hilbert_index(x, y, order, &h);
        if (st != QMC_OK)
            fail(st, last_error());
        // radical_inverse_tabled_fixed(h, 3, base3_four_digit_table()) ==
        // radical_inverse_fixed(h, 1): i %= 3^20, reversed digits / 3^digits
        uint32_t i = static_cast<uint32_t>(h) % 3486784401u;
        uint64_t acc = 0, scale = 1;
        do {
            acc = acc * 3 + i % 3;
            i /= 3;
            scale *= 3;
        } while (i != 0);
        if (!out)
            fail(QMC_INVALID_ARGUMENT, "output pointer is null");
        *out = static_cast<uint32_t>((acc << 32) / scale);
    });
}

qmc_status qmc_hilbert_xy(uint64_t d, uint32_t order, uint32_t* x, uint32_t* y)
{
    return guard([&] {
        if (!x || !y)
            fail(QMC_INVALID_ARGUMENT, "output pointer is null");
        if (order == 0 || order > 31)
            fail(QMC_INVALID_ARGUMENT, "hilbert_xy: order must be in [1, 31]");
        if (d >= (1ull << (2 * order)))
            fail(QMC_OUT_OF_RANGE, "hilbert_xy: index beyond 4^order");
        hilbert_xy_host(d, order, *x, *y);
    });
}

uint64_t qmc_digit_reverse(uint64_t v, uint32_t base, uint32_t digits)
{
    return base < 2 ? 0 : digit_reverse_host(v, base, digits);
}

qmc_status qmc_lattice_shift_fixed(uint32_t k, uint32_t m, const uint32_t* g, uint32_t dims,
                                   uint32_t* out)
{
    return guard([&] {
        if ((!g || !out) && dims)
            fail(QMC_INVALID_ARGUMENT, "generator or output pointer is null");
        if (m > 32)
            fail(QMC_INVALID_ARGUMENT, "lattice_shift: m must be <= 32");
        const uint64_t scaled = static_cast<uint64_t>(k) << m;
        if (scaled > 0xffffffffull)
            fail(QMC_OVERFLOW, "lattice_shift: k * 2^m does not fit 32 bits");
        const uint32_t rev = brev_host(static_cast<uint32_t>(scaled));
        for (uint32_t j = 0; j < dims; ++j)
            out[j] = rev * g[j];
    });
}

uint32_t qmc_hilbert_order_for(uint32_t width, uint32_t height)
{
    return hilbert_order(width, height);
}

qmc_status qmc_partition_by_extra_dimension(uint32_t part, uint32_t parts, uint32_t base,
                                            uint64_t* remainder, uint64_t* modulus)
{
    return guard([&] {
        if (base < 2)
            fail(QMC_INVALID_ARGUMENT, "partition_by_extra_dimension: base must be >= 2");
        uint32_t k = 0;
        uint64_t p = 1;
        while (p < parts) {
            p *= base;
            ++k;
        }
        if (p != parts)
            fail(QMC_CONFIG, "partition_by_extra_dimension: parts must be a power of the base");
        if (part >= parts)
            fail(QMC_OUT_OF_RANGE, "partition_by_extra_dimension: part index beyond parts");
        *remainder = digit_reverse_host(part, base, k);
        *modulus = parts;
    });
}

qmc_status qmc_halton_pixel_enumeration(uint32_t width, uint32_t height, uint32_t px, uint32_t py,
                                        qmc_halton_enumeration* e, uint64_t* offset)
{
    return guard([&] {
        const HaltonEnum h = halton_enum(width, height);
        if (px >= h.sx || py >= h.sy)
            fail(QMC_OUT_OF_RANGE, "HaltonPixelEnumeration: pixel outside the scaled grid");
        if (e)
            *e = qmc_halton_enumeration{h.sx, h.sy, h.ex, h.ey, h.stride};
        if (offset) {
            const uint64_t r2 = digit_reverse_host(px, 2, h.ex);
            const uint64_t r3 = digit_reverse_host(py, 3, h.ey);
            *offset = (r2 * h.crt_x % h.stride + r3 * h.crt_y % h.stride) % h.stride;
        }
    });
}

// ------------------------------------------------------------- matrices

static qmc_matrices* new_matrices(std::vector<uint32_t> cols, uint32_t dims)
{
    auto* m = new qmc_matrices();
    m->dims = dims;
    m->columns = std::move(cols);
    return m;
}

qmc_status qmc_matrices_builtin(uint32_t dims, qmc_matrices** out)
{
    return guard([&] { *out = new_matrices(build_columns(builtin_rows(), dims), dims); });
}

qmc_status qmc_matrices_from_text(const char* text, uint32_t dims, qmc_matrices** out)
{
    return guard([&] {
        if (!text)
            fail(QMC_INVALID_ARGUMENT, "direction number text is null");
        *out = new_matrices(build_columns(parse_rows(text), dims), dims);
    });
}

qmc_status qmc_matrices_from_columns(const uint32_t* columns, uint32_t dims, qmc_matrices** out)
{
    return guard([&] {
        if (!columns && dims)
            fail(QMC_INVALID_ARGUMENT, "columns pointer is null");
        *out = new_matrices(std::vector<uint32_t>(columns, columns + static_cast<size_t>(dims) * 52),
                            dims);
    });
}

uint32_t qmc_matrices_dims(const qmc_matrices* m) { return m ? m->dims : 0; }

qmc_status qmc_matrices_columns(const qmc_matrices* m, uint32_t* out)
{
    return guard([&] {
        if (!m)
            fail(QMC_INVALID_ARGUMENT, "matrices handle is null");
        std::memcpy(out, m->columns.data(), m->columns.size() * 4);
    });
}

void qmc_matrices_destroy(qmc_matrices* m) { delete m; }

// ----------------------------------------------------------------- fills

qmc_status qmc_sobol_fill(const qmc_matrices* m, uint64_t first_index, uint64_t n, uint32_t dims,
                          qmc_sobol_scramble scramble, const uint32_t* words, qmc_output kind,
                          void* out, qmc_stream stream)
{
    return guard([&] {
        const NvtxRange nvtx("qmc_sobol_fill");
        sobol_fill_impl(const_cast<qmc_matrices*>(m), first_index, n, dims, scramble, words, kind,
                        out, as_stream(stream));
    });
}

static void halton_fill_impl(uint64_t first, uint64_t n, uint32_t dims, uint32_t first_prime,
                             qmc_radical_scramble sc, const uint32_t* factors, qmc_output kind,
                             void* out, cudaStream_t s)
{
    if (sc != QMC_RADICAL_PLAIN && sc != QMC_RADICAL_LINEAR && sc != QMC_RADICAL_FAURE)
        fail(QMC_INVALID_ARGUMENT, "halton: unknown scramble kind");
    const bool u32 = kind == QMC_OUT_U32;
    if (dims == 1 && first_prime == 0) { // van der Corput: every scramble is the identity
        if (sc == QMC_RADICAL_LINEAR && factors && factors[0] != 1)
            fail(QMC_INVALID_ARGUMENT, "radical_inverse_linscramble: factor must be in [1, base)");
        place_fill(out, first, n, 1, s, [&](const FillRange& r, cudaStream_t st) {
            return launch_vdc(u32, r, st);
        });
        return;
    }
    std::vector<uint32_t> pool;
    std::vector<size_t> soff;
    auto rd = radical_dims(dims, first_prime, sc, factors, pool, soff);
    if (n == 0 || dims == 0)
        return;
    CallArgs pargs(s);
    pool.push_back(0u); // never empty
    pargs.add(pool.data(), pool.size() * 4);
    pargs.upload();
    const uint32_t* pool_dev = pargs.at<uint32_t>(0);
    for (size_t j = 0; j < rd.size(); ++j)
        if (soff[j] != SIZE_MAX)
            rd[j].sigma = pool_dev + soff[j];
    CallArgs args(s);
    const size_t off = args.add(rd.data(), rd.size() * sizeof(RadicalDim));
    args.upload();
    const RadicalDim* rdev = args.at<RadicalDim>(off);
    place_fill(out, first, n, dims, s, [&](const FillRange& r, cudaStream_t st) {
        return launch_halton(rdev, dims, u32, r, st, rd.data());
    });
}

qmc_status qmc_halton_fill(uint64_t first_index, uint64_t n, uint32_t dims,
                           qmc_radical_scramble scramble, const uint32_t* factors,
                           qmc_output kind, void* out, qmc_stream stream)
{
    return guard([&] {
        const NvtxRange nvtx("qmc_halton_fill");
        if (dims > kPrimes)
            fail(QMC_INVALID_ARGUMENT, "halton_point: dims beyond the prime table");
        halton_fill_impl(first_index, n, dims, 0, scramble, factors, kind, out,
                         as_stream(stream));
    });
}

qmc_status qmc_radical_inverse_fill(uint64_t first_index, uint64_t n, uint32_t prime_index,
                                    qmc_radical_scramble scramble, uint32_t factor,
                                    qmc_output kind, void* out, qmc_stream stream)
{
    return guard([&] {
        const NvtxRange nvtx("qmc_radical_inverse_fill");
        prime_at(prime_index); // out_of_range like prime()
        halton_fill_impl(first_index, n, 1, prime_index, scramble, &factor, kind, out,
                         as_stream(stream));
    });
}

static void lattice_fill_impl(const uint32_t* g, const uint32_t* shifts, uint32_t dims,
                              uint64_t first, uint64_t n, qmc_output kind, void* out,
                              cudaStream_t s)
{
    if (n == 0 || dims == 0)
        return;
    if (!g)
        fail(QMC_INVALID_ARGUMENT, "generator vector is null");
    CallArgs args(s);
    SmallArgs small{};
    SmallStage stage;
    set_small(small, stage, 0, g, dims, args);
    if (shifts)
        set_small(small, stage, 1, shifts, dims, args);
    args.upload();
    finish_small(small, stage, args);
    const bool u32 = kind == QMC_OUT_U32;
    place_fill(out, first, n, dims, s, [&](const FillRange& r, cudaStream_t st) {
        return launch_lattice(small, dims, u32, r, st);
    });
}

qmc_status qmc_lattice_fill(const uint32_t* g, const uint32_t* shifts, uint32_t dims,
                            uint64_t first_index, uint64_t n, qmc_output kind, void* out,
                            qmc_stream stream)
{
    return guard([&] {
        const NvtxRange nvtx("qmc_lattice_fill");
        lattice_fill_impl(g, shifts, dims, first_index, n, kind, out, as_stream(stream));
    });
}

// ------------------------------------------------------ SampleStream façade

static const char* const kKindNames[] = {"sobol",
                                         "halton",
                                         "lattice",
                                         "halton-hilbert",
                                         "pixel-shifted-lattice",
                                         "pixel-random-lattice",
                                         "image-plane-halton",
                                         "sobol-xor-table"};

qmc_status qmc_sampler_kind_from_name(const char* name, qmc_sampler_kind* out)
{
    return guard([&] {
        const std::string n = name ? name : "";
        for (int k = 0; k < 8; ++k)
            if (n == kKindNames[k]) {
                *out = static_cast<qmc_sampler_kind>(k);
                return;
            }
        fail(QMC_CONFIG, "unknown sampler: " + n);
    });
}

const char* qmc_sampler_kind_name(qmc_sampler_kind kind)
{
    return (kind >= 0 && kind < 8) ? kKindNames[kind] : "";
}

namespace {

// make_stream (imageplane.cpp:310-416) for one pixel context: validates the
// parameters with the reference's ConfigError conditions and resolves the
// device-side state the kernels read. Owns every device resource until it
// goes out of scope (callers synchronize before that).
struct ResolvedStream {
    PixelStreamParams q{};
    std::unique_ptr<qmc_matrices> own_matrices;
    qmc_matrices* matrices = nullptr; // sobol
    std::vector<uint32_t> sobol_words; // sobol scrambles (may be empty)
    XorTablesDev xt;
    std::vector<uint32_t> pool;
    std::vector<size_t> soff;
    std::vector<RadicalDim> rd;
    size_t goff = SIZE_MAX, roff = SIZE_MAX, woff = SIZE_MAX;
    qmc_radical_scramble halton_sc = QMC_RADICAL_PLAIN;
};

void resolve_stream(qmc_sampler_kind kind, const qmc_stream_params* p, cudaStream_t s,
                    ResolvedStream& r, CallArgs& args, CallArgs& pargs)
{
    if (!p)
        fail(QMC_INVALID_ARGUMENT, "stream params are null");
    if (kind < 0 || kind > 7)
        fail(QMC_CONFIG, "unknown sampler kind");
    require(p->dims >= 1, "make_stream: dims must be >= 1");
    const uint32_t dims = p->dims;
    auto halton_scramble = [&]() -> qmc_radical_scramble {
        if (p->halton_scramble > 2)
            fail(QMC_CONFIG, "make_stream: scramble must be plain, faure, or linear");
        if (p->halton_scramble == QMC_RADICAL_LINEAR && p->linear_factors)
            require(p->linear_factors_len >= dims,
                    "make_stream: linear factor list shorter than dims");
        return static_cast<qmc_radical_scramble>(p->halton_scramble);
    };
    auto lattice_vector = [&]() {
        require(p->generator && p->generator_dims > 0, "make_stream: generator vector required");
        for (uint32_t j = 0; j < p->generator_dims; ++j)
            require(p->generator[j] & 1u, "make_stream: generator components must be odd");
        require(dims <= p->generator_dims, "make_stream: dims beyond the generator vector");
        r.goff = args.add(p->generator, dims * 4);
    };
    auto validate_pixel = [&]() {
        require(p->order >= 1 && p->order <= 31, "make_stream: pixel order must be in [1, 31]");
        require(p->px < (1u << p->order) && p->py < (1u << p->order),
                "make_stream: pixel outside the 2^order grid");
    };
    PixelStreamParams& q = r.q;
    q.tab3 = digit_table(3, 0, 0).ptr;
    q.kind = kind;
    q.dims = dims;
    q.px = p->px;
    q.py = p->py;
    q.order = p->order;
    q.spp = p->spp;
    q.width = p->width;
    q.height = p->height;
    switch (kind) {
    case QMC_KIND_SOBOL:
        r.matrices = const_cast<qmc_matrices*>(p->matrices);
        if (!r.matrices)
            r.matrices = builtin_matrices(dims);
        require(dims <= r.matrices->dims, "make_stream: dims beyond the generator matrices");
        if (p->sobol_scrambles) {
            require(p->sobol_scrambles_len >= dims, "make_stream: scramble list shorter than dims");
            r.sobol_words.assign(p->sobol_scrambles, p->sobol_scrambles + dims);
            r.woff = args.add(r.sobol_words.data(), dims * 4);
        }
        break;
    case QMC_KIND_HALTON:
        require(dims <= kPrimes, "make_stream: dims beyond the prime table");
        r.halton_sc = halton_scramble();
        r.rd = radical_dims(dims, 0, r.halton_sc, p->linear_factors, r.pool, r.soff);
        break;
    case QMC_KIND_LATTICE:
        lattice_vector();
        break;
    case QMC_KIND_HALTON_HILBERT:
        require(p->spp >= 1, "make_stream: spp must be >= 1");
        validate_pixel();
        require(dims <= kPrimes, "halton_point: dims beyond the prime table");
        r.rd = radical_dims(dims, 0, halton_scramble(), p->linear_factors, r.pool, r.soff);
        break;
    case QMC_KIND_PIXEL_SHIFTED_LATTICE:
        validate_pixel();
        lattice_vector();
        break;
    case QMC_KIND_PIXEL_RANDOM_LATTICE:
        break;
    case QMC_KIND_IMAGE_PLANE_HALTON: {
        require(p->width >= 1 && p->height >= 1,
                "make_stream: image size required for image-plane halton");
        require(p->px < p->width && p->py < p->height, "make_stream: pixel outside the image");
        require(dims <= kPrimes, "make_stream: dims beyond the prime table");
        const HaltonEnum e = halton_enum(p->width, p->height);
        if (p->linear_factors)
            require(p->linear_factors_len >= dims,
                    "make_stream: linear factor list shorter than dims");
        r.rd = radical_dims(dims, 0, QMC_RADICAL_LINEAR, p->linear_factors, r.pool, r.soff);
        q.scale_x = e.sx;
        q.scale_y = e.sy;
        q.exp_x = e.ex;
        q.exp_y = e.ey;
        q.stride = e.stride;
        q.crt_x = e.crt_x;
        q.crt_y = e.crt_y;
        break;
    }
    case QMC_KIND_SOBOL_XOR_TABLE: {
        r.xt = xor_view(p->xor_tables, dims, p->xor_point_count, p->xor_seed, s);
        require(dims <= r.xt.dims, "make_stream: dims beyond the stored point set");
        q.xor_reorder = r.xt.reorder;
        q.xor_scramble = r.xt.scramble;
        q.xor_points = r.xt.points;
        q.xor_point_count = r.xt.point_count;
        q.xor_dims = r.xt.dims;
        break;
    }
    }
    // radical tables: the permutation pool goes first (its device address is
    // patched into the RadicalDim records), then everything else
    if (!r.rd.empty()) {
        r.pool.push_back(0u); // never empty
        pargs.add(r.pool.data(), r.pool.size() * 4);
        pargs.upload();
        const uint32_t* pool_dev = pargs.at<uint32_t>(0);
        for (size_t j = 0; j < r.rd.size(); ++j)
            if (r.soff[j] != SIZE_MAX)
                r.rd[j].sigma = pool_dev + r.soff[j];
        r.roff = args.add(r.rd.data(), r.rd.size() * sizeof(RadicalDim));
    }
    args.upload();
    if (r.goff != SIZE_MAX)
        q.generator = args.at<uint32_t>(r.goff);
    if (r.roff != SIZE_MAX)
        q.radical_dims = args.at<RadicalDim>(r.roff);
}

} // namespace

qmc_status qmc_stream_fill(qmc_sampler_kind kind, const qmc_stream_params* p,
                           uint64_t first_index, uint64_t n, qmc_output out_kind, void* out,
                           qmc_stream stream)
{
    return guard([&] {
        const NvtxRange nvtx("qmc_stream_fill");
        const cudaStream_t s = as_stream(stream);
        if (!p)
            fail(QMC_INVALID_ARGUMENT, "stream params are null");
        const uint32_t dims = p->dims;
        // the non-pixel kinds are the batched fills
        if (kind == QMC_KIND_SOBOL || kind == QMC_KIND_HALTON || kind == QMC_KIND_LATTICE) {
            CallArgs args(s), pargs(s);
            ResolvedStream r;
            resolve_stream(kind, p, s, r, args, pargs);
            if (kind == QMC_KIND_SOBOL) {
                sobol_fill_impl(r.matrices, first_index, n, dims,
                                r.sobol_words.empty() ? QMC_SOBOL_NONE : QMC_SOBOL_XOR,
                                r.sobol_words.empty() ? nullptr : r.sobol_words.data(), out_kind,
                                out, s);
            } else if (kind == QMC_KIND_HALTON) {
                // SampleStream::sample casts the index to 32 bits (the kernel wraps too)
                halton_fill_impl(first_index, n, dims, 0, r.halton_sc, p->linear_factors,
                                 out_kind, out, s);
            } else {
                lattice_fill_impl(p->generator, nullptr, dims, first_index, n, out_kind, out, s);
            }
            cuda_ok(cudaStreamSynchronize(s), "sync");
            return;
        }
        CallArgs args(s), pargs(s);
        ResolvedStream r;
        resolve_stream(kind, p, s, r, args, pargs);
        if (kind == QMC_KIND_HALTON_HILBERT && (first_index >= p->spp || n > p->spp - first_index))
            fail(QMC_OUT_OF_RANGE, "SampleStream: sample index beyond the pixel block");
        if (kind == QMC_KIND_SOBOL_XOR_TABLE &&
            (first_index >= r.q.xor_point_count || n > r.q.xor_point_count - first_index))
            fail(QMC_OUT_OF_RANGE, "xor_table_sample: index beyond the stored point set");
        if (n == 0)
            return;
        if (kind == QMC_KIND_PIXEL_SHIFTED_LATTICE) {
            // (brev(i) + shift) * g_j == brev(i) * g_j + shift * g_j (mod 2^32):
            // the pixel's stream is the CP-rotated lattice with integer
            // shifts s_j = shift * g_j (imageplane.hpp:26-31), so it takes
            // the HBM-bound lattice fill
            uint32_t shift = 0;
            const qmc_status st = qmc_hilbert_phi3_fixed(p->px, p->py, p->order, &shift);
            if (st != QMC_OK)
                fail(st, last_error());
            std::vector<uint32_t> sh(dims);
            for (uint32_t j = 0; j < dims; ++j)
                sh[j] = shift * p->generator[j];
            lattice_fill_impl(p->generator, sh.data(), dims, first_index, n, out_kind, out, s);
            cuda_ok(cudaStreamSynchronize(s), "sync");
            return;
        }
        if (kind == QMC_KIND_HALTON_HILBERT) {
            // sample(i, j) = halton_component(u32(block_start + i), j)
            // (imageplane.cpp:378, :439-442): the contiguous Halton fill
            const uint64_t block = hilbert_index(p->px, p->py, p->order) * p->spp;
            halton_fill_impl(block + first_index, n, dims, 0,
                             static_cast<qmc_radical_scramble>(p->halton_scramble),
                             p->linear_factors, out_kind, out, s);
            cuda_ok(cudaStreamSynchronize(s), "sync");
            return;
        }
        const bool u32 = out_kind == QMC_OUT_U32;
        place_fill(out, first_index, n, dims, s, [&](const FillRange& fr, cudaStream_t st) {
            return launch_pixel_stream(r.q, u32, fr, st);
        });
        cuda_ok(cudaStreamSynchronize(s), "sync"); // tables owned by this call
    });
}

// --------------------------------------------------------------- integrate

static const char* const kIntegrandNames[] = {"product-sine", "product-poly", "indicator"};

qmc_status qmc_builtin_integrand(const char* name, uint32_t dims, qmc_integrand_kind* kind,
                                 double* exact_integral)
{
    return guard([&] {
        if (dims == 0)
            fail(QMC_INVALID_ARGUMENT, "builtin_integrands: dims must be >= 1");
        const std::string n = name ? name : "";
        for (int k = 0; k < 3; ++k)
            if (n == kIntegrandNames[k]) {
                if (kind)
                    *kind = static_cast<qmc_integrand_kind>(k);
                if (exact_integral) // quality.cpp:38-66
                    *exact_integral = k == 2 ? std::pow(0.7, static_cast<double>(dims)) : 1.0;
                return;
            }
        fail(QMC_CONFIG, "unknown integrand: " + n);
    });
}

} // extern "C"

namespace {

// integrate() (quality.cpp:214-282) over the 4096-index chunks [c0, c1) of
// [0, n): validation with the reference's conditions, one launch, and the
// per-chunk Kahan partials (kahan mode) or the exact int64 sum (int mode).
void integrate_chunks(qmc_sampler_kind kind, const qmc_stream_params* p, qmc_integrand_kind f,
                      uint32_t f_dims, uint64_t n, uint64_t c0, uint64_t c1, qmc_accum mode,
                      cudaStream_t s, std::vector<double>& partials, long long& isum)
{
    if (f < 0 || f > 2)
        fail(QMC_CONFIG, "unknown integrand");
    if (f_dims == 0)
        fail(QMC_INVALID_ARGUMENT, "builtin_integrands: dims must be >= 1");
    if (mode != QMC_ACCUM_KAHAN && mode != QMC_ACCUM_INT)
        fail(QMC_CONFIG, "accumulation mode must be 'kahan' or 'int'");
    if (n == 0)
        fail(QMC_INVALID_ARGUMENT, "integrate: n must be >= 1");
    if (!p)
        fail(QMC_INVALID_ARGUMENT, "stream params are null");
    if (p->dims < f_dims)
        fail(QMC_INVALID_ARGUMENT, "integrate: stream has fewer dimensions than the integrand");
    const uint64_t chunks = (n + 4095) / 4096;
    if (c0 > c1 || c1 > chunks)
        fail(QMC_OUT_OF_RANGE, "integrate: chunk range outside [0, ceil(n / 4096))");
    CallArgs args(s), pargs(s);
    ResolvedStream r;
    resolve_stream(kind, p, s, r, args, pargs);
    // sample-time preconditions of SampleStream::sample over [0, n)
    if (kind == QMC_KIND_SOBOL && n > (1ull << 52))
        fail(QMC_INVALID_ARGUMENT, "sobol_component: index must be below 2^52");
    if (kind == QMC_KIND_HALTON_HILBERT && n > p->spp)
        fail(QMC_OUT_OF_RANGE, "SampleStream: sample index beyond the pixel block");
    if (kind == QMC_KIND_SOBOL_XOR_TABLE && n > r.q.xor_point_count)
        fail(QMC_OUT_OF_RANGE, "xor_table_sample: index beyond the stored point set");
    if (kind == QMC_KIND_HALTON || kind == QMC_KIND_HALTON_HILBERT ||
        kind == QMC_KIND_IMAGE_PLANE_HALTON)
        for (const RadicalDim& d : r.rd)
            if (d.mode == 1 && (d.factor == 0 || d.factor >= d.base))
                fail(QMC_INVALID_ARGUMENT,
                     "radical_inverse_linscramble: factor must be in [1, base)");

    const uint32_t dims_of_integrand = p->dims; // stream dims (>= f_dims)
    IntegrateParams ip{};
    ip.pix = r.q;
    ip.fn = f;
    ip.fdims = f_dims;
    ip.n = n;
    ip.sc = make_scene_consts();
    ip.chunk0 = c0;
    ip.nchunks = c1 - c0;
    if (kind == QMC_KIND_SOBOL) {
        const auto& dev = r.matrices->on_device(dims_of_integrand);
        ip.colsT = static_cast<const uint32_t*>(dev.colsT.get());
        ip.mdims = dims_of_integrand;
        ip.words = r.woff == SIZE_MAX ? nullptr : args.at<uint32_t>(r.woff);
    }
    const uint64_t nc = c1 - c0;
    double* partial = nullptr;
    unsigned long long* scal = nullptr; // [0] int sum, [1] first bad index
    cuda_ok(cudaMallocAsync(&partial, nc * 8 + 8, s), "cudaMallocAsync");
    cuda_ok(cudaMallocAsync(&scal, 16, s), "cudaMallocAsync");
    const unsigned long long init[2] = {0ull, ~0ull};
    cuda_ok(cudaMemcpyAsync(scal, init, 16, cudaMemcpyHostToDevice, s), "H2D");
    cuda_ok(launch_integrate(ip, mode, partial, scal, scal + 1, s), "launch_integrate");
    partials.assign(mode == QMC_ACCUM_KAHAN ? nc : 0, 0.0);
    unsigned long long hs[2] = {0, 0};
    if (!partials.empty())
        cuda_ok(cudaMemcpyAsync(partials.data(), partial, nc * 8, cudaMemcpyDeviceToHost, s),
                "D2H");
    cuda_ok(cudaMemcpyAsync(hs, scal, 16, cudaMemcpyDeviceToHost, s), "D2H");
    cudaFreeAsync(partial, s);
    cudaFreeAsync(scal, s);
    cuda_ok(cudaStreamSynchronize(s), "sync");
    if (hs[1] != ~0ull)
        fail(QMC_INTERNAL, std::string("integrate: non-finite value of '") + kIntegrandNames[f] +
                               "' at index " + std::to_string(hs[1]));
    isum = static_cast<long long>(hs[0]);
}

// CompensatedSum (quality.hpp:18-33) over values in the given order.
double compensated_sum(const double* v, uint64_t count)
{
    double sum = 0.0, comp = 0.0;
    for (uint64_t k = 0; k < count; ++k) {
        const double t = sum + v[k];
        if (std::fabs(sum) >= std::fabs(v[k]))
            comp += (sum - t) + v[k];
        else
            comp += (v[k] - t) + sum;
        sum = t;
    }
    return sum + comp;
}

} // namespace

extern "C" {

qmc_status qmc_integrate(qmc_sampler_kind kind, const qmc_stream_params* p,
                         qmc_integrand_kind f, uint32_t f_dims, uint64_t n, qmc_accum mode,
                         qmc_integration_row* row, qmc_stream stream)
{
    return guard([&] {
        const NvtxRange nvtx("qmc_integrate");
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<double> partials;
        long long isum = 0;
        integrate_chunks(kind, p, f, f_dims, n, 0, (n + 4095) / 4096, mode, as_stream(stream),
                         partials, isum);
        // rank-ordered CompensatedSum of the chunk partials (quality.cpp:262-267),
        // or the exact 64-bit sum (quality.cpp:268-272)
        const double estimate =
            mode == QMC_ACCUM_KAHAN
                ? compensated_sum(partials.data(), partials.size()) / static_cast<double>(n)
                : static_cast<double>(isum) / 4294967296.0 / static_cast<double>(n);
        double exact = 1.0;
        qmc_builtin_integrand(kIntegrandNames[f], f_dims, nullptr, &exact);
        if (row) {
            row->n = n;
            row->estimate = estimate;
            row->abs_error = std::fabs(estimate - exact);
            row->seconds =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
    });
}

qmc_status qmc_integrate_partials(qmc_sampler_kind kind, const qmc_stream_params* p,
                                  qmc_integrand_kind f, uint32_t f_dims, uint64_t n,
                                  uint64_t chunk_begin, uint64_t chunk_end, qmc_accum mode,
                                  double* partials, int64_t* int_sum, qmc_stream stream)
{
    return guard([&] {
        const NvtxRange nvtx("qmc_integrate_partials");
        if (mode == QMC_ACCUM_KAHAN && !partials && chunk_end > chunk_begin)
            fail(QMC_INVALID_ARGUMENT, "partials pointer is null");
        if (mode == QMC_ACCUM_INT && !int_sum)
            fail(QMC_INVALID_ARGUMENT, "int_sum pointer is null");
        std::vector<double> hp;
        long long isum = 0;
        integrate_chunks(kind, p, f, f_dims, n, chunk_begin, chunk_end, mode, as_stream(stream),
                         hp, isum);
        if (mode == QMC_ACCUM_KAHAN)
            std::memcpy(partials, hp.data(), hp.size() * 8);
        else
            *int_sum = isum;
    });
}

qmc_status qmc_reduce_deterministic(const uint64_t* ranks, const double* values, uint64_t count,
                                    double* out)
{
    return guard([&] {
        if (!out || (count && (!ranks || !values)))
            fail(QMC_INVALID_ARGUMENT, "null pointer");
        std::vector<uint64_t> order(count);
        for (uint64_t k = 0; k < count; ++k)
            order[k] = k;
        std::stable_sort(order.begin(), order.end(),
                         [&](uint64_t a, uint64_t b) { return ranks[a] < ranks[b]; });
        std::vector<double> v(count);
        for (uint64_t k = 0; k < count; ++k)
            v[k] = values[order[k]];
        *out = compensated_sum(v.data(), count);
    });
}

// --------------------------------------------------------------- XOR tables

qmc_status qmc_xor_tables_white_noise(uint32_t dims, uint32_t point_count, uint32_t seed,
                                      qmc_xor_tables** out)
{
    return guard([&] { *out = make_white_noise(dims, point_count, seed).release(); });
}

// load_xor_tables (imageplane.cpp:163-195): "XQT1", 128^2 reorder words (used
// modulo point_count), then 128^2 * dims scramble words, little-endian.
qmc_status qmc_xor_tables_load(const void* bytes, size_t len, uint32_t dims,
                               const uint32_t* points, uint32_t point_count,
                               qmc_xor_tables** out)
{
    return guard([&] {
        if (dims == 0)
            fail(QMC_CONFIG, "load_xor_tables: dims must be >= 1");
        if (point_count == 0 || (point_count & (point_count - 1)) != 0)
            fail(QMC_CONFIG, "load_xor_tables: point count must be a power of two");
        if (!points)
            fail(QMC_CONFIG, "load_xor_tables: point set size does not match point_count * dims");
        const unsigned char* b = static_cast<const unsigned char*>(bytes);
        if (!b || len < 4 || std::memcmp(b, "XQT1", 4) != 0)
            fail(QMC_CONFIG, "xor table file: bad magic, expected XQT1");
        size_t pos = 4;
        auto word = [&]() -> uint32_t {
            if (pos + 4 > len)
                fail(QMC_CONFIG, "xor table file: truncated");
            const uint32_t v = static_cast<uint32_t>(b[pos]) | (static_cast<uint32_t>(b[pos + 1]) << 8) |
                               (static_cast<uint32_t>(b[pos + 2]) << 16) |
                               (static_cast<uint32_t>(b[pos + 3]) << 24);
            pos += 4;
            return v;
        };
        auto t = std::make_unique<qmc_xor_tables>();
        t->dims = dims;
        t->point_count = point_count;
        t->reorder.resize(kXorTile);
        for (auto& v : t->reorder)
            v = word() & (point_count - 1);
        t->scramble.resize(kXorTile * dims);
        for (auto& v : t->scramble)
            v = word();
        t->points.assign(points, points + static_cast<size_t>(point_count) * dims);
        *out = t.release();
    });
}

// write_xor_table_file (imageplane.cpp:154-161).
qmc_status qmc_xor_tables_write(const qmc_xor_tables* t, void* bytes, size_t* len)
{
    return guard([&] {
        if (!t || !len)
            fail(QMC_INVALID_ARGUMENT, "xor tables: null argument");
        const size_t need = 4 + 4 * (t->reorder.size() + t->scramble.size());
        if (!bytes || *len < need) {
            *len = need;
            if (bytes)
                fail(QMC_INVALID_ARGUMENT, "xor tables: output buffer too small");
            return;
        }
        unsigned char* o = static_cast<unsigned char*>(bytes);
        std::memcpy(o, "XQT1", 4);
        size_t pos = 4;
        auto put = [&](uint32_t v) {
            o[pos] = v & 0xff;
            o[pos + 1] = (v >> 8) & 0xff;
            o[pos + 2] = (v >> 16) & 0xff;
            o[pos + 3] = (v >> 24) & 0xff;
            pos += 4;
        };
        for (uint32_t v : t->reorder)
            put(v);
        for (uint32_t v : t->scramble)
            put(v);
        *len = need;
    });
}

uint32_t qmc_xor_tables_dims(const qmc_xor_tables* t) { return t ? t->dims : 0; }
uint32_t qmc_xor_tables_point_count(const qmc_xor_tables* t) { return t ? t->point_count : 0; }
void qmc_xor_tables_destroy(qmc_xor_tables* t) { delete t; }

// ------------------------------------------------------------ quality metrics

namespace {

double pairwise_metric(const float* points, uint64_t n, uint32_t dims, cudaStream_t s, bool l2)
{
    if (dims > quality_max_dims())
        fail(QMC_INVALID_ARGUMENT, "quality metric: at most 256 dimensions on the device");
    if (n > 0x7fffffffull)
        fail(QMC_INVALID_ARGUMENT, "quality metric: at most 2^31 - 1 points");
    pool_keep_memory();
    DevPoints dp(points, n * dims, s);
    double* scratch = nullptr;
    cuda_ok(cudaMallocAsync(&scratch, (2 * n + 1) * 8, s), "cudaMallocAsync");
    cuda_ok(l2 ? launch_l2star(dp.ptr, n, dims, scratch + 1, scratch, s)
               : launch_mindist(dp.ptr, n, dims, scratch + 1, scratch, s),
            "launch quality");
    double r = 0.0;
    cuda_ok(cudaMemcpyAsync(&r, scratch, 8, cudaMemcpyDeviceToHost, s), "D2H");
    cudaFreeAsync(scratch, s);
    cuda_ok(cudaStreamSynchronize(s), "sync");
    return r;
}

} // namespace

qmc_status qmc_l2_star_discrepancy(const float* points, uint64_t n, uint32_t dims, double* out,
                                   qmc_stream stream)
{
    return guard([&] {
        const NvtxRange nvtx("qmc_l2_star_discrepancy");
        if (n == 0 || dims == 0)
            fail(QMC_INVALID_ARGUMENT, "l2_star_discrepancy: empty point set");
        if (!points || !out)
            fail(QMC_INVALID_ARGUMENT, "l2_star_discrepancy: null pointer");
        *out = pairwise_metric(points, n, dims, as_stream(stream), true);
    });
}

qmc_status qmc_min_toroidal_distance(const float* points, uint64_t n, uint32_t dims, double* out,
                                     qmc_stream stream)
{
    return guard([&] {
        const NvtxRange nvtx("qmc_min_toroidal_distance");
        if (n < 2)
            fail(QMC_INVALID_ARGUMENT, "min_toroidal_distance: need at least two points");
        if (!points || !out)
            fail(QMC_INVALID_ARGUMENT, "min_toroidal_distance: null pointer");
        *out = pairwise_metric(points, n, dims, as_stream(stream), false);
    });
}

qmc_status qmc_check_1d_stratification(qmc_sampler_kind kind, const qmc_stream_params* params,
                                       uint32_t j, uint32_t m, int* ok, uint32_t* histogram,
                                       qmc_stream stream)
{
    return guard([&] {
        if (m > 20)
            fail(QMC_INVALID_ARGUMENT, "check_1d_stratification: m must be <= 20");
        if (!params)
            fail(QMC_INVALID_ARGUMENT, "stream params are null");
        if (j >= params->dims)
            fail(QMC_OUT_OF_RANGE, "SampleStream: dimension beyond the stream");
        const cudaStream_t s = as_stream(stream);
        pool_keep_memory();
        const uint32_t count = 1u << m;
        float* pts = nullptr;
        uint32_t* hist = nullptr;
        unsigned int* bad = nullptr;
        cuda_ok(cudaMallocAsync(&pts, static_cast<size_t>(count) * params->dims * 4 + 32, s),
                "cudaMallocAsync");
        cuda_ok(cudaMallocAsync(&hist, static_cast<size_t>(count) * 4 + 4, s), "cudaMallocAsync");
        cuda_ok(cudaMemsetAsync(hist, 0, static_cast<size_t>(count) * 4 + 4, s), "memset");
        const qmc_status st = qmc_stream_fill(kind, params, 0, count, QMC_OUT_F32, pts, stream);
        if (st != QMC_OK) {
            cudaFreeAsync(pts, s);
            cudaFreeAsync(hist, s);
            fail(st, last_error());
        }
        bad = reinterpret_cast<unsigned int*>(hist + count);
        cuda_ok(launch_stratification(pts, m, params->dims, j, hist, bad, s), "launch");
        unsigned int hbad = 0;
        cuda_ok(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, s), "D2H");
        if (histogram)
            cuda_ok(cudaMemcpyAsync(histogram, hist, static_cast<size_t>(count) * 4,
                                    cudaMemcpyDeviceToHost, s),
                    "D2H");
        cudaFreeAsync(pts, s);
        cudaFreeAsync(hist, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
        *ok = hbad == 0;
    });
}

// ------------------------------------------------------------------ formats

// load_generator_vector (lattice.cpp:21-46): one decimal component per line,
// '#' comments; ConfigError for components beyond 32 bits, even components,
// or an empty file.
qmc_status qmc_load_generator_vector(const char* text, uint32_t* out, uint32_t capacity,
                                     uint32_t* dims)
{
    return guard([&] {
        if (!text || !dims)
            fail(QMC_INVALID_ARGUMENT, "load_generator_vector: null argument");
        std::istringstream in(text);
        std::string line;
        size_t no = 0;
        std::vector<uint32_t> g;
        while (std::getline(in, line)) {
            ++no;
            const auto hash = line.find('#');
            if (hash != std::string::npos)
                line.erase(hash);
            std::istringstream ls(line);
            uint64_t v = 0;
            if (!(ls >> v))
                continue;
            if (v > 0xffffffffull)
                fail(QMC_CONFIG, "generator vector, line " + std::to_string(no) +
                                     ": component beyond 32 bits");
            if (v % 2 == 0)
                fail(QMC_CONFIG,
                     "generator vector, line " + std::to_string(no) + ": component is even");
            g.push_back(static_cast<uint32_t>(v));
        }
        if (g.empty())
            fail(QMC_CONFIG, "generator vector file holds no components");
        *dims = static_cast<uint32_t>(g.size());
        if (out) {
            if (capacity < g.size())
                fail(QMC_INVALID_ARGUMENT, "load_generator_vector: output capacity too small");
            std::memcpy(out, g.data(), g.size() * 4);
        }
    });
}

// load_linear_factors (radical.cpp:281-306): "base factor" lines override the
// default factor (base - 1) of the matching prime among the first dims.
qmc_status qmc_load_linear_factors(const char* text, uint32_t dims, uint32_t* out)
{
    return guard([&] {
        if (!text || !out)
            fail(QMC_INVALID_ARGUMENT, "load_linear_factors: null argument");
        if (dims > kPrimes)
            fail(QMC_INVALID_ARGUMENT, "default_linear_factors: dims beyond the prime table");
        std::vector<uint32_t> f(dims);
        for (uint32_t j = 0; j < dims; ++j)
            f[j] = primes().p[j] - 1;
        std::istringstream in(text);
        std::string line;
        size_t no = 0;
        while (std::getline(in, line)) {
            ++no;
            const auto hash = line.find('#');
            if (hash != std::string::npos)
                line.erase(hash);
            std::istringstream ls(line);
            uint64_t base = 0, factor = 0;
            if (!(ls >> base))
                continue;
            if (!(ls >> factor))
                fail(QMC_CONFIG, "scramble factor file, line " + std::to_string(no) +
                                     ": expected 'base factor'");
            if (base < 2 || factor == 0 || factor >= base)
                fail(QMC_CONFIG, "scramble factor file, line " + std::to_string(no) +
                                     ": factor must be in [1, base)");
            for (uint32_t j = 0; j < dims; ++j)
                if (primes().p[j] == base)
                    f[j] = static_cast<uint32_t>(factor);
        }
        std::memcpy(out, f.data(), f.size() * 4);
    });
}

// fnv1a64 (image.cpp:54-63) — checksum of serialized output.
uint64_t qmc_fnv1a64(const void* data, uint64_t size)
{
    const unsigned char* p = static_cast<const unsigned char*>(data);
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t k = 0; k < size; ++k) {
        h ^= p[k];
        h *= 0x100000001b3ull;
    }
    return h;
}

// `qmckit points --format csv` rows (qmckit.cpp:225-235): "%.9f" per
// component, comma-separated, one line per point. Host formatting of a
// device or host float array; bytes = NULL queries the size.
qmc_status qmc_write_points_csv(const float* points, uint64_t n, uint32_t dims, void* bytes,
                                size_t* len, qmc_stream stream)
{
    return guard([&] {
        if (!len || (!points && n))
            fail(QMC_INVALID_ARGUMENT, "write_points_csv: null argument");
        std::vector<float> host;
        const float* p = points;
        if (n && is_device_pointer(points)) {
            host.resize(n * dims);
            const cudaStream_t s = as_stream(stream);
            cuda_ok(cudaMemcpyAsync(host.data(), points, host.size() * 4, cudaMemcpyDeviceToHost,
                                    s),
                    "D2H");
            cuda_ok(cudaStreamSynchronize(s), "sync");
            p = host.data();
        }
        std::string text;
        text.reserve(n * dims * 12);
        char buf[32];
        for (uint64_t i = 0; i < n; ++i) {
            for (uint32_t j = 0; j < dims; ++j) {
                std::snprintf(buf, sizeof buf, "%.9f", static_cast<double>(p[i * dims + j]));
                if (j)
                    text += ',';
                text += buf;
            }
            text += '\n';
        }
        if (bytes) {
            if (*len < text.size())
                fail(QMC_INVALID_ARGUMENT, "write_points_csv: output buffer too small");
            std::memcpy(bytes, text.data(), text.size());
        }
        *len = text.size();
    });
}

// write_pgm / write_ppm (image.cpp:34-52): header on the host, the per-pixel
// quantization (image.cpp:25-30) on the device.
qmc_status qmc_write_pnm(const float* image, uint32_t width, uint32_t height, uint32_t channels,
                         void* bytes, size_t* len, qmc_stream stream)
{
    return guard([&] {
        if (!len)
            fail(QMC_INVALID_ARGUMENT, "write_pnm: null length");
        if (channels != 1 && channels != 3)
            fail(QMC_INVALID_ARGUMENT, "write_pnm: channels must be 1 (P5) or 3 (P6)");
        if (width == 0 || height == 0)
            fail(QMC_INVALID_ARGUMENT, "make_image: image must be at least 1x1");
        const std::string header = std::string(channels == 1 ? "P5\n" : "P6\n") +
                                   std::to_string(width) + " " + std::to_string(height) +
                                   "\n255\n";
        const uint64_t npix = static_cast<uint64_t>(width) * height;
        const size_t need = header.size() + npix * channels;
        if (!bytes || *len < need) {
            *len = need;
            if (bytes)
                fail(QMC_INVALID_ARGUMENT, "write_pnm: output buffer too small");
            return;
        }
        if (!image)
            fail(QMC_INVALID_ARGUMENT, "write_pnm: null image");
        const cudaStream_t s = as_stream(stream);
        pool_keep_memory();
        DevPoints dv(image, npix, s);
        unsigned char* d = nullptr;
        cuda_ok(cudaMallocAsync(&d, npix * channels + 1, s), "cudaMallocAsync");
        cuda_ok(launch_quantize(dv.ptr, npix, channels, d, s), "launch_quantize");
        unsigned char* o = static_cast<unsigned char*>(bytes);
        std::memcpy(o, header.data(), header.size());
        cuda_ok(cudaMemcpyAsync(o + header.size(), d, npix * channels, cudaMemcpyDeviceToHost, s),
                "D2H");
        cudaFreeAsync(d, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
        *len = need;
    });
}

} // extern "C"
