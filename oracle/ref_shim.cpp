// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (qmckit `qmc::`,
// /root/reference/proj/src/*.cpp, compiled from where it lies by
// oracle/Makefile into oracle/_ref/libqmcref.so). Only tests/, bench.py's
// cpu_baseline / --impl reference leg and __graft_entry__.smoke() load it,
// and only as the checker or the timed CPU baseline.
//
// Every function catches the reference's C++ exceptions and turns them into
// a status code (0 ok, 1 ConfigError, 2 invalid_argument, 3 out_of_range,
// 4 overflow_error, 9 other) plus a thread-local message, so Python tests can
// assert the same error classes the product's C-ABI reports.

#include "qmc/bench.hpp"
#include "qmc/digitalnet.hpp"
#include "qmc/errors.hpp"
#include "qmc/hilbert.hpp"
#include "qmc/image.hpp"
#include "qmc/imageplane.hpp"
#include "qmc/lattice.hpp"
#include "qmc/primes.hpp"
#include "qmc/quality.hpp"
#include "qmc/radical.hpp"
#include "qmc/render.hpp"
#include "qmc/unitfloat.hpp"

#include <bit>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f)
{
    try {
        f();
        return 0;
    } catch (const qmc::ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 2;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 3;
    } catch (const std::overflow_error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

// Runs body(begin, end) over [0, n) split into `threads` contiguous ranges.
template <typename Body>
void parallel_ranges(std::uint64_t n, int threads, Body&& body)
{
    if (threads <= 1 || n < 4096) {
        body(std::uint64_t{0}, n);
        return;
    }
    std::vector<std::thread> pool;
    std::exception_ptr failure;
    std::mutex m;
    for (int t = 0; t < threads; ++t) {
        const std::uint64_t b = n * t / threads, e = n * (t + 1) / threads;
        pool.emplace_back([&, b, e]() {
            try {
                body(b, e);
            } catch (...) {
                std::lock_guard<std::mutex> lk(m);
                if (!failure)
                    failure = std::current_exception();
            }
        });
    }
    for (auto& th : pool)
        th.join();
    if (failure)
        std::rethrow_exception(failure);
}

std::shared_ptr<const qmc::GeneratorMatrixSet> builtin_matrices(std::uint32_t dims)
{
    return std::make_shared<qmc::GeneratorMatrixSet>(
        qmc::build_matrices(qmc::builtin_direction_numbers(), dims));
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- L0 -------------------------------------------------------------------
std::uint32_t ref_map_bits(std::uint32_t u)
{
    return std::bit_cast<std::uint32_t>(qmc::map_u32_to_unifloat(u));
}
void ref_map_bulk(const std::uint32_t* in, std::uint32_t* out, std::uint64_t n)
{
    for (std::uint64_t k = 0; k < n; ++k)
        out[k] = std::bit_cast<std::uint32_t>(qmc::map_u32_to_unifloat(in[k]));
}
// Map of the contiguous range [u0, u0 + n): used for stratified map checks.
void ref_map_range(std::uint32_t u0, std::uint64_t n, std::uint32_t* out)
{
    for (std::uint64_t k = 0; k < n; ++k)
        out[k] = std::bit_cast<std::uint32_t>(
            qmc::map_u32_to_unifloat(static_cast<std::uint32_t>(u0 + k)));
}
std::uint32_t ref_bit_reverse32(std::uint32_t v) { return qmc::bit_reverse32(v); }
std::uint32_t ref_clz32(std::uint32_t v) { return qmc::count_leading_zeros32(v); }

int ref_prime(std::uint32_t idx, std::uint32_t* out)
{
    return guard([&] { *out = qmc::prime(idx); });
}
int ref_prime_max_power(std::uint32_t idx, std::uint32_t* out)
{
    return guard([&] { *out = qmc::prime_max_power(idx); });
}

// ---- radical --------------------------------------------------------------
// mode: 0 plain, 1 linear(factor), 2 faure
int ref_radical_fixed_fill(std::uint32_t first, std::uint64_t n, std::uint32_t prime_index,
                           int mode, std::uint32_t factor, std::uint32_t* out)
{
    return guard([&] {
        qmc::DigitPermutation sigma;
        if (mode == 2)
            sigma = qmc::faure_permutation(qmc::prime(prime_index));
        for (std::uint64_t k = 0; k < n; ++k) {
            const auto i = static_cast<std::uint32_t>(first + k);
            if (mode == 0)
                out[k] = qmc::radical_inverse_fixed(i, prime_index);
            else if (mode == 1)
                out[k] = qmc::radical_inverse_linscramble_fixed(i, prime_index, factor);
            else
                out[k] = qmc::radical_inverse_permuted_fixed(i, prime_index, sigma);
        }
    });
}
int ref_radical_tabled_fixed_fill(std::uint32_t first, std::uint64_t n, int which,
                                  std::uint32_t* out)
{
    // which: 0 base3 two-digit, 1 base5 two-digit (Faure), 2 base3 four-digit
    return guard([&] {
        const qmc::MultiDigitTable& t = which == 0   ? qmc::base3_two_digit_table()
                                        : which == 1 ? qmc::base5_two_digit_table()
                                                     : qmc::base3_four_digit_table();
        for (std::uint64_t k = 0; k < n; ++k)
            out[k] = qmc::radical_inverse_tabled_fixed(static_cast<std::uint32_t>(first + k),
                                                       t.base, t);
    });
}
int ref_faure_permutation(std::uint32_t b, std::uint32_t* out)
{
    return guard([&] {
        const auto s = qmc::faure_permutation(b);
        std::memcpy(out, s.map.data(), s.map.size() * 4);
    });
}
int ref_tensor_table(const std::uint32_t* sigma, std::uint32_t b, std::uint32_t d,
                     std::uint32_t* out, std::uint32_t* group_base)
{
    return guard([&] {
        qmc::DigitPermutation p{b, std::vector<std::uint32_t>(sigma, sigma + b)};
        const auto t = qmc::tensor_digit_table(p, d);
        std::memcpy(out, t.table.data(), t.table.size() * 4);
        *group_base = t.group_base;
    });
}
// Tabled Halton component (TabledHalton, radical.cpp:308-350), default factors.
int ref_tabled_halton_fixed_fill(std::uint32_t first, std::uint64_t n, std::uint32_t dims,
                                 std::uint32_t* out)
{
    return guard([&] {
        const qmc::TabledHalton th(dims);
        for (std::uint64_t k = 0; k < n; ++k)
            for (std::uint32_t j = 0; j < dims; ++j)
                out[k * dims + j] = th.component_fixed(static_cast<std::uint32_t>(first + k), j);
    });
}

// ---- digitalnet -----------------------------------------------------------
int ref_build_matrices_builtin(std::uint32_t dims, std::uint32_t* out)
{
    return guard([&] {
        const auto m = qmc::build_matrices(qmc::builtin_direction_numbers(), dims);
        for (std::uint32_t j = 0; j < dims; ++j)
            std::memcpy(out + j * qmc::kSobolColumns, m.columns(j).data(),
                        qmc::kSobolColumns * 4);
    });
}
int ref_build_matrices_text(const char* text, std::uint32_t dims, std::uint32_t* out)
{
    return guard([&] {
        const auto dns = qmc::parse_direction_numbers(std::string(text));
        const auto m = qmc::build_matrices(dns, dims);
        for (std::uint32_t j = 0; j < dims; ++j)
            std::memcpy(out + j * qmc::kSobolColumns, m.columns(j).data(),
                        qmc::kSobolColumns * 4);
    });
}
// Sobol' integer stage, row-major [n][dims]; scrambles may be null.
int ref_sobol_fixed_fill(std::uint64_t first, std::uint64_t n, std::uint32_t dims,
                         const std::uint32_t* scrambles, std::uint32_t* out, int threads)
{
    return guard([&] {
        const auto m = builtin_matrices(dims);
        parallel_ranges(n, threads, [&](std::uint64_t b, std::uint64_t e) {
            for (std::uint64_t k = b; k < e; ++k)
                for (std::uint32_t j = 0; j < dims; ++j)
                    out[k * dims + j] =
                        qmc::sobol_component_fixed(first + k, j, *m, scrambles ? scrambles[j] : 0u);
        });
    });
}
// Float Sobol' through the public float API (qmc::sobol_component) — also the
// timed CPU baseline for configs C2/C3(XOR).
int ref_sobol_fill(std::uint64_t first, std::uint64_t n, std::uint32_t dims,
                   const std::uint32_t* scrambles, float* out, int threads)
{
    return guard([&] {
        const auto m = builtin_matrices(dims);
        parallel_ranges(n, threads, [&](std::uint64_t b, std::uint64_t e) {
            for (std::uint64_t k = b; k < e; ++k)
                for (std::uint32_t j = 0; j < dims; ++j)
                    out[k * dims + j] =
                        qmc::sobol_component(first + k, j, *m, scrambles ? scrambles[j] : 0u);
        });
    });
}

// ---- lattice --------------------------------------------------------------
std::uint32_t ref_pixel_hash(std::uint32_t j, std::uint32_t px, std::uint32_t py)
{
    return qmc::pixel_hash(j, px, py);
}
int ref_lfsr_generator_vector(std::uint32_t seed, std::uint32_t dims, std::uint32_t* out)
{
    return guard([&] {
        const auto g = qmc::lfsr_generator_vector(seed, dims);
        std::memcpy(out, g.g.data(), dims * 4);
    });
}
// x = map(lattice_component_fixed(i, g_j) + s_j): the reference composition
// for the CP-rotated lattice. shifts may be null.
int ref_lattice_fill(std::uint64_t first, std::uint64_t n, std::uint32_t dims,
                     const std::uint32_t* g, const std::uint32_t* shifts, float* out, int threads)
{
    return guard([&] {
        parallel_ranges(n, threads, [&](std::uint64_t b, std::uint64_t e) {
            for (std::uint64_t k = b; k < e; ++k)
                for (std::uint32_t j = 0; j < dims; ++j) {
                    const auto i = static_cast<std::uint32_t>(first + k);
                    out[k * dims + j] =
                        shifts ? qmc::map_u32_to_unifloat(qmc::lattice_component_fixed(i, g[j]) +
                                                          shifts[j])
                               : qmc::lattice_component(i, g[j]);
                }
        });
    });
}
int ref_lattice_shift_fixed(std::uint32_t k, std::uint32_t m, const std::uint32_t* g,
                            std::uint32_t dims, std::uint32_t* out)
{
    return guard([&] {
        qmc::GeneratorVector gv{std::vector<std::uint32_t>(g, g + dims)};
        const auto d = qmc::lattice_shift_fixed(k, m, gv);
        std::memcpy(out, d.data(), dims * 4);
    });
}

// ---- hilbert / imageplane -------------------------------------------------
int ref_hilbert_index(std::uint32_t x, std::uint32_t y, std::uint32_t order, std::uint64_t* out)
{
    return guard([&] { *out = qmc::hilbert_index(qmc::PixelCoord{x, y, order}); });
}
int ref_hilbert_xy(std::uint64_t d, std::uint32_t order, std::uint32_t* x, std::uint32_t* y)
{
    return guard([&] {
        const auto p = qmc::hilbert_xy(d, order);
        *x = p.x;
        *y = p.y;
    });
}
int ref_hilbert_phi3_fixed(std::uint32_t x, std::uint32_t y, std::uint32_t order,
                           std::uint32_t* out)
{
    return guard([&] { *out = qmc::hilbert_phi3_fixed(qmc::PixelCoord{x, y, order}); });
}
int ref_halton_pixel_enum(std::uint32_t w, std::uint32_t h, std::uint32_t px, std::uint32_t py,
                          std::uint64_t* offset, std::uint64_t* stride, std::uint32_t* exps)
{
    return guard([&] {
        const qmc::HaltonPixelEnumeration e(w, h);
        *offset = e.offset(px, py);
        *stride = e.stride();
        exps[0] = e.exponent_x();
        exps[1] = e.exponent_y();
        exps[2] = e.scale_x();
        exps[3] = e.scale_y();
    });
}
std::uint64_t ref_digit_reverse(std::uint64_t v, std::uint32_t base, std::uint32_t digits)
{
    return qmc::digit_reverse(v, base, digits);
}
int ref_partition(std::uint32_t part, std::uint32_t parts, std::uint32_t base,
                  std::uint64_t* rem, std::uint64_t* mod)
{
    return guard([&] {
        const auto c = qmc::partition_by_extra_dimension(part, parts, base);
        *rem = c.remainder;
        *mod = c.modulus;
    });
}

// Generic stream fill through make_stream / SampleStream::sample
// (imageplane.cpp:310-461): float bits, row-major [n][dims].
int ref_stream_fill(const char* kind, std::uint32_t dims, std::uint32_t seed,
                    const char* scramble, std::uint32_t px, std::uint32_t py, std::uint32_t order,
                    std::uint32_t spp, std::uint32_t width, std::uint32_t height,
                    std::uint64_t first, std::uint64_t n, std::uint32_t* out)
{
    return guard([&] {
        const qmc::SamplerKind k = qmc::sampler_kind_from_name(kind);
        qmc::StreamParams p;
        p.dims = dims;
        p.scramble = scramble;
        p.pixel = qmc::PixelCoord{px, py, order};
        p.spp = spp;
        p.width = width;
        p.height = height;
        if (k == qmc::SamplerKind::lattice || k == qmc::SamplerKind::pixel_shifted_lattice)
            p.generator = qmc::lfsr_generator_vector(seed ? seed : qmc::kDefaultGeneratorSeed,
                                                     std::max(dims, 2u));
        if (k == qmc::SamplerKind::sobol) {
            p.matrices = builtin_matrices(dims);
            if (seed)
                for (std::uint32_t j = 0; j < dims; ++j)
                    p.sobol_scrambles.push_back(qmc::pixel_hash(j, seed, 0x5eedu));
        }
        if (k == qmc::SamplerKind::sobol_xor_table)
            p.tables = std::make_shared<qmc::XorTables>(qmc::white_noise_xor_tables(
                dims, std::bit_ceil(std::max<std::uint32_t>(static_cast<std::uint32_t>(n + first), 1u)),
                seed));
        const qmc::SampleStream s = qmc::make_stream(k, std::move(p));
        for (std::uint64_t i = 0; i < n; ++i)
            for (std::uint32_t j = 0; j < dims; ++j)
                out[i * dims + j] = std::bit_cast<std::uint32_t>(s.sample(first + i, j));
    });
}

// ---- render / quality / image ---------------------------------------------
int ref_render(std::uint32_t w, std::uint32_t h, std::uint32_t spp, const char* kind,
               const char* accum, std::uint32_t seed, std::uint32_t workers, float* out)
{
    return guard([&] {
        qmc::RenderJob job;
        job.width = w;
        job.height = h;
        job.spp = spp;
        job.kind = qmc::sampler_kind_from_name(kind);
        job.accum = qmc::accum_mode_from_name(accum);
        job.seed = seed;
        job.workers = workers;
        const qmc::ImageBuffer img = qmc::render(job);
        std::memcpy(out, img.values.data(), img.values.size() * 4);
    });
}
double ref_scene_value(double x, double y) { return qmc::scene_value(x, y); }
std::uint32_t ref_hilbert_order_for(std::uint32_t w, std::uint32_t h)
{
    return qmc::hilbert_order_for(w, h);
}
std::uint64_t ref_fnv1a64(const void* data, std::uint64_t size)
{
    return qmc::fnv1a64(data, size);
}
int ref_run_bench_kernel(const char* name, std::uint64_t count, std::uint32_t dims,
                         double* comps_per_s, std::uint64_t* checksum)
{
    return guard([&] {
        const auto r = qmc::run_bench_kernel(name, count, dims);
        *comps_per_s = r.components_per_second;
        *checksum = r.checksum;
    });
}
// integrate (quality.cpp:214-282) over a stream built like ref_stream_fill.
int ref_integrate(const char* kind, std::uint32_t dims, std::uint32_t seed, const char* integrand,
                  std::uint64_t n, const char* accum, std::uint32_t workers, double* estimate)
{
    return guard([&] {
        const qmc::SamplerKind k = qmc::sampler_kind_from_name(kind);
        qmc::StreamParams p;
        p.dims = dims;
        if (k == qmc::SamplerKind::lattice)
            p.generator = qmc::lfsr_generator_vector(seed ? seed : qmc::kDefaultGeneratorSeed,
                                                     std::max(dims, 2u));
        if (k == qmc::SamplerKind::sobol) {
            p.matrices = builtin_matrices(dims);
            if (seed)
                for (std::uint32_t j = 0; j < dims; ++j)
                    p.sobol_scrambles.push_back(qmc::pixel_hash(j, seed, 0x5eedu));
        }
        const qmc::SampleStream s = qmc::make_stream(k, std::move(p));
        const auto f = qmc::builtin_integrand(integrand, dims);
        *estimate =
            qmc::integrate(s, f, n, qmc::accum_mode_from_name(accum), workers).estimate;
    });
}
// integrate over a Sobol' stream with caller direction numbers (any dims the
// text defines; parse_direction_numbers + build_matrices, digitalnet.cpp:23-109).
int ref_integrate_sobol_text(const char* text, std::uint32_t dims, const char* integrand,
                             std::uint64_t n, const char* accum, std::uint32_t workers,
                             double* estimate)
{
    return guard([&] {
        qmc::StreamParams p;
        p.dims = dims;
        p.matrices = std::make_shared<qmc::GeneratorMatrixSet>(
            qmc::build_matrices(qmc::parse_direction_numbers(std::string(text)), dims));
        const qmc::SampleStream s = qmc::make_stream(qmc::SamplerKind::sobol, std::move(p));
        const auto f = qmc::builtin_integrand(integrand, dims);
        *estimate =
            qmc::integrate(s, f, n, qmc::accum_mode_from_name(accum), workers).estimate;
    });
}
// CPU float radical inverse fill through the public API (qmc::radical_inverse,
// radical.cpp:210-213) on `threads` threads — config C1's timed CPU baseline.
int ref_radical_fill(std::uint64_t first, std::uint64_t n, std::uint32_t prime_index, float* out,
                     int threads)
{
    return guard([&] {
        parallel_ranges(n, threads, [&](std::uint64_t b, std::uint64_t e) {
            for (std::uint64_t k = b; k < e; ++k)
                out[k] = qmc::radical_inverse(static_cast<std::uint32_t>(first + k), prime_index);
        });
    });
}
// CPU linearly scrambled Halton points through the public API
// (qmc::halton_point with qmc::default_linear_factors, radical.cpp:260-279)
// on `threads` threads, rows of `dims` floats — the Halton fill's CPU baseline.
int ref_halton_linear_fill(std::uint64_t first, std::uint64_t n, std::uint32_t dims, float* out,
                           int threads)
{
    return guard([&] {
        const std::vector<std::uint32_t> f = qmc::default_linear_factors(dims);
        parallel_ranges(n, threads, [&](std::uint64_t b, std::uint64_t e) {
            for (std::uint64_t k = b; k < e; ++k) {
                const std::vector<float> x =
                    qmc::halton_point(static_cast<std::uint32_t>(first + k), dims, f);
                std::copy(x.begin(), x.end(), out + k * dims);
            }
        });
    });
}
int ref_l2_star(const float* pts, std::uint64_t n, std::uint32_t dims, double* out)
{
    return guard([&] {
        *out = qmc::l2_star_discrepancy(std::span<const float>(pts, n * dims), n, dims);
    });
}
int ref_min_toroidal(const float* pts, std::uint64_t n, std::uint32_t dims, double* out)
{
    return guard([&] {
        *out = qmc::min_toroidal_distance(std::span<const float>(pts, n * dims), n, dims);
    });
}
// check_1d_stratification over the stream built as in ref_stream_fill.
int ref_stratification(const char* kind, std::uint32_t dims, std::uint32_t seed, std::uint32_t j,
                       std::uint32_t m, int* ok)
{
    return guard([&] {
        const qmc::SamplerKind k = qmc::sampler_kind_from_name(kind);
        qmc::StreamParams p;
        p.dims = dims;
        if (k == qmc::SamplerKind::lattice || k == qmc::SamplerKind::pixel_shifted_lattice)
            p.generator = qmc::lfsr_generator_vector(seed ? seed : qmc::kDefaultGeneratorSeed,
                                                     std::max(dims, 2u));
        if (k == qmc::SamplerKind::sobol) {
            p.matrices = builtin_matrices(dims);
            if (seed)
                for (std::uint32_t d = 0; d < dims; ++d)
                    p.sobol_scrambles.push_back(qmc::pixel_hash(d, seed, 0x5eedu));
        }
        const qmc::SampleStream s = qmc::make_stream(k, std::move(p));
        *ok = qmc::check_1d_stratification(s, j, m).ok ? 1 : 0;
    });
}
// write_xor_table_file(white_noise_xor_tables(dims, pc, seed)) into `out`.
int ref_white_noise_xor_file(std::uint32_t dims, std::uint32_t pc, std::uint32_t seed,
                             unsigned char* out, std::uint64_t* len)
{
    return guard([&] {
        std::ostringstream os;
        qmc::write_xor_table_file(os, qmc::white_noise_xor_tables(dims, pc, seed));
        const std::string b = os.str();
        if (out && *len >= b.size())
            std::memcpy(out, b.data(), b.size());
        *len = b.size();
    });
}
// Tables loaded from an XQT1 image with the CLI's point set (qmckit.cpp:
// 121-139: Sobol' points, scrambles pixel_hash(j, seed, 0x5eed) when seeded),
// then SampleStream(sobol_xor_table)::sample — float bits [n][dims].
int ref_xor_stream_fill(const unsigned char* bytes, std::uint64_t len, std::uint32_t dims,
                        std::uint32_t seed, std::uint32_t pc, std::uint32_t px, std::uint32_t py,
                        std::uint64_t first, std::uint64_t n, std::uint32_t* out)
{
    return guard([&] {
        const auto m = builtin_matrices(dims);
        std::vector<std::uint32_t> pts(static_cast<std::size_t>(pc) * dims);
        for (std::uint32_t i = 0; i < pc; ++i)
            for (std::uint32_t j = 0; j < dims; ++j)
                pts[static_cast<std::size_t>(i) * dims + j] = qmc::sobol_component_fixed(
                    i, j, *m, seed ? qmc::pixel_hash(j, seed, 0x5eedu) : 0u);
        std::istringstream in(std::string(reinterpret_cast<const char*>(bytes), len));
        qmc::StreamParams p;
        p.dims = dims;
        p.pixel = qmc::PixelCoord{px, py, 8};
        p.tables = std::make_shared<qmc::XorTables>(qmc::load_xor_tables(in, dims, pts, pc));
        const qmc::SampleStream s = qmc::make_stream(qmc::SamplerKind::sobol_xor_table, std::move(p));
        for (std::uint64_t i = 0; i < n; ++i)
            for (std::uint32_t j = 0; j < dims; ++j)
                out[i * dims + j] = std::bit_cast<std::uint32_t>(s.sample(first + i, j));
    });
}
int ref_load_generator_vector(const char* text, std::uint32_t* out, std::uint32_t cap,
                              std::uint32_t* dims)
{
    return guard([&] {
        std::istringstream in(text);
        const auto g = qmc::load_generator_vector(in);
        *dims = g.dims();
        if (out && cap >= g.dims())
            std::memcpy(out, g.g.data(), g.g.size() * 4);
    });
}
int ref_load_linear_factors(const char* text, std::uint32_t dims, std::uint32_t* out)
{
    return guard([&] {
        std::istringstream in(text);
        const auto f = qmc::load_linear_factors(in, dims);
        std::memcpy(out, f.data(), f.size() * 4);
    });
}
// write_pgm (p6 = 0) / write_ppm (p6 = 1) of a float image into `out`.
int ref_write_pnm(const float* values, std::uint32_t w, std::uint32_t h, int p6,
                  unsigned char* out, std::uint64_t* len)
{
    return guard([&] {
        qmc::ImageBuffer img = qmc::make_image(w, h);
        std::memcpy(img.values.data(), values, img.values.size() * 4);
        std::ostringstream os;
        if (p6)
            qmc::write_ppm(img, os);
        else
            qmc::write_pgm(img, os);
        const std::string b = os.str();
        if (out && *len >= b.size())
            std::memcpy(out, b.data(), b.size());
        *len = b.size();
    });
}
double ref_neumaier(const double* v, std::uint64_t n)
{
    qmc::CompensatedSum s;
    for (std::uint64_t k = 0; k < n; ++k)
        s.add(v[k]);
    return s.value();
}

// reduce_deterministic (quality.cpp:158-166) over (rank, value) pairs
double ref_reduce_deterministic(const std::uint32_t* ranks, const double* values, std::uint64_t n)
{
    std::vector<qmc::RankedPartial> p(n);
    for (std::uint64_t k = 0; k < n; ++k)
        p[k] = qmc::RankedPartial{ranks[k], values[k]};
    return qmc::reduce_deterministic(std::move(p));
}

} // extern "C"
