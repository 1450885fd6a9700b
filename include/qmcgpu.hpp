// qmcgpu.hpp — header-only C++ wrapper that re-exposes the reference's
// `qmc::` call shapes (/root/reference/proj/include/qmc/*.hpp) on top of the
// C-ABI in qmcgpu.h, so reference callers switch with a header change.
// Errors are rethrown as the reference's exception classes (errors.hpp:13-15
// ConfigError, std::invalid_argument, std::out_of_range, std::overflow_error).
// Per-component scalar functions of the reference become batched calls: the
// GPU computes whole index ranges (there is no scalar CPU fallback).
#pragma once

#include "qmcgpu.h"

#include <cstdint>
#include <istream>
#include <iterator>
#include <memory>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

namespace qmcgpu {

struct ConfigError : std::runtime_error { // errors.hpp:13-15
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(qmc_status s)
{
    if (s == QMC_OK)
        return;
    const std::string msg = qmc_last_error();
    switch (s) {
    case QMC_CONFIG: throw ConfigError(msg);
    case QMC_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case QMC_OUT_OF_RANGE: throw std::out_of_range(msg);
    case QMC_OVERFLOW: throw std::overflow_error(msg);
    case QMC_CUDA:
    case QMC_NCCL: throw CudaError(msg);
    default: throw std::runtime_error(msg);
    }
}

// ------------------------------------------------ host setup (primes.hpp etc.)
inline std::uint32_t prime(std::uint32_t index)
{
    std::uint32_t v = 0;
    check(qmc_prime(index, &v));
    return v;
}
inline std::uint32_t prime_max_power(std::uint32_t index)
{
    std::uint32_t v = 0;
    check(qmc_prime_max_power(index, &v));
    return v;
}
inline std::vector<std::uint32_t> faure_permutation(std::uint32_t base) // radical.hpp:32-36
{
    std::vector<std::uint32_t> s(base ? base : 1);
    check(qmc_faure_permutation(base, s.data()));
    return s;
}

struct GeneratorVector { // lattice.hpp:17-23
    std::vector<std::uint32_t> g;
    std::uint32_t dims() const { return static_cast<std::uint32_t>(g.size()); }
};
inline GeneratorVector lfsr_generator_vector(std::uint32_t seed, std::uint32_t dims)
{
    GeneratorVector v{std::vector<std::uint32_t>(dims ? dims : 1)};
    check(qmc_lfsr_generator_vector(seed, dims, v.g.data()));
    return v;
}
inline std::uint32_t pixel_hash(std::uint32_t j, std::uint32_t px, std::uint32_t py)
{
    return qmc_pixel_hash(j, px, py);
}
inline std::uint32_t hilbert_order_for(std::uint32_t w, std::uint32_t h)
{
    return qmc_hilbert_order_for(w, h);
}

inline std::uint64_t digit_reverse(std::uint64_t v, std::uint32_t base, std::uint32_t digits)
{ // imageplane.cpp:43-51
    return qmc_digit_reverse(v, base, digits);
}
// lattice_shift_fixed (lattice.cpp:157-170): pass as lattice_points' shifts
inline std::vector<std::uint32_t> lattice_shift_fixed(std::uint32_t k, std::uint32_t m,
                                                      const GeneratorVector& g)
{
    std::vector<std::uint32_t> d(g.dims() ? g.dims() : 1);
    check(qmc_lattice_shift_fixed(k, m, g.g.data(), g.dims(), d.data()));
    d.resize(g.dims());
    return d;
}

struct IndexCongruence { // imageplane.hpp:77-84
    std::uint64_t remainder = 0, modulus = 1;
    bool contains(std::uint64_t i) const { return i % modulus == remainder; }
    std::uint64_t index(std::uint64_t k) const { return remainder + k * modulus; }
};
inline IndexCongruence partition_by_extra_dimension(std::uint32_t part, std::uint32_t parts,
                                                    std::uint32_t base)
{
    IndexCongruence c;
    check(qmc_partition_by_extra_dimension(part, parts, base, &c.remainder, &c.modulus));
    return c;
}

class HaltonPixelEnumeration { // imageplane.hpp:42-68
public:
    HaltonPixelEnumeration(std::uint32_t w, std::uint32_t h) : w_(w), h_(h)
    {
        check(qmc_halton_pixel_enumeration(w, h, 0, 0, &e_, nullptr));
    }
    std::uint64_t stride() const { return e_.stride; }
    std::uint32_t scale_x() const { return e_.scale_x; }
    std::uint32_t scale_y() const { return e_.scale_y; }
    std::uint32_t exponent_x() const { return e_.exponent_x; }
    std::uint32_t exponent_y() const { return e_.exponent_y; }
    std::uint64_t offset(std::uint32_t px, std::uint32_t py) const
    {
        std::uint64_t o = 0;
        check(qmc_halton_pixel_enumeration(w_, h_, px, py, nullptr, &o));
        return o;
    }
    std::uint64_t index(std::uint32_t px, std::uint32_t py, std::uint64_t k) const
    {
        return offset(px, py) + k * stride();
    }

private:
    std::uint32_t w_, h_;
    qmc_halton_enumeration e_{};
};

// ---------------------------------------------------- digitalnet.hpp:50-84
class GeneratorMatrixSet {
public:
    static GeneratorMatrixSet builtin(std::uint32_t dims)
    {
        qmc_matrices* m = nullptr;
        check(qmc_matrices_builtin(dims, &m));
        return GeneratorMatrixSet(m);
    }
    static GeneratorMatrixSet from_text(const std::string& text, std::uint32_t dims)
    {
        qmc_matrices* m = nullptr;
        check(qmc_matrices_from_text(text.c_str(), dims, &m));
        return GeneratorMatrixSet(m);
    }
    std::uint32_t dimensions() const { return qmc_matrices_dims(m_.get()); }
    std::vector<std::uint32_t> columns() const
    {
        std::vector<std::uint32_t> c(static_cast<size_t>(dimensions()) * 52);
        check(qmc_matrices_columns(m_.get(), c.data()));
        return c;
    }
    const qmc_matrices* handle() const { return m_.get(); }

private:
    struct Del {
        void operator()(qmc_matrices* m) const { qmc_matrices_destroy(m); }
    };
    explicit GeneratorMatrixSet(qmc_matrices* m) : m_(m, Del{}) {}
    std::shared_ptr<qmc_matrices> m_;
};

// Batched sobol_point (digitalnet.hpp:80-84) for indices [first, first + n):
// row-major [n][dims] floats. `out` may be device or host memory.
inline void sobol_points(const GeneratorMatrixSet& m, std::uint64_t first, std::uint64_t n,
                         std::uint32_t dims, float* out,
                         const std::vector<std::uint32_t>& scrambles = {},
                         qmc_stream stream = nullptr)
{
    check(qmc_sobol_fill(m.handle(), first, n, dims, scrambles.empty() ? QMC_SOBOL_NONE : QMC_SOBOL_XOR,
                         scrambles.empty() ? nullptr : scrambles.data(), QMC_OUT_F32, out, stream));
}
inline std::vector<float> sobol_points(const GeneratorMatrixSet& m, std::uint64_t first,
                                       std::uint64_t n, std::uint32_t dims,
                                       const std::vector<std::uint32_t>& scrambles = {})
{
    std::vector<float> v(n * dims);
    sobol_points(m, first, n, dims, v.data(), scrambles);
    return v;
}

// Batched lattice_point (lattice.cpp:48-55), optional integer CP rotation.
inline std::vector<float> lattice_points(const GeneratorVector& g, std::uint64_t first,
                                         std::uint64_t n,
                                         const std::vector<std::uint32_t>& shifts = {})
{
    std::vector<float> v(n * g.dims());
    check(qmc_lattice_fill(g.g.data(), shifts.empty() ? nullptr : shifts.data(), g.dims(), first,
                           n, QMC_OUT_F32, v.data(), nullptr));
    return v;
}

// Batched halton_point (radical.cpp:240-269).
inline std::vector<float> halton_points(std::uint64_t first, std::uint64_t n, std::uint32_t dims,
                                        qmc_radical_scramble scramble = QMC_RADICAL_PLAIN,
                                        const std::vector<std::uint32_t>& factors = {})
{
    std::vector<float> v(n * dims);
    check(qmc_halton_fill(first, n, dims, scramble, factors.empty() ? nullptr : factors.data(),
                          QMC_OUT_F32, v.data(), nullptr));
    return v;
}

inline std::vector<std::uint32_t> default_linear_factors(std::uint32_t dims); // below

// Faure permutations for the first dims prime bases (radical.hpp:80-89).
class FaurePermutations {
public:
    explicit FaurePermutations(std::uint32_t dims)
    {
        for (std::uint32_t j = 0; j < dims; ++j)
            perms_.push_back(faure_permutation(prime(j)));
    }
    std::uint32_t dims() const { return static_cast<std::uint32_t>(perms_.size()); }
    const std::vector<std::uint32_t>& for_prime_index(std::uint32_t j) const { return perms_.at(j); }

private:
    std::vector<std::vector<std::uint32_t>> perms_;
};

// TabledHalton (radical.hpp:110-121): linearly scrambled Halton. The
// reference evaluates it through per-base multi-digit tables; the values
// equal the single-digit linear scramble, which the GPU fill computes.
class TabledHalton {
public:
    explicit TabledHalton(std::uint32_t dims, std::vector<std::uint32_t> linear_factors = {})
        : dims_(dims), factors_(linear_factors.empty() ? default_linear_factors(dims)
                                                         : std::move(linear_factors))
    {
        if (factors_.size() < dims_)
            throw std::invalid_argument("TabledHalton: linear factor list shorter than dims");
    }
    std::uint32_t dims() const { return dims_; }
    // rows [first, first + n) x dims, row-major
    std::vector<float> points(std::uint64_t first, std::uint64_t n) const
    {
        std::vector<float> v(n * dims_);
        check(qmc_halton_fill(first, n, dims_, QMC_RADICAL_LINEAR, factors_.data(), QMC_OUT_F32,
                              v.data(), nullptr));
        return v;
    }
    std::uint32_t component_fixed(std::uint32_t i, std::uint32_t j) const
    {
        if (j >= dims_)
            throw std::out_of_range("TabledHalton: dimension out of range");
        std::vector<std::uint32_t> v(dims_);
        check(qmc_halton_fill(i, 1, dims_, QMC_RADICAL_LINEAR, factors_.data(), QMC_OUT_U32,
                              v.data(), nullptr));
        return v[j];
    }
    float component(std::uint32_t i, std::uint32_t j) const
    {
        if (j >= dims_)
            throw std::out_of_range("TabledHalton: dimension out of range");
        return points(i, 1)[j];
    }

private:
    std::uint32_t dims_;
    std::vector<std::uint32_t> factors_;
};

// ------------------------------------------------ render.hpp:31-54
struct ImageBuffer { // image.hpp:13-23
    std::uint32_t width = 0, height = 0;
    std::vector<float> values;
};

struct RenderJob {
    std::uint32_t width = 0, height = 0, spp = 1;
    qmc_sampler_kind kind = QMC_KIND_PIXEL_SHIFTED_LATTICE;
    qmc_accum accum = QMC_ACCUM_KAHAN;
    std::uint32_t seed = 0;
    GeneratorVector generator;
};

inline ImageBuffer render(const RenderJob& job)
{
    qmc_render_job j{};
    j.width = job.width;
    j.height = job.height;
    j.spp = job.spp;
    j.kind = job.kind;
    j.accum = job.accum;
    j.seed = job.seed;
    j.generator = job.generator.g.empty() ? nullptr : job.generator.g.data();
    j.generator_dims = job.generator.dims();
    ImageBuffer img{job.width, job.height,
                    std::vector<float>(static_cast<size_t>(job.width) * job.height)};
    check(qmc_render(&j, 0, job.height, img.values.data(), nullptr));
    return img;
}

// render(job) across several GPUs of this process (row bands; host image).
inline ImageBuffer render_devices(const RenderJob& job, const std::vector<int>& devices)
{
    qmc_render_job j{};
    j.width = job.width;
    j.height = job.height;
    j.spp = job.spp;
    j.kind = job.kind;
    j.accum = job.accum;
    j.seed = job.seed;
    j.generator = job.generator.g.empty() ? nullptr : job.generator.g.data();
    j.generator_dims = job.generator.dims();
    ImageBuffer img{job.width, job.height,
                    std::vector<float>(static_cast<size_t>(job.width) * job.height)};
    check(qmc_render_devices(&j, devices.data(), static_cast<std::uint32_t>(devices.size()),
                             img.values.data()));
    return img;
}

// The paper's sample partition across GPUs of this process, with the int64
// reduction fused into the render kernels (atomic adds into one accumulator
// over peer access). Int accumulator; a power-of-two device count.
inline ImageBuffer render_samples_devices(const RenderJob& job, const std::vector<int>& devices)
{
    qmc_render_job j{};
    j.width = job.width;
    j.height = job.height;
    j.spp = job.spp;
    j.kind = job.kind;
    j.accum = QMC_ACCUM_INT;
    j.seed = job.seed;
    j.generator = job.generator.g.empty() ? nullptr : job.generator.g.data();
    j.generator_dims = job.generator.dims();
    ImageBuffer img{job.width, job.height,
                    std::vector<float>(static_cast<size_t>(job.width) * job.height)};
    check(qmc_render_samples_devices(&j, devices.data(),
                                     static_cast<std::uint32_t>(devices.size()),
                                     img.values.data()));
    return img;
}

// render(job) across distinct GPUs of this process over NCCL, inside the
// library (qmc_render_nccl_devices): row bands + ncclAllGather
// (QMC_PARTITION_ROWS) or the sample partition + int64 ncclAllReduce
// (QMC_PARTITION_SAMPLES, int accumulator). Host image.
inline ImageBuffer render_nccl_devices(const RenderJob& job, const std::vector<int>& devices,
                                       qmc_partition mode = QMC_PARTITION_ROWS)
{
    qmc_render_job j{};
    j.width = job.width;
    j.height = job.height;
    j.spp = job.spp;
    j.kind = job.kind;
    j.accum = job.accum;
    j.seed = job.seed;
    j.generator = job.generator.g.empty() ? nullptr : job.generator.g.data();
    j.generator_dims = job.generator.dims();
    ImageBuffer img{job.width, job.height,
                    std::vector<float>(static_cast<size_t>(job.width) * job.height)};
    check(qmc_render_nccl_devices(&j, devices.data(), static_cast<std::uint32_t>(devices.size()),
                                  mode, img.values.data()));
    return img;
}

inline qmc_sampler_kind sampler_kind_from_name(const std::string& name)
{
    qmc_sampler_kind k{};
    check(qmc_sampler_kind_from_name(name.c_str(), &k));
    return k;
}
inline std::string sampler_kind_name(qmc_sampler_kind kind) { return qmc_sampler_kind_name(kind); }

// ------------------------------------------------ radical.hpp:65-77, :100-105
// Batched radical_inverse / _linscramble / _permuted for one prime (u32
// indices as the reference's, so first + n wraps at 2^32).
inline std::vector<float> radical_inverse_points(std::uint64_t first, std::uint64_t n,
                                                 std::uint32_t prime_index,
                                                 qmc_radical_scramble scramble = QMC_RADICAL_PLAIN,
                                                 std::uint32_t factor = 1)
{
    std::vector<float> v(n);
    check(qmc_radical_inverse_fill(first, n, prime_index, scramble, factor, QMC_OUT_F32, v.data(),
                                   nullptr));
    return v;
}
inline float radical_inverse(std::uint32_t i, std::uint32_t prime_index)
{
    return radical_inverse_points(i, 1, prime_index)[0];
}
inline std::vector<std::uint32_t> default_linear_factors(std::uint32_t dims)
{
    std::vector<std::uint32_t> f(dims ? dims : 1);
    check(qmc_default_linear_factors(dims, f.data()));
    f.resize(dims);
    return f;
}

// ------------------------------------------------------ file formats
inline std::string slurp(std::istream& in)
{
    return std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}
inline GeneratorVector load_generator_vector(std::istream& in) // lattice.cpp:21-46
{
    const std::string text = slurp(in);
    std::uint32_t dims = 0;
    check(qmc_load_generator_vector(text.c_str(), nullptr, 0, &dims));
    GeneratorVector g{std::vector<std::uint32_t>(dims)};
    check(qmc_load_generator_vector(text.c_str(), g.g.data(), dims, &dims));
    return g;
}
inline std::vector<std::uint32_t> load_linear_factors(std::istream& in, std::uint32_t dims)
{ // radical.cpp:281-306
    const std::string text = slurp(in);
    std::vector<std::uint32_t> f(dims ? dims : 1);
    check(qmc_load_linear_factors(text.c_str(), dims, f.data()));
    f.resize(dims);
    return f;
}
inline std::uint64_t fnv1a64(const void* data, std::size_t size) // image.cpp:54-63
{
    return qmc_fnv1a64(data, size);
}
inline void write_pnm(const ImageBuffer& image, std::uint32_t channels, std::ostream& out)
{
    size_t len = 0;
    check(qmc_write_pnm(image.values.data(), image.width, image.height, channels, nullptr, &len,
                        nullptr));
    std::string bytes(len, '\0');
    check(qmc_write_pnm(image.values.data(), image.width, image.height, channels, &bytes[0], &len,
                        nullptr));
    out.write(bytes.data(), static_cast<std::streamsize>(len));
}
inline void write_pgm(const ImageBuffer& image, std::ostream& out) { write_pnm(image, 1, out); }
inline void write_ppm(const ImageBuffer& image, std::ostream& out) { write_pnm(image, 3, out); }

// ------------------------------------------- XOR tables (imageplane.hpp:92-120)
class XorTables {
public:
    static XorTables white_noise(std::uint32_t dims, std::uint32_t point_count, std::uint32_t seed)
    {
        qmc_xor_tables* t = nullptr;
        check(qmc_xor_tables_white_noise(dims, point_count, seed, &t));
        return XorTables(t);
    }
    // load_xor_tables(in, dims, points, point_count): XQT1 bytes + the stored
    // integer-stage point set [point_count][dims]
    static XorTables load(std::istream& in, std::uint32_t dims,
                          const std::vector<std::uint32_t>& points, std::uint32_t point_count)
    {
        const std::string bytes = slurp(in);
        qmc_xor_tables* t = nullptr;
        check(qmc_xor_tables_load(bytes.data(), bytes.size(), dims, points.data(), point_count,
                                  &t));
        return XorTables(t);
    }
    void write(std::ostream& out) const // write_xor_table_file
    {
        size_t len = 0;
        check(qmc_xor_tables_write(t_.get(), nullptr, &len));
        std::string bytes(len, '\0');
        check(qmc_xor_tables_write(t_.get(), &bytes[0], &len));
        out.write(bytes.data(), static_cast<std::streamsize>(len));
    }
    std::uint32_t dims() const { return qmc_xor_tables_dims(t_.get()); }
    std::uint32_t point_count() const { return qmc_xor_tables_point_count(t_.get()); }
    const qmc_xor_tables* handle() const { return t_.get(); }

private:
    struct Del {
        void operator()(qmc_xor_tables* t) const { qmc_xor_tables_destroy(t); }
    };
    explicit XorTables(qmc_xor_tables* t) : t_(t, Del{}) {}
    std::shared_ptr<qmc_xor_tables> t_;
};

// ------------------------------- StreamParams / SampleStream (imageplane.hpp:139-199)
struct PixelCoord { // hilbert.hpp:14-18
    std::uint32_t x = 0, y = 0, order = 0;
};
inline std::uint64_t hilbert_index(const PixelCoord& p) // hilbert.hpp:39-56
{
    std::uint64_t d = 0;
    check(qmc_hilbert_index(p.x, p.y, p.order, &d));
    return d;
}
inline std::uint32_t hilbert_phi3_fixed(const PixelCoord& p) // imageplane.cpp:16-21
{
    std::uint32_t v = 0;
    check(qmc_hilbert_phi3_fixed(p.x, p.y, p.order, &v));
    return v;
}
inline PixelCoord hilbert_xy(std::uint64_t d, std::uint32_t order) // hilbert.hpp:59-78
{
    PixelCoord p{0, 0, order};
    check(qmc_hilbert_xy(d, order, &p.x, &p.y));
    return p;
}

struct StreamParams {
    std::uint32_t dims = 2;
    GeneratorVector generator;                           // lattice family
    std::shared_ptr<const GeneratorMatrixSet> matrices;  // sobol (null = builtin)
    std::vector<std::uint32_t> sobol_scrambles;          // empty = plain sequence
    std::string scramble = "plain";                      // halton: plain | faure | linear
    std::vector<std::uint32_t> linear_factors;           // empty = default factors
    PixelCoord pixel{0, 0, 1};
    std::uint32_t spp = 1;                               // halton_hilbert block size
    std::uint32_t width = 0, height = 0;                 // image_plane_halton
    std::shared_ptr<const XorTables> tables;             // sobol_xor_table
    // sobol_xor_table without `tables`: white-noise tables made per call
    std::uint32_t xor_seed = 0, xor_point_count = 1024;
};

// A validated stream (make_stream): sample(i, j) and batched points().
class SampleStream {
public:
    std::uint32_t dims() const { return p_.dims; }
    qmc_sampler_kind kind() const { return kind_; }

    // rows [first, first + n) x dims, row-major, into `out` (device or host)
    void points(std::uint64_t first, std::uint64_t n, float* out, qmc_stream stream = nullptr) const
    {
        const qmc_stream_params c = c_params();
        check(qmc_stream_fill(kind_, &c, first, n, QMC_OUT_F32, out, stream));
    }
    std::vector<float> points(std::uint64_t first, std::uint64_t n) const
    {
        std::vector<float> v(n * p_.dims);
        points(first, n, v.data());
        return v;
    }
    // SampleStream::sample(index, dim): one GPU call per point; use points()
    // for anything but spot checks
    float sample(std::uint64_t index, std::uint32_t dim) const
    {
        if (dim >= p_.dims)
            throw std::out_of_range("SampleStream::sample: dimension out of range");
        return points(index, 1)[dim];
    }
    qmc_stream_params c_params() const
    {
        qmc_stream_params c{};
        c.dims = p_.dims;
        c.generator = p_.generator.g.empty() ? nullptr : p_.generator.g.data();
        c.generator_dims = p_.generator.dims();
        c.matrices = p_.matrices ? p_.matrices->handle() : nullptr;
        c.sobol_scrambles = p_.sobol_scrambles.empty() ? nullptr : p_.sobol_scrambles.data();
        c.sobol_scrambles_len = static_cast<std::uint32_t>(p_.sobol_scrambles.size());
        c.halton_scramble = scramble_;
        c.linear_factors = p_.linear_factors.empty() ? nullptr : p_.linear_factors.data();
        c.linear_factors_len = static_cast<std::uint32_t>(p_.linear_factors.size());
        c.px = p_.pixel.x;
        c.py = p_.pixel.y;
        c.order = p_.pixel.order;
        c.spp = p_.spp;
        c.width = p_.width;
        c.height = p_.height;
        c.xor_seed = p_.xor_seed;
        c.xor_point_count = p_.xor_point_count;
        c.xor_tables = p_.tables ? p_.tables->handle() : nullptr;
        return c;
    }

private:
    friend SampleStream make_stream(qmc_sampler_kind kind, StreamParams params);
    SampleStream(qmc_sampler_kind kind, StreamParams p) : kind_(kind), p_(std::move(p)) {}
    qmc_sampler_kind kind_;
    StreamParams p_;
    std::uint32_t scramble_ = QMC_RADICAL_PLAIN;
};

// make_stream (imageplane.cpp:310-416): the C-ABI runs the reference's
// ConfigError checks; a zero-length fill validates without sampling.
inline SampleStream make_stream(qmc_sampler_kind kind, StreamParams params)
{
    SampleStream s(kind, std::move(params));
    const std::string& sc = s.p_.scramble;
    if (sc == "plain")
        s.scramble_ = QMC_RADICAL_PLAIN;
    else if (sc == "faure")
        s.scramble_ = QMC_RADICAL_FAURE;
    else if (sc == "linear")
        s.scramble_ = QMC_RADICAL_LINEAR;
    else
        throw ConfigError("make_stream: scramble must be plain, faure, or linear");
    const qmc_stream_params c = s.c_params();
    check(qmc_stream_fill(kind, &c, 0, 0, QMC_OUT_F32, nullptr, nullptr));
    return s;
}

// ------------------------------------------ quality.hpp:37-104 (integration)
struct TestIntegrand { // quality.hpp:40-48
    std::string name;
    qmc_integrand_kind kind;
    std::uint32_t dims;
    double exact_integral;
};
inline TestIntegrand builtin_integrand(const std::string& name, std::uint32_t dims)
{
    TestIntegrand f{name, QMC_PRODUCT_SINE, dims, 0.0};
    check(qmc_builtin_integrand(name.c_str(), dims, &f.kind, &f.exact_integral));
    return f;
}
struct IntegrationRow { // quality.hpp:90-95
    std::uint64_t n = 0;
    double estimate = 0, abs_error = 0, seconds = 0;
};
inline IntegrationRow integrate(const SampleStream& stream, const TestIntegrand& f,
                                std::uint64_t n, qmc_accum mode = QMC_ACCUM_KAHAN)
{
    const qmc_stream_params c = stream.c_params();
    qmc_integration_row r{};
    check(qmc_integrate(stream.kind(), &c, f.kind, f.dims, n, mode, &r, nullptr));
    return {r.n, r.estimate, r.abs_error, r.seconds};
}

// ------------------------------------------- quality.hpp:56-71 (point-set metrics)
inline double l2_star_discrepancy(const std::vector<float>& points, std::size_t n,
                                  std::size_t dims)
{
    double d = 0;
    check(qmc_l2_star_discrepancy(points.data(), n, static_cast<std::uint32_t>(dims), &d,
                                  nullptr));
    return d;
}
inline double min_toroidal_distance(const std::vector<float>& points, std::size_t n,
                                    std::size_t dims)
{
    double d = 0;
    check(qmc_min_toroidal_distance(points.data(), n, static_cast<std::uint32_t>(dims), &d,
                                    nullptr));
    return d;
}
struct StratificationResult { // quality.hpp:61-66
    bool ok = false;
    std::vector<std::uint32_t> histogram;
};
inline StratificationResult check_1d_stratification(const SampleStream& stream, std::uint32_t j,
                                                    std::uint32_t m)
{
    const qmc_stream_params c = stream.c_params();
    StratificationResult r;
    r.histogram.assign(m <= 20 ? (1u << m) : 1u, 0u); // the C-ABI rejects m > 20
    int ok = 0;
    check(qmc_check_1d_stratification(stream.kind(), &c, j, m, &ok, r.histogram.data(), nullptr));
    r.ok = ok != 0;
    return r;
}

} // namespace qmcgpu
