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
#include <memory>
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

inline qmc_sampler_kind sampler_kind_from_name(const std::string& name)
{
    qmc_sampler_kind k{};
    check(qmc_sampler_kind_from_name(name.c_str(), &k));
    return k;
}

} // namespace qmcgpu
