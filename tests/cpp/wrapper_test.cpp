// Reference-style caller of the qmc::-shaped C++ wrapper (include/qmcgpu.hpp):
// the same calls a qmckit caller makes (sobol_point, lattice_point, render),
// checked against golden checksums recorded from the reference build.
#include "qmcgpu.hpp"

#include <cstdio>
#include <cstring>

static std::uint64_t fnv(const void* p, size_t n)
{
    const unsigned char* b = static_cast<const unsigned char*>(p);
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (size_t k = 0; k < n; ++k) {
        h ^= b[k];
        h *= 0x100000001b3ull;
    }
    return h;
}

int main(int argc, char** argv)
{
    if (argc < 3)
        return 2;
    const std::uint64_t want_sobol = std::strtoull(argv[1], nullptr, 16);
    const std::uint64_t want_render = std::strtoull(argv[2], nullptr, 16);
    int bad = 0;
    const auto m = qmcgpu::GeneratorMatrixSet::builtin(32);
    const auto pts = qmcgpu::sobol_points(m, 0, 1 << 16, 32);
    if (fnv(pts.data(), pts.size() * 4) != want_sobol) {
        std::printf("sobol checksum mismatch\n");
        ++bad;
    }
    qmcgpu::RenderJob job;
    job.width = job.height = 64;
    job.spp = 16;
    const auto img = qmcgpu::render(job);
    if (fnv(img.values.data(), img.values.size() * 4) != want_render) {
        std::printf("render checksum mismatch\n");
        ++bad;
    }
    try {
        qmcgpu::GeneratorMatrixSet::builtin(65);
        ++bad;
    } catch (const qmcgpu::ConfigError&) {
    }
    try {
        qmcgpu::sobol_points(m, (1ull << 52) - 1, 2, 4);
        ++bad;
    } catch (const std::invalid_argument&) {
    }
    try {
        qmcgpu::prime(1000);
        ++bad;
    } catch (const std::out_of_range&) {
    }
    const auto g = qmcgpu::lfsr_generator_vector(0xace1, 4);
    const auto lat = qmcgpu::lattice_points(g, 1, 1);
    if (lat.size() != 4 || lat[0] != 0.5f) {
        std::printf("lattice mismatch\n");
        ++bad;
    }
    std::printf(bad ? "FAIL %d\n" : "OK\n", bad);
    return bad ? 1 : 0;
}
