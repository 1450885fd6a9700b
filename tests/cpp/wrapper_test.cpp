// Reference-style caller of the qmc::-shaped C++ wrapper (include/qmcgpu.hpp):
// the same calls a qmckit caller makes (sobol_point, lattice_point,
// halton_point, make_stream / sample, integrate, the point-set metrics, the
// file formats, render), checked against golden checksums recorded from the
// reference build and against each other.
//   wrapper_test --host                  host-only calls (no GPU needed)
//   wrapper_test <sobol fnv> <render fnv>  everything, on a GPU
#include "qmcgpu.hpp"

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <sstream>

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

#define EXPECT(cond)                                                                               \
    do {                                                                                           \
        if (!(cond)) {                                                                             \
            std::printf("FAILED: %s (line %d)\n", #cond, __LINE__);                                \
            ++bad;                                                                                 \
        }                                                                                          \
    } while (0)

template <typename E, typename F>
static bool throws(F&& f)
{
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static int host_checks()
{
    int bad = 0;
    EXPECT(qmcgpu::prime(0) == 2 && qmcgpu::prime(999) == 7919);
    EXPECT(throws<std::out_of_range>([] { qmcgpu::prime(1000); }));
    EXPECT(qmcgpu::prime_max_power(1) == 3486784401u);
    const auto g = qmcgpu::lfsr_generator_vector(0xace1, 2);
    EXPECT(g.g[0] == 1u && g.g[1] == 1276675999u);
    EXPECT(qmcgpu::hilbert_order_for(3840, 2160) == 12);
    const qmcgpu::HaltonPixelEnumeration e(3840, 2160);
    EXPECT(e.stride() == 8957952u && e.scale_x() == 4096 && e.scale_y() == 2187);
    EXPECT(qmcgpu::hilbert_index({0, 1, 1}) == 1 && qmcgpu::hilbert_index({1, 0, 1}) == 3);
    // SURVEY §4 goldens
    EXPECT(qmcgpu::hilbert_phi3_fixed({1, 0, 12}) == 0x55555555u);
    EXPECT(qmcgpu::hilbert_phi3_fixed({0, 1, 12}) == 0x1c71c71cu);
    const auto hp = qmcgpu::hilbert_xy(qmcgpu::hilbert_index({5, 9, 4}), 4);
    EXPECT(hp.x == 5 && hp.y == 9);
    EXPECT(throws<std::invalid_argument>([] { qmcgpu::hilbert_index({0, 0, 0}); }));
    EXPECT(throws<std::out_of_range>([] { qmcgpu::hilbert_index({16, 0, 4}); }));
    EXPECT(qmcgpu::digit_reverse(5, 2, 3) == 5 && qmcgpu::digit_reverse(1, 3, 2) == 3);
    EXPECT(throws<std::overflow_error>([&] { qmcgpu::lattice_shift_fixed(2, 32, g); }));
    EXPECT(qmcgpu::lattice_shift_fixed(1, 31, g)[0] == 1u);
    const auto c = qmcgpu::partition_by_extra_dimension(1, 4, 2);
    EXPECT(c.remainder == 2 && c.modulus == 4);
    std::istringstream gv("# comment\n1\n1276675999 # second\n");
    const auto lg = qmcgpu::load_generator_vector(gv);
    EXPECT(lg.dims() == 2 && lg.g[1] == 1276675999u);
    std::istringstream bad_gv("1\n4\n");
    EXPECT(throws<qmcgpu::ConfigError>([&] { qmcgpu::load_generator_vector(bad_gv); }));
    std::istringstream lf("3 2\n");
    const auto f = qmcgpu::load_linear_factors(lf, 3);
    EXPECT(f.size() == 3 && f[0] == 1 && f[1] == 2 && f[2] == 4);
    EXPECT(qmcgpu::default_linear_factors(3) == (std::vector<std::uint32_t>{1, 2, 4}));
    const char msg[] = "qmc";
    EXPECT(qmcgpu::fnv1a64(msg, 3) == fnv(msg, 3));
    const auto ti = qmcgpu::builtin_integrand("indicator", 3);
    EXPECT(std::fabs(ti.exact_integral - 0.343) < 1e-15);
    EXPECT(throws<qmcgpu::ConfigError>([] { qmcgpu::builtin_integrand("gauss", 2); }));
    EXPECT(qmcgpu::sampler_kind_from_name("image-plane-halton") == QMC_KIND_IMAGE_PLANE_HALTON);
    EXPECT(qmcgpu::sampler_kind_name(QMC_KIND_SOBOL_XOR_TABLE) == "sobol-xor-table");
    EXPECT(throws<qmcgpu::ConfigError>([] { qmcgpu::sampler_kind_from_name("sobol2"); }));
    return bad;
}

int main(int argc, char** argv)
{
    if (argc >= 2 && std::strcmp(argv[1], "--host") == 0) {
        const int bad = host_checks();
        std::printf(bad ? "FAIL %d\n" : "OK\n", bad);
        return bad ? 1 : 0;
    }
    if (argc < 3)
        return 2;
    const std::uint64_t want_sobol = std::strtoull(argv[1], nullptr, 16);
    const std::uint64_t want_render = std::strtoull(argv[2], nullptr, 16);
    int bad = host_checks();

    // sobol_point / render goldens
    const auto m = qmcgpu::GeneratorMatrixSet::builtin(32);
    const auto pts = qmcgpu::sobol_points(m, 0, 1 << 16, 32);
    EXPECT(fnv(pts.data(), pts.size() * 4) == want_sobol);
    qmcgpu::RenderJob job;
    job.width = job.height = 64;
    job.spp = 16;
    const auto img = qmcgpu::render(job);
    EXPECT(fnv(img.values.data(), img.values.size() * 4) == want_render);
    const auto img3 = qmcgpu::render_devices(job, {0, 0, 0}); // row bands, one thread each
    EXPECT(img3.values == img.values);
    qmcgpu::RenderJob ijob = job;
    ijob.accum = QMC_ACCUM_INT;
    const auto iimg = qmcgpu::render(ijob);
    const auto iimg4 = qmcgpu::render_samples_devices(ijob, {0, 0, 0, 0}); // fused reduction
    EXPECT(iimg4.values == iimg.values);
    // the collective inside the library: NCCL communicator over device 0
    // (world size 1 on a one-GPU box; every distinct GPU on a bigger one)
    const int ndev = argc > 3 ? std::atoi(argv[3]) : 1;
    std::vector<int> devs;
    for (int d = 0; d < ndev && d < 8; ++d)
        devs.push_back(d);
    const auto nimg = qmcgpu::render_nccl_devices(job, devs, QMC_PARTITION_ROWS);
    EXPECT(nimg.values == img.values);
    if ((devs.size() & (devs.size() - 1)) == 0) {
        const auto nimg2 = qmcgpu::render_nccl_devices(ijob, devs, QMC_PARTITION_SAMPLES);
        EXPECT(nimg2.values == iimg.values);
    }
    EXPECT(throws<qmcgpu::ConfigError>([] { qmcgpu::GeneratorMatrixSet::builtin(65); }));
    EXPECT(throws<std::invalid_argument>([&] { qmcgpu::sobol_points(m, (1ull << 52) - 1, 2, 4); }));

    // lattice_point, radical_inverse, halton_point
    const auto g = qmcgpu::lfsr_generator_vector(0xace1, 4);
    const auto lat = qmcgpu::lattice_points(g, 1, 1);
    EXPECT(lat.size() == 4 && lat[0] == 0.5f);
    EXPECT(qmcgpu::radical_inverse(1, 0) == 0.5f && qmcgpu::radical_inverse(1, 1) == 1.0f / 3);
    const auto hal = qmcgpu::halton_points(100, 50, 5, QMC_RADICAL_LINEAR);
    const auto rad = qmcgpu::radical_inverse_points(100, 50, 3, QMC_RADICAL_LINEAR, 6);
    for (int k = 0; k < 50; ++k)
        EXPECT(hal[k * 5 + 3] == rad[k]);

    // TabledHalton equals the linearly scrambled Halton; Faure tables
    const qmcgpu::TabledHalton th(5);
    EXPECT(th.points(100, 50) == hal);
    EXPECT(th.component(107, 3) == hal[7 * 5 + 3]);
    const qmcgpu::FaurePermutations fp(4);
    EXPECT(fp.dims() == 4 && fp.for_prime_index(2) == qmcgpu::faure_permutation(5));

    // make_stream / SampleStream: the halton kind equals halton_point
    qmcgpu::StreamParams sp;
    sp.dims = 5;
    sp.scramble = "linear";
    const auto hs = qmcgpu::make_stream(QMC_KIND_HALTON, sp);
    EXPECT(hs.points(100, 50) == hal);
    EXPECT(hs.sample(107, 2) == hal[7 * 5 + 2]);
    qmcgpu::StreamParams bad_sp;
    bad_sp.scramble = "owen";
    EXPECT(throws<qmcgpu::ConfigError>([&] { qmcgpu::make_stream(QMC_KIND_HALTON, bad_sp); }));
    qmcgpu::StreamParams lat_sp;
    lat_sp.dims = 2;
    lat_sp.generator = qmcgpu::GeneratorVector{{1, 4}};
    EXPECT(throws<qmcgpu::ConfigError>([&] { qmcgpu::make_stream(QMC_KIND_LATTICE, lat_sp); }));
    qmcgpu::StreamParams px;
    px.dims = 2;
    px.pixel = {5, 9, 4};
    px.generator = qmcgpu::lfsr_generator_vector(0xace1, 2);
    const auto psl = qmcgpu::make_stream(QMC_KIND_PIXEL_SHIFTED_LATTICE, px);
    EXPECT(qmcgpu::check_1d_stratification(psl, 0, 8).ok);

    // XOR tables: write -> load round trip gives the same stream
    const auto wn = std::make_shared<const qmcgpu::XorTables>(
        qmcgpu::XorTables::white_noise(2, 64, 7));
    std::stringstream xqt;
    wn->write(xqt);
    EXPECT(xqt.str().size() > 0 && wn->dims() == 2 && wn->point_count() == 64);

    // integrate and the point-set metrics
    qmcgpu::StreamParams sob;
    sob.dims = 4;
    const auto ss = qmcgpu::make_stream(QMC_KIND_SOBOL, sob);
    const auto row = qmcgpu::integrate(ss, qmcgpu::builtin_integrand("product-sine", 4), 1 << 16);
    EXPECT(row.n == (1u << 16) && std::fabs(row.estimate - 1.0) < 1e-3);
    const auto s256 = qmcgpu::sobol_points(m, 0, 256, 2);
    EXPECT(qmcgpu::l2_star_discrepancy(s256, 256, 2) > 0.0);
    EXPECT(qmcgpu::min_toroidal_distance(s256, 256, 2) > 0.0);

    // write_pgm: P5 header + one byte per pixel
    std::ostringstream pgm;
    qmcgpu::write_pgm(img, pgm);
    EXPECT(pgm.str().compare(0, 2, "P5") == 0 && pgm.str().size() > 64 * 64);

    std::printf(bad ? "FAIL %d\n" : "OK\n", bad);
    return bad ? 1 : 0;
}
