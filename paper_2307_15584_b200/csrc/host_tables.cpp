// host_tables.cpp — the immutable tables the reference builds on the host
// (primes, Faure permutations, direction numbers and generator matrices,
// generator vectors, Halton pixel enumeration, multi-digit tables). Each
// function cites the reference file:line it restates.
#include "host.hpp"

#include <cstdlib>
#include <cmath>
#include <map>
#include <sstream>
#include <tuple>

namespace qmcgpu {
namespace host {

// ---------------------------------------------------------- prime table

const PrimeTable& primes()
{
    static const PrimeTable t;
    return t;
}

uint32_t prime_at(uint32_t index)
{
    if (index >= kPrimes)
        fail(QMC_OUT_OF_RANGE, "prime: index beyond the bundled prime table");
    return primes().p[index];
}

// radical.cpp:50-74
std::vector<uint32_t> faure(uint32_t b)
{
    if (b < 2)
        fail(QMC_INVALID_ARGUMENT, "faure_permutation: base must be >= 2");
    if (b == 2)
        return {0u, 1u};
    std::vector<uint32_t> s;
    s.reserve(b);
    if (b % 2 == 0) {
        const auto h = faure(b / 2);
        for (uint32_t v : h)
            s.push_back(2 * v);
        for (uint32_t v : h)
            s.push_back(2 * v + 1);
    } else {
        const auto prev = faure(b - 1);
        const uint32_t mid = (b - 1) / 2;
        for (uint32_t k = 0; k < prev.size(); ++k) {
            if (k == mid)
                s.push_back(mid);
            s.push_back(prev[k] >= mid ? prev[k] + 1 : prev[k]);
        }
    }
    return s;
}

// ------------------------------------------------- direction numbers

struct BuiltinRow {
    uint32_t s, a;
    uint32_t m[32];
};
const BuiltinRow kJoeKuo[] = {
#include "joe_kuo_64.inc"
};

std::vector<DirRow> builtin_rows()
{
    std::vector<DirRow> rows;
    for (const BuiltinRow& r : kJoeKuo)
        rows.push_back(DirRow{r.s, r.a, std::vector<uint32_t>(r.m, r.m + r.s)});
    return rows;
}

// digitalnet.cpp:23-65 — same grammar, checks and ConfigError messages.
std::vector<DirRow> parse_rows(const std::string& text)
{
    std::vector<DirRow> rows;
    std::istringstream in(text);
    std::string line;
    size_t no = 0;
    bool header = false;
    auto bad = [&](const std::string& w) {
        fail(QMC_CONFIG, "direction numbers, line " + std::to_string(no) + ": " + w);
    };
    while (std::getline(in, line)) {
        ++no;
        if (!header) {
            header = true;
            continue;
        }
        std::istringstream ls(line);
        uint32_t d = 0, s = 0, a = 0;
        if (!(ls >> d))
            continue;
        if (!(ls >> s >> a))
            bad("expected 'd s a m_1 ... m_s'");
        if (d != rows.size() + 2)
            bad("dimensions must be consecutive starting at 2");
        if (s == 0 || s > 32)
            bad("degree s out of range");
        if (s > 1 && a >= (1u << (s - 1)))
            bad("coefficient a has more than s-1 bits");
        DirRow row{s, a, {}};
        for (uint32_t k = 1; k <= s; ++k) {
            uint64_t mk = 0;
            if (!(ls >> mk))
                bad("expected " + std::to_string(s) + " direction numbers");
            if (mk % 2 == 0)
                bad("direction number m_" + std::to_string(k) + " is even");
            if (mk >= (1ull << k))
                bad("direction number m_" + std::to_string(k) + " must be < 2^" +
                    std::to_string(k));
            row.m.push_back(static_cast<uint32_t>(mk));
        }
        std::string rest;
        if (ls >> rest)
            bad("trailing tokens after the m values");
        rows.push_back(std::move(row));
    }
    return rows;
}

// digitalnet.cpp:79-109 — MSB-aligned columns, 52 per dimension.
std::vector<uint32_t> build_columns(const std::vector<DirRow>& rows, uint32_t dims)
{
    if (dims > rows.size() + 1)
        fail(QMC_CONFIG, "build_matrices: requested " + std::to_string(dims) +
                             " dimensions, direction numbers provide " +
                             std::to_string(rows.size() + 1));
    std::vector<uint32_t> c(static_cast<size_t>(dims) * 52, 0u);
    if (dims == 0)
        return c;
    for (uint32_t k = 0; k < 32; ++k)
        c[k] = 0x80000000u >> k;
    for (uint32_t j = 1; j < dims; ++j) {
        const DirRow& r = rows[j - 1];
        uint32_t* v = c.data() + static_cast<size_t>(j) * 52;
        for (uint32_t k = 0; k < r.s && k < 52; ++k)
            v[k] = r.m[k] << (31 - k);
        for (uint32_t k = r.s; k < 52; ++k) {
            uint32_t x = v[k - r.s] ^ (v[k - r.s] >> r.s);
            for (uint32_t l = 1; l < r.s; ++l)
                if ((r.a >> (r.s - 1 - l)) & 1u)
                    x ^= v[k - l];
            v[k] = x;
        }
    }
    return c;
}

uint32_t brev_host(uint32_t v)
{
    uint32_t r = 0;
    for (int k = 0; k < 32; ++k)
        r |= ((v >> k) & 1u) << (31 - k);
    return r;
}

// lattice.cpp:59-77
uint32_t fmix_host(uint32_t h)
{
    h = (h ^ (h >> 16)) * 0x85ebca6bu;
    h = (h ^ (h >> 13)) * 0xc2b2ae35u;
    return h ^ (h >> 16);
}
uint32_t pixel_hash_host(uint32_t j, uint32_t px, uint32_t py)
{
    return fmix_host(fmix_host(fmix_host(0x9e3779b9u ^ j) ^ px) ^ py);
}

std::vector<uint32_t> lfsr(uint32_t seed, uint32_t dims)
{
    if (seed == 0)
        fail(QMC_INVALID_ARGUMENT, "lfsr_generator_vector: zero seed is the absorbing state");
    if (dims < 1)
        fail(QMC_INVALID_ARGUMENT, "lfsr_generator_vector: dims must be >= 1");
    std::vector<uint32_t> g{1u};
    uint32_t x = seed;
    for (uint32_t j = 1; j < dims; ++j) {
        x ^= x << 13;
        x ^= x >> 17;
        x ^= x << 5;
        g.push_back(2u * x + 1u);
    }
    return g;
}

uint32_t hilbert_order(uint32_t w, uint32_t h)
{
    uint32_t o = 1;
    while (o < 32 && ((1ull << o) < w || (1ull << o) < h))
        ++o;
    return o;
}

// ------------------------------------------ Halton pixel enumeration

uint64_t inverse_mod(uint64_t a, uint64_t n)
{
    if (n == 1)
        return 0;
    int64_t r0 = static_cast<int64_t>(n), r1 = static_cast<int64_t>(a % n), t0 = 0, t1 = 1;
    while (r1) {
        const int64_t q = r0 / r1;
        const int64_t r2 = r0 - q * r1, t2 = t0 - q * t1;
        r0 = r1;
        r1 = r2;
        t0 = t1;
        t1 = t2;
    }
    const int64_t m = static_cast<int64_t>(n);
    return static_cast<uint64_t>(((t0 % m) + m) % m);
}

// imageplane.cpp:80-98
HaltonEnum halton_enum(uint32_t w, uint32_t h)
{
    if (w == 0 || h == 0)
        fail(QMC_CONFIG, "HaltonPixelEnumeration: image must be at least 1x1");
    if (w > (1u << 20) || h > 1594323u)
        fail(QMC_CONFIG, "HaltonPixelEnumeration: image too large for the index range");
    HaltonEnum e;
    while (e.sx < w) {
        e.sx *= 2;
        ++e.ex;
    }
    while (e.sy < h) {
        e.sy *= 3;
        ++e.ey;
    }
    e.stride = static_cast<uint64_t>(e.sx) * e.sy;
    e.crt_x = e.sy * inverse_mod(e.sy % e.sx, e.sx);
    e.crt_y = e.sx * inverse_mod(e.sx % e.sy, e.sy);
    return e;
}

// hilbert.hpp:59-78, the inverse of hilbert_index for its orientation
// (order validated by the caller).
void hilbert_xy_host(uint64_t d, uint32_t order, uint32_t& x, uint32_t& y)
{
    x = y = 0;
    const uint32_t n = 1u << order;
    for (uint32_t s = 1; s < n; s <<= 1, d >>= 2) {
        const uint32_t rx = 1u & static_cast<uint32_t>(d >> 1);
        const uint32_t ry = 1u & static_cast<uint32_t>(d ^ rx);
        if (ry == 0) { // rotate the s x s quadrant
            if (rx == 1) {
                x = s - 1 - x;
                y = s - 1 - y;
            }
            const uint32_t tmp = x;
            x = y;
            y = tmp;
        }
        x += s * rx;
        y += s * ry;
    }
}

uint64_t digit_reverse_host(uint64_t v, uint32_t base, uint32_t digits)
{
    uint64_t r = 0;
    for (uint32_t k = 0; k < digits; ++k) {
        r = r * base + v % base;
        v /= base;
    }
    return r;
}

// Multi-digit tables (tensor_digit_table, radical.cpp:76-110) on the device:
// d = the most base-b digits with b^d <= 4096 (so a table stays 16 KB and
// L1-resident), entry v = the d digits of v permuted by sigma and mirrored.
// Built once per (device, base, scramble) and kept for the process.
DigitTable digit_table(uint32_t b, uint32_t mode, uint32_t factor, uint32_t min_digits,
                       uint32_t max_entries, bool with_quotients)
{
    struct Slot {
        DevPtr t, qx;
        uint32_t group = 0;
    };
    static std::mutex mu;
    static std::map<std::tuple<int, uint32_t, uint32_t, uint32_t, uint32_t, bool>, Slot> cache;
    uint32_t d = 0, group = 1;
    while (static_cast<uint64_t>(group) * b <= max_entries) {
        group *= b;
        ++d;
    }
    if (d < min_digits || d == 0)
        return {};
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    auto& slot = cache[{dev, b, mode, factor, max_entries, with_quotients}];
    if (!slot.t) {
        std::vector<uint32_t> sigma(b);
        if (mode == 2) {
            sigma = faure(b);
        } else {
            for (uint32_t a = 0; a < b; ++a)
                sigma[a] = mode == 1 ? static_cast<uint32_t>((uint64_t(factor) * a) % b) : a;
        }
        std::vector<uint32_t> t(group + 8, 0u);
        for (uint32_t v = 0; v < group; ++v) {
            uint32_t rem = v, out = 0;
            for (uint32_t k = 0; k < d; ++k) {
                out = out * b + sigma[rem % b];
                rem /= b;
            }
            t[v] = out;
        }
        if (with_quotients) {
            // T * 2^32 = q * group + r: the contiguous fill adds the
            // warp-uniform quotient of the high digits and a carry (r >= thr)
            std::vector<uint32_t> qx(group + 8, 0u);
            for (uint32_t v = 0; v < group; ++v)
                qx[v] = static_cast<uint32_t>((static_cast<uint64_t>(t[v]) << 32) / group);
            slot.qx = dev_upload(qx.data(), qx.size() * 4);
        }
        slot.t = dev_upload(t.data(), t.size() * 4);
        slot.group = group;
    }
    return {static_cast<const uint32_t*>(slot.t.get()), slot.group,
            static_cast<const uint32_t*>(slot.qx.get())};
}

// Column order of k_render's warps at spp >= 8: the columns whose pixel
// footprints keep one sine quadrant of sin(8 pi x) with an even quadrant
// count first, then those with an odd count, then the few that cross a
// quadrant boundary — so nearly every warp of 32 consecutive entries shares
// its quadrant parity and takes the specialised loop. The order only decides
// which thread renders which pixel; every pixel's value is unchanged. The
// classification restates sin_fixed_quadrant (device.cuh).
const uint32_t* render_column_order(uint32_t width)
{
    static std::mutex mu;
    static std::map<std::pair<int, uint32_t>, DevPtr> cache;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    auto& slot = cache[{dev, width}];
    if (!slot) {
        const SceneConsts c = make_scene_consts();
        const double inv_w = 1.0 / width;
        std::vector<uint32_t> cls[3];
        for (uint32_t px = 0; px < width; ++px) {
            const double t0 = px * inv_w * c.k8pi * c.two_over_pi;
            const double t1 = (px + 1.0) * inv_w * c.k8pi * c.two_over_pi;
            const double n = std::rint(t0);
            const bool fixed = t0 > n - 0.5 + 1e-9 && t1 < n + 0.5 - 1e-9;
            cls[fixed ? static_cast<int64_t>(n) & 1 : 2].push_back(px);
        }
        std::vector<uint32_t> order;
        order.reserve(width);
        for (const auto& v : cls)
            order.insert(order.end(), v.begin(), v.end());
        slot = dev_upload(order.data(), order.size() * 4);
    }
    return static_cast<const uint32_t*>(slot.get());
}

// [floor(T[v] 2^32 / 3^7) | floor(T[v] 2^32 / 3^14)], v < 3^7, T[v] the
// 7-digit base-3 reversal of v (kernels_render.cu, phi3_q).
const uint32_t* render_phi3_quotients()
{
    static std::mutex mu;
    static std::map<int, DevPtr> cache;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    auto& slot = cache[dev];
    if (!slot) {
        std::vector<uint32_t> q(2 * 2187);
        for (uint32_t v = 0; v < 2187; ++v) {
            uint32_t t = 0;
            for (uint32_t k = 0, r = v; k < 7; ++k, r /= 3)
                t = t * 3 + r % 3;
            q[v] = static_cast<uint32_t>((static_cast<uint64_t>(t) << 32) / 2187u);
            q[2187 + v] = static_cast<uint32_t>((static_cast<uint64_t>(t) << 32) / 4782969u);
        }
        slot = dev_upload(q.data(), q.size() * 4);
    }
    return static_cast<const uint32_t*>(slot.get());
}

// The render's staged phi_3 tables in one 16-B padded device buffer, laid out
// as k_render's shared copy (RenderSmem tab3 then q3): [T (3^7 words), 0,
// QL (3^7), QH (3^7), 0, 0], so one cp.async.bulk copies them.
const uint32_t* render_t3q3()
{
    static std::mutex mu;
    static std::map<int, DevPtr> cache;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    auto& slot = cache[dev];
    if (!slot) {
        std::vector<uint32_t> z(kRenderT3Q3Words, 0u);
        slot = dev_upload(z.data(), z.size() * 4);
        cuda_ok(cudaMemcpy(slot.get(), digit_table(3, 0, 0).ptr, 2187 * 4, cudaMemcpyDeviceToDevice),
                "cudaMemcpy D2D");
        cuda_ok(cudaMemcpy(static_cast<uint32_t*>(slot.get()) + 2188, render_phi3_quotients(),
                           2 * 2187 * 4, cudaMemcpyDeviceToDevice),
                "cudaMemcpy D2D");
    }
    return static_cast<const uint32_t*>(slot.get());
}

const uint64_t* pow_magic(uint32_t b)
{
    static std::mutex mu;
    static std::map<std::pair<int, uint32_t>, DevPtr> cache;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    auto& slot = cache[{dev, b}];
    if (!slot) {
        std::vector<uint64_t> m(33, 0);
        uint64_t p = 1;
        for (uint32_t d = 0; d < 33 && p < (1ull << 32); ++d, p *= b)
            m[d] = p == 1 ? ~0ull : ~0ull / p; // b odd: floor((2^64-1)/p) = floor(2^64/p)
        slot = dev_upload(m.data(), m.size() * 8);
    }
    return static_cast<const uint64_t*>(slot.get());
}

// RadicalDim table for `dims` prime bases (radical.cpp:130-181).
std::vector<RadicalDim> radical_dims(uint32_t dims, uint32_t first_prime, qmc_radical_scramble sc,
                                     const uint32_t* factors, std::vector<uint32_t>& sigma_pool,
                                     std::vector<size_t>& sigma_off)
{
    std::vector<RadicalDim> rd(dims);
    sigma_off.assign(dims, SIZE_MAX);
    for (uint32_t j = 0; j < dims; ++j) {
        const uint32_t pi = first_prime + j;
        const uint32_t b = prime_at(pi);
        RadicalDim& r = rd[j];
        r.base = b;
        r.maxpow = primes().maxpow[pi];
        r.divb = make_div32(b);
        r.divmp = make_div32(r.maxpow);
        r.mode = 0;
        r.factor = 0;
        r.sigma = nullptr;
        r.table = nullptr;
        r.group = 0;
        r.divg = Div32{0, 0};
        if (sc == QMC_RADICAL_LINEAR) {
            const uint32_t f = factors ? factors[j] : b - 1;
            if (f == 0 || f >= b)
                fail(QMC_INVALID_ARGUMENT,
                     "radical_inverse_linscramble: factor must be in [1, base)");
            r.mode = 1;
            r.factor = f;
        } else if (sc == QMC_RADICAL_FAURE) {
            const auto s = faure(b);
            sigma_off[j] = sigma_pool.size();
            sigma_pool.insert(sigma_pool.end(), s.begin(), s.end());
            r.mode = 2;
        }
        r.ftable = nullptr;
        r.fqx = nullptr;
        r.magic = nullptr;
        r.gdigits = r.fgroup = r.fdigits = r.himod = 0;
        r.fdivg = Div32{0, 0};
        if (b > 2) {
            r.magic = pow_magic(b);
            const DigitTable t = digit_table(b, r.mode, r.factor);
            if (t.ptr) {
                r.table = t.ptr;
                r.group = t.group;
                r.divg = make_div32(t.group);
                for (uint32_t g = t.group; g > 1; g /= b)
                    ++r.gdigits;
            }
            const DigitTable f = digit_table(b, r.mode, r.factor, 1, kFillTableMax, true);
            if (f.ptr) {
                r.ftable = f.ptr;
                r.fqx = f.qx;
                r.fgroup = f.group;
                r.fdivg = make_div32(f.group);
                for (uint32_t g = f.group; g > 1; g /= b)
                    ++r.fdigits;
                r.himod = r.maxpow / f.group;
            }
        }
    }
    return rd;
}

} // namespace host
} // namespace qmcgpu
