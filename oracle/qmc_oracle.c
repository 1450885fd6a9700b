/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference QMC sampling
 * path (see qmc_oracle.h for the contract and how it is pinned).
 * Citations are relative to /root/reference/proj.
 */
#include "qmc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- unitfloat */

/* include/qmc/unitfloat.hpp:13-16 — clz with clz(0) = 32 */
uint32_t qo_clz32(uint32_t v)
{
    uint32_t n = 0;
    if (v == 0)
        return 32;
    while (!(v & 0x80000000u)) {
        v <<= 1;
        ++n;
    }
    return n;
}

/* include/qmc/unitfloat.hpp:20-28 — bit k of the result is bit 31-k */
uint32_t qo_brev32(uint32_t v)
{
    uint32_t r = 0;
    for (int k = 0; k < 32; ++k)
        r |= ((v >> k) & 1u) << (31 - k);
    return r;
}

/* include/qmc/unitfloat.hpp:34-50 — nearest binary32 to u*2^-32 in [0,1),
 * ties on the 9 dropped bits toward zero, 0 -> 0, 1 -> 2^-32, clamp below 1. */
uint32_t qo_map_bits(uint32_t u)
{
    if (u == 0)
        return 0;
    if (u == 1)
        return 95u << 23;
    const uint32_t z = qo_clz32(u);
    const uint32_t w = u << (z + 1); /* leading one dropped */
    uint32_t bits = ((126u - z) << 23) | (w >> 9);
    if ((w & 0x1ffu) > 0x100u)
        bits += 1;
    return bits >= 0x3f800000u ? 0x3f7fffffu : bits;
}

void qo_map_range(uint32_t u0, uint64_t n, uint32_t* out)
{
    for (uint64_t k = 0; k < n; ++k)
        out[k] = qo_map_bits((uint32_t)(u0 + k));
}

/* ------------------------------------------------------------------- primes */

/* src/primes.cpp:14-44 — first 1000 primes and per prime the largest power
 * below 2^32, by trial division (computed once). */
#define QO_PRIMES 1000
static uint32_t g_primes[QO_PRIMES];
static uint32_t g_maxpow[QO_PRIMES];
static int g_primes_ready;

static void primes_init(void)
{
    if (g_primes_ready)
        return;
    uint32_t count = 0;
    for (uint32_t c = 2; count < QO_PRIMES; ++c) {
        int prime = 1;
        for (uint32_t k = 0; k < count && g_primes[k] * g_primes[k] <= c; ++k)
            if (c % g_primes[k] == 0) {
                prime = 0;
                break;
            }
        if (prime)
            g_primes[count++] = c;
    }
    for (uint32_t k = 0; k < QO_PRIMES; ++k)
        g_maxpow[k] = qo_max_power_fitting_u32(g_primes[k]);
    g_primes_ready = 1;
}

/* src/primes.cpp:50-62 */
int qo_prime(uint32_t index, uint32_t* out)
{
    primes_init();
    if (index >= QO_PRIMES)
        return 3;
    *out = g_primes[index];
    return 0;
}

int qo_prime_max_power(uint32_t index, uint32_t* out)
{
    primes_init();
    if (index >= QO_PRIMES)
        return 3;
    *out = g_maxpow[index];
    return 0;
}

/* src/primes.cpp:64-72 */
uint32_t qo_max_power_fitting_u32(uint32_t base)
{
    uint64_t p = base;
    while (p * base <= 0xffffffffull)
        p *= base;
    return (uint32_t)p;
}

/* ------------------------------------------------------------------ radical */

/* Shared digit loop of src/radical.cpp:130-181: least significant digit of
 * i becomes the most significant digit of the result, digit count >= 1, and
 * the fixed-point value is floor(result * 2^32 / base^digits). */
static uint32_t radical_core(uint32_t i, uint32_t base, uint32_t modulus, const uint32_t* sigma,
                             uint32_t factor)
{
    i %= modulus;
    uint32_t scale = 1, acc = 0;
    do {
        uint32_t digit = i % base;
        if (sigma)
            digit = sigma[digit];
        else if (factor)
            digit = (uint32_t)(((uint64_t)factor * digit) % base);
        acc = acc * base + digit;
        i /= base;
        scale *= base;
    } while (i != 0);
    return (uint32_t)(((uint64_t)acc << 32) / scale);
}

/* src/radical.cpp:130-142 */
uint32_t qo_radical_inverse_fixed(uint32_t i, uint32_t prime_index)
{
    primes_init();
    return radical_core(i, g_primes[prime_index], g_maxpow[prime_index], NULL, 0);
}

/* src/radical.cpp:144-164 — digit a -> (factor * a) mod base */
uint32_t qo_radical_inverse_linscramble_fixed(uint32_t i, uint32_t prime_index, uint32_t factor)
{
    primes_init();
    return radical_core(i, g_primes[prime_index], g_maxpow[prime_index], NULL, factor);
}

/* src/radical.cpp:166-181 */
uint32_t qo_radical_inverse_permuted_fixed(uint32_t i, uint32_t prime_index,
                                           const uint32_t* sigma)
{
    primes_init();
    return radical_core(i, g_primes[prime_index], g_maxpow[prime_index], sigma, 0);
}

/* src/radical.cpp:50-74 — sigma_2 = (0,1); even b: 2*sigma_{b/2} then
 * 2*sigma_{b/2}+1; odd b: sigma_{b-1} with values >= (b-1)/2 bumped and
 * (b-1)/2 inserted in the middle. */
void qo_faure_permutation(uint32_t base, uint32_t* out)
{
    if (base == 2) {
        out[0] = 0;
        out[1] = 1;
        return;
    }
    uint32_t* prev = (uint32_t*)malloc(sizeof(uint32_t) * base);
    if (base % 2 == 0) {
        const uint32_t h = base / 2;
        qo_faure_permutation(h, prev);
        for (uint32_t k = 0; k < h; ++k) {
            out[k] = 2 * prev[k];
            out[h + k] = 2 * prev[k] + 1;
        }
    } else {
        const uint32_t mid = (base - 1) / 2;
        qo_faure_permutation(base - 1, prev);
        uint32_t o = 0;
        for (uint32_t k = 0; k < base - 1; ++k) {
            if (k == mid)
                out[o++] = mid;
            out[o++] = prev[k] >= mid ? prev[k] + 1 : prev[k];
        }
    }
    free(prev);
}

/* src/radical.cpp:76-110 — entry v: the d base-b digits of v permuted by
 * sigma and mirrored inside the group. */
uint32_t qo_tensor_digit_table(const uint32_t* sigma, uint32_t base, uint32_t d, uint32_t* table)
{
    uint64_t group = 1;
    for (uint32_t k = 0; k < d; ++k) {
        group *= base;
        if (group > 65536u)
            return 0;
    }
    for (uint32_t v = 0; v < group; ++v) {
        uint32_t rem = v, out = 0;
        for (uint32_t k = 0; k < d; ++k) {
            out = out * base + sigma[rem % base];
            rem /= base;
        }
        table[v] = out;
    }
    return (uint32_t)group;
}

/* src/radical.cpp:183-208 — count digits, invert full groups by table,
 * then the remaining most significant digits singly. */
uint32_t qo_radical_inverse_tabled_fixed(uint32_t i, uint32_t base, uint32_t digits_per_step,
                                         const uint32_t* table, const uint32_t* sigma)
{
    uint32_t group = 1;
    for (uint32_t k = 0; k < digits_per_step; ++k)
        group *= base;
    i %= qo_max_power_fitting_u32(base);
    uint32_t digits = 1;
    for (uint32_t v = i / base; v; v /= base)
        ++digits;
    uint32_t scale = 1, acc = 0;
    for (uint32_t g = digits / digits_per_step; g; --g) {
        acc = acc * group + table[i % group];
        i /= group;
        scale *= group;
    }
    for (uint32_t r = digits % digits_per_step; r; --r) {
        acc = acc * base + sigma[i % base];
        i /= base;
        scale *= base;
    }
    return (uint32_t)(((uint64_t)acc << 32) / scale);
}

/* --------------------------------------------------------------- digitalnet */

/* src/digitalnet.cpp:79-109 — 52 MSB-aligned column words per dimension;
 * dimension 0 is the identity (zero past column 31); dimension j >= 1 takes
 * m_k << (31-k) for k < s and the primitive-polynomial recurrence beyond. */
void qo_build_matrices(uint32_t dims, const uint32_t* s, const uint32_t* a,
                       const uint32_t* const* m, uint32_t* columns)
{
    memset(columns, 0, sizeof(uint32_t) * 52u * dims);
    if (dims == 0)
        return;
    for (uint32_t k = 0; k < 32; ++k)
        columns[k] = 0x80000000u >> k;
    for (uint32_t j = 1; j < dims; ++j) {
        uint32_t* v = columns + 52u * j;
        const uint32_t deg = s[j - 1], poly = a[j - 1];
        for (uint32_t k = 0; k < deg && k < 52; ++k)
            v[k] = m[j - 1][k] << (31 - k);
        for (uint32_t k = deg; k < 52; ++k) {
            uint32_t x = v[k - deg] ^ (v[k - deg] >> deg);
            for (uint32_t l = 1; l < deg; ++l)
                if ((poly >> (deg - 1 - l)) & 1u)
                    x ^= v[k - l];
            v[k] = x;
        }
    }
}

/* src/digitalnet.cpp:111-131 — scramble XOR the columns selected by the
 * index bits (low 32, then the high 20). */
uint32_t qo_sobol_component_fixed(uint64_t i, const uint32_t* c, uint32_t scramble)
{
    uint32_t r = scramble;
    for (uint32_t k = 0; k < 52 && i; ++k, i >>= 1)
        if (i & 1u)
            r ^= c[k];
    return r;
}

void qo_sobol_fill_fixed(uint64_t first, uint64_t n, uint32_t dims, const uint32_t* columns,
                         const uint32_t* scrambles, uint32_t* out)
{
    for (uint64_t k = 0; k < n; ++k)
        for (uint32_t j = 0; j < dims; ++j)
            out[k * dims + j] = qo_sobol_component_fixed(first + k, columns + 52u * j,
                                                         scrambles ? scrambles[j] : 0u);
}

/* sobol_point as floats (digitalnet.cpp:141-151 + unitfloat.hpp:34-50): the
 * CPU "port" timing of bench.py --impl reference when the reference build is
 * absent (the checker is never the thing measured on the GPU side). */
void qo_sobol_fill_f32(uint64_t first, uint64_t n, uint32_t dims, const uint32_t* columns,
                       const uint32_t* scrambles, float* out)
{
    for (uint64_t k = 0; k < n; ++k)
        for (uint32_t j = 0; j < dims; ++j) {
            const uint32_t b = qo_map_bits(qo_sobol_component_fixed(
                first + k, columns + 52u * j, scrambles ? scrambles[j] : 0u));
            memcpy(out + k * dims + j, &b, 4);
        }
}

/* Hash-based Owen scrambling — BUILDER-DEFINED, no reference counterpart
 * (SPEC.md:271 lists Owen trees as a non-goal). The 32-bit
 * fixed-point value v is bit-reversed, so digit k (from the most significant
 * end) sits at bit k; then a hash whose every step keeps "output bit k =
 * input bit k XOR f(input bits < k, seed)" (x ^= x*even, x += c, x *= odd)
 * flips each digit as a function of the seed and all preceding digits, which
 * is the nested-uniform (Owen) structure; finally reversed back. Constants:
 * Vegdahl, "Building a Better LK Hash" (2021), an improved Laine-Karras hash. */
uint32_t qo_owen_scramble(uint32_t v, uint32_t seed)
{
    uint32_t x = qo_brev32(v);
    x ^= x * 0x3d20adeau;
    x += seed;
    x *= (seed >> 16) | 1u;
    x ^= x * 0x05526c56u;
    x ^= x * 0x53a22864u;
    return qo_brev32(x);
}

void qo_sobol_owen_fill_fixed(uint64_t first, uint64_t n, uint32_t dims, const uint32_t* columns,
                              const uint32_t* seeds, uint32_t* out)
{
    for (uint64_t k = 0; k < n; ++k)
        for (uint32_t j = 0; j < dims; ++j)
            out[k * dims + j] = qo_owen_scramble(
                qo_sobol_component_fixed(first + k, columns + 52u * j, 0u), seeds[j]);
}

/* ------------------------------------------------------------------ lattice */

/* include/qmc/lattice.hpp:31-34 — brev(i) * g mod 2^32 */
uint32_t qo_lattice_component_fixed(uint32_t i, uint32_t g) { return qo_brev32(i) * g; }

/* Integer Cranley-Patterson rotation: (phi_2(i) g + s) mod 1 in 32-bit
 * fixed point — the composition lattice_component_fixed + wrapping add
 * (SURVEY §8a A14). s = 0 is the plain lattice. */
uint32_t qo_lattice_cp_fixed(uint32_t i, uint32_t g, uint32_t shift)
{
    return qo_brev32(i) * g + shift;
}

/* src/lattice.cpp:59-67 — murmur3 fmix32 */
static uint32_t fmix32(uint32_t h)
{
    h = (h ^ (h >> 16)) * 0x85ebca6bu;
    h = (h ^ (h >> 13)) * 0xc2b2ae35u;
    return h ^ (h >> 16);
}

/* src/lattice.cpp:71-77 */
uint32_t qo_pixel_hash(uint32_t j, uint32_t px, uint32_t py)
{
    return fmix32(fmix32(fmix32(0x9e3779b9u ^ j) ^ px) ^ py);
}

/* include/qmc/lattice.hpp:51-56 — g = hash | 1, index enumerated backwards */
uint32_t qo_random_lattice_component_fixed(uint32_t i, uint32_t j, uint32_t px, uint32_t py)
{
    return qo_brev32(~i) * (qo_pixel_hash(j, px, py) | 1u);
}

/* src/lattice.cpp:81-104 — g_0 = 1, g_j = 2*xorshift32(13,17,5) + 1 */
int qo_lfsr_generator_vector(uint32_t seed, uint32_t dims, uint32_t* out)
{
    if (seed == 0 || dims < 1)
        return 2;
    out[0] = 1;
    uint32_t x = seed;
    for (uint32_t j = 1; j < dims; ++j) {
        x ^= x << 13;
        x ^= x >> 17;
        x ^= x << 5;
        out[j] = 2u * x + 1u;
    }
    return 0;
}

/* src/lattice.cpp:157-170 — Delta_k = brev(k * 2^m) * g */
int qo_lattice_shift_fixed(uint32_t k, uint32_t m, const uint32_t* g, uint32_t dims,
                           uint32_t* out)
{
    if (m > 32)
        return 2;
    const uint64_t scaled = (uint64_t)k << m;
    if (scaled > 0xffffffffull)
        return 4;
    const uint32_t r = qo_brev32((uint32_t)scaled);
    for (uint32_t j = 0; j < dims; ++j)
        out[j] = r * g[j];
    return 0;
}

/* ---------------------------------------------------------------- hilbert */

/* include/qmc/hilbert.hpp:39-56 — orientation (0,0),(0,1),(1,1),(1,0) */
int qo_hilbert_index(uint32_t x, uint32_t y, uint32_t order, uint64_t* out)
{
    if (order == 0 || order > 31)
        return 2;
    const uint32_t n = 1u << order;
    if (x >= n || y >= n)
        return 3;
    uint64_t d = 0;
    for (uint32_t s = n >> 1; s; s >>= 1) {
        const uint32_t rx = (x & s) != 0, ry = (y & s) != 0;
        d += (uint64_t)s * s * ((3u * rx) ^ ry);
        if (!ry) {
            if (rx) {
                x = n - 1 - x;
                y = n - 1 - y;
            }
            const uint32_t t = x;
            x = y;
            y = t;
        }
    }
    *out = d;
    return 0;
}

/* include/qmc/hilbert.hpp:59-78 */
int qo_hilbert_xy(uint64_t d, uint32_t order, uint32_t* px, uint32_t* py)
{
    if (order == 0 || order > 31)
        return 2;
    if (d >= (1ull << (2 * order)))
        return 3;
    const uint32_t n = 1u << order;
    uint32_t x = 0, y = 0;
    for (uint32_t s = 1; s < n; s <<= 1) {
        const uint32_t rx = 1u & (uint32_t)(d >> 1);
        const uint32_t ry = 1u & (uint32_t)(d ^ rx);
        if (!ry) {
            if (rx) {
                x = s - 1 - x;
                y = s - 1 - y;
            }
            const uint32_t t = x;
            x = y;
            y = t;
        }
        x += s * rx;
        y += s * ry;
        d >>= 2;
    }
    *px = x;
    *py = y;
    return 0;
}

/* src/imageplane.cpp:16-21 — phi_3 of the Hilbert index (the reference
 * inverts four ternary digits per step through the identity base-81 table,
 * which equals plain phi_3: SPEC acceptance 2). */
uint32_t qo_hilbert_phi3_fixed(uint32_t x, uint32_t y, uint32_t order)
{
    uint64_t h = 0;
    qo_hilbert_index(x, y, order, &h);
    static const uint32_t id3[3] = {0, 1, 2};
    uint32_t table[81];
    qo_tensor_digit_table(id3, 3, 4, table);
    return qo_radical_inverse_tabled_fixed((uint32_t)h, 3, 4, table, id3);
}

/* src/imageplane.cpp:43-51 */
uint64_t qo_digit_reverse(uint64_t v, uint32_t base, uint32_t digits)
{
    uint64_t r = 0;
    for (uint32_t k = 0; k < digits; ++k) {
        r = r * base + v % base;
        v /= base;
    }
    return r;
}

/* a^-1 mod n by the iterative extended Euclid (imageplane.cpp:55-76). */
static uint64_t inverse_mod(uint64_t a, uint64_t n)
{
    if (n == 1)
        return 0;
    int64_t r0 = (int64_t)n, r1 = (int64_t)(a % n), t0 = 0, t1 = 1;
    while (r1) {
        const int64_t q = r0 / r1, r2 = r0 - q * r1, t2 = t0 - q * t1;
        r0 = r1;
        r1 = r2;
        t0 = t1;
        t1 = t2;
    }
    const int64_t m = (int64_t)n;
    return (uint64_t)(((t0 % m) + m) % m);
}

/* src/imageplane.cpp:80-98 */
int qo_halton_enum_init(uint32_t width, uint32_t height, qo_halton_enum* e)
{
    if (width == 0 || height == 0 || width > (1u << 20) || height > 1594323u)
        return 1;
    e->scale_x = e->scale_y = 1;
    e->exp_x = e->exp_y = 0;
    while (e->scale_x < width) {
        e->scale_x *= 2;
        ++e->exp_x;
    }
    while (e->scale_y < height) {
        e->scale_y *= 3;
        ++e->exp_y;
    }
    e->stride = (uint64_t)e->scale_x * e->scale_y;
    e->crt_x = e->scale_y * inverse_mod(e->scale_y % e->scale_x, e->scale_x);
    e->crt_y = e->scale_x * inverse_mod(e->scale_x % e->scale_y, e->scale_y);
    return 0;
}

/* src/imageplane.cpp:100-106 */
uint64_t qo_halton_enum_offset(const qo_halton_enum* e, uint32_t px, uint32_t py)
{
    const uint64_t r2 = qo_digit_reverse(px, 2, e->exp_x);
    const uint64_t r3 = qo_digit_reverse(py, 3, e->exp_y);
    return (r2 * e->crt_x % e->stride + r3 * e->crt_y % e->stride) % e->stride;
}

/* src/imageplane.cpp:114-130 */
int qo_partition(uint32_t part, uint32_t parts, uint32_t base, uint64_t* rem, uint64_t* mod)
{
    if (base < 2)
        return 2;
    uint32_t k = 0;
    uint64_t p = 1;
    while (p < parts) {
        p *= base;
        ++k;
    }
    if (p != parts)
        return 1;
    if (part >= parts)
        return 3;
    *rem = qo_digit_reverse(part, base, k);
    *mod = parts;
    return 0;
}

/* ------------------------------------------------------------------- render */

/* src/render.cpp:17-26 with the constants of include/qmc/render.hpp:24-27 */
double qo_scene_value(double x, double y)
{
    const double pi = 3.14159265358979323846;
    const double s = sin(8.0 * pi * x) * sin(8.0 * pi * y);
    double v = 0.5 * (1.0 + s);
    const double dx = x - 0.5, dy = y - 0.5;
    if (dx * dx + dy * dy < 0.3 * 0.3)
        v += 0.25;
    return v;
}

/* src/render.cpp:28-34 */
uint32_t qo_hilbert_order_for(uint32_t w, uint32_t h)
{
    uint32_t o = 1;
    while ((1u << o) < w || (1u << o) < h)
        ++o;
    return o;
}

static float map_float(uint32_t u)
{
    const uint32_t b = qo_map_bits(u);
    float f;
    memcpy(&f, &b, 4);
    return f;
}

/* render.cpp:38-143 for one pixel with the per-kind stream state of
 * imageplane.cpp:310-461 (dims = 2). */
int qo_render(uint32_t w, uint32_t h, uint32_t spp, int kind, int accum, uint32_t seed,
              const uint32_t* cols2, float* out)
{
    if (w == 0 || h == 0 || spp == 0)
        return 1;
    const uint32_t order = qo_hilbert_order_for(w, h);
    uint32_t g[2];
    qo_lfsr_generator_vector(seed ? seed : 0xace1u, 2, g);
    uint32_t scr[2] = {0, 0};
    if (kind == QO_SOBOL && seed) {
        scr[0] = qo_pixel_hash(0, seed, 0);
        scr[1] = qo_pixel_hash(1, seed, 0);
    }
    qo_halton_enum he;
    if (kind == QO_IMAGE_PLANE_HALTON && qo_halton_enum_init(w, h, &he))
        return 1;
    const double inv_w = 1.0 / w, inv_h = 1.0 / h;
    for (uint32_t py = 0; py < h; ++py)
        for (uint32_t px = 0; px < w; ++px) {
            uint32_t shift = 0;
            uint64_t block = 0, offset = 0;
            if (kind == QO_PIXEL_SHIFTED_LATTICE)
                shift = qo_hilbert_phi3_fixed(px, py, order);
            if (kind == QO_HALTON_HILBERT) {
                qo_hilbert_index(px, py, order, &block);
                block *= spp;
            }
            if (kind == QO_IMAGE_PLANE_HALTON)
                offset = qo_halton_enum_offset(&he, px, py);
            double sum = 0.0, comp = 0.0;
            int64_t isum = 0;
            for (uint32_t i = 0; i < spp; ++i) {
                float uv[2];
                for (uint32_t j = 0; j < 2; ++j) {
                    uint32_t fx = 0;
                    switch (kind) {
                    case QO_SOBOL: fx = qo_sobol_component_fixed(i, cols2 + 52 * j, scr[j]); break;
                    case QO_HALTON: fx = qo_radical_inverse_fixed(i, j); break;
                    case QO_LATTICE: fx = qo_lattice_component_fixed(i, g[j]); break;
                    case QO_HALTON_HILBERT:
                        fx = qo_radical_inverse_fixed((uint32_t)(block + i), j);
                        break;
                    case QO_PIXEL_SHIFTED_LATTICE: fx = (qo_brev32(i) + shift) * g[j]; break;
                    case QO_PIXEL_RANDOM_LATTICE:
                        fx = qo_random_lattice_component_fixed(i, j, px, py);
                        break;
                    case QO_IMAGE_PLANE_HALTON: {
                        const uint64_t gl = offset + (uint64_t)i * he.stride;
                        fx = j == 0 ? qo_radical_inverse_fixed((uint32_t)(gl >> he.exp_x), 0)
                                    : qo_radical_inverse_fixed((uint32_t)(gl / he.scale_y), 1);
                        break;
                    }
                    default: return 2;
                    }
                    uv[j] = map_float(fx);
                }
                const double u = uv[0], v = uv[1];
                const double f = qo_scene_value((px + u) * inv_w, (py + v) * inv_h);
                if (accum == 0) { /* quality.hpp:22-30 Neumaier */
                    const double t = sum + f;
                    if (fabs(sum) >= fabs(f))
                        comp += (sum - t) + f;
                    else
                        comp += (f - t) + sum;
                    sum = t;
                } else {
                    isum += llround(f * 4294967296.0);
                }
            }
            out[(uint64_t)py * w + px] = accum == 0
                                             ? (float)((sum + comp) / spp)
                                             : (float)((double)isum / 4294967296.0 / spp);
        }
    return 0;
}

/* Int-mode render restricted to the samples i == rem (mod mod) — the
 * per-part accumulators of the paper's sample partition;
 * int64 sums of llround(f * 2^32) per pixel (render.cpp:72-78). */
int qo_render_partial_int(uint32_t w, uint32_t h, uint32_t spp, int kind, uint32_t seed,
                          const uint32_t* cols2, uint32_t rem, uint32_t mod, int64_t* acc)
{
    /* render the per-sample values through qo_render's sampling by running
     * one-sample renders is wasteful; restate the loop directly */
    if (w == 0 || h == 0 || spp == 0 || mod == 0)
        return 1;
    const uint32_t order = qo_hilbert_order_for(w, h);
    uint32_t g[2];
    qo_lfsr_generator_vector(seed ? seed : 0xace1u, 2, g);
    uint32_t scr[2] = {0, 0};
    if (kind == QO_SOBOL && seed) {
        scr[0] = qo_pixel_hash(0, seed, 0);
        scr[1] = qo_pixel_hash(1, seed, 0);
    }
    qo_halton_enum he;
    if (kind == QO_IMAGE_PLANE_HALTON && qo_halton_enum_init(w, h, &he))
        return 1;
    const double inv_w = 1.0 / w, inv_h = 1.0 / h;
    for (uint32_t py = 0; py < h; ++py)
        for (uint32_t px = 0; px < w; ++px) {
            uint32_t shift = 0;
            uint64_t block = 0, offset = 0;
            if (kind == QO_PIXEL_SHIFTED_LATTICE)
                shift = qo_hilbert_phi3_fixed(px, py, order);
            if (kind == QO_HALTON_HILBERT) {
                qo_hilbert_index(px, py, order, &block);
                block *= spp;
            }
            if (kind == QO_IMAGE_PLANE_HALTON)
                offset = qo_halton_enum_offset(&he, px, py);
            int64_t isum = 0;
            for (uint32_t i = rem; i < spp; i += mod) {
                float uv[2];
                for (uint32_t j = 0; j < 2; ++j) {
                    uint32_t fx = 0;
                    switch (kind) {
                    case QO_SOBOL: fx = qo_sobol_component_fixed(i, cols2 + 52 * j, scr[j]); break;
                    case QO_HALTON: fx = qo_radical_inverse_fixed(i, j); break;
                    case QO_LATTICE: fx = qo_lattice_component_fixed(i, g[j]); break;
                    case QO_HALTON_HILBERT:
                        fx = qo_radical_inverse_fixed((uint32_t)(block + i), j);
                        break;
                    case QO_PIXEL_SHIFTED_LATTICE: fx = (qo_brev32(i) + shift) * g[j]; break;
                    case QO_PIXEL_RANDOM_LATTICE:
                        fx = qo_random_lattice_component_fixed(i, j, px, py);
                        break;
                    case QO_IMAGE_PLANE_HALTON: {
                        const uint64_t gl = offset + (uint64_t)i * he.stride;
                        fx = j == 0 ? qo_radical_inverse_fixed((uint32_t)(gl >> he.exp_x), 0)
                                    : qo_radical_inverse_fixed((uint32_t)(gl / he.scale_y), 1);
                        break;
                    }
                    default: return 2;
                    }
                    uv[j] = map_float(fx);
                }
                const double u = uv[0], v = uv[1];
                isum += llround(qo_scene_value((px + u) * inv_w, (py + v) * inv_h) * 4294967296.0);
            }
            acc[(uint64_t)py * w + px] = isum;
        }
    return 0;
}

/* src/image.cpp:54-63 */
uint64_t qo_fnv1a64(const void* data, uint64_t size)
{
    const unsigned char* p = (const unsigned char*)data;
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t k = 0; k < size; ++k) {
        h ^= p[k];
        h *= 0x100000001b3ull;
    }
    return h;
}
