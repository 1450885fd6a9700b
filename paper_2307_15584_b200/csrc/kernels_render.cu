// kernels_render.cu — per-pixel sample enumeration and the fused per-pixel
// integro-approximation (config C5) for sm_100a.
//
// render: one thread owns one pixel of the band, derives its pixel state
// (Hilbert index + phi_3 shift, Halton CRT offset, hashed generator) on the
// device, and walks its spp samples in the reference order (render.cpp:
// 58-79): sample -> scene_value in FP64 -> Neumaier (or int64 fixed-point)
// accumulation -> one fp32 store. Points are never materialised; the only
// HBM traffic is the 4 B per pixel image write. The per-pixel sequential sum
// keeps the reference's summation order, so the Kahan path only differs from
// the CPU where device sin() differs from libm's.
#include <cstdint>

#include <type_traits>

#include "device.cuh"
#include "internal.hpp"

namespace qmcgpu {

namespace {

constexpr int kBlock = 128;

// Per-pixel state of the SampleStream kinds (imageplane.cpp:366-405).
struct PixelState {
    uint32_t shift;     // pixel_shifted_lattice
    uint32_t g0, g1;    // pixel_random_lattice (hash | 1)
    uint64_t block;     // halton_hilbert: hilbert_index * spp
    uint32_t ipx0, ipy0; // image_plane_halton: (uint32)(offset >> a), (uint32)(offset / 3^b)
    uint32_t cell;      // sobol_xor_table: tile cell
};

__device__ __forceinline__ uint64_t digit_reverse(uint64_t v, uint32_t base, uint32_t digits)
{
    uint64_t r = 0;
    for (uint32_t k = 0; k < digits; ++k) {
        r = r * base + v % base;
        v /= base;
    }
    return r;
}

// a mod m for a < 2^64 and m < 2^32 with mg = floor((2^64 - 1) / m): the
// multiply-high quotient is at most two low
__device__ __forceinline__ uint64_t mod_by_magic(uint64_t a, uint64_t m, uint64_t mg)
{
    uint64_t r = a - __umul64hi(a, mg) * m;
    r = r >= m ? r - m : r;
    return r >= m ? r - m : r;
}

// imageplane.cpp:100-106: CRT combination of the reversed digits. mg: the
// magic of a stride below 2^32 (every image up to 2^16 x 3^10 pixels, 4K
// included), else 0 and the plain 64-bit remainders
__device__ __forceinline__ uint64_t halton_offset(uint32_t px, uint32_t py, uint32_t exp_x,
                                                  uint32_t exp_y, uint64_t stride, uint64_t crt_x,
                                                  uint64_t crt_y, uint64_t mg)
{
    if (mg != 0) {
        const uint64_t r2 = exp_x == 0 ? 0 : __brevll(px) >> (64 - exp_x);
        uint32_t r3 = 0, v = py;
        for (uint32_t k = 0; k < exp_y; ++k) { // digit_reverse(py, 3, exp_y) in 32 bits
            const uint32_t q = __umulhi(v, 0xaaaaaaabu) >> 1;
            r3 = r3 * 3u + (v - 3u * q);
            v = q;
        }
        const uint64_t s = mod_by_magic(r2 * crt_x, stride, mg) +
                           mod_by_magic(static_cast<uint64_t>(r3) * crt_y, stride, mg);
        return s >= stride ? s - stride : s;
    }
    // digit_reverse(px, 2, exp_x) = the exp_x low bits of px mirrored
    const uint64_t r2 = exp_x == 0 ? 0 : __brevll(px) >> (64 - exp_x);
    const uint64_t r3 = digit_reverse(py, 3, exp_y);
    return (r2 * crt_x % stride + r3 * crt_y % stride) % stride;
}

template <uint32_t KIND>
__device__ __forceinline__ PixelState pixel_state(uint32_t px, uint32_t py, const RenderParams& p)
{
    PixelState s{};
    if (KIND == 4) // pixel_shifted_lattice: phi_3(hilbert_index), imageplane.cpp:16-21
        s.shift = phi3_fixed(static_cast<uint32_t>(hilbert_index(px, py, p.order)), p.tab3);
    if (KIND == 5) { // pixel_random_lattice, lattice.hpp:51-56
        s.g0 = pixel_hash(0, px, py) | 1u;
        s.g1 = pixel_hash(1, px, py) | 1u;
    }
    if (KIND == 3) // halton_hilbert, imageplane.cpp:373-379
        s.block = hilbert_index(px, py, p.order) * p.spp;
    if (KIND == 6) {
        const uint64_t off =
            halton_offset(px, py, p.exp_x, p.exp_y, p.stride, p.crt_x, p.crt_y, p.stride_magic);
        s.ipx0 = static_cast<uint32_t>(off >> p.exp_x);
        s.ipy0 = static_cast<uint32_t>(off / p.scale_y);
    }
    if (KIND == 7)
        s.cell = (px % 128u) + (py % 128u) * 128u;
    return s;
}

__device__ __forceinline__ uint32_t rad2(uint32_t i) { return brev32(i & 0x7fffffffu); }

// Component j in {0,1} of sample i (SampleStream::sample, imageplane.cpp:
// 427-461) at the integer stage, for the render's 2-dim streams.
// SMEM_T3: t3 is a shared-memory copy of the 3^7-entry phi_3 table.
// phi_3 (u32 fixed point) of n = hi * 3^7 + lo < 3^14 from the quotient
// tables q3 = [floor(T[v] 2^32 / 3^7) | floor(T[v] 2^32 / 3^14)], T the
// 7-digit reversal: phi_3(n) = floor(2^32 (T[lo] / 3^7 + T[hi] / 3^14)). With
// S = q3[lo] + q3[3^7 + hi], the dropped fractions sum to F / 3^14 with
// F < 2 * 3^14 < 2^32 and 3^14 (S + F / 3^14) = 2^32 (T[lo] 3^7 + T[hi]), so
// F = -3^14 S mod 2^32 and phi_3(n) = S + (F >= 3^14) — the same value as
// phi3_fixed's two-step branch (frac_div_magic of T[lo] 3^7 + T[hi]).
// a_lo, a_hi: the shared-memory addresses of q3[lo] and q3[3^7 + hi].
__device__ __forceinline__ uint32_t lds_u32(uint32_t a)
{
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a)); // read-only after staging
    return v;
}
__device__ __forceinline__ uint32_t phi3_q(uint32_t a_lo, uint32_t a_hi)
{
    const uint32_t s = lds_u32(a_lo) + lds_u32(a_hi);
    return s + (s * (0u - 4782969u) >= 4782969u ? 1u : 0u);
}

// INC3 (KIND 1 and 6): sob0 / sob1 carry the shared-memory addresses of
// q3[lo] and q3[3^7 + hi] for the (lo, hi) base-3^7 digits of the phi_3
// index, advanced by the caller.
// INC3 with KIND 3 (halton_hilbert, n = block + i up to 3^20): sob1 is the
// shared-memory address of q3[lo] for n = H * 3^7 + lo and rec = {floor(W /
// 3^7), 2^32 - (3^7 - W mod 3^7)} with W = phi_3(H): phi_3(n) = q3[lo] +
// rec.x + (r >= 3^7 - W mod 3^7), r = -q3[lo] * 3^7 mod 2^32 (the split of
// the level-table Halton fill, kernels_fill.cu k_halton_lv, with G0 = 3^7).
template <uint32_t KIND, bool SMEM_T3 = false, bool INC3 = false>
__device__ __forceinline__ void sample2(uint32_t i, const PixelState& s, const RenderParams& p,
                                        uint32_t& x0, uint32_t& x1, uint32_t& sob0,
                                        uint32_t& sob1, const uint32_t* t3, uint2 rec = {})
{
    if (INC3 && KIND == 3) {
        x0 = rad2(static_cast<uint32_t>(s.block + i));
        const uint32_t q = lds_u32(sob1);
        uint32_t dummy;
        asm("{\n\t"
            "add.cc.u32 %1, %2, %3;\n\t"
            "addc.u32 %0, %4, %5;\n\t}"
            : "=r"(x1), "=r"(dummy)
            : "r"(q * (0u - 2187u)), "r"(rec.y), "r"(q), "r"(rec.x));
    } else if (INC3 && (KIND == 1 || KIND == 6)) {
        x0 = KIND == 1 ? rad2(i) : rad2(s.ipx0 + i * p.scale_y);
        x1 = phi3_q(sob0, sob1);
    } else if (KIND == 0) { // sobol: natural-order incremental, caller advances
        x0 = sob0;
        x1 = sob1;
    } else if (KIND == 1) { // halton (plain)
        x0 = rad2(i);
        x1 = phi3_fixed<SMEM_T3>(i, t3);
    } else if (KIND == 2) { // lattice
        const uint32_t b = brev32(i);
        x0 = b * p.g0;
        x1 = b * p.g1;
    } else if (KIND == 3) { // halton_hilbert
        const uint32_t gi = static_cast<uint32_t>(s.block + i);
        x0 = rad2(gi);
        x1 = phi3_fixed<SMEM_T3>(gi, t3);
    } else if (KIND == 4) { // pixel_shifted_lattice (Eq. 3)
        const uint32_t b = brev32(i) + s.shift;
        x0 = b * p.g0;
        x1 = b * p.g1;
    } else if (KIND == 5) { // pixel_random_lattice (backwards)
        const uint32_t b = brev32(~i);
        x0 = b * s.g0;
        x1 = b * s.g1;
    } else if (KIND == 6) { // image_plane_halton: (offset + i*stride)>>a, / 3^b
        x0 = rad2(s.ipx0 + i * p.scale_y);
        x1 = phi3_fixed<SMEM_T3>(s.ipy0 + i * p.scale_x, t3);
    } else { // sobol_xor_table, imageplane.cpp:231-243
        const uint32_t k = i ^ __ldg(p.xor_reorder + s.cell);
        const uint64_t pk = static_cast<uint64_t>(k) * p.xor_dims;
        const uint32_t sc = s.cell * p.xor_dims;
        x0 = __ldg(p.xor_points + pk) ^ __ldg(p.xor_scramble + sc);
        x1 = __ldg(p.xor_points + pk + 1) ^ __ldg(p.xor_scramble + sc + 1);
    }
}

// ---- per-pixel building blocks shared by the render kernels

// Pixel of band index q (row-major over rows [row_begin, row_end)).
__device__ __forceinline__ void band_pixel(uint64_t q, const RenderParams& p, uint32_t& px,
                                           uint32_t& py)
{
    if (p.small_band) { // a 32-bit multiply-high instead of a 64-bit division
        const uint32_t q32 = static_cast<uint32_t>(q);
        const uint32_t r = p.width == 1 ? q32 : div32(q32, p.divw);
        py = p.row_begin + r;
        px = q32 - r * p.width;
        return;
    }
    py = p.row_begin + static_cast<uint32_t>(q / p.width);
    px = static_cast<uint32_t>(q % p.width);
}

// Direct Sobol' value (both render dims) of index i (digitalnet.cpp:111-131).
__device__ __forceinline__ void sobol_direct2(uint32_t i, const RenderParams& p, uint32_t& s0,
                                              uint32_t& s1)
{
    s0 = p.scr0;
    s1 = p.scr1;
    for (uint32_t k = 0, v = i; v; ++k, v >>= 1)
        if (v & 1u) {
            s0 ^= __ldg(p.cols2 + k);
            s1 ^= __ldg(p.cols2 + 52 + k);
        }
}

// scene_value at sample i of the pixel (render.cpp:61-68): the two fp32
// sample components, the sample point ((px + u) / W, (py + v) / H) in FP64
// and the integrand. sob0/sob1: the Sobol' value of index i (KIND 0).
// UQ >= 0: the warp shares qx and qy, UQ = their parities (scene_value_uq).
template <uint32_t KIND, bool DISC_TEST = true, bool FIXED_Q = false, bool SMEM_T3 = false,
          int UQ = -1, bool INC3 = false>
__device__ __forceinline__ double pixel_sample(uint32_t i, const PixelState& s,
                                               const RenderParams& p, double fx, double fy,
                                               const double2* s_poly, uint32_t sob0,
                                               uint32_t sob1, bool inside_px = false, int qx = 0,
                                               int qy = 0, const uint32_t* s_tab3 = nullptr,
                                               uint2 rec = {})
{
    uint32_t a, b;
    sample2<KIND, SMEM_T3, INC3>(i, s, p, a, b, sob0, sob1, SMEM_T3 || INC3 ? s_tab3 : p.tab3,
                                 rec);
    const double u = static_cast<double>(map_u32(a));
    const double v = static_cast<double>(map_u32(b));
    const double x = __dmul_rn(__dadd_rn(fx, u), p.inv_w);
    const double y = __dmul_rn(__dadd_rn(fy, v), p.inv_h);
    if constexpr (UQ >= 0)
        return scene_value_uq<UQ, DISC_TEST>(x, y, p.sc, inside_px, qx, qy);
    else
        return scene_value<true, DISC_TEST, FIXED_Q>(x, y, p.sc, s_poly, inside_px, qx, qy);
}

// render.cpp:72-78: llround(f * 2^32), the int accumulator's term.
__device__ __forceinline__ long long int_term(double f)
{
    return llround(__dmul_rn(f, 4294967296.0));
}

// float(value() / spp) (kahan) and float(sum / 2^32 / spp) (int).
// x / spp; when spp is a power of two the quotient is exact, so the product
// with the exact reciprocal inv_spp is the same double without a DDIV
__device__ __forceinline__ double div_spp(double x, uint32_t spp, double inv_spp)
{
    return inv_spp != 0.0 ? __dmul_rn(x, inv_spp) : __ddiv_rn(x, static_cast<double>(spp));
}
__device__ __forceinline__ float finish_kahan(double sum, double comp, uint32_t spp,
                                              double inv_spp = 0.0)
{
    return __double2float_rn(div_spp(__dadd_rn(sum, comp), spp, inv_spp));
}
__device__ __forceinline__ float finish_int(long long isum, uint32_t spp, double inv_spp = 0.0)
{
    // / 2^32 is exact (a power of two)
    return __double2float_rn(
        div_spp(__dmul_rn(static_cast<double>(isum), 0x1p-32), spp, inv_spp));
}

// The sequential per-pixel sample loop of k_render (render.cpp:61-78).
// INC3: s_tab3 is the q3 quotient table and the phi_3 index advances as
// base-3^7 digits (the caller checked that it stays below 3^14).
template <uint32_t KIND, uint32_t ACCUM, bool DISC_TEST, bool FIXED_Q, int UQ = -1,
          bool INC3 = false>
__device__ __forceinline__ float render_pixel(const PixelState& s, const RenderParams& p,
                                              double fx, double fy, const double2* s_poly,
                                              const uint32_t* sob_d, bool inside_px, int qx,
                                              int qy, const uint32_t* s_tab3)
{
    constexpr bool kSmemT3 = KIND == 1 || KIND == 3 || KIND == 6;
    uint32_t sob0 = p.scr0, sob1 = p.scr1; // sobol index 0 value
    uint32_t dlo = 0, dhi = 0, a_end = 0;
    uint2 rec{}, rec2{}; // halton_hilbert: the records of H and H + 1
    if (INC3 && KIND == 3) {
        // n0 = the pixel's first index mod 3^20 (render_classified checked
        // that its spp indices neither cross 3^20 nor wrap u32, spp <= 2187)
        uint32_t n0 = static_cast<uint32_t>(s.block);
        if (n0 >= 3486784401u)
            n0 -= 3486784401u;
        const uint32_t H = n0 / 2187u, base = static_cast<uint32_t>(__cvta_generic_to_shared(s_tab3));
        sob1 = base + 4u * (n0 - 2187u * H);
        a_end = base + 4u * 2187u;
        const uint32_t* t7 = s_tab3 - 2188; // RenderSmem: tab3 (2188 words) precedes q3
        const uint32_t W = phi3_fixed<true>(H, t7), W2 = phi3_fixed<true>(H + 1u, t7);
        const uint32_t qw = W / 2187u, qw2 = W2 / 2187u;
        rec = make_uint2(qw, 0u - (2187u - (W - 2187u * qw)));
        rec2 = make_uint2(qw2, 0u - (2187u - (W2 - 2187u * qw2)));
    } else if (INC3) { // image-plane halton: n = ipy0 + i * scale_x; halton: n = i
        const uint32_t n0 = KIND == 6 ? s.ipy0 : 0u;
        const uint32_t hi = n0 / 2187u, base = static_cast<uint32_t>(__cvta_generic_to_shared(s_tab3));
        sob0 = base + 4u * (n0 - 2187u * hi);
        sob1 = base + 4u * (2187u + hi);
        a_end = base + 4u * 2187u;
        dlo = 4u * (KIND == 6 ? p.dlo3 : 1u);
        dhi = 4u * (KIND == 6 ? p.dhi3 : 0u);
    }
    double sum = 0.0, comp = 0.0;
    long long isum = 0;
    // BIG: Neumaier's |sum| >= |v| branch is known to hold
    auto run = [&](uint32_t i0, uint32_t i1, auto big) {
#pragma unroll 2
        for (uint32_t i = i0; i < i1; ++i) {
            const double f = pixel_sample<KIND, DISC_TEST, FIXED_Q, kSmemT3, UQ, INC3>(
                i, s, p, fx, fy, s_poly, sob0, sob1, inside_px, qx, qy, s_tab3, rec);
            if (ACCUM != 0)
                isum += int_term(f);
            else if (decltype(big)::value)
                neumaier_add_big(sum, comp, f);
            else
                neumaier_add(sum, comp, f);
            if (INC3 && KIND == 3) {
                sob1 += 4u;
                if (sob1 >= a_end) {
                    sob1 -= 4u * 2187u;
                    rec = rec2;
                }
            } else if (INC3) {
                sob0 += dlo;
                sob1 += dhi;
                if (sob0 >= a_end) {
                    sob0 -= 4u * 2187u;
                    sob1 += 4u;
                }
            } else if (KIND == 0) { // x(i+1) = x(i) ^ D[ctz(i+1)], D[c] = C[0] ^ ... ^ C[c]
                const uint32_t c = __ffs(static_cast<int>(i + 1)) - 1;
                sob0 ^= sob_d[c];
                sob1 ^= sob_d[32 + c];
            }
        }
    };
    if (ACCUM != 0) {
        run(0, p.spp, std::false_type{});
        return finish_int(isum, p.spp, p.inv_spp);
    }
    // scene_value lies in [0, 1.25] and the sum never decreases, so once the
    // whole warp has sum >= 1.25 every later step takes the first branch
    const uint32_t k0 = p.spp < 8u ? p.spp : 8u;
    run(0, k0, std::false_type{});
    if (__all_sync(__activemask(), sum >= 1.25))
        run(k0, p.spp, std::true_type{});
    else
        run(k0, p.spp, std::false_type{});
    return finish_kahan(sum, comp, p.spp, p.inv_spp);
}

// Low-spp grid-stride rendering for the kinds that stage tables per CTA
// (Sobol' prefix XORs, the Halton kinds' phi_3 table): +15-50 % at 1-4 spp
// for Sobol' and Halton, while the lattice kinds measured faster with one
// pixel per thread.
template <uint32_t KIND>
constexpr bool kLowSppStride = KIND == 0 || KIND == 1 || KIND == 3;

// Per-warp classification of k_render's pixels (spp >= 8). Thread q takes
// the pixel in row q / W of the band and column colmap[q % W] (host::
// render_column_order groups the columns by sine-quadrant parity, so nearly
// every warp is uniform below); o is that pixel's offset in the band.
// valid: the lane has a pixel; every vote is over the whole warp and counts
// valid lanes only, so all k_render modes classify every warp identically.
struct WarpClass {
    uint64_t o;
    uint32_t px, py;
    int qx, qy;     // the lane's fixed quadrant counts (when fixed)
    bool inside;    // the lane's pixel lies inside the disc
    bool test;      // some lane's footprint crosses the disc's edge
    bool fixed;     // every lane keeps one sine quadrant per axis
    bool uniform;   // fixed, and all lanes share the parities of qx and qy
};

__device__ __forceinline__ WarpClass classify_warp(bool valid, uint64_t q, const RenderParams& p)
{
    WarpClass c{};
    int disc = kDiscOutside;
    bool fixed = true;
    if (valid) {
        band_pixel(q, p, c.px, c.py);
        c.o = q;
        if (p.colmap) {
            c.px = __ldg(p.colmap + c.px);
            c.o = static_cast<uint64_t>(c.py - p.row_begin) * p.width + c.px;
        }
        const double fx = static_cast<double>(c.px), fy = static_cast<double>(c.py);
        disc = disc_class(c.px, c.py, p.inv_w, p.inv_h, p.sc.disc_r2);
        fixed = sin_fixed_quadrant(fx * p.inv_w, (fx + 1.0) * p.inv_w, p.sc, c.qx) &&
                sin_fixed_quadrant(fy * p.inv_h, (fy + 1.0) * p.inv_h, p.sc, c.qy);
    }
    const unsigned vmask = __ballot_sync(0xffffffffu, valid);
    c.inside = disc == kDiscInside;
    c.test = __any_sync(0xffffffffu, disc == kDiscTest);
    c.fixed = __all_sync(0xffffffffu, fixed);
    const int par = (c.qx & 1) | (c.qy & 1) << 1;
    const int lead = vmask ? __ffs(vmask) - 1 : 0;
    const int par0 = __shfl_sync(0xffffffffu, par, lead);
    c.uniform = vmask != 0 && c.fixed && __all_sync(0xffffffffu, !valid || par == par0);
    return c;
}

// k_render. At spp >= 8 every warp is classified. With UQ, the warps whose
// lanes share the quadrant parities per axis (uniform) run sine polynomials
// specialised on those parities, with the coefficients in the constant bank
// (scene_value_uq); every other warp (and every warp without UQ) runs the
// per-lane quadrant / per-sample paths. Each pixel is rendered by one thread
// in the reference's per-pixel sample order, so neither the column order
// nor the path changes an output bit. UQ costs registers (the generic paths
// and the specialised loops in one kernel), so render_kind launches the UQ
// instance only at spp >= 8 and for the kinds where it measured faster.
// Shared-memory tables of the render kernels: the Sobol' prefix XORs (KIND
// 0), the phi_3 table (the Halton kinds) and the sine coefficients.
template <uint32_t KIND, bool Q3 = false>
struct RenderSmem {
    static constexpr bool kT3 = KIND == 1 || KIND == 3 || KIND == 6;
    static constexpr bool kQ3 = Q3 && (KIND == 1 || KIND == 3 || KIND == 6); // k_render's INC3 kinds
    double2 poly[8];
    uint32_t sob_d[KIND == 0 ? 64 : 4]; // sobol: prefix XORs of the columns
    // halton kinds: 3^7 words (+1 pad), then phi3_q's quotient tables, laid
    // out as the padded device buffer p.t3q3 so one bulk copy stages both
    alignas(16) uint32_t tab3[kT3 ? 2188 : 4];
    uint32_t q3[kQ3 ? 2 * 2187 + 2 : 4];
    uint64_t bar;
};

// The phi_3 tables are staged by one cp.async.bulk (TMA) copy from thread 0
// into the CTA's shared memory, completing on an mbarrier: no per-thread
// load/store loop (image-plane Halton stages 26 KB per 128-pixel CTA).
template <uint32_t KIND, bool Q3>
__device__ __forceinline__ void stage_render_smem(RenderSmem<KIND, Q3>& sm, const RenderParams& p)
{
    using S = RenderSmem<KIND, Q3>;
    const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(&sm.bar));
    if (S::kT3 && threadIdx.x == 0) {
        constexpr uint32_t bytes = (S::kQ3 ? 2188 + 2 * 2187 + 2 : 2188) * 4;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], "
                     "%2, [%3];" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(sm.tab3))),
                     "l"(p.t3q3), "r"(bytes), "r"(bar)
                     : "memory");
    }
    if (KIND == 0 && threadIdx.x < 64) {
        const uint32_t dim = threadIdx.x >> 5, c = threadIdx.x & 31u;
        uint32_t d = 0;
        for (uint32_t k = 0; k <= c; ++k)
            d ^= __ldg(p.cols2 + 52 * dim + k);
        sm.sob_d[threadIdx.x] = d;
    }
    load_sin_poly(sm.poly); // includes the barrier (the mbarrier init is visible after it)
    if (S::kT3) {
        uint32_t ok;
        do {
            asm volatile("{\n\t.reg .pred p;\n\t"
                         "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok)
                         : "r"(bar)
                         : "memory");
        } while (!ok);
    }
}

// spp < 8: too few samples to repay the per-warp classification. The kinds
// that stage tables per CTA run a grid-stride loop (render_kind sizes the
// grid to the resident CTAs) to spread the staging over many pixels.
template <uint32_t KIND, uint32_t ACCUM>
__global__ void __launch_bounds__(kBlock) k_render_low(RenderParams p, float* __restrict__ out)
{
    __shared__ RenderSmem<KIND> sm;
    stage_render_smem(sm, p);
    const uint64_t npix = static_cast<uint64_t>(p.row_end - p.row_begin) * p.width;
    const uint64_t step = kLowSppStride<KIND> ? static_cast<uint64_t>(gridDim.x) * blockDim.x : npix;
    for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < npix;
         q += step) {
        uint32_t px, py;
        band_pixel(q, p, px, py);
        const PixelState s = pixel_state<KIND>(px, py, p);
        out[q] = render_pixel<KIND, ACCUM, true, false>(s, p, static_cast<double>(px),
                                                         static_cast<double>(py), sm.poly, sm.sob_d,
                                                         false, 0, 0, sm.tab3);
    }
}

// spp >= 8. Every warp is classified (classify_warp). With UQ, the warps
// whose lanes share the quadrant parities per axis (uniform) run sine
// polynomials specialised on those parities, with the coefficients in the
// constant bank (scene_value_uq); every other warp (and every warp without
// UQ) runs the per-lane quadrant / per-sample paths. Each pixel is rendered
// by one thread in the reference's per-pixel sample order, so neither the
// column order nor the path changes an output bit. UQ costs registers (the
// generic paths and the specialised loops share the kernel), so render_kind
// launches the UQ instance only for the kinds where it measured faster.
template <uint32_t KIND, uint32_t ACCUM, bool UQ, bool Q3>
__device__ __forceinline__ void render_classified(const WarpClass& wc,
                                                  const RenderSmem<KIND, Q3>& sm,
                                                  const RenderParams& p, float* __restrict__ out)
{
    const PixelState s = pixel_state<KIND>(wc.px, wc.py, p);
    const double fx = static_cast<double>(wc.px), fy = static_cast<double>(wc.py);
    const bool inside = wc.inside;
    const int qx = wc.qx, qy = wc.qy;
    float r;
    if constexpr (RenderSmem<KIND, Q3>::kQ3) {
        // the phi_3 index of every sample below 3^14: the incremental
        // quotient-table path (phi3_q), warp-uniform
        bool inc;
        if (KIND == 3) { // halton_hilbert: no 3^20 reduction or u32 wrap inside the pixel
            const uint64_t g0 = static_cast<uint32_t>(s.block), g1 = g0 + (p.spp - 1);
            inc = p.spp <= 2187u && (g0 < 3486784401ull ? g1 < 3486784401ull : g1 <= 0xffffffffull);
        } else {
            const uint64_t nmax = (KIND == 6 ? static_cast<uint64_t>(s.ipy0) : 0ull) +
                                  static_cast<uint64_t>(p.spp - 1) * (KIND == 6 ? p.scale_x : 1u);
            inc = nmax < 4782969ull;
        }
        if (__all_sync(__activemask(), inc)) {
            if (UQ && wc.uniform) {
#define QMC_UQ3_CASE(U)                                                                            \
    r = wc.test ? render_pixel<KIND, ACCUM, true, true, U, true>(s, p, fx, fy, sm.poly, sm.sob_d,  \
                                                                 false, qx, qy, sm.q3)            \
                : render_pixel<KIND, ACCUM, false, true, U, true>(s, p, fx, fy, sm.poly, sm.sob_d, \
                                                                  inside, qx, qy, sm.q3)
                switch ((qx & 1) | (qy & 1) << 1) {
                case 0: QMC_UQ3_CASE(0); break;
                case 1: QMC_UQ3_CASE(1); break;
                case 2: QMC_UQ3_CASE(2); break;
                default: QMC_UQ3_CASE(3); break;
                }
#undef QMC_UQ3_CASE
            } else if (wc.fixed)
                r = wc.test ? render_pixel<KIND, ACCUM, true, true, -1, true>(
                                  s, p, fx, fy, sm.poly, sm.sob_d, false, qx, qy, sm.q3)
                            : render_pixel<KIND, ACCUM, false, true, -1, true>(
                                  s, p, fx, fy, sm.poly, sm.sob_d, inside, qx, qy, sm.q3);
            else
                r = wc.test ? render_pixel<KIND, ACCUM, true, false, -1, true>(
                                  s, p, fx, fy, sm.poly, sm.sob_d, false, 0, 0, sm.q3)
                            : render_pixel<KIND, ACCUM, false, false, -1, true>(
                                  s, p, fx, fy, sm.poly, sm.sob_d, inside, 0, 0, sm.q3);
            out[wc.o] = r;
            return;
        }
    }
    if (UQ && wc.uniform) {
        // four parities x disc test: warp-uniform choices
#define QMC_UQ_CASE(U)                                                                             \
    r = wc.test ? render_pixel<KIND, ACCUM, true, true, U>(s, p, fx, fy, sm.poly, sm.sob_d, false, \
                                                           qx, qy, sm.tab3)                        \
                : render_pixel<KIND, ACCUM, false, true, U>(s, p, fx, fy, sm.poly, sm.sob_d,       \
                                                            inside, qx, qy, sm.tab3)
        switch ((qx & 1) | (qy & 1) << 1) {
        case 0: QMC_UQ_CASE(0); break;
        case 1: QMC_UQ_CASE(1); break;
        case 2: QMC_UQ_CASE(2); break;
        default: QMC_UQ_CASE(3); break;
        }
#undef QMC_UQ_CASE
    } else if (wc.fixed) {
        // warps with no pixel on the disc's edge skip the per-sample disc
        // test; warps whose footprints each keep one sine quadrant per axis
        // skip the per-sample quadrant count (both choices warp-uniform)
        r = wc.test ? render_pixel<KIND, ACCUM, true, true>(s, p, fx, fy, sm.poly, sm.sob_d, false,
                                                             qx, qy, sm.tab3)
                    : render_pixel<KIND, ACCUM, false, true>(s, p, fx, fy, sm.poly, sm.sob_d,
                                                              inside, qx, qy, sm.tab3);
    } else {
        r = wc.test ? render_pixel<KIND, ACCUM, true, false>(s, p, fx, fy, sm.poly, sm.sob_d, false,
                                                              0, 0, sm.tab3)
                    : render_pixel<KIND, ACCUM, false, false>(s, p, fx, fy, sm.poly, sm.sob_d,
                                                               inside, 0, 0, sm.tab3);
    }
    out[wc.o] = r;
}

// Q3: the incremental phi3_q path of the image-plane / plain Halton kinds
// (17.5 KB of quotient tables per CTA: render_kind enables it from 32 spp,
// where the per-CTA staging is repaid).
#ifndef QMC_RENDER_Q3_MINB
#define QMC_RENDER_Q3_MINB 0
#endif
template <uint32_t KIND, uint32_t ACCUM, bool UQ, bool Q3>
__global__ void __launch_bounds__(kBlock, Q3 ? QMC_RENDER_Q3_MINB : 0)
    k_render(RenderParams p, float* __restrict__ out)
{
    const uint64_t npix = static_cast<uint64_t>(p.row_end - p.row_begin) * p.width;
    const uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const WarpClass wc = classify_warp(q < npix, q, p);
    __shared__ RenderSmem<KIND, Q3> sm;
    stage_render_smem(sm, p);
    if (q < npix)
        render_classified<KIND, ACCUM, UQ, Q3>(wc, sm, p, out);
}

// Few pixels, many samples (npix < kWarpPixels, spp >= 64): one warp per
// pixel, lane l takes samples l, l + 32, ... and the warp reduces with
// shuffles. int: exact int64 butterfly sum -> bit-identical to the
// sequential sum. kahan: per-lane Neumaier, lanes combined by a fixed
// compensated butterfly -> deterministic, within ~1e-16 relative of the
// reference's sequential order (north_star tolerance 1e-6).
template <uint32_t KIND, uint32_t ACCUM>
__global__ void __launch_bounds__(kBlock) k_render_warp(RenderParams p, float* __restrict__ out)
{
    __shared__ double2 s_poly[8];
    // sobol: D32[c] = C[5] ^ ... ^ C[5 + c] per dim (lane l takes samples
    // l + 32 m: X = X(l) ^ X(32 m), and m -> m + 1 flips X(32 m) by D32)
    __shared__ uint32_t s_d32[KIND == 0 ? 64 : 1];
    constexpr bool kSmemT3 = KIND == 1 || KIND == 3 || KIND == 6;
    __shared__ uint32_t s_tab3[kSmemT3 ? 2187 : 1];
    if (KIND == 0 && threadIdx.x < 64) {
        const uint32_t dim = threadIdx.x >> 5, c = threadIdx.x & 31u;
        uint32_t d = 0;
        for (uint32_t k = 0; k <= c && 5 + k < 52; ++k)
            d ^= __ldg(p.cols2 + 52 * dim + 5 + k);
        s_d32[threadIdx.x] = d;
    }
    if (kSmemT3)
        for (uint32_t e = threadIdx.x; e < 2187; e += blockDim.x)
            s_tab3[e] = __ldg(p.tab3 + e);
    load_sin_poly(s_poly); // includes the barrier
    const uint64_t npix = static_cast<uint64_t>(p.row_end - p.row_begin) * p.width;
    const uint64_t q = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31u;
    if (q >= npix)
        return; // whole warp
    uint32_t px, py;
    band_pixel(q, p, px, py);
    const PixelState s = pixel_state<KIND>(px, py, p);
    double sum = 0.0, comp = 0.0;
    long long isum = 0;
    const double fx = static_cast<double>(px), fy = static_cast<double>(py);
    uint32_t xl0 = p.scr0, xl1 = p.scr1; // sobol: scramble ^ X(lane)
    if (KIND == 0)
        sobol_direct2(lane, p, xl0, xl1);
    auto run = [&](auto test, auto fixed, bool inside_px, int qx, int qy) {
        uint32_t h0 = 0, h1 = 0; // sobol: X(32 m)
        for (uint32_t m = 0, i = lane; i < p.spp; ++m, i += 32) {
            const double f = pixel_sample<KIND, decltype(test)::value, decltype(fixed)::value,
                                          kSmemT3>(i, s, p, fx, fy, s_poly, xl0 ^ h0, xl1 ^ h1,
                                                   inside_px, qx, qy, s_tab3);
            if (ACCUM == 0)
                neumaier_add(sum, comp, f);
            else
                isum += int_term(f);
            if (KIND == 0) {
                const uint32_t c = __ffs(static_cast<int>(m + 1)) - 1;
                h0 ^= s_d32[c];
                h1 ^= s_d32[32 + c];
            }
        }
    };
    // one pixel per warp: the disc and quadrant classifications are uniform
    const int disc = disc_class(px, py, p.inv_w, p.inv_h, p.sc.disc_r2);
    int qx, qy;
    const bool fixed = sin_fixed_quadrant(fx * p.inv_w, (fx + 1.0) * p.inv_w, p.sc, qx) &&
                       sin_fixed_quadrant(fy * p.inv_h, (fy + 1.0) * p.inv_h, p.sc, qy);
    const bool inside = disc == kDiscInside;
    if (fixed) {
        if (disc == kDiscTest)
            run(std::true_type{}, std::true_type{}, false, qx, qy);
        else
            run(std::false_type{}, std::true_type{}, inside, qx, qy);
    } else {
        if (disc == kDiscTest)
            run(std::true_type{}, std::false_type{}, false, 0, 0);
        else
            run(std::false_type{}, std::false_type{}, inside, 0, 0);
    }
    for (int o = 16; o; o >>= 1) {
        if (ACCUM == 0) {
            const double os = __shfl_xor_sync(0xffffffffu, sum, o);
            const double oc = __shfl_xor_sync(0xffffffffu, comp, o);
            neumaier_add(sum, comp, os);
            comp = __dadd_rn(comp, oc);
        } else {
            isum += __shfl_xor_sync(0xffffffffu, isum, o);
        }
    }
    if (lane == 0)
        out[q] = ACCUM == 0 ? finish_kahan(sum, comp, p.spp, p.inv_spp)
                            : finish_int(isum, p.spp, p.inv_spp);
}

// Sample-partitioned render (PAPER.md:498-509 / imageplane.cpp:114-130:
// the sequence split by an extra radical-inverse dimension): accumulate, in
// int mode, only the samples i = first, first + step, ... of every pixel
// into an int64 per pixel. The int accumulation (llround(f * 2^32) summed in
// int64, render.cpp:72-78) is exactly associative, so summing the partials
// of all parts (one NCCL all-reduce across GPUs) and finalizing is
// bit-identical to the single-GPU int render.
// ADD: atomically add into acc instead of storing — the fused reduction of
// qmc_render_samples_devices, where acc may be another GPU's memory (peer
// access over NVLink): every part's kernel adds its int64 partials straight
// into the one accumulator, no separate collective.
template <uint32_t KIND, bool ADD = false>
__global__ void __launch_bounds__(kBlock)
    k_render_partial(RenderParams p, uint32_t first, uint32_t step, long long* __restrict__ acc)
{
    __shared__ double2 s_poly[8];
    // sobol: the part's samples first + step * m (step = 2^lp, first < step)
    // are X(first) ^ X(step * m); m -> m + 1 flips X(step * m) by
    // D[c] = C[lp] ^ ... ^ C[lp + c]
    __shared__ uint32_t s_dp[KIND == 0 ? 64 : 1];
    constexpr bool kSmemT3 = KIND == 1 || KIND == 3 || KIND == 6;
    __shared__ uint32_t s_tab3[kSmemT3 ? 2187 : 1];
    if (KIND == 0 && threadIdx.x < 64) {
        const uint32_t dim = threadIdx.x >> 5, c = threadIdx.x & 31u;
        const uint32_t lp = __ffs(static_cast<int>(step)) - 1;
        uint32_t d = 0;
        for (uint32_t k = 0; k <= c && lp + k < 52; ++k)
            d ^= __ldg(p.cols2 + 52 * dim + lp + k);
        s_dp[threadIdx.x] = d;
    }
    if (kSmemT3)
        for (uint32_t e = threadIdx.x; e < 2187; e += blockDim.x)
            s_tab3[e] = __ldg(p.tab3 + e);
    load_sin_poly(s_poly); // includes the barrier
    const uint64_t npix = static_cast<uint64_t>(p.row_end - p.row_begin) * p.width;
    const uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= npix)
        return;
    uint32_t px, py;
    band_pixel(q, p, px, py);
    const PixelState s = pixel_state<KIND>(px, py, p);
    long long isum = 0;
    const double fx = static_cast<double>(px), fy = static_cast<double>(py);
    uint32_t xf0 = p.scr0, xf1 = p.scr1; // sobol: scramble ^ X(first)
    if (KIND == 0)
        sobol_direct2(first, p, xf0, xf1);
    auto run = [&](auto test, auto fixed, bool inside_px, int qx, int qy) {
        uint32_t h0 = 0, h1 = 0; // sobol: X(step * m)
        for (uint32_t m = 0, i = first; i < p.spp; ++m, i += step) {
            isum += int_term(pixel_sample<KIND, decltype(test)::value, decltype(fixed)::value,
                                          kSmemT3>(i, s, p, fx, fy, s_poly, xf0 ^ h0, xf1 ^ h1,
                                                   inside_px, qx, qy, s_tab3));
            if (KIND == 0) {
                const uint32_t c = __ffs(static_cast<int>(m + 1)) - 1;
                h0 ^= s_dp[c];
                h1 ^= s_dp[32 + c];
            }
        }
    };
    // the same warp-uniform skips as k_render (disc_class, sin_fixed_quadrant)
    const int disc = disc_class(px, py, p.inv_w, p.inv_h, p.sc.disc_r2);
    int qx, qy;
    const bool fixed = sin_fixed_quadrant(fx * p.inv_w, (fx + 1.0) * p.inv_w, p.sc, qx) &&
                       sin_fixed_quadrant(fy * p.inv_h, (fy + 1.0) * p.inv_h, p.sc, qy);
    const unsigned mask = __activemask();
    const bool test = __any_sync(mask, disc == kDiscTest), inside = disc == kDiscInside;
    if (__all_sync(mask, fixed)) {
        if (test)
            run(std::true_type{}, std::true_type{}, false, qx, qy);
        else
            run(std::false_type{}, std::true_type{}, inside, qx, qy);
    } else {
        if (test)
            run(std::true_type{}, std::false_type{}, false, 0, 0);
        else
            run(std::false_type{}, std::false_type{}, inside, 0, 0);
    }
    if (ADD)
        atomicAdd(reinterpret_cast<unsigned long long*>(acc) + q,
                  static_cast<unsigned long long>(isum)); // two's complement: exact
    else
        acc[q] = isum;
}

__global__ void k_render_finalize(const long long* __restrict__ acc, uint64_t npix, uint32_t spp,
                                  float* __restrict__ out)
{
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < npix;
         k += stride)
        out[k] = finish_int(acc[k], spp);
}

// --------------------------------------------- stream fill of pixel kinds

template <uint32_t KIND, bool U32OUT>
__global__ void __launch_bounds__(256)
    k_pixel_stream(PixelStreamParams p, Div32 div_dims, uint64_t first, uint32_t elems,
                   uint32_t* __restrict__ out)
{
    // per-pixel state, recomputed per thread (a few dozen integer ops)
    uint32_t shift = 0, ipx0 = 0, ipy0 = 0, cell = 0;
    uint64_t block = 0, off = 0;
    if (KIND == 4)
        shift = phi3_fixed(static_cast<uint32_t>(hilbert_index(p.px, p.py, p.order)), p.tab3);
    if (KIND == 3)
        block = hilbert_index(p.px, p.py, p.order) * p.spp;
    if (KIND == 6) {
        off = halton_offset(p.px, p.py, p.exp_x, p.exp_y, p.stride, p.crt_x, p.crt_y, 0);
        ipx0 = static_cast<uint32_t>(off >> p.exp_x);
        ipy0 = static_cast<uint32_t>(off / p.scale_y);
    }
    if (KIND == 7)
        cell = (p.px % 128u) + (p.py % 128u) * 128u;
    const RadicalDim* rd = static_cast<const RadicalDim*>(p.radical_dims);
    // pixel_random_lattice: the per-dimension hashed generator depends on the
    // pixel only (lattice.hpp:51-56), so it is hashed once per block
    __shared__ uint32_t s_gen[KIND == 5 ? 256 : 1];
    const bool gen_cached = KIND == 5 && p.dims <= 256;
    if (gen_cached) {
        for (uint32_t j = threadIdx.x; j < p.dims; j += blockDim.x)
            s_gen[j] = pixel_hash(j, p.px, p.py) | 1u;
        __syncthreads();
    }

    auto value = [&](uint32_t pt, uint32_t j) {
        const uint64_t idx = first + pt;
        const uint32_t i = static_cast<uint32_t>(idx);
        uint32_t x;
        if (KIND == 3) {
            x = radical_fixed(static_cast<uint32_t>(block + idx), rd[j]);
        } else if (KIND == 4) {
            x = (brev32(i) + shift) * __ldg(p.generator + j);
        } else if (KIND == 5) {
            x = brev32(~i) * (gen_cached ? s_gen[j] : (pixel_hash(j, p.px, p.py) | 1u));
        } else if (KIND == 6) { // imageplane.cpp:448-456
            if (j == 0)
                x = rad2(ipx0 + i * p.scale_y);
            else if (j == 1)
                x = phi3_fixed(ipy0 + i * p.scale_x, p.tab3);
            else
                x = radical_fixed(static_cast<uint32_t>(off + idx * p.stride), rd[j]);
        } else { // KIND == 7
            const uint32_t k = i ^ __ldg(p.xor_reorder + cell);
            x = __ldg(p.xor_points + static_cast<uint64_t>(k) * p.xor_dims + j) ^
                __ldg(p.xor_scramble + cell * p.xor_dims + j);
        }
        return U32OUT ? x : map_bits(x);
    };
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t t0 = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t e0 = 0;
    if ((reinterpret_cast<uintptr_t>(out) & 15u) == 0) {
        // four consecutive elements per thread, one 16-B streaming store
        const uint32_t quads = elems >> 2;
        e0 = quads << 2;
        for (uint32_t qd = t0; qd < quads; qd += stride) {
            uint32_t pt = p.dims == 1 ? qd * 4 : div32(qd * 4, div_dims);
            uint32_t j = qd * 4 - pt * p.dims;
            uint32_t v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                v[k] = value(pt, j);
                if (++j == p.dims) {
                    j = 0;
                    ++pt;
                }
            }
            __stcs(reinterpret_cast<uint4*>(out) + qd, make_uint4(v[0], v[1], v[2], v[3]));
        }
    }
    for (uint32_t e = e0 + t0; e < elems; e += stride) {
        const uint32_t pt = p.dims == 1 ? e : div32(e, div_dims);
        out[e] = value(pt, e - pt * p.dims);
    }
}

// image.cpp:25-30: clamp to [0,1], round half up in fp32 (mul then add, no
// FMA, as the x86 reference), min 255; `channels` copies per pixel (P5: 1,
// P6: 3).
__global__ void k_quantize(const float* __restrict__ v, uint64_t npix, uint32_t channels,
                           unsigned char* __restrict__ out)
{
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < npix;
         k += stride) {
        float c = v[k];
        c = c < 0.0f ? 0.0f : (1.0f < c ? 1.0f : c);
        const int q = __float2int_rz(__fadd_rn(__fmul_rn(c, 255.0f), 0.5f));
        const unsigned char b = static_cast<unsigned char>(q < 255 ? q : 255);
        for (uint32_t ch = 0; ch < channels; ++ch)
            out[k * channels + ch] = b;
    }
}

__global__ void k_scene_value(const double* __restrict__ xy, double* __restrict__ out, uint64_t n)
{
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
         k += stride)
        out[k] = scene_value(xy[2 * k], xy[2 * k + 1]);
}

// The kinds whose k_render<.., true> measured faster (4K, 8-64 spp): sobol,
// lattice, pixel-shifted / pixel-random lattice, sobol-xor-table. The
// Halton kinds' phi_3 digit work needs the registers more: +8-16 % without.
#ifndef QMC_RENDER_UQ_KINDS
#define QMC_RENDER_UQ_KINDS 0xb5u
#endif
constexpr uint32_t kRenderUqKinds = QMC_RENDER_UQ_KINDS;

constexpr uint64_t kWarpPixels = 32768; // below this (and spp >= 64): warp per pixel

template <uint32_t KIND>
cudaError_t render_kind(const RenderParams& p, uint32_t accum, float* out, cudaStream_t s)
{
    const uint64_t npix = static_cast<uint64_t>(p.row_end - p.row_begin) * p.width;
    if (npix < kWarpPixels && p.spp >= 64) {
        const unsigned wgrid = static_cast<unsigned>((npix * 32 + kBlock - 1) / kBlock);
        if (accum == 0)
            k_render_warp<KIND, 0><<<wgrid, kBlock, 0, s>>>(p, out);
        else
            k_render_warp<KIND, 1><<<wgrid, kBlock, 0, s>>>(p, out);
        return cudaGetLastError();
    }
    unsigned grid = static_cast<unsigned>((npix + kBlock - 1) / kBlock);
    if (p.spp < 8) {
        if (kLowSppStride<KIND>) // grid-stride: about one wave of resident CTAs
            grid = std::min(grid, static_cast<unsigned>(sm_count()) * 8u);
        if (accum == 0)
            k_render_low<KIND, 0><<<grid, kBlock, 0, s>>>(p, out);
        else
            k_render_low<KIND, 1><<<grid, kBlock, 0, s>>>(p, out);
        return cudaGetLastError();
    }
    constexpr bool kUq = (kRenderUqKinds >> KIND) & 1u;
    constexpr bool kHasQ3 = KIND == 1 || KIND == 3 || KIND == 6;
    if (kHasQ3 && p.spp >= 32) { // the phi3_q path, with the specialised sine loop
        if (accum == 0)
            k_render<KIND, 0, true, kHasQ3><<<grid, kBlock, 0, s>>>(p, out);
        else
            k_render<KIND, 1, true, kHasQ3><<<grid, kBlock, 0, s>>>(p, out);
    } else if (accum == 0) {
        k_render<KIND, 0, kUq, false><<<grid, kBlock, 0, s>>>(p, out);
    } else {
        k_render<KIND, 1, kUq, false><<<grid, kBlock, 0, s>>>(p, out);
    }
    return cudaGetLastError();
}

template <uint32_t KIND>
cudaError_t pixel_stream_kind(const PixelStreamParams& p, bool u32, const FillRange& r,
                              cudaStream_t s)
{
    const Div32 d = p.dims >= 2 ? make_div32(p.dims) : Div32{0, 0};
    const uint64_t max_pts = (1ull << 30) / p.dims;
    for (uint64_t done = 0; done < r.n; done += max_pts) {
        const uint64_t pts = r.n - done < max_pts ? r.n - done : max_pts;
        const uint32_t elems = static_cast<uint32_t>(pts * p.dims);
        uint64_t want = (elems + 255) / 256;
        const uint64_t cap = static_cast<uint64_t>(sm_count()) * 8;
        const unsigned grid = static_cast<unsigned>(want < cap ? want : cap);
        uint32_t* o = static_cast<uint32_t*>(r.out) + done * p.dims;
        if (u32)
            k_pixel_stream<KIND, true><<<grid, 256, 0, s>>>(p, d, r.first + done, elems, o);
        else
            k_pixel_stream<KIND, false><<<grid, 256, 0, s>>>(p, d, r.first + done, elems, o);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess)
            return e;
    }
    return cudaSuccess;
}

} // namespace

cudaError_t launch_render(const RenderParams& p, uint32_t kind, uint32_t accum, float* out,
                          cudaStream_t s)
{
    if (p.row_end <= p.row_begin || p.width == 0)
        return cudaSuccess;
    switch (kind) {
    case 0: return render_kind<0>(p, accum, out, s);
    case 1: return render_kind<1>(p, accum, out, s);
    case 2: return render_kind<2>(p, accum, out, s);
    case 3: return render_kind<3>(p, accum, out, s);
    case 4: return render_kind<4>(p, accum, out, s);
    case 5: return render_kind<5>(p, accum, out, s);
    case 6: return render_kind<6>(p, accum, out, s);
    case 7: return render_kind<7>(p, accum, out, s);
    }
    return cudaErrorInvalidValue;
}

template <uint32_t KIND>
cudaError_t render_partial_kind(const RenderParams& p, uint32_t first, uint32_t step,
                                long long* acc, bool add, cudaStream_t s)
{
    const uint64_t npix = static_cast<uint64_t>(p.row_end - p.row_begin) * p.width;
    const unsigned grid = static_cast<unsigned>((npix + kBlock - 1) / kBlock);
    if (add)
        k_render_partial<KIND, true><<<grid, kBlock, 0, s>>>(p, first, step, acc);
    else
        k_render_partial<KIND, false><<<grid, kBlock, 0, s>>>(p, first, step, acc);
    return cudaGetLastError();
}

cudaError_t launch_render_partial(const RenderParams& p, uint32_t kind, uint32_t first,
                                  uint32_t step, long long* acc, cudaStream_t s, bool add)
{
    if (p.row_end <= p.row_begin || p.width == 0)
        return cudaSuccess;
    switch (kind) {
    case 0: return render_partial_kind<0>(p, first, step, acc, add, s);
    case 1: return render_partial_kind<1>(p, first, step, acc, add, s);
    case 2: return render_partial_kind<2>(p, first, step, acc, add, s);
    case 3: return render_partial_kind<3>(p, first, step, acc, add, s);
    case 4: return render_partial_kind<4>(p, first, step, acc, add, s);
    case 5: return render_partial_kind<5>(p, first, step, acc, add, s);
    case 6: return render_partial_kind<6>(p, first, step, acc, add, s);
    case 7: return render_partial_kind<7>(p, first, step, acc, add, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_render_finalize(const long long* acc, uint64_t npix, uint32_t spp, float* out,
                                   cudaStream_t s)
{
    if (npix == 0)
        return cudaSuccess;
    const uint64_t want = (npix + 255) / 256, cap = static_cast<uint64_t>(sm_count()) * 8;
    k_render_finalize<<<static_cast<unsigned>(want < cap ? want : cap), 256, 0, s>>>(acc, npix,
                                                                                      spp, out);
    return cudaGetLastError();
}

cudaError_t launch_pixel_stream(const PixelStreamParams& p, bool u32, const FillRange& r,
                                cudaStream_t s)
{
    if (r.n == 0)
        return cudaSuccess;
    switch (p.kind) {
    case 3: return pixel_stream_kind<3>(p, u32, r, s);
    case 4: return pixel_stream_kind<4>(p, u32, r, s);
    case 5: return pixel_stream_kind<5>(p, u32, r, s);
    case 6: return pixel_stream_kind<6>(p, u32, r, s);
    case 7: return pixel_stream_kind<7>(p, u32, r, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_quantize(const float* v, uint64_t npix, uint32_t channels, unsigned char* out,
                            cudaStream_t s)
{
    if (npix == 0)
        return cudaSuccess;
    const uint64_t want = (npix + 255) / 256, cap = static_cast<uint64_t>(sm_count()) * 8;
    k_quantize<<<static_cast<unsigned>(want < cap ? want : cap), 256, 0, s>>>(v, npix, channels,
                                                                              out);
    return cudaGetLastError();
}

cudaError_t launch_scene_value(const double* xy, double* out, uint64_t n, cudaStream_t s)
{
    if (n == 0)
        return cudaSuccess;
    const uint64_t want = (n + 255) / 256, cap = static_cast<uint64_t>(sm_count()) * 8;
    k_scene_value<<<static_cast<unsigned>(want < cap ? want : cap), 256, 0, s>>>(xy, out, n);
    return cudaGetLastError();
}

} // namespace qmcgpu
