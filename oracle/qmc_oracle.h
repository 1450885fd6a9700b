/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the QMC sampling path.
 *
 * A plain-C11 restatement of the reference algorithms (qmckit `qmc::`,
 * /root/reference/proj); every function cites the reference file:line it
 * follows. Only tests/, bench.py's cpu_baseline leg and
 * __graft_entry__.smoke() may load it, and only as the checker. The product
 * (paper_2307_15584_b200/libqmcgpu.so) never links or calls it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 * the reference itself (oracle/_ref/libqmcref.so, built from the reference
 * sources by oracle/Makefile) and against the golden vectors in
 * tests/golden/ (made by tests/golden/make_golden.py from the same build).
 * Two functions have no reference counterpart and are *defined* here:
 * qo_owen_scramble (hash-based Owen scrambling: parity
 * unpinned, pinned by properties instead) and the CP-rotated lattice
 * qo_lattice_cp_fixed (a composition of reference functions).
 */
#ifndef QMC_ORACLE_H
#define QMC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* unitfloat.hpp */
uint32_t qo_clz32(uint32_t v);
uint32_t qo_brev32(uint32_t v);
uint32_t qo_map_bits(uint32_t u); /* bits of map_u32_to_unifloat(u) */
void qo_map_range(uint32_t u0, uint64_t n, uint32_t* out);

/* primes.cpp */
int qo_prime(uint32_t index, uint32_t* out);           /* 0 ok, 3 out_of_range */
int qo_prime_max_power(uint32_t index, uint32_t* out); /* 0 ok, 3 out_of_range */
uint32_t qo_max_power_fitting_u32(uint32_t base);

/* radical.cpp */
uint32_t qo_radical_inverse_fixed(uint32_t i, uint32_t prime_index);
uint32_t qo_radical_inverse_linscramble_fixed(uint32_t i, uint32_t prime_index, uint32_t factor);
uint32_t qo_radical_inverse_permuted_fixed(uint32_t i, uint32_t prime_index,
                                           const uint32_t* sigma);
void qo_faure_permutation(uint32_t base, uint32_t* out);
/* table[b^d]; returns b^d, or 0 when the table would exceed 2^16 entries */
uint32_t qo_tensor_digit_table(const uint32_t* sigma, uint32_t base, uint32_t d,
                               uint32_t* table);
uint32_t qo_radical_inverse_tabled_fixed(uint32_t i, uint32_t base, uint32_t digits_per_step,
                                         const uint32_t* table, const uint32_t* sigma);

/* digitalnet.cpp: rows of (s, a, m[0..s-1]) for dimensions 1..rows */
void qo_build_matrices(uint32_t dims, const uint32_t* s, const uint32_t* a,
                       const uint32_t* const* m, uint32_t* columns /* dims*52 */);
uint32_t qo_sobol_component_fixed(uint64_t i, const uint32_t* columns_j, uint32_t scramble);
void qo_sobol_fill_fixed(uint64_t first, uint64_t n, uint32_t dims, const uint32_t* columns,
                         const uint32_t* scrambles, uint32_t* out);
void qo_sobol_fill_f32(uint64_t first, uint64_t n, uint32_t dims, const uint32_t* columns,
                       const uint32_t* scrambles, float* out);

/* Builder-defined hash-based Owen scramble (no reference). */
uint32_t qo_owen_scramble(uint32_t v, uint32_t seed);
void qo_sobol_owen_fill_fixed(uint64_t first, uint64_t n, uint32_t dims, const uint32_t* columns,
                              const uint32_t* seeds, uint32_t* out);

/* lattice.cpp / lattice.hpp */
uint32_t qo_lattice_component_fixed(uint32_t i, uint32_t g);
uint32_t qo_lattice_cp_fixed(uint32_t i, uint32_t g, uint32_t shift);
uint32_t qo_pixel_hash(uint32_t j, uint32_t px, uint32_t py);
uint32_t qo_random_lattice_component_fixed(uint32_t i, uint32_t j, uint32_t px, uint32_t py);
int qo_lfsr_generator_vector(uint32_t seed, uint32_t dims, uint32_t* out);
int qo_lattice_shift_fixed(uint32_t k, uint32_t m, const uint32_t* g, uint32_t dims,
                           uint32_t* out);

/* hilbert.hpp / imageplane.cpp */
int qo_hilbert_index(uint32_t x, uint32_t y, uint32_t order, uint64_t* out);
int qo_hilbert_xy(uint64_t d, uint32_t order, uint32_t* x, uint32_t* y);
uint32_t qo_hilbert_phi3_fixed(uint32_t x, uint32_t y, uint32_t order);
uint64_t qo_digit_reverse(uint64_t v, uint32_t base, uint32_t digits);

typedef struct qo_halton_enum {
    uint32_t scale_x, scale_y, exp_x, exp_y;
    uint64_t stride, crt_x, crt_y;
} qo_halton_enum;
int qo_halton_enum_init(uint32_t width, uint32_t height, qo_halton_enum* e);
uint64_t qo_halton_enum_offset(const qo_halton_enum* e, uint32_t px, uint32_t py);
int qo_partition(uint32_t part, uint32_t parts, uint32_t base, uint64_t* rem, uint64_t* mod);

/* render.cpp / quality.hpp */
double qo_scene_value(double x, double y);
uint32_t qo_hilbert_order_for(uint32_t w, uint32_t h);

/* kinds follow imageplane.hpp:122-131 order */
enum { QO_SOBOL = 0, QO_HALTON, QO_LATTICE, QO_HALTON_HILBERT, QO_PIXEL_SHIFTED_LATTICE,
       QO_PIXEL_RANDOM_LATTICE, QO_IMAGE_PLANE_HALTON };

/* Per-pixel render of the synthetic scene (render.cpp:58-143), single
 * thread, kinds above (sobol uses `columns` for 2 dims; scrambles derived
 * from seed as render.cpp:52-54). accum: 0 kahan, 1 int. */
int qo_render(uint32_t w, uint32_t h, uint32_t spp, int kind, int accum, uint32_t seed,
              const uint32_t* sobol_columns2, float* out);

/* int-mode render over samples i == rem (mod mod): int64 per-pixel sums */
int qo_render_partial_int(uint32_t w, uint32_t h, uint32_t spp, int kind, uint32_t seed,
                          const uint32_t* cols2, uint32_t rem, uint32_t mod, int64_t* acc);

uint64_t qo_fnv1a64(const void* data, uint64_t size);

#ifdef __cplusplus
}
#endif
#endif
