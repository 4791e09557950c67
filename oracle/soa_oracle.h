/* TEST INFRASTRUCTURE — CPU oracle for the AoS<->SoA + reduced-precision SPH
 * hot path.  A plain-C restatement of the reference algorithms, each function
 * citing the reference file:line it follows (paths relative to
 * /root/reference/proj).  Parity is pinned against the reference itself
 * (oracle/_ref, tests/test_oracle_pinning.py) and the golden vectors in
 * tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library — as the checker, never as the thing measured/shipped. */
#ifndef SOA_ORACLE_H
#define SOA_ORACLE_H
#include <stdint.h>

/* Storage format codes for one lane.
 *   7..64      compressed T-bit float (fpcodec::layout_for(T), fpcodec.cpp:28-37)
 *   1000+T     native: T-bit value expanded to its base IEEE width
 *              (PrecisionTag::Native, layout_ops.cpp:164-191)
 *   OR_BF16    bfloat16 = narrow_to_ieee(x, 8, 7) (fpcodec.cpp:39-90); not a
 *              reference PrecisionSpec, restated for the new bf16 mode
 *   OR_I64     raw 64-bit integer lane (copied bit-exactly)            */
#define OR_BF16 (-2)
#define OR_I64 (-1)
#define OR_NATIVE(T) (1000 + (T))

int or_layout_for(int total_bits, int* exponent_bits, int* mantissa_bits);
int or_fmt_width(int fmt);
uint64_t or_narrow_to_ieee(double x, int exponent_bits, int mantissa_bits);
double or_widen_from_ieee(uint64_t bits, int exponent_bits, int mantissa_bits);
uint64_t or_expand_to_base_bits(uint64_t bits, int total_bits);
uint64_t or_truncate_from_base_bits(uint64_t base_bits, int total_bits);
uint64_t or_encode_bits(double x, int total_bits);
double or_decode_bits(uint64_t bits, int total_bits);
double or_quantize(double x, int total_bits);
uint64_t or_encode_fmt(double x, int fmt);
double or_decode_fmt(uint64_t bits, int fmt);
void or_encode_array(const double* x, uint64_t n, int fmt, uint64_t* out);
void or_decode_array(const uint64_t* bits, uint64_t n, int fmt, double* out);

void or_write_bits(uint8_t* buf, uint64_t offset_bits, int width, uint64_t value);
uint64_t or_read_bits(const uint8_t* buf, uint64_t offset_bits, int width);

/* One field's lanes moved from a source to a destination bit stream:
 * lane l of record r sits at base + r*stride + l*width on each side.
 * AoS: base = field prefix, stride = record_bits;  SoA: base = stream
 * base, stride = arity*width (layout_ops.cpp:25-39). */
typedef struct {
    int arity;
    int src_fmt, dst_fmt;
    uint64_t src_base, src_stride;
    uint64_t dst_base, dst_stride;
} or_move;
/* dst lane = encode(decode(src lane)) (fpcodec.cpp:137-155); raw copy when
 * the formats are equal (layout_ops.cpp:150-191). */
void or_apply_moves(const uint8_t* src, uint8_t* dst, uint64_t count, const or_move* moves,
                    int nmoves);

uint64_t or_checksum(const uint8_t* bytes, uint64_t nbytes, uint64_t length_bits);

/* sph.cpp:17-24 */
double or_w(double r, double h);
/* sph.cpp:176-199 over contiguous buffers of `bs` (sph.cpp:286-308).  When
 * rho_fmt != 0 the accumulator is quantized through it after every
 * neighbour (Writeback::PerAccess). */
void or_density_buffer(const double* x, const double* m, const double* h, uint64_t n,
                       uint64_t bs, int rho_fmt, double* rho);
/* Cell-linked restatement: same pair formula, j over every particle with
 * |x_i - x_j| < 2 h_ij, summed in ascending particle index order.  Pairs
 * beyond the support add exactly +0.0 in the reference, so this equals the
 * all-pairs sum over any candidate superset. */
void or_density_cells(const double* x, const double* m, const double* h, uint64_t n,
                      double box_lo, double box_hi, double cell, double* rho);
/* The same sums for the listed homes only (every particle a candidate). */
void or_density_cells_at(const double* x, const double* m, const double* h, uint64_t n, double lo, double hi,
                         double cell, const uint64_t* homes, uint64_t nh, double* rho);
double or_dw_dr(double r, double h);
int or_force_cells(const double* x, const double* v, const double* m, const double* h, const double* rho,
                   const double* P, uint64_t n, double lo, double hi, double cell, double* a, double* du,
                   double* a_scale, double* du_scale);
int or_force_cells_at(const double* x, const double* v, const double* m, const double* h, const double* rho,
                      const double* P, uint64_t n, double lo, double hi, double cell, const uint64_t* homes,
                      uint64_t nh, double* a, double* du, double* a_scale, double* du_scale);

/* sph.cpp:325-349 (mt19937_64 + libstdc++ uniform_real_distribution);
 * accel_seed != 0 additionally draws a ~ U(-1,1)^3, du ~ U(-1,1). */
void or_random_ics(uint64_t n, uint64_t seed, uint64_t accel_seed, double dt, double* x,
                   double* v, double* a, double* u, double* m, double* h, double* rho,
                   double* P, double* cs, double* du, double* dtf, int64_t* id);
#endif
