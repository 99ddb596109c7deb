/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the hot path of
 * arXiv 2109.05410 ("Accelerating GPU-Based Out-of-Core Stencil Computation
 * with On-the-Fly Compression").  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load liboracle.so.
 * The product path (paper_2109_05410_b200/, include/oocz.h) never includes,
 * links or calls anything here, and nothing here includes product headers.
 *
 * Citations: PAPER.md:N is a line of /root/reference/PAPER.md; SURVEY.md
 * sections are the build blueprint (Appendix A = the ZFP fixed-rate format).
 *
 * Parity pins live in tests/test_oracle_*.py.  Functions whose parity with
 * an external implementation cannot be checked here say so ("parity
 * unpinned") -- see DESIGN.md "Oracle pins".
 */
#ifndef OOCZ_ORACLE_H
#define OOCZ_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------- ZFP-style fixed-rate codec, fp32, 3-D (zfp_ref.c) ----------------
 * PAPER.md:120-123 (Sec. IV: cuZFP, "specify the number of bits to use to
 * preserve a value"), PAPER.md:202 (cuZFP 0.5.5).  Format: SURVEY Appendix A. */

/* individual steps, exposed for the pins */
int32_t  orc_exponent_max(const float x[64]);           /* emax, or -127 for an all-zero block */
void     orc_fwd_cast(const float x[64], int emax, int32_t q[64]);
void     orc_inv_cast(const int32_t q[64], int emax, float x[64]);
void     orc_fwd_lift(int32_t v[4]);                     /* one 4-vector, in place */
void     orc_inv_lift(int32_t v[4]);
void     orc_fwd_xform(int32_t q[64]);                   /* lifting along x, then y, then z */
void     orc_inv_xform(int32_t q[64]);                   /* lifting along z, then y, then x */
uint32_t orc_int2uint(int32_t x);                        /* negabinary */
int32_t  orc_uint2int(uint32_t u);
const uint8_t* orc_perm3(void);                          /* coefficient order, 64 entries */

/* whole-block coder; out/in hold `rate` uint64 words; returns the number of
 * bits the coder actually emitted (before zero padding) */
int orc_encode_block(const float x[64], int rate, uint64_t* out);
int orc_decode_block(const uint64_t* in, int rate, float x[64]);
/* integer-stage only (bit-plane coder on 64 negabinary words, budget in bits) */
int orc_encode_ints(const uint32_t u[64], int budget_bits, uint64_t* words, int bit_offset);
int orc_decode_ints(const uint64_t* words, int bit_offset, int budget_bits, uint32_t u[64]);

/* whole array: x fastest, each extent a multiple of 4; block order bz,by,bx */
size_t orc_zfp_bytes(int nx, int ny, int nz, int rate);
int    orc_zfp_encode(const float* f, int nx, int ny, int nz, int rate, uint64_t* out);
int    orc_zfp_decode(const uint64_t* in, int nx, int ny, int nz, int rate, float* f);
/* RT_r(.) = decode(encode(.)), in place; identity for rate == 0 (raw) */
int    orc_roundtrip(float* f, int nx, int ny, int nz, int rate);

/* ---------------- the same codec for fp64 (zfp_ref64.c) ----------------
 * The paper's precision and rates (32/64, 24/64: PAPER.md:213-215):
 * EBITS 11, EBIAS 1023, 64 bit planes, q = trunc(x * 2^(62 - emax)). */
int32_t  orc64_exponent_max(const double x[64]);
void     orc64_fwd_cast(const double x[64], int emax, int64_t q[64]);
void     orc64_inv_cast(const int64_t q[64], int emax, double x[64]);
void     orc64_fwd_lift(int64_t v[4]);
void     orc64_inv_lift(int64_t v[4]);
void     orc64_fwd_xform(int64_t q[64]);
void     orc64_inv_xform(int64_t q[64]);
uint64_t orc64_int2uint(int64_t x);
int64_t  orc64_uint2int(uint64_t u);
int orc64_encode_ints(const uint64_t u[64], int budget_bits, uint64_t* words, int bit_offset);
int orc64_decode_ints(const uint64_t* words, int bit_offset, int budget_bits, uint64_t u[64]);
int orc64_encode_block(const double x[64], int rate, uint64_t* out);
int orc64_decode_block(const uint64_t* in, int rate, double x[64]);
int orc64_zfp_encode(const double* f, int nx, int ny, int nz, int rate, uint64_t* out);
int orc64_zfp_decode(const uint64_t* in, int nx, int ny, int nz, int rate, double* f);
int orc64_roundtrip(double* f, int nx, int ny, int nz, int rate);

/* ---------------- 25-point leapfrog (stencil_ref.c) ----------------
 * PAPER.md:208 (Sec. VI: 25-point acoustic propagator, two read-write
 * datasets, one write-only intermediate, one read-only dataset),
 * PAPER.md:188 (HALO = 4).  Arithmetic order: SURVEY 8(c) c.1. */
void orc_default_coeffs(float c[5]);
/* one step over the whole grid: out = 2u - uprev + m*L(u), zero ghost of depth 4 */
void orc_step(const float* u, const float* uprev, const float* m, float* out,
              int nx, int ny, int nz, const float c[5]);
void orc_step_f64(const double* u, const double* uprev, const double* m, double* out,
                  int nx, int ny, int nz, const double c[5]);
/* one step restricted to global planes [z0, z1); planes of out outside are untouched */
void orc_step_planes(const float* u, const float* uprev, const float* m, float* out,
                     int nx, int ny, int nz, const float c[5], int z0, int z1);

void orc_step_planes_f64(const double* u, const double* uprev, const double* m, double* out,
                         int nx, int ny, int nz, const double c[5], int z0, int z1);

/* the schedule the out-of-core method reduces to.
 * Advances (u, uprev) by nsteps: floor(n/T) sweeps of T steps and one of
 * n mod T, with RT_rate[f] applied to u and uprev after every sweep.
 * (set_field's round trip of all three fields is orc_roundtrip, done by the caller.) */
int orc_advance(float* u, float* uprev, const float* m, int nx, int ny, int nz,
                const float c[5], int T, const int rate[3], long nsteps);
/* the same schedule in fp64 (orc_step_f64 + orc64_roundtrip) */
int orc64_advance(double* u, double* uprev, const double* m, int nx, int ny, int nz,
                  const double c[5], int T, const int rate[3], long nsteps);

/* ---------------- literal out-of-core emulator (ooc_emul.c) ----------------
 * PAPER.md:112-113 (Sec. III region sharing), PAPER.md:130-160 (Sec. V.A,
 * Fig. 4 separate compression).  Follows the block/region bookkeeping
 * literally (compressed store per region, per-block slab, time-t copy of the
 * common region, cone-limited steps), optionally split into G z-slabs that
 * exchange compressed boundary regions.  stats: [0] H2D bytes, [1] D2H bytes,
 * [2] halo bytes sent between slabs (all summed over the run). */
int orc_ooc_emulate(float* u, float* uprev, const float* m, int nx, int ny, int nz,
                    const float c[5], int T, int P, int G, const int rate[3],
                    long nsteps, int poison, uint64_t stats[3]);
/* the same literal emulation in the paper's precision (fp64 fields, the fp64
 * codec orc64_* and orc_step_planes_f64; ooc_emul64.c instantiates ooc_emul.c) */
int orc64_ooc_emulate(double* u, double* uprev, const double* m, int nx, int ny, int nz,
                      const double c[5], int T, int P, int G, const int rate[3],
                      long nsteps, int poison, uint64_t stats[3]);

#ifdef __cplusplus
}
#endif
#endif
