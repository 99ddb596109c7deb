/*
 * zfp_ref.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Bit-serial ZFP-style fixed-rate coder for fp32 3-D arrays, written step by
 * step in the order of SURVEY.md Appendix A (the zfp 0.5.5 fixed-rate format
 * that cuZFP 0.5.5 mirrors; the paper uses cuZFP 0.5.5, and
 * only fixes "a number of bits to preserve a value").
 *
 *   encode: gather 4^3 -> zero test -> emax -> 9 exponent bits ->
 *           q = trunc(x * 2^(30-emax)) (exact, fp64) -> lifting x,y,z ->
 *           PERM -> negabinary -> embedded group-tested bit planes 31..0
 *           under a budget of 64*rate-9 bits -> zero pad to 64*rate bits
 *   decode: the mirror image, including zfp's budget-exhaustion behaviour
 *
 * Bits are written one at a time: bit j of block b is global bit
 * 64*rate*b + j, i.e. word (p>>6), bit (p&63), little-endian uint64 words.
 *
 * Parity vs real zfp / cuZFP: UNPINNED (no zfp on this machine); pinned
 * instead by the closed forms and invariants in tests/test_oracle_zfp.py.
 * Readings (R9-R12): exact fp64 scale factors; -0.0 blocks are zero
 * blocks; extents are multiples of 4 (no partial blocks).
 */
#include "oracle.h"
#include <math.h>
#include <string.h>
#include <stdlib.h>

#define EBITS 8
#define EBIAS 127
#define NBMASK 0xaaaaaaaau

/* ---- 32-bit wraparound helpers: the lifting is defined on 32-bit two's
 * complement integers with arithmetic right shift. ---- */
static int32_t wadd(int32_t a, int32_t b) { return (int32_t)((uint32_t)a + (uint32_t)b); }
static int32_t wsub(int32_t a, int32_t b) { return (int32_t)((uint32_t)a - (uint32_t)b); }
static int32_t wshl1(int32_t a) { return (int32_t)((uint32_t)a << 1); }
static int32_t asr1(int32_t a) { return (int32_t)(a >> 1); } /* gcc: arithmetic */

/* ---- block-floating-point: common exponent (App. A "Exponent") ---- */
int32_t orc_exponent_max(const float x[64])
{
    float mx = 0.0f;
    for (int i = 0; i < 64; i++) {
        float a = fabsf(x[i]);
        if (a > mx) mx = a;
    }
    if (mx == 0.0f) return -EBIAS;          /* zero block */
    int e;
    frexp((double)mx, &e);                  /* mx = f * 2^e, f in [0.5, 1) */
    return e < 1 - EBIAS ? 1 - EBIAS : e;   /* emax = max(e, -126) */
}

/* q = trunc(x * 2^(30-emax)); the product is exact in fp64 (reading R10) */
void orc_fwd_cast(const float x[64], int emax, int32_t q[64])
{
    double s = ldexp(1.0, 30 - emax);
    for (int i = 0; i < 64; i++) q[i] = (int32_t)trunc((double)x[i] * s);
}

/* x = fl32( fl32(q) * 2^(emax-30) ): one RNE rounding of the exact product */
void orc_inv_cast(const int32_t q[64], int emax, float x[64])
{
    double s = ldexp(1.0, emax - 30);
    for (int i = 0; i < 64; i++) x[i] = (float)((double)(float)q[i] * s);
}

/* ---- decorrelating transform (App. A "Forward lifting") ---- */
void orc_fwd_lift(int32_t v[4])
{
    int32_t x = v[0], y = v[1], z = v[2], w = v[3];
    x = wadd(x, w); x = asr1(x); w = wsub(w, x);
    z = wadd(z, y); z = asr1(z); y = wsub(y, z);
    x = wadd(x, z); x = asr1(x); z = wsub(z, x);
    w = wadd(w, y); w = asr1(w); y = wsub(y, w);
    w = wadd(w, asr1(y)); y = wsub(y, asr1(w));
    v[0] = x; v[1] = y; v[2] = z; v[3] = w;
}

void orc_inv_lift(int32_t v[4])
{
    int32_t x = v[0], y = v[1], z = v[2], w = v[3];
    y = wadd(y, asr1(w)); w = wsub(w, asr1(y));
    y = wadd(y, w); w = wshl1(w); w = wsub(w, y);
    z = wadd(z, x); x = wshl1(x); x = wsub(x, z);
    y = wadd(y, z); z = wshl1(z); z = wsub(z, y);
    w = wadd(w, x); x = wshl1(x); x = wsub(x, w);
    v[0] = x; v[1] = y; v[2] = z; v[3] = w;
}

/* apply a lift to the 4 values p[b], p[b+s], p[b+2s], p[b+3s] */
static void lift_line(int32_t* p, int b, int s, int inverse)
{
    int32_t v[4] = { p[b], p[b + s], p[b + 2 * s], p[b + 3 * s] };
    if (inverse) orc_inv_lift(v); else orc_fwd_lift(v);
    p[b] = v[0]; p[b + s] = v[1]; p[b + 2 * s] = v[2]; p[b + 3 * s] = v[3];
}

/* local index l = i + 4j + 16k (i along x) */
void orc_fwd_xform(int32_t q[64])
{
    for (int k = 0; k < 4; k++)             /* along x */
        for (int j = 0; j < 4; j++) lift_line(q, 4 * j + 16 * k, 1, 0);
    for (int k = 0; k < 4; k++)             /* along y */
        for (int i = 0; i < 4; i++) lift_line(q, i + 16 * k, 4, 0);
    for (int j = 0; j < 4; j++)             /* along z */
        for (int i = 0; i < 4; i++) lift_line(q, i + 4 * j, 16, 0);
}

void orc_inv_xform(int32_t q[64])
{
    for (int j = 0; j < 4; j++)             /* along z */
        for (int i = 0; i < 4; i++) lift_line(q, i + 4 * j, 16, 1);
    for (int k = 0; k < 4; k++)             /* along y */
        for (int i = 0; i < 4; i++) lift_line(q, i + 16 * k, 4, 1);
    for (int k = 0; k < 4; k++)             /* along x */
        for (int j = 0; j < 4; j++) lift_line(q, 4 * j + 16 * k, 1, 1);
}

/* ---- ordering and negabinary (App. A "Order and negabinary") ---- */
static const uint8_t PERM3[64] = {
    0, 1, 4, 16, 20, 17, 5, 2, 8, 32, 21, 6, 18, 24, 9, 33,
    36, 3, 12, 48, 22, 25, 37, 40, 34, 10, 7, 19, 28, 13, 49, 52,
    41, 38, 26, 23, 29, 53, 11, 35, 44, 14, 50, 56, 42, 27, 39, 45,
    30, 54, 57, 60, 51, 15, 43, 46, 58, 61, 55, 31, 62, 59, 47, 63 };

const uint8_t* orc_perm3(void) { return PERM3; }

uint32_t orc_int2uint(int32_t x) { return ((uint32_t)x + NBMASK) ^ NBMASK; }
int32_t  orc_uint2int(uint32_t u) { return (int32_t)((u ^ NBMASK) - NBMASK); }

/* ---- bit I/O, one bit at a time ---- */
typedef struct { uint64_t* w; long pos; } bw_t;
static void put_bit(bw_t* s, unsigned bit)
{
    if (bit) s->w[s->pos >> 6] |= (uint64_t)1 << (s->pos & 63);
    s->pos++;
}
typedef struct { const uint64_t* w; long pos; } br_t;
static unsigned get_bit(br_t* s)
{
    unsigned b = (unsigned)((s->w[s->pos >> 6] >> (s->pos & 63)) & 1u);
    s->pos++;
    return b;
}

/* ---- embedded bit-plane coder with group testing (App. A "Embedded coder") ----
 * Writes into words starting at bit_offset (the words must be zeroed by the
 * caller); returns the number of bits written (<= budget_bits). */
int orc_encode_ints(const uint32_t u[64], int budget_bits, uint64_t* words, int bit_offset)
{
    bw_t s = { words, bit_offset };
    int bits = budget_bits;
    int n = 0;                                  /* coefficients already significant */
    for (int k = 31; k >= 0 && bits > 0; k--) {
        /* step 1: bit plane k as a 64-bit word, coefficient i -> bit i */
        uint64_t x = 0;
        for (int i = 0; i < 64; i++) x += (uint64_t)((u[i] >> k) & 1u) << i;
        /* step 2: first n bits verbatim */
        int m = n < bits ? n : bits;
        bits -= m;
        for (int i = 0; i < m; i++) { put_bit(&s, (unsigned)(x & 1u)); x >>= 1; }
        /* step 3: unary run-length (group test) coding of the rest */
        while (n < 64 && bits > 0) {
            bits--;
            put_bit(&s, x != 0);
            if (x == 0) break;
            while (n < 63 && bits > 0) {
                bits--;
                unsigned b = (unsigned)(x & 1u);
                put_bit(&s, b);
                if (b) break;
                x >>= 1; n++;
            }
            x >>= 1; n++;
        }
    }
    return budget_bits - bits;
}

int orc_decode_ints(const uint64_t* words, int bit_offset, int budget_bits, uint32_t u[64])
{
    br_t s = { words, bit_offset };
    int bits = budget_bits;
    int n = 0;
    for (int i = 0; i < 64; i++) u[i] = 0;
    for (int k = 31; k >= 0 && bits > 0; k--) {
        int m = n < bits ? n : bits;
        bits -= m;
        uint64_t x = 0;
        for (int i = 0; i < m; i++) x |= (uint64_t)get_bit(&s) << i;
        while (n < 64 && bits > 0) {
            bits--;
            if (!get_bit(&s)) break;            /* group is empty */
            while (n < 63 && bits > 0) {
                bits--;
                if (get_bit(&s)) break;
                n++;
            }
            /* zfp deposits a one at position n even when the budget ran out
             * inside the scan (App. A, decoder note) */
            x += (uint64_t)1 << n;
            n++;
        }
        for (int i = 0; i < 64; i++) u[i] += (uint32_t)((x >> i) & 1u) << k;
    }
    return budget_bits - bits;
}

/* ---- one 4^3 block ---- */
int orc_encode_block(const float x[64], int rate, uint64_t* out)
{
    const int maxbits = 64 * rate;
    memset(out, 0, sizeof(uint64_t) * (size_t)rate);
    bw_t s = { out, 0 };
    int emax = orc_exponent_max(x);
    int e = emax + EBIAS;                       /* biased; 0 <=> all-zero block */
    if (e == 0) {
        put_bit(&s, 0);                         /* then zero padding */
        return 1;
    }
    /* 1 + EBITS bits: the value 2e+1, LSB first */
    unsigned ev = 2u * (unsigned)e + 1u;
    for (int i = 0; i < 1 + EBITS; i++) put_bit(&s, (ev >> i) & 1u);
    int32_t q[64];
    orc_fwd_cast(x, emax, q);
    orc_fwd_xform(q);
    uint32_t u[64];
    for (int i = 0; i < 64; i++) u[i] = orc_int2uint(q[PERM3[i]]);
    int used = orc_encode_ints(u, maxbits - (1 + EBITS), out, 1 + EBITS);
    return 1 + EBITS + used;
}

int orc_decode_block(const uint64_t* in, int rate, float x[64])
{
    const int maxbits = 64 * rate;
    br_t s = { in, 0 };
    if (!get_bit(&s)) {
        for (int i = 0; i < 64; i++) x[i] = 0.0f;
        return 1;
    }
    unsigned e = 0;
    for (int i = 0; i < EBITS; i++) e |= get_bit(&s) << i;
    int emax = (int)e - EBIAS;
    uint32_t u[64];
    int used = orc_decode_ints(in, 1 + EBITS, maxbits - (1 + EBITS), u);
    int32_t q[64];
    for (int i = 0; i < 64; i++) q[PERM3[i]] = orc_uint2int(u[i]);
    orc_inv_xform(q);
    orc_inv_cast(q, emax, x);
    return 1 + EBITS + used;
}

/* ---- whole arrays ---- */
size_t orc_zfp_bytes(int nx, int ny, int nz, int rate)
{
    return (size_t)(nx / 4) * (size_t)(ny / 4) * (size_t)(nz / 4) * 8u * (size_t)rate;
}

static int bad_args(int nx, int ny, int nz, int rate)
{
    return nx < 0 || ny < 0 || nz < 0 || nx % 4 || ny % 4 || nz % 4 || rate < 1 || rate > 64;
}

int orc_zfp_encode(const float* f, int nx, int ny, int nz, int rate, uint64_t* out)
{
    if (bad_args(nx, ny, nz, rate)) return -1;
    const long bx_n = nx / 4, by_n = ny / 4, bz_n = nz / 4;
    #pragma omp parallel for schedule(static)
    for (long bz = 0; bz < bz_n; bz++)
        for (long by = 0; by < by_n; by++)
            for (long bx = 0; bx < bx_n; bx++) {
                float blk[64];
                for (int k = 0; k < 4; k++)
                    for (int j = 0; j < 4; j++)
                        for (int i = 0; i < 4; i++)
                            blk[i + 4 * j + 16 * k] =
                                f[((size_t)(4 * bz + k) * ny + (size_t)(4 * by + j)) * nx + (size_t)(4 * bx + i)];
                long b = bx + bx_n * (by + by_n * bz);
                orc_encode_block(blk, rate, out + (size_t)b * (size_t)rate);
            }
    return 0;
}

int orc_zfp_decode(const uint64_t* in, int nx, int ny, int nz, int rate, float* f)
{
    if (bad_args(nx, ny, nz, rate)) return -1;
    const long bx_n = nx / 4, by_n = ny / 4, bz_n = nz / 4;
    #pragma omp parallel for schedule(static)
    for (long bz = 0; bz < bz_n; bz++)
        for (long by = 0; by < by_n; by++)
            for (long bx = 0; bx < bx_n; bx++) {
                float blk[64];
                long b = bx + bx_n * (by + by_n * bz);
                orc_decode_block(in + (size_t)b * (size_t)rate, rate, blk);
                for (int k = 0; k < 4; k++)
                    for (int j = 0; j < 4; j++)
                        for (int i = 0; i < 4; i++)
                            f[((size_t)(4 * bz + k) * ny + (size_t)(4 * by + j)) * nx + (size_t)(4 * bx + i)] =
                                blk[i + 4 * j + 16 * k];
            }
    return 0;
}

int orc_roundtrip(float* f, int nx, int ny, int nz, int rate)
{
    if (rate == 0) return 0;                    /* raw field: identity */
    if (bad_args(nx, ny, nz, rate)) return -1;
    size_t nb = orc_zfp_bytes(nx, ny, nz, rate);
    uint64_t* buf = (uint64_t*)malloc(nb ? nb : 8);
    if (!buf) return -2;
    orc_zfp_encode(f, nx, ny, nz, rate, buf);
    orc_zfp_decode(buf, nx, ny, nz, rate, f);
    free(buf);
    return 0;
}
