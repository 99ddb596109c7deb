/*
 * zfp_ref64.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Bit-serial ZFP-style fixed-rate coder for fp64 3-D arrays: the same format
 * as zfp_ref.c instantiated for double precision, the
 * paper's own precision (its codes 2-4 use 32/64 and 24/64 bits
 * per value):
 *   EBITS = 11, EBIAS = 1023, integer precision 64 (64 bit planes),
 *   NBMASK = 0xaaaaaaaaaaaaaaaa, q = trunc(x * 2^(62 - emax)),
 *   header = 1 + 11 bits (2e + 1), bit-plane budget 64*rate - 12.
 * Readings (R10 for fp64): quantise with ldexp (exact, no overflow
 * of an intermediate scale factor) and truncate; dequantise as one RNE rounding
 * of fl64(q) * 2^(emax - 62) (ldexp of the rounded integer).
 * Parity vs real zfp: UNPINNED (no zfp here); pinned by tests/test_oracle_zfp64.py.
 */
#include "oracle.h"
#include <math.h>
#include <string.h>
#include <stdlib.h>

#define EBITS64 11
#define EBIAS64 1023
#define NBMASK64 0xaaaaaaaaaaaaaaaaull

static int64_t wadd64(int64_t a, int64_t b) { return (int64_t)((uint64_t)a + (uint64_t)b); }
static int64_t wsub64(int64_t a, int64_t b) { return (int64_t)((uint64_t)a - (uint64_t)b); }
static int64_t wshl1_64(int64_t a) { return (int64_t)((uint64_t)a << 1); }
static int64_t asr1_64(int64_t a) { return (int64_t)(a >> 1); } /* gcc: arithmetic */

int32_t orc64_exponent_max(const double x[64])
{
    double mx = 0.0;
    for (int i = 0; i < 64; i++) {
        double a = fabs(x[i]);
        if (a > mx) mx = a;
    }
    if (mx == 0.0) return -EBIAS64;
    int e;
    frexp(mx, &e);
    return e < 1 - EBIAS64 ? 1 - EBIAS64 : e;   /* max(e, -1022) */
}

void orc64_fwd_cast(const double x[64], int emax, int64_t q[64])
{
    for (int i = 0; i < 64; i++) q[i] = (int64_t)trunc(ldexp(x[i], 62 - emax));
}

void orc64_inv_cast(const int64_t q[64], int emax, double x[64])
{
    for (int i = 0; i < 64; i++) x[i] = ldexp((double)q[i], emax - 62);
}

void orc64_fwd_lift(int64_t v[4])
{
    int64_t x = v[0], y = v[1], z = v[2], w = v[3];
    x = wadd64(x, w); x = asr1_64(x); w = wsub64(w, x);
    z = wadd64(z, y); z = asr1_64(z); y = wsub64(y, z);
    x = wadd64(x, z); x = asr1_64(x); z = wsub64(z, x);
    w = wadd64(w, y); w = asr1_64(w); y = wsub64(y, w);
    w = wadd64(w, asr1_64(y)); y = wsub64(y, asr1_64(w));
    v[0] = x; v[1] = y; v[2] = z; v[3] = w;
}

void orc64_inv_lift(int64_t v[4])
{
    int64_t x = v[0], y = v[1], z = v[2], w = v[3];
    y = wadd64(y, asr1_64(w)); w = wsub64(w, asr1_64(y));
    y = wadd64(y, w); w = wshl1_64(w); w = wsub64(w, y);
    z = wadd64(z, x); x = wshl1_64(x); x = wsub64(x, z);
    y = wadd64(y, z); z = wshl1_64(z); z = wsub64(z, y);
    w = wadd64(w, x); x = wshl1_64(x); x = wsub64(x, w);
    v[0] = x; v[1] = y; v[2] = z; v[3] = w;
}

static void lift_line64(int64_t* p, int b, int s, int inverse)
{
    int64_t v[4] = { p[b], p[b + s], p[b + 2 * s], p[b + 3 * s] };
    if (inverse) orc64_inv_lift(v); else orc64_fwd_lift(v);
    p[b] = v[0]; p[b + s] = v[1]; p[b + 2 * s] = v[2]; p[b + 3 * s] = v[3];
}

void orc64_fwd_xform(int64_t q[64])
{
    for (int k = 0; k < 4; k++)
        for (int j = 0; j < 4; j++) lift_line64(q, 4 * j + 16 * k, 1, 0);
    for (int k = 0; k < 4; k++)
        for (int i = 0; i < 4; i++) lift_line64(q, i + 16 * k, 4, 0);
    for (int j = 0; j < 4; j++)
        for (int i = 0; i < 4; i++) lift_line64(q, i + 4 * j, 16, 0);
}

void orc64_inv_xform(int64_t q[64])
{
    for (int j = 0; j < 4; j++)
        for (int i = 0; i < 4; i++) lift_line64(q, i + 4 * j, 16, 1);
    for (int k = 0; k < 4; k++)
        for (int i = 0; i < 4; i++) lift_line64(q, i + 16 * k, 4, 1);
    for (int k = 0; k < 4; k++)
        for (int j = 0; j < 4; j++) lift_line64(q, 4 * j + 16 * k, 1, 1);
}

uint64_t orc64_int2uint(int64_t x) { return ((uint64_t)x + NBMASK64) ^ NBMASK64; }
int64_t  orc64_uint2int(uint64_t u) { return (int64_t)((u ^ NBMASK64) - NBMASK64); }

typedef struct { uint64_t* w; long pos; } bw64_t;
static void put_bit64(bw64_t* s, unsigned bit)
{
    if (bit) s->w[s->pos >> 6] |= (uint64_t)1 << (s->pos & 63);
    s->pos++;
}
typedef struct { const uint64_t* w; long pos; } br64_t;
static unsigned get_bit64(br64_t* s)
{
    unsigned b = (unsigned)((s->w[s->pos >> 6] >> (s->pos & 63)) & 1u);
    s->pos++;
    return b;
}

/* embedded group-tested coder over 64 bit planes (k = 63 .. 0) of 64 values */
int orc64_encode_ints(const uint64_t u[64], int budget_bits, uint64_t* words, int bit_offset)
{
    bw64_t s = { words, bit_offset };
    int bits = budget_bits;
    int n = 0;
    for (int k = 63; k >= 0 && bits > 0; k--) {
        uint64_t x = 0;
        for (int i = 0; i < 64; i++) x += ((u[i] >> k) & 1u) << i;
        int m = n < bits ? n : bits;
        bits -= m;
        for (int i = 0; i < m; i++) { put_bit64(&s, (unsigned)(x & 1u)); x >>= 1; }
        while (n < 64 && bits > 0) {
            bits--;
            put_bit64(&s, x != 0);
            if (x == 0) break;
            while (n < 63 && bits > 0) {
                bits--;
                unsigned b = (unsigned)(x & 1u);
                put_bit64(&s, b);
                if (b) break;
                x >>= 1; n++;
            }
            x >>= 1; n++;
        }
    }
    return budget_bits - bits;
}

int orc64_decode_ints(const uint64_t* words, int bit_offset, int budget_bits, uint64_t u[64])
{
    br64_t s = { words, bit_offset };
    int bits = budget_bits;
    int n = 0;
    for (int i = 0; i < 64; i++) u[i] = 0;
    for (int k = 63; k >= 0 && bits > 0; k--) {
        int m = n < bits ? n : bits;
        bits -= m;
        uint64_t x = 0;
        for (int i = 0; i < m; i++) x |= (uint64_t)get_bit64(&s) << i;
        while (n < 64 && bits > 0) {
            bits--;
            if (!get_bit64(&s)) break;
            while (n < 63 && bits > 0) {
                bits--;
                if (get_bit64(&s)) break;
                n++;
            }
            x += (uint64_t)1 << n;               /* zfp's deposit, also when the budget ran out */
            n++;
        }
        for (int i = 0; i < 64; i++) u[i] += ((x >> i) & 1u) << k;
    }
    return budget_bits - bits;
}

extern const uint8_t* orc_perm3(void);

int orc64_encode_block(const double x[64], int rate, uint64_t* out)
{
    const int maxbits = 64 * rate;
    memset(out, 0, sizeof(uint64_t) * (size_t)rate);
    bw64_t s = { out, 0 };
    int emax = orc64_exponent_max(x);
    int e = emax + EBIAS64;
    if (e == 0) { put_bit64(&s, 0); return 1; }
    unsigned ev = 2u * (unsigned)e + 1u;
    for (int i = 0; i < 1 + EBITS64; i++) put_bit64(&s, (ev >> i) & 1u);
    int64_t q[64];
    orc64_fwd_cast(x, emax, q);
    orc64_fwd_xform(q);
    const uint8_t* perm = orc_perm3();
    uint64_t u[64];
    for (int i = 0; i < 64; i++) u[i] = orc64_int2uint(q[perm[i]]);
    int used = orc64_encode_ints(u, maxbits - (1 + EBITS64), out, 1 + EBITS64);
    return 1 + EBITS64 + used;
}

int orc64_decode_block(const uint64_t* in, int rate, double x[64])
{
    const int maxbits = 64 * rate;
    br64_t s = { in, 0 };
    if (!get_bit64(&s)) {
        for (int i = 0; i < 64; i++) x[i] = 0.0;
        return 1;
    }
    unsigned e = 0;
    for (int i = 0; i < EBITS64; i++) e |= get_bit64(&s) << i;
    int emax = (int)e - EBIAS64;
    uint64_t u[64];
    int used = orc64_decode_ints(in, 1 + EBITS64, maxbits - (1 + EBITS64), u);
    const uint8_t* perm = orc_perm3();
    int64_t q[64];
    for (int i = 0; i < 64; i++) q[perm[i]] = orc64_uint2int(u[i]);
    orc64_inv_xform(q);
    orc64_inv_cast(q, emax, x);
    return 1 + EBITS64 + used;
}

static int bad_args64(int nx, int ny, int nz, int rate)
{
    return nx < 0 || ny < 0 || nz < 0 || nx % 4 || ny % 4 || nz % 4 || rate < 1 || rate > 64;
}

int orc64_zfp_encode(const double* f, int nx, int ny, int nz, int rate, uint64_t* out)
{
    if (bad_args64(nx, ny, nz, rate)) return -1;
    const long bx_n = nx / 4, by_n = ny / 4, bz_n = nz / 4;
    #pragma omp parallel for schedule(static)
    for (long bz = 0; bz < bz_n; bz++)
        for (long by = 0; by < by_n; by++)
            for (long bx = 0; bx < bx_n; bx++) {
                double blk[64];
                for (int k = 0; k < 4; k++)
                    for (int j = 0; j < 4; j++)
                        for (int i = 0; i < 4; i++)
                            blk[i + 4 * j + 16 * k] =
                                f[((size_t)(4 * bz + k) * ny + (size_t)(4 * by + j)) * nx + (size_t)(4 * bx + i)];
                long b = bx + bx_n * (by + by_n * bz);
                orc64_encode_block(blk, rate, out + (size_t)b * (size_t)rate);
            }
    return 0;
}

int orc64_zfp_decode(const uint64_t* in, int nx, int ny, int nz, int rate, double* f)
{
    if (bad_args64(nx, ny, nz, rate)) return -1;
    const long bx_n = nx / 4, by_n = ny / 4, bz_n = nz / 4;
    #pragma omp parallel for schedule(static)
    for (long bz = 0; bz < bz_n; bz++)
        for (long by = 0; by < by_n; by++)
            for (long bx = 0; bx < bx_n; bx++) {
                double blk[64];
                long b = bx + bx_n * (by + by_n * bz);
                orc64_decode_block(in + (size_t)b * (size_t)rate, rate, blk);
                for (int k = 0; k < 4; k++)
                    for (int j = 0; j < 4; j++)
                        for (int i = 0; i < 4; i++)
                            f[((size_t)(4 * bz + k) * ny + (size_t)(4 * by + j)) * nx + (size_t)(4 * bx + i)] =
                                blk[i + 4 * j + 16 * k];
            }
    return 0;
}

int orc64_roundtrip(double* f, int nx, int ny, int nz, int rate)
{
    if (rate == 0) return 0;
    if (bad_args64(nx, ny, nz, rate)) return -1;
    size_t nb = orc_zfp_bytes(nx, ny, nz, rate);
    uint64_t* buf = (uint64_t*)malloc(nb ? nb : 8);
    if (!buf) return -2;
    orc64_zfp_encode(f, nx, ny, nz, rate, buf);
    orc64_zfp_decode(buf, nx, ny, nz, rate, f);
    free(buf);
    return 0;
}

/* SURVEY 8(c) c.0 schedule in fp64 (the fp64 twin of orc_advance) */
int orc64_advance(double* u, double* uprev, const double* m, int nx, int ny, int nz,
                  const double c[5], int T, const int rate[3], long nsteps)
{
    if (T < 1 || nsteps < 0) return -1;
    size_t n = (size_t)nx * ny * nz;
    double* nxt = (double*)malloc((n ? n : 1) * sizeof(double));
    if (!nxt) return -2;
    long done = 0;
    while (done < nsteps) {
        long ts = nsteps - done < T ? nsteps - done : T;
        for (long s = 0; s < ts; s++) {
            orc_step_f64(u, uprev, m, nxt, nx, ny, nz, c);
            memcpy(uprev, u, n * sizeof(double));
            memcpy(u, nxt, n * sizeof(double));
        }
        orc64_roundtrip(u, nx, ny, nz, rate[0]);
        orc64_roundtrip(uprev, nx, ny, nz, rate[1]);
        done += ts;
    }
    free(nxt);
    return 0;
}
