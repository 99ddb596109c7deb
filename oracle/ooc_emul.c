/*
 * ooc_emul.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Literal emulation of the paper's out-of-core schedule on tiny grids, used
 * to pin the reduction of SURVEY 8(c) c.0 (out-of-core result == in-core
 * steps + whole-field round trip after every sweep), and to count bytes.
 *
 *  - Decomposition into blocks of P planes along z, temporal blocking of T
 *    steps per residency with halo h = 4T (Sec. III; Fig. 1b;
 *    D = 8, T = 12 in PAPER.md:217).
 *  - Region sharing (Fig. 3): contiguous blocks share the
 *    common region C_i = [(i+1)P-h, (i+1)P+h); remainders
 *    R_i = [iP+h, (i+1)P-h) (R_0 starts at the slab top, R_{D-1} ends at the
 *    slab bottom).
 *  - Separate compression (Sec. V.A, Fig. 4): every R_i and
 *    every C_i is its own compressed payload.  Before computing, block i
 *    decompresses R_i and C_i (Fig. 4a); C_{i-1} is already on the GPU.  After
 *    computing, the results are compressed to update the i-th remainder and the
 *    (i-1)-th common region (Fig. 4b caption, reading R13).  The time-t copy of
 *    C_i needed by block i+1 is kept (reading R14).
 *  - The read-only dataset is compressed once and never re-encoded
 *    (reading R15).
 *  - Multi-GPU extension (reading R20): G contiguous z-slabs, each with its
 *    own store; at the start of a sweep each slab receives the time-t
 *    boundary h planes of its neighbours (compressed form), m halos once.
 *  - poison != 0: before every step, planes outside the still-valid cone are
 *    set to NaN (SPEC.md:231 poison test); results must not change.
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* Element type and the codec / stencil of that precision.  Defaults: fp32.
 * ooc_emul64.c defines these for fp64 and includes this file (the schedule
 * below is written once, for both precisions). */
#ifndef OOC_REAL
#define OOC_REAL float
#define OOC_BYTES orc_zfp_bytes
#define OOC_ENCODE orc_zfp_encode
#define OOC_DECODE orc_zfp_decode
#define OOC_STEP_PLANES orc_step_planes
#define OOC_EMULATE orc_ooc_emulate
#define OOC_NAN nanf("")
#endif
typedef OOC_REAL real;

typedef struct {
    int z0, z1;          /* global planes [z0, z1) */
    size_t bytes;
    void* payload;       /* uint64 words (rate > 0) or raw values (rate == 0) */
} region_t;

static size_t plane_elems(int nx, int ny) { return (size_t)nx * (size_t)ny; }

static size_t region_bytes(int nx, int ny, int nplanes, int rate)
{
    if (rate == 0) return plane_elems(nx, ny) * (size_t)nplanes * sizeof(real);
    return OOC_BYTES(nx, ny, nplanes, rate);
}

/* compress planes src[0 .. nplanes) into a region payload */
static void region_put(region_t* r, const real* src, int nx, int ny, int rate)
{
    int np = r->z1 - r->z0;
    r->bytes = region_bytes(nx, ny, np, rate);
    free(r->payload);
    r->payload = malloc(r->bytes ? r->bytes : 8);
    if (rate == 0) memcpy(r->payload, src, r->bytes);
    else OOC_ENCODE(src, nx, ny, np, rate, (uint64_t*)r->payload);
}

static void region_get(const region_t* r, real* dst, int nx, int ny, int rate)
{
    int np = r->z1 - r->z0;
    if (rate == 0) memcpy(dst, r->payload, r->bytes);
    else OOC_DECODE((const uint64_t*)r->payload, nx, ny, np, rate, dst);
}

/* region index: 2i = R_i, 2i+1 = C_i */
static void region_bounds(int g, int i_reg, int S, int P, int h, int D, int* z0, int* z1)
{
    int base = g * S;
    int i = i_reg / 2;
    if (i_reg % 2 == 1) {                       /* C_i */
        *z0 = base + (i + 1) * P - h;
        *z1 = base + (i + 1) * P + h;
    } else {                                    /* R_i */
        *z0 = i == 0 ? base : base + i * P + h;
        *z1 = i == D - 1 ? base + S : base + (i + 1) * P - h;
    }
}

/* decode the planes [z0, z1) of slab g's field from whichever region holds them */
static void slab_planes(region_t* regs, int nreg, int z0, int z1, real* dst,
                        int nx, int ny, int rate)
{
    size_t pe = plane_elems(nx, ny);
    for (int r = 0; r < nreg; r++) {
        int a = regs[r].z0, b = regs[r].z1;
        int lo = z0 > a ? z0 : a, hi = z1 < b ? z1 : b;
        if (lo >= hi) continue;
        real* tmp = (real*)malloc(pe * (size_t)(b - a) * sizeof(real) + 4);
        region_get(&regs[r], tmp, nx, ny, rate);
        memcpy(dst + pe * (size_t)(lo - z0), tmp + pe * (size_t)(lo - a), pe * (size_t)(hi - lo) * sizeof(real));
        free(tmp);
    }
}

static void poison_outside(real* buf, int zlo, int L, int nz, int v0, int v1, size_t pe)
{
    const real nanv = OOC_NAN;
    for (int zl = 0; zl < L; zl++) {
        int z = zlo + zl;
        if (z < 0 || z >= nz) continue;         /* Dirichlet ghost planes stay 0 */
        if (z >= v0 && z < v1) continue;
        for (size_t e = 0; e < pe; e++) buf[(size_t)zl * pe + e] = nanv;
    }
}

int OOC_EMULATE(real* u, real* uprev, const real* m, int nx, int ny, int nz,
                const real c[5], int T, int P, int G, const int rate[3],
                    long nsteps, int poison, uint64_t stats[3])
{
    const int h = 4 * T;
    if (T < 1 || G < 1 || nz % G) return -1;
    const int S = nz / G;
    if (P < 2 * h || P % 4 || h % 4 || S % P || nx % 4 || ny % 4) return -1;
    const int D = S / P;
    const int nreg = 2 * D - 1;
    const size_t pe = plane_elems(nx, ny);
    stats[0] = stats[1] = stats[2] = 0;

    /* store[f][g][r] */
    region_t* store = (region_t*)calloc((size_t)3 * G * nreg, sizeof(region_t));
    #define REG(f, g, r) store[((size_t)(f) * G + (g)) * nreg + (r)]
    const real* init[3] = { u, uprev, m };
    /* set_field: initial compression of every region of every field */
    for (int f = 0; f < 3; f++)
        for (int g = 0; g < G; g++)
            for (int r = 0; r < nreg; r++) {
                region_t* R = &REG(f, g, r);
                region_bounds(g, r, S, P, h, D, &R->z0, &R->z1);
                region_put(R, init[f] + pe * (size_t)R->z0, nx, ny, rate[f]);
            }

    /* m halos (read-only): exchanged once, compressed (reading R20) */
    real* mtop = (real*)calloc(pe * (size_t)h * G + 1, sizeof(real));
    real* mbot = (real*)calloc(pe * (size_t)h * G + 1, sizeof(real));
    for (int g = 0; g < G; g++) {
        if (g > 0) {
            slab_planes(&REG(2, g - 1, 0), nreg, g * S - h, g * S, mtop + pe * (size_t)h * g, nx, ny, rate[2]);
            stats[2] += region_bytes(nx, ny, h, rate[2]);
        }
        if (g < G - 1) {
            slab_planes(&REG(2, g + 1, 0), nreg, (g + 1) * S, (g + 1) * S + h, mbot + pe * (size_t)h * g, nx, ny, rate[2]);
            stats[2] += region_bytes(nx, ny, h, rate[2]);
        }
    }

    const int L = P + 2 * h;                    /* slab planes per block */
    real* A = (real*)malloc(pe * L * sizeof(real) + 4);
    real* B = (real*)malloc(pe * L * sizeof(real) + 4);
    real* M = (real*)malloc(pe * L * sizeof(real) + 4);
    real* ccopy[3];                            /* time-t copy of C_i */
    real* keep[2];                             /* t+T values of C_i's upper half */
    for (int f = 0; f < 3; f++) ccopy[f] = (real*)malloc(pe * 2 * h * sizeof(real) + 4);
    for (int f = 0; f < 2; f++) keep[f] = (real*)malloc(pe * h * sizeof(real) + 4);
    real* top[2]; real* bot[2];
    for (int f = 0; f < 2; f++) {
        top[f] = (real*)calloc(pe * (size_t)h * G + 1, sizeof(real));
        bot[f] = (real*)calloc(pe * (size_t)h * G + 1, sizeof(real));
    }

    long done = 0;
    while (done < nsteps) {
        const int ts = (int)(nsteps - done < T ? nsteps - done : T);
        /* halo snapshot at time t: compressed boundary planes from the neighbours */
        for (int g = 0; g < G; g++)
            for (int f = 0; f < 2; f++) {
                if (g > 0) {
                    slab_planes(&REG(f, g - 1, 0), nreg, g * S - h, g * S, top[f] + pe * (size_t)h * g, nx, ny, rate[f]);
                    stats[2] += region_bytes(nx, ny, h, rate[f]);
                }
                if (g < G - 1) {
                    slab_planes(&REG(f, g + 1, 0), nreg, (g + 1) * S, (g + 1) * S + h, bot[f] + pe * (size_t)h * g, nx, ny, rate[f]);
                    stats[2] += region_bytes(nx, ny, h, rate[f]);
                }
            }
        for (int g = 0; g < G; g++) {
            for (int i = 0; i < D; i++) {
                const int zlo = g * S + i * P - h, zhi = g * S + (i + 1) * P + h;
                real* F[3] = { A, B, M };
                for (int f = 0; f < 3; f++) memset(F[f], 0, pe * L * sizeof(real));
                /* top 2h planes: C_{i-1} from the previous block, or the halo from slab g-1 */
                if (i > 0) {
                    for (int f = 0; f < 3; f++) memcpy(F[f], ccopy[f], pe * 2 * h * sizeof(real));
                } else if (g > 0) {
                    memcpy(A, top[0] + pe * (size_t)h * g, pe * h * sizeof(real));
                    memcpy(B, top[1] + pe * (size_t)h * g, pe * h * sizeof(real));
                    memcpy(M, mtop + pe * (size_t)h * g, pe * h * sizeof(real));
                }
                /* Fig. 4a: decompress this block's remainder and common region */
                int regs[2] = { 2 * i, 2 * i + 1 };
                int nr = i < D - 1 ? 2 : 1;
                for (int k = 0; k < nr; k++)
                    for (int f = 0; f < 3; f++) {
                        region_t* R = &REG(f, g, regs[k]);
                        region_get(R, F[f] + pe * (size_t)(R->z0 - zlo), nx, ny, rate[f]);
                        stats[0] += R->bytes;
                    }
                if (i == D - 1 && g < G - 1) {
                    int off = (g + 1) * S - zlo;
                    memcpy(A + pe * (size_t)off, bot[0] + pe * (size_t)h * g, pe * h * sizeof(real));
                    memcpy(B + pe * (size_t)off, bot[1] + pe * (size_t)h * g, pe * h * sizeof(real));
                    memcpy(M + pe * (size_t)off, mbot + pe * (size_t)h * g, pe * h * sizeof(real));
                }
                /* keep the time-t C_i for block i+1 (reading R14) */
                if (i < D - 1)
                    for (int f = 0; f < 3; f++)
                        memcpy(ccopy[f], F[f] + pe * (size_t)(P), pe * 2 * h * sizeof(real));
                /* temporal blocking: step s updates the cone [zlo+4s, zhi-4s) */
                real* cu = A; real* cp = B;
                for (int s = 1; s <= ts; s++) {
                    if (poison) {
                        poison_outside(cu, zlo, L, nz, zlo + 4 * (s - 1), zhi - 4 * (s - 1), pe);
                        poison_outside(cp, zlo, L, nz, zlo + 4 * (s - 1), zhi - 4 * (s - 1), pe);
                    }
                    int g0 = zlo + 4 * s > 0 ? zlo + 4 * s : 0;
                    int g1 = zhi - 4 * s < nz ? zhi - 4 * s : nz;
                    /* in place: u+ overwrites u- (only the same point is read) */
                    OOC_STEP_PLANES(cu, cp, M, cp, nx, ny, L, c, g0 - zlo, g1 - zlo);
                    real* t = cu; cu = cp; cp = t;
                }
                /* Fig. 4b: compress R_i and C_{i-1} and write them back */
                real* out[2] = { cu, cp };
                for (int f = 0; f < 2; f++) {
                    region_t* R = &REG(f, g, 2 * i);
                    region_put(R, out[f] + pe * (size_t)(R->z0 - zlo), nx, ny, rate[f]);
                    stats[1] += R->bytes;
                    if (i > 0) {
                        region_t* C = &REG(f, g, 2 * i - 1);
                        real* tmp = (real*)malloc(pe * 2 * h * sizeof(real));
                        memcpy(tmp, keep[f], pe * h * sizeof(real));
                        memcpy(tmp + pe * h, out[f] + pe * (size_t)h, pe * h * sizeof(real));
                        region_put(C, tmp, nx, ny, rate[f]);
                        stats[1] += C->bytes;
                        free(tmp);
                    }
                    if (i < D - 1)  /* upper half of C_i: own planes, kept for block i+1 */
                        memcpy(keep[f], out[f] + pe * (size_t)P, pe * h * sizeof(real));
                }
            }
        }
        done += ts;
    }

    /* read back */
    for (int g = 0; g < G; g++) {
        slab_planes(&REG(0, g, 0), nreg, g * S, (g + 1) * S, u + pe * (size_t)g * S, nx, ny, rate[0]);
        slab_planes(&REG(1, g, 0), nreg, g * S, (g + 1) * S, uprev + pe * (size_t)g * S, nx, ny, rate[1]);
    }
    #undef REG
    for (size_t k = 0; k < (size_t)3 * G * nreg; k++) free(store[k].payload);
    free(store); free(A); free(B); free(M); free(mtop); free(mbot);
    for (int f = 0; f < 3; f++) free(ccopy[f]);
    for (int f = 0; f < 2; f++) { free(keep[f]); free(top[f]); free(bot[f]); }
    return 0;
}
