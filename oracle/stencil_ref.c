/*
 * stencil_ref.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * In-core 25-point (radius-4, 8th-order in space) leapfrog for the acoustic
 * wave equation, the propagator of PAPER.md:208 (Sec. VI; HALO = 4 in
 * Table I).  The paper does not print the scheme; the readings
 * (R1-R5) are:
 *   u+ = 2u - u- + m * L(u),   L(u) = 3*c0*u + sum_{k=1..4} c_k * s_k,
 *   s_k = sum of the 6 axis neighbours at distance k, zero outside the grid,
 *   c = (-205/72, 8/5, -1/5, 8/315, -1/560), m = (v dt/dx)^2 (read-only field).
 * Evaluation order, fp32 round-to-nearest, no contraction
 * (compiled with -ffp-contract=off), explicit fmaf:
 *   s_d = ((u[x-d]+u[x+d]) + (u[y-d]+u[y+d])) + (u[z-d]+u[z+d])
 *   L = c0x3*u0; L = fmaf(c1,s1,L); ...; L = fmaf(c4,s4,L)
 *   u+ = fmaf(m, L, fmaf(2, u0, -u-))
 *
 * orc_advance is the reduced form of the out-of-core method (SURVEY 8(c)
 * c.0): in-core steps with the whole-field codec round trip RT applied to the
 * two read-write fields at the end of every sweep of T steps.
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

void orc_default_coeffs(float c[5])
{
    /* standard 8th-order central second-derivative weights, rounded to fp32 */
    c[0] = (float)(-205.0 / 72.0);
    c[1] = (float)(8.0 / 5.0);
    c[2] = (float)(-1.0 / 5.0);
    c[3] = (float)(8.0 / 315.0);
    c[4] = (float)(-1.0 / 560.0);
}

static float at(const float* u, int nx, int ny, int nz, long x, long y, long z)
{
    if (x < 0 || y < 0 || z < 0 || x >= nx || y >= ny || z >= nz) return 0.0f; /* Dirichlet ghost */
    return u[((size_t)z * ny + (size_t)y) * nx + (size_t)x];
}

static double atd(const double* u, int nx, int ny, int nz, long x, long y, long z)
{
    if (x < 0 || y < 0 || z < 0 || x >= nx || y >= ny || z >= nz) return 0.0;
    return u[((size_t)z * ny + (size_t)y) * nx + (size_t)x];
}

void orc_step_planes(const float* u, const float* uprev, const float* m, float* out,
                     int nx, int ny, int nz, const float c[5], int z0, int z1)
{
    const float c0x3 = 3.0f * c[0];
    if (z0 < 0) z0 = 0;
    if (z1 > nz) z1 = nz;
    #pragma omp parallel for schedule(static)
    for (long z = z0; z < z1; z++)
        for (long y = 0; y < ny; y++)
            for (long x = 0; x < nx; x++) {
                size_t idx = ((size_t)z * ny + (size_t)y) * nx + (size_t)x;
                float u0 = u[idx];
                float s[5];
                for (int d = 1; d <= 4; d++) {
                    float ax = at(u, nx, ny, nz, x - d, y, z) + at(u, nx, ny, nz, x + d, y, z);
                    float ay = at(u, nx, ny, nz, x, y - d, z) + at(u, nx, ny, nz, x, y + d, z);
                    float az = at(u, nx, ny, nz, x, y, z - d) + at(u, nx, ny, nz, x, y, z + d);
                    s[d] = (ax + ay) + az;
                }
                float L = c0x3 * u0;
                L = fmaf(c[1], s[1], L);
                L = fmaf(c[2], s[2], L);
                L = fmaf(c[3], s[3], L);
                L = fmaf(c[4], s[4], L);
                out[idx] = fmaf(m[idx], L, fmaf(2.0f, u0, -uprev[idx]));
            }
}

void orc_step(const float* u, const float* uprev, const float* m, float* out,
              int nx, int ny, int nz, const float c[5])
{
    orc_step_planes(u, uprev, m, out, nx, ny, nz, c, 0, nz);
}

void orc_step_planes_f64(const double* u, const double* uprev, const double* m, double* out,
                         int nx, int ny, int nz, const double c[5], int z0, int z1)
{
    const double c0x3 = 3.0 * c[0];
    if (z0 < 0) z0 = 0;
    if (z1 > nz) z1 = nz;
    #pragma omp parallel for schedule(static)
    for (long z = z0; z < z1; z++)
        for (long y = 0; y < ny; y++)
            for (long x = 0; x < nx; x++) {
                size_t idx = ((size_t)z * ny + (size_t)y) * nx + (size_t)x;
                double u0 = u[idx];
                double s[5];
                for (int d = 1; d <= 4; d++) {
                    double ax = atd(u, nx, ny, nz, x - d, y, z) + atd(u, nx, ny, nz, x + d, y, z);
                    double ay = atd(u, nx, ny, nz, x, y - d, z) + atd(u, nx, ny, nz, x, y + d, z);
                    double az = atd(u, nx, ny, nz, x, y, z - d) + atd(u, nx, ny, nz, x, y, z + d);
                    s[d] = (ax + ay) + az;
                }
                double L = c0x3 * u0;
                L = fma(c[1], s[1], L);
                L = fma(c[2], s[2], L);
                L = fma(c[3], s[3], L);
                L = fma(c[4], s[4], L);
                out[idx] = fma(m[idx], L, fma(2.0, u0, -uprev[idx]));
            }
}

void orc_step_f64(const double* u, const double* uprev, const double* m, double* out,
                  int nx, int ny, int nz, const double c[5])
{
    orc_step_planes_f64(u, uprev, m, out, nx, ny, nz, c, 0, nz);
}

int orc_advance(float* u, float* uprev, const float* m, int nx, int ny, int nz,
                const float c[5], int T, const int rate[3], long nsteps)
{
    if (T < 1 || nsteps < 0) return -1;
    size_t n = (size_t)nx * ny * nz;
    float* nxt = (float*)malloc((n ? n : 1) * sizeof(float));
    if (!nxt) return -2;
    long done = 0;
    while (done < nsteps) {
        long ts = nsteps - done < T ? nsteps - done : T;   /* last sweep: n mod T */
        for (long s = 0; s < ts; s++) {
            /* (U, U-) <- (leap(U, U-, M), U) */
            orc_step(u, uprev, m, nxt, nx, ny, nz, c);
            memcpy(uprev, u, n * sizeof(float));
            memcpy(u, nxt, n * sizeof(float));
        }
        /* every sweep ends with the read-write fields re-encoded (Fig. 4b) */
        orc_roundtrip(u, nx, ny, nz, rate[0]);
        orc_roundtrip(uprev, nx, ny, nz, rate[1]);
        done += ts;
    }
    free(nxt);
    return 0;
}
