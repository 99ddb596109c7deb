// stencil.cu -- 25-point (radius-4) leapfrog step for sm_100a.
//
// The acoustic propagator of PAPER.md:208 (Sec. VI): two read-write time
// levels, a read-only model m, and a "write-only dataset" for intermediates,
// which here is fused away into registers.  HALO = 4.  One
// launch is one cone-limited step of temporal blocking:
// it updates planes [z0, z1) of a z-slab in place (u+ overwrites u-).
//
// Design (HBM-bound: >= 16 B per cell-update: read u, u-, m, write u+):
//  * CTA tile 128 (x) x 15 (y) cells marched along z; warp-specialised:
//    warp 0 is a TMA producer (one elected lane), warps 1..15 compute one row
//    each, 4 consecutive x per thread.  16 warps of <= 96 registers: each SM
//    sub-partition keeps room for one codec warp of the concurrent decode /
//    encode streams, and a 512^2 plane is 140 tiles (<= 148 SMs).
//  * Producer: cp.async.bulk.tensor.3d loads of
//      - the u plane tile with its radius-4 x/y halo (136 x 23 floats) into an
//        8-stage ring; TMA out-of-bounds fill gives the zero Dirichlet ghost in
//        x, y and z (the tensor map covers only the planes [zv0, zv1) that hold
//        data);
//      - the u- and m tiles (128 x 15 each) into a 4-stage ring (161 KiB of
//        shared memory in all, so a codec CTA fits next to it).
//    full/empty mbarrier pairs per stage: every consumer thread releases a
//    stage once its own loads from it have returned (no CTA-wide barrier per
//    plane; see "release discipline" below), so
//    the producer stays 3 u planes / 3 u-,m planes ahead.
//  * Persistent: one CTA per SM; work items (z chunk, tile) in chunk-major
//    order, CTA b takes items b, b + G, ...: all CTAs stay in the same z chunk
//    (halo rows hit in L2) and one continuous producer pipeline per CTA runs
//    across items (no relaunch, no per-item pipeline drain).
//  * Consumers: z-neighbours from a float4 register queue (values, not
//    partial sums, so the prescribed summation order is kept), advanced two
//    planes per iteration (fp32); x/y neighbours and u-, m from shared memory
//    with 128-bit loads; u+ with 128-bit stores.
//  * Arithmetic: DESIGN.md R5 order with __fadd_rn / __fmul_rn / __fmaf_rn, so
//    results are bit-identical to the fp32 oracle; in fp32 as packed pairs
//    (__fadd2_rn / __fmul2_rn / __ffma2_rn: per lane the same roundings).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include <mutex>

#include "common.cuh"

namespace oocz {
namespace {

#ifndef OOCZ_STENCIL_NU
#define OOCZ_STENCIL_NU 8
#endif
#ifndef OOCZ_STENCIL_NR
#define OOCZ_STENCIL_NR 4
#endif
#ifndef OOCZ_STENCIL_CTAS
#define OOCZ_STENCIL_CTAS 148
#endif
constexpr int kStencilCTAs = OOCZ_STENCIL_CTAS;  // persistent CTAs (one per SM at most)
constexpr int TX = 128;                           // 32 lanes x 4 consecutive x

// Tile shape per element type.  fp32: 128 x 15 cells, 15 consumer warps, ring
// depths NU / NR (measured on one C2 slab: 128 x 16 with rings 10 / 5, 17 warps,
// 111 us; 128 x 15 with rings 8 / 4, 16 warps, 106.5 us).  fp64 (the paper's precision): 128 x 8 cells,
// 8 consumer warps (the register queue is twice as wide; 288 threads leave
// 224 registers per thread), u ring 8, u-/m ring 4: 203 KiB of shared memory.
template <class T> struct Tile;
#ifndef OOCZ_STENCIL_TY
#define OOCZ_STENCIL_TY 15
#endif
#ifndef OOCZ_STENCIL_LB
#define OOCZ_STENCIL_LB 640
#endif
// LB: the thread count __launch_bounds__ is given (0: the real one).  A larger
// bound caps the registers (65536 / LB), e.g. 640 -> 96 with 16 warps, which
// leaves each SM sub-partition room for one codec warp next to the stencil.
template <> struct Tile<float> {
    static constexpr int TY = OOCZ_STENCIL_TY, NU = OOCZ_STENCIL_NU, NR = OOCZ_STENCIL_NR, LB = OOCZ_STENCIL_LB;
};
#ifndef OOCZ_STENCIL64_TY
#define OOCZ_STENCIL64_TY 8
#endif
#ifndef OOCZ_STENCIL64_NU
#define OOCZ_STENCIL64_NU 8
#endif
#ifndef OOCZ_STENCIL64_NR
#define OOCZ_STENCIL64_NR 4
#endif
template <> struct Tile<double> {
    static constexpr int TY = OOCZ_STENCIL64_TY, NU = OOCZ_STENCIL64_NU, NR = OOCZ_STENCIL64_NR, LB = 0;
};

template <class T> struct K {
    static constexpr int TY = Tile<T>::TY, NU = Tile<T>::NU, NR = Tile<T>::NR;
    static_assert(NU >= 6 && NR >= 2, "the u ring holds planes z..z+4 plus at least one in flight");
    static constexpr int SW = TX + 8, SH = TY + 8;            // u tile incl. halo
    // elements per u stage: the TMA box, padded to a 128 B multiple
    static constexpr int kUStage = (int)(((SW * SH * sizeof(T) + 127) / 128 * 128) / sizeof(T));
    static constexpr int kRStage = 2 * TX * TY;               // u- tile then m tile
    static constexpr int kConsumerWarps = TY;
    static constexpr int kThreads = 32 * (1 + kConsumerWarps);
    static constexpr int kBoundThreads = Tile<T>::LB ? Tile<T>::LB : kThreads;
    static constexpr unsigned kUBytes = kUStage * sizeof(T);          // stage stride
    static constexpr unsigned kUBoxBytes = SW * SH * sizeof(T);       // bytes one TMA box delivers
    static constexpr unsigned kRTileBytes = TX * TY * sizeof(T);
    static constexpr size_t kSmemBytes =
        (size_t)NU * kUBytes + (size_t)NR * 2 * kRTileBytes + 2 * (NU + NR) * sizeof(uint64_t);
    static_assert(kUBytes % 128 == 0 && kRTileBytes % 128 == 0, "TMA destinations stay 128 B aligned");
};

template <class T> struct Coeffs { T c0x3, c1, c2, c3, c4; };

// The 4 cells a lane owns, and how they are loaded / stored.
//   fp32: x = x0 + 4 lane + {0,1,2,3}: one 16-B access, a warp covers 512
//         contiguous bytes (4 shared-memory wavefronts, conflict-free).
//   fp64: x = x0 + 2 lane + {0,1} and x0 + 64 + 2 lane + {0,1}: two 16-B
//         accesses, each covering 512 contiguous bytes per warp.  (Four
//         consecutive doubles per lane would put 32-B strides on the banks:
//         twice the wavefronts; ncu measured the kernel shared-memory bound.)
template <class T> struct V4 { T v[4]; };
template <class T> struct Lanes;
template <> struct Lanes<float> {
    static constexpr int kLaneStride = 4;
};
template <> struct Lanes<double> {
    static constexpr int kLaneStride = 2;
};
__device__ __forceinline__ V4<float> ld4(const float* p) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    return V4<float>{{a.x, a.y, a.z, a.w}};
}
__device__ __forceinline__ V4<double> ld4(const double* p) {
    const double2 a = *reinterpret_cast<const double2*>(p), b = *reinterpret_cast<const double2*>(p + 64);
    return V4<double>{{a.x, a.y, b.x, b.y}};
}
// store the lane's 4 results; gx = x of its first cell (columns >= nx are not stored)
__device__ __forceinline__ void st4(float* p, const float r[4], int gx, int nx) {
    if (gx < nx) *reinterpret_cast<float4*>(p) = make_float4(r[0], r[1], r[2], r[3]);
}
__device__ __forceinline__ void st4(double* p, const double r[4], int gx, int nx) {
    if (gx < nx) *reinterpret_cast<double2*>(p) = make_double2(r[0], r[1]);
    if (gx + 64 < nx) *reinterpret_cast<double2*>(p + 64) = make_double2(r[2], r[3]);
}

// Packed fp32 (FADD2 / FMUL2 / FFMA2, sm_100): two lanes of one 64-bit register
// pair per instruction, each lane rounded exactly as __fadd_rn / __fmul_rn /
// __fmaf_rn, so results are bit-identical to the scalar forms.  The FMA pipe
// runs them at half the issue rate of the scalar forms (the same flops per
// cycle, tools/probe/ffma2_rate.cu), so they save issue slots, not pipe time.
#ifndef OOCZ_STENCIL_ZU
#define OOCZ_STENCIL_ZU 2
#endif
#ifndef OOCZ_STENCIL_F2
#define OOCZ_STENCIL_F2 1
#endif
__device__ __forceinline__ float2 lo2(const V4<float>& v) { return make_float2(v.v[0], v.v[1]); }
__device__ __forceinline__ float2 hi2(const V4<float>& v) { return make_float2(v.v[2], v.v[3]); }
__device__ __forceinline__ float2 half2of(const V4<float>& v, int p) { return p ? hi2(v) : lo2(v); }

__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
#if !OOCZ_STENCIL_F2   // the scalar fp32 forms (A/B builds only)
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
#endif
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }

// x-neighbour pairs ax[d-1][o] = u[x_o - d] + u[x_o + d] of the lane's cells;
// crow points at the lane's first cell in the u stage, uc holds its centres
#if !OOCZ_STENCIL_F2
__device__ __forceinline__ void x_pairs(const float* crow, const V4<float>& uc, float ax[4][4]) {
    const V4<float> xl = ld4(crow - 4), xr = ld4(crow + 4);
    const float w[12] = {xl.v[0], xl.v[1], xl.v[2], xl.v[3], uc.v[0], uc.v[1], uc.v[2], uc.v[3],
                         xr.v[0], xr.v[1], xr.v[2], xr.v[3]};
#pragma unroll
    for (int o = 0; o < 4; o++)
#pragma unroll
        for (int d = 1; d <= 4; d++) ax[d - 1][o] = add_rn(w[4 + o - d], w[4 + o + d]);
}
#endif
__device__ __forceinline__ void x_pairs(const double* crow, const V4<double>& uc, double ax[4][4]) {
#pragma unroll
    for (int g = 0; g < 2; g++) {                  // the two 2-cell groups, 64 apart
        const double* c = crow + 64 * g;
        const double2 a = *reinterpret_cast<const double2*>(c - 4), b = *reinterpret_cast<const double2*>(c - 2);
        const double2 e = *reinterpret_cast<const double2*>(c + 2), f = *reinterpret_cast<const double2*>(c + 4);
        const double w[10] = {a.x, a.y, b.x, b.y, uc.v[2 * g], uc.v[2 * g + 1], e.x, e.y, f.x, f.y};
#pragma unroll
        for (int o = 0; o < 2; o++)
#pragma unroll
            for (int d = 1; d <= 4; d++) ax[d - 1][2 * g + o] = add_rn(w[4 + o - d], w[4 + o + d]);
    }
}

// Ring-slot release discipline.  A shared-memory load (LDS) may still be in
// flight when a later mbarrier.arrive issues: ptxas does not wait for a load's
// scoreboard before SYNCS.ARRIVE unless the arrive depends on the loaded
// register, and the producer's next TMA write into the slot is not ordered
// after loads still in flight -- a write-after-read race, seen on B200 as rare
// wrong neighbours (first in fp64 on ragged tiles; later, with 8-deep rings,
// as wrong first planes of a segment on ragged tiles while a codec kernel ran
// concurrently: the prologue's loads were released with no instruction
// reading them -- an empty asm "use" emits no SASS).  So every release carries
// a real data dependency on one register of every load from the slot: the
// words are XORed into an accumulator (real instructions that wait for the
// loads), ANDed with a kernel-parameter zero that ptxas cannot fold, OR-reduced
// over the warp (REDUX reads every lane's value), and added to the barrier
// address of the single arrive.
__device__ __forceinline__ void dep_add(uint32_t& acc, float v) { acc ^= __float_as_uint(v); }
__device__ __forceinline__ void dep_add(uint32_t& acc, double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    acc ^= (uint32_t)b ^ (uint32_t)(b >> 32);
}
// one register of each 16-B load behind a V4 (fp32: one load; fp64: two)
template <class T> __device__ __forceinline__ void dep_add4(uint32_t& acc, const V4<T>& v) {
    dep_add(acc, v.v[0]);
    if (sizeof(T) == 8) dep_add(acc, v.v[2]);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// a consumer thread's release of a ring slot: every consumer thread arrives
// (the empty barriers count threads), at an address that depends on the
// thread's own loads from the slot (acc, see dep_add; zero is 0 at run time).
// Barriers are passed as shared-window addresses computed once per thread: the
// compiler does not hoist the generic-to-shared conversion across the asm's
// memory clobbers, so per-plane conversions cost instructions.
__device__ __forceinline__ void release_slot_s(uint32_t bar, uint32_t acc, uint32_t zero) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar + (acc & zero)) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// Work item `it` of the chunk-major enumeration (z chunk, tile): CTA b takes
// items b, b + G, b + 2G, ... so at any time all CTAs work in the same z chunk
// and a tile's radius-4 y/x halo rows are L2 hits from its neighbours' loads.
struct Seg { int x0, y0, zb, ze; };

template <int TY>
__device__ __forceinline__ bool next_seg(long& it, long items, long tiles, int ntx, int z0, int z1, int chunk,
                                         Seg& sg) {
    if (it >= items) return false;
    const long c = it / tiles, t = it - c * tiles;
    sg.x0 = (int)(t % ntx) * TX;
    sg.y0 = (int)(t / ntx) * TY;
    sg.zb = z0 + (int)c * chunk;
    sg.ze = min(sg.zb + chunk, z1);
    it += gridDim.x;
    return true;
}

template <class T>
__global__ void __launch_bounds__(K<T>::kBoundThreads, 1)
stencil25_kernel(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_up,
                 const __grid_constant__ CUtensorMap tm_m, T* __restrict__ uprev, int nx, int ny,
                 int z0, int z1, int chunk, int ntx, long tiles, int zv0, Coeffs<T> cf, uint32_t zero)
{
    constexpr int TY = K<T>::TY, NU = K<T>::NU, NR = K<T>::NR, SW = K<T>::SW;
    constexpr int kUStage = K<T>::kUStage, kRStage = K<T>::kRStage, kConsumerWarps = K<T>::kConsumerWarps;
    constexpr unsigned kUBoxBytes = K<T>::kUBoxBytes, kRTileBytes = K<T>::kRTileBytes;
    constexpr bool kPacked = sizeof(T) == 4 && OOCZ_STENCIL_F2;
    constexpr int kZU = sizeof(T) == 4 ? OOCZ_STENCIL_ZU : 1;   // planes per march iteration
    // dynamic smem only (no static shared variables before it), 1024-aligned, and
    // pointers derived from it directly so the compiler emits LDS, not generic LD
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    T* uring = reinterpret_cast<T*>(smem_raw);
    T* rring = uring + NU * kUStage;
    uint64_t* bars = reinterpret_cast<uint64_t*>(uring + NU * kUStage + NR * kRStage);
    uint64_t* ufull = bars;
    uint64_t* uempty = bars + NU;
    uint64_t* rfull = bars + 2 * NU;
    uint64_t* rempty = bars + 2 * NU + NR;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // persistent: items blockIdx.x, + gridDim.x, ... of (z chunk, tile)
    const long items = tiles * ((z1 - z0 + chunk - 1) / chunk);

    if (threadIdx.x == 0) {
        for (int s = 0; s < NU; s++) { mbar_init(&ufull[s], 1); mbar_init(&uempty[s], 32 * kConsumerWarps); }
        for (int s = 0; s < NR; s++) { mbar_init(&rfull[s], 1); mbar_init(&rempty[s], 32 * kConsumerWarps); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        // issues every segment's u planes [zb-4, ze+4) and u-/m planes [zb, ze)
        // in consumption order; ring slots and phases follow global counters
        // that run on across segments, so the pipeline never drains in between
        if (lane == 0) {
            long it = blockIdx.x;
            unsigned gu = 0, gr = 0;
            Seg sg;
            while (next_seg<TY>(it, items, tiles, ntx, z0, z1, chunk, sg)) {
                for (int p = sg.zb - 4; p < sg.ze + 4; p++, gu++) {
                    const int s = gu % NU;
                    if (gu >= NU) mbar_wait(&uempty[s], ((gu / NU) & 1) ^ 1);
                    mbar_expect_tx(&ufull[s], kUBoxBytes);
                    tma_load_3d(uring + s * kUStage, &tm_u, sg.x0 - 4, sg.y0 - 4, p - zv0, &ufull[s]);
                    const int z = p - 4;                   // u-, m of plane z go with u plane z+4
                    if (z >= sg.zb) {
                        const int r = gr % NR;
                        if (gr >= NR) mbar_wait(&rempty[r], ((gr / NR) & 1) ^ 1);
                        mbar_expect_tx(&rfull[r], 2 * kRTileBytes);
                        T* dst = rring + r * kRStage;
                        tma_load_3d(dst, &tm_up, sg.x0, sg.y0, z, &rfull[r]);
                        tma_load_3d(dst + TX * TY, &tm_m, sg.x0, sg.y0, z, &rfull[r]);
                        gr++;
                    }
                }
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int ty = warp - 1;
    const size_t plane = (size_t)nx * ny;
    constexpr int LS = Lanes<T>::kLaneStride;
    const int cidx = (ty + 4) * SW + 4 + LS * lane;  // this thread's (first) centre in a u stage
    const int ridx = ty * TX + LS * lane;            // ... in a u- / m tile
    const uint32_t ufull_s = smem_u32(ufull), uempty_s = smem_u32(uempty);
    const uint32_t rfull_s = smem_u32(rfull), rempty_s = smem_u32(rempty);
    long it = blockIdx.x;
    unsigned gu0 = 0, gr0 = 0;                       // global index of the segment's first u / u- plane
    Seg sg;
    while (next_seg<TY>(it, items, tiles, ntx, z0, z1, chunk, sg)) {
        const int zb = sg.zb, ze = sg.ze, pfirst = zb - 4;
        const int gx = sg.x0 + LS * lane, gy = sg.y0 + ty;
        const bool active = gy < ny;                 // (columns: checked per store)
        const size_t col = (size_t)gy * nx + gx;
        auto uslot = [&](int p) { return (gu0 + (unsigned)(p - pfirst)) % NU; };
        auto wait_u = [&](int p) -> const T* {
            const unsigned g = gu0 + (unsigned)(p - pfirst);
            mbar_wait_s(ufull_s + 8 * (g % NU), (g / NU) & 1);
            return uring + (g % NU) * kUStage;
        };
        auto release_u = [&](int p, uint32_t acc) { release_slot_s(uempty_s + 8 * uslot(p), acc, zero); };

        V4<T> q[8 + kZU];
        // centres of planes zb-4 .. zb+3; a plane outside [zb, ze) is released as soon
        // as its centre is read (its only use), so the ring never needs more than
        // 5 stages to get through this prologue
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int p = pfirst + i;
            q[i] = ld4(wait_u(p) + cidx);
            if (p < zb || p >= ze) {
                uint32_t acc = 0;
                dep_add4(acc, q[i]);
                release_u(p, acc);
            }
        }

        // one plane z of the march; qq[0..8] are the u centres of planes z-4 .. z+4
        auto plane_step = [&](const int z, const V4<T>* qq, T* outz) {
                const unsigned g = gr0 + (unsigned)(z - zb);
                const T* rt = rring + (g % NR) * kRStage;
                const T* crow = uring + uslot(z) * kUStage + cidx;  // plane z already landed
                T res[4];
                if constexpr (kPacked) {
                    // the same arithmetic on the lane's cell pairs (0, 1) and (2, 3)
                    float2 ay[4][2];
#pragma unroll
                    for (int d = 1; d <= 4; d++) {
                        const V4<T> a = ld4(crow - d * SW);
                        const V4<T> b = ld4(crow + d * SW);
                        ay[d - 1][0] = __fadd2_rn(lo2(a), lo2(b));
                        ay[d - 1][1] = __fadd2_rn(hi2(a), hi2(b));
                    }
                    const V4<T> uc = qq[4];
                    const V4<T> xl = ld4(crow - 4), xr = ld4(crow + 4);
                    const float w[12] = {xl.v[0], xl.v[1], xl.v[2], xl.v[3], uc.v[0], uc.v[1], uc.v[2], uc.v[3],
                                         xr.v[0], xr.v[1], xr.v[2], xr.v[3]};
                    // x pairs at even distance are aligned register pairs; at odd distance
                    // they straddle two pairs, so those are two scalar additions
                    float2 ax[4][2];
#pragma unroll
                    for (int p = 0; p < 2; p++)
#pragma unroll
                        for (int d = 1; d <= 4; d++) {
                            const int lo = 4 + 2 * p - d, hi = 4 + 2 * p + d;
                            ax[d - 1][p] = (d & 1) ? make_float2(__fadd_rn(w[lo], w[hi]), __fadd_rn(w[lo + 1], w[hi + 1]))
                                                   : __fadd2_rn(make_float2(w[lo], w[lo + 1]), make_float2(w[hi], w[hi + 1]));
                        }
                    // the release depends on every load from slot z (see the scalar path)
                    uint32_t acc = 0;
#pragma unroll
                    for (int d = 0; d < 4; d++) dep_add(acc, ay[d][0].x);
                    dep_add(acc, ax[3][0].x);
                    release_u(z, acc);
                    if (z + 4 >= ze) {
                        uint32_t acc8 = 0;
                        dep_add4(acc8, qq[8]);
                        release_u(z + 4, acc8);
                    }
                    const float2 c0x3 = make_float2(cf.c0x3, cf.c0x3), c1 = make_float2(cf.c1, cf.c1),
                                 c2 = make_float2(cf.c2, cf.c2), c3 = make_float2(cf.c3, cf.c3),
                                 c4 = make_float2(cf.c4, cf.c4);
                    float2 Lv[2];
#pragma unroll
                    for (int p = 0; p < 2; p++) {
                        float2 sd[4];
#pragma unroll
                        for (int d = 1; d <= 4; d++) {
                            const float2 az = __fadd2_rn(half2of(qq[4 - d], p), half2of(qq[4 + d], p));
                            sd[d - 1] = __fadd2_rn(__fadd2_rn(ax[d - 1][p], ay[d - 1][p]), az);
                        }
                        float2 L = __fmul2_rn(c0x3, half2of(uc, p));
                        L = __ffma2_rn(c1, sd[0], L);
                        L = __ffma2_rn(c2, sd[1], L);
                        L = __ffma2_rn(c3, sd[2], L);
                        L = __ffma2_rn(c4, sd[3], L);
                        Lv[p] = L;
                    }
                    mbar_wait_s(rfull_s + 8 * (g % NR), (g / NR) & 1);
                    const V4<T> upv = ld4(rt + ridx);
                    const V4<T> mv = ld4(rt + TX * TY + ridx);
#pragma unroll
                    for (int p = 0; p < 2; p++) {
                        const float2 up2 = half2of(upv, p);
                        const float2 r = __ffma2_rn(half2of(mv, p), Lv[p],
                                                    __ffma2_rn(make_float2(2.f, 2.f), half2of(uc, p),
                                                               make_float2(-up2.x, -up2.y)));
                        res[2 * p] = r.x;
                        res[2 * p + 1] = r.y;
                    }
                    uint32_t accr = 0;
                    dep_add4(accr, upv);
                    dep_add4(accr, mv);
                    release_slot_s(rempty_s + 8 * (g % NR), accr, zero);
                } else {
                    // y-neighbour pairs are summed as they arrive (ay[d][o] = u[y-d] + u[y+d]),
                    // which is the first addition of the prescribed order anyway
                    T ay[4][4];
#pragma unroll
                    for (int d = 1; d <= 4; d++) {
                        const V4<T> a = ld4(crow - d * SW);
                        const V4<T> b = ld4(crow + d * SW);
#pragma unroll
                        for (int o = 0; o < 4; o++) ay[d - 1][o] = add_rn(a.v[o], b.v[o]);
                    }
                    // x-neighbour pairs (the first addition of the prescribed order too)
                    const V4<T> uc = qq[4];
                    T ax[4][4];
                    x_pairs(crow, uc, ax);
                    // the release depends on every load from slot z through the pair sums:
                    // ay[d][0] reads both y loads of distance d and ax[3][0] = xl + xr both x
                    // loads; fp64 loads each 4-cell vector in two halves, 64 apart, so also
                    // ay[d][2], and its x pairs come from four loads per half (ax[3] and ax[1])
                    uint32_t acc = 0;
#pragma unroll
                    for (int d = 0; d < 4; d++) dep_add(acc, ay[d][0]);
                    dep_add(acc, ax[3][0]);
                    if (sizeof(T) == 8) {
#pragma unroll
                        for (int d = 0; d < 4; d++) dep_add(acc, ay[d][2]);
                        dep_add(acc, ax[1][0]);
                        dep_add(acc, ax[3][2]);
                        dep_add(acc, ax[1][2]);
                    }
                    release_u(z, acc);
                    if (z + 4 >= ze) {
                        uint32_t acc8 = 0;
                        dep_add4(acc8, qq[8]);
                        release_u(z + 4, acc8);
                    }

                    T Lv[4];
#pragma unroll
                    for (int o = 0; o < 4; o++) {
                        const T u0 = uc.v[o];
                        T sd[4];
#pragma unroll
                        for (int d = 1; d <= 4; d++) {
                            const T az = add_rn(qq[4 - d].v[o], qq[4 + d].v[o]);
                            sd[d - 1] = add_rn(add_rn(ax[d - 1][o], ay[d - 1][o]), az);
                        }
                        T L = mul_rn(cf.c0x3, u0);
                        L = fma_rn(cf.c1, sd[0], L);
                        L = fma_rn(cf.c2, sd[1], L);
                        L = fma_rn(cf.c3, sd[2], L);
                        L = fma_rn(cf.c4, sd[3], L);
                        Lv[o] = L;
                    }
                    // u- and m are read only now, when they are needed
                    mbar_wait_s(rfull_s + 8 * (g % NR), (g / NR) & 1);
                    const V4<T> upv = ld4(rt + ridx);
                    const V4<T> mv = ld4(rt + TX * TY + ridx);
#pragma unroll
                    for (int o = 0; o < 4; o++) res[o] = fma_rn(mv.v[o], Lv[o], fma_rn((T)2, uc.v[o], -upv.v[o]));
                    {
                        uint32_t accr = 0;
                        dep_add4(accr, upv);
                        dep_add4(accr, mv);
                        release_slot_s(rempty_s + 8 * (g % NR), accr, zero);
                    }
                }
                if (active) st4(outz, res, gx, nx);
        };
        T* outz = uprev + (size_t)zb * plane + col;   // u+ of plane z (advanced per plane)
        for (int z = zb; z < ze; z += kZU, outz += kZU * plane) {
#pragma unroll
            for (int j = 0; j < kZU; j++) {
                if (z + j < ze) {
                    q[8 + j] = ld4(wait_u(z + j + 4) + cidx);
                    plane_step(z + j, q + j, outz + j * plane);
                }
            }
            // shift the queue by kZU planes (kZU = 2 halves the moves per plane; an
            // unroll by 9 to rotate by renaming measured slower: 9x the code,
            // instruction-cache and register pressure)
#pragma unroll
            for (int i = 0; i < 8; i++) q[i] = q[i + kZU];
        }
        gu0 += (unsigned)(ze - zb + 8);
        gr0 += (unsigned)(ze - zb);
    }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

template <class T>
bool make_map(CUtensorMap* map, const T* base, int nx, int ny, int nplanes, int bx, int by) {
    auto encode = get_encode_fn();
    if (!encode) return false;
    const cuuint64_t gdim[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nplanes};
    const cuuint64_t gstride[2] = {(cuuint64_t)nx * sizeof(T), (cuuint64_t)nx * ny * sizeof(T)};
    const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    const cuuint32_t estride[3] = {1, 1, 1};
    const CUtensorMapDataType dt = sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    return encode(map, dt, 3, const_cast<T*>(base), gdim, gstride, box,
                  estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <class T>
cudaError_t launch_stencil_step_t(const T* u, T* uprev, const T* m, int nx, int ny, int nz,
                                  const T c[5], int z0, int z1, int zv0, int zv1, cudaStream_t s)
{
    using KT = K<T>;
    if (nx <= 0 || ny <= 0 || nx % 4 || z0 < 0 || z1 > nz || zv0 < 0 || zv1 > nz || zv0 >= zv1)
        return cudaErrorInvalidValue;
    if (z1 <= z0) return cudaSuccess;
    CUtensorMap mu, mup, mm;
    if (!make_map(&mu, u + (size_t)zv0 * nx * ny, nx, ny, zv1 - zv0, KT::SW, KT::SH) ||
        !make_map(&mup, (const T*)uprev, nx, ny, nz, TX, KT::TY) || !make_map(&mm, m, nx, ny, nz, TX, KT::TY))
        return cudaErrorInvalidValue;
    static std::atomic<uint64_t> attr_done{0};
    {
        cudaError_t e = kernel_smem_setup((const void*)stencil25_kernel<T>, (int)KT::kSmemBytes, attr_done);
        if (e != cudaSuccess) return e;
    }
    Coeffs<T> cf{(T)3 * c[0], c[1], c[2], c[3], c[4]};  // fl(3 c0) in T, as the oracle
    // persistent CTAs.  If the plane's tiles fit on the SMs, one CTA per tile
    // marches the whole z range (no chunk prologues; the SMs left over run the
    // decode stream's kernels concurrently).  Otherwise kStencilCTAs CTAs and the
    // chunk count minimising the busiest CTA's load ceil(items / G) x (chunk + 8)
    // (a chunk re-reads 8 halo planes and refills its pipeline).  Measured on
    // 512^2 (128 tiles): 128 CTAs x 1 chunk 108.6 us vs 148 CTAs x 8 chunks 114.7 us.
    const int ntx = (nx + TX - 1) / TX;
    const long tiles = (long)ntx * ((ny + KT::TY - 1) / KT::TY);
    const int nzu = z1 - z0;
    int chunk = nzu;
    if (tiles > kStencilCTAs) {
        double best = 1e300;
        for (int nch = 1; nch <= std::max(1, nzu / 8); nch++) {
            const int c = (nzu + nch - 1) / nch;
            const long items = tiles * ((nzu + c - 1) / c);
            const long per = (items + kStencilCTAs - 1) / kStencilCTAs;
            const double cost = (double)per * (c + 8.0);
            if (cost < best - 1e-9) { best = cost; chunk = c; }
        }
    }
    const long items = tiles * ((nzu + chunk - 1) / chunk);
    const int grid = (int)std::min<long>(kStencilCTAs, items);
    stencil25_kernel<T><<<grid, KT::kThreads, KT::kSmemBytes, s>>>(mu, mup, mm, uprev, nx, ny, z0, z1, chunk, ntx,
                                                                   tiles, zv0, cf, 0u);
    note_launches(1);
    return cudaGetLastError();
}

template <class T>
oocz_status stencil_steps_t(T* d_u, T* d_uprev, const T* d_m, int nx, int ny, int nz, const T c[5], int nsteps,
                            cudaStream_t s)
{
    T* a = d_u;
    T* b = d_uprev;
    for (int k = 0; k < nsteps; k++) {
        cudaError_t e = launch_stencil_step_t<T>(a, b, d_m, nx, ny, nz, c, 0, nz, 0, nz, s);
        if (e != cudaSuccess) return stateless_status(e, "oocz_stencil_steps");
        T* t = a; a = b; b = t;  // newest level now in a
    }
    if (a != d_u) {  // odd count: move the levels back into the caller's roles
        const size_t bytes = (size_t)nx * ny * nz * sizeof(T);
        void* tmp = nullptr;
        cudaError_t e = cudaMallocAsync(&tmp, bytes, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(tmp, d_u, bytes, cudaMemcpyDeviceToDevice, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(d_u, d_uprev, bytes, cudaMemcpyDeviceToDevice, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(d_uprev, tmp, bytes, cudaMemcpyDeviceToDevice, s);
        if (e == cudaSuccess) e = cudaFreeAsync(tmp, s);
        if (e != cudaSuccess) return stateless_status(e, "oocz_stencil_steps");
    }
    return OOCZ_OK;
}

}  // namespace

cudaError_t launch_stencil_step(const float* u, float* uprev, const float* m, int nx, int ny, int nz,
                                const float c[5], int z0, int z1, int zv0, int zv1, cudaStream_t s)
{
    return launch_stencil_step_t<float>(u, uprev, m, nx, ny, nz, c, z0, z1, zv0, zv1, s);
}

cudaError_t launch_stencil_step(const double* u, double* uprev, const double* m, int nx, int ny, int nz,
                                const double c[5], int z0, int z1, int zv0, int zv1, cudaStream_t s)
{
    return launch_stencil_step_t<double>(u, uprev, m, nx, ny, nz, c, z0, z1, zv0, zv1, s);
}

}  // namespace oocz

// ------------------------------------------------------------------ C ABI
namespace {
template <class T>
oocz_status step_planes_abi(const T* d_u, T* d_uprev, const T* d_m, int32_t nx, int32_t ny, int32_t nz,
                            const T c[5], int32_t z0, int32_t z1, int32_t zv0, int32_t zv1, void* stream,
                            const char* fn)
{
    if (nx % 4) return OOCZ_EALIGN;
    if (!d_u || !d_uprev || !d_m || !c || nx <= 0 || ny <= 0 || nz <= 0 || z0 < 0 || z1 > nz ||
        zv0 < 0 || zv1 > nz || zv0 >= zv1)
        return OOCZ_EINVAL;
    cudaError_t e = oocz::launch_stencil_step(d_u, d_uprev, d_m, nx, ny, nz, c, z0, z1, zv0, zv1,
                                              (cudaStream_t)stream);
    return oocz::stateless_status(e, fn);
}
}  // namespace

extern "C" oocz_status oocz_stencil_step_planes(const float* d_u, float* d_uprev, const float* d_m,
                                                int32_t nx, int32_t ny, int32_t nz, const float c[5],
                                                int32_t z0, int32_t z1, int32_t zv0, int32_t zv1,
                                                void* stream)
{
    return step_planes_abi(d_u, d_uprev, d_m, nx, ny, nz, c, z0, z1, zv0, zv1, stream, __func__);
}

extern "C" oocz_status oocz_stencil_step_planes_f64(const double* d_u, double* d_uprev, const double* d_m,
                                                    int32_t nx, int32_t ny, int32_t nz, const double c[5],
                                                    int32_t z0, int32_t z1, int32_t zv0, int32_t zv1,
                                                    void* stream)
{
    return step_planes_abi(d_u, d_uprev, d_m, nx, ny, nz, c, z0, z1, zv0, zv1, stream, __func__);
}

extern "C" oocz_status oocz_stencil_steps(float* d_u, float* d_uprev, const float* d_m, int32_t nx,
                                          int32_t ny, int32_t nz, const float c[5], int32_t nsteps,
                                          void* stream)
{
    if (nx % 4) return OOCZ_EALIGN;
    if (!d_u || !d_uprev || !d_m || !c || nx <= 0 || ny <= 0 || nz <= 0 || nsteps < 0) return OOCZ_EINVAL;
    return oocz::stencil_steps_t<float>(d_u, d_uprev, d_m, nx, ny, nz, c, nsteps, (cudaStream_t)stream);
}

extern "C" oocz_status oocz_stencil_steps_f64(double* d_u, double* d_uprev, const double* d_m, int32_t nx,
                                              int32_t ny, int32_t nz, const double c[5], int32_t nsteps,
                                              void* stream)
{
    if (nx % 4) return OOCZ_EALIGN;
    if (!d_u || !d_uprev || !d_m || !c || nx <= 0 || ny <= 0 || nz <= 0 || nsteps < 0) return OOCZ_EINVAL;
    return oocz::stencil_steps_t<double>(d_u, d_uprev, d_m, nx, ny, nz, c, nsteps, (cudaStream_t)stream);
}
