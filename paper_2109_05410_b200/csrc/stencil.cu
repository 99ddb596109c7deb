// stencil.cu -- 25-point (radius-4) leapfrog step for sm_100a.
//
// The acoustic propagator of PAPER.md:208 (Sec. VI): two read-write time
// levels, a read-only model m, and a "write-only dataset" for intermediates,
// which here is fused away into registers.  HALO = 4.  One
// launch is one cone-limited step of temporal blocking:
// it updates planes [z0, z1) of a z-slab in place (u+ overwrites u-).
//
// Design (HBM-bound: >= 16 B per cell-update: read u, u-, m, write u+):
//  * CTA tile 128 (x) x 8 (y) cells, 256 threads, each thread 4 consecutive x.
//  * The u plane tile with its radius-4 x/y halo (136 x 16 floats) arrives by
//    TMA (cp.async.bulk.tensor.3d) into an 8-stage shared-memory ring guarded
//    by mbarriers; planes are prefetched 3 ahead.  TMA out-of-bounds fill gives
//    the zero Dirichlet ghost in x, y and z for free: the tensor map covers only
//    the planes [zv0, zv1) that hold data.
//  * z-neighbours come from a 9-deep register queue of float4 (values, not
//    partial sums, so the prescribed summation order is kept); x/y neighbours
//    are 128-bit shared-memory loads.
//  * u- and m are streamed with 128-bit loads one plane ahead; u+ is stored
//    with 128-bit stores.
//  * Each CTA marches a 32-plane z chunk (8 halo planes of extra TMA traffic,
//    mostly L2 hits) so that a 512^2 x 160 slab gives ~1300 CTAs.
//  * Arithmetic: DESIGN.md R5 order with __fadd_rn / __fmul_rn / __fmaf_rn, so
//    results are bit-identical to the fp32 oracle.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <mutex>

#include "common.cuh"

namespace oocz {
namespace {

constexpr int TX = 128, TY = 8;
constexpr int SW = TX + 8, SH = TY + 8;         // smem tile incl. halo
constexpr int kStageFloats = SW * SH;          // 2176 floats = 8704 B (128 B multiple)
constexpr int NS = 8;                          // ring stages
constexpr int ZCHUNK = 32;
constexpr int kThreads = 32 * TY;
constexpr unsigned kStageBytes = kStageFloats * sizeof(float);
constexpr size_t kSmemBytes = (size_t)NS * kStageBytes + 128;

struct Coeffs { float c0x3, c1, c2, c3, c4; };

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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(float* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

__global__ void __launch_bounds__(kThreads, 2)
stencil25_kernel(const __grid_constant__ CUtensorMap tm_u, float* __restrict__ uprev,
                 const float* __restrict__ m, int nx, int ny, int z0, int z1, int zv0, Coeffs cf)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* ring = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    __shared__ __align__(8) uint64_t full[NS];

    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int zb = z0 + blockIdx.z * ZCHUNK;
    const int ze = min(zb + ZCHUNK, z1);
    const int pfirst = zb - 4, plast = ze + 4;  // u planes needed: [pfirst, plast)
    const bool leader = threadIdx.x == 0;

    if (leader) {
        for (int s = 0; s < NS; s++) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto issue = [&](int p) {  // leader only
        const int s = (p - pfirst) % NS;
        mbar_expect_tx(&full[s], kStageBytes);
        tma_load_3d(ring + s * kStageFloats, &tm_u, x0 - 4, y0 - 4, p - zv0, &full[s]);
    };
    auto wait_plane = [&](int p) -> const float* {
        const int s = (p - pfirst) % NS;
        mbar_wait(&full[s], (uint32_t)(((p - pfirst) / NS) & 1));
        return ring + s * kStageFloats;
    };

    if (leader)
        for (int p = pfirst; p < min(pfirst + NS, plast); p++) issue(p);

    const int gx = x0 + 4 * tx, gy = y0 + ty;
    const bool active = gx < nx && gy < ny;
    const size_t plane = (size_t)nx * ny;
    const size_t col = (size_t)gy * nx + gx;
    const int cidx = (ty + 4) * SW + 4 + 4 * tx;  // this thread's centre in a stage

    // register queue: planes z-4 .. z+4
    float4 q[9];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const float* st = wait_plane(pfirst + i);
        q[i] = *reinterpret_cast<const float4*>(st + cidx);
    }
    __syncthreads();  // halo stages (planes zb-4 .. zb-1) are free again
    if (leader) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int p = pfirst + NS; p < min(pfirst + NS + 4, plast); p++) issue(p);
    }

    float4 up_n = make_float4(0.f, 0.f, 0.f, 0.f), m_n = up_n;
    if (active && zb < ze) {
        up_n = *reinterpret_cast<const float4*>(uprev + (size_t)zb * plane + col);
        m_n = __ldg(reinterpret_cast<const float4*>(m + (size_t)zb * plane + col));
    }

    for (int z = zb; z < ze; z++) {
        const float4 upv = up_n, mv = m_n;
        if (active && z + 1 < ze) {  // stream u-, m one plane ahead
            up_n = *reinterpret_cast<const float4*>(uprev + (size_t)(z + 1) * plane + col);
            m_n = __ldg(reinterpret_cast<const float4*>(m + (size_t)(z + 1) * plane + col));
        }
        {
            const float* st4 = wait_plane(z + 4);
            q[8] = *reinterpret_cast<const float4*>(st4 + cidx);
        }
        const float* st = wait_plane(z);
        const float* crow = st + cidx;
        const float4 xl = *reinterpret_cast<const float4*>(crow - 4);
        const float4 xr = *reinterpret_cast<const float4*>(crow + 4);
        float4 ym[4], yp[4];
#pragma unroll
        for (int d = 1; d <= 4; d++) {
            ym[d - 1] = *reinterpret_cast<const float4*>(crow - d * SW);
            yp[d - 1] = *reinterpret_cast<const float4*>(crow + d * SW);
        }
        const float4 uc = q[4];
        const float w[12] = {xl.x, xl.y, xl.z, xl.w, uc.x, uc.y, uc.z, uc.w, xr.x, xr.y, xr.z, xr.w};
        const float ucv[4] = {uc.x, uc.y, uc.z, uc.w};
        const float upa[4] = {upv.x, upv.y, upv.z, upv.w};
        const float ma[4] = {mv.x, mv.y, mv.z, mv.w};
        float res[4];
#pragma unroll
        for (int o = 0; o < 4; o++) {
            const float u0 = ucv[o];
            float s[4];
#pragma unroll
            for (int d = 1; d <= 4; d++) {
                const float* ymd = reinterpret_cast<const float*>(&ym[d - 1]);
                const float* ypd = reinterpret_cast<const float*>(&yp[d - 1]);
                const float* zmd = reinterpret_cast<const float*>(&q[4 - d]);
                const float* zpd = reinterpret_cast<const float*>(&q[4 + d]);
                const float ax = __fadd_rn(w[4 + o - d], w[4 + o + d]);
                const float ay = __fadd_rn(ymd[o], ypd[o]);
                const float az = __fadd_rn(zmd[o], zpd[o]);
                s[d - 1] = __fadd_rn(__fadd_rn(ax, ay), az);
            }
            float L = __fmul_rn(cf.c0x3, u0);
            L = __fmaf_rn(cf.c1, s[0], L);
            L = __fmaf_rn(cf.c2, s[1], L);
            L = __fmaf_rn(cf.c3, s[2], L);
            L = __fmaf_rn(cf.c4, s[3], L);
            res[o] = __fmaf_rn(ma[o], L, __fmaf_rn(2.0f, u0, -upa[o]));
        }
        if (active)
            *reinterpret_cast<float4*>(uprev + (size_t)z * plane + col) = make_float4(res[0], res[1], res[2], res[3]);
#pragma unroll
        for (int i = 0; i < 8; i++) q[i] = q[i + 1];
        __syncthreads();  // stage of plane z is free
        if (leader && z + NS < plast) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(z + NS);
        }
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

}  // namespace

cudaError_t launch_stencil_step(const float* u, float* uprev, const float* m, int nx, int ny, int nz,
                                const float c[5], int z0, int z1, int zv0, int zv1, cudaStream_t s)
{
    if (nx <= 0 || ny <= 0 || nx % 4 || z0 < 0 || z1 > nz || zv0 < 0 || zv1 > nz || zv0 >= zv1)
        return cudaErrorInvalidValue;
    if (z1 <= z0) return cudaSuccess;
    auto encode = get_encode_fn();
    if (!encode) return cudaErrorNotSupported;
    CUtensorMap map;
    const cuuint64_t gdim[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)(zv1 - zv0)};
    const cuuint64_t gstride[2] = {(cuuint64_t)nx * sizeof(float), (cuuint64_t)nx * ny * sizeof(float)};
    const cuuint32_t box[3] = {SW, SH, 1};
    const cuuint32_t estride[3] = {1, 1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                        const_cast<float*>(u) + (size_t)zv0 * nx * ny, gdim, gstride, box, estride,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(stencil25_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kSmemBytes);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    Coeffs cf{3.0f * c[0], c[1], c[2], c[3], c[4]};  // fl32(3 c0), as the oracle
    dim3 grid((nx + TX - 1) / TX, (ny + TY - 1) / TY, (z1 - z0 + ZCHUNK - 1) / ZCHUNK);
    stencil25_kernel<<<grid, kThreads, kSmemBytes, s>>>(map, uprev, m, nx, ny, z0, z1, zv0, cf);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace oocz

// ------------------------------------------------------------------ C ABI
extern "C" oocz_status oocz_stencil_step_planes(const float* d_u, float* d_uprev, const float* d_m,
                                                int32_t nx, int32_t ny, int32_t nz, const float c[5],
                                                int32_t z0, int32_t z1, int32_t zv0, int32_t zv1,
                                                void* stream)
{
    if (nx % 4) return OOCZ_EALIGN;
    if (!d_u || !d_uprev || !d_m || !c || nx <= 0 || ny <= 0 || nz <= 0 || z0 < 0 || z1 > nz ||
        zv0 < 0 || zv1 > nz || zv0 >= zv1)
        return OOCZ_EINVAL;
    cudaError_t e = oocz::launch_stencil_step(d_u, d_uprev, d_m, nx, ny, nz, c, z0, z1, zv0, zv1,
                                              (cudaStream_t)stream);
    return e == cudaSuccess ? OOCZ_OK : OOCZ_ECUDA;
}

extern "C" oocz_status oocz_stencil_steps(float* d_u, float* d_uprev, const float* d_m, int32_t nx,
                                          int32_t ny, int32_t nz, const float c[5], int32_t nsteps,
                                          void* stream)
{
    if (nx % 4) return OOCZ_EALIGN;
    if (!d_u || !d_uprev || !d_m || !c || nx <= 0 || ny <= 0 || nz <= 0 || nsteps < 0) return OOCZ_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    float* a = d_u;
    float* b = d_uprev;
    for (int k = 0; k < nsteps; k++) {
        cudaError_t e = oocz::launch_stencil_step(a, b, d_m, nx, ny, nz, c, 0, nz, 0, nz, s);
        if (e != cudaSuccess) return OOCZ_ECUDA;
        float* t = a; a = b; b = t;  // newest level now in a
    }
    if (a != d_u) {  // odd count: move the levels back into the caller's roles
        const size_t bytes = (size_t)nx * ny * nz * sizeof(float);
        void* tmp = nullptr;
        if (cudaMallocAsync(&tmp, bytes, s) != cudaSuccess) return OOCZ_ECUDA;
        if (cudaMemcpyAsync(tmp, d_u, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
            cudaMemcpyAsync(d_u, d_uprev, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
            cudaMemcpyAsync(d_uprev, tmp, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
            cudaFreeAsync(tmp, s) != cudaSuccess)
            return OOCZ_ECUDA;
    }
    return OOCZ_OK;
}
