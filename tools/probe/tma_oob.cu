// Probe: does a cp.async.bulk.tensor.3d load whose box is partly out of bounds
// zero-fill the out-of-bounds elements (fp64 and fp32), every time?
// Each CTA pre-fills its smem with a sentinel, issues one box load, waits on an
// mbarrier, and dumps smem; the host checks in-bound = source, OOB = 0.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <class T>
__global__ void probe(const __grid_constant__ CUtensorMap map, int bx, int by, int ny, int ntiles_y, T* out, int reps)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    T* buf = reinterpret_cast<T*>(sm);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + ((bx * by * sizeof(T) + 127) / 128) * 128);
    const int tile = blockIdx.x % ntiles_y;
    const int z = blockIdx.x / ntiles_y;
    const int y0 = tile * (by - 8);
    for (int r = 0; r < reps; r++) {
        for (int i = threadIdx.x; i < bx * by; i += blockDim.x) buf[i] = (T)-12345.0;
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bar)) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)),
                         "r"((unsigned)(bx * by * sizeof(T))) : "memory");
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(sa(buf)), "l"(reinterpret_cast<uint64_t>(&map)),
                         "r"(-4), "r"(y0 - 4), "r"(z), "r"(sa(bar)) : "memory");
        }
        asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}"
                     ::"r"(sa(bar)) : "memory");
        // count mismatches against the expected box
        for (int i = threadIdx.x; i < bx * by; i += blockDim.x) {
            const int x = i % bx - 4, y = i / bx + y0 - 4;
            const bool in = x >= 0 && x < bx - 8 && y >= 0 && y < ny;
            const T want = in ? (T)(z * 100000 + y * 1000 + x) : (T)0;
            if (buf[i] != want) atomicAdd(reinterpret_cast<unsigned long long*>(out), 1ull);
        }
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(sa(bar)) : "memory");
        __syncthreads();
    }
}

template <class T>
int run(int nx, int ny, int nz, int by, int reps, const char* name)
{
    std::vector<T> h((size_t)nx * ny * nz);
    for (int z = 0; z < nz; z++)
        for (int y = 0; y < ny; y++)
            for (int x = 0; x < nx; x++) h[((size_t)z * ny + y) * nx + x] = (T)(z * 100000 + y * 1000 + x);
    T* d;
    cudaMalloc(&d, h.size() * sizeof(T));
    cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    CUtensorMap map;
    const int bx = nx + 8;
    cuuint64_t gdim[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
    cuuint64_t gstr[2] = {(cuuint64_t)nx * sizeof(T), (cuuint64_t)nx * ny * sizeof(T)};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d,
                     gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("%s: encode failed %d\n", name, (int)r); return 1; }
    unsigned long long* bad;
    cudaMalloc(&bad, 8);
    cudaMemset(bad, 0, 8);
    const int ntiles_y = (ny + (by - 8) - 1) / (by - 8);
    const size_t smem = ((bx * by * sizeof(T) + 127) / 128) * 128 + 64;
    cudaFuncSetAttribute(probe<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<T><<<ntiles_y * nz, 256, smem>>>(map, bx, by, ny, ntiles_y, reinterpret_cast<T*>(bad), reps);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long nb = 0;
    cudaMemcpy(&nb, bad, 8, cudaMemcpyDeviceToHost);
    printf("%-6s nx=%d ny=%d by=%d box_bytes=%zu tiles=%d reps=%d: mismatches %llu (%s)\n", name, nx, ny, by,
           bx * by * sizeof(T), ntiles_y * nz, reps, nb, cudaGetErrorString(e));
    cudaFree(d);
    cudaFree(bad);
    return 0;
}

int main()
{
    for (int ny : {10, 12, 20})
        for (int by : {12, 16, 24}) {
            run<double>(128, ny, 64, by, 200, "fp64");
            run<float>(128, ny, 64, by, 200, "fp32");
        }
    run<double>(248, 10, 64, 16, 200, "fp64");
    run<double>(64, 10, 64, 16, 200, "fp64");
    return 0;
}
