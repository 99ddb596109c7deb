// common.cuh -- shared plumbing of liboocz.so (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstddef>
#include <atomic>

#include "../../include/oocz.h"

#if defined(__CUDACC__)
#define OOCZ_HD __host__ __device__ __forceinline__
#else
#define OOCZ_HD inline
#endif

namespace oocz {

// count of this library's kernel launches (oocz_kernel_launch_count)
void note_launches(uint64_t n);
// record a failure of a stateless call (oocz_last_error(NULL)); returns s
oocz_status stateless_status(cudaError_t e, const char* what);

// launch-configuration helpers
constexpr int kNumSMs = 148;  // B200

inline const char* cuda_str(cudaError_t e) { return cudaGetErrorString(e); }

#ifndef OOCZ_CARVEOUT
#define OOCZ_CARVEOUT 1
#endif
// Once per kernel: allow `dyn_bytes` of dynamic shared memory, and (unless
// built with OOCZ_CARVEOUT=0) ask for the largest shared-memory carveout, so
// an SM configured for one of the pipeline's kernels can take another's CTA.
// Function attributes belong to a device's context: `done` holds one bit per
// device already configured (setting them twice is harmless, so concurrent
// first calls need no lock).
inline cudaError_t kernel_smem_setup(const void* fn, int dyn_bytes, std::atomic<uint64_t>& done)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_bytes);
    if (e == cudaSuccess && OOCZ_CARVEOUT)
        e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

// internal launchers (stream-ordered, no synchronisation)
cudaError_t launch_zfp_encode(const float* in, int nx, int ny, int nz, int rate,
                              uint64_t* out, cudaStream_t s);
cudaError_t launch_zfp_decode(const uint64_t* in, int nx, int ny, int nz, int rate,
                              float* out, cudaStream_t s);
cudaError_t launch_zfp_encode64(const double* in, int nx, int ny, int nz, int rate,
                                uint64_t* out, cudaStream_t s);
cudaError_t launch_zfp_decode64(const uint64_t* in, int nx, int ny, int nz, int rate,
                                double* out, cudaStream_t s);
// nplanes of an nx*ny field of element size esz (4: fp32, 8: fp64): fixed-rate
// encode / decode, or a raw device copy for rate 0
cudaError_t field_encode(const void* src, int esz, int nx, int ny, int nplanes, int rate, void* dst,
                         cudaStream_t s);
cudaError_t field_decode(const void* src, int esz, int nx, int ny, int nplanes, int rate, void* dst,
                         cudaStream_t s);
// one cone-limited step: planes [z0, z1) of uprev <- u+; u planes outside
// [zv0, zv1) read as zero
cudaError_t launch_stencil_step(const float* u, float* uprev, const float* m,
                                int nx, int ny, int nz, const float c[5],
                                int z0, int z1, int zv0, int zv1, cudaStream_t s);
cudaError_t launch_stencil_step(const double* u, double* uprev, const double* m,
                                int nx, int ny, int nz, const double c[5],
                                int z0, int z1, int zv0, int zv1, cudaStream_t s);
// checks used by set_field: flags[0] |= non-finite seen; flags[1] = max(bits of m) (m >= 0)
cudaError_t launch_scan_field(const float* in, size_t n, unsigned int* flags, cudaStream_t s);
// fp64: flags[0] as above; *mx64 = max(bits of |x|) as a 64-bit word
cudaError_t launch_scan_field(const double* in, size_t n, unsigned int* flags, unsigned long long* mx64,
                              cudaStream_t s);

}  // namespace oocz
