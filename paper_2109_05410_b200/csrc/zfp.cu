// zfp.cu -- fixed-rate ZFP-style encode / decode kernels for fp32 3-D fields (sm_100a).
//
// PAPER.md:120-125 (Sec. IV): a fixed-rate codec, so compressed sizes are known
// in advance and device buffers are pre-allocated; PAPER.md:155-160 (Fig. 4):
// blocks are decompressed on arrival and compressed before leaving the GPU.
// Format: zfp 0.5.5 fixed-rate layout; per-block logic in
// zfp_block.cuh.
//
// Kernel shape: one thread per 4^3 block (NB = 1 block per thread; NB = 2,
// two interleaved event streams per thread, measured slower on B200: the
// doubled shared memory halves occupancy).  Block b of the CTA's range is
// owned by thread b % 128: consecutive threads own consecutive bx, so the
// float4 row loads / stores of a warp are coalesced.  The 32
// bit-plane words of each block live in shared memory in a [plane][thread]
// layout (conflict-free).  The decoder stages its compressed words through
// shared memory (coalesced loads); the encoder writes its words directly (the
// warp's 32 streams are adjacent, so L2 merges the partial-sector writes).
#include "common.cuh"
#include "zfp_block.cuh"

namespace oocz {
namespace {

constexpr int kThreads = 128;
constexpr int NB = 1;                       // blocks (event streams) per thread
#ifndef OOCZ_ENC_THREADS
#define OOCZ_ENC_THREADS 128
#endif
constexpr int kEncThreads = OOCZ_ENC_THREADS;       // fp32 encoder CTA size
#ifndef OOCZ_DEC_THREADS
#define OOCZ_DEC_THREADS 128
#endif
constexpr int kDecThreads = OOCZ_DEC_THREADS;       // fp32 decoder CTA size

struct BlockPos { long long bx, by, bz; };

#ifdef OOCZ_DEC_NOSTORE
// A/B bound only (tools/fusion_bound.sh): the decoder skips its slab stores once
// a context has made OOCZ_DEC_NOSTORE_AFTER decode launches (default 40: the
// warm-up sweeps), so the slabs hold real data from earlier blocks and the
// stencil and encoder see realistic values (with stores skipped from the first
// launch the slabs stay zero and the encoder codes all-zero blocks -- the
// round-2 bound measured that, not the stores)
__device__ int g_dec_skip_store;
std::atomic<int> g_dec_launches{0};
#endif

// Prefetch of the input of the CTA one resident wave ahead into L2 (one bulk
// prefetch of its contiguous words): the decoder is not persistent, and each
// CTA used to start with its input loads exposed (ncu: ~14 % of its stall
// samples).  Measured: decode 149.5 -> 147.5 us at rate 16, 188 -> 178 us at
// 24.  (The encoder's row-segment prefetch measured slower, 143 -> 148 us.)
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}

// the decoder's slab stores / the encoder's slab loads (streaming cache hints
// measured no different on the pipelined device path: DESIGN.md section 13)
__device__ __forceinline__ void st_slab(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float4 ld_slab(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }


// Coalesced stage-in of a CTA's contiguous stream words into shared memory,
// block by block with a row stride of S words: word w goes to words[(w / rate)
// S + w % rate].  Then each row's words [rate, S) are zeroed: the padded
// decoder reads up to 3 words past the stream.
// The quotient and remainder advance with w instead of being recomputed (an
// integer division per word was 7.5 % of the decoder's instructions).
template <int NT>
__device__ __forceinline__ void stage_words(uint64_t* words, const uint64_t* __restrict__ src, int total, int rate,
                                            int S)
{
    const int t = threadIdx.x;
    const int dq = NT / rate, dr = NT - dq * rate;
    int q = t / rate, r = t - q * rate;
#pragma unroll 4
    for (int w = t; w < total; w += NT) {
        words[q * S + r] = __ldg(src + w);
        q += dq;
        r += dr;
        if (r >= rate) { r -= rate; q++; }
    }
    for (int w = rate; w < S; w++) words[t * S + w] = 0ull;
}
// decoder row stride: the stream, 3 zero words, odd (bank spread)
__host__ __device__ __forceinline__ int dec_row_stride(int rate) { return (rate + 3) | 1; }

__device__ __forceinline__ BlockPos block_pos(long long b, int nbx, int nby) {
    BlockPos p;
    if (b < 0x7fffffffLL) {          // 32-bit division (a 64-bit one is a long software sequence)
        const unsigned ub = (unsigned)b, r = ub / (unsigned)nbx;
        p.bx = ub - r * (unsigned)nbx;
        p.bz = r / (unsigned)nby;
        p.by = r - (unsigned)p.bz * (unsigned)nby;
        return p;
    }
    p.bx = b % nbx;
    long long r = b / nbx;
    p.by = r % nby;
    p.bz = r / nby;
    return p;
}

// Encoder shared memory: one row of S words per thread that holds both the
// block's bit planes and its output stream.  Plane k sits at word kPlaneBase +
// (top - k); the planes are consumed in the order top, top - 1, ... while the
// stream is written from word 0 up, and the stream never overtakes an unread
// plane: with c planes started, at most 9 + 64 c (heads) + 64 (zero runs and
// ones, each position scanned once) + 64 (1 flags) + c (0 flags) = 137 + 65 c
// bits are out (fp64: 140 + 65 c), so the writer's words w, w + 1 stay below
// word kPlaneBase + c of the next unread plane for every c <= top (base 4 for
// 32 planes, 5 for 64).  S is odd, so a warp's rows start in different banks
// and the coalesced copy-out reads one row's consecutive words conflict-free.
constexpr int kPlaneBase32 = 4, kPlaneBase64 = 5;

// Coalesced copy of nb rows' first rate words (the CTA's contiguous streams)
// from shared memory to global.  Word i = (row r, column c), advanced with i
// instead of divided.
template <int NT>
__device__ __forceinline__ void copy_rows_out(const uint64_t* rows, int S, uint64_t* __restrict__ dst, int nb, int rate)
{
    const int t = threadIdx.x;
    const int total = nb * rate;
    const int dq = NT / rate, dr = NT - dq * rate;
    int r = t / rate, c = t - r * rate;
#pragma unroll 4
    for (int i = t; i < total; i += NT) {
        dst[i] = rows[r * S + c];
        r += dq;
        c += dr;
        if (c >= rate) { c -= rate; r++; }
    }
}

__host__ __device__ __forceinline__ int enc_row_stride(int rate, int planes, int base) {
    const int need = rate + 1 > base + planes ? rate + 1 : base + planes;
    return need | 1;
}

#ifndef OOCZ_ENC_MINB
#define OOCZ_ENC_MINB 5
#endif
__global__ void __launch_bounds__(kEncThreads, OOCZ_ENC_MINB)
zfp_encode_kernel(const float* __restrict__ in, int nx, int ny, int nbx, int nby,
                  long long nblocks, int rate, uint64_t* __restrict__ out)
{
    extern __shared__ __align__(16) uint64_t rows[];   // [kEncThreads][S]: planes and stream (above)
    const int S = enc_row_stride(rate, 32, kPlaneBase32);
    const int t = threadIdx.x;
    const long long b0 = (long long)blockIdx.x * kEncThreads;
    const long long b = b0 + t;
    zb::RowWriter bw{rows + t * S, 0, 0};
    bw.row[0] = 0ull;
    if (b < nblocks) {
#ifdef OOCZ_ENC_L2IN        // A/B bound for fusion (tools/fusion_bound.py): inputs from a 1 MB, L2-resident range
        const BlockPos p = block_pos(b & 4095, nbx, nby);
#else
        const BlockPos p = block_pos(b, nbx, nby);
#endif
        const float* base = in + ((size_t)(4 * p.bz) * ny + (size_t)(4 * p.by)) * nx + 4 * p.bx;
        uint32_t v[64];
#pragma unroll
        for (int k = 0; k < 4; k++)
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const float4 f = ld_slab(base + ((size_t)k * ny + j) * nx);
                v[16 * k + 4 * j + 0] = __float_as_uint(f.x);
                v[16 * k + 4 * j + 1] = __float_as_uint(f.y);
                v[16 * k + 4 * j + 2] = __float_as_uint(f.z);
                v[16 * k + 4 * j + 3] = __float_as_uint(f.w);
            }
        const int Emax = zb::block_exponent(v);
        if (Emax < 0) {
            bw.put(0, 1);                              // all-zero block: one 0 bit
        } else {
            const uint32_t e = (uint32_t)Emax + 1u;    // emax + 127, emax = Emax - 126
            bw.put(2u * e + 1u, zb::kHeaderBits);
            // q = trunc(x 2^(30 - emax)).  When 2^(30 - emax) is a normal fp32 (emax >= -97)
            // and the block is finite, x * 2^(30 - emax) is exact wherever |q| >= 1 (an
            // underflowing product is < 1 in magnitude and truncates to 0 either way):
            // one FMUL + one F2I.TRUNC per value, off the integer ALU pipe that binds
            // this kernel.  Otherwise the bit-field path.
            int32_t q[64];
            if (Emax >= 29 && Emax < 255) {
                const float sc = __int_as_float((283 - Emax) << 23);   // 2^(30 - emax), emax = Emax - 126
#pragma unroll
                for (int i = 0; i < 64; i++) q[i] = __float2int_rz(__fmul_rn(__uint_as_float(v[i]), sc));
            } else {
#pragma unroll
                for (int i = 0; i < 64; i++) q[i] = zb::quantize(v[i], Emax);
            }
            zb::fwd_xform(q);
            constexpr int perm[64] = OOCZ_PERM3;
            // negabinary (q + M) ^ M, M = 0xaaaaaaaa: the add here, the XOR folded into
            // the transposes (it complements the odd planes)
            uint32_t lo[32], hi[32];
#pragma unroll
            for (int i = 0; i < 32; i++) {
                lo[i] = (uint32_t)q[perm[i]] + zb::kNBMask;
                hi[i] = (uint32_t)q[perm[i + 32]] + zb::kNBMask;
            }
            zb::transpose32<true>(lo);
            zb::transpose32<true>(hi);
            uint64_t* pl = rows + t * S + kPlaneBase32 + 31;      // plane k at pl[-k]
#pragma unroll
            for (int k = 0; k < 32; k++) pl[-k] = ((uint64_t)hi[k] << 32) | lo[k];
            zb::encode_planes_rows([&](int k) { return pl[-k]; }, 31, 64 * rate, bw);
        }
        bw.zero_tail(rate);
    }
    __syncthreads();
    copy_rows_out<kEncThreads>(rows, S, out + (size_t)b0 * rate, nblocks - b0 < kEncThreads ? (int)(nblocks - b0) : kEncThreads,
                              rate);
}

__global__ void __launch_bounds__(kDecThreads)
zfp_decode_kernel(const uint64_t* __restrict__ in, int nx, int ny, int nbx, int nby,
                  long long nblocks, int rate, float* __restrict__ out, int ahead)
{
    __shared__ uint64_t planes_all[NB * 32 * kDecThreads];   // [32][kDecThreads]
    extern __shared__ __align__(16) uint64_t words[];      // [kDecThreads][S]
    const int t = threadIdx.x;
    const int S = dec_row_stride(rate);
    const long long b0 = (long long)blockIdx.x * kDecThreads;
    const long long nb = nblocks - b0 < kDecThreads ? nblocks - b0 : kDecThreads;
    if (ahead && t == 0) {          // the words of CTA + ahead, contiguous
        const long long f0 = b0 + (long long)ahead * kDecThreads;
        if (f0 < nblocks)
            prefetch_l2(in + (size_t)f0 * rate,
                        (uint32_t)((nblocks - f0 < kDecThreads ? nblocks - f0 : kDecThreads) * rate * 8) & ~15u);
    }
    stage_words<kDecThreads>(words, in + (size_t)b0 * rate, (int)nb * rate, rate, S);
    __syncthreads();

    int emax[NB];
    bool zero[NB];
    static_assert(NB == 1, "one event stream per thread");
    {
        const uint32_t* row = reinterpret_cast<const uint32_t*>(words + (size_t)t * S);
        emax[0] = 0;
        zero[0] = true;
        uint64_t* planes = planes_all + t;
        if (t < nb && (row[0] & 1u)) {
            zero[0] = false;
            emax[0] = (int)((row[0] >> 1) & 0xffu) - 127;
            zb::decode_planes_padded([&](int k, uint64_t x) { planes[k * kDecThreads] = x; }, 31, 64 * rate,
                                     zb::kHeaderBits, row);
        }
    }
#pragma unroll
    for (int s = 0; s < NB; s++) {
        const int bb = s * kDecThreads + t;
        if (bb >= nb) continue;
        const BlockPos p = block_pos(b0 + bb, nbx, nby);
        float* base = out + ((size_t)(4 * p.bz) * ny + (size_t)(4 * p.by)) * nx + 4 * p.bx;
        if (zero[s]) {                                 // zero block -> +0.0
#pragma unroll
            for (int k = 0; k < 4; k++)
#pragma unroll
                for (int j = 0; j < 4; j++)
                    st_slab(base + ((size_t)k * ny + j) * nx, make_float4(0.f, 0.f, 0.f, 0.f));
            continue;
        }
        uint64_t* planes = planes_all + s * 32 * kDecThreads;
        uint32_t lo[32], hi[32];
#pragma unroll
        for (int k = 0; k < 32; k++) {
            const uint64_t x = planes[k * kDecThreads + t];
            lo[k] = (uint32_t)x;
            hi[k] = (uint32_t)(x >> 32);
        }
        // negabinary (u ^ M) - M, M = 0xaaaaaaaa: the XOR folded into the transposes
        zb::transpose32<false, true>(lo);
        zb::transpose32<false, true>(hi);
        constexpr int perm[64] = OOCZ_PERM3;
        int32_t q[64];
#pragma unroll
        for (int i = 0; i < 32; i++) {
            q[perm[i]] = (int32_t)(lo[i] - zb::kNBMask);
            q[perm[i + 32]] = (int32_t)(hi[i] - zb::kNBMask);
        }
        zb::inv_xform(q);
        // dequantise: one branch per block (not per value, which the compiler
        // if-converts into both paths); emax >= -96 is the FMUL path of
        // zb::dequantize, the rest its fp64 path
        const int em = emax[s];
#ifdef OOCZ_DEC_NOSTORE     // A/B bound for fusion (tools/fusion_bound.sh): all the work, no output stores
        if (em >= -96 && g_dec_skip_store) {
            const float sc = __int_as_float((em - 30 + 127) << 23);
            uint32_t acc = 0;
#pragma unroll
            for (int l = 0; l < 64; l++) acc ^= __float_as_uint(__fmul_rn(__int2float_rn(q[l]), sc));
            if (nx < 0) *reinterpret_cast<uint32_t*>(base) = acc;
            continue;
        }
#endif
        if (em >= -96) {
            const float sc = __int_as_float((em - 30 + 127) << 23);
#pragma unroll
            for (int k = 0; k < 4; k++)
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int l = 16 * k + 4 * j;
                    st_slab(base + ((size_t)k * ny + j) * nx,
                            make_float4(__fmul_rn(__int2float_rn(q[l]), sc), __fmul_rn(__int2float_rn(q[l + 1]), sc),
                                        __fmul_rn(__int2float_rn(q[l + 2]), sc), __fmul_rn(__int2float_rn(q[l + 3]), sc)));
                }
        } else {
#pragma unroll
            for (int k = 0; k < 4; k++)
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int l = 16 * k + 4 * j;
                    st_slab(base + ((size_t)k * ny + j) * nx,
                            make_float4(zb::dequantize(q[l], em), zb::dequantize(q[l + 1], em),
                                        zb::dequantize(q[l + 2], em), zb::dequantize(q[l + 3], em)));
                }
        }
    }
}

// ---------------------------------------------------------------- fp64
// The paper's own precision.  Same shape as the fp32 kernels;
// 64 bit planes of 64 coefficients each, formed by four 32x32 transposes
// (coefficients 0-31 / 32-63 x integer bits 0-31 / 32-63).  Both kernels keep
// the planes in dynamic shared memory, [64][kThreads].
// plane k (0..63) of the 64 negabinary integers to pl[-k]
__device__ __forceinline__ void planes_from_ints64(const uint64_t u[64], uint64_t* pl) {
    uint32_t a[32], b[32];
#pragma unroll
    for (int half = 0; half < 2; half++) {     // integer bits 0-31, then 32-63
#pragma unroll
        for (int i = 0; i < 32; i++) {
            a[i] = (uint32_t)(u[i] >> (32 * half));
            b[i] = (uint32_t)(u[i + 32] >> (32 * half));
        }
        zb::transpose32<true>(a);             // (the negabinary XOR: odd planes complemented)
        zb::transpose32<true>(b);
#pragma unroll
        for (int k = 0; k < 32; k++) pl[-(32 * half + k)] = ((uint64_t)b[k] << 32) | a[k];
    }
}

// three CTAs per SM: a 69-word row per thread (planes and stream, as the fp32
// encoder), <= 168 registers
__global__ void __launch_bounds__(kThreads, 3)
zfp_encode64_kernel(const double* __restrict__ in, int nx, int ny, int nbx, int nby,
                    long long nblocks, int rate, uint64_t* __restrict__ out)
{
    extern __shared__ __align__(16) uint64_t rows[];   // [kThreads][S]
    const int S = enc_row_stride(rate, 64, kPlaneBase64);
    const int t = threadIdx.x;
    const long long b0 = (long long)blockIdx.x * kThreads;
    const long long b = b0 + t;
    zb::RowWriter bw{rows + t * S, 0, 0};
    bw.row[0] = 0ull;
    if (b < nblocks) {
        const BlockPos p = block_pos(b, nbx, nby);
        const double* base = in + ((size_t)(4 * p.bz) * ny + (size_t)(4 * p.by)) * nx + 4 * p.bx;
        uint64_t v[64];
#pragma unroll
        for (int k = 0; k < 4; k++)
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const double2* row = reinterpret_cast<const double2*>(base + ((size_t)k * ny + j) * nx);
                const double2 f0 = __ldg(row), f1 = __ldg(row + 1);
                v[16 * k + 4 * j + 0] = (uint64_t)__double_as_longlong(f0.x);
                v[16 * k + 4 * j + 1] = (uint64_t)__double_as_longlong(f0.y);
                v[16 * k + 4 * j + 2] = (uint64_t)__double_as_longlong(f1.x);
                v[16 * k + 4 * j + 3] = (uint64_t)__double_as_longlong(f1.y);
            }
        const int Emax = zb::block_exponent64(v);
        if (Emax < 0) {
            bw.put(0, 1);                                  // all-zero block: one 0 bit
        } else {
            bw.put(2ull * (uint64_t)(Emax + 1) + 1ull, zb::kHeaderBits64);   // e = emax + 1023
            int64_t q[64];
#pragma unroll
            for (int i = 0; i < 64; i++) q[i] = zb::quantize64(v[i], Emax);
            zb::fwd_xform(q);
            constexpr int perm[64] = OOCZ_PERM3;
            uint64_t u[64];
#pragma unroll
            for (int i = 0; i < 64; i++) u[i] = (uint64_t)q[perm[i]] + zb::kNBMask64;   // (^ M in the transposes)
            uint64_t* pl = rows + t * S + kPlaneBase64 + 63;   // plane k at pl[-k]
            planes_from_ints64(u, pl);
            zb::encode_planes_rows([&](int k) { return pl[-k]; }, 63, 64 * rate, bw);
        }
        bw.zero_tail(rate);
    }
    __syncthreads();
    copy_rows_out<kThreads>(rows, S, out + (size_t)b0 * rate, nblocks - b0 < kThreads ? (int)(nblocks - b0) : kThreads, rate);
}

// Two phases of 32 planes so that only 32 planes (32 KiB) are in shared memory
// at a time: planes 63..32 are decoded and transposed into the high halves of
// the 64 coefficients (kept in registers), then planes 31..0 reuse the same
// shared memory.  65 KiB per CTA at rate 32, three CTAs per SM (the 64-plane
// layout, 97 KiB, allowed two: the kernel is occupancy-limited).
__global__ void __launch_bounds__(kThreads, 3)
zfp_decode64_kernel(const uint64_t* __restrict__ in, int nx, int ny, int nbx, int nby,
                    long long nblocks, int rate, double* __restrict__ out)
{
    extern __shared__ __align__(16) uint64_t smem[];   // planes [32][kThreads], then words
    uint64_t* planes = smem;
    uint64_t* words = smem + 32 * kThreads;            // [kThreads][S]
    const int t = threadIdx.x;
    const int stride = dec_row_stride(rate);
    const long long b0 = (long long)blockIdx.x * kThreads;
    const long long nb = nblocks - b0 < kThreads ? nblocks - b0 : kThreads;
    stage_words<kThreads>(words, in + (size_t)b0 * rate, (int)nb * rate, rate, stride);
    __syncthreads();
    if (t >= nb) return;
    const BlockPos p = block_pos(b0 + t, nbx, nby);
    double* base = out + ((size_t)(4 * p.bz) * ny + (size_t)(4 * p.by)) * nx + 4 * p.bx;
    zb::BitReader br{words + (size_t)t * stride, 0};
    if (!br.read(1)) {                                 // zero block -> +0.0
#pragma unroll
        for (int k = 0; k < 4; k++)
#pragma unroll
            for (int j = 0; j < 4; j++) {
                double2* row = reinterpret_cast<double2*>(base + ((size_t)k * ny + j) * nx);
                row[0] = make_double2(0.0, 0.0);
                row[1] = make_double2(0.0, 0.0);
            }
        return;
    }
    const int emax = (int)br.read(zb::kEBits64) - 1023;
    uint64_t* pl = planes + t;
    zb::PadDecState st{63, 0, zb::kHeaderBits64, 0u, 0u, 0u};
    const uint32_t* p32 = reinterpret_cast<const uint32_t*>(words + (size_t)t * stride);
    uint32_t hi[64];                                   // bits 32..63 of the 64 coefficients
#pragma unroll
    for (int half = 1; half >= 0; half--) {
        const int kmin = 32 * half;
        zb::decode_planes_padded(st, kmin, [&](int k, uint64_t x) { pl[(k - kmin) * kThreads] = x; }, 64 * rate,
                                 p32);
        uint32_t a[32], b[32];
#pragma unroll
        for (int k = 0; k < 32; k++) {
            const uint64_t x = pl[k * kThreads];
            a[k] = (uint32_t)x;
            b[k] = (uint32_t)(x >> 32);
        }
        zb::transpose32<false, true>(a);      // (the negabinary XOR folded in)
        zb::transpose32<false, true>(b);
        if (half == 1) {
#pragma unroll
            for (int i = 0; i < 32; i++) { hi[i] = a[i]; hi[i + 32] = b[i]; }
            continue;
        }
        constexpr int perm[64] = OOCZ_PERM3;
        int64_t q[64];
#pragma unroll
        for (int i = 0; i < 32; i++) {
            const uint64_t u0 = ((uint64_t)hi[i] << 32) | a[i], u1 = ((uint64_t)hi[i + 32] << 32) | b[i];
            q[perm[i]] = (int64_t)(u0 - zb::kNBMask64);
            q[perm[i + 32]] = (int64_t)(u1 - zb::kNBMask64);
        }
        zb::inv_xform(q);
        // one branch per block: emax >= -960 is zb::dequantize64's one-DMUL path
        if (emax >= -960) {
            const double sc = __longlong_as_double((long long)(emax - 62 + 1023) << 52);
#pragma unroll
            for (int k = 0; k < 4; k++)
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int l = 16 * k + 4 * j;
                    double2* row = reinterpret_cast<double2*>(base + ((size_t)k * ny + j) * nx);
                    row[0] = make_double2(__dmul_rn(__ll2double_rn(q[l]), sc), __dmul_rn(__ll2double_rn(q[l + 1]), sc));
                    row[1] = make_double2(__dmul_rn(__ll2double_rn(q[l + 2]), sc),
                                          __dmul_rn(__ll2double_rn(q[l + 3]), sc));
                }
        } else {
#pragma unroll
            for (int k = 0; k < 4; k++)
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int l = 16 * k + 4 * j;
                    double2* row = reinterpret_cast<double2*>(base + ((size_t)k * ny + j) * nx);
                    row[0] = make_double2(zb::dequantize64(q[l], emax), zb::dequantize64(q[l + 1], emax));
                    row[1] = make_double2(zb::dequantize64(q[l + 2], emax), zb::dequantize64(q[l + 3], emax));
                }
        }
    }
}

size_t encode64_smem_bytes(int rate) { return sizeof(uint64_t) * (size_t)kThreads * enc_row_stride(rate, 64, kPlaneBase64); }
size_t decode64_smem_bytes(int rate) { return sizeof(uint64_t) * (size_t)(32 * kThreads + kThreads * dec_row_stride(rate)); }

size_t encode_smem_bytes(int rate) { return sizeof(uint64_t) * (size_t)kEncThreads * enc_row_stride(rate, 32, kPlaneBase32); }
size_t decode_smem_bytes(int rate) { return sizeof(uint64_t) * (size_t)kDecThreads * dec_row_stride(rate); }

// resident CTAs of a codec kernel on the whole GPU at this rate's shared memory
// (the prefetch lookahead); OOCZ_PREFETCH=0 turns the prefetch off (A/B)
int resident_ctas(const void* fn, int threads, size_t smem) {
    static const bool off = getenv("OOCZ_PREFETCH") && atoi(getenv("OOCZ_PREFETCH")) == 0;
    if (off) return 0;
    int dev = 0, sms = 0, per = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return per * sms;
}

bool codec_args_ok(int nx, int ny, int nz, int rate) {
    return nx >= 0 && ny >= 0 && nz >= 0 && nx % 4 == 0 && ny % 4 == 0 && nz % 4 == 0 &&
           rate >= 1 && rate <= 64;
}

}  // namespace

cudaError_t launch_zfp_encode(const float* in, int nx, int ny, int nz, int rate,
                              uint64_t* out, cudaStream_t s)
{
    if (!codec_args_ok(nx, ny, nz, rate)) return cudaErrorInvalidValue;
    const long long nblocks = (long long)(nx / 4) * (ny / 4) * (nz / 4);
    if (nblocks == 0) return cudaSuccess;
    static std::atomic<uint64_t> attr_done{0};
    {
        cudaError_t e = kernel_smem_setup((const void*)zfp_encode_kernel, (int)encode_smem_bytes(64), attr_done);
        if (e != cudaSuccess) return e;
    }
    const long long grid = (nblocks + kEncThreads - 1) / kEncThreads;
    zfp_encode_kernel<<<(unsigned)grid, kEncThreads, encode_smem_bytes(rate), s>>>(in, nx, ny, nx / 4, ny / 4,
                                                                           nblocks, rate, out);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_zfp_decode(const uint64_t* in, int nx, int ny, int nz, int rate,
                              float* out, cudaStream_t s)
{
    if (!codec_args_ok(nx, ny, nz, rate)) return cudaErrorInvalidValue;
    const long long nblocks = (long long)(nx / 4) * (ny / 4) * (nz / 4);
    if (nblocks == 0) return cudaSuccess;
    static std::atomic<uint64_t> attr_done{0};
    {
        cudaError_t e = kernel_smem_setup((const void*)zfp_decode_kernel, (int)decode_smem_bytes(64), attr_done);
        if (e != cudaSuccess) return e;
    }
    const long long grid = (nblocks + kDecThreads - 1) / kDecThreads;
#ifdef OOCZ_DEC_NOSTORE
    {
        static const int after = getenv("OOCZ_DEC_NOSTORE_AFTER") ? atoi(getenv("OOCZ_DEC_NOSTORE_AFTER")) : 40;
        const int nth = g_dec_launches++;
        if (nth == 0 || nth == after) {
            const int v = nth >= after ? 1 : 0;
            cudaMemcpyToSymbolAsync(g_dec_skip_store, &v, sizeof v, 0, cudaMemcpyHostToDevice, s);
        }
    }
#endif
    const int ahead = resident_ctas((const void*)zfp_decode_kernel, kDecThreads, decode_smem_bytes(rate));
    zfp_decode_kernel<<<(unsigned)grid, kDecThreads, decode_smem_bytes(rate), s>>>(in, nx, ny, nx / 4, ny / 4,
                                                                               nblocks, rate, out, ahead);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_zfp_encode64(const double* in, int nx, int ny, int nz, int rate,
                                uint64_t* out, cudaStream_t s)
{
    if (!codec_args_ok(nx, ny, nz, rate)) return cudaErrorInvalidValue;
    const long long nblocks = (long long)(nx / 4) * (ny / 4) * (nz / 4);
    if (nblocks == 0) return cudaSuccess;
    static std::atomic<uint64_t> attr_done{0};
    {
        cudaError_t e = kernel_smem_setup((const void*)zfp_encode64_kernel, (int)encode64_smem_bytes(64), attr_done);
        if (e != cudaSuccess) return e;
    }
    const long long grid = (nblocks + kThreads - 1) / kThreads;
    zfp_encode64_kernel<<<(unsigned)grid, kThreads, encode64_smem_bytes(rate), s>>>(in, nx, ny, nx / 4, ny / 4,
                                                                               nblocks, rate, out);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_zfp_decode64(const uint64_t* in, int nx, int ny, int nz, int rate,
                                double* out, cudaStream_t s)
{
    if (!codec_args_ok(nx, ny, nz, rate)) return cudaErrorInvalidValue;
    const long long nblocks = (long long)(nx / 4) * (ny / 4) * (nz / 4);
    if (nblocks == 0) return cudaSuccess;
    static std::atomic<uint64_t> attr_done{0};
    {
        cudaError_t e = kernel_smem_setup((const void*)zfp_decode64_kernel, (int)decode64_smem_bytes(64), attr_done);
        if (e != cudaSuccess) return e;
    }
    const long long grid = (nblocks + kThreads - 1) / kThreads;
    zfp_decode64_kernel<<<(unsigned)grid, kThreads, decode64_smem_bytes(rate), s>>>(in, nx, ny, nx / 4, ny / 4,
                                                                                   nblocks, rate, out);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t field_encode(const void* src, int esz, int nx, int ny, int nplanes, int rate, void* dst,
                         cudaStream_t s)
{
    if (rate == 0)
        return cudaMemcpyAsync(dst, src, (size_t)nplanes * nx * ny * esz, cudaMemcpyDeviceToDevice, s);
    return esz == 8 ? launch_zfp_encode64(static_cast<const double*>(src), nx, ny, nplanes, rate,
                                          static_cast<uint64_t*>(dst), s)
                    : launch_zfp_encode(static_cast<const float*>(src), nx, ny, nplanes, rate,
                                        static_cast<uint64_t*>(dst), s);
}

cudaError_t field_decode(const void* src, int esz, int nx, int ny, int nplanes, int rate, void* dst,
                         cudaStream_t s)
{
    if (rate == 0)
        return cudaMemcpyAsync(dst, src, (size_t)nplanes * nx * ny * esz, cudaMemcpyDeviceToDevice, s);
    return esz == 8 ? launch_zfp_decode64(static_cast<const uint64_t*>(src), nx, ny, nplanes, rate,
                                          static_cast<double*>(dst), s)
                    : launch_zfp_decode(static_cast<const uint64_t*>(src), nx, ny, nplanes, rate,
                                        static_cast<float*>(dst), s);
}

#ifdef OOCZ_DEC_NOSTORE
void zfp_ab_reset() { g_dec_launches = 0; }
#endif

}  // namespace oocz

// ------------------------------------------------------------------ C ABI
extern "C" size_t oocz_zfp_bytes(int32_t nx, int32_t ny, int32_t nz, int32_t rate)
{
    if (nx < 0 || ny < 0 || nz < 0 || rate < 0) return 0;
    return (size_t)(nx / 4) * (size_t)(ny / 4) * (size_t)(nz / 4) * 8u * (size_t)rate;
}

extern "C" oocz_status oocz_zfp_encode(const float* d_in, int32_t nx, int32_t ny, int32_t nz,
                                       int32_t rate, uint64_t* d_out, void* stream)
{
    if (nx % 4 || ny % 4 || nz % 4) return OOCZ_EALIGN;
    if (nx < 0 || ny < 0 || nz < 0 || rate < 1 || rate > 64 || ((!d_in || !d_out) && (size_t)nx * ny * nz != 0))
        return OOCZ_EINVAL;
    cudaError_t e = oocz::launch_zfp_encode(d_in, nx, ny, nz, rate, d_out, (cudaStream_t)stream);
    return oocz::stateless_status(e, __func__);
}

extern "C" oocz_status oocz_zfp_decode(const uint64_t* d_in, int32_t nx, int32_t ny, int32_t nz,
                                       int32_t rate, float* d_out, void* stream)
{
    if (nx % 4 || ny % 4 || nz % 4) return OOCZ_EALIGN;
    if (nx < 0 || ny < 0 || nz < 0 || rate < 1 || rate > 64 || ((!d_in || !d_out) && (size_t)nx * ny * nz != 0))
        return OOCZ_EINVAL;
    cudaError_t e = oocz::launch_zfp_decode(d_in, nx, ny, nz, rate, d_out, (cudaStream_t)stream);
    return oocz::stateless_status(e, __func__);
}

extern "C" oocz_status oocz_zfp_encode_f64(const double* d_in, int32_t nx, int32_t ny, int32_t nz,
                                           int32_t rate, uint64_t* d_out, void* stream)
{
    if (nx % 4 || ny % 4 || nz % 4) return OOCZ_EALIGN;
    if (nx < 0 || ny < 0 || nz < 0 || rate < 1 || rate > 64 || ((!d_in || !d_out) && (size_t)nx * ny * nz != 0))
        return OOCZ_EINVAL;
    cudaError_t e = oocz::launch_zfp_encode64(d_in, nx, ny, nz, rate, d_out, (cudaStream_t)stream);
    return oocz::stateless_status(e, __func__);
}

extern "C" oocz_status oocz_zfp_decode_f64(const uint64_t* d_in, int32_t nx, int32_t ny, int32_t nz,
                                           int32_t rate, double* d_out, void* stream)
{
    if (nx % 4 || ny % 4 || nz % 4) return OOCZ_EALIGN;
    if (nx < 0 || ny < 0 || nz < 0 || rate < 1 || rate > 64 || ((!d_in || !d_out) && (size_t)nx * ny * nz != 0))
        return OOCZ_EINVAL;
    cudaError_t e = oocz::launch_zfp_decode64(d_in, nx, ny, nz, rate, d_out, (cudaStream_t)stream);
    return oocz::stateless_status(e, __func__);
}
