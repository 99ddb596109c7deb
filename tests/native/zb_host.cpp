// Test-only host build of the CUDA path's per-block coder (zfp_block.cuh), so the
// word-parallel logic can be compared with the bit-serial oracle without a GPU.
// Not part of liboocz.so; loaded by tests/test_codec_host_logic.py via ctypes.
#include <cstdint>
#include <cstring>
#include "../../paper_2109_05410_b200/csrc/zfp_block.cuh"

using namespace oocz::zb;

extern "C" int zb_encode_block(const float* x, int rate, uint64_t* out) {
    uint32_t v[64];
    std::memcpy(v, x, sizeof v);
    uint64_t row[66];                      // the kernel's shared-memory row: rate + 1 words
    std::memset(row, 0xa5, sizeof row);    // (garbage: every kept word must be written)
    RowWriter bw{row, 0ull, 0, 0};
    const int Emax = block_exponent(v);
    if (Emax < 0) {
        bw.put(0, 1);
    } else {
        bw.put(2u * (uint32_t)(Emax + 1) + 1u, kHeaderBits);
        int32_t q[64];
        for (int i = 0; i < 64; i++) q[i] = quantize(v[i], Emax);
        fwd_xform(q);
        const int perm[64] = OOCZ_PERM3;
        uint32_t lo[32], hi[32];
        for (int i = 0; i < 32; i++) {
            lo[i] = ((uint32_t)q[perm[i]] + kNBMask) ^ kNBMask;
            hi[i] = ((uint32_t)q[perm[i + 32]] + kNBMask) ^ kNBMask;
        }
        transpose32(lo);
        transpose32(hi);
        uint64_t planes[32];
        for (int k = 0; k < 32; k++) planes[k] = ((uint64_t)hi[k] << 32) | lo[k];
        encode_planes_rows([&](int k) { return planes[k]; }, 31, 64 * rate, bw);
    }
    bw.zero_tail(rate);
    std::memcpy(out, row, sizeof(uint64_t) * (size_t)rate);
    return 0;
}

extern "C" int zb_decode_block(const uint64_t* in_words, int rate, float* x) {
    uint64_t in[66] = {0};                 // spare words, as the kernel's smem staging has
    std::memcpy(in, in_words, sizeof(uint64_t) * (size_t)rate);
    BitReader br{in, 0};
    if (!br.read(1)) { for (int i = 0; i < 64; i++) x[i] = 0.0f; return 0; }
    const int emax = (int)br.read(kEBits) - 127;
    uint64_t planes[32];
    decode_planes([&](int k, uint64_t w) { planes[k] = w; }, 64 * rate - kHeaderBits, br);
    uint32_t lo[32], hi[32];
    for (int k = 0; k < 32; k++) { lo[k] = (uint32_t)planes[k]; hi[k] = (uint32_t)(planes[k] >> 32); }
    transpose32(lo);
    transpose32(hi);
    const int perm[64] = OOCZ_PERM3;
    int32_t q[64];
    for (int i = 0; i < 32; i++) {
        q[perm[i]] = (int32_t)((lo[i] ^ kNBMask) - kNBMask);
        q[perm[i + 32]] = (int32_t)((hi[i] ^ kNBMask) - kNBMask);
    }
    inv_xform(q);
    for (int i = 0; i < 64; i++) x[i] = dequantize(q[i], emax);
    return 0;
}

// ---- fp64: 64 bit planes of 64 coefficients; plane words from four 32x32 transposes
static void planes_from_ints64(const uint64_t u[64], uint64_t planes[64]) {
    uint32_t a[32], b[32], c[32], d[32];   // coeff 0-31 / 32-63, bits 0-31 / 32-63
    for (int i = 0; i < 32; i++) {
        a[i] = (uint32_t)u[i];       b[i] = (uint32_t)u[i + 32];
        c[i] = (uint32_t)(u[i] >> 32); d[i] = (uint32_t)(u[i + 32] >> 32);
    }
    transpose32(a); transpose32(b); transpose32(c); transpose32(d);
    for (int k = 0; k < 32; k++) {
        planes[k] = ((uint64_t)b[k] << 32) | a[k];
        planes[k + 32] = ((uint64_t)d[k] << 32) | c[k];
    }
}

static void ints_from_planes64(const uint64_t planes[64], uint64_t u[64]) {
    uint32_t a[32], b[32], c[32], d[32];
    for (int k = 0; k < 32; k++) {
        a[k] = (uint32_t)planes[k];      b[k] = (uint32_t)(planes[k] >> 32);
        c[k] = (uint32_t)planes[k + 32]; d[k] = (uint32_t)(planes[k + 32] >> 32);
    }
    transpose32(a); transpose32(b); transpose32(c); transpose32(d);
    for (int i = 0; i < 32; i++) {
        u[i] = ((uint64_t)c[i] << 32) | a[i];
        u[i + 32] = ((uint64_t)d[i] << 32) | b[i];
    }
}

extern "C" int zb_encode_block64(const double* x, int rate, uint64_t* out) {
    uint64_t v[64];
    std::memcpy(v, x, sizeof v);
    uint64_t row[66];
    std::memset(row, 0xa5, sizeof row);
    RowWriter bw{row, 0ull, 0, 0};
    const int Emax = block_exponent64(v);
    if (Emax < 0) {
        bw.put(0, 1);
    } else {
        bw.put(2ull * (uint64_t)(Emax + 1) + 1ull, kHeaderBits64);
        int64_t q[64];
        for (int i = 0; i < 64; i++) q[i] = quantize64(v[i], Emax);
        fwd_xform(q);
        const int perm[64] = OOCZ_PERM3;
        uint64_t u[64], planes[64];
        for (int i = 0; i < 64; i++) u[i] = ((uint64_t)q[perm[i]] + kNBMask64) ^ kNBMask64;
        planes_from_ints64(u, planes);
        encode_planes_rows([&](int k) { return planes[k]; }, 63, 64 * rate, bw);
    }
    bw.zero_tail(rate);
    std::memcpy(out, row, sizeof(uint64_t) * (size_t)rate);
    return 0;
}

extern "C" int zb_decode_block64(const uint64_t* in_words, int rate, double* x) {
    uint64_t in[66] = {0};
    std::memcpy(in, in_words, sizeof(uint64_t) * (size_t)rate);
    BitReader br{in, 0};
    if (!br.read(1)) { for (int i = 0; i < 64; i++) x[i] = 0.0; return 0; }
    const int emax = (int)br.read(kEBits64) - 1023;
    uint64_t planes[64], u[64];
    decode_planes([&](int k, uint64_t w) { planes[k] = w; }, 64 * rate - kHeaderBits64, br, 63);
    ints_from_planes64(planes, u);
    const int perm[64] = OOCZ_PERM3;
    int64_t q[64];
    for (int i = 0; i < 64; i++) q[perm[i]] = (int64_t)((u[i] ^ kNBMask64) - kNBMask64);
    inv_xform(q);
    for (int i = 0; i < 64; i++) x[i] = dequantize64(q[i], emax);
    return 0;
}
