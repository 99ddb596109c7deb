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
    BitWriter bw{out, 0ull, 0, 0};
    const int Emax = block_exponent(v);
    if (Emax < 0) { bw.put(0, 1); bw.finish(rate); return 0; }
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
    encode_planes([&](int k) { return planes[k]; }, 64 * rate - kHeaderBits, bw);
    bw.finish(rate);
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
