// Test-only host build of the CUDA path's per-block coder (zfp_block.cuh), so the
// word-parallel logic can be compared with the bit-serial oracle without a GPU.
// Not part of liboocz.so; loaded by tests/test_codec_host_logic.py via ctypes.
#include <cstdint>
#include <cstring>
#include "../../paper_2109_05410_b200/csrc/zfp_block.cuh"

using namespace oocz::zb;

// The kernels' shared-memory row: planes at word base + (top - k), the stream
// written from word 0 up over them (zfp.cu, "Encoder shared memory"); the row
// is filled with garbage first so that an overtaken plane or an unwritten kept
// word shows up as a mismatch.
static int row_stride(int rate, int planes, int base) {
    const int need = rate + 1 > base + planes ? rate + 1 : base + planes;
    return need | 1;
}
template <int TOP, int BASE>
static void encode_rows(const uint64_t planes[TOP + 1], int header, uint64_t hv, int rate, uint64_t* out) {
    uint64_t row[80];
    std::memset(row, 0xa5, sizeof row);
    (void)row_stride;
    uint64_t* pl = row + BASE + TOP;
    for (int k = 0; k <= TOP; k++) pl[-k] = planes[k];
    RowWriter bw{row, 0, 0};
    row[0] = 0ull;
    bw.put(hv, header);
    encode_planes_rows([&](int k) { return pl[-k]; }, TOP, 64 * rate, bw);
    bw.zero_tail(rate);
    std::memcpy(out, row, sizeof(uint64_t) * (size_t)rate);
}

// the plane coder alone on 64 arbitrary negabinary integers (after a header of
// `header` zero bits): the adversarial inputs of the overlap bound
extern "C" int zb_encode_ints_rows(const uint32_t* u, int header, int rate, uint64_t* out) {
    uint32_t lo[32], hi[32];
    for (int i = 0; i < 32; i++) { lo[i] = u[i]; hi[i] = u[i + 32]; }
    transpose32(lo);
    transpose32(hi);
    uint64_t planes[32];
    for (int k = 0; k < 32; k++) planes[k] = ((uint64_t)hi[k] << 32) | lo[k];
    encode_rows<31, 4>(planes, header, 0, rate, out);
    return 0;
}

extern "C" int zb_encode_block(const float* x, int rate, uint64_t* out) {
    uint32_t v[64];
    std::memcpy(v, x, sizeof v);
    const int Emax = block_exponent(v);
    if (Emax < 0) {                        // all-zero block: one 0 bit
        uint64_t row[66];
        std::memset(row, 0xa5, sizeof row);
        RowWriter bw{row, 0, 0};
    row[0] = 0ull;
        bw.put(0, 1);
        bw.zero_tail(rate);
        std::memcpy(out, row, sizeof(uint64_t) * (size_t)rate);
        return 0;
    }
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
    encode_rows<31, 4>(planes, kHeaderBits, 2u * (uint32_t)(Emax + 1) + 1u, rate, out);
    return 0;
}

extern "C" int zb_decode_block(const uint64_t* in_words, int rate, float* x) {
    uint64_t in[68] = {0};                 // 3 zero words past the stream, as the kernel's staging
    std::memcpy(in, in_words, sizeof(uint64_t) * (size_t)rate);
    BitReader br{in, 0};
    if (!br.read(1)) { for (int i = 0; i < 64; i++) x[i] = 0.0f; return 0; }
    const int emax = (int)br.read(kEBits) - 127;
    uint64_t planes[32];
    decode_planes_padded([&](int k, uint64_t w) { planes[k] = w; }, 31, 64 * rate, br.pos,
                         reinterpret_cast<const uint32_t*>(in));
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
    const int Emax = block_exponent64(v);
    if (Emax < 0) {
        uint64_t row[66];
        std::memset(row, 0xa5, sizeof row);
        RowWriter bw{row, 0, 0};
    row[0] = 0ull;
        bw.put(0, 1);
        bw.zero_tail(rate);
        std::memcpy(out, row, sizeof(uint64_t) * (size_t)rate);
        return 0;
    }
    int64_t q[64];
    for (int i = 0; i < 64; i++) q[i] = quantize64(v[i], Emax);
    fwd_xform(q);
    const int perm[64] = OOCZ_PERM3;
    uint64_t u[64], planes[64];
    for (int i = 0; i < 64; i++) u[i] = ((uint64_t)q[perm[i]] + kNBMask64) ^ kNBMask64;
    planes_from_ints64(u, planes);
    encode_rows<63, 5>(planes, kHeaderBits64, 2ull * (uint64_t)(Emax + 1) + 1ull, rate, out);
    return 0;
}

extern "C" int zb_encode_ints64_rows(const uint64_t* u, int header, int rate, uint64_t* out) {
    uint64_t planes[64];
    planes_from_ints64(u, planes);
    encode_rows<63, 5>(planes, header, 0, rate, out);
    return 0;
}

extern "C" int zb_decode_block64(const uint64_t* in_words, int rate, double* x) {
    uint64_t in[68] = {0};
    std::memcpy(in, in_words, sizeof(uint64_t) * (size_t)rate);
    BitReader br{in, 0};
    if (!br.read(1)) { for (int i = 0; i < 64; i++) x[i] = 0.0; return 0; }
    const int emax = (int)br.read(kEBits64) - 1023;
    uint64_t planes[64], u[64];
    decode_planes_padded([&](int k, uint64_t w) { planes[k] = w; }, 63, 64 * rate, br.pos,
                         reinterpret_cast<const uint32_t*>(in));
    ints_from_planes64(planes, u);
    const int perm[64] = OOCZ_PERM3;
    int64_t q[64];
    for (int i = 0; i < 64; i++) q[perm[i]] = (int64_t)((u[i] ^ kNBMask64) - kNBMask64);
    inv_xform(q);
    for (int i = 0; i < 64; i++) x[i] = dequantize64(q[i], emax);
    return 0;
}
