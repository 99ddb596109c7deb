// zfp_block.cuh -- per-4^3-block ZFP fixed-rate coder, word-parallel.
//
// Format (zfp 0.5.5 fixed-rate fp32 3-D, the layout of the
// cuZFP 0.5.5 library the paper uses): 1 flag bit,
// 8 exponent bits, group-tested bit planes 31..0 of the negabinary,
// sequency-ordered coefficients of the lifted block-floating-point integers,
// truncated at 64*rate bits.
//
// This is NOT a transcription of a bit-serial coder.  One thread owns one
// block and works on whole 64-bit bit planes:
//   * quantisation straight from the fp32 bit fields (integer ops, exact),
//   * 32x32 bit-matrix transposes to turn 64 coefficients into 32 planes,
//   * each group test emits/consumes a whole zero run at once (ctz on the
//     plane word / on the next <=63 stream bits), so the coder's cost is
//     O(planes + newly significant coefficients) instead of O(bits).
// Functions are __host__ __device__ only so that a stand-alone CPU build of
// this header (tests/native/zb_host.cpp) can exercise the same logic; the
// library itself only calls them from CUDA kernels.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>

#if defined(__CUDACC__)
#define ZB_HD __host__ __device__ __forceinline__
#else
#define ZB_HD inline
#endif
#if defined(__CUDA_ARCH__)
#define ZB_UNROLL _Pragma("unroll")
#else
#define ZB_UNROLL
#endif

namespace oocz {
namespace zb {

constexpr uint32_t kNBMask = 0xaaaaaaaau;
constexpr int kEBits = 8;
constexpr int kHeaderBits = 1 + kEBits;

// sequency order of the 64 coefficients (by i+j+k, then i^2+j^2+k^2)
#define OOCZ_PERM3                                                                  \
    { 0, 1, 4, 16, 20, 17, 5, 2, 8, 32, 21, 6, 18, 24, 9, 33,                         \
      36, 3, 12, 48, 22, 25, 37, 40, 34, 10, 7, 19, 28, 13, 49, 52,                   \
      41, 38, 26, 23, 29, 53, 11, 35, 44, 14, 50, 56, 42, 27, 39, 45,                 \
      30, 54, 57, 60, 51, 15, 43, 46, 58, 61, 55, 31, 62, 59, 47, 63 }

ZB_HD int ctz64(uint64_t x) {
#if defined(__CUDA_ARCH__)
    return __ffsll((long long)x) - 1;
#else
    return __builtin_ctzll(x);
#endif
}

ZB_HD uint64_t lowmask(int m) { return m >= 64 ? ~0ull : ((1ull << m) - 1ull); }
ZB_HD uint64_t shr64(uint64_t x, int s) { return s >= 64 ? 0ull : (x >> s); }

// Two's-complement wraparound arithmetic with arithmetic >> (App. A), on the
// block's integer type I (int32_t for fp32 data, int64_t for fp64 data)
template <class I> struct UnsignedOf;
template <> struct UnsignedOf<int32_t> { using type = uint32_t; };
template <> struct UnsignedOf<int64_t> { using type = uint64_t; };
template <class I> ZB_HD I add(I a, I b) { using U = typename UnsignedOf<I>::type; return (I)((U)a + (U)b); }
template <class I> ZB_HD I sub(I a, I b) { using U = typename UnsignedOf<I>::type; return (I)((U)a - (U)b); }
template <class I> ZB_HD I shl1(I a) { using U = typename UnsignedOf<I>::type; return (I)((U)a << 1); }
template <class I> ZB_HD I asr1(I a) { return a >> 1; }

template <class I>
ZB_HD void fwd_lift(I& x, I& y, I& z, I& w) {
    x = add(x, w); x = asr1(x); w = sub(w, x);
    z = add(z, y); z = asr1(z); y = sub(y, z);
    x = add(x, z); x = asr1(x); z = sub(z, x);
    w = add(w, y); w = asr1(w); y = sub(y, w);
    w = add(w, asr1(y)); y = sub(y, asr1(w));
}

template <class I>
ZB_HD void inv_lift(I& x, I& y, I& z, I& w) {
    y = add(y, asr1(w)); w = sub(w, asr1(y));
    y = add(y, w); w = shl1(w); w = sub(w, y);
    z = add(z, x); x = shl1(x); x = sub(x, z);
    y = add(y, z); z = shl1(z); z = sub(z, y);
    w = add(w, x); x = shl1(x); x = sub(x, w);
}

// q[i + 4j + 16k]; lines along x, then y, then z
template <class I>
ZB_HD void fwd_xform(I q[64]) {
ZB_UNROLL
    for (int l = 0; l < 16; l++) { int b = 4 * l; fwd_lift(q[b], q[b + 1], q[b + 2], q[b + 3]); }
ZB_UNROLL
    for (int l = 0; l < 16; l++) { int b = (l & 3) + 16 * (l >> 2); fwd_lift(q[b], q[b + 4], q[b + 8], q[b + 12]); }
ZB_UNROLL
    for (int l = 0; l < 16; l++) { int b = l; fwd_lift(q[b], q[b + 16], q[b + 32], q[b + 48]); }
}

template <class I>
ZB_HD void inv_xform(I q[64]) {
ZB_UNROLL
    for (int l = 0; l < 16; l++) { int b = l; inv_lift(q[b], q[b + 16], q[b + 32], q[b + 48]); }
ZB_UNROLL
    for (int l = 0; l < 16; l++) { int b = (l & 3) + 16 * (l >> 2); inv_lift(q[b], q[b + 4], q[b + 8], q[b + 12]); }
ZB_UNROLL
    for (int l = 0; l < 16; l++) { int b = 4 * l; inv_lift(q[b], q[b + 1], q[b + 2], q[b + 3]); }
}

#if defined(__CUDA_ARCH__)
// (m & a) | (~m & b) and its complement as ONE LOP3 (written out, ptxas splits the
// disjoint OR into two LOP3s and an add)
__device__ __forceinline__ uint32_t bitsel(uint32_t m, uint32_t a, uint32_t b) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xca;" : "=r"(r) : "r"(m), "r"(a), "r"(b));   // m ? a : b (LUT over 0xf0, 0xcc, 0xaa)
    return r;
}
__device__ __forceinline__ uint32_t bitsel_na(uint32_t m, uint32_t a, uint32_t b) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0x3a;" : "=r"(r) : "r"(m), "r"(a), "r"(b));   // m ? ~a : b
    return r;
}
__device__ __forceinline__ uint32_t bitsel_nb(uint32_t m, uint32_t a, uint32_t b) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xc5;" : "=r"(r) : "r"(m), "r"(a), "r"(b));   // m ? a : ~b
    return r;
}
__device__ __forceinline__ uint32_t bitsel_not(uint32_t m, uint32_t a, uint32_t b) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0x35;" : "=r"(r) : "r"(m), "r"(a), "r"(b));   // ~(m ? a : b)
    return r;
}
#endif

// In-place 32x32 bit transpose, LSB = column 0: afterwards bit i of a[k] is
// the former bit k of a[i].  5 butterfly levels of 16 masked swaps.
// NB_ODD (encoder): also complement the odd output words, i.e. transpose the
// input XORed with 0xaaaaaaaa in every word (the negabinary XOR, folded into
// the last level's LOP3s for free).
// NB_IN (decoder): transpose the input with its odd words complemented, i.e.
// XOR every output word with 0xaaaaaaaa.  The 16-, 8-, 4- and 2-bit levels only
// combine words of equal parity, so the complement of the odd words carries
// through them untouched (the shifted-in bits fall outside the select masks);
// the 1-bit level, which pairs word k with k + 1, applies it with two other
// LOP3 tables.
template <bool NB_ODD = false, bool NB_IN = false>
ZB_HD void transpose32(uint32_t a[32]) {
#if defined(__CUDA_ARCH__)
    // the 16- and 8-bit levels are whole half-word / byte exchanges: one PRMT
    // per output word instead of shift / xor / and / xor / shift / xor
ZB_UNROLL
    for (int k = 0; k < 16; k++) {
        const uint32_t x = a[k], y = a[k + 16];
        a[k] = __byte_perm(x, y, 0x5410);          // (x.lo, y.lo)
        a[k + 16] = __byte_perm(x, y, 0x7632);     // (x.hi, y.hi)
    }
ZB_UNROLL
    for (int k = 0; k < 32; k++) {
        if ((k & 8) == 0) {
            const uint32_t x = a[k], y = a[k + 8];
            a[k] = __byte_perm(x, y, 0x6240);      // (x.b0, y.b0, x.b2, y.b2)
            a[k + 8] = __byte_perm(x, y, 0x7351);  // (x.b1, y.b1, x.b3, y.b3)
        }
    }
    // the 4-, 2- and 1-bit levels as two bit-selects per pair,
    //   a' = (a & ~(m << j)) | ((b << j) & (m << j)),  b' = (b & ~m) | ((a >> j) & m),
    // each one LOP3 on the ALU pipe, with the shifts on the FMA pipe (IMAD.SHL,
    // and the logical right shift as IMAD.HI): the ALU pipe binds the codec
    uint32_t m = 0x0f0f0f0fu;
ZB_UNROLL
    for (int j = 4; j != 0; j >>= 1) {
        const uint32_t mj = m << j;
ZB_UNROLL
        for (int k = 0; k < 32; k++) {
            if ((k & j) == 0) {
                const uint32_t x = a[k], y = a[k + j];
                const uint32_t xs = __umulhi(x, 1u << (32 - j)), ys = y * (1u << j);
                if (NB_IN && j == 1) {                      // y is an odd word: use ~y
                    a[k] = bitsel_na(mj, ys, x);
                    a[k + j] = bitsel_nb(m, xs, y);
                } else {
                    a[k] = bitsel(mj, ys, x);
                    a[k + j] = (NB_ODD && j == 1) ? bitsel_not(m, xs, y) : bitsel(m, xs, y);   // (k + 1 is odd)
                }
            }
        }
        m ^= m << (j >> 1);
    }
#else
    uint32_t m = 0x0000ffffu;
    for (int j = 16; j != 0; j >>= 1) {
        for (int k = 0; k < 32; k++) {
            if ((k & j) == 0) {
                uint32_t t = ((a[k] >> j) ^ a[k + j]) & m;
                a[k + j] ^= t;
                a[k] ^= t << j;
            }
        }
        m ^= m << (j >> 1);
    }
    if (NB_ODD)
        for (int k = 1; k < 32; k += 2) a[k] = ~a[k];
    if (NB_IN)
        for (int k = 0; k < 32; k++) a[k] ^= 0xaaaaaaaau;
#endif
}

// Common exponent from fp32 bit patterns: returns the biased exponent E of the
// largest magnitude (emax = E - 126, i.e. max(frexp exponent, -126); E = 0 for
// an all-denormal block), or -1 for an all-zero block.
ZB_HD int block_exponent(const uint32_t v[64]) {
    // max of the bit patterns shifted left by one (the sign bit dropped: a
    // multiply by 2 on the FMA pipe instead of an AND on the ALU pipe)
    uint32_t mx = 0;
ZB_UNROLL
    for (int i = 0; i < 64; i++) { uint32_t a = v[i] * 2u; mx = a > mx ? a : mx; }
    return mx == 0 ? -1 : (int)(mx >> 24);
}

// q = trunc(x * 2^(30 - emax)), built from the bit fields: x = mant * 2^(max(E,1)-150)
ZB_HD int32_t quantize(uint32_t bits, int Emax) {
    int E = (int)((bits >> 23) & 0xffu);
    uint32_t mant = (bits & 0x7fffffu) | (E ? 0x800000u : 0u);
    int s = (E < 1 ? 1 : E) - Emax + 6;                       // <= 6
    uint32_t a = s >= 0 ? (mant << s) : (s > -32 ? (mant >> (-s)) : 0u);
    return (bits >> 31) ? -(int32_t)a : (int32_t)a;
}

// x = fl32(fl32(q) * 2^(emax-30)), one rounding of the exact product
ZB_HD float dequantize(int32_t q, int emax) {
    int64_t sb = (int64_t)(emax - 30 + 1023) << 52;
#if defined(__CUDA_ARCH__)
    // emax >= -96: every nonzero |fl32(q)| * 2^(emax-30) is >= 2^-126 (normal), so
    // the fp32 product by a power of two is exact (or overflows exactly as the
    // rounded fp64 product does): the same bits as the fp64 path, one FMUL
    if (emax >= -96) return __fmul_rn(__int2float_rn(q), __int_as_float((emax - 30 + 127) << 23));
    double s = __longlong_as_double(sb);
    return __double2float_rn(__dmul_rn((double)__int2float_rn(q), s));
#else
    double s;
    std::memcpy(&s, &sb, sizeof s);
    return (float)((double)(float)q * s);
#endif
}

// ---- fp64 (EBITS 11, EBIAS 1023, 64 bit planes, q = trunc(x * 2^(62 - emax)))
constexpr uint64_t kNBMask64 = 0xaaaaaaaaaaaaaaaaull;
constexpr int kEBits64 = 11;
constexpr int kHeaderBits64 = 1 + kEBits64;

// biased exponent E of the largest magnitude (emax = E - 1022, E = 0 for an
// all-denormal block), or -1 for an all-zero block
ZB_HD int block_exponent64(const uint64_t v[64]) {
    uint64_t mx = 0;
ZB_UNROLL
    for (int i = 0; i < 64; i++) { uint64_t a = v[i] & 0x7fffffffffffffffull; mx = a > mx ? a : mx; }
    return mx == 0 ? -1 : (int)(mx >> 52);
}

// q = trunc(x * 2^(62 - emax)) from the bit fields: x = mant * 2^(max(E,1) - 1075)
ZB_HD int64_t quantize64(uint64_t bits, int Emax) {
    int E = (int)((bits >> 52) & 0x7ffu);
    uint64_t mant = (bits & 0xfffffffffffffull) | (E ? 0x10000000000000ull : 0ull);
    int s = (E < 1 ? 1 : E) - Emax + 9;                         // <= 9
    uint64_t a = s >= 0 ? (mant << s) : (s > -64 ? (mant >> (-s)) : 0ull);
    return (bits >> 63) ? -(int64_t)a : (int64_t)a;
}

// x = fl64(fl64(q) * 2^(emax - 62)), one rounding of the exact product (ldexp)
ZB_HD double dequantize64(int64_t q, int emax) {
#if defined(__CUDA_ARCH__)
    const double a = __ll2double_rn(q);
    if (emax >= -960)            // every nonzero result is normal: the product is exact
        return __dmul_rn(a, __longlong_as_double((long long)(emax - 62 + 1023) << 52));
    // subnormal results: an exact scaling by 2^-64 first, then one rounding
    return __dmul_rn(__dmul_rn(a, 0x1p-64), __longlong_as_double((long long)(emax - 62 + 64 + 1023) << 52));
#else
    return std::ldexp((double)q, emax - 62);
#endif
}

// ---------------------------------------------------------------- bit I/O
struct BitWriter {
    uint64_t* p;      // output words of this block
    uint64_t acc;     // pending bits (LSB first)
    int nb;           // number of pending bits, < 64
    int words;        // words stored so far
    // append the low n bits of v (1 <= n <= 64, v < 2^n)
    ZB_HD void put(uint64_t v, int n) {
        acc |= v << nb;
        nb += n;
        if (nb >= 64) {
            p[words++] = acc;
            nb -= 64;
            acc = nb ? (v >> (n - nb)) : 0ull;
        }
    }
    // the same for 0 <= n <= 65 (bit 64 of a 65-bit emission is 0: the closing
    // flag), with no data-dependent branch: the word stores are predicated
    ZB_HD void put_fast(uint64_t v, int n) {
        acc |= v << nb;
        const uint64_t spill = shr64(v, 64 - nb);   // the bits of v past the word
        nb += n;
        const bool f1 = nb >= 64;
        if (f1) p[words] = acc;
        words += f1 ? 1 : 0;
        acc = f1 ? spill : acc;
        nb -= f1 ? 64 : 0;
        const bool f2 = nb >= 64;                   // only after 65 bits from nb = 63
        if (f2) p[words] = acc;
        words += f2 ? 1 : 0;
        acc = f2 ? 0ull : acc;
        nb -= f2 ? 64 : 0;
    }
    ZB_HD void finish(int total_words) {       // zero padding to the fixed size
        if (nb) { p[words++] = acc; acc = 0; nb = 0; }
        while (words < total_words) p[words++] = 0ull;
    }
};

struct BitReader {
    const uint64_t* p;  // stream words of this block
    int pos;            // bit position
    // next m bits (0 <= m <= 64) without consuming them; never reads past the
    // word holding the last requested bit
    ZB_HD uint64_t peek(int m) const {
        if (m == 0) return 0ull;
        const int w = pos >> 6, o = pos & 63;
        uint64_t v = p[w] >> o;
        if (o + m > 64) v |= p[w + 1] << (64 - o);
        return v & lowmask(m);
    }
    ZB_HD uint64_t read(int m) { uint64_t v = peek(m); pos += m; return v; }
    // the 64 stream bits from pos on, as two 32-bit halves (reads the 32-bit
    // words at pos/32 + 0..2: up to 8 bytes past the last bit, so the stream
    // needs one spare word after it -- the staged copies have one)
    ZB_HD void window(uint32_t& wl, uint32_t& wh) const;
};

// ---------------------------------------------------------------- plane coder
// Both coders run ONE flat loop of per-lane "events" whose body is
// straight-line code (both alternatives computed, then selected), so the 32
// lanes of a warp -- 32 different blocks -- never wait for each other's group
// tests and the compiler has no branch to re-nest into an inner loop:
//   plane start : the first n bits of plane k verbatim, plus the group flag 0
//                 when nothing new is significant in the plane (plane done);
//   found one   : flag 1, the zero run and the one (1 | 2 << tz: tz + 2 bits;
//                 tz + 1 bits when the one sits at position 63, which is never
//                 sent), plus the closing flag 0 when no one is left.
// The encoded stream is exactly the bit-serial coder's, cut at the budget.

// ---- 32-bit helpers: each is one or two SASS instructions on the device
ZB_HD uint32_t fshr32(uint32_t lo, uint32_t hi, int s) {   // ((hi:lo) >> s) & 0xffffffff, 0 <= s < 32
#if defined(__CUDA_ARCH__)
    return __funnelshift_r(lo, hi, s);
#else
    return s ? (lo >> s) | (hi << (32 - s)) : lo;
#endif
}
ZB_HD uint32_t bmask32(int m) {                            // low clamp(m, 0, 32) bits set
#if defined(__CUDA_ARCH__)
    uint32_t r;
    asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(r) : "r"(m < 0 ? 0 : m));
    return r;
#else
    return m <= 0 ? 0u : (m >= 32 ? ~0u : ((1u << m) - 1u));
#endif
}
ZB_HD int ctz32nz(uint32_t x) {                            // x != 0
#if defined(__CUDA_ARCH__)
    return __ffs((int)x) - 1;
#else
    return __builtin_ctz(x);
#endif
}
ZB_HD uint32_t bit64(uint32_t lo, uint32_t hi, int p) {    // bit p (0..63) of hi:lo
    return (p < 32 ? fshr32(lo, hi, p) : (hi >> (p & 31))) & 1u;
}

ZB_HD void BitReader::window(uint32_t& wl, uint32_t& wh) const {
    const uint32_t* p32 = reinterpret_cast<const uint32_t*>(p) + (pos >> 5);
    const int o = pos & 31;
    const uint32_t w0 = p32[0], w1 = p32[1], w2 = p32[2];
    wl = fshr32(w0, w1, o);
    wh = fshr32(w1, w2, o);
}

// Emit the low `len` bits of v (len <= 65: a 0 flag after a full word), cut at
// the remaining budget.
// FAST: the caller guarantees bits >= 65 (no event emits more), so no cut.
template <bool FAST = false>
ZB_HD void emit(BitWriter& bw, uint64_t v, int len, int& bits) {
    if (FAST) {
        bw.put_fast(v, len);
    } else {
        if (len > bits) { len = bits; v &= lowmask(len); }
        if (len > 64) { bw.put(v, 64); bw.put(0, len - 64); }
        else if (len > 0) bw.put(v, len);
    }
    bits -= len;
}

// One encoder event.  State: plane index k, significant count n, whether the
// group tests of plane k are under way, remaining budget.  The remaining plane
// bits y = x >> n drive both alternatives:
//   plane start : x & mask(n), then a 0 flag if y == 0 (plane done);
//   found one   : tz = ctz(y): 1 | 2 << tz (tz + 2 bits; tz + 1 if the one is at
//                 63, which is implied), then a closing 0 flag if y had a single
//                 one left (y & (y - 1) == 0).
struct EncState {
    int k, n, bits;
    bool inplane;
    ZB_HD bool active() const { return k >= 0 && bits > 0; }
};

template <bool FAST = false, class PlaneAt>
ZB_HD void encode_event(EncState& st, PlaneAt plane_at, BitWriter& bw) {
    const int n = st.n;
    const uint64_t x = plane_at(st.k);
    const uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
    // y = x >> n on 32-bit halves (n in 0..64)
    const uint32_t yl = n < 32 ? fshr32(xl, xh, n) : (n < 64 ? xh >> (n & 31) : 0u);
    const uint32_t yh = n < 32 ? xh >> n : 0u;
    const int tz = yl ? ctz32nz(yl) : 32 + ctz32nz(yh | 0x80000000u);
    const bool implied = n + tz >= 63;
    const bool lastone = yl ? ((yl & (yl - 1u)) == 0u && yh == 0u) : ((yh & (yh - 1u)) == 0u);
    // found one: 1 | 2 << tz
    const int t1 = tz + 1;
    const uint32_t vBl = implied ? 1u : (1u | (t1 < 32 ? 1u << (t1 & 31) : 0u));
    const uint32_t vBh = implied ? 0u : (t1 >= 32 ? 1u << (t1 & 31) : 0u);
    const int lenB = implied ? tz + 1 : tz + 2 + (lastone ? 1 : 0);
    const bool doneB = implied || lastone;
    const int nB = implied ? 64 : n + t1;
    // plane start: x & mask(n)
    const bool yz = (yl | yh) == 0u;
    const uint32_t vAl = xl & bmask32(n), vAh = xh & bmask32(n - 32);
    const int lenA = n + ((n < 64 && yz) ? 1 : 0);
    const bool doneA = n >= 64 || yz;
    const bool ip = st.inplane;
    const uint32_t vl = ip ? vBl : vAl, vh = ip ? vBh : vAh;
    emit<FAST>(bw, ((uint64_t)vh << 32) | vl, ip ? lenB : lenA, st.bits);
    const bool done = ip ? doneB : doneA;
    st.n = ip ? nB : n;
    st.k -= done ? 1 : 0;
    st.inplane = !done;
}

// The budget-free (bits >= 65) event that also merges a plane start with the
// plane's first unit: at a plane start with something newly significant, the
// n verbatim bits and the unit (flag 1, zero run, one, closing flag) go out as
// ONE emission.  Its length is n + tz + 2 + lastone <= 65 (n + tz <= 62 unless
// the one at 63 is implied, and then it is n + tz + 1 = 64), and a 65th bit is
// the closing 0 flag, so one put always suffices.  A plane with j >= 1 new
// ones takes j events instead of j + 1 (measured on the C2 data: 35 events per
// block instead of 48, the warp's maximum 42 instead of 55).
template <class PlaneAt>
ZB_HD void encode_event_merged(EncState& st, PlaneAt plane_at, BitWriter& bw) {
    const int n = st.n;
    const uint64_t x = plane_at(st.k);
    const uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
    const uint32_t yl = n < 32 ? fshr32(xl, xh, n) : (n < 64 ? xh >> (n & 31) : 0u);
    const uint32_t yh = n < 32 ? xh >> n : 0u;
    const int tz = yl ? ctz32nz(yl) : 32 + ctz32nz(yh | 0x80000000u);
    const bool implied = n + tz >= 63;
    const bool lastone = yl ? ((yl & (yl - 1u)) == 0u && yh == 0u) : ((yh & (yh - 1u)) == 0u);
    const int t1 = tz + 1;
    const uint64_t vB = implied ? 1ull : (1ull | (1ull << (t1 & 63)));
    const int lenB = implied ? tz + 1 : tz + 2 + (lastone ? 1 : 0);
    const bool doneB = implied || lastone;
    const int nB = implied ? 64 : n + t1;
    const bool yz = (yl | yh) == 0u;
    const bool ip = st.inplane;
    const bool unit = ip || (!yz && n < 64);         // (!ip: a plane start)
    const uint64_t vA = ((uint64_t)(xh & bmask32(n - 32)) << 32) | (xl & bmask32(n));
    const int sh = ip ? 0 : (n & 63);                 // the unit's bits follow the head's
    const uint64_t v = (ip ? 0ull : vA) | (unit ? (vB << sh) : 0ull);
    const int len = (ip ? 0 : n) + (unit ? lenB : (n < 64 ? 1 : 0));
    emit<true>(bw, v, len, st.bits);
    const bool done = unit ? doneB : true;
    st.n = unit ? nB : n;
    st.k -= done ? 1 : 0;
    st.inplane = !done;
}

// ---------------------------------------------------------------- lean encoder
// 64-bit shifts with PTX's clamping (an amount >= 64 gives 0): one SHF pair,
// no select for the edge cases.
ZB_HD uint64_t shl64c(uint64_t v, int s) {
#if defined(__CUDA_ARCH__)
    uint64_t r;
    asm("shl.b64 %0, %1, %2;" : "=l"(r) : "l"(v), "r"(s));
    return r;
#else
    return s >= 64 ? 0ull : v << s;
#endif
}
ZB_HD uint64_t shr64c(uint64_t v, int s) {
#if defined(__CUDA_ARCH__)
    uint64_t r;
    asm("shr.b64 %0, %1, %2;" : "=l"(r) : "l"(v), "r"(s));
    return r;
#else
    return s >= 64 ? 0ull : v >> s;
#endif
}
// a + b on the FMA pipe: an IMAD whose multiplier is a constant-bank word
// ptxas cannot fold (so it does not turn it back into an IADD3).  The decoder's
// event loop is bound by the integer ALU pipe while the FMA pipe has room
// (ncu: ALU 78 %, FMA 27 %): its additions go there (ALU-pipe instructions per
// event 53 -> 47; decode64 288.8 -> 283.5 us, fp32 decode within the noise; the
// same in the encoder's loop measured no faster: tools/ab_fma_adds.sh,
// profiles/r02_ab_fma_adds.txt).  OOCZ_FMA_ADDS=0 gives plain additions.
#ifndef OOCZ_FMA_ADDS
#define OOCZ_FMA_ADDS 1
#endif
#if defined(__CUDACC__)
static __constant__ int zb_one = 1;
#endif
ZB_HD int addf(int a, int b) {
#if defined(__CUDA_ARCH__) && OOCZ_FMA_ADDS
    int r;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(zb_one), "r"(b));
    return r;
#else
    return a + b;
#endif
}
// low min(m, 32) bits set for m >= 0: one BMSK
ZB_HD uint32_t bmask32p(int m) {
#if defined(__CUDA_ARCH__)
    uint32_t r;
    asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(r) : "r"(m));
    return r;
#else
    return m >= 32 ? ~0u : ((1u << m) - 1u);
#endif
}
// x >> s with PTX's clamping (s >= 32 gives 0), s >= 0
ZB_HD uint32_t shr32c(uint32_t x, int s) {
#if defined(__CUDA_ARCH__)
    uint32_t r;
    asm("shr.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s));
    return r;
#else
    return s >= 32 ? 0u : x >> s;
#endif
}
// low clamp(m, 0, 64) bits set: two BMSK
ZB_HD uint64_t bmask64(int m) { return ((uint64_t)bmask32(m - 32) << 32) | bmask32(m); }

// A thread's output stream as a row of words in shared memory.  Each emission
// writes the word being filled and the next one unconditionally (no branch, no
// global address arithmetic); the partial word is not kept in registers but
// read back from the row (an LDS instead of the selects that would track it),
// so the row must hold 0 at word 0 before the first put, and a 65-bit emission
// that ends exactly on a word boundary zeroes the word after (the only case
// where the next word was not just written).  The row needs two words of room
// past the last one kept; the caller copies the row out (coalesced).
struct RowWriter {
    uint64_t* row;
    int nb, w;        // bits [0, nb) of word w are written
    ZB_HD int pos() const { return 64 * w + nb; }
    // append the low len bits of v (len <= 65: bit 64 of a 65-bit emission is
    // the closing 0 flag; v has no bits at or above len)
    ZB_HD void put(uint64_t v, int len) {
        row[w] |= shl64c(v, nb);
        row[w + 1] = shr64c(v, 64 - nb);
        const int t = nb + len;
        if (t >= 128) row[w + 2] = 0ull;
        w += t >> 6;
        nb = t & 63;
    }
    // zero the words of [pos, 64 * words) not yet written
    ZB_HD void zero_tail(int words) {
        for (int i = w + (nb ? 1 : 0); i < words; i++) row[i] = 0ull;
    }
};

// The encoder as one flat loop of straight-line events with no budget test
// inside: the fixed-rate stream is a prefix of the unbounded one (zfp stops
// writing when the budget is spent and writes nothing else), so the loop
// emits until 64 * rate bits are out and the caller keeps the first rate
// words.  State: x = plane k at a plane start, else only its ones not yet
// coded (all at or above n); ip = inside plane k's group tests.  Each event
// is a head (plane start: the n verbatim bits) plus a unit:
//   ones left r = x & ~mask(n):
//     none      : the 0 group flag (when n < 64); plane done;
//     next at tz: flag 1, the tz - n zeros, the one (implied at 63: not sent),
//                 and the closing 0 flag when it was the last one (tz < 63).
// A plane start with new ones is merged with its first unit, so a plane with
// j >= 1 new ones takes j events (encode_event_merged's schedule, ~half the
// instructions: no both-alternatives select, no budget clamps, no global
// stores).
template <class PlaneAt>
ZB_HD void encode_planes_rows(PlaneAt plane_at, int top_plane, int limit, RowWriter& bw) {
    int k = top_plane, n = 0;
    uint32_t ipm = 0u;                                 // ~0 inside a plane's group tests
    uint64_t x = plane_at(k);
    const int wlimit = limit >> 6;                     // (limit is a whole number of words)
    while (k >= 0 && bw.w < wlimit) {
        const uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
        const uint32_t ml = bmask32p(n), mh = shr32c(~0u, 64 - n);
        // head (plane start only): x & mask(n); ones left: x & ~mask(n) (inside a
        // plane x holds no bit below n, so the same masking gives x)
        const uint64_t head = ((uint64_t)(xh & mh & ~ipm) << 32) | (xl & ml & ~ipm);
        const uint32_t rl = xl & ~ml, rh = xh & ~mh;
        const bool lnz = rl != 0u;
        const bool has = lnz || rh != 0u;
        const int tz = ctz32nz(lnz ? rl : (rh | 0x80000000u)) + (lnz ? 0 : 32);
        const uint64_t r = ((uint64_t)rh << 32) | rl;
        const uint64_t r2 = r & (r - 1ull);
        const bool last = r2 == 0ull;
        const bool implied = tz == 63;
        const int nsub = n & (int)ipm;                 // unit start: 0 at a plane start, n inside
        const int tz1 = tz + 1;
        const int onep = tz1 - nsub;             // position of the one in the emission
        const int fpos = has ? (n & ~(int)ipm) : 64;   // the 1 flag after the head (none: no bit)
        const int opos = (has && !implied) ? onep : 64;
        const uint64_t v = head | shl64c(1ull, fpos) | shl64c(1ull, opos);
        const int n1 = n + 1, lenu = onep + (implied ? 0 : (last ? 2 : 1));
        const int len = has ? lenu : (n < 64 ? n1 : 64);
        bw.put(v, len);
        const bool done = !has || last;
        n = has ? tz1 : n;
        k -= done ? 1 : 0;
        ipm = done ? 0u : ~0u;
        x = done ? plane_at(k & top_plane) : r2;      // (k = -1 reads a valid plane, unused)
    }
}

template <class PlaneAt>
ZB_HD void encode_planes(PlaneAt plane_at, int bits, BitWriter& bw, int top_plane = 31) {
    EncState st{top_plane, 0, bits, false};
    // no event emits more than 65 bits: while that many are left, no budget cut
    while (st.k >= 0 && st.bits >= 65) encode_event_merged(st, plane_at, bw);
    while (st.active()) encode_event(st, plane_at, bw);
}

// One decoder event on a 64-bit window wl:wh of the stream (three 32-bit
// words funnel-shifted: no 64-bit shifts, no predication):
//   plane start : n verbatim bits, then the first group flag;
//   found one   : the zero run -- r = ctz(w | ~0 << L) is the distance to the
//                 next one, or L when there is none within the L = min(63 - n,
//                 budget) scan bits -- the deposit at n + r (found, implied at 63,
//                 or budget end: zfp's rule), then the next group flag.
struct DecState {
    int k, n, bits;
    bool inplane;
    uint32_t xlo, xhi;               // plane k being assembled
    ZB_HD bool active() const { return k >= 0 && (bits > 0 || inplane); }
};

// FAST: the caller guarantees bits >= 66 (an event consumes at most 65), so
// every budget clamp below is the identity; the plane being assembled is then
// stored on every event (plane_set is an unconditional shared-memory store:
// the last store of plane k is its final value), with no branch.
template <bool FAST = false, class PlaneSet>
ZB_HD void decode_event(DecState& st, BitReader& br, PlaneSet plane_set) {
    const int n = st.n, bits = FAST ? 1 << 20 : st.bits;
    const uint32_t* p32 = reinterpret_cast<const uint32_t*>(br.p) + (br.pos >> 5);
    const int o = br.pos & 31;
    const uint32_t w0 = p32[0], w1 = p32[1], w2 = p32[2];
    const uint32_t wl = fshr32(w0, w1, o), wh = fshr32(w1, w2, o);
    // plane start
    const int mA = n < bits ? n : bits;
    const uint32_t aLo = wl & bmask32(mA), aHi = wh & bmask32(mA - 32);
    const uint32_t fA = (uint32_t)(n < 64) & (uint32_t)(bits > mA);   // a flag follows
    const uint32_t contA = fA & bit64(wl, wh, mA & 63);               // (no short-circuit branch)
    const int cA = mA + (int)fA;
    // found one
    const int L = 63 - n < bits ? 63 - n : bits;
    const uint32_t tLo = wl | ~bmask32(L), tHi = wh | ~bmask32(L - 32);
    const int r = tLo ? ctz32nz(tLo) : 32 + ctz32nz(tHi | 0x80000000u);
    const int c0 = r + (r < L ? 1 : 0);
    const int nB = n + r;
    const uint32_t bLo = st.xlo | (nB < 32 ? 1u << (nB & 31) : 0u);
    const uint32_t bHi = st.xhi | (nB >= 32 ? 1u << (nB & 31) : 0u);
    const uint32_t fB = (uint32_t)(nB < 63) & (uint32_t)(bits > c0);
    const uint32_t contB = fB & bit64(wl, wh, c0 & 63);
    const int cB = c0 + (int)fB;
    // select
    const bool ip = st.inplane;
    st.xlo = ip ? bLo : aLo;
    st.xhi = ip ? bHi : aHi;
    const int c = ip ? cB : cA;
    const bool cont = (ip ? contB : contA) != 0u;
    st.n = ip ? nB + 1 : n;
    br.pos += c;
    st.bits -= c;
    if (FAST) {
        plane_set(st.k, ((uint64_t)st.xhi << 32) | st.xlo);
        st.k -= cont ? 0 : 1;
    } else if (!cont) {
        plane_set(st.k, ((uint64_t)st.xhi << 32) | st.xlo);
        st.k -= 1;
    }
    st.inplane = cont;
}

// The FAST event written out without any budget term (the caller guarantees
// bits >= 66): same result as decode_event<true>, fewer instructions.
template <class PlaneSet>
ZB_HD void decode_event_fast(DecState& st, BitReader& br, PlaneSet plane_set) {
    const int n = st.n;
    const uint32_t* p32 = reinterpret_cast<const uint32_t*>(br.p) + (br.pos >> 5);
    const int o = br.pos & 31;
    const uint32_t w0 = p32[0], w1 = p32[1], w2 = p32[2];
    const uint32_t wl = fshr32(w0, w1, o), wh = fshr32(w1, w2, o);
    // plane start: the n (<= 64) verbatim bits, then a group flag unless n == 64
    const uint32_t aLo = wl & bmask32(n), aHi = wh & bmask32(n > 32 ? n - 32 : 0);
    const uint32_t fA = (uint32_t)(n < 64);
    const uint32_t contA = fA & bit64(wl, wh, n & 63);
    const int cA = n + (int)fA;
    // found one (n <= 63): r = length of the zero run, L = 63 - n if no one
    // follows within the scan (the one at 63 is then implied)
    const int L = 63 - n;
    const uint32_t tLo = wl | ~bmask32(L), tHi = wh | ~bmask32(L > 32 ? L - 32 : 0);
    const int r = tLo ? ctz32nz(tLo) : 32 + ctz32nz(tHi);
    const int c0 = r + (r < L ? 1 : 0);
    const int nB = n + r;
    const uint32_t one = 1u << (nB & 31);
    const uint32_t bLo = st.xlo | (nB < 32 ? one : 0u);
    const uint32_t bHi = st.xhi | (nB >= 32 ? one : 0u);
    const uint32_t fB = (uint32_t)(nB < 63);
    const uint32_t contB = fB & bit64(wl, wh, c0 & 63);
    const int cB = c0 + (int)fB;
    // select
    const bool ip = st.inplane;
    st.xlo = ip ? bLo : aLo;
    st.xhi = ip ? bHi : aHi;
    const int c = ip ? cB : cA;
    const bool cont = (ip ? contB : contA) != 0u;
    st.n = ip ? nB + 1 : n;
    br.pos += c;
    st.bits -= c;
    plane_set(st.k, ((uint64_t)st.xhi << 32) | st.xlo);   // unconditional: the last store is final
    st.k -= cont ? 0 : 1;
    st.inplane = cont;
}

// The budget-free (bits >= 131) event that merges a plane start with the
// plane's first unit (the decoder's side of encode_event_merged): the head is
// read from the window at pos, the unit from a second window right after it.
template <class PlaneSet>
ZB_HD void decode_event_merged(DecState& st, BitReader& br, PlaneSet plane_set) {
    const int n = st.n;
    const bool ip = st.inplane;
    uint32_t wl, wh;
    br.window(wl, wh);
    // plane start: the n (<= 64) verbatim bits, then the group flag unless n == 64
    const uint32_t aLo = wl & bmask32(n), aHi = wh & bmask32(n > 32 ? n - 32 : 0);
    const uint32_t fA = (uint32_t)(n < 64);
    const uint32_t flagA = fA & bit64(wl, wh, n & 63);
    const int hl = ip ? 0 : n + (int)fA;
    const bool unit = ip || flagA != 0u;
    // a unit on the window after the head: zero run r < L, or none (r = L: the
    // one at 63 is implied), the deposit, the next flag
    uint32_t ul, uh;
    BitReader{br.p, br.pos + hl}.window(ul, uh);
    const int L = 63 - n;
    const uint32_t tLo = ul | ~bmask32(L), tHi = uh | ~bmask32(L > 32 ? L - 32 : 0);
    const int r = tLo ? ctz32nz(tLo) : 32 + ctz32nz(tHi | 0x80000000u);
    const int c0 = r + (r < L ? 1 : 0);
    const int nB = n + r;
    const uint32_t baseLo = ip ? st.xlo : aLo, baseHi = ip ? st.xhi : aHi;
    const uint32_t one = 1u << (nB & 31);
    const uint32_t bLo = baseLo | (nB < 32 ? one : 0u);
    const uint32_t bHi = baseHi | (nB >= 32 ? one : 0u);
    const uint32_t fB = (uint32_t)(nB < 63);
    const uint32_t contB = fB & bit64(ul, uh, c0 & 63);
    const int cB = c0 + (int)fB;
    st.xlo = unit ? bLo : aLo;
    st.xhi = unit ? bHi : aHi;
    const bool cont = unit && contB != 0u;
    st.n = unit ? nB + 1 : n;
    const int c = hl + (unit ? cB : 0);
    br.pos += c;
    st.bits -= c;
    plane_set(st.k, ((uint64_t)st.xhi << 32) | st.xlo);   // unconditional: the last store is final
    st.k -= cont ? 0 : 1;
    st.inplane = cont;
}

// The decoder as one flat loop of merged events with a single budget term.
// The stream must be followed by >= 3 zero words past the limit (64 * rate
// bits incl. the header).  Reading past the budget then reproduces zfp's
// truncation everywhere but in one place: verbatim bits and group flags past
// the budget read as 0 (zfp leaves those bits 0 and stops), and the one place
// that differs -- a zero-run scan cut by the budget, after which zfp deposits
// the one where the budget ended -- is the scan length clamp L = min(63 - n,
// limit - u0).  The loop ends once the position reaches the limit; the planes
// not reached stay 0 (the caller's).  Event (state: plane k being assembled in
// xl:xh, n, ipm = ~0 inside the plane's group tests):
//   plane start : the n verbatim bits, then the group flag (n < 64);
//   unit        : (in-plane, or after a 1 flag) the zero run r <= L from u0,
//                 the deposit at n + r, then the next flag unless n + r == 63.
struct PadDecState {
    int k, n, pos;
    uint32_t ipm, xl, xh;
};

// planes k >= kmin (resumable: the fp64 decoder runs it in two halves)
template <class PlaneSet>
ZB_HD void decode_planes_padded(PadDecState& st, int kmin, PlaneSet plane_set, int limit, const uint32_t* p32) {
    int k = st.k, n = st.n, pos = st.pos;
    uint32_t ipm = st.ipm, xl = st.xl, xh = st.xh;
    // (a 1 flag that is the budget's last bit still gets its deposit: zfp's
    // scan reads nothing and puts the one at n, the event below with L = 0)
    while (k >= kmin && (pos < limit || ipm != 0u)) {
        const uint32_t* q = p32 + (pos >> 5);
        const int o = pos & 31;
        const uint64_t W = ((uint64_t)fshr32(q[1], q[2], o) << 32) | fshr32(q[0], q[1], o);
        const uint64_t head = W & (((uint64_t)shr32c(~0u, addf(-n, 64)) << 32) | bmask32p(n));
        const uint32_t fA = (uint32_t)(n < 64);
        const uint32_t flagA = fA & (uint32_t)(W >> (n & 63));    // (bit 0 only)
        const bool unit = ipm != 0u || (flagA & 1u) != 0u;
        const int u0 = addf(pos, addf(n, (int)fA) & ~(int)ipm);   // after the head and its flag
        // the unit's window: inside a plane it starts at pos (the window above);
        // at a plane start after the head (predicated loads: no shared-memory
        // wavefronts for the lanes that are inside a plane)
        uint64_t U = W;
        if (ipm == 0u) {
            const uint32_t* qu = p32 + (u0 >> 5);
            const int ou = u0 & 31;
            U = ((uint64_t)fshr32(qu[1], qu[2], ou) << 32) | fshr32(qu[0], qu[1], ou);
        }
        const int rem = limit - u0;
        const int L = 63 - n < rem ? 63 - n : rem;                   // (>= 0 whenever unit)
        const uint32_t tLo = (uint32_t)U | ~bmask32p(L), tHi = (uint32_t)(U >> 32) | ~shr32c(~0u, addf(-L, 64));
        const int r = addf(ctz32nz(tLo ? tLo : tHi), tLo ? 0 : 32);  // (bit 63 of ~mask(L) is set)
        const int c0 = addf(r, r < L ? 1 : 0);
        const int nB = addf(n, r);                                   // <= 63
        const uint64_t x = ipm ? (((uint64_t)xh << 32) | xl) : head;
        const uint64_t b = x | (1ull << nB);
        const uint32_t fB = (uint32_t)(nB < 63);
        const uint32_t contB = fB & (uint32_t)(U >> (c0 & 63));     // (bit 0 only)
        const uint64_t xn = unit ? b : head;
        xl = (uint32_t)xn;
        xh = (uint32_t)(xn >> 32);
        const bool cont = unit && (contB & 1u) != 0u;
        const int nB1 = addf(nB, 1), pn = addf(u0, addf(c0, (int)fB));
        n = unit ? nB1 : n;
        pos = unit ? pn : u0;
        plane_set(k, xn);                          // unconditional: the last store of plane k is final
        k = addf(k, cont ? 0 : -1);
        ipm = cont ? ~0u : 0u;
    }
    for (; k >= kmin; --k) plane_set(k, 0ull);
    st = PadDecState{k, n, pos, ipm, xl, xh};
}

template <class PlaneSet>
ZB_HD void decode_planes_padded(PlaneSet plane_set, int top_plane, int limit, int pos, const uint32_t* p32) {
    PadDecState st{top_plane, 0, pos, 0u, 0u, 0u};
    decode_planes_padded(st, 0, plane_set, limit, p32);
}

template <class PlaneSet>
ZB_HD void decode_planes(PlaneSet plane_set, int bits, BitReader& br, int top_plane = 31) {
    DecState st{top_plane, 0, bits, false, 0u, 0u};
    while (st.k >= 0 && st.bits >= 131) decode_event_merged(st, br, plane_set);
    while (st.k >= 0 && st.bits >= 66) decode_event_fast(st, br, plane_set);
    while (st.active()) decode_event(st, br, plane_set);
    for (int k = st.k; k >= 0; --k) plane_set(k, 0ull);
}

}  // namespace zb
}  // namespace oocz
