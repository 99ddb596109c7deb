// engine.cu -- out-of-core sweep engine behind the C ABI (include/oocz.h).
//
// The paper's method (PAPER.md:112-113 Sec. III, :130-179 Sec. V):
//  * the datasets are split along z into blocks of P planes that are streamed
//    host -> GPU -> host; each residency advances T steps (temporal blocking,
//    halo h = 4T);
//  * contiguous blocks share their common region C_i = [(i+1)P-h, (i+1)P+h) on
//    the GPU (region sharing, Fig. 3), so each plane crosses the host link once
//    per direction per sweep;
//  * remainders and common regions are compressed separately (Fig. 4): with
//    h a multiple of 4, every region boundary is a ZFP block-row boundary, so
//    the per-field store is one fixed-rate stream of 4-plane block-rows and any
//    region is one contiguous byte range.  Block i reads [iP+h, (i+1)P+h)
//    (block 0: [0, P+h)) and writes back its own planes [iP, (i+1)P), which
//    are exactly "the i-th remainder and the (i-1)-th common region" halves it
//    owns (reading R13);
//  * the time-t copy of C_i is kept on the GPU for block i+1 (reading R14);
//  * temporal blocking (beyond the paper, reading R26): parallelogram tiles --
//    in an ascending sweep block i > 0 updates [iP + 4(ts-s), (i+1)P + 4(ts-s))
//    in step s and takes the strip [iP-4, iP+4ts-4) at its last two time levels
//    from block i-1 (descending sweeps mirror it) -- so every cell is updated
//    once per step instead of the paper's trapezoid cone [iP-h+4s, (i+1)P+h-4s);
//  * copies, codec and stencil overlap on CUDA streams (Fig. 5): h2d, decode,
//    compute (stencil), encode, d2h.  Blocks rotate through `slab_sets` slab
//    sets, so the decode of block i+1 and the encode of block i-1 (integer-ALU
//    bound) run while block i's stencil (HBM bound) does.  One set serialises
//    decode -> stencil -> encode on the device (the copies still overlap) and
//    is for grids whose compressed store nearly fills HBM.
//
// Device-side data layout (per rank):
//   slab[s][f]: `slab_sets` sets (blocks rotate through them; default 2) of
//               (P + 2h) planes of nx*ny fp32,
//               slab plane 0 = rank plane iP - h
//   ccopy[f]  : 2h planes, time-t copy of C_i (u, u-, m); with parallelogram
//               tiles only its upper h planes for u, u-
//   pcopy[2]  : h planes of u, u-: the parallelogram strip for block i+1
//   in[slot]  : H2D staging of one read unit (3 fields), `slots` deep
//   out[slot] : D2H staging of one write unit (2 read-write fields)
//   store[f]  : pinned host (OOCZ_STORE_HOST) or device (OOCZ_STORE_DEVICE)
//               stream of S/4 block-rows
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include <sys/mman.h>

#include "common.cuh"
#include "halo.h"

static cudaError_t pinned_alloc(void** out, size_t bytes, unsigned flags);   // (below, with oocz_host_alloc)
static void pinned_free(void* p);

namespace oocz {

static std::atomic<uint64_t> g_launches{0};
void note_launches(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static thread_local std::string g_stateless_err;
oocz_status stateless_status(cudaError_t e, const char* what)
{
    if (e == cudaSuccess) return OOCZ_OK;
    g_stateless_err = std::string(what) + ": " + cudaGetErrorString(e);
    return OOCZ_ECUDA;
}

namespace {

__global__ void scan_field_kernel(const float* __restrict__ in, size_t n, unsigned int* flags)
{
    unsigned int nonfinite = 0, neg = 0, mx = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const unsigned int b = __float_as_uint(in[i]);
        const unsigned int a = b & 0x7fffffffu;
        nonfinite |= a >= 0x7f800000u;
        neg |= (b >> 31) && a;                // negative and not -0.0
        mx = max(mx, a);
    }
    nonfinite = __reduce_or_sync(0xffffffffu, nonfinite);
    neg = __reduce_or_sync(0xffffffffu, neg);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) {
        if (nonfinite) atomicOr(&flags[0], 1u);
        if (neg) atomicOr(&flags[0], 2u);
        atomicMax(&flags[1], mx);
    }
}

__global__ void scan_field64_kernel(const double* __restrict__ in, size_t n, unsigned int* flags,
                                    unsigned long long* mx64)
{
    unsigned int nonfinite = 0, neg = 0;
    unsigned long long mx = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(in[i]);
        const unsigned long long a = b & 0x7fffffffffffffffull;
        nonfinite |= a >= 0x7ff0000000000000ull;
        neg |= (b >> 63) && a;
        mx = max(mx, a);
    }
    nonfinite = __reduce_or_sync(0xffffffffu, nonfinite);
    neg = __reduce_or_sync(0xffffffffu, neg);
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) {
        if (nonfinite) atomicOr(&flags[0], 1u);
        if (neg) atomicOr(&flags[0], 2u);
        atomicMax(mx64, mx);
    }
}

}  // namespace

cudaError_t launch_scan_field(const double* in, size_t n, unsigned int* flags, unsigned long long* mx64,
                              cudaStream_t s)
{
    if (n == 0) return cudaSuccess;
    size_t blocks = std::min<size_t>((n + 255) / 256, (size_t)kNumSMs * 8);
    scan_field64_kernel<<<(unsigned)blocks, 256, 0, s>>>(in, n, flags, mx64);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_scan_field(const float* in, size_t n, unsigned int* flags, cudaStream_t s)
{
    if (n == 0) return cudaSuccess;
    size_t blocks = std::min<size_t>((n + 255) / 256, (size_t)kNumSMs * 8);
    scan_field_kernel<<<(unsigned)blocks, 256, 0, s>>>(in, n, flags);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace oocz

using namespace oocz;

// ------------------------------------------------------------------ context
#ifndef OOCZ_IN_SLOTS
#define OOCZ_IN_SLOTS 3
#endif
static constexpr int kInSlots = OOCZ_IN_SLOTS;   // input staging slots at most (host store)

struct Geom {
    int rd0, rd1;      // read unit, rank-local planes
    int own0, own1;    // write unit
    int slab0;         // rank-local plane of slab plane 0 (= iP - h)
    int vlo, vhi;      // slab planes holding data (others read as zero ghost)
};

struct oocz_ctx {
    oocz_config cfg{};
    int rank = 0, world = 1, device = 0;
    int S = 0, P = 0, D = 0, h = 0, T = 0, L = 0;   // slab planes, block, blocks, halo, depth, slab len
    int nx = 0, ny = 0;
    int esz = 4;                            // element size: 4 (precision 32) or 8 (precision 64)
    size_t plane_elems = 0, pb = 0;         // elements / bytes per plane
    size_t row_bytes[3] = {0, 0, 0};       // bytes per 4-plane block-row in the store
    bool field_set[3] = {false, false, false};
    std::vector<uint8_t> rows_set[3];       // 4-plane rows of each field set so far
    bool poisoned = false;
    std::string err;

    std::vector<Geom> geom;
    // device buffers
    // (byte pointers: fp32 or fp64 planes of pb bytes)
    static constexpr int kMaxSets = 4;
    int nsets = 2;                          // slab sets in rotation (cfg.slab_sets, default 2)
    uint8_t* slab[kMaxSets][3] = {};
    uint8_t* ccopy[3] = {nullptr, nullptr, nullptr};
    uint8_t* pcopy[2] = {nullptr, nullptr};  // parallelogram strip of u, u- for the next block
    bool para = false;                      // parallelogram tiles (reading R26)
    int cbase[3] = {0, 0, 0};               // first C plane ccopy[f] holds (h for u, u- with para)
    uint8_t* m_full = nullptr;              // m_resident: decoded m, planes [-h, S + h)
    std::vector<uint8_t*> in_slot, out_slot;
    size_t in_off[3] = {0, 0, 0}, out_off[2] = {0, 0};
    size_t in_slot_bytes = 0, out_slot_bytes = 0;
    unsigned int* d_flags = nullptr;        // two scan records (input, RT(m)): [0] flags, [1] fp32 max bits, [2..3] fp64 max bits
    // store
    // The stored rows of planes [0, zres) are in HBM (dstore), those of [zres, S) in
    // store: zres = S with OOCZ_STORE_DEVICE (dstore aliases store), K * P with
    // resident_blocks = K on a host store (a hybrid), 0 otherwise.  rows_ptr() maps.
    uint8_t* store[3] = {nullptr, nullptr, nullptr};
    uint8_t* dstore[3] = {nullptr, nullptr, nullptr};
    int zres[3] = {0, 0, 0};                // per field (m_hbm: m's whole stream in HBM)
    size_t store_bytes[3] = {0, 0, 0};
    bool store_external = false;            // host store carved from a caller-owned arena (oocz_create_ex)
    // streams / events
    cudaStream_t s_h2d = nullptr, s_dec = nullptr, s_comp = nullptr, s_enc = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_decoded[kMaxSets] = {}, ev_slab_free[kMaxSets] = {}, ev_stepped[kMaxSets] = {};
    cudaEvent_t ev_join_enc = nullptr;
    cudaEvent_t ev_join_dec = nullptr;
    std::vector<cudaEvent_t> ev_in_ready, ev_in_free, ev_out_ready, ev_out_free, ev_written, ev_encoded;
    long long seq = 0;                      // global block sequence number
    std::vector<int> last_slot;             // staging slot of each block's latest encode (host store)
    std::vector<long long> last_seq;        // ... and its block sequence number (-1: not in a slot)
    std::vector<uint8_t> kept;              // its latest rows are only in that slot (D2H skipped, R22)
    // halo exchange (world > 1)
    HaloComm* halo = nullptr;
    // profiling
    struct Prof { int sweep, block, stage, lane; cudaEvent_t a, b; uint64_t bytes; };
    std::vector<Prof> prof;
    std::vector<cudaEvent_t> ev_pool;       // timing events, reused across calls
    size_t ev_used = 0;
    cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr, ev_join_h2d = nullptr, ev_join_comp = nullptr;
    std::vector<oocz_event> events;
    oocz_stats stats{};
    // CUDA graphs (cfg.graphs): one executable graph per chunk length in steps
    struct Graph { cudaGraphExec_t exec; uint64_t launches; int sweeps; };
    std::map<int64_t, Graph> graph_cache;
    bool capturing = false;                 // inside a capture: slab sets by block index
    cudaEvent_t ev_g_fork = nullptr, ev_g_join[4] = {};
};

namespace {

oocz_status fail(oocz_ctx* c, oocz_status s, const char* fmt, ...) __attribute__((format(printf, 3, 4)));
oocz_status fail(oocz_ctx* c, oocz_status s, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) {
        c->err = buf;
        if (s == OOCZ_ECUDA || s == OOCZ_ENCCL) c->poisoned = true;
    }
    return s;
}

#define CK(call)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fail(ctx, OOCZ_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                            \
    } while (0)

size_t row_bytes_for(int nx, int ny, int rate, int esz)
{
    return rate == 0 ? (size_t)nx * ny * 4 * esz : (size_t)(nx / 4) * (ny / 4) * 8u * (size_t)rate;
}

int esz_of(const oocz_config* cfg) { return cfg->precision == 64 ? 8 : 4; }

template <class C>
double cfl_limit(const C c[5])
{
    // m_max = 4 / (3 max_theta |S(theta)|), S = c0 + 2 sum c_k cos(k theta) (R2)
    double mx = 0.0;
    const int N = 20000;
    for (int i = 0; i <= N; i++) {
        const double th = M_PI * i / N;
        double s = c[0];
        for (int k = 1; k <= 4; k++) s += 2.0 * c[k] * std::cos(k * th);
        mx = std::max(mx, std::fabs(s));
    }
    return mx > 0 ? 4.0 / (3.0 * mx) : INFINITY;
}

// one 4-aligned plane range of a field's store as a byte range
inline size_t rows_off(const oocz_ctx* c, int f, int plane) { return (size_t)(plane / 4) * c->row_bytes[f]; }
// where the stored rows from `plane` on live (a block's rows are all in one place)
inline bool rows_on_device(const oocz_ctx* c, int f, int plane) { return plane < c->zres[f]; }
inline uint8_t* rows_ptr(const oocz_ctx* c, int f, int plane)
{
    return plane < c->zres[f] ? c->dstore[f] + rows_off(c, f, plane)
                              : c->store[f] + (rows_off(c, f, plane) - rows_off(c, f, c->zres[f]));
}
// the end of a chunk of stored rows starting at plane z that stays in one place
inline int rows_chunk_end(const oocz_ctx* c, int f, int z, int end)
{
    return z < c->zres[f] ? std::min(end, c->zres[f]) : end;
}

cudaError_t encode_or_copy(oocz_ctx* c, int f, const uint8_t* src, int nplanes, uint8_t* dst, cudaStream_t s)
{
    return field_encode(src, c->esz, c->nx, c->ny, nplanes, c->cfg.rate[f], dst, s);
}

cudaError_t decode_or_copy(oocz_ctx* c, int f, const uint8_t* src, int nplanes, uint8_t* dst, cudaStream_t s)
{
    return field_decode(src, c->esz, c->nx, c->ny, nplanes, c->cfg.rate[f], dst, s);
}

// one cone-limited step in the context's precision
cudaError_t stencil_step(oocz_ctx* c, uint8_t* u, uint8_t* uprev, const uint8_t* m, int z0, int z1, int zv0,
                         int zv1, cudaStream_t s)
{
    if (c->esz == 8)
        return launch_stencil_step(reinterpret_cast<const double*>(u), reinterpret_cast<double*>(uprev),
                                   reinterpret_cast<const double*>(m), c->nx, c->ny, c->L, c->cfg.c64, z0, z1,
                                   zv0, zv1, s);
    return launch_stencil_step(reinterpret_cast<const float*>(u), reinterpret_cast<float*>(uprev),
                               reinterpret_cast<const float*>(m), c->nx, c->ny, c->L, c->cfg.c, z0, z1, zv0, zv1, s);
}

cudaEvent_t pool_event(oocz_ctx* c)
{
    if (c->ev_used == c->ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        c->ev_pool.push_back(e);
    }
    return c->ev_pool[c->ev_used++];
}

void prof_begin(oocz_ctx* c, int sweep, int block, int stage, int lane, cudaStream_t s, uint64_t bytes)
{
    if (!c->cfg.profile) return;
    oocz_ctx::Prof p{sweep, block, stage, lane, pool_event(c), pool_event(c), bytes};
    cudaEventRecord(p.a, s);
    c->prof.push_back(p);
}
void prof_end(oocz_ctx* c, cudaStream_t s)
{
    if (!c->cfg.profile) return;
    cudaEventRecord(c->prof.back().b, s);
}

}  // namespace

// ------------------------------------------------------------------ library
extern "C" int32_t oocz_abi_version(void) { return OOCZ_ABI_VERSION; }

extern "C" uint64_t oocz_kernel_launch_count(void) { return g_launches.load(); }

extern "C" const char* oocz_status_string(oocz_status s)
{
    switch (s) {
        case OOCZ_OK: return "ok";
        case OOCZ_EINVAL: return "invalid argument";
        case OOCZ_EALIGN: return "extent not a multiple of 4";
        case OOCZ_ECFL: return "stability (CFL) bound violated";
        case OOCZ_ECAPACITY: return "memory budget too small";
        case OOCZ_ENONFINITE: return "non-finite value in field";
        case OOCZ_ESTATE: return "invalid state";
        case OOCZ_ECUDA: return "CUDA error";
        case OOCZ_ENCCL: return "NCCL error";
    }
    return "unknown status";
}

extern "C" void oocz_default_config(oocz_config* cfg, int32_t nx, int32_t ny, int32_t nz)
{
    std::memset(cfg, 0, sizeof *cfg);
    cfg->nx = nx; cfg->ny = ny; cfg->nz = nz;
    cfg->c[0] = (float)(-205.0 / 72.0);
    cfg->c[1] = (float)(8.0 / 5.0);
    cfg->c[2] = (float)(-1.0 / 5.0);
    cfg->c[3] = (float)(8.0 / 315.0);
    cfg->c[4] = (float)(-1.0 / 560.0);
    cfg->c64[0] = -205.0 / 72.0;
    cfg->c64[1] = 8.0 / 5.0;
    cfg->c64[2] = -1.0 / 5.0;
    cfg->c64[3] = 8.0 / 315.0;
    cfg->c64[4] = -1.0 / 560.0;
    cfg->precision = 32;
    cfg->tb = 4;
    cfg->block_planes = nz;
    cfg->rate[0] = cfg->rate[1] = cfg->rate[2] = 16;
    cfg->store = OOCZ_STORE_HOST;
    cfg->slots = 2;
}

extern "C" double oocz_cfl_limit(const float c[5]) { return c ? cfl_limit(c) : 0.0; }
extern "C" double oocz_cfl_limit_f64(const double c[5]) { return c ? cfl_limit(c) : 0.0; }

extern "C" oocz_status oocz_validate(const oocz_config* cfg, int32_t world, char* msg, size_t msg_len)
{
    char buf[256] = "";
    oocz_status st = OOCZ_OK;
#define BAD(code, ...) do { snprintf(buf, sizeof buf, __VA_ARGS__); st = code; goto done; } while (0)
    if (!cfg) BAD(OOCZ_EINVAL, "null config");
    if (world < 1) BAD(OOCZ_EINVAL, "world (%d) < 1", world);
    if (cfg->nx <= 0 || cfg->ny <= 0 || cfg->nz <= 0)
        BAD(OOCZ_EINVAL, "extents must be positive (%d, %d, %d)", cfg->nx, cfg->ny, cfg->nz);
    if (cfg->nx % 4 || cfg->ny % 4 || cfg->nz % 4)
        BAD(OOCZ_EALIGN, "nx, ny, nz (%d, %d, %d) must be multiples of 4", cfg->nx, cfg->ny, cfg->nz);
    if (cfg->nz % world) BAD(OOCZ_EINVAL, "world (%d) does not divide nz (%d)", world, cfg->nz);
    {
        const int S = cfg->nz / world;
        if (S % 4) BAD(OOCZ_EALIGN, "nz/world (%d) must be a multiple of 4", S);
        if (cfg->tb < 1) BAD(OOCZ_EINVAL, "tb (%d) < 1", cfg->tb);
        const int h = 4 * cfg->tb;
        const int P = cfg->block_planes;
        if (P <= 0 || P % 4) BAD(OOCZ_EALIGN, "P (%d) must be a positive multiple of 4", P);
        if (P < 2 * h) BAD(OOCZ_EINVAL, "P (%d) < 2h (%d)", P, 2 * h);
        if (S % P) BAD(OOCZ_EINVAL, "P (%d) does not divide nz/world (%d)", P, S);
    }
    for (int f = 0; f < 3; f++)
        if (cfg->rate[f] < 0 || cfg->rate[f] > 64) BAD(OOCZ_EINVAL, "rate[%d] (%d) outside [0, 64]", f, cfg->rate[f]);
    if (cfg->store != OOCZ_STORE_HOST && cfg->store != OOCZ_STORE_DEVICE)
        BAD(OOCZ_EINVAL, "store (%d) unknown", cfg->store);
    if (cfg->store == OOCZ_STORE_HOST && cfg->slots < 2) BAD(OOCZ_EINVAL, "slots (%d) < 2", cfg->slots);
    if (cfg->slab_sets < 0 || cfg->slab_sets > 4)
        BAD(OOCZ_EINVAL, "slab_sets (%d) outside {0 (= 2), 1, 2, 3, 4}", cfg->slab_sets);
    if (cfg->graphs != 0 && cfg->graphs != 1) BAD(OOCZ_EINVAL, "graphs (%d) must be 0 or 1", cfg->graphs);
    if (cfg->cone != 0 && cfg->cone != 1) BAD(OOCZ_EINVAL, "cone (%d) must be 0 or 1", cfg->cone);
    if (cfg->resident_blocks < -1 || cfg->resident_blocks > cfg->nz / world / cfg->block_planes)
        BAD(OOCZ_EINVAL, "resident_blocks (%d) outside [-1 (auto), D = %d]", cfg->resident_blocks,
            cfg->nz / world / cfg->block_planes);
    if (cfg->m_hbm != 0 && cfg->m_hbm != 1) BAD(OOCZ_EINVAL, "m_hbm (%d) must be 0 or 1", cfg->m_hbm);
    if (cfg->m_hbm && cfg->store != OOCZ_STORE_HOST) BAD(OOCZ_EINVAL, "m_hbm needs store = OOCZ_STORE_HOST");
    if (cfg->resident_blocks != 0 && cfg->store != OOCZ_STORE_HOST)
        BAD(OOCZ_EINVAL, "resident_blocks (%d) needs store = OOCZ_STORE_HOST", cfg->resident_blocks);
    if (cfg->precision != 32 && cfg->precision != 64)
        BAD(OOCZ_EINVAL, "precision (%d) must be 32 or 64", cfg->precision);
    for (int k = 0; k < 5; k++)
        if (cfg->precision == 32 ? !std::isfinite(cfg->c[k]) : !std::isfinite(cfg->c64[k]))
            BAD(OOCZ_EINVAL, "c[%d] not finite", k);
#undef BAD
done:
    if (msg && msg_len) snprintf(msg, msg_len, "%s", buf);
    return st;
}

extern "C" oocz_status oocz_get_nccl_id(uint8_t id[128])
{
    return halo_get_unique_id(id) ? OOCZ_OK : OOCZ_ENCCL;
}

// bytes of one field's store, rounded up so that stores carved from one arena stay 4 KiB aligned
static size_t arena_field_bytes(size_t b) { return (b + 4095) / 4096 * 4096; }

#ifdef OOCZ_DEC_NOSTORE
namespace oocz { void zfp_ab_reset(); }
using oocz::zfp_ab_reset;
#endif
static oocz_status create_impl(const oocz_config* cfg, int32_t rank, int32_t world, const uint8_t* nccl_id,
                               int32_t device, HaloComm* preset_halo, uint8_t* arena, size_t arena_bytes,
                               oocz_ctx** out)
{
#ifdef OOCZ_DEC_NOSTORE
    zfp_ab_reset();   // A/B bound only (zfp.cu)
#endif
    if (!out) return OOCZ_EINVAL;
    *out = nullptr;
    char msg[256];
    oocz_status st = oocz_validate(cfg, world, msg, sizeof msg);
    if (st != OOCZ_OK) {
        fprintf(stderr, "oocz_create: %s\n", msg);
        return st;
    }
    if (rank < 0 || rank >= world || (world > 1 && !nccl_id && !preset_halo)) return OOCZ_EINVAL;
    oocz_ctx* ctx = new oocz_ctx;
    ctx->cfg = *cfg;
    ctx->rank = rank; ctx->world = world; ctx->device = device;
    ctx->nx = cfg->nx; ctx->ny = cfg->ny;
    ctx->S = cfg->nz / world;
    ctx->T = cfg->tb; ctx->h = 4 * cfg->tb; ctx->P = cfg->block_planes;
    ctx->D = ctx->S / ctx->P;
    for (int f = 0; f < 3; f++) ctx->rows_set[f].assign(ctx->S / 4, 0);
    ctx->L = ctx->P + 2 * ctx->h;
    ctx->plane_elems = (size_t)cfg->nx * cfg->ny;
    ctx->nsets = cfg->slab_sets ? cfg->slab_sets : 2;
    ctx->esz = esz_of(cfg);
    ctx->pb = ctx->plane_elems * ctx->esz;
    for (int f = 0; f < 3; f++) ctx->row_bytes[f] = row_bytes_for(cfg->nx, cfg->ny, cfg->rate[f], ctx->esz);

    auto cleanup_fail = [&](oocz_status s) { oocz_destroy(ctx); return s; };
#define CKC(call)                                                                                 \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) {                                                                  \
            fprintf(stderr, "oocz_create: %s: %s\n", #call, cudaGetErrorString(e_));              \
            return cleanup_fail(e_ == cudaErrorMemoryAllocation ? OOCZ_ECAPACITY : OOCZ_ECUDA);   \
        }                                                                                         \
    } while (0)

    CKC(cudaSetDevice(device));
    // block geometry (rank-local planes)
    const int S = ctx->S, P = ctx->P, h = ctx->h, D = ctx->D;
    const bool has_up = rank > 0, has_down = rank < world - 1;
    for (int i = 0; i < D; i++) {
        Geom g;
        g.slab0 = i * P - h;
        g.rd0 = i == 0 ? 0 : i * P + h;
        g.rd1 = std::min((i + 1) * P + h, S);
        g.own0 = i * P;
        g.own1 = (i + 1) * P;
        const int lo = (i == 0 && !has_up) ? 0 : i * P - h;
        const int hi = (i == D - 1 && !has_down) ? S : (i + 1) * P + h;
        g.vlo = lo - g.slab0;
        g.vhi = hi - g.slab0;
        ctx->geom.push_back(g);
    }
    // memory plan and budget check
    const size_t pb = ctx->pb;
    // slab sets (m is not streamed into them when it is resident) + the C_i copy
    const int slab_fields = cfg->m_resident ? 2 : 3;    // also the streamed fields
    // cfg->cone = 1: the paper's trapezoid cone on every block;
    // 0: parallelogram tiles (reading R26).  Same bits either way.
    ctx->para = cfg->cone == 0;
    // with parallelogram tiles and ascending sweeps only, only C planes
    // [h + 4ts - 4, 2h) of u, u- are kept (descending sweeps need [0, h - 4ts + 4))
    for (int f = 0; f < 2; f++) ctx->cbase[f] = ctx->para && !cfg->serpentine ? h : 0;
    size_t need = (size_t)ctx->nsets * slab_fields * (size_t)ctx->L * pb;
    for (int f = 0; f < slab_fields; f++) need += (size_t)(2 * h - ctx->cbase[f]) * pb;
    if (ctx->para) need += 2 * (size_t)h * pb;   // pcopy
    const bool host = cfg->store == OOCZ_STORE_HOST;
    const int rd_max_planes = std::min(P + h, S);
    if (host) {
        // an input slot holds one read unit of each streamed field; set_field /
        // get_field also stage P planes of any one field through slot 0
        size_t one_field = 0;
        for (int f = 0; f < slab_fields; f++) {
            if (f == OOCZ_M && cfg->m_hbm) continue;          // m's rows are read in HBM
            ctx->in_off[f] = ctx->in_slot_bytes;
            ctx->in_slot_bytes += (size_t)(rd_max_planes / 4) * ctx->row_bytes[f];
        }
        for (int f = 0; f < 3; f++) one_field = std::max(one_field, (size_t)(P / 4) * ctx->row_bytes[f]);
        ctx->in_slot_bytes = std::max(ctx->in_slot_bytes, one_field);
        for (int f = 0; f < 2; f++) {
            ctx->out_off[f] = ctx->out_slot_bytes;
            ctx->out_slot_bytes += (size_t)(P / 4) * ctx->row_bytes[f];
        }
        // staging: `slots` output slots (their depth is what keeps recently encoded
        // rows on the device, R22) and at most kInSlots input slots (H2D runs that far
        // ahead of the decode)
        need += (size_t)std::min(cfg->slots, kInSlots) * ctx->in_slot_bytes + (size_t)cfg->slots * ctx->out_slot_bytes;
    }
    for (int f = 0; f < 3; f++) ctx->store_bytes[f] = (size_t)(S / 4) * ctx->row_bytes[f];
    if (world > 1) need += halo_device_bytes(ctx->plane_elems, h, cfg->rate, ctx->row_bytes);
    if (cfg->m_resident) need += (size_t)(S + 2 * h) * pb;
    {
        size_t fr = 0, tot = 0;
        CKC(cudaMemGetInfo(&fr, &tot));
        const size_t budget = cfg->device_bytes ? cfg->device_bytes : fr;
        int K = cfg->resident_blocks;
        const bool m_hbm = host && cfg->m_hbm;
        if (m_hbm) need += rows_off(ctx, OOCZ_M, S);        // m's whole compressed stream in HBM
        if (host && K < 0) {    // auto: as many leading blocks as the budget leaves room for
            size_t per = 0;
            for (int f = 0; f < 3; f++)
                if (!(m_hbm && f == OOCZ_M)) per += rows_off(ctx, f, P);
            K = budget > need ? (int)std::min<size_t>((size_t)D, (budget - need) / std::max<size_t>(per, 1)) : 0;
            ctx->cfg.resident_blocks = K;
        }
        for (int f = 0; f < 3; f++) {
            ctx->zres[f] = host ? std::min(std::max(K, 0) * P, S) : S;
            if (m_hbm && f == OOCZ_M) ctx->zres[f] = S;
            else need += rows_off(ctx, f, ctx->zres[f]);   // the rows kept in HBM
        }
        if (need > budget) {
            fprintf(stderr, "oocz_create: device memory %zu B needed > budget %zu B\n", need, budget);
            return cleanup_fail(OOCZ_ECAPACITY);
        }
    }
    for (int f = 0; f < 3; f++) {
        for (int k = 0; k < ctx->nsets && f < slab_fields; k++) {
            CKC(cudaMalloc(&ctx->slab[k][f], (size_t)ctx->L * pb));
            CKC(cudaMemset(ctx->slab[k][f], 0, (size_t)ctx->L * pb));
        }
        if (f < slab_fields) CKC(cudaMalloc(&ctx->ccopy[f], (size_t)(2 * h - ctx->cbase[f]) * pb));
    }
    if (ctx->para)
        for (auto& q : ctx->pcopy) CKC(cudaMalloc(&q, (size_t)h * pb));
    CKC(cudaMalloc(&ctx->d_flags, 8 * sizeof(unsigned int)));
    if (cfg->m_resident) {
        CKC(cudaMalloc(&ctx->m_full, (size_t)(S + 2 * h) * pb));
        CKC(cudaMemset(ctx->m_full, 0, (size_t)(S + 2 * h) * pb));
    }
    if (host) {
        for (int s = 0; s < cfg->slots; s++) {
            uint8_t* a = nullptr;
            uint8_t* b = nullptr;
            if (s < kInSlots) {
                CKC(cudaMalloc(&a, ctx->in_slot_bytes));
                ctx->in_slot.push_back(a);
            }
            CKC(cudaMalloc(&b, ctx->out_slot_bytes));
            ctx->out_slot.push_back(b);
        }
        for (int f = 0; f < 3; f++)
            if (ctx->zres[f] > 0) CKC(cudaMalloc(&ctx->dstore[f], std::max<size_t>(rows_off(ctx, f, ctx->zres[f]), 1)));
        auto host_part = [&](int f) { return ctx->store_bytes[f] - rows_off(ctx, f, ctx->zres[f]); };
        if (arena) {
            size_t want = 0;
            for (int f = 0; f < 3; f++) want += arena_field_bytes(host_part(f));
            cudaPointerAttributes pa{};
            CKC(cudaPointerGetAttributes(&pa, arena));
            if (pa.type != cudaMemoryTypeHost) {
                fprintf(stderr, "oocz_create_ex: the arena is not pinned host memory\n");
                return cleanup_fail(OOCZ_EINVAL);
            }
            if (arena_bytes < want) {
                fprintf(stderr, "oocz_create_ex: arena %zu B < %zu B needed\n", arena_bytes, want);
                return cleanup_fail(OOCZ_ECAPACITY);
            }
            ctx->store_external = true;
            for (int f = 0; f < 3; f++) {
                ctx->store[f] = arena;
                arena += arena_field_bytes(host_part(f));
            }
        } else {
            for (int f = 0; f < 3; f++) {
                CKC(pinned_alloc(reinterpret_cast<void**>(&ctx->store[f]), std::max<size_t>(host_part(f), 1),
                                 cudaHostAllocDefault));
                ctx->stats.host_bytes_pinned += host_part(f);
            }
        }
    } else {
        for (int f = 0; f < 3; f++) {
            CKC(cudaMalloc(&ctx->store[f], std::max<size_t>(ctx->store_bytes[f], 1)));
            ctx->dstore[f] = ctx->store[f];
        }
    }
    ctx->stats.device_bytes_used = need;
    CKC(cudaStreamCreateWithFlags(&ctx->s_h2d, cudaStreamNonBlocking));
    {
        // Equal priorities.  Giving the compute stream (stencil, encode) the higher
        // priority ran the in-step stencil at 5.2 instead of 4.3 TB/s but slowed the
        // decodes more: 121 vs 124.5 G cell-updates/s over the sweep (A/B, tools/ab_prio.sh).
        // OOCZ_STREAM_PRIORITY=1 turns it on for experiments.
        int lo = 0, hi = 0;
        const char* sp = getenv("OOCZ_STREAM_PRIORITY");
        if (sp && sp[0] == '1') CKC(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CKC(cudaStreamCreateWithPriority(&ctx->s_comp, cudaStreamNonBlocking, hi));
        CKC(cudaStreamCreateWithPriority(&ctx->s_dec, cudaStreamNonBlocking, lo));
        // The encode has its own stream, so the next block's stencil overlaps this
        // block's encode (+1.5 %).  (-DOOCZ_ENCODE_ON_COMPUTE puts it back on the
        // compute stream; the rare wrong results first blamed on this stream were
        // a ring-slot race in the stencil, see stencil.cu "release discipline".)
#ifdef OOCZ_ENCODE_ON_COMPUTE
        ctx->s_enc = ctx->s_comp;
#else
        CKC(cudaStreamCreateWithPriority(&ctx->s_enc, cudaStreamNonBlocking, lo));
#endif
    }
    for (int k = 0; k < ctx->nsets; k++) {
        CKC(cudaEventCreateWithFlags(&ctx->ev_decoded[k], cudaEventDisableTiming));
        CKC(cudaEventCreateWithFlags(&ctx->ev_slab_free[k], cudaEventDisableTiming));
        CKC(cudaEventCreateWithFlags(&ctx->ev_stepped[k], cudaEventDisableTiming));
    }
    CKC(cudaEventCreateWithFlags(&ctx->ev_join_enc, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&ctx->ev_join_dec, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&ctx->ev_g_fork, cudaEventDisableTiming));
    for (auto& e : ctx->ev_g_join) CKC(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CKC(cudaStreamCreateWithFlags(&ctx->s_d2h, cudaStreamNonBlocking));
    const int nslots = host ? cfg->slots : 1;
    auto mk = [&](std::vector<cudaEvent_t>& v, int n) -> cudaError_t {
        for (int k = 0; k < n; k++) {
            cudaEvent_t e;
            cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            if (r != cudaSuccess) return r;
            v.push_back(e);
        }
        return cudaSuccess;
    };
    CKC(mk(ctx->ev_in_ready, std::min(nslots, kInSlots)));
    CKC(mk(ctx->ev_in_free, std::min(nslots, kInSlots)));
    CKC(mk(ctx->ev_out_ready, nslots));
    CKC(mk(ctx->ev_out_free, nslots));
    CKC(mk(ctx->ev_written, D));
    CKC(mk(ctx->ev_encoded, D));
    ctx->last_slot.assign(D, 0);
    ctx->last_seq.assign(D, -1);
    ctx->kept.assign(D, 0);
    CKC(cudaEventCreate(&ctx->ev_t0));
    CKC(cudaEventCreate(&ctx->ev_t1));
    CKC(cudaEventCreateWithFlags(&ctx->ev_join_h2d, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&ctx->ev_join_comp, cudaEventDisableTiming));
    if (preset_halo) {
        ctx->halo = preset_halo;
    } else if (world > 1) {
        std::string herr;
        ctx->halo = halo_create(rank, world, nccl_id, device, ctx->plane_elems, ctx->esz, h, cfg->rate,
                                ctx->row_bytes, &herr);
        if (!ctx->halo) {
            fprintf(stderr, "oocz_create: %s\n", herr.c_str());
            return cleanup_fail(OOCZ_ENCCL);
        }
    }
#undef CKC
    *out = ctx;
    return OOCZ_OK;
}

extern "C" oocz_status oocz_create(const oocz_config* cfg, int32_t rank, int32_t world, const uint8_t* nccl_id,
                                   int32_t device, oocz_ctx** out)
{
    return create_impl(cfg, rank, world, nccl_id, device, nullptr, nullptr, 0, out);
}

extern "C" oocz_status oocz_create_ex(const oocz_config* cfg, int32_t rank, int32_t world, const uint8_t* nccl_id,
                                      int32_t device, void* host_arena, size_t arena_bytes, oocz_ctx** out)
{
    if (host_arena && cfg && cfg->store != OOCZ_STORE_HOST) return OOCZ_EINVAL;
    return create_impl(cfg, rank, world, nccl_id, device, nullptr, static_cast<uint8_t*>(host_arena), arena_bytes,
                       out);
}

extern "C" size_t oocz_host_store_bytes(const oocz_config* cfg, int32_t world)
{
    if (!cfg || world < 1 || cfg->nz % world) return 0;
    const int S = cfg->nz / world;
    // (auto, -1: the bytes for K = 0, an upper bound)
    const int zres = cfg->resident_blocks > 0 ? std::min(cfg->resident_blocks * cfg->block_planes, S) : 0;
    size_t t = 0;
    for (int f = 0; f < 3; f++)
        t += arena_field_bytes((size_t)((S - (cfg->m_hbm && f == OOCZ_M ? S : zres)) / 4) *
                               row_bytes_for(cfg->nx, cfg->ny, cfg->rate[f], esz_of(cfg)));
    return t;
}

// Pinned host memory.  Large buffers (>= 1 GiB: the compressed stores) are an
// anonymous mapping advised to transparent huge pages and registered with
// cudaHostRegister: pinning 48 GB took 5.9 s instead of cudaHostAlloc's 18.5 s
// and copies ran at the same rate (profiles/r02_link_arena.txt); a 155 GB C3
// arena pins in ~20 s instead of ~60 s.  Anything that fails falls back to
// cudaHostAlloc.  pinned_free() releases either kind.
namespace {
std::mutex g_maps_mu;
std::map<void*, std::pair<void*, size_t>> g_maps;   // registered pointer -> (mapping, length)
}  // namespace

static cudaError_t pinned_alloc(void** out, size_t bytes, unsigned flags)
{
    constexpr size_t kHuge = 2u << 20;
    if (bytes >= (1ull << 30) && !getenv("OOCZ_NO_THP")) {
        const size_t len = (bytes + kHuge - 1) / kHuge * kHuge + kHuge;
        void* m = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
        if (m != MAP_FAILED) {
            void* p = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(m) + kHuge - 1) / kHuge * kHuge);
            madvise(p, len - kHuge, MADV_HUGEPAGE);
            if (cudaHostRegister(p, bytes, flags == cudaHostAllocPortable ? cudaHostRegisterPortable
                                                                         : cudaHostRegisterDefault) == cudaSuccess) {
                std::lock_guard<std::mutex> lk(g_maps_mu);
                g_maps[p] = {m, len};
                *out = p;
                return cudaSuccess;
            }
            cudaGetLastError();
            munmap(m, len);
        }
    }
    return cudaHostAlloc(out, std::max<size_t>(bytes, 1), flags);
}

static void pinned_free(void* p)
{
    if (!p) return;
    {
        std::lock_guard<std::mutex> lk(g_maps_mu);
        auto it = g_maps.find(p);
        if (it != g_maps.end()) {
            cudaHostUnregister(p);
            munmap(it->second.first, it->second.second);
            g_maps.erase(it);
            return;
        }
    }
    cudaFreeHost(p);
}

extern "C" oocz_status oocz_host_alloc(size_t bytes, void** out)
{
    if (!out) return OOCZ_EINVAL;
    *out = nullptr;
    const cudaError_t e = pinned_alloc(out, bytes, cudaHostAllocPortable);
    if (e != cudaSuccess) {
        *out = nullptr;
        return stateless_status(e, "cudaHostAlloc");
    }
    return OOCZ_OK;
}

extern "C" void oocz_host_free(void* p)
{
    pinned_free(p);
}

extern "C" oocz_status oocz_create_local_group(const oocz_config* cfg, int32_t world, int32_t device,
                                               oocz_ctx** outs)
{
    if (!outs || world < 1) return OOCZ_EINVAL;
    char msg[256];
    oocz_status st = oocz_validate(cfg, world, msg, sizeof msg);
    if (st != OOCZ_OK) {
        fprintf(stderr, "oocz_create_local_group: %s\n", msg);
        return st;
    }
    if (cudaSetDevice(device) != cudaSuccess) return OOCZ_ECUDA;
    size_t rb[3];
    for (int f = 0; f < 3; f++) rb[f] = row_bytes_for(cfg->nx, cfg->ny, cfg->rate[f], esz_of(cfg));
    HaloComm** hs = nullptr;
    if (world > 1) {
        std::string herr;
        hs = halo_create_local_group(world, device, (size_t)cfg->nx * cfg->ny, esz_of(cfg), 4 * cfg->tb, cfg->rate,
                                     rb, &herr);
        if (!hs) {
            fprintf(stderr, "oocz_create_local_group: %s\n", herr.c_str());
            return OOCZ_ECAPACITY;
        }
    }
    std::vector<HaloComm*> halos(world, nullptr);
    for (int r = 0; r < world && hs; r++) halos[r] = hs[r];
    for (int r = 0; r < world; r++) {
        st = create_impl(cfg, r, world, nullptr, device, halos[r], nullptr, 0, &outs[r]);
        if (st != OOCZ_OK) {
            for (int k = 0; k < r; k++) { oocz_destroy(outs[k]); outs[k] = nullptr; }
            for (int k = r; k < world; k++) if (halos[k]) halo_destroy(halos[k]);
            return st;
        }
        halos[r] = nullptr;   // owned by the context now
    }
    return OOCZ_OK;
}

extern "C" void oocz_destroy(oocz_ctx* ctx)
{
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->s_h2d) cudaStreamSynchronize(ctx->s_h2d);
    if (ctx->s_comp) cudaStreamSynchronize(ctx->s_comp);
    if (ctx->s_enc) cudaStreamSynchronize(ctx->s_enc);
    if (ctx->s_dec) cudaStreamSynchronize(ctx->s_dec);
    if (ctx->s_d2h) cudaStreamSynchronize(ctx->s_d2h);
    if (ctx->halo) halo_destroy(ctx->halo);
    for (int f = 0; f < 3; f++) {
        for (int k = 0; k < oocz_ctx::kMaxSets; k++) cudaFree(ctx->slab[k][f]);
        cudaFree(ctx->ccopy[f]);
        if (f < 2) cudaFree(ctx->pcopy[f]);
        if (ctx->cfg.store == OOCZ_STORE_HOST) {
            if (!ctx->store_external) pinned_free(ctx->store[f]);
            cudaFree(ctx->dstore[f]);
        }
        else cudaFree(ctx->store[f]);
    }
    for (auto p : ctx->in_slot) cudaFree(p);
    for (auto p : ctx->out_slot) cudaFree(p);
    cudaFree(ctx->d_flags);
    cudaFree(ctx->m_full);
    for (auto* v : {&ctx->ev_in_ready, &ctx->ev_in_free, &ctx->ev_out_ready, &ctx->ev_out_free, &ctx->ev_written,
                    &ctx->ev_encoded})
        for (auto e : *v) cudaEventDestroy(e);
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : {ctx->ev_t0, ctx->ev_t1, ctx->ev_join_h2d, ctx->ev_join_comp})
        if (e) cudaEventDestroy(e);
    if (ctx->s_h2d) cudaStreamDestroy(ctx->s_h2d);
    if (ctx->s_comp) cudaStreamDestroy(ctx->s_comp);
    if (ctx->s_enc && ctx->s_enc != ctx->s_comp) cudaStreamDestroy(ctx->s_enc);
    if (ctx->ev_join_enc) cudaEventDestroy(ctx->ev_join_enc);
    if (ctx->s_dec) cudaStreamDestroy(ctx->s_dec);
    for (int k = 0; k < oocz_ctx::kMaxSets; k++) {
        if (ctx->ev_decoded[k]) cudaEventDestroy(ctx->ev_decoded[k]);
        if (ctx->ev_slab_free[k]) cudaEventDestroy(ctx->ev_slab_free[k]);
        if (ctx->ev_stepped[k]) cudaEventDestroy(ctx->ev_stepped[k]);
    }
    if (ctx->ev_join_dec) cudaEventDestroy(ctx->ev_join_dec);
    for (auto& kv : ctx->graph_cache) cudaGraphExecDestroy(kv.second.exec);
    if (ctx->ev_g_fork) cudaEventDestroy(ctx->ev_g_fork);
    for (auto e : ctx->ev_g_join)
        if (e) cudaEventDestroy(e);
    if (ctx->s_d2h) cudaStreamDestroy(ctx->s_d2h);
    delete ctx;
}

extern "C" const char* oocz_last_error(const oocz_ctx* ctx)
{
    return ctx ? ctx->err.c_str() : g_stateless_err.c_str();
}

extern "C" oocz_status oocz_get_stats(const oocz_ctx* ctx, oocz_stats* out)
{
    if (!ctx || !out) return OOCZ_EINVAL;
    *out = ctx->stats;
    return OOCZ_OK;
}

extern "C" oocz_status oocz_get_config(const oocz_ctx* ctx, oocz_config* out)
{
    if (!ctx || !out) return OOCZ_EINVAL;
    *out = ctx->cfg;
    return OOCZ_OK;
}

extern "C" oocz_status oocz_get_events(const oocz_ctx* ctx, oocz_event* evs, size_t cap, size_t* n)
{
    if (!ctx || !n) return OOCZ_EINVAL;
    *n = ctx->events.size();
    if (evs) std::memcpy(evs, ctx->events.data(), std::min(cap, ctx->events.size()) * sizeof(oocz_event));
    return OOCZ_OK;
}

// ------------------------------------------------------------------ set / get
// Max |value| (as a double) and flags from one scan record of d_flags:
// rec[0] bit 0 non-finite, bit 1 negative; rec[1] fp32 max bits; rec[2..3] fp64 max bits.
static double scan_max(const oocz_ctx* ctx, const unsigned int* rec)
{
    if (ctx->esz == 8) {
        double mx;
        std::memcpy(&mx, &rec[2], sizeof mx);
        return mx;
    }
    float m32;
    std::memcpy(&m32, &rec[1], sizeof m32);
    return m32;
}

static cudaError_t scan_planes(oocz_ctx* ctx, const uint8_t* buf, size_t n, unsigned int* rec, cudaStream_t s)
{
    if (ctx->esz == 8)
        return launch_scan_field(reinterpret_cast<const double*>(buf), n, rec,
                                 reinterpret_cast<unsigned long long*>(rec + 2), s);
    return launch_scan_field(reinterpret_cast<const float*>(buf), n, rec, s);
}

// Compress planes [z0, z0 + nplanes) (rank-local, 4-aligned) of field f from src
// into the store (the initial round trip).  The field counts as set
// once every 4-plane row has been set; then its halos are (re)published.
//
// Two passes, so that a rejected call changes nothing ("a failed
// validation leaves the state unchanged"):
//   1. validate: every chunk is scanned for NaN / Inf and, for m, sign and the
//      CFL bound -- both on the input and on its fixed-rate round trip RT(m),
//      which is what the stencil will read (encode into scratch, decode, scan);
//      nothing is written to the store, rows_set or m_full;
//   2. write: encode into the store (and decode RT(m) into m_full if resident).
static oocz_status set_planes_impl(oocz_ctx* ctx, int32_t field, int32_t z0, int32_t nplanes, const void* src_v,
                                   bool on_device)
{
    if (!ctx) return OOCZ_EINVAL;
    if (ctx->poisoned) return fail(ctx, OOCZ_ESTATE, "context poisoned by an earlier error: %s", ctx->err.c_str());
    if (field < 0 || field > 2) return fail(ctx, OOCZ_EINVAL, "unknown field %d", field);
    if (z0 % 4 || nplanes % 4) return fail(ctx, OOCZ_EALIGN, "z0 (%d) and nplanes (%d) must be multiples of 4", z0, nplanes);
    if (z0 < 0 || nplanes < 0 || z0 + nplanes > ctx->S)
        return fail(ctx, OOCZ_EINVAL, "planes [%d, %d) outside [0, %d)", z0, z0 + nplanes, ctx->S);
    if (!src_v && nplanes) return fail(ctx, OOCZ_EINVAL, "null source");
    CK(cudaSetDevice(ctx->device));
    // a device source may still be being written on a stream of the caller's
    // (the copies below run on the library's own non-blocking stream)
    if (on_device) CK(cudaDeviceSynchronize());
    cudaStream_t s = ctx->s_comp;
    const double mmax = ctx->esz == 8 ? cfl_limit(ctx->cfg.c64) : cfl_limit(ctx->cfg.c);
    const uint8_t* src = static_cast<const uint8_t*>(src_v);
    const cudaMemcpyKind in_kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    const int rate = ctx->cfg.rate[field];
    const bool check_rt = field == OOCZ_M && rate > 0;
    // ---- pass 1: validate (scratch only: slab set 0, which holds nothing between steps)
    {
        // the encoded chunk goes to slab[0][1]: half a block of planes fits even at
        // rate 64 in fp32 (8 B per value <= 4 B x (P + 2h) / (P / 2) planes)
        const int chunk = check_rt ? std::max(4, ctx->P / 2 / 4 * 4) : ctx->P;
        CK(cudaMemsetAsync(ctx->d_flags, 0, 8 * sizeof(unsigned int), s));
        for (int z = z0; z < z0 + nplanes; z += chunk) {
            const int np = std::min(chunk, z0 + nplanes - z);
            const size_t n = (size_t)np * ctx->plane_elems;
            uint8_t* buf = ctx->slab[0][0];
            CK(cudaMemcpyAsync(buf, src + (size_t)(z - z0) * ctx->pb, (size_t)np * ctx->pb, in_kind, s));
            CK(scan_planes(ctx, buf, n, ctx->d_flags, s));
            if (check_rt) {       // RT(m): encode -> decode over the raw chunk -> scan
                uint8_t* enc = ctx->slab[0][1];
                CK(encode_or_copy(ctx, field, buf, np, enc, s));
                CK(decode_or_copy(ctx, field, enc, np, buf, s));
                CK(scan_planes(ctx, buf, n, ctx->d_flags + 4, s));
            }
        }
        unsigned int flags[8] = {};
        CK(cudaMemcpyAsync(flags, ctx->d_flags, sizeof flags, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (flags[0] & 1u) return fail(ctx, OOCZ_ENONFINITE, "field %d contains NaN or Inf", field);
        if (field == OOCZ_M) {
            if (flags[0] & 2u) return fail(ctx, OOCZ_ECFL, "m has negative values");
            const double mx = scan_max(ctx, flags);
            if (mx > mmax) return fail(ctx, OOCZ_ECFL, "max m (%.9g) > m_max(c) (%.9g)", mx, mmax);
            if (check_rt) {
                if (flags[4] & 1u)
                    return fail(ctx, OOCZ_ENONFINITE, "m at rate %d decodes to NaN or Inf", rate);
                if (flags[4] & 2u)
                    return fail(ctx, OOCZ_ECFL, "m at rate %d decodes to negative values", rate);
                const double mrt = scan_max(ctx, flags + 4);
                if (mrt > mmax)
                    return fail(ctx, OOCZ_ECFL, "max m decoded at rate %d (%.9g) > m_max(c) (%.9g)", rate, mrt, mmax);
            }
        }
    }
    // ---- pass 2: write.  Rows of this range count as unset until it succeeds.
    for (int r = z0 / 4; r < (z0 + nplanes) / 4; r++) ctx->rows_set[field][r] = 0;
    ctx->field_set[field] = false;
    std::fill(ctx->last_seq.begin(), ctx->last_seq.end(), -1LL);   // the store changes outside the slots
    const int chunk = ctx->P;                       // planes per pass, <= slab capacity
    for (int z = z0, np; z < z0 + nplanes; z += np) {
        np = rows_chunk_end(ctx, field, z, std::min(z + chunk, z0 + nplanes)) - z;
        uint8_t* buf = ctx->slab[0][0];              // scratch between steps
        CK(cudaMemcpyAsync(buf, src + (size_t)(z - z0) * ctx->pb, (size_t)np * ctx->pb, in_kind, s));
        const size_t bytes = (size_t)(np / 4) * ctx->row_bytes[field];
        const uint8_t* coded;
        if (!rows_on_device(ctx, field, z)) {
            uint8_t* dev = ctx->in_slot[0];         // device staging of the encoded rows
            CK(encode_or_copy(ctx, field, buf, np, dev, s));
            CK(cudaMemcpyAsync(rows_ptr(ctx, field, z), dev, bytes, cudaMemcpyDeviceToHost, s));
            coded = dev;
        } else {
            CK(encode_or_copy(ctx, field, buf, np, rows_ptr(ctx, field, z), s));
            coded = rows_ptr(ctx, field, z);
        }
        if (field == OOCZ_M && ctx->m_full)         // m_resident: keep the decoded RT(m)
            CK(decode_or_copy(ctx, field, coded, np, ctx->m_full + (size_t)(ctx->h + z) * ctx->pb, s));
    }
    CK(cudaStreamSynchronize(s));
    for (int r = z0 / 4; r < (z0 + nplanes) / 4; r++) ctx->rows_set[field][r] = 1;
    ctx->field_set[field] = std::all_of(ctx->rows_set[field].begin(), ctx->rows_set[field].end(),
                                        [](uint8_t v) { return v != 0; });
    if (!ctx->field_set[field]) return OOCZ_OK;
    if (field != OOCZ_M && ctx->halo) {
        std::string herr;
        if (!halo_capture_store(ctx->halo, field, rows_ptr(ctx, field, 0), rows_ptr(ctx, field, ctx->S - ctx->h), s, &herr) ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return fail(ctx, OOCZ_ENCCL, "halo capture: %s", herr.c_str());
    }
    if (field == OOCZ_M && ctx->halo) {
        // m halos are read-only: exchange them once (compressed form, reading R20)
        std::string herr;
        if (!halo_exchange_m(ctx->halo, rows_ptr(ctx, OOCZ_M, 0), rows_ptr(ctx, OOCZ_M, ctx->S - ctx->h), s, &herr))
            return fail(ctx, OOCZ_ENCCL, "m halo exchange: %s", herr.c_str());
    }
    return OOCZ_OK;
}

static oocz_status set_field_impl(oocz_ctx* ctx, int32_t field, const void* src_v, size_t count, bool on_device)
{
    if (!ctx) return OOCZ_EINVAL;
    const size_t want = ctx->plane_elems * (size_t)ctx->S;
    if (count != want) return fail(ctx, OOCZ_EINVAL, "count (%zu) != nx*ny*nz/world (%zu)", count, want);
    return set_planes_impl(ctx, field, 0, ctx->S, src_v, on_device);
}

extern "C" oocz_status oocz_set_field(oocz_ctx* ctx, int32_t field, const void* src, size_t count)
{
    return set_field_impl(ctx, field, src, count, false);
}
extern "C" oocz_status oocz_set_field_device(oocz_ctx* ctx, int32_t field, const void* d_src, size_t count)
{
    return set_field_impl(ctx, field, d_src, count, true);
}
extern "C" oocz_status oocz_set_field_planes(oocz_ctx* ctx, int32_t field, int32_t z0, int32_t nplanes,
                                             const void* src, int32_t src_on_device)
{
    return set_planes_impl(ctx, field, z0, nplanes, src, src_on_device != 0);
}

// Decode planes [z0, z0 + nplanes) (rank-local, 4-aligned) of field f into dst.
static oocz_status get_planes_impl(oocz_ctx* ctx, int32_t field, int32_t z0, int32_t nplanes, void* dst_v,
                                   bool on_device)
{
    if (!ctx) return OOCZ_EINVAL;
    if (ctx->poisoned) return fail(ctx, OOCZ_ESTATE, "context poisoned by an earlier error: %s", ctx->err.c_str());
    if (field < 0 || field > 2) return fail(ctx, OOCZ_EINVAL, "unknown field %d", field);
    if (!ctx->field_set[field]) return fail(ctx, OOCZ_ESTATE, "field %d was never set", field);
    if (z0 % 4 || nplanes % 4) return fail(ctx, OOCZ_EALIGN, "z0 (%d) and nplanes (%d) must be multiples of 4", z0, nplanes);
    if (z0 < 0 || nplanes < 0 || z0 + nplanes > ctx->S)
        return fail(ctx, OOCZ_EINVAL, "planes [%d, %d) outside [0, %d)", z0, z0 + nplanes, ctx->S);
    if (!dst_v && nplanes) return fail(ctx, OOCZ_EINVAL, "null destination");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->s_comp;
    const int chunk = ctx->P;
    uint8_t* dst = static_cast<uint8_t*>(dst_v);
    for (int z = z0, np; z < z0 + nplanes; z += np) {
        np = rows_chunk_end(ctx, field, z, std::min(z + chunk, z0 + nplanes)) - z;
        const size_t bytes = (size_t)(np / 4) * ctx->row_bytes[field];
        uint8_t* buf = ctx->slab[0][0];              // scratch between steps
        if (!rows_on_device(ctx, field, z)) {
            uint8_t* dev = ctx->in_slot[0];
            CK(cudaMemcpyAsync(dev, rows_ptr(ctx, field, z), bytes, cudaMemcpyHostToDevice, s));
            CK(decode_or_copy(ctx, field, dev, np, buf, s));
        } else {
            CK(decode_or_copy(ctx, field, rows_ptr(ctx, field, z), np, buf, s));
        }
        CK(cudaMemcpyAsync(dst + (size_t)(z - z0) * ctx->pb, buf, (size_t)np * ctx->pb,
                           on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    return OOCZ_OK;
}

static oocz_status get_field_impl(oocz_ctx* ctx, int32_t field, void* dst_v, size_t count, bool on_device)
{
    if (!ctx) return OOCZ_EINVAL;
    const size_t want = ctx->plane_elems * (size_t)ctx->S;
    if (count != want) return fail(ctx, OOCZ_EINVAL, "count (%zu) != nx*ny*nz/world (%zu)", count, want);
    return get_planes_impl(ctx, field, 0, ctx->S, dst_v, on_device);
}

extern "C" oocz_status oocz_get_field_planes(oocz_ctx* ctx, int32_t field, int32_t z0, int32_t nplanes, void* dst,
                                             int32_t dst_on_device)
{
    return get_planes_impl(ctx, field, z0, nplanes, dst, dst_on_device != 0);
}

extern "C" oocz_status oocz_get_field(oocz_ctx* ctx, int32_t field, void* dst, size_t count)
{
    return get_field_impl(ctx, field, dst, count, false);
}
extern "C" oocz_status oocz_get_field_device(oocz_ctx* ctx, int32_t field, void* d_dst, size_t count)
{
    return get_field_impl(ctx, field, d_dst, count, true);
}

// ------------------------------------------------------------------ checkpoint
extern "C" size_t oocz_store_bytes(const oocz_ctx* ctx, int32_t field)
{
    return (ctx && field >= 0 && field <= 2) ? ctx->store_bytes[field] : 0;
}

extern "C" oocz_status oocz_save_store(oocz_ctx* ctx, int32_t field, void* dst, size_t bytes)
{
    if (!ctx) return OOCZ_EINVAL;
    if (ctx->poisoned) return fail(ctx, OOCZ_ESTATE, "context poisoned by an earlier error: %s", ctx->err.c_str());
    if (field < 0 || field > 2) return fail(ctx, OOCZ_EINVAL, "unknown field %d", field);
    if (!ctx->field_set[field]) return fail(ctx, OOCZ_ESTATE, "field %d was never set", field);
    if (bytes != ctx->store_bytes[field] || (!dst && bytes))
        return fail(ctx, OOCZ_EINVAL, "bytes (%zu) != store size (%zu)", bytes, ctx->store_bytes[field]);
    CK(cudaSetDevice(ctx->device));
    const size_t dev_bytes = rows_off(ctx, field, ctx->zres[field]);   // the rows kept in HBM come first
    if (dev_bytes) CK(cudaMemcpy(dst, ctx->dstore[field], dev_bytes, cudaMemcpyDeviceToHost));
    if (bytes > dev_bytes) std::memcpy(static_cast<uint8_t*>(dst) + dev_bytes, ctx->store[field], bytes - dev_bytes);
    return OOCZ_OK;
}

extern "C" oocz_status oocz_load_store(oocz_ctx* ctx, int32_t field, const void* src, size_t bytes)
{
    if (!ctx) return OOCZ_EINVAL;
    if (ctx->poisoned) return fail(ctx, OOCZ_ESTATE, "context poisoned by an earlier error: %s", ctx->err.c_str());
    if (field < 0 || field > 2) return fail(ctx, OOCZ_EINVAL, "unknown field %d", field);
    if (bytes != ctx->store_bytes[field] || (!src && bytes))
        return fail(ctx, OOCZ_EINVAL, "bytes (%zu) != store size (%zu)", bytes, ctx->store_bytes[field]);
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->s_comp;
    ctx->field_set[field] = false;
    std::fill(ctx->rows_set[field].begin(), ctx->rows_set[field].end(), 0);
    std::fill(ctx->last_seq.begin(), ctx->last_seq.end(), -1LL);   // the store changes outside the slots
    {
        const size_t dev_bytes = rows_off(ctx, field, ctx->zres[field]);
        if (dev_bytes) CK(cudaMemcpy(ctx->dstore[field], src, dev_bytes, cudaMemcpyHostToDevice));
        if (bytes > dev_bytes)
            std::memcpy(ctx->store[field], static_cast<const uint8_t*>(src) + dev_bytes, bytes - dev_bytes);
    }
    if (field == OOCZ_M && ctx->m_full) {       // m_resident: decode the loaded stream once
        for (int z = 0; z < ctx->S; z += ctx->P) {
            const int np = std::min(ctx->P, ctx->S - z);
            const uint8_t* coded = rows_ptr(ctx, field, z);
            if (!rows_on_device(ctx, field, z)) {
                CK(cudaMemcpyAsync(ctx->in_slot[0], coded, (size_t)(np / 4) * ctx->row_bytes[field],
                                   cudaMemcpyHostToDevice, s));
                coded = ctx->in_slot[0];
            }
            CK(decode_or_copy(ctx, field, coded, np, ctx->m_full + (size_t)(ctx->h + z) * ctx->pb, s));
        }
        CK(cudaStreamSynchronize(s));
    }
    std::fill(ctx->rows_set[field].begin(), ctx->rows_set[field].end(), 1);
    ctx->field_set[field] = true;
    if (ctx->halo) {                            // the neighbours' halos come from the store
        std::string herr;
        const bool ok = field == OOCZ_M
            ? halo_exchange_m(ctx->halo, rows_ptr(ctx, OOCZ_M, 0), rows_ptr(ctx, OOCZ_M, ctx->S - ctx->h), s, &herr)
            : halo_capture_store(ctx->halo, field, rows_ptr(ctx, field, 0), rows_ptr(ctx, field, ctx->S - ctx->h), s, &herr);
        if (!ok || cudaStreamSynchronize(s) != cudaSuccess)
            return fail(ctx, OOCZ_ENCCL, "halo refresh: %s", herr.c_str());
    }
    return OOCZ_OK;
}

// ------------------------------------------------------------------ step
// Is block j's latest encoded own rows still intact in its staging slot for a
// decode enqueued now?  (Slot k is next overwritten by the encode of block
// sequence number last_seq + nslots, which is enqueued after this decode.)
static bool rows_in_slot(const oocz_ctx* ctx, int j)
{
    if (!ctx->cfg.serpentine) return false;                  // the paper-faithful schedule stays literal
    const long long ls = ctx->last_seq[j];
    return ls >= 0 && ctx->seq <= ls + (long long)ctx->out_slot.size();
}

// Enqueue one block of one sweep (ts steps).
//   dir  : +1 ascending (the paper's order, R17), -1 descending (serpentine
//          sweeps, reading R22);
//   turn : serpentine turnaround -- block i was the last block of the previous
//          sweep of this call: m is still decoded in its slab;
//   keep : block i is the last block of a sweep that is followed by a
//          turnaround in this call -- its compressed rows stay in the staging
//          slot (no D2H; the turnaround reads them and the store rows are
//          rewritten next sweep).
// Host store: rows of the read unit that are still in a staging slot (encoded
// by a recent block -- always the turnaround's, and with slots >= 3 the next
// block's own rows too) are decoded from the device; only the rest crosses the
// host link (region sharing carried across the sweep boundary, reading R22).
static oocz_status enqueue_block(oocz_ctx* ctx, int sweep, int i, int ts, int dir, bool turn, bool keep)
{
    const Geom& g = ctx->geom[i];
    const int h = ctx->h, P = ctx->P, D = ctx->D, S = ctx->S;
    const size_t pb = ctx->pb;
    // this block's rows stream over the host link (not kept in HBM: device store or
    // resident_blocks)
    const bool host = !rows_on_device(ctx, OOCZ_U, g.own0);
    const int islot = (int)(ctx->seq % (long long)ctx->ev_in_ready.size());    // input staging slot
    const int slot = (int)(ctx->seq % (long long)ctx->ev_out_ready.size());    // output staging slot
    // slab set: blocks rotate through nsets; with serpentine sweeps by block
    // index, so a turnaround block finds its own slab (and its decoded m) again;
    // in a graph capture by block
    // index too (a captured graph must not depend on the call's block count)
    const int set = ctx->cfg.serpentine || ctx->capturing ? i % ctx->nsets : (int)(ctx->seq % ctx->nsets);
    // m_resident: m is read in place from the decoded copy, never streamed
    const int nf = ctx->m_full ? 2 : 3;
    uint8_t* slab[3] = {ctx->slab[set][0], ctx->slab[set][1],
                        ctx->m_full ? ctx->m_full + (size_t)(g.slab0 + h) * pb : ctx->slab[set][2]};
    // read unit: ascending [iP+h, (i+1)P+h) (block 0 from 0); descending
    // [iP-h, (i+1)P-h) (block D-1 to S); both partition [0, S)
    const int rd0 = dir > 0 ? g.rd0 : std::max(i * P - h, 0);
    const int rd1 = dir > 0 ? g.rd1 : (i == D - 1 ? S : (i + 1) * P - h);
    const int rd_planes = rd1 - rd0;
    cudaStream_t sd = ctx->s_dec, sc = ctx->s_comp, se = ctx->s_enc;
    const int nb = dir > 0 ? std::min(i + 1, D - 1) : std::max(i - 1, 0);   // the read unit's other owner

    // ---- the read unit as (at most) two parts per field: the own rows and the
    // neighbour block's rows; each from the device (store or staging slot) or
    // from the host store through the staging slot `in`
    struct Part { int z0, z1; const uint8_t* src; bool h2d; };
    Part part[3][2];
    int nparts[3] = {0, 0, 0};
    const int own0 = std::max(rd0, g.own0), own1 = std::min(rd1, g.own1);
    for (int f = 0; f < nf; f++) {
        if (f == OOCZ_M && turn) continue;                    // still decoded in this slab
        auto add = [&](int z0, int z1, int owner) {
            if (z1 <= z0) return;
            Part q{z0, z1, nullptr, false};
            if (rows_on_device(ctx, f, z0)) {
                q.src = rows_ptr(ctx, f, z0);
            } else if (f != OOCZ_M && rows_in_slot(ctx, owner)) {
                q.src = ctx->out_slot[ctx->last_slot[owner]] + ctx->out_off[f] +
                        (size_t)((z0 - owner * P) / 4) * ctx->row_bytes[f];
            } else {
                q.src = ctx->in_slot[islot] + ctx->in_off[f] + (size_t)((z0 - rd0) / 4) * ctx->row_bytes[f];
                q.h2d = true;
            }
            part[f][nparts[f]++] = q;
        };
        if (dir > 0) { add(own0, own1, i); add(own1, rd1, nb); }
        else { add(rd0, own0, nb); add(own0, own1, i); }
    }

    // ---- (a2) H2D of the parts not on the device, once the previous sweep has
    // written those rows back
    bool any_h2d = false;
    for (int f = 0; f < nf; f++)
        for (int k = 0; k < nparts[f]; k++) any_h2d |= part[f][k].h2d;
    auto owner_of = [&](const Part& q) { return q.z0 >= g.own0 && q.z0 < g.own1 ? i : nb; };
    if (any_h2d) {
        cudaStream_t sh = ctx->s_h2d;
        CK(cudaStreamWaitEvent(sh, ctx->ev_in_free[islot], 0));
        for (int f = 0; f < nf; f++)
            for (int k = 0; k < nparts[f]; k++)
                if (part[f][k].h2d) CK(cudaStreamWaitEvent(sh, ctx->ev_written[owner_of(part[f][k])], 0));
        uint64_t bytes = 0;
        for (int f = 0; f < nf; f++)
            for (int k = 0; k < nparts[f]; k++)
                if (part[f][k].h2d) bytes += (uint64_t)((part[f][k].z1 - part[f][k].z0) / 4) * ctx->row_bytes[f];
        prof_begin(ctx, sweep, i, OOCZ_ST_H2D, 0, sh, bytes);
        for (int f = 0; f < nf; f++)
            for (int k = 0; k < nparts[f]; k++) {
                const Part& q = part[f][k];
                if (!q.h2d) continue;
                CK(cudaMemcpyAsync(const_cast<uint8_t*>(q.src), rows_ptr(ctx, f, q.z0),
                                   (size_t)((q.z1 - q.z0) / 4) * ctx->row_bytes[f], cudaMemcpyHostToDevice, sh));
            }
        prof_end(ctx, sh);
        ctx->stats.h2d_bytes += bytes;
        CK(cudaEventRecord(ctx->ev_in_ready[islot], sh));
        CK(cudaStreamWaitEvent(sd, ctx->ev_in_ready[islot], 0));
    }
    // rows read from the device: the encodes that wrote them must be done
    for (int f = 0; f < nf; f++)
        for (int k = 0; k < nparts[f]; k++)
            if (!part[f][k].h2d) CK(cudaStreamWaitEvent(sd, ctx->ev_encoded[owner_of(part[f][k])], 0));

    // ---- (a4) slab assembly on the decode stream, once this slab set is free
    CK(cudaStreamWaitEvent(sd, ctx->ev_slab_free[set], 0));
    const bool has_c = !turn && (dir > 0 ? i > 0 : i < D - 1);   // the shared region kept by the previous block
    // Parallelogram tiling (reading R26).  Ascending: a block with a block before
    // it in the sweep updates [iP + 4(ts-s), (i+1)P + 4(ts-s)) in step s instead
    // of the cone [iP - h + 4s, (i+1)P + h - 4s); the planes below that it reads
    // come at their last two time levels from block i-1 (pcopy -> slab
    // [h-4, h+4ts-4)), so of the time-t C_{i-1} only slab [h+4ts-4, 2h) of u, u-
    // is needed.  Descending sweeps mirror it: [iP - 4(ts-s), (i+1)P - 4(ts-s)),
    // the strip from block i+1 at slab [P+h-4ts+4, P+h+4), and C_i's slab
    // [P, P+h-4ts+4).  The first block of a sweep keeps the cone on that side.
    const bool para = ctx->para;
    const bool has_next = dir > 0 ? i < D - 1 : i > 0;
    // the planes [cr0, cr1) of the 2h-plane C region that are needed (u, u-)
    const int cr0 = para && dir > 0 ? h + 4 * ts - 4 : 0;
    const int cr1 = para && dir < 0 ? h - 4 * ts + 4 : 2 * h;
    auto c_lo = [&](int f) { return f == OOCZ_M ? 0 : cr0; };
    auto c_hi = [&](int f) { return f == OOCZ_M ? 2 * h : cr1; };
    if (has_c) {
        // ascending: C_{i-1} -> slab [0, 2h); descending: C_i -> slab [P, P+2h)
        const size_t dst = dir > 0 ? 0 : (size_t)P * pb;
        uint64_t cb = 0;
        for (int f = 0; f < nf; f++) cb += 2 * (uint64_t)(c_hi(f) - c_lo(f)) * pb;
        prof_begin(ctx, sweep, i, OOCZ_ST_COPY, 4, sd, cb);
        for (int f = 0; f < nf; f++) {
            const size_t o = (size_t)c_lo(f) * pb;
            CK(cudaMemcpyAsync(slab[f] + dst + o, ctx->ccopy[f] + o - (size_t)ctx->cbase[f] * pb,
                               (size_t)(c_hi(f) - c_lo(f)) * pb, cudaMemcpyDeviceToDevice, sd));
        }
        prof_end(ctx, sd);
    }
    if (ctx->halo) {  // neighbour-rank halos received at the sweep start
        std::string herr;
        if (!halo_insert(ctx->halo, i == 0, i == D - 1, slab, g.slab0, S, ctx->nx, ctx->ny, sd, &herr))
            return fail(ctx, OOCZ_ENCCL, "halo insert: %s", herr.c_str());
    }
    // ---- (a3) decode the read unit into the slab
    for (int f = 0; f < nf; f++) {
        if (!nparts[f]) continue;
        // algorithmic bytes: compressed (or raw) read unit in + decoded planes out
        uint64_t bytes = 0;
        for (int k = 0; k < nparts[f]; k++)
            bytes += (uint64_t)((part[f][k].z1 - part[f][k].z0) / 4) * ctx->row_bytes[f] +
                     (uint64_t)(part[f][k].z1 - part[f][k].z0) * pb;
        prof_begin(ctx, sweep, i, OOCZ_ST_DECODE, 4, sd, bytes);
        for (int k = 0; k < nparts[f]; k++) {
            const Part& q = part[f][k];
            CK(decode_or_copy(ctx, f, q.src, q.z1 - q.z0, slab[f] + (size_t)(q.z0 - g.slab0) * pb, sd));
        }
        prof_end(ctx, sd);
    }
    (void)rd_planes;
    if (any_h2d) CK(cudaEventRecord(ctx->ev_in_free[islot], sd));
    // a kept block's slot (its rows were never written back) is free once the
    // decodes that read it are done: the encode that reuses it waits on this
    for (int f = 0; f < nf; f++)
        for (int k = 0; k < nparts[f]; k++) {
            const int o = owner_of(part[f][k]);
            if (!part[f][k].h2d && ctx->kept[o] && !rows_on_device(ctx, f, part[f][k].z0))
                CK(cudaEventRecord(ctx->ev_out_free[ctx->last_slot[o]], sd));
        }
    // keep the time-t shared region for the next block (reading R14):
    // ascending C_i = slab [P, P+2h), descending C_{i-1} = slab [0, 2h)
    if (has_next) {
        const size_t off = dir > 0 ? (size_t)P * pb : 0;
        uint64_t cb = 0;
        for (int f = 0; f < nf; f++) cb += 2 * (uint64_t)(c_hi(f) - c_lo(f)) * pb;
        prof_begin(ctx, sweep, i, OOCZ_ST_COPY, 4, sd, cb);
        for (int f = 0; f < nf; f++) {
            const size_t o = (size_t)c_lo(f) * pb;
            CK(cudaMemcpyAsync(ctx->ccopy[f] + o - (size_t)ctx->cbase[f] * pb, slab[f] + off + o,
                               (size_t)(c_hi(f) - c_lo(f)) * pb, cudaMemcpyDeviceToDevice, sd));
        }
        prof_end(ctx, sd);
    }
    CK(cudaEventRecord(ctx->ev_decoded[set], sd));

    // ---- (a5) T cone-limited steps, in place, roles swapping (compute stream)
    CK(cudaStreamWaitEvent(sc, ctx->ev_decoded[set], 0));
    uint8_t* cu = slab[OOCZ_U];
    uint8_t* cp = slab[OOCZ_UPREV];
    const size_t strip = (size_t)(4 * ts) * pb;
    if (para && has_c) {          // the previous block's strip, both leapfrog buffers
        const size_t at = (size_t)(dir > 0 ? h - 4 : P + h - 4 * ts + 4) * pb;
        prof_begin(ctx, sweep, i, OOCZ_ST_COPY, 1, sc, 4 * (uint64_t)strip);
        CK(cudaMemcpyAsync(cu + at, ctx->pcopy[0], strip, cudaMemcpyDeviceToDevice, sc));
        CK(cudaMemcpyAsync(cp + at, ctx->pcopy[1], strip, cudaMemcpyDeviceToDevice, sc));
        prof_end(ctx, sc);
    }
    for (int s = 1; s <= ts; s++) {
        const int cone0 = std::max(4 * s, g.vlo), cone1 = std::min(ctx->L - 4 * s, g.vhi);
        int z0 = cone0, z1 = cone1;
        if (para && dir > 0) {
            if (has_c) z0 = h + 4 * (ts - s);
            z1 = std::min(P + h + 4 * (ts - s), g.vhi);
        } else if (para) {
            z0 = std::max(h - 4 * (ts - s), g.vlo);
            if (has_c) z1 = P + h - 4 * (ts - s);
        }
#ifdef OOCZ_AB_HALF_STEPS
        // A/B bound only (tools/fusion_bound.sh): every second step's launch is
        // skipped, i.e. two leapfrog steps cost one pass over the slab -- the
        // ceiling of on-chip temporal blocking by 2 with no halo recompute
        if (s % 2 == 0) { std::swap(cu, cp); continue; }
#endif
        // algorithmic bytes: read u, u-, m and write u+ once per updated cell
        prof_begin(ctx, sweep, i, OOCZ_ST_STENCIL, 1, sc, 4ull * (uint64_t)std::max(z1 - z0, 0) * pb);
        CK(stencil_step(ctx, cu, cp, slab[OOCZ_M], z0, z1, g.vlo, g.vhi, sc));
        prof_end(ctx, sc);
        std::swap(cu, cp);
    }

    if (para && has_next) {       // the strip for the next block: ascending rank planes
        // [(i+1)P-4, (i+1)P+4ts-4), descending [iP-4ts+4, iP+4)
        const size_t from = (size_t)(dir > 0 ? P + h - 4 : h - 4 * ts + 4) * pb;
        prof_begin(ctx, sweep, i, OOCZ_ST_COPY, 1, sc, 4 * (uint64_t)strip);
        CK(cudaMemcpyAsync(ctx->pcopy[0], slab[OOCZ_U] + from, strip, cudaMemcpyDeviceToDevice, sc));
        CK(cudaMemcpyAsync(ctx->pcopy[1], slab[OOCZ_UPREV] + from, strip, cudaMemcpyDeviceToDevice, sc));
        prof_end(ctx, sc);
    }

    // ---- (a6) encode own planes [iP, (i+1)P) = slab [h, P + h) of u, u-, on
    // the encode stream: the next block's stencil need not wait for it (the
    // slab is free once the strip above is copied out)
    CK(cudaEventRecord(ctx->ev_stepped[set], sc));
    CK(cudaStreamWaitEvent(se, ctx->ev_stepped[set], 0));
    const uint8_t* own[2] = {cu + (size_t)h * pb, cp + (size_t)h * pb};
    if (ctx->halo) {
        std::string herr;
        if (!halo_capture(ctx->halo, i == 0, i == D - 1, own, P, ctx->nx, ctx->ny, se, &herr))
            return fail(ctx, OOCZ_ENCCL, "halo capture: %s", herr.c_str());
    }
    if (host) {
        CK(cudaStreamWaitEvent(se, ctx->ev_out_free[slot], 0));
        for (int f = 0; f < 2; f++) {
            prof_begin(ctx, sweep, i, OOCZ_ST_ENCODE, 5, se, (uint64_t)P * pb + (uint64_t)(P / 4) * ctx->row_bytes[f]);
            CK(encode_or_copy(ctx, f, own[f], P, ctx->out_slot[slot] + ctx->out_off[f], se));
            prof_end(ctx, se);
        }
        CK(cudaEventRecord(ctx->ev_slab_free[set], se));
        ctx->last_slot[i] = slot;
        ctx->last_seq[i] = ctx->seq;
        ctx->kept[i] = keep;
        CK(cudaEventRecord(ctx->ev_encoded[i], se));
        if (keep) {
            // rows stay in the slot for the turnaround; its decode frees the slot
            CK(cudaEventRecord(ctx->ev_written[i], se));
        } else {
            CK(cudaEventRecord(ctx->ev_out_ready[slot], se));
            // ---- (a7) D2H into the store, in place
            cudaStream_t so = ctx->s_d2h;
            CK(cudaStreamWaitEvent(so, ctx->ev_out_ready[slot], 0));
            uint64_t bytes = 0;
            for (int f = 0; f < 2; f++) bytes += (uint64_t)(P / 4) * ctx->row_bytes[f];
            prof_begin(ctx, sweep, i, OOCZ_ST_D2H, 2, so, bytes);
            for (int f = 0; f < 2; f++)
                CK(cudaMemcpyAsync(rows_ptr(ctx, f, g.own0), ctx->out_slot[slot] + ctx->out_off[f],
                                   (size_t)(P / 4) * ctx->row_bytes[f], cudaMemcpyDeviceToHost, so));
            prof_end(ctx, so);
            ctx->stats.d2h_bytes += bytes;
            CK(cudaEventRecord(ctx->ev_out_free[slot], so));
            CK(cudaEventRecord(ctx->ev_written[i], so));
        }
    } else {
        for (int f = 0; f < 2; f++) {
            prof_begin(ctx, sweep, i, OOCZ_ST_ENCODE, 5, se, (uint64_t)P * pb + (uint64_t)(P / 4) * ctx->row_bytes[f]);
            CK(encode_or_copy(ctx, f, own[f], P, rows_ptr(ctx, f, g.own0), se));
            prof_end(ctx, se);
        }
        CK(cudaEventRecord(ctx->ev_slab_free[set], se));
        CK(cudaEventRecord(ctx->ev_written[i], se));
        CK(cudaEventRecord(ctx->ev_encoded[i], se));
    }
#ifdef OOCZ_DEBUG_SERIAL_ENC      // debugging: the next stencil waits for this encode
    CK(cudaEventRecord(ctx->ev_join_enc, se));
    CK(cudaStreamWaitEvent(sc, ctx->ev_join_enc, 0));
#endif
#ifdef OOCZ_DEBUG_SERIAL_DEC      // debugging: the next decode waits for this encode
    CK(cudaEventRecord(ctx->ev_join_enc, se));
    CK(cudaStreamWaitEvent(sd, ctx->ev_join_enc, 0));
#endif
    ctx->seq++;
    return OOCZ_OK;
}

static oocz_status step_begin(oocz_ctx* ctx, int64_t nsteps, cudaEvent_t* base)
{
    if (!ctx) return OOCZ_EINVAL;
    if (ctx->poisoned) return fail(ctx, OOCZ_ESTATE, "context poisoned by an earlier error: %s", ctx->err.c_str());
    if (nsteps < 0) return fail(ctx, OOCZ_EINVAL, "nsteps (%lld) < 0", (long long)nsteps);
    for (int f = 0; f < 3; f++)
        if (!ctx->field_set[f]) return fail(ctx, OOCZ_ESTATE, "field %d was never set", f);
    CK(cudaSetDevice(ctx->device));
    ctx->prof.clear();
    ctx->events.clear();
    ctx->ev_used = 0;
    // device-side timing of the whole call: all three streams start after t0
    *base = ctx->ev_t0;
    CK(cudaEventRecord(ctx->ev_t0, ctx->s_h2d));
    CK(cudaStreamWaitEvent(ctx->s_comp, ctx->ev_t0, 0));
    CK(cudaStreamWaitEvent(ctx->s_enc, ctx->ev_t0, 0));
    CK(cudaStreamWaitEvent(ctx->s_dec, ctx->ev_t0, 0));
    CK(cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_t0, 0));
    halo_step_begin(ctx->halo);
    return OOCZ_OK;
}

static oocz_status step_end(oocz_ctx* ctx, int64_t nsteps, cudaEvent_t base)
{
    CK(cudaSetDevice(ctx->device));
    // join the other streams into s_d2h and stamp t1 there
    CK(cudaEventRecord(ctx->ev_join_h2d, ctx->s_h2d));
    CK(cudaEventRecord(ctx->ev_join_comp, ctx->s_comp));
    CK(cudaEventRecord(ctx->ev_join_enc, ctx->s_enc));
    CK(cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_join_enc, 0));
    CK(cudaEventRecord(ctx->ev_join_dec, ctx->s_dec));
    CK(cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_join_dec, 0));
    CK(cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_join_h2d, 0));
    CK(cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_join_comp, 0));
    if (ctx->halo) {
        std::string herr;
        if (!halo_join(ctx->halo, ctx->s_d2h, &herr)) return fail(ctx, OOCZ_ECUDA, "halo join: %s", herr.c_str());
    }
    CK(cudaEventRecord(ctx->ev_t1, ctx->s_d2h));
    if (ctx->halo) {      // NCCL: poll for asynchronous communicator errors instead of hanging
        std::string herr;
        if (!halo_wait(ctx->halo, ctx->ev_t1, &herr)) return fail(ctx, OOCZ_ENCCL, "halo: %s", herr.c_str());
    }
    CK(cudaStreamSynchronize(ctx->s_h2d));
    CK(cudaStreamSynchronize(ctx->s_comp));
    CK(cudaStreamSynchronize(ctx->s_enc));
    CK(cudaStreamSynchronize(ctx->s_dec));
    CK(cudaStreamSynchronize(ctx->s_d2h));
    {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, ctx->ev_t0, ctx->ev_t1));
        ctx->stats.last_step_device_ms = ms;
        ctx->stats.step_device_ms += ms;
    }
    ctx->stats.steps += (uint64_t)nsteps;
    ctx->stats.halo_bytes = halo_bytes_sent(ctx->halo);
    if (ctx->cfg.profile && base) {
        for (auto& p : ctx->prof) {
            float a = 0, b = 0;
            CK(cudaEventElapsedTime(&a, base, p.a));
            CK(cudaEventElapsedTime(&b, base, p.b));
            ctx->events.push_back(oocz_event{p.sweep, p.block, p.stage, p.lane, a, b, p.bytes});
            const double d = b - a;
            switch (p.stage) {
                case OOCZ_ST_H2D: ctx->stats.h2d_ms += d; break;
                case OOCZ_ST_DECODE: ctx->stats.decode_ms += d; break;
                case OOCZ_ST_STENCIL: ctx->stats.stencil_ms += d; break;
                case OOCZ_ST_ENCODE: ctx->stats.encode_ms += d; break;
                case OOCZ_ST_D2H: ctx->stats.d2h_ms += d; break;
                case OOCZ_ST_HALO: ctx->stats.halo_ms += d; break;
                case OOCZ_ST_COPY: ctx->stats.copy_ms += d; break;
            }
        }
    }
    return OOCZ_OK;
}

// ---- CUDA graphs (cfg.graphs).  A chunk of up to kGraphSweeps sweeps is
// captured once per length in steps and replayed on the decode stream.  The
// capture forks every stream from the decode stream, re-records every event the
// blocks wait on at the fork (so the graph depends on nothing outside itself)
// and joins all streams back at the end; consecutive replays are ordered by the
// decode stream, so sweep k+1 of the next chunk starts after the whole chunk.
// The enqueued work is exactly the eager path's (enqueue_block), slab sets
// chosen by block index.
static constexpr int kGraphSweeps = 16;

// In core: with every field raw and the store in HBM, the store IS the grid (the
// [z][y][x] planes of each field), so a sweep is T whole-grid steps in place, the
// two time levels swapping roles by pointer -- what the block schedule computes
// with raw round trips (the schedule equals the in-core leapfrog),
// without its slab copies.  The paper-faithful schedule (cone = 1) keeps its blocks.
static bool in_core_eligible(const oocz_ctx* c)
{
    return c->cfg.store == OOCZ_STORE_DEVICE && c->world == 1 && !c->halo && c->cfg.cone == 0 &&
           c->cfg.rate[0] == 0 && c->cfg.rate[1] == 0 && c->cfg.rate[2] == 0;
}

static oocz_status in_core_sweep(oocz_ctx* ctx, int sweep, int ts)
{
    for (int s = 0; s < ts; s++) {
        uint8_t* u = ctx->store[OOCZ_U];
        uint8_t* up = ctx->store[OOCZ_UPREV];
        const uint8_t* m = ctx->store[OOCZ_M];
        const int S = ctx->S;
        prof_begin(ctx, sweep, 0, OOCZ_ST_STENCIL, 1, ctx->s_comp, 4ull * (uint64_t)S * ctx->pb);
        cudaError_t e = ctx->esz == 8
            ? launch_stencil_step(reinterpret_cast<const double*>(u), reinterpret_cast<double*>(up),
                                  reinterpret_cast<const double*>(m), ctx->nx, ctx->ny, S, ctx->cfg.c64, 0, S, 0, S,
                                  ctx->s_comp)
            : launch_stencil_step(reinterpret_cast<const float*>(u), reinterpret_cast<float*>(up),
                                  reinterpret_cast<const float*>(m), ctx->nx, ctx->ny, S, ctx->cfg.c, 0, S, 0, S,
                                  ctx->s_comp);
        CK(e);
        prof_end(ctx, ctx->s_comp);
        // u+ was written over u-: it is the new u, the old u the new u-
        std::swap(ctx->store[OOCZ_U], ctx->store[OOCZ_UPREV]);
        std::swap(ctx->dstore[OOCZ_U], ctx->dstore[OOCZ_UPREV]);
    }
    return OOCZ_OK;
}

static bool graph_eligible(const oocz_ctx* c)
{
    return c->cfg.graphs && c->cfg.store == OOCZ_STORE_DEVICE && c->world == 1 && !c->halo && !c->cfg.profile &&
           !c->cfg.serpentine && !in_core_eligible(c);
}

static oocz_status capture_chunk(oocz_ctx* ctx, int64_t nsteps, int* sweeps)
{
    cudaStream_t o = ctx->s_dec;
    cudaStream_t others[4] = {ctx->s_h2d, ctx->s_comp, ctx->s_enc, ctx->s_d2h};
    CK(cudaEventRecord(ctx->ev_g_fork, o));
    for (cudaStream_t s : others) CK(cudaStreamWaitEvent(s, ctx->ev_g_fork, 0));
    for (int k = 0; k < ctx->nsets; k++) {
        CK(cudaEventRecord(ctx->ev_decoded[k], o));
        CK(cudaEventRecord(ctx->ev_slab_free[k], o));
        CK(cudaEventRecord(ctx->ev_stepped[k], o));
    }
    for (int i = 0; i < ctx->D; i++) {
        CK(cudaEventRecord(ctx->ev_encoded[i], o));
        CK(cudaEventRecord(ctx->ev_written[i], o));
    }
    int64_t done = 0;
    int sweep = 0;
    while (done < nsteps) {
        const int ts = (int)std::min<int64_t>(ctx->T, nsteps - done);
        for (int i = 0; i < ctx->D; i++) {
            oocz_status st = enqueue_block(ctx, sweep, i, ts, 1, false, false);
            if (st != OOCZ_OK) return st;
        }
        done += ts;
        sweep++;
    }
    for (int k = 0; k < 4; k++) {
        CK(cudaEventRecord(ctx->ev_g_join[k], others[k]));
        CK(cudaStreamWaitEvent(o, ctx->ev_g_join[k], 0));
    }
    *sweeps = sweep;
    return OOCZ_OK;
}

// Builds (captures and instantiates) the graph of a chunk of nsteps if it is not
// cached yet.  Called before the call's t0, so device timing excludes it.
static oocz_status ensure_graph(oocz_ctx* ctx, int64_t nsteps)
{
    auto it = ctx->graph_cache.find(nsteps);
    if (it == ctx->graph_cache.end()) {
        cudaStream_t o = ctx->s_dec;
        const long long seq0 = ctx->seq;
        const uint64_t l0 = g_launches.load();
        CK(cudaStreamBeginCapture(o, cudaStreamCaptureModeRelaxed));
        ctx->capturing = true;
        int sweeps = 0;
        oocz_status st = capture_chunk(ctx, nsteps, &sweeps);
        ctx->capturing = false;
        cudaGraph_t g = nullptr;
        const cudaError_t e = cudaStreamEndCapture(o, &g);
        ctx->seq = seq0;
        const uint64_t launches = g_launches.load() - l0;
        g_launches.fetch_sub(launches);          // captured, not launched: counted per replay
        if (st != OOCZ_OK) {
            if (g) cudaGraphDestroy(g);
            return st;
        }
        if (e != cudaSuccess) return fail(ctx, OOCZ_ECUDA, "graph capture: %s", cudaGetErrorString(e));
        cudaGraphExec_t x = nullptr;
        const cudaError_t ei = cudaGraphInstantiate(&x, g, 0);
        cudaGraphDestroy(g);
        if (ei != cudaSuccess) return fail(ctx, OOCZ_ECUDA, "graph instantiate: %s", cudaGetErrorString(ei));
        ctx->graph_cache.emplace(nsteps, oocz_ctx::Graph{x, launches, sweeps});
    }
    return OOCZ_OK;
}

static oocz_status run_graph_chunk(oocz_ctx* ctx, int64_t nsteps)
{
    auto it = ctx->graph_cache.find(nsteps);
    if (it == ctx->graph_cache.end()) return fail(ctx, OOCZ_ESTATE, "graph for %lld steps not built", (long long)nsteps);
    CK(cudaGraphLaunch(it->second.exec, ctx->s_dec));
    note_launches(it->second.launches);
    ctx->seq += (long long)it->second.sweeps * ctx->D;
    ctx->stats.sweeps += (uint64_t)it->second.sweeps;
    return OOCZ_OK;
}

// Enqueue all sweeps of every context in lockstep (one context unless this is
// an in-process local group), then wait.
static oocz_status step_group(oocz_ctx* const* ctxs, int n, int64_t nsteps)
{
    if (!ctxs || n < 1) return OOCZ_EINVAL;
    const auto t0 = std::chrono::steady_clock::now();
    const bool graphed = n == 1 && graph_eligible(ctxs[0]);
    if (graphed && nsteps > 0) {
        oocz_ctx* ctx = ctxs[0];
        if (ctx->poisoned) return fail(ctx, OOCZ_ESTATE, "context poisoned by an earlier error: %s", ctx->err.c_str());
        CK(cudaSetDevice(ctx->device));
        const int64_t chunk = (int64_t)kGraphSweeps * ctx->T;
        for (int64_t k : {std::min<int64_t>(chunk, nsteps), nsteps % chunk}) {
            if (k <= 0) continue;
            oocz_status st = ensure_graph(ctx, k);
            if (st != OOCZ_OK) return st;
        }
    }
    const uint64_t launches0 = g_launches.load();
    std::vector<cudaEvent_t> base(n, nullptr);
    for (int r = 0; r < n; r++) {
        oocz_status st = step_begin(ctxs[r], nsteps, &base[r]);
        if (st != OOCZ_OK) return st;
    }
    const int T = ctxs[0]->T;
    int64_t done = 0;
    int sweep = 0;
    if (graphed) {
        const int64_t chunk = (int64_t)kGraphSweeps * T;
        while (done < nsteps) {
            const int64_t k = std::min<int64_t>(chunk, nsteps - done);
            oocz_status st = run_graph_chunk(ctxs[0], k);
            if (st != OOCZ_OK) return st;
            done += k;
        }
    }
    while (done < nsteps) {
        const int ts = (int)std::min<int64_t>(T, nsteps - done);
        for (int r = 0; r < n; r++) {
            oocz_ctx* ctx = ctxs[r];
            if (ctx->halo) {
                // both directions start as soon as their own captures (previous
                // sweep) and inserts are done, on the halo's own streams
                std::string herr;
                CK(cudaSetDevice(ctx->device));
                if (!halo_sweep_begin(ctx->halo, &herr))
                    return fail(ctx, OOCZ_ENCCL, "halo exchange: %s", herr.c_str());
            }
        }
        const bool last_sweep = done + ts >= nsteps;
        for (int r = 0; r < n; r++) {
            oocz_ctx* ctx = ctxs[r];
            if (in_core_eligible(ctx)) {
                oocz_status st = in_core_sweep(ctx, sweep, ts);
                if (st != OOCZ_OK) return st;
                ctx->stats.sweeps++;
                continue;
            }
            const int D = ctx->D;
            // serpentine (reading R22): odd sweeps of the call descend, and the block
            // at each turn is processed twice in a row without leaving the device
            const bool serp = ctx->cfg.serpentine != 0;
            const int dir = serp && (sweep & 1) ? -1 : 1;
            for (int k = 0; k < D; k++) {
                const int i = dir > 0 ? k : D - 1 - k;
                const bool turn = serp && sweep > 0 && k == 0;
                // the last nkeep blocks before a turnaround keep their rows in their slots
                // (no D2H): the first nkeep blocks after it read them from there before
                // re-encoding them, which needs slots >= 2 nkeep - 1 (R22)
                const int nkeep = std::min(D, ((int)ctx->out_slot.size() + 1) / 2);
                const bool keep = serp && !last_sweep && k >= D - nkeep;
                oocz_status st = enqueue_block(ctx, sweep, i, ts, dir, turn, keep);
                if (st != OOCZ_OK) return st;
            }
            ctx->stats.sweeps++;
        }
        done += ts;
        sweep++;
    }
    for (int r = 0; r < n; r++) {
        oocz_status st = step_end(ctxs[r], nsteps, base[r]);
        if (st != OOCZ_OK) return st;
    }
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    const uint64_t launched = g_launches.load() - launches0;
    for (int r = 0; r < n; r++) {
        ctxs[r]->stats.step_ms += ms;
        ctxs[r]->stats.kernel_launches += launched;
    }
    return OOCZ_OK;
}

extern "C" oocz_status oocz_step(oocz_ctx* ctx, int64_t nsteps)
{
    return step_group(&ctx, 1, nsteps);
}

extern "C" oocz_status oocz_step_local_group(oocz_ctx* const* ctxs, int32_t world, int64_t nsteps)
{
    if (!ctxs || world < 1) return OOCZ_EINVAL;
    for (int r = 0; r < world; r++)
        if (!ctxs[r] || ctxs[r]->rank != r || ctxs[r]->world != world) return OOCZ_EINVAL;
    return step_group(ctxs, world, nsteps);
}
