/*
 * oocz.h -- C ABI of liboocz.so: out-of-core 25-point stencil time stepping
 * with on-the-fly ZFP-style fixed-rate compression, B200 (sm_100a).
 *
 * Method: Shen, Wu, Okita, Ino, "Accelerating GPU-Based Out-of-Core Stencil
 * Computation with On-the-Fly Compression", arXiv 2109.05410.
 * The calls follow the paper's problem statement (Sec. VI):
 * given two read-write time levels u^t, u^{t-1}, a read-only model m, a
 * 25-point stencil and a compression rate, advance n steps and read back.
 *
 * Conventions
 *  - Every call returns oocz_status: 0 = OK, < 0 = error.  A failed call
 *    leaves the context unchanged unless it returns OOCZ_ECUDA / OOCZ_ENCCL,
 *    which poison the context (every later call returns OOCZ_ESTATE).
 *  - Fields are fp32 (precision 32) or fp64 (precision 64: the paper's own,
 *    PAPER.md:208), x fastest then y then z ("C order" [z][y][x]).
 *  - A context is used by one host thread at a time.
 *  - Pointers named d_* are device pointers on the context's device; all
 *    others are host pointers.  The caller owns every pointer it passes; the
 *    library never keeps one past the call (except the stream handles passed
 *    to the codec / kernel calls, used only during the call).
 *  - No torch types, no C++ types: plain pointers, sizes, and PODs.
 */
#ifndef OOCZ_H
#define OOCZ_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OOCZ_ABI_VERSION 6

typedef enum {
    OOCZ_OK = 0,
    OOCZ_EINVAL = -1,      /* bad value: P < 2h, P does not divide nz/world, rate > 64, ... */
    OOCZ_EALIGN = -2,      /* nx, ny, nz, P or h not a multiple of 4 (ZFP blocks are 4^3) */
    OOCZ_ECFL = -3,        /* max m exceeds the leapfrog stability bound m_max(c), or m < 0 */
    OOCZ_ECAPACITY = -4,   /* device (or pinned host) memory budget too small */
    OOCZ_ENONFINITE = -5,  /* NaN or Inf in a field passed to set_field */
    OOCZ_ESTATE = -6,      /* step before all fields were set, or poisoned context */
    OOCZ_ECUDA = -7,       /* CUDA runtime / driver failure (poisons the context) */
    OOCZ_ENCCL = -8        /* NCCL failure (poisons the context) */
} oocz_status;

/* field ids ("two read-write datasets ... and a read-only dataset") */
enum { OOCZ_U = 0,        /* u^t       (read-write) */
       OOCZ_UPREV = 1,    /* u^{t-1}   (read-write) */
       OOCZ_M = 2 };      /* m = (v dt / dx)^2 (read-only) */

/* where the per-field store lives */
enum { OOCZ_STORE_HOST = 0,    /* pinned host DRAM: the paper's out-of-core path */
       OOCZ_STORE_DEVICE = 1 };/* resident in HBM: same pipeline, no host link (measures the kernels) */

typedef struct {
    int32_t  nx, ny, nz;   /* GLOBAL interior extent; multiples of 4.  Rank r of `world`
                              owns planes [r*nz/world, (r+1)*nz/world).                   */
    float    c[5];         /* 1-D second-derivative weights c0..c4 (radius 4);
                              oocz_default_config fills the 8th-order set (R1). */
    int32_t  tb;           /* temporal blocking depth T >= 1 (PAPER.md:217 uses 12); halo h = 4T */
    int32_t  block_planes; /* P: z-planes per block; multiple of 4, P >= 2h, P | nz/world     */
    int32_t  rate[3];      /* bits per value for {U, UPREV, M}: 0 = raw fp32, 1..64 = fixed-rate
                              ZFP ("the number of bits to preserve a value") */
    int32_t  store;        /* OOCZ_STORE_HOST or OOCZ_STORE_DEVICE.  DEVICE with every rate 0,
                              world = 1 and cone = 0 is the in-core problem: oocz_step then
                              steps the store in place (one whole-grid launch per step, no
                              blocks); results identical                                   */
    int32_t  slots;        /* staging slots (>= 2), host store only: `slots` output slots for
                              encoded rows (with serpentine, the last (slots + 1) / 2 blocks
                              before a turnaround keep their rows there instead of writing
                              them back) and min(slots, 3) input slots for the H2D of read
                              units.  Results identical.                                     */
    int32_t  profile;      /* 1: record per-stage CUDA events (oocz_get_events)               */
    uint64_t device_bytes; /* device memory budget; 0 = whatever cudaMemGetInfo reports free  */
    int32_t  m_resident;   /* 1: decode the read-only m ONCE into HBM (nx*ny*(nz/world + 8T)
                              values) and keep it, instead of streaming and decoding it every
                              sweep: orchestration beyond the paper (the
                              paper's future work PAPER.md:254).  Results are identical.     */
    int32_t  precision;    /* 32: fp32 fields, arithmetic and codec (uses c);  64: fp64 (uses
                              c64; the paper's precision; rates 32/64 and 24/64,
                              PAPER.md:213-215).  Raw rate 0 stores 4 resp. 8 B per value.   */
    double   c64[5];       /* the weights for precision 64 (default: the exact decimals)      */
    int32_t  serpentine;   /* 1: sweeps alternate ascending / descending inside one oocz_step,
                              and the block at each turn is processed twice in a row on the
                              device: its compressed rows never cross the host link in between
                              (1/D of the traffic per sweep saved).  Orchestration beyond the
                              paper (R22).  Results identical.  */
    int32_t  slab_sets;    /* device slab sets the blocks rotate through: 0 (= 2), 1, 2, 3 or 4.
                              Each set is (P + 8T) planes per streamed field.  With more sets
                              block i+1 decodes and block i-1 encodes while block i runs its
                              stencil (the encode has its own stream); with 1 those run one
                              after another (least HBM: a compressed store that nearly fills
                              the GPU, e.g. C3 with store = OOCZ_STORE_DEVICE).  Results
                              identical.  Out of range: OOCZ_EINVAL. */
    int32_t  graphs;       /* 1: replay each oocz_step's sweeps as a captured CUDA graph (built
                              on the first call with that nsteps, cached per context, chunks of
                              at most 16 sweeps).  Takes effect with store = OOCZ_STORE_DEVICE,
                              world = 1, profile = 0 and serpentine = 0; otherwise ignored.  For
                              launch-bound small grids.  Results identical.  0 or 1, else
                              OOCZ_EINVAL. */
    int32_t  cone;         /* temporal-blocking tile shape.  1: the paper's trapezoid cone
                              (PAPER.md:112, :217): block i updates planes [iP - h + 4s,
                              (i+1)P + h - 4s) in step s, recomputing the overlap with its
                              neighbours.  0 (default): parallelogram tiles (R26),
                              every cell updated once per step, the overlap's last two time
                              levels handed from block to block.  Results identical.  0 or
                              1, else OOCZ_EINVAL. */
    int32_t  resident_blocks; /* K: with store = OOCZ_STORE_HOST, the compressed rows of
                              z-blocks 0 .. K-1 (all three fields) live in HBM and never cross
                              the host link; blocks K .. D-1 stream from pinned host memory
                              as usual.  The host store then holds only the streamed rows,
                              so a store larger than host RAM runs when its resident part
                              fits HBM (a hybrid of the two placements; the paper streams
                              everything, PAPER.md:254 names orchestration future work).
                              0 (default) = all rows on the host; K = D equals
                              OOCZ_STORE_DEVICE.  -1 = auto: the largest K whose rows fit
                              the device budget (device_bytes, or the free memory) beside
                              everything else; oocz_get_config reports the K chosen, and
                              oocz_host_store_bytes the K = 0 size (an upper bound).  Per
                              rank with world > 1 (D = nz / world / P).  Needs store =
                              HOST when nonzero; -1 <= K <= D, else OOCZ_EINVAL.  Results
                              identical. */
    int32_t  m_hbm;        /* 1: with store = OOCZ_STORE_HOST, the read-only m's compressed
                              stream lives in HBM whole (decoded per block, never crossing the
                              host link), whatever resident_blocks says for u and u-.  Half
                              the HBM of m_resident's decoded m at rate 16, for more output
                              slots.  0 or 1 (1 needs store = HOST), else OOCZ_EINVAL.
                              Results identical. */
} oocz_config;

typedef struct {
    uint64_t steps, sweeps;           /* totals since create                                */
    uint64_t h2d_bytes, d2h_bytes;    /* host<->device bytes moved by oocz_step             */
    uint64_t halo_bytes;              /* bytes sent to neighbour ranks by oocz_step          */
    uint64_t kernel_launches;         /* this library's kernel launches in oocz_step         */
    uint64_t device_bytes_used;       /* device memory held by the context                   */
    uint64_t host_bytes_pinned;       /* pinned host memory held by the context              */
    double   step_ms;                 /* host wall time spent inside oocz_step               */
    /* per-stage device time summed over blocks (profile = 1 only), ms */
    double   h2d_ms, decode_ms, stencil_ms, encode_ms, d2h_ms, copy_ms, halo_ms;
    /* device time of oocz_step calls (CUDA events on the library's own streams:
       from the first enqueued operation to the join of all streams), ms */
    double   last_step_device_ms, step_device_ms;
} oocz_stats;

/* one pipeline stage of one block (profile = 1), times relative to the
 * first event of the last oocz_step call (SPEC.md:282-287 StageEvent) */
enum { OOCZ_ST_H2D = 0, OOCZ_ST_DECODE = 1, OOCZ_ST_STENCIL = 2, OOCZ_ST_ENCODE = 3,
       OOCZ_ST_D2H = 4, OOCZ_ST_HALO = 5, OOCZ_ST_COPY = 6 };
/* events are per operation: one per stencil launch, one per field for decode /
 * encode; `bytes` is that operation's ALGORITHMIC byte count (DESIGN.md
 * "Roofline"): stencil 16 B per updated cell; decode/encode the compressed bytes
 * plus 4 B per value; copies and transfers the bytes moved. */
typedef struct {
    int32_t  sweep, block, stage, lane;   /* lane: 0 = h2d, 1 = compute (stencil), 2 = d2h, 3 = comm,
                                             4 = decode, 5 = encode */
    double   start_ms, end_ms;
    uint64_t bytes;
} oocz_event;

typedef struct oocz_ctx oocz_ctx;

/* ---------------------------------------------------------------- library */
int32_t     oocz_abi_version(void);
const char* oocz_status_string(oocz_status s);
/* fills defaults: precision 32, 8th-order c / c64, tb = 4, rates 16, host store, 2 slots */
void        oocz_default_config(oocz_config* cfg, int32_t nx, int32_t ny, int32_t nz);
/* m_max(c) = 4 / (3 max_theta |S(theta)|), S = c0 + 2 sum c_k cos(k theta); 105/512 for
 * the default c (R2).  oocz_set_field(M) rejects larger m with OOCZ_ECFL. */
double      oocz_cfl_limit(const float c[5]);
double      oocz_cfl_limit_f64(const double c[5]);
/* validate a config for (rank, world) without allocating; msg (may be NULL) receives
 * the violated constraint, e.g. "P (36) < 2h (40)" */
oocz_status oocz_validate(const oocz_config* cfg, int32_t world, char* msg, size_t msg_len);

/* ---------------------------------------------------------------- stepper
 * Multi-GPU (world > 1): one process per GPU; z-slabs of nz/world planes; the
 * 128-byte NCCL unique id comes from oocz_get_nccl_id on rank 0 and is
 * broadcast by the caller (e.g. torch.distributed).  oocz_create and
 * oocz_step are collective over the world. */
oocz_status oocz_get_nccl_id(uint8_t id[128]);
oocz_status oocz_create(const oocz_config* cfg, int32_t rank, int32_t world,
                        const uint8_t* nccl_id /* NULL if world == 1 */,
                        int32_t device, oocz_ctx** out);
/* Caller-owned host store (one pinned arena reused by several contexts in turn,
 * e.g. the benchmark's schedules over one 155 GB store: pinning takes ~0.45 s
 * per GiB, the allocation, not the stepping, would dominate).
 *  - oocz_host_store_bytes: arena bytes a host-store context for (cfg, world)
 *    needs on each rank (the three field stores, each rounded up to 4 KiB; with
 *    resident_blocks K > 0 only the streamed rows); 0 if nz is not divisible by
 *    world.
 *  - oocz_host_alloc / oocz_host_free: pinned, portable host memory
 *    (cudaHostAlloc); OOCZ_ECUDA if the allocation fails (oocz_last_error(NULL)).
 *  - oocz_create_ex: oocz_create, but with store = OOCZ_STORE_HOST the stores
 *    are carved from `host_arena` (pinned host memory of arena_bytes >=
 *    oocz_host_store_bytes, else OOCZ_EINVAL / OOCZ_ECAPACITY), which the
 *    caller owns and frees after oocz_destroy.  host_arena == NULL: the
 *    context allocates its own (= oocz_create).  A non-NULL arena with
 *    store = OOCZ_STORE_DEVICE is OOCZ_EINVAL.  One arena serves one live
 *    context at a time. */
size_t      oocz_host_store_bytes(const oocz_config* cfg, int32_t world);
oocz_status oocz_host_alloc(size_t bytes, void** out);
void        oocz_host_free(void* p);
oocz_status oocz_create_ex(const oocz_config* cfg, int32_t rank, int32_t world,
                           const uint8_t* nccl_id, int32_t device,
                           void* host_arena, size_t arena_bytes, oocz_ctx** out);
/* Copy this rank's slab (count = nx*ny*nz/world values: float for precision 32,
 * double for precision 64) of field f into the
 * store, compressing it on the GPU (the initial round trip).
 * Rejects NaN/Inf (OOCZ_ENONFINITE) and, for OOCZ_M, m < 0 or m > m_max (OOCZ_ECFL),
 * checked on the input AND on its fixed-rate round trip RT(m) (what the stencil
 * reads).  Validation runs before anything is written: a rejected call leaves
 * the previous field (store, set state) unchanged. */
oocz_status oocz_set_field(oocz_ctx* ctx, int32_t field, const void* src, size_t count);
oocz_status oocz_set_field_device(oocz_ctx* ctx, int32_t field, const void* d_src, size_t count);
/* Advance n steps: floor(n/T) sweeps of T steps, then one sweep of n mod T.
 * Every sweep streams each z-block through decode -> T cone-limited stencil
 * steps -> encode (Fig. 4), with copies, codec and stencil on
 * separate CUDA streams (Fig. 5).  Blocks until done.
 * Results depend on how n is split across calls (each sweep ends with a
 * re-encode); R16. */
oocz_status oocz_step(oocz_ctx* ctx, int64_t nsteps);
/* Decode this rank's slab of field f into dst (count values of the context's precision). */
oocz_status oocz_get_field(oocz_ctx* ctx, int32_t field, void* dst, size_t count);
/* The same two calls on a z-range, for slabs too large to hold in host memory
 * at once (3 x 103 GB raw per GPU).  Planes [z0, z0 + nplanes)
 * of this rank's slab (rank-local, both multiples of 4: whole ZFP block-rows,
 * else OOCZ_EALIGN; outside [0, nz/world): OOCZ_EINVAL); src / dst hold
 * nplanes * nx * ny values (x fastest), in device memory if *_on_device != 0,
 * else host memory (pageable or pinned).  A field counts as set once every
 * block-row has been set (oocz_step needs all three; get_* needs the field);
 * set_field_planes applies the same checks as set_field to its planes (NaN /
 * Inf, m range) and, on failure, leaves the context unchanged.  A device source is
 * read after a device-wide synchronisation (it may be produced on any stream);
 * the calls return once dst is written. */
oocz_status oocz_set_field_planes(oocz_ctx* ctx, int32_t field, int32_t z0, int32_t nplanes,
                                  const void* src, int32_t src_on_device);
oocz_status oocz_get_field_planes(oocz_ctx* ctx, int32_t field, int32_t z0, int32_t nplanes,
                                  void* dst, int32_t dst_on_device);
oocz_status oocz_get_field_device(oocz_ctx* ctx, int32_t field, void* d_dst, size_t count);
/* Checkpoint / restore.  Between oocz_step calls the
 * compressed store IS the whole state; a decode -> encode round trip is not
 * idempotent, so a faithful checkpoint keeps the compressed bytes.
 * oocz_store_bytes: this rank's store size for field f (0 for a bad field).
 * oocz_save_store copies it to host memory `dst` (exactly that many bytes);
 * oocz_load_store replaces it from `src` and marks the field set; a context
 * created with the same config then continues bit for bit (collective for
 * world > 1: the halos are refreshed from the loaded stores). */
size_t      oocz_store_bytes(const oocz_ctx* ctx, int32_t field);
oocz_status oocz_save_store(oocz_ctx* ctx, int32_t field, void* dst, size_t bytes);
oocz_status oocz_load_store(oocz_ctx* ctx, int32_t field, const void* src, size_t bytes);
oocz_status oocz_get_stats(const oocz_ctx* ctx, oocz_stats* out);
/* the configuration the context was created with */
oocz_status oocz_get_config(const oocz_ctx* ctx, oocz_config* out);
/* In-process z-partitioned group on ONE device: `world` contexts (ranks 0..world-1)
 * that exchange their halos with device copies instead of NCCL, stepped in
 * lockstep by oocz_step_local_group.  Same engine, same halo protocol as the
 * multi-process path; used to check on a single GPU that a partitioned run is
 * bit-identical to world = 1.  Each context is destroyed with oocz_destroy. */
oocz_status oocz_create_local_group(const oocz_config* cfg, int32_t world, int32_t device, oocz_ctx** outs);
oocz_status oocz_step_local_group(oocz_ctx* const* ctxs, int32_t world, int64_t nsteps);
/* copy up to cap events of the last oocz_step (profile = 1) into evs; *n = total */
oocz_status oocz_get_events(const oocz_ctx* ctx, oocz_event* evs, size_t cap, size_t* n);
/* owned by ctx; valid until the next call.  With ctx == NULL: the last failure of a
 * stateless codec / kernel call on this host thread. */
const char* oocz_last_error(const oocz_ctx* ctx);
void        oocz_destroy(oocz_ctx* ctx);

/* ---------------------------------------------------------------- codec / kernels
 * Stateless entry points used by the parity tests and the benchmark.  All
 * pointers are device pointers, caller-owned; `stream` is a cudaStream_t (NULL
 * = legacy default stream).  The call enqueues work and returns; errors in
 * argument checking are returned synchronously. */

/* exact compressed size: (nx/4)(ny/4)(nz/4) * 8 * rate bytes (fixed rate) */
size_t      oocz_zfp_bytes(int32_t nx, int32_t ny, int32_t nz, int32_t rate);
/* ZFP fixed-rate fp32 3-D encode: 4^3 blocks in order bz, by, bx; block b occupies
 * words [rate*b, rate*b + rate) of d_out (little-endian uint64, bits LSB first).
 * Format: DESIGN.md "Codec" (zfp 0.5.5 fixed-rate layout).  rate in 1..64. */
oocz_status oocz_zfp_encode(const float* d_in, int32_t nx, int32_t ny, int32_t nz,
                            int32_t rate, uint64_t* d_out, void* stream);
oocz_status oocz_zfp_decode(const uint64_t* d_in, int32_t nx, int32_t ny, int32_t nz,
                            int32_t rate, float* d_out, void* stream);
/* nsteps in-core leapfrog steps on a whole nx*ny*nz grid with a zero Dirichlet ghost of
 * depth 4: (u, uprev) <- (2u - uprev + m L(u), u), arithmetic order of DESIGN.md R5.
 * On return d_u holds the newest level and d_uprev the one before. */
oocz_status oocz_stencil_steps(float* d_u, float* d_uprev, const float* d_m,
                               int32_t nx, int32_t ny, int32_t nz, const float c[5],
                               int32_t nsteps, void* stream);
/* one step restricted to planes [z0, z1) of an nz-plane array: d_uprev[z] <- u+ there,
 * nothing else written; planes outside [zv0, zv1) of d_u are read as zero (ghost).
 * This is the engine's cone-limited primitive (temporal blocking). */
oocz_status oocz_stencil_step_planes(const float* d_u, float* d_uprev, const float* d_m,
                                     int32_t nx, int32_t ny, int32_t nz, const float c[5],
                                     int32_t z0, int32_t z1, int32_t zv0, int32_t zv1,
                                     void* stream);
/* fp64 twins (the paper's own precision; rates 32/64 and 24/64 at
 * PAPER.md:213-215).  Format: the same layout with an 11-bit exponent (bias 1023),
 * a 12-bit header and 64 bit planes, q = trunc(x 2^(62 - emax)) (DESIGN.md
 * "Codec", fp64).  Same sizes (8 * rate bytes per 4^3 block), same block order. */
oocz_status oocz_zfp_encode_f64(const double* d_in, int32_t nx, int32_t ny, int32_t nz,
                                int32_t rate, uint64_t* d_out, void* stream);
oocz_status oocz_zfp_decode_f64(const uint64_t* d_in, int32_t nx, int32_t ny, int32_t nz,
                                int32_t rate, double* d_out, void* stream);
/* fp64 stencil: the same step in fp64 arithmetic (same order, fl64(3 c0)) */
oocz_status oocz_stencil_steps_f64(double* d_u, double* d_uprev, const double* d_m,
                                   int32_t nx, int32_t ny, int32_t nz, const double c[5],
                                   int32_t nsteps, void* stream);
oocz_status oocz_stencil_step_planes_f64(const double* d_u, double* d_uprev, const double* d_m,
                                         int32_t nx, int32_t ny, int32_t nz, const double c[5],
                                         int32_t z0, int32_t z1, int32_t zv0, int32_t zv1,
                                         void* stream);
/* number of this library's kernels launched by this process so far */
uint64_t    oocz_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* OOCZ_H */
