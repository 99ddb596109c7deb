// halo.cu -- z-halo exchange between z-slabs: NCCL point-to-point between
// processes (one per GPU), or device copies inside one process (local group).
// Protocol: halo.h.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"
#include "halo.h"

namespace oocz {
namespace {

// NCCL is resolved at run time (dlopen) so that the library links without it
// and shares the libnccl.so.2 that torch already loaded, if any.
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;   // optional
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.CommAbort = reinterpret_cast<decltype(api.CommAbort)>(sym("ncclCommAbort"));
        api.CommGetAsyncError = reinterpret_cast<decltype(api.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
        api.CommSplit = reinterpret_cast<decltype(api.CommSplit)>(sym("ncclCommSplit"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.CommAbort &&
                 api.CommGetAsyncError && api.GroupStart && api.GroupEnd && api.Send && api.Recv &&
                 api.GetErrorString;
    });
    return api;
}

struct LocalGroup {
    std::vector<HaloComm*> members;
    int alive = 0;
};

}  // namespace

// Directions (halo.h): "dn" carries rank g's bottom planes to rank g+1 (its
// top halo), "up" carries rank g's top planes to rank g-1 (its bottom halo).
struct HaloComm {
    int rank = 0, world = 1;
    LocalGroup* group = nullptr;          // non-null: in-process transport
    ncclComm_t comm_dn = nullptr;         // NCCL: one communicator per direction, so the two
    ncclComm_t comm_up = nullptr;         // directions complete independently (== comm_dn if one group)
    bool one_group = false;               // both directions in one group on one stream (A/B, or no CommSplit)
    int h = 0;
    size_t plane_elems = 0;
    int esz = 4;                          // element size: 4 fp32, 8 fp64
    int rate[3] = {0, 0, 0};
    size_t bytes[3] = {0, 0, 0};          // h planes of each field, as stored
    uint8_t* send_top[3] = {};
    uint8_t* send_bot[3] = {};
    uint8_t* recv_top[3] = {};
    uint8_t* recv_bot[3] = {};
    bool m_pending = false;
    cudaStream_t s_dn = nullptr, s_up = nullptr;
    // capture done (send buffer holds the next halo), transfer done (recv buffer
    // filled, send buffer free again), insert done (recv buffer consumed)
    cudaEvent_t ev_capt_top = nullptr, ev_capt_bot = nullptr;
    cudaEvent_t ev_dn = nullptr, ev_up = nullptr;
    cudaEvent_t ev_ins_top = nullptr, ev_ins_bot = nullptr;
    std::vector<cudaEvent_t> progress;    // one per exchange of the current step call (NCCL watchdog)
    size_t progress_used = 0;
    uint64_t sent = 0;
};

namespace {

bool set_err(std::string* err, const std::string& m) { if (err) *err = m; return false; }

bool cuda_ok(cudaError_t e, std::string* err, const char* what)
{
    if (e == cudaSuccess) return true;
    return set_err(err, std::string(what) + ": " + cudaGetErrorString(e));
}

bool nccl_ok(ncclResult_t r, std::string* err, const char* what)
{
    if (r == ncclSuccess) return true;
    return set_err(err, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
}

HaloComm* alloc_halo(int rank, int world, int device, size_t plane_elems, int esz, int h, const int rate[3],
                     const size_t row_bytes[3], std::string* err)
{
    HaloComm* hc = new HaloComm;
    hc->rank = rank; hc->world = world; hc->h = h; hc->plane_elems = plane_elems; hc->esz = esz;
    const char* og = getenv("OOCZ_HALO_ONE_GROUP");
    hc->one_group = og && og[0] == '1';
    bool ok = cuda_ok(cudaSetDevice(device), err, "cudaSetDevice");
    for (int f = 0; f < 3 && ok; f++) {
        hc->rate[f] = rate[f];
        hc->bytes[f] = (size_t)(h / 4) * row_bytes[f];
        ok = cuda_ok(cudaMalloc(&hc->send_top[f], hc->bytes[f]), err, "cudaMalloc") &&
             cuda_ok(cudaMalloc(&hc->send_bot[f], hc->bytes[f]), err, "cudaMalloc") &&
             cuda_ok(cudaMalloc(&hc->recv_top[f], hc->bytes[f]), err, "cudaMalloc") &&
             cuda_ok(cudaMalloc(&hc->recv_bot[f], hc->bytes[f]), err, "cudaMalloc");
    }
    for (cudaEvent_t* e : {&hc->ev_capt_top, &hc->ev_capt_bot, &hc->ev_dn, &hc->ev_up, &hc->ev_ins_top,
                           &hc->ev_ins_bot})
        ok = ok && cuda_ok(cudaEventCreateWithFlags(e, cudaEventDisableTiming), err, "event");
    ok = ok && cuda_ok(cudaStreamCreateWithFlags(&hc->s_dn, cudaStreamNonBlocking), err, "stream") &&
         cuda_ok(cudaStreamCreateWithFlags(&hc->s_up, cudaStreamNonBlocking), err, "stream");
    if (!ok) { halo_destroy(hc); return nullptr; }
    return hc;
}

cudaError_t code(const HaloComm* hc, int f, const uint8_t* src, int nx, int ny, uint8_t* dst, cudaStream_t s)
{
    return field_encode(src, hc->esz, nx, ny, hc->h, hc->rate[f], dst, s);
}

cudaError_t uncode(const HaloComm* hc, int f, const uint8_t* src, int nx, int ny, uint8_t* dst, cudaStream_t s)
{
    return field_decode(src, hc->esz, nx, ny, hc->h, hc->rate[f], dst, s);
}

bool fill_from_store(HaloComm* hc, int f, const uint8_t* top, const uint8_t* bot, cudaStream_t s, std::string* err)
{
    // pinned host or device rows: unified addressing tells the copy which
    const size_t n = hc->bytes[f];
    return cuda_ok(cudaMemcpyAsync(hc->send_top[f], top, n, cudaMemcpyDefault, s), err, "halo fill") &&
           cuda_ok(cudaMemcpyAsync(hc->send_bot[f], bot, n, cudaMemcpyDefault, s), err, "halo fill");
}

// One NCCL group: send `snd` to peer `to`, receive `rcv` from peer `from` (either
// peer may be absent, -1), fields [0, nf).  ncclGroupEnd is always called once
// ncclGroupStart succeeded, also when a send / recv fails to enqueue.
bool nccl_pair(HaloComm* hc, ncclComm_t comm, uint8_t* const snd[3], int to, uint8_t* const rcv[3], int from,
               int nf, cudaStream_t s, std::string* err)
{
    NcclApi& n = nccl();
    if (!nccl_ok(n.GroupStart(), err, "ncclGroupStart")) return false;
    bool ok = true;
    for (int f = 0; f < nf && ok; f++) {
        if (to >= 0) {
            ok = nccl_ok(n.Send(snd[f], hc->bytes[f], ncclUint8, to, comm, s), err, "ncclSend");
            if (ok) hc->sent += hc->bytes[f];
        }
        if (ok && from >= 0) ok = nccl_ok(n.Recv(rcv[f], hc->bytes[f], ncclUint8, from, comm, s), err, "ncclRecv");
    }
    const ncclResult_t e = n.GroupEnd();
    return ok && nccl_ok(e, err, "ncclGroupEnd");
}

void abort_comms(HaloComm* hc)
{
    if (!nccl().ok) return;
    if (hc->comm_up && hc->comm_up != hc->comm_dn) nccl().CommAbort(hc->comm_up);
    if (hc->comm_dn) nccl().CommAbort(hc->comm_dn);
    hc->comm_up = hc->comm_dn = nullptr;
}

}  // namespace

bool halo_get_unique_id(uint8_t id[128])
{
    if (!nccl().ok) return false;
    ncclUniqueId u;
    if (nccl().GetUniqueId(&u) != ncclSuccess) return false;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(id, &u, 128);
    return true;
}

size_t halo_device_bytes(size_t, int h, const int[3], const size_t row_bytes[3])
{
    size_t t = 0;
    for (int f = 0; f < 3; f++) t += 4 * (size_t)(h / 4) * row_bytes[f];
    return t;
}

HaloComm* halo_create(int rank, int world, const uint8_t* id, int device, size_t plane_elems, int esz, int h,
                      const int rate[3], const size_t row_bytes[3], std::string* err)
{
    if (!nccl().ok) { set_err(err, "libnccl.so.2 not loadable"); return nullptr; }
    HaloComm* hc = alloc_halo(rank, world, device, plane_elems, esz, h, rate, row_bytes, err);
    if (!hc) return nullptr;
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    if (!nccl_ok(nccl().CommInitRank(&hc->comm_dn, world, u, rank), err, "ncclCommInitRank")) {
        halo_destroy(hc);
        return nullptr;
    }
    // the second direction gets its own communicator (collective over the world)
    if (!hc->one_group && nccl().CommSplit) {
        if (!nccl_ok(nccl().CommSplit(hc->comm_dn, 0, rank, &hc->comm_up, nullptr), err, "ncclCommSplit")) {
            halo_destroy(hc);
            return nullptr;
        }
    } else {
        hc->one_group = true;
        hc->comm_up = hc->comm_dn;
    }
    return hc;
}

HaloComm** halo_create_local_group(int world, int device, size_t plane_elems, int esz, int h, const int rate[3],
                                   const size_t row_bytes[3], std::string* err)
{
    LocalGroup* g = new LocalGroup;
    for (int r = 0; r < world; r++) {
        HaloComm* hc = alloc_halo(r, world, device, plane_elems, esz, h, rate, row_bytes, err);
        if (!hc) {
            for (auto* m : g->members) halo_destroy(m);
            delete g;
            return nullptr;
        }
        hc->group = g;
        g->members.push_back(hc);
    }
    g->alive = world;
    return g->members.data();
}

void halo_destroy(HaloComm* hc)
{
    if (!hc) return;
    if (hc->s_dn) cudaStreamSynchronize(hc->s_dn);
    if (hc->s_up) cudaStreamSynchronize(hc->s_up);
    if (nccl().ok) {
        if (hc->comm_up && hc->comm_up != hc->comm_dn) nccl().CommDestroy(hc->comm_up);
        if (hc->comm_dn) nccl().CommDestroy(hc->comm_dn);
    }
    for (int f = 0; f < 3; f++) {
        cudaFree(hc->send_top[f]); cudaFree(hc->send_bot[f]);
        cudaFree(hc->recv_top[f]); cudaFree(hc->recv_bot[f]);
    }
    for (cudaEvent_t e : {hc->ev_capt_top, hc->ev_capt_bot, hc->ev_dn, hc->ev_up, hc->ev_ins_top, hc->ev_ins_bot})
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : hc->progress) cudaEventDestroy(e);
    if (hc->s_dn) cudaStreamDestroy(hc->s_dn);
    if (hc->s_up) cudaStreamDestroy(hc->s_up);
    if (hc->group) {
        LocalGroup* g = hc->group;
        for (auto*& m : g->members) if (m == hc) m = nullptr;
        if (--g->alive == 0) delete g;
    }
    delete hc;
}

bool halo_capture_store(HaloComm* hc, int field, const uint8_t* top, const uint8_t* bot, cudaStream_t s,
                        std::string* err)
{
    // the previous transfers must be done reading the send buffers
    return cuda_ok(cudaStreamWaitEvent(s, hc->ev_dn, 0), err, "wait") &&
           cuda_ok(cudaStreamWaitEvent(s, hc->ev_up, 0), err, "wait") &&
           fill_from_store(hc, field, top, bot, s, err) &&
           cuda_ok(cudaEventRecord(hc->ev_capt_top, s), err, "event") &&
           cuda_ok(cudaEventRecord(hc->ev_capt_bot, s), err, "event");
}

bool halo_exchange_m(HaloComm* hc, const uint8_t* top, const uint8_t* bot, cudaStream_t s, std::string* err)
{
    if (!cuda_ok(cudaStreamWaitEvent(s, hc->ev_dn, 0), err, "wait") ||
        !cuda_ok(cudaStreamWaitEvent(s, hc->ev_up, 0), err, "wait") ||
        !fill_from_store(hc, 2, top, bot, s, err))
        return false;
    if (!cuda_ok(cudaStreamSynchronize(s), err, "sync")) return false;
    hc->m_pending = true;
    return true;
}

void halo_step_begin(HaloComm* hc)
{
    if (hc) hc->progress_used = 0;
}

bool halo_sweep_begin(HaloComm* hc, std::string* err)
{
    const int nf = hc->m_pending ? 3 : 2;
    const bool up = hc->rank > 0, down = hc->rank < hc->world - 1;
    // stream of each direction: with one group both run on s_dn, one after the other
    cudaStream_t sdn = hc->s_dn, sup = hc->one_group ? hc->s_dn : hc->s_up;
    HaloComm* above = nullptr;
    HaloComm* below = nullptr;
    if (hc->group) {
        above = up ? hc->group->members[hc->rank - 1] : nullptr;
        below = down ? hc->group->members[hc->rank + 1] : nullptr;
        if ((up && !above) || (down && !below)) return set_err(err, "local group member destroyed");
    }
    // dn: my send_bot (captured by my last block) -> rank+1; rank-1's -> my recv_top,
    // once my first block has consumed the previous recv_top
    bool ok = cuda_ok(cudaStreamWaitEvent(sdn, hc->ev_capt_bot, 0), err, "wait") &&
              cuda_ok(cudaStreamWaitEvent(sdn, hc->ev_ins_top, 0), err, "wait");
    if (ok && hc->one_group)
        ok = cuda_ok(cudaStreamWaitEvent(sdn, hc->ev_capt_top, 0), err, "wait") &&
             cuda_ok(cudaStreamWaitEvent(sdn, hc->ev_ins_bot, 0), err, "wait");
    if (!ok) return false;
    if (hc->group) {
        // receiver-driven device copies: the sender's capture must be done
        if (above) {
            if (!cuda_ok(cudaStreamWaitEvent(sdn, above->ev_capt_bot, 0), err, "wait")) return false;
            for (int f = 0; f < nf; f++)
                if (!cuda_ok(cudaMemcpyAsync(hc->recv_top[f], above->send_bot[f], hc->bytes[f],
                                             cudaMemcpyDeviceToDevice, sdn), err, "halo copy"))
                    return false;
        }
        for (int f = 0; f < nf && down; f++) hc->sent += hc->bytes[f];   // what a real transport sends
    } else if (!nccl_pair(hc, hc->comm_dn, hc->send_bot, down ? hc->rank + 1 : -1, hc->recv_top,
                          up ? hc->rank - 1 : -1, nf, sdn, err)) {
        return false;
    }
    if (!cuda_ok(cudaEventRecord(hc->ev_dn, sdn), err, "event")) return false;
    // up: my send_top (captured by my first block) -> rank-1; rank+1's -> my recv_bot
    if (!hc->one_group &&
        !(cuda_ok(cudaStreamWaitEvent(sup, hc->ev_capt_top, 0), err, "wait") &&
          cuda_ok(cudaStreamWaitEvent(sup, hc->ev_ins_bot, 0), err, "wait")))
        return false;
    if (hc->group) {
        if (below) {
            if (!cuda_ok(cudaStreamWaitEvent(sup, below->ev_capt_top, 0), err, "wait")) return false;
            for (int f = 0; f < nf; f++)
                if (!cuda_ok(cudaMemcpyAsync(hc->recv_bot[f], below->send_top[f], hc->bytes[f],
                                             cudaMemcpyDeviceToDevice, sup), err, "halo copy"))
                    return false;
        }
        for (int f = 0; f < nf && up; f++) hc->sent += hc->bytes[f];
    } else if (!nccl_pair(hc, hc->comm_up, hc->send_top, up ? hc->rank - 1 : -1, hc->recv_bot,
                          down ? hc->rank + 1 : -1, nf, sup, err)) {
        return false;
    }
    if (!cuda_ok(cudaEventRecord(hc->ev_up, sup), err, "event")) return false;
    // watchdog progress marker: both directions of this exchange done
    if (hc->progress_used == hc->progress.size()) {
        cudaEvent_t e;
        if (!cuda_ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), err, "event")) return false;
        hc->progress.push_back(e);
    }
    cudaEvent_t pe = hc->progress[hc->progress_used++];
    if (!cuda_ok(cudaStreamWaitEvent(sdn, hc->ev_up, 0), err, "wait") ||
        !cuda_ok(cudaEventRecord(pe, sdn), err, "event"))
        return false;
    hc->m_pending = false;
    return true;
}

bool halo_insert(HaloComm* hc, bool first_block, bool last_block, uint8_t* const slab[3], int slab0, int S,
                 int nx, int ny, cudaStream_t s, std::string* err)
{
    if (first_block && hc->rank > 0) {
        if (!cuda_ok(cudaStreamWaitEvent(s, hc->ev_dn, 0), err, "wait")) return false;
        for (int f = 0; f < 3; f++)
            if (!cuda_ok(uncode(hc, f, hc->recv_top[f], nx, ny, slab[f], s), err, "halo decode")) return false;
        if (!cuda_ok(cudaEventRecord(hc->ev_ins_top, s), err, "event")) return false;
    }
    if (last_block && hc->rank < hc->world - 1) {
        if (!cuda_ok(cudaStreamWaitEvent(s, hc->ev_up, 0), err, "wait")) return false;
        for (int f = 0; f < 3; f++)
            if (!cuda_ok(uncode(hc, f, hc->recv_bot[f], nx, ny, slab[f] + (size_t)(S - slab0) * hc->plane_elems * hc->esz, s),
                         err, "halo decode"))
                return false;
        if (!cuda_ok(cudaEventRecord(hc->ev_ins_bot, s), err, "event")) return false;
    }
    return true;
}

bool halo_capture(HaloComm* hc, bool first_block, bool last_block, const uint8_t* const own[2], int P, int nx,
                  int ny, cudaStream_t s, std::string* err)
{
    // a send buffer is rewritten once the transfer that reads it is done: the own
    // NCCL group, or, in a local group, the neighbour's copy out of it
    if (first_block && hc->rank > 0) {
        const cudaEvent_t done = hc->group ? hc->group->members[hc->rank - 1]->ev_up : hc->ev_up;
        if (!cuda_ok(cudaStreamWaitEvent(s, done, 0), err, "wait")) return false;
        for (int f = 0; f < 2; f++)
            if (!cuda_ok(code(hc, f, own[f], nx, ny, hc->send_top[f], s), err, "halo encode")) return false;
        if (!cuda_ok(cudaEventRecord(hc->ev_capt_top, s), err, "event")) return false;
    }
    if (last_block && hc->rank < hc->world - 1) {
        const cudaEvent_t done = hc->group ? hc->group->members[hc->rank + 1]->ev_dn : hc->ev_dn;
        if (!cuda_ok(cudaStreamWaitEvent(s, done, 0), err, "wait")) return false;
        for (int f = 0; f < 2; f++)
            if (!cuda_ok(code(hc, f, own[f] + (size_t)(P - hc->h) * hc->plane_elems * hc->esz, nx, ny, hc->send_bot[f], s), err,
                         "halo encode"))
                return false;
        if (!cuda_ok(cudaEventRecord(hc->ev_capt_bot, s), err, "event")) return false;
    }
    return true;
}

bool halo_wait(HaloComm* hc, cudaEvent_t done, std::string* err)
{
    if (!hc || hc->group) return true;            // device copies cannot hang on a peer
    // NCCL: poll instead of blocking, so that an asynchronous communicator error
    // (a dead peer, a network failure) or a stall surfaces as an error instead of a hang
    const char* t = getenv("OOCZ_NCCL_TIMEOUT_S");
    const double timeout = t ? atof(t) : 600.0;   // seconds without any completed exchange
    size_t seen = 0;
    auto last = std::chrono::steady_clock::now();
    for (;;) {
        const cudaError_t q = cudaEventQuery(done);
        if (q == cudaSuccess) return true;
        if (q != cudaErrorNotReady) return cuda_ok(q, err, "cudaEventQuery");
        for (ncclComm_t c : {hc->comm_dn, hc->comm_up}) {
            ncclResult_t ae = ncclSuccess;
            if (c && nccl().CommGetAsyncError(c, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress) {
                set_err(err, std::string("NCCL asynchronous error: ") + nccl().GetErrorString(ae));
                abort_comms(hc);
                return false;
            }
        }
        while (seen < hc->progress_used && cudaEventQuery(hc->progress[seen]) == cudaSuccess) {
            seen++;
            last = std::chrono::steady_clock::now();
        }
        if (timeout > 0 &&
            std::chrono::duration<double>(std::chrono::steady_clock::now() - last).count() > timeout) {
            set_err(err, "no halo exchange completed for " + std::to_string(timeout) +
                             " s (OOCZ_NCCL_TIMEOUT_S): communicators aborted");
            abort_comms(hc);
            return false;
        }
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
}

bool halo_join(HaloComm* hc, cudaStream_t s, std::string* err)
{
    return cuda_ok(cudaStreamWaitEvent(s, hc->ev_dn, 0), err, "wait") &&
           cuda_ok(cudaStreamWaitEvent(s, hc->ev_up, 0), err, "wait");
}

uint64_t halo_bytes_sent(const HaloComm* hc) { return hc ? hc->sent : 0; }

bool halo_one_group(const HaloComm* hc) { return hc && hc->one_group; }

}  // namespace oocz
