// halo.cu -- z-halo exchange between z-slabs: NCCL point-to-point between
// processes (one per GPU), or device copies inside one process (local group).
// Protocol: halo.h.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
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
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart && api.GroupEnd &&
                 api.Send && api.Recv && api.GetErrorString;
    });
    return api;
}

struct LocalGroup {
    std::vector<HaloComm*> members;
    int alive = 0;
};

}  // namespace

struct HaloComm {
    int rank = 0, world = 1;
    LocalGroup* group = nullptr;          // non-null: in-process transport
    ncclComm_t comm = nullptr;
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
    cudaEvent_t ev_capt_top = nullptr, ev_capt_bot = nullptr, ev_recv_top = nullptr, ev_recv_bot = nullptr;
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
    bool ok = cuda_ok(cudaSetDevice(device), err, "cudaSetDevice");
    for (int f = 0; f < 3 && ok; f++) {
        hc->rate[f] = rate[f];
        hc->bytes[f] = (size_t)(h / 4) * row_bytes[f];
        ok = cuda_ok(cudaMalloc(&hc->send_top[f], hc->bytes[f]), err, "cudaMalloc") &&
             cuda_ok(cudaMalloc(&hc->send_bot[f], hc->bytes[f]), err, "cudaMalloc") &&
             cuda_ok(cudaMalloc(&hc->recv_top[f], hc->bytes[f]), err, "cudaMalloc") &&
             cuda_ok(cudaMalloc(&hc->recv_bot[f], hc->bytes[f]), err, "cudaMalloc");
    }
    ok = ok && cuda_ok(cudaEventCreateWithFlags(&hc->ev_capt_top, cudaEventDisableTiming), err, "event") &&
         cuda_ok(cudaEventCreateWithFlags(&hc->ev_capt_bot, cudaEventDisableTiming), err, "event") &&
         cuda_ok(cudaEventCreateWithFlags(&hc->ev_recv_top, cudaEventDisableTiming), err, "event") &&
         cuda_ok(cudaEventCreateWithFlags(&hc->ev_recv_bot, cudaEventDisableTiming), err, "event");
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

bool fill_from_store(HaloComm* hc, int f, const uint8_t* store, bool host_store, int S, size_t row_bytes,
                     cudaStream_t s, std::string* err)
{
    const cudaMemcpyKind k = host_store ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    const size_t n = hc->bytes[f];
    return cuda_ok(cudaMemcpyAsync(hc->send_top[f], store, n, k, s), err, "halo fill") &&
           cuda_ok(cudaMemcpyAsync(hc->send_bot[f], store + (size_t)((S - hc->h) / 4) * row_bytes, n, k, s), err,
                   "halo fill");
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
    if (!nccl_ok(nccl().CommInitRank(&hc->comm, world, u, rank), err, "ncclCommInitRank")) {
        halo_destroy(hc);
        return nullptr;
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
    if (hc->comm && nccl().ok) nccl().CommDestroy(hc->comm);
    for (int f = 0; f < 3; f++) {
        cudaFree(hc->send_top[f]); cudaFree(hc->send_bot[f]);
        cudaFree(hc->recv_top[f]); cudaFree(hc->recv_bot[f]);
    }
    for (cudaEvent_t e : {hc->ev_capt_top, hc->ev_capt_bot, hc->ev_recv_top, hc->ev_recv_bot})
        if (e) cudaEventDestroy(e);
    if (hc->group) {
        LocalGroup* g = hc->group;
        for (auto*& m : g->members) if (m == hc) m = nullptr;
        if (--g->alive == 0) delete g;
    }
    delete hc;
}

bool halo_capture_store(HaloComm* hc, int field, const uint8_t* store, bool host_store, int S, size_t row_bytes,
                        cudaStream_t s, std::string* err)
{
    return fill_from_store(hc, field, store, host_store, S, row_bytes, s, err) &&
           cuda_ok(cudaEventRecord(hc->ev_capt_top, s), err, "event") &&
           cuda_ok(cudaEventRecord(hc->ev_capt_bot, s), err, "event");
}

bool halo_exchange_m(HaloComm* hc, const uint8_t* store_m, bool host_store, int S, size_t row_bytes,
                     cudaStream_t s, std::string* err)
{
    if (!fill_from_store(hc, 2, store_m, host_store, S, row_bytes, s, err)) return false;
    if (!cuda_ok(cudaStreamSynchronize(s), err, "sync")) return false;
    hc->m_pending = true;
    return true;
}

bool halo_sweep_begin(HaloComm* hc, cudaStream_t s, std::string* err)
{
    const int nf = hc->m_pending ? 3 : 2;
    const bool up = hc->rank > 0, down = hc->rank < hc->world - 1;
    if (hc->group) {
        HaloComm* above = up ? hc->group->members[hc->rank - 1] : nullptr;
        HaloComm* below = down ? hc->group->members[hc->rank + 1] : nullptr;
        if ((up && !above) || (down && !below)) return set_err(err, "local group member destroyed");
        if (above && !cuda_ok(cudaStreamWaitEvent(s, above->ev_capt_bot, 0), err, "wait")) return false;
        if (below && !cuda_ok(cudaStreamWaitEvent(s, below->ev_capt_top, 0), err, "wait")) return false;
        for (int f = 0; f < nf; f++) {
            if (above && !cuda_ok(cudaMemcpyAsync(hc->recv_top[f], above->send_bot[f], hc->bytes[f],
                                                  cudaMemcpyDeviceToDevice, s), err, "halo copy"))
                return false;
            if (below && !cuda_ok(cudaMemcpyAsync(hc->recv_bot[f], below->send_top[f], hc->bytes[f],
                                                  cudaMemcpyDeviceToDevice, s), err, "halo copy"))
                return false;
            // bytes a real transport would send from this rank
            hc->sent += (up ? hc->bytes[f] : 0) + (down ? hc->bytes[f] : 0);
        }
        if (!cuda_ok(cudaEventRecord(hc->ev_recv_top, s), err, "event") ||
            !cuda_ok(cudaEventRecord(hc->ev_recv_bot, s), err, "event"))
            return false;
    } else {
        NcclApi& n = nccl();
        if (!nccl_ok(n.GroupStart(), err, "ncclGroupStart")) return false;
        for (int f = 0; f < nf; f++) {
            if (down) {
                if (!nccl_ok(n.Send(hc->send_bot[f], hc->bytes[f], ncclUint8, hc->rank + 1, hc->comm, s), err, "ncclSend") ||
                    !nccl_ok(n.Recv(hc->recv_bot[f], hc->bytes[f], ncclUint8, hc->rank + 1, hc->comm, s), err, "ncclRecv"))
                    return false;
                hc->sent += hc->bytes[f];
            }
            if (up) {
                if (!nccl_ok(n.Send(hc->send_top[f], hc->bytes[f], ncclUint8, hc->rank - 1, hc->comm, s), err, "ncclSend") ||
                    !nccl_ok(n.Recv(hc->recv_top[f], hc->bytes[f], ncclUint8, hc->rank - 1, hc->comm, s), err, "ncclRecv"))
                    return false;
                hc->sent += hc->bytes[f];
            }
        }
        if (!nccl_ok(n.GroupEnd(), err, "ncclGroupEnd")) return false;
    }
    hc->m_pending = false;
    return true;
}

bool halo_insert(HaloComm* hc, bool first_block, bool last_block, uint8_t* const slab[3], int slab0, int S,
                 int nx, int ny, cudaStream_t s, std::string* err)
{
    if (first_block && hc->rank > 0)
        for (int f = 0; f < 3; f++)
            if (!cuda_ok(uncode(hc, f, hc->recv_top[f], nx, ny, slab[f], s), err, "halo decode")) return false;
    if (last_block && hc->rank < hc->world - 1)
        for (int f = 0; f < 3; f++)
            if (!cuda_ok(uncode(hc, f, hc->recv_bot[f], nx, ny, slab[f] + (size_t)(S - slab0) * hc->plane_elems * hc->esz, s),
                         err, "halo decode"))
                return false;
    return true;
}

bool halo_capture(HaloComm* hc, bool first_block, bool last_block, const uint8_t* const own[2], int P, int nx,
                  int ny, cudaStream_t s, std::string* err)
{
    if (first_block && hc->rank > 0) {
        if (hc->group && !cuda_ok(cudaStreamWaitEvent(s, hc->group->members[hc->rank - 1]->ev_recv_bot, 0), err, "wait"))
            return false;
        for (int f = 0; f < 2; f++)
            if (!cuda_ok(code(hc, f, own[f], nx, ny, hc->send_top[f], s), err, "halo encode")) return false;
        if (!cuda_ok(cudaEventRecord(hc->ev_capt_top, s), err, "event")) return false;
    }
    if (last_block && hc->rank < hc->world - 1) {
        if (hc->group && !cuda_ok(cudaStreamWaitEvent(s, hc->group->members[hc->rank + 1]->ev_recv_top, 0), err, "wait"))
            return false;
        for (int f = 0; f < 2; f++)
            if (!cuda_ok(code(hc, f, own[f] + (size_t)(P - hc->h) * hc->plane_elems * hc->esz, nx, ny, hc->send_bot[f], s), err,
                         "halo encode"))
                return false;
        if (!cuda_ok(cudaEventRecord(hc->ev_capt_bot, s), err, "event")) return false;
    }
    return true;
}

uint64_t halo_bytes_sent(const HaloComm* hc) { return hc ? hc->sent : 0; }

}  // namespace oocz
