// halo.h -- radius-4 z-halo exchange between z-slabs (reading R20).
//
// Rank g owns planes [gS, (g+1)S).  Its first block needs the h = 4T planes
// above the slab, its last block the h planes below, both at the sweep's
// start time t.  They travel in COMPRESSED form (the same fixed-rate bytes
// the neighbour's own store holds), so a partitioned run decodes exactly the
// round-tripped values a single-GPU run would: results are bit-identical to
// world = 1.  The read-only m halos are exchanged once.
//
// Per sweep, on the compute stream:
//   capture : block 0 encodes its planes [0, h) into send_top, block D-1 its
//             planes [S-h, S) into send_bot (time t+T, for the next sweep);
//             set_field fills them from the store for the first sweep;
//   begin   : send_bot -> rank g+1's recv_top, send_top -> rank g-1's recv_bot
//             (NCCL send/recv in one group; or device copies for the local
//             in-process group used to test the logic on one GPU);
//   insert  : block 0 decodes recv_top into slab planes [0, h), block D-1
//             decodes recv_bot into slab planes [P+h, P+2h).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <string>

namespace oocz {

struct HaloComm;

bool halo_get_unique_id(uint8_t id[128]);
size_t halo_device_bytes(size_t plane_elems, int h, const int rate[3], const size_t row_bytes[3]);
// NCCL transport (one process per GPU); esz = element size (4: fp32, 8: fp64)
HaloComm* halo_create(int rank, int world, const uint8_t* id, int device, size_t plane_elems, int esz, int h,
                      const int rate[3], const size_t row_bytes[3], std::string* err);
// in-process transport: `world` halves sharing one registry (local group)
HaloComm** halo_create_local_group(int world, int device, size_t plane_elems, int esz, int h, const int rate[3],
                                   const size_t row_bytes[3], std::string* err);
void halo_destroy(HaloComm* hc);

// copy the store's first / last h planes of a read-write field into the send buffers
bool halo_capture_store(HaloComm* hc, int field, const uint8_t* store, bool host_store, int S,
                        size_t row_bytes, cudaStream_t s, std::string* err);
// m: fill send buffers from the store and mark the m halos stale (exchanged at the next sweep)
bool halo_exchange_m(HaloComm* hc, const uint8_t* store_m, bool host_store, int S, size_t row_bytes,
                     cudaStream_t s, std::string* err);
bool halo_sweep_begin(HaloComm* hc, cudaStream_t s, std::string* err);
bool halo_insert(HaloComm* hc, bool first_block, bool last_block, uint8_t* const slab[3], int slab0, int S,
                 int nx, int ny, cudaStream_t s, std::string* err);
bool halo_capture(HaloComm* hc, bool first_block, bool last_block, const uint8_t* const own[2], int P, int nx,
                  int ny, cudaStream_t s, std::string* err);
uint64_t halo_bytes_sent(const HaloComm* hc);

}  // namespace oocz
