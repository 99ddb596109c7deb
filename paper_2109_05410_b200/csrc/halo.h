// halo.h -- radius-4 z-halo exchange between z-slabs (reading R20).
//
// Rank g owns planes [gS, (g+1)S).  Its first block (i = 0) needs the h = 4T
// planes above the slab, its last block (i = D-1) the h planes below, both at
// the sweep's start time t.  They travel in COMPRESSED form (the same
// fixed-rate bytes the neighbour's own store holds), so a partitioned run
// decodes exactly the round-tripped values a single-GPU run would: results are
// bit-identical to world = 1.  The read-only m halos are exchanged once.
//
// Two independent directions, each with its own stream (and, with NCCL, its
// own communicator, so neither waits for the other):
//   dn : rank g's send_bot -> rank g+1's recv_top (rank g+1's block 0 needs it)
//   up : rank g's send_top -> rank g-1's recv_bot (rank g-1's block D-1 needs it)
// Per sweep:
//   capture : block 0 encodes its planes [0, h) into send_top, block D-1 its
//             planes [S-h, S) into send_bot (time t+T, for the next sweep),
//             once the previous transfer out of that buffer is done;
//             set_field fills them from the store for the first sweep;
//   begin   : each direction waits for its own capture and for the previous
//             sweep's insert out of its receive buffer, then transfers (NCCL
//             send/recv group, or device copies in an in-process local group);
//   insert  : block 0 decodes recv_top into slab planes [0, h) after the dn
//             transfer, block D-1 decodes recv_bot into [P+h, P+2h) after up.
// So a rank's first block waits only for the neighbour's LAST block of the
// previous sweep (ascending sweeps: inherent; serpentine sweeps turn it into
// the neighbour's FIRST block of the previous sweep, i.e. no per-sweep drain),
// never for a whole sweep's encodes.  OOCZ_HALO_ONE_GROUP=1 puts both
// directions into one group on one stream (the round-1 protocol, for A/B).
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
// (top / bot: the stored rows of planes [0, h) and [S - h, S), each in host or
// device memory -- a store split by resident_blocks has one of each)
bool halo_capture_store(HaloComm* hc, int field, const uint8_t* top, const uint8_t* bot, cudaStream_t s,
                        std::string* err);
// m: fill send buffers from the store and mark the m halos stale (exchanged at the next sweep)
bool halo_exchange_m(HaloComm* hc, const uint8_t* top, const uint8_t* bot, cudaStream_t s, std::string* err);
// start of an oocz_step call (resets the watchdog's progress markers)
void halo_step_begin(HaloComm* hc);
bool halo_sweep_begin(HaloComm* hc, std::string* err);
bool halo_insert(HaloComm* hc, bool first_block, bool last_block, uint8_t* const slab[3], int slab0, int S,
                 int nx, int ny, cudaStream_t s, std::string* err);
bool halo_capture(HaloComm* hc, bool first_block, bool last_block, const uint8_t* const own[2], int P, int nx,
                  int ny, cudaStream_t s, std::string* err);
// make stream s wait for both directions' latest transfers
bool halo_join(HaloComm* hc, cudaStream_t s, std::string* err);
// NCCL: wait for event `done` while polling ncclCommGetAsyncError and a progress
// watchdog (OOCZ_NCCL_TIMEOUT_S seconds without a completed exchange, default
// 600, 0 = none); on failure the communicators are aborted and false returned.
// Local groups return immediately (true).
bool halo_wait(HaloComm* hc, cudaEvent_t done, std::string* err);
uint64_t halo_bytes_sent(const HaloComm* hc);
bool halo_one_group(const HaloComm* hc);

}  // namespace oocz
