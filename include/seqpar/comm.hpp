// B200 mirror of the reference communication API (/root/reference/proj/include/seqpar/comm.hpp).
//
// The reference runs ranks as threads over an in-process rendezvous fabric (comm.cpp:160-231).
// Here a rank is a GPU stream with a Transport:
//   * NcclTransport     — one process per GPU, NCCL over NVLink/NVSwitch (grouped send/recv);
//   * LoopbackFabric    — the CommFabric analog: `world` ranks as host threads sharing ONE
//                         device, each with its own stream; collectives are stream-ordered
//                         peer reads of device memory (the same copy kernels an NVSwitch
//                         peer-memory path runs), or emulated messages (force_messages) so the
//                         NCCL pack -> send/recv -> unpack code path is testable on one GPU.
// Byte counters are send-side per primitive per rank, like PrimitiveStats (comm.hpp:30-33).
#pragma once
#include <cuda_runtime.h>

#include <array>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "seqpar/partition.hpp"

namespace seqpar {

enum class Primitive { all_to_all = 0, all_gather, p2p, all_reduce, broadcast };  // comm.hpp:19
constexpr int kPrimitiveCount = 5;
const char* primitive_name(Primitive p);

struct PrimitiveStats {
  int64_t calls = 0;
  int64_t bytes = 0;
};

// comm.hpp:37-44: ordered rank list
struct CommGroup {
  std::vector<int> ranks;
  int size() const { return static_cast<int>(ranks.size()); }
  int index_of(int rank) const;
  bool contains(int rank) const;
  std::string key() const;
};

// Raised in ranks blocked on a rendezvous after a peer failed (comm.cpp:10-14).
struct PeerAbort : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Msg {
  int peer;  // index within the group
  void* ptr;
  size_t bytes;
};

class Transport {
 public:
  virtual ~Transport() = default;
  // true when peers' device pointers may be read directly (same device / mapped peer memory)
  virtual bool peer_access() const = 0;
  // Publish `mine` (ready once the work queued so far on `stream` completes); returns every
  // member's pointer in group order and makes `stream` wait for every member's readiness.
  virtual std::vector<void*> exchange_ptrs(const CommGroup& g, int my_rank, void* mine,
                                           cudaStream_t stream) = 0;
  // Ends a peer-read phase: `stream`'s reads are done; waits for every member's reads.
  virtual void release(const CommGroup& g, int my_rank, cudaStream_t stream) = 0;
  // Grouped point-to-point messages on `stream` (all sends and receives in one group call).
  virtual void send_recv(const CommGroup& g, int my_rank, const std::vector<Msg>& sends,
                         const std::vector<Msg>& recvs, cudaStream_t stream) = 0;
  // Diagnostics (collective over every rank of the transport): a message of `bytes` to this
  // rank itself through every entry point the transport uses; throws on a mismatch.
  virtual void self_test(int my_rank, size_t bytes, cudaStream_t stream);
};

// comm.hpp:63-82 RankCtx: this rank's transport, SP group, stream and counters.
struct RankCtx {
  Transport* transport = nullptr;
  int rank = 0;
  int device = 0;
  CommGroup sp_group;
  cudaStream_t stream = nullptr;       // compute stream (caller-provided or owned)
  cudaStream_t comm_stream = nullptr;  // collectives overlapped with compute (ring)
  std::array<PrimitiveStats, kPrimitiveCount> stats{};
  int64_t flops = 0;

  void count(Primitive p, int64_t bytes) {
    auto& s = stats[static_cast<int>(p)];
    ++s.calls;
    s.bytes += bytes;
  }
  void add_flops(int64_t n) { flops += n; }
  int64_t total_bytes() const {
    int64_t t = 0;
    for (const auto& s : stats) t += s.bytes;
    return t;
  }
  void reset_stats() {
    stats = {};
    flops = 0;
  }
};

// CommFabric analog (comm.cpp:185-231): `world` ranks as threads on one device; SP groups are
// consecutive ranks (sp_group_of, comm.cpp:81-87). run() rethrows the first rank error by rank
// order; blocked peers see PeerAbort.
class LoopbackFabric {
 public:
  LoopbackFabric(int world, int sp, int device, bool force_messages = false);
  ~LoopbackFabric();
  int world_size() const { return world_; }
  int sp() const { return sp_; }
  CommGroup sp_group_of(int rank) const;
  RankCtx& ctx(int rank) { return *ctxs_[static_cast<size_t>(rank)]; }
  void run(const std::function<void(RankCtx&)>& body);
  void set_force_messages(bool on) { force_messages_ = on; }

  struct Deposit {
    void* ptr = nullptr;
    cudaEvent_t ev = nullptr;
    std::shared_ptr<std::vector<Msg>> sends;
  };
  std::vector<Deposit> rendezvous(const CommGroup& g, int my_rank, Deposit d);
  bool force_messages() const { return force_messages_; }

 private:
  struct Slot {
    std::vector<Deposit> dep;
    std::vector<Deposit> result[2];
    int arrived = 0;
    uint64_t gen = 0;
  };
  int world_, sp_, device_;
  bool force_messages_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::map<std::string, Slot> slots_;
  bool abort_ = false;
  std::vector<std::unique_ptr<Transport>> transports_;
  std::vector<std::unique_ptr<RankCtx>> ctxs_;
  std::vector<cudaStream_t> own_streams_;
};

// One process per GPU; NCCL loaded at run time (libnccl.so.2, the copy torch already mapped).
// `unique_id` is the 128-byte ncclUniqueId rank 0 created (spattn_nccl_unique_id) and the
// launcher broadcast.
// broadcast_bytes (comm.hpp:159-161, comm.cpp:526-545): the root RANK's bytes reach every member;
// counted as bytes * (g - 1) / g per rank. ConfigError when root is not in the group.
std::vector<uint8_t> broadcast_bytes(RankCtx& ctx, const CommGroup& group, const std::vector<uint8_t>& payload,
                                     int root);

// replicate_packing_mask (partition.cpp:222-227) over broadcast_bytes (comm.cpp:526-545):
// group index 0 supplies the neat-packing mask (other ranks pass anything, e.g. empty); every
// member returns the root's bytes. The mask is replicated, not split. Counted
// as one broadcast of size*(g-1)/g bytes per rank, as the reference counts it.
std::vector<uint8_t> replicate_packing_mask(RankCtx& ctx, const CommGroup& group,
                                            const std::vector<uint8_t>& mask);

std::unique_ptr<Transport> make_nccl_transport(int rank, int world, const void* unique_id,
                                               int device);
void nccl_unique_id(void* out128);

}  // namespace seqpar
