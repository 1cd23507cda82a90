// Transports for the SP collectives: a single-device loopback fabric (ranks = host threads,
// mirroring CommFabric, /root/reference/proj/src/comm.cpp:127-231) and NCCL (one process per
// GPU over NVLink/NVSwitch), NCCL resolved at run time with dlopen.
#include <algorithm>
#include <dlfcn.h>
#include <nccl.h>

#include <functional>

#include <cstring>
#include <exception>
#include <sstream>
#include <thread>

#include "seqpar/comm.hpp"

namespace seqpar {

#define SP_CUDA(x)                                                                       \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) throw StateError(std::string("CUDA: ") + cudaGetErrorString(e_) + \
                                            " at " #x);                                  \
  } while (0)

const char* primitive_name(Primitive p) {
  static const char* n[] = {"all_to_all", "all_gather", "p2p", "all_reduce", "broadcast"};
  return n[static_cast<int>(p)];
}

int CommGroup::index_of(int rank) const {
  for (size_t i = 0; i < ranks.size(); ++i)
    if (ranks[i] == rank) return static_cast<int>(i);
  throw ConfigError("rank " + std::to_string(rank) + " is not in group " + key());
}
bool CommGroup::contains(int rank) const {
  for (int r : ranks)
    if (r == rank) return true;
  return false;
}
std::string CommGroup::key() const {
  std::ostringstream os;
  for (size_t i = 0; i < ranks.size(); ++i) os << (i ? "," : "") << ranks[i];
  return os.str();
}

// ------------------------------------------------------------------------------ loopback
namespace {

class LoopbackTransport : public Transport {
 public:
  LoopbackTransport(LoopbackFabric* f, int device) : f_(f) {
    SP_CUDA(cudaSetDevice(device));
    SP_CUDA(cudaEventCreateWithFlags(&ev_ready_, cudaEventDisableTiming));
    SP_CUDA(cudaEventCreateWithFlags(&ev_done_, cudaEventDisableTiming));
  }
  ~LoopbackTransport() override {
    cudaEventDestroy(ev_ready_);
    cudaEventDestroy(ev_done_);
  }
  bool peer_access() const override { return !f_->force_messages(); }

  std::vector<void*> exchange_ptrs(const CommGroup& g, int my_rank, void* mine,
                                   cudaStream_t s) override {
    SP_CUDA(cudaEventRecord(ev_ready_, s));
    auto dep = f_->rendezvous(g, my_rank, {mine, ev_ready_, nullptr});
    std::vector<void*> out;
    const int me = g.index_of(my_rank);
    for (int i = 0; i < g.size(); ++i) {
      out.push_back(dep[static_cast<size_t>(i)].ptr);
      if (i != me) SP_CUDA(cudaStreamWaitEvent(s, dep[static_cast<size_t>(i)].ev, 0));
    }
    return out;
  }

  void release(const CommGroup& g, int my_rank, cudaStream_t s) override {
    SP_CUDA(cudaEventRecord(ev_done_, s));
    auto dep = f_->rendezvous(g, my_rank, {nullptr, ev_done_, nullptr});
    const int me = g.index_of(my_rank);
    for (int i = 0; i < g.size(); ++i)
      if (i != me) SP_CUDA(cudaStreamWaitEvent(s, dep[static_cast<size_t>(i)].ev, 0));
  }

  // Emulated messages: every receiver copies the matching send out of the sender's buffer
  // (k-th message from a to b pairs with the k-th receive on b from a, as NCCL orders them).
  void send_recv(const CommGroup& g, int my_rank, const std::vector<Msg>& sends,
                 const std::vector<Msg>& recvs, cudaStream_t s) override {
    SP_CUDA(cudaEventRecord(ev_ready_, s));
    auto mine = std::make_shared<std::vector<Msg>>(sends);
    auto dep = f_->rendezvous(g, my_rank, {nullptr, ev_ready_, mine});
    const int me = g.index_of(my_rank);
    std::vector<int> taken(static_cast<size_t>(g.size()), 0);
    for (const Msg& r : recvs) {
      const auto& src = *dep[static_cast<size_t>(r.peer)].sends;
      int seen = 0;
      const Msg* hit = nullptr;
      for (const Msg& m : src)
        if (m.peer == me && seen++ == taken[static_cast<size_t>(r.peer)]) {
          hit = &m;
          break;
        }
      if (!hit || hit->bytes != r.bytes)
        throw StateError("loopback send_recv: unmatched message from group index " +
                         std::to_string(r.peer));
      ++taken[static_cast<size_t>(r.peer)];
      if (r.peer != me) SP_CUDA(cudaStreamWaitEvent(s, dep[static_cast<size_t>(r.peer)].ev, 0));
      if (r.bytes) SP_CUDA(cudaMemcpyAsync(r.ptr, hit->ptr, r.bytes, cudaMemcpyDeviceToDevice, s));
    }
    release(g, my_rank, s);
  }

 private:
  LoopbackFabric* f_;
  cudaEvent_t ev_ready_ = nullptr, ev_done_ = nullptr;
};

}  // namespace

LoopbackFabric::LoopbackFabric(int world, int sp, int device, bool force_messages)
    : world_(world), sp_(sp), device_(device), force_messages_(force_messages) {
  if (world <= 0 || sp <= 0 || world % sp) throw ConfigError("fabric: world must be a multiple of sp");
  SP_CUDA(cudaSetDevice(device));
  for (int r = 0; r < world; ++r) {
    transports_.push_back(std::make_unique<LoopbackTransport>(this, device));
    auto c = std::make_unique<RankCtx>();
    c->transport = transports_.back().get();
    c->rank = r;
    c->device = device;
    c->sp_group = sp_group_of(r);
    SP_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    SP_CUDA(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    own_streams_.push_back(c->stream);
    own_streams_.push_back(c->comm_stream);
    ctxs_.push_back(std::move(c));
  }
}

LoopbackFabric::~LoopbackFabric() {
  // only the streams this fabric created: a context's compute stream may have been replaced by
  // the caller's (spattn_ctx_set_stream) and is not ours to destroy
  for (auto& c : ctxs_) cudaStreamSynchronize(c->stream);
  for (cudaStream_t s : own_streams_) {
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
}

CommGroup LoopbackFabric::sp_group_of(int rank) const {
  CommGroup g;
  const int base = rank / sp_ * sp_;
  for (int i = 0; i < sp_; ++i) g.ranks.push_back(base + i);
  return g;
}

std::vector<LoopbackFabric::Deposit> LoopbackFabric::rendezvous(const CommGroup& g, int my_rank,
                                                                 Deposit d) {
  std::unique_lock<std::mutex> lk(mu_);
  if (abort_) throw PeerAbort("peer rank failed");
  Slot& s = slots_[g.key()];
  if (s.dep.size() != static_cast<size_t>(g.size())) s.dep.assign(static_cast<size_t>(g.size()), {});
  const uint64_t gen = s.gen;
  s.dep[static_cast<size_t>(g.index_of(my_rank))] = std::move(d);
  if (++s.arrived == g.size()) {
    s.result[gen & 1] = s.dep;
    s.arrived = 0;
    ++s.gen;
    cv_.notify_all();
  } else {
    cv_.wait(lk, [&] { return s.gen != gen || abort_; });
    if (s.gen == gen) throw PeerAbort("peer rank failed");
  }
  return s.result[gen & 1];
}

void LoopbackFabric::run(const std::function<void(RankCtx&)>& body) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    abort_ = false;
    slots_.clear();
  }
  std::vector<std::exception_ptr> err(static_cast<size_t>(world_));
  std::vector<std::thread> th;
  for (int r = 0; r < world_; ++r) {
    th.emplace_back([&, r] {
      try {
        cudaSetDevice(device_);
        body(*ctxs_[static_cast<size_t>(r)]);
        SP_CUDA(cudaStreamSynchronize(ctxs_[static_cast<size_t>(r)]->stream));
      } catch (...) {
        err[static_cast<size_t>(r)] = std::current_exception();
        std::lock_guard<std::mutex> lk(mu_);
        abort_ = true;
        cv_.notify_all();
      }
    });
  }
  for (auto& t : th) t.join();
  // root cause first: a real error beats the PeerAbort it triggered elsewhere
  for (auto& e : err) {
    if (!e) continue;
    try {
      std::rethrow_exception(e);
    } catch (const PeerAbort&) {
      continue;
    } catch (...) {
      throw;
    }
  }
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

namespace {
// one self message on `c` (or through send_recv on the single-member group when c is null)
void self_message(Transport& t, int my_rank, size_t bytes, cudaStream_t s,
                  const std::function<void(void*, void*, size_t)>& send_self) {
  void *a = nullptr, *b = nullptr;
  SP_CUDA(cudaMallocAsync(&a, bytes, s));
  SP_CUDA(cudaMallocAsync(&b, bytes, s));
  SP_CUDA(cudaMemsetAsync(a, 0x5a, bytes, s));
  SP_CUDA(cudaMemsetAsync(b, 0, bytes, s));
  if (send_self) {
    send_self(a, b, bytes);
  } else {
    CommGroup g;
    g.ranks = {my_rank};
    t.send_recv(g, my_rank, {{0, a, bytes}}, {{0, b, bytes}}, s);
  }
  std::vector<unsigned char> h(bytes);
  SP_CUDA(cudaMemcpyAsync(h.data(), b, bytes, cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaFreeAsync(a, s));
  SP_CUDA(cudaFreeAsync(b, s));
  SP_CUDA(cudaStreamSynchronize(s));
  for (unsigned char c : h)
    if (c != 0x5a) throw StateError("transport self-test: received bytes differ from the sent ones");
}
}  // namespace

void Transport::self_test(int my_rank, size_t bytes, cudaStream_t s) {
  self_message(*this, my_rank, bytes, s, nullptr);
}

// ---------------------------------------------------------------------------------- NCCL
namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!a.h) a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.h) throw StateError(std::string("NCCL: cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char* n) {
      void* p = dlsym(a.h, n);
      if (!p) throw StateError(std::string("NCCL: missing symbol ") + n);
      return p;
    };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommSplit = reinterpret_cast<decltype(a.CommSplit)>(sym("ncclCommSplit"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.CommAbort = reinterpret_cast<decltype(a.CommAbort)>(sym("ncclCommAbort"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    return a;
  }();
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw StateError(std::string("NCCL ") + what + ": " + nccl().GetErrorString(r));
}

class NcclTransport : public Transport {
 public:
  NcclTransport(int rank, int world, const void* uid, int device) : rank_(rank), world_(world) {
    SP_CUDA(cudaSetDevice(device));
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    nccl_check(nccl().CommInitRank(&world_comm_, world, id, rank), "CommInitRank");
  }
  ~NcclTransport() override {
    // after a failed NCCL call the communicators may hold operations that never complete:
    // abort them (the reference aborts the group on a peer failure, comm.cpp:206-230)
    auto end = failed_ ? nccl().CommAbort : nccl().CommDestroy;
    for (auto& kv : sub_) end(kv.second);
    if (world_comm_) end(world_comm_);
  }
  bool peer_access() const override { return false; }
  std::vector<void*> exchange_ptrs(const CommGroup&, int, void*, cudaStream_t) override {
    throw StateError("NCCL transport has no peer-pointer path");
  }
  void release(const CommGroup&, int, cudaStream_t) override {}

  // ncclCommSplit (collective: every rank calls it) + a grouped ncclSend/ncclRecv to itself on
  // the split communicator and on the world one, then ncclCommDestroy of the split
  void self_test(int my_rank, size_t bytes, cudaStream_t s) override {
    ncclComm_t c = nullptr;
    nccl_check(nccl().CommSplit(world_comm_, 7, my_rank, &c, nullptr), "CommSplit");
    for (ncclComm_t comm : {c, world_comm_}) {
      self_message(*this, my_rank, bytes, s, [&](void* a, void* b, size_t n) {
        nccl_check(nccl().GroupStart(), "GroupStart");
        nccl_check(nccl().Send(a, n, ncclUint8, my_rank, comm, s), "Send");
        nccl_check(nccl().Recv(b, n, ncclUint8, my_rank, comm, s), "Recv");
        nccl_check(nccl().GroupEnd(), "GroupEnd");
      });
    }
    nccl_check(nccl().CommDestroy(c), "CommDestroy");
  }

  void send_recv(const CommGroup& g, int, const std::vector<Msg>& sends,
                 const std::vector<Msg>& recvs, cudaStream_t s) override {
    try {
      ncclComm_t c = comm_for(g);
      nccl_check(nccl().GroupStart(), "GroupStart");
      for (const Msg& m : sends)
        if (m.bytes) nccl_check(nccl().Send(m.ptr, m.bytes, ncclUint8, m.peer, c, s), "Send");
      for (const Msg& m : recvs)
        if (m.bytes) nccl_check(nccl().Recv(m.ptr, m.bytes, ncclUint8, m.peer, c, s), "Recv");
      nccl_check(nccl().GroupEnd(), "GroupEnd");
    } catch (...) {
      failed_ = true;
      throw;
    }
  }

 private:
  // Sub-groups (USP inner/outer) get a communicator split from the world one; every rank
  // requests its groups in the same program order, so the collective splits line up.
  ncclComm_t comm_for(const CommGroup& g) {
    if (g.size() == world_) {
      bool identity = true;
      for (int i = 0; i < world_; ++i) identity &= g.ranks[static_cast<size_t>(i)] == i;
      if (identity) return world_comm_;
    }
    const std::string k = g.key();
    auto it = sub_.find(k);
    if (it != sub_.end()) return it->second;
    // every split call partitions the ranks into disjoint groups (the USP inner / outer
    // groups), so the group's lowest rank is a collision-free colour
    const int color = *std::min_element(g.ranks.begin(), g.ranks.end());
    ncclComm_t c;
    nccl_check(nccl().CommSplit(world_comm_, color, g.index_of(rank_), &c, nullptr), "CommSplit");
    sub_[k] = c;
    return c;
  }

  int rank_, world_;
  bool failed_ = false;
  ncclComm_t world_comm_ = nullptr;
  std::map<std::string, ncclComm_t> sub_;
};

}  // namespace

std::unique_ptr<Transport> make_nccl_transport(int rank, int world, const void* uid, int device) {
  return std::make_unique<NcclTransport>(rank, world, uid, device);
}

void nccl_unique_id(void* out128) {
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "GetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

std::vector<uint8_t> broadcast_bytes(RankCtx& ctx, const CommGroup& group, const std::vector<uint8_t>& payload,
                                     int root) {
  const int g = group.size();
  const int me = group.index_of(ctx.rank);
  if (!group.contains(root)) throw ConfigError("broadcast root not in group");
  const int ri = group.index_of(root);
  const bool is_root = me == ri;
  cudaStream_t s = ctx.stream;
  if (g == 1) {
    ctx.count(Primitive::broadcast, 0);
    return payload;
  }
  // the root's size first (members do not know it), then the payload; both staged in device
  // memory so the NCCL transport can carry them
  int64_t* dsize = nullptr;
  SP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dsize), sizeof(int64_t), s));
  int64_t n = is_root ? static_cast<int64_t>(payload.size()) : 0;
  if (is_root) SP_CUDA(cudaMemcpyAsync(dsize, &n, sizeof(n), cudaMemcpyHostToDevice, s));
  std::vector<Msg> sends, recvs;
  if (is_root) {
    for (int j = 0; j < g; ++j)
      if (j != ri) sends.push_back({j, dsize, sizeof(int64_t)});
  } else {
    recvs.push_back({ri, dsize, sizeof(int64_t)});
  }
  ctx.transport->send_recv(group, ctx.rank, sends, recvs, s);
  SP_CUDA(cudaMemcpyAsync(&n, dsize, sizeof(n), cudaMemcpyDeviceToHost, s));
  SP_CUDA(cudaStreamSynchronize(s));
  SP_CUDA(cudaFreeAsync(dsize, s));
  std::vector<uint8_t> out(static_cast<size_t>(n));
  if (n > 0) {
    void* buf = nullptr;
    SP_CUDA(cudaMallocAsync(&buf, static_cast<size_t>(n), s));
    if (is_root) SP_CUDA(cudaMemcpyAsync(buf, payload.data(), static_cast<size_t>(n), cudaMemcpyHostToDevice, s));
    sends.clear();
    recvs.clear();
    if (is_root) {
      for (int j = 0; j < g; ++j)
        if (j != ri) sends.push_back({j, buf, static_cast<size_t>(n)});
    } else {
      recvs.push_back({ri, buf, static_cast<size_t>(n)});
    }
    ctx.transport->send_recv(group, ctx.rank, sends, recvs, s);
    SP_CUDA(cudaMemcpyAsync(out.data(), buf, static_cast<size_t>(n), cudaMemcpyDeviceToHost, s));
    SP_CUDA(cudaFreeAsync(buf, s));
    SP_CUDA(cudaStreamSynchronize(s));
  }
  ctx.count(Primitive::broadcast, n * (g - 1) / g);
  return out;
}

std::vector<uint8_t> replicate_packing_mask(RankCtx& ctx, const CommGroup& group,
                                            const std::vector<uint8_t>& mask) {
  return broadcast_bytes(ctx, group, mask, group.ranks.front());
}

}  // namespace seqpar
