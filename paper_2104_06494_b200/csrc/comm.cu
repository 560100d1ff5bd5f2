// Transports for the sharded driver (see comm.hpp).
#include "comm.hpp"

#include <dlfcn.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>

#include "driver.hpp"

namespace pgn {

namespace {

constexpr uint32_t kCommMagic = 0x50474e43u;  // 'PGNC'

// ---- NCCL through dlopen ------------------------------------------------------
// Minimal ABI subset (nccl.h): opaque communicator, 128-byte unique id, the
// uint8 datatype, and the entry points used here.
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[PAGANI_COMM_ID_BYTES];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclUint8 = 1;  // ncclUint8

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(api.h, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(api.h, "ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(api.h, "ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(api.h, "ncclAllGather"));
    api.Send = reinterpret_cast<decltype(api.Send)>(dlsym(api.h, "ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(dlsym(api.h, "ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(api.h, "ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(api.h, "ncclGroupEnd"));
    api.GetErrorString =
        reinterpret_cast<decltype(api.GetErrorString)>(dlsym(api.h, "ncclGetErrorString"));
  });
  if (!api.h) throw NcclError("NCCL (libnccl.so.2) is not available");
  if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.AllGather || !api.Send ||
      !api.Recv || !api.GroupStart || !api.GroupEnd)
    throw NcclError("libnccl.so.2 lacks an entry point this library uses (need NCCL >= 2.7)");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != 0) {
    const char* s = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
    throw NcclError(std::string("NCCL error ") + std::to_string(r) + " (" + s + ") at " + what);
  }
}

class NcclComm final : public Comm {
 public:
  NcclComm(const uint8_t* id, int nranks, int rank, int device)
      : rank_(rank), size_(nranks), device_(device) {
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, PAGANI_COMM_ID_BYTES);
    PGN_CK(cudaSetDevice(device));
    nccl_check(nccl().CommInitRank(&comm_, nranks, uid, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) nccl().CommDestroy(comm_);
  }
  int rank() const override { return rank_; }
  int size() const override { return size_; }
  int device() const override { return device_; }
  void allgather(const void* s, void* r, size_t bytes, cudaStream_t st) override {
    nccl_check(nccl().AllGather(s, r, bytes, kNcclUint8, comm_, st), "ncclAllGather");
  }
  void exchange(const std::vector<Transfer>& sends, const std::vector<Transfer>& recvs,
                cudaStream_t st) override {
    if (sends.empty() && recvs.empty()) return;
    nccl_check(nccl().GroupStart(), "ncclGroupStart");
    for (const Transfer& t : sends)
      if (t.bytes) nccl_check(nccl().Send(t.dev, t.bytes, kNcclUint8, t.peer, comm_, st), "ncclSend");
    for (const Transfer& t : recvs)
      if (t.bytes) nccl_check(nccl().Recv(t.dev, t.bytes, kNcclUint8, t.peer, comm_, st), "ncclRecv");
    nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  }

 private:
  ncclComm_t comm_ = nullptr;
  int rank_, size_, device_;
};

// ---- host-callback transport ---------------------------------------------------
class HostComm final : public Comm {
 public:
  HostComm(const pagani_host_transport& t, int device) : t_(t), device_(device) {}
  int rank() const override { return t_.rank; }
  int size() const override { return t_.size; }
  int device() const override { return device_; }
  void allgather(const void* s, void* r, size_t bytes, cudaStream_t st) override {
    hs_.resize(bytes);
    hr_.resize(bytes * t_.size);
    if (bytes) PGN_CK(cudaMemcpyAsync(hs_.data(), s, bytes, cudaMemcpyDeviceToHost, st));
    PGN_CK(cudaStreamSynchronize(st));
    if (t_.allgather(hs_.data(), hr_.data(), bytes, t_.user) != 0)
      throw NcclError("host transport allgather failed");
    if (bytes) PGN_CK(cudaMemcpyAsync(r, hr_.data(), bytes * t_.size, cudaMemcpyHostToDevice, st));
    PGN_CK(cudaStreamSynchronize(st));
  }
  void exchange(const std::vector<Transfer>& sends, const std::vector<Transfer>& recvs,
                cudaStream_t st) override {
    std::vector<std::vector<uint8_t>> sb(sends.size()), rb(recvs.size());
    std::vector<int> sp, rp;
    std::vector<const void*> sptr;
    std::vector<void*> rptr;
    std::vector<size_t> sn, rn;
    for (size_t i = 0; i < sends.size(); ++i) {
      sb[i].resize(sends[i].bytes);
      if (sends[i].bytes)
        PGN_CK(cudaMemcpyAsync(sb[i].data(), sends[i].dev, sends[i].bytes, cudaMemcpyDeviceToHost, st));
      sp.push_back(sends[i].peer);
      sptr.push_back(sb[i].data());
      sn.push_back(sends[i].bytes);
    }
    for (size_t i = 0; i < recvs.size(); ++i) {
      rb[i].resize(recvs[i].bytes);
      rp.push_back(recvs[i].peer);
      rptr.push_back(rb[i].data());
      rn.push_back(recvs[i].bytes);
    }
    PGN_CK(cudaStreamSynchronize(st));
    if (t_.exchange(static_cast<int>(sends.size()), sp.data(), sptr.data(), sn.data(),
                    static_cast<int>(recvs.size()), rp.data(), rptr.data(), rn.data(), t_.user) != 0)
      throw NcclError("host transport exchange failed");
    for (size_t i = 0; i < recvs.size(); ++i)
      if (recvs[i].bytes)
        PGN_CK(cudaMemcpyAsync(recvs[i].dev, rb[i].data(), recvs[i].bytes, cudaMemcpyHostToDevice, st));
    PGN_CK(cudaStreamSynchronize(st));
  }

 private:
  pagani_host_transport t_;
  int device_;
  std::vector<uint8_t> hs_, hr_;
};

struct Handle {
  uint32_t magic = kCommMagic;
  Comm* comm = nullptr;
};

template <class Fn>
int comm_guard(Fn&& fn) {
  try {
    fn();
    return PAGANI_OK;
  } catch (const NcclError& e) {
    set_last_error(e.what());
    return PAGANI_E_NCCL;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return PAGANI_E_INVALID;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return PAGANI_E_CUDA;
  }
}

}  // namespace

Comm* comm_from_handle(void* handle) {
  if (!handle) return nullptr;
  auto* h = static_cast<Handle*>(handle);
  if (h->magic != kCommMagic || !h->comm) throw std::invalid_argument("invalid communicator handle");
  return h->comm;
}

}  // namespace pgn

extern "C" {

int pagani_comm_unique_id(uint8_t* unique_id) {
  return pgn::comm_guard([&] {
    pgn::ncclUniqueId id;
    pgn::nccl_check(pgn::nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(unique_id, id.internal, PAGANI_COMM_ID_BYTES);
  });
}

int pagani_comm_init_rank(const uint8_t* unique_id, int nranks, int rank, int device,
                          void** comm) {
  return pgn::comm_guard([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank/size");
    // the communicator first: if ncclCommInitRank throws, nothing leaks
    std::unique_ptr<pgn::Comm> c(new pgn::NcclComm(unique_id, nranks, rank, device));
    auto* h = new pgn::Handle();
    h->comm = c.release();
    *comm = h;
  });
}

int pagani_comm_init_host(const pagani_host_transport* t, int device, void** comm) {
  return pgn::comm_guard([&] {
    if (!t || !t->allgather || !t->exchange || t->size < 1 || t->rank < 0 || t->rank >= t->size)
      throw std::invalid_argument("bad host transport");
    std::unique_ptr<pgn::Comm> c(new pgn::HostComm(*t, device));
    auto* h = new pgn::Handle();
    h->comm = c.release();
    *comm = h;
  });
}

int pagani_shard_bounds(int64_t m, int nranks, int64_t* bounds) {
  return pgn::comm_guard([&] {
    if (nranks < 1 || m < 0) throw std::invalid_argument("bad shard arguments");
    const std::vector<int64_t> b = pgn::shard_bounds(m, nranks);
    for (int r = 0; r <= nranks; ++r) bounds[r] = b[r];
  });
}

int pagani_shard_plan(int nranks, int rank, const int64_t* kept, int max_pieces, int32_t* n_send,
                      int64_t* sends, int32_t* n_recv, int64_t* recvs) {
  return pgn::comm_guard([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank/size");
    const std::vector<int64_t> k(kept, kept + nranks + 1);
    const std::vector<int64_t> next = pgn::shard_bounds(2 * k[nranks], nranks);
    std::vector<pgn::Piece> s, r;
    pgn::exchange_plan(nranks, rank, k, next, s, r);
    if (static_cast<int>(s.size()) > max_pieces || static_cast<int>(r.size()) > max_pieces)
      throw std::invalid_argument("shard plan: too many pieces");
    *n_send = static_cast<int32_t>(s.size());
    *n_recv = static_cast<int32_t>(r.size());
    for (size_t i = 0; i < s.size(); ++i) {
      sends[4 * i] = s[i].peer, sends[4 * i + 1] = s[i].src_off;
      sends[4 * i + 2] = s[i].dst_off, sends[4 * i + 3] = s[i].count;
    }
    for (size_t i = 0; i < r.size(); ++i) {
      recvs[4 * i] = r[i].peer, recvs[4 * i + 1] = r[i].src_off;
      recvs[4 * i + 2] = r[i].dst_off, recvs[4 * i + 3] = r[i].count;
    }
  });
}

int pagani_comm_destroy(void* comm) {
  return pgn::comm_guard([&] {
    if (!comm) return;
    auto* h = static_cast<pgn::Handle*>(comm);
    if (h->magic != pgn::kCommMagic) throw std::invalid_argument("invalid communicator handle");
    delete h->comm;
    h->magic = 0;
    delete h;
  });
}

}  // extern "C"
