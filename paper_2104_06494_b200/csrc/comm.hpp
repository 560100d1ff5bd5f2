// Multi-GPU transport for the sharded PAGANI loop (one process per GPU).
//
// Two implementations behind one interface:
//  * NcclComm -- NCCL over NVLink/NVSwitch (libnccl.so.2 is dlopen'ed, so the
//    library has no link-time NCCL dependency and shares the process's NCCL
//    if torch already loaded one).
//  * HostComm -- caller-provided host callbacks (e.g. torch.distributed/gloo);
//    device buffers are staged through host memory.  Used to run R ranks on a
//    single GPU in tests, and by hosts without NCCL.
// Every collective the driver issues is tiny (block partials, counts) except
// the region exchange after bisection.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pagani.h"

namespace pgn {

struct NcclError : std::runtime_error {
  explicit NcclError(const std::string& s) : std::runtime_error(s) {}
};

void set_last_error(const std::string& msg);  // capi.cu (pagani_last_error)

struct Transfer {
  int peer;
  void* dev;  // device pointer
  size_t bytes;
};

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  virtual int device() const = 0;
  // Equal-size allgather of device buffers: recv holds size() * bytes.
  virtual void allgather(const void* dsend, void* drecv, size_t bytes, cudaStream_t st) = 0;
  // Point-to-point exchange (one group); self transfers are not allowed here.
  virtual void exchange(const std::vector<Transfer>& sends, const std::vector<Transfer>& recvs,
                        cudaStream_t st) = 0;
};

Comm* comm_from_handle(void* handle);

}  // namespace pgn
