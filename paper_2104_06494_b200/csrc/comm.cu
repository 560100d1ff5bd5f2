// Multi-GPU communicator (one process per GPU).  Placeholder until the
// sharded driver lands: every entry point reports PAGANI_E_UNSUPPORTED.
#include "driver.hpp"

extern "C" {

int pagani_comm_unique_id(uint8_t*) { return PAGANI_E_UNSUPPORTED; }
int pagani_comm_init_rank(const uint8_t*, int, int, int, void**) { return PAGANI_E_UNSUPPORTED; }
int pagani_comm_destroy(void*) { return PAGANI_E_UNSUPPORTED; }

}  // extern "C"
