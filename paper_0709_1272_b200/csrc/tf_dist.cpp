// tf_dist.cpp — multi-GPU entry points (placeholder until the NCCL path lands).
#include <cstdint>
#include "../../include/tilefact.h"

extern "C" {
int tile_chol_dist(int64_t, int64_t, int64_t, int, int, double*, int32_t*, void*, tf_stream_t) {
  return TF_ERR_UNSUPPORTED;
}
int64_t tile_dist_local_tiles(int64_t, int64_t, int, int, int, int) { return -1; }
int tile_nccl_id_bytes(void) { return 128; }
int tile_nccl_get_unique_id(void*) { return TF_ERR_UNSUPPORTED; }
int tile_nccl_comm_init(void*, int, int, void**) { return TF_ERR_UNSUPPORTED; }
int tile_nccl_comm_destroy(void*) { return TF_ERR_UNSUPPORTED; }
}
