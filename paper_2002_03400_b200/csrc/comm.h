// comm.h -- NCCL plumbing for the rank-sharded construction (one process per
// GPU; every level's probes are split across ranks and the new factor
// blocks are all-gathered over NVLink).
#pragma once

#include <cstdint>

#include "context.h"

namespace bfly {

void comm_unique_id(uint8_t* id_out);
void comm_init(Ctx* c, int rank, int world, const uint8_t* id);
void comm_destroy(Ctx* c);
// element counts in bytes; in place when send == recv + rank*bytes
void comm_allgather_bytes(Ctx* c, const void* send, void* recv, size_t bytes_per_rank);
void comm_allreduce_max_i32(Ctx* c, int32_t* buf, size_t count);
void comm_allreduce_sum_f64(Ctx* c, double* buf, size_t count);
void comm_allreduce_sum_f32(Ctx* c, float* buf, size_t count);
// point-to-point (distributed apply exchanges), grouped between start/end
void comm_group_start();
void comm_group_end();
void comm_send(Ctx* c, const void* buf, size_t bytes, int peer);
void comm_recv(Ctx* c, void* buf, size_t bytes, int peer);
void comm_barrier(Ctx* c);

}  // namespace bfly
