// comm.h -- collectives of the rank-sharded construction (one process per
// GPU; every level's probes are split across ranks and the new factor
// blocks are all-gathered) and of the distributed apply.
//
// Two transports behind one interface:
//   * NCCL (bfly_ctx_set_comm): device buffers, stream-ordered, NVLink;
//   * host-staged (bfly_ctx_set_host_comm): the library synchronizes its
//     stream, stages the buffers through pinned host memory and calls the
//     caller's collective functions (e.g. torch.distributed over gloo).  For
//     processes that share one GPU (NCCL rejects two ranks on one device) and
//     for hosts without peer access; no kernel ever waits on another rank.
#pragma once

#include <cstdint>

#include "../../include/bfly_b200.h"
#include "context.h"

namespace bfly {

void comm_unique_id(uint8_t* id_out);
void comm_init(Ctx* c, int rank, int world, const uint8_t* id);
void comm_init_host(Ctx* c, int rank, int world, const bfly_host_comm* hc);
void comm_destroy(Ctx* c);
// true when a transport (NCCL or host-staged) connects world > 1 ranks
bool comm_active(const Ctx* c);
// element counts in bytes; in place when send == recv + rank*bytes
void comm_allgather_bytes(Ctx* c, const void* send, void* recv, size_t bytes_per_rank);
void comm_allreduce_max_i32(Ctx* c, int32_t* buf, size_t count);
void comm_allreduce_sum_f64(Ctx* c, double* buf, size_t count);
void comm_allreduce_sum_f32(Ctx* c, float* buf, size_t count);
// point-to-point (distributed apply exchanges), grouped between start/end
void comm_group_start(Ctx* c);
void comm_group_end(Ctx* c);
void comm_send(Ctx* c, const void* buf, size_t bytes, int peer);
void comm_recv(Ctx* c, void* buf, size_t bytes, int peer);
void comm_barrier(Ctx* c);

}  // namespace bfly
