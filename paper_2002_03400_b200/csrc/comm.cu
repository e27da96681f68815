// comm.cu -- NCCL communicator management and the few collectives the
// sharded construction needs.
#include <nccl.h>

#include <cstring>

#include "comm.h"

namespace bfly {

#define BFLY_NCCL(call)                                                                                 \
  do {                                                                                                  \
    ncclResult_t r_ = (call);                                                                           \
    if (r_ != ncclSuccess) fail(NCCL_ERR, std::string(#call) + ": " + ncclGetErrorString(r_));          \
  } while (0)

void comm_unique_id(uint8_t* id_out) {
  ncclUniqueId id;
  BFLY_NCCL(ncclGetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof id);
}

void comm_init(Ctx* c, int rank, int world, const uint8_t* id_bytes) {
  if (world < 1 || rank < 0 || rank >= world) fail(PRECONDITION, "comm: bad rank/world");
  comm_destroy(c);
  c->rank = rank;
  c->world = world;
  if (world == 1) return;
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, sizeof id);
  ncclComm_t comm;
  BFLY_NCCL(ncclCommInitRank(&comm, world, id, rank));
  c->comm = comm;
}

void comm_destroy(Ctx* c) {
  if (c && c->comm) {
    ncclCommDestroy(c->comm);
    c->comm = nullptr;
  }
  if (c) {
    c->rank = 0;
    c->world = 1;
  }
}

void comm_allgather_bytes(Ctx* c, const void* send, void* recv, size_t bytes) {
  if (c->world == 1 || !c->comm) return;
  BFLY_NCCL(ncclAllGather(send, recv, bytes, ncclUint8, c->comm, c->stream));
}

void comm_allreduce_max_i32(Ctx* c, int32_t* buf, size_t count) {
  if (c->world == 1 || !c->comm) return;
  BFLY_NCCL(ncclAllReduce(buf, buf, count, ncclInt32, ncclMax, c->comm, c->stream));
}

void comm_allreduce_sum_f64(Ctx* c, double* buf, size_t count) {
  if (c->world == 1 || !c->comm) return;
  BFLY_NCCL(ncclAllReduce(buf, buf, count, ncclFloat64, ncclSum, c->comm, c->stream));
}

void comm_barrier(Ctx* c) {
  if (c->world == 1 || !c->comm) return;
  DBuf<int32_t> one(c, 1);
  one.zero();
  comm_allreduce_max_i32(c, one.p, 1);
  c->sync();
}

}  // namespace bfly
