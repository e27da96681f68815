// comm.cu -- NCCL communicator management and the few collectives the
// sharded construction needs.
//
// libnccl is bound lazily with dlopen on first use, so the library never
// forces a particular libnccl.so.2 into a process: when PyTorch has already
// loaded its bundled NCCL, dlopen returns that same object (same soname).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "comm.h"

namespace bfly {

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static bool loaded = false;
  if (loaded) return api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) fail(NCCL_ERR, std::string("cannot load libnccl.so.2: ") + dlerror());
  auto sym = [&](const char* name) {
    void* p = dlsym(h, name);
    if (!p) fail(NCCL_ERR, std::string("libnccl.so.2 lacks ") + name);
    return p;
  };
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
  api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
  api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
  api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
  api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
  api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
  api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
  api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  loaded = true;
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(NCCL_ERR, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace

void comm_unique_id(uint8_t* id_out) {
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
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
  nccl_check(nccl().CommInitRank(&comm, world, id, rank), "ncclCommInitRank");
  c->comm = comm;
}

void comm_destroy(Ctx* c) {
  if (c && c->comm) {
    nccl().CommDestroy(c->comm);
    c->comm = nullptr;
  }
  if (c) {
    c->rank = 0;
    c->world = 1;
  }
}

void comm_allgather_bytes(Ctx* c, const void* send, void* recv, size_t bytes) {
  if (c->world == 1 || !c->comm) return;
  nccl_check(nccl().AllGather(send, recv, bytes, ncclUint8, c->comm, c->stream), "ncclAllGather");
}

void comm_allreduce_max_i32(Ctx* c, int32_t* buf, size_t count) {
  if (c->world == 1 || !c->comm) return;
  nccl_check(nccl().AllReduce(buf, buf, count, ncclInt32, ncclMax, c->comm, c->stream), "ncclAllReduce");
}

void comm_allreduce_sum_f64(Ctx* c, double* buf, size_t count) {
  if (c->world == 1 || !c->comm) return;
  nccl_check(nccl().AllReduce(buf, buf, count, ncclFloat64, ncclSum, c->comm, c->stream), "ncclAllReduce");
}

void comm_allreduce_sum_f32(Ctx* c, float* buf, size_t count) {
  if (c->world == 1 || !c->comm) return;
  nccl_check(nccl().AllReduce(buf, buf, count, ncclFloat32, ncclSum, c->comm, c->stream), "ncclAllReduce");
}

void comm_group_start() { nccl_check(nccl().GroupStart(), "ncclGroupStart"); }
void comm_group_end() { nccl_check(nccl().GroupEnd(), "ncclGroupEnd"); }

void comm_send(Ctx* c, const void* buf, size_t bytes, int peer) {
  nccl_check(nccl().Send(buf, bytes, ncclUint8, peer, c->comm, c->stream), "ncclSend");
}
void comm_recv(Ctx* c, void* buf, size_t bytes, int peer) {
  nccl_check(nccl().Recv(buf, bytes, ncclUint8, peer, c->comm, c->stream), "ncclRecv");
}

void comm_barrier(Ctx* c) {
  if (c->world == 1 || !c->comm) return;
  DBuf<int32_t> one(c, 1);
  one.zero();
  comm_allreduce_max_i32(c, one.p, 1);
  c->sync();
}

}  // namespace bfly
