// comm.cu -- communicators (NCCL, or host-staged through the caller's
// collectives) and the few collectives the sharded construction and the
// distributed apply need.
//
// libnccl is bound lazily with dlopen on first use, so the library never
// forces a particular libnccl.so.2 into a process: when PyTorch has already
// loaded its bundled NCCL, dlopen returns that same object (same soname).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
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

namespace {
void log_join(const Ctx* c, const char* transport) {
  if (std::getenv("BFLY_QUIET")) return;
  std::fprintf(stderr, "bfly: rank %d of %d joined the %s communicator (device %d)\n", c->rank, c->world, transport,
               c->device);
}
}  // namespace

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
  log_join(c, "NCCL");
}

void comm_init_host(Ctx* c, int rank, int world, const bfly_host_comm* hc) {
  if (world < 1 || rank < 0 || rank >= world) fail(PRECONDITION, "comm: bad rank/world");
  if (world > 1 && (!hc || !hc->allgather || !hc->allreduce || !hc->sendrecv))
    fail(PRECONDITION, "host comm: allgather, allreduce and sendrecv are required");
  comm_destroy(c);
  c->rank = rank;
  c->world = world;
  if (world == 1) return;
  c->host = std::make_unique<HostComm>();
  c->host->fns = *hc;
  log_join(c, "host-staged");
}

void comm_destroy(Ctx* c) {
  if (c && c->comm) {
    nccl().CommDestroy(c->comm);
    c->comm = nullptr;
  }
  if (c) {
    c->host.reset();
    c->rank = 0;
    c->world = 1;
  }
}

bool comm_active(const Ctx* c) { return c->world > 1 && (c->comm || c->host); }

namespace {
// host staging: the library stream is drained, so the device buffers are final
void host_rc(int rc, const char* what) {
  if (rc != 0) fail(NCCL_ERR, std::string("host comm ") + what + " failed (" + std::to_string(rc) + ")");
}
}  // namespace

void comm_allgather_bytes(Ctx* c, const void* send, void* recv, size_t bytes) {
  if (!comm_active(c)) return;
  if (c->comm) {
    nccl_check(nccl().AllGather(send, recv, bytes, ncclUint8, c->comm, c->stream), "ncclAllGather");
    return;
  }
  HostComm& h = *c->host;
  unsigned char* hs = h.stage(c, 0, bytes);
  unsigned char* hr = h.stage(c, 1, bytes * (size_t)c->world);
  if (bytes) BFLY_CUDA(cudaMemcpyAsync(hs, send, bytes, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  host_rc(h.fns.allgather(h.fns.user, hs, hr, (int64_t)bytes), "allgather");
  if (bytes) BFLY_CUDA(cudaMemcpyAsync(recv, hr, bytes * (size_t)c->world, cudaMemcpyHostToDevice, c->stream));
  c->sync();
}

namespace {
void host_allreduce(Ctx* c, void* buf, size_t count, size_t elem, int dtype, int op) {
  HostComm& h = *c->host;
  const size_t bytes = count * elem;
  unsigned char* hb = h.stage(c, 0, bytes);
  if (bytes) BFLY_CUDA(cudaMemcpyAsync(hb, buf, bytes, cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  host_rc(h.fns.allreduce(h.fns.user, hb, (int64_t)count, dtype, op), "allreduce");
  if (bytes) BFLY_CUDA(cudaMemcpyAsync(buf, hb, bytes, cudaMemcpyHostToDevice, c->stream));
  c->sync();
}
}  // namespace

void comm_allreduce_max_i32(Ctx* c, int32_t* buf, size_t count) {
  if (!comm_active(c)) return;
  if (c->host) return host_allreduce(c, buf, count, sizeof(int32_t), 0, 1);
  nccl_check(nccl().AllReduce(buf, buf, count, ncclInt32, ncclMax, c->comm, c->stream), "ncclAllReduce");
}

void comm_allreduce_sum_f64(Ctx* c, double* buf, size_t count) {
  if (!comm_active(c)) return;
  if (c->host) return host_allreduce(c, buf, count, sizeof(double), 1, 0);
  nccl_check(nccl().AllReduce(buf, buf, count, ncclFloat64, ncclSum, c->comm, c->stream), "ncclAllReduce");
}

void comm_allreduce_sum_f32(Ctx* c, float* buf, size_t count) {
  if (!comm_active(c)) return;
  if (c->host) return host_allreduce(c, buf, count, sizeof(float), 2, 0);
  nccl_check(nccl().AllReduce(buf, buf, count, ncclFloat32, ncclSum, c->comm, c->stream), "ncclAllReduce");
}

void comm_group_start(Ctx* c) {
  if (c->host) {
    c->host->pending.clear();
    c->host->grouped = true;
    return;
  }
  nccl_check(nccl().GroupStart(), "ncclGroupStart");
}

void comm_group_end(Ctx* c) {
  if (!c->host) {
    nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
    return;
  }
  HostComm& h = *c->host;
  h.grouped = false;
  // stage every send, run the group on the host, copy every receive back
  size_t sb = 0, rb = 0;
  for (const auto& t : h.pending) (t.send ? sb : rb) += (t.bytes + 255) / 256 * 256;
  unsigned char* hs = h.stage(c, 0, sb);
  unsigned char* hr = h.stage(c, 1, rb);
  std::vector<int32_t> sp, rp;
  std::vector<void*> sbuf, rbuf;
  std::vector<int64_t> sn, rn;
  size_t so = 0, ro = 0;
  for (const auto& t : h.pending) {
    const size_t pad = (t.bytes + 255) / 256 * 256;
    if (t.send) {
      if (t.bytes) BFLY_CUDA(cudaMemcpyAsync(hs + so, t.dev, t.bytes, cudaMemcpyDeviceToHost, c->stream));
      sp.push_back(t.peer);
      sbuf.push_back(hs + so);
      sn.push_back((int64_t)t.bytes);
      so += pad;
    } else {
      rp.push_back(t.peer);
      rbuf.push_back(hr + ro);
      rn.push_back((int64_t)t.bytes);
      ro += pad;
    }
  }
  c->sync();
  host_rc(h.fns.sendrecv(h.fns.user, (int)sp.size(), sp.data(), sbuf.data(), sn.data(), (int)rp.size(), rp.data(),
                         rbuf.data(), rn.data()),
          "sendrecv");
  ro = 0;
  for (const auto& t : h.pending)
    if (!t.send) {
      if (t.bytes) BFLY_CUDA(cudaMemcpyAsync(t.dev, hr + ro, t.bytes, cudaMemcpyHostToDevice, c->stream));
      ro += (t.bytes + 255) / 256 * 256;
    }
  c->sync();
  h.pending.clear();
}

void comm_send(Ctx* c, const void* buf, size_t bytes, int peer) {
  if (c->host) {
    c->host->pending.push_back(HostComm::Xfer{true, peer, const_cast<void*>(buf), bytes});
    return;
  }
  nccl_check(nccl().Send(buf, bytes, ncclUint8, peer, c->comm, c->stream), "ncclSend");
}
void comm_recv(Ctx* c, void* buf, size_t bytes, int peer) {
  if (c->host) {
    c->host->pending.push_back(HostComm::Xfer{false, peer, buf, bytes});
    return;
  }
  nccl_check(nccl().Recv(buf, bytes, ncclUint8, peer, c->comm, c->stream), "ncclRecv");
}

void comm_barrier(Ctx* c) {
  if (!comm_active(c)) return;
  DBuf<int32_t> one(c, 1);
  one.zero();
  comm_allreduce_max_i32(c, one.p, 1);
  c->sync();
}

// pinned staging slot `i` of at least `bytes` (grown geometrically, kept)
unsigned char* HostComm::stage(Ctx*, int i, size_t bytes) {
  if (bytes > cap[i]) {
    if (buf[i]) cudaFreeHost(buf[i]);
    buf[i] = nullptr;
    const size_t want = std::max<size_t>(bytes, cap[i] * 2);
    BFLY_CUDA(cudaMallocHost(reinterpret_cast<void**>(&buf[i]), want));
    cap[i] = want;
  }
  return buf[i];
}

HostComm::~HostComm() {
  for (auto* b : buf)
    if (b) cudaFreeHost(b);
}

}  // namespace bfly
