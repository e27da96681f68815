// dist.cu -- butterfly apply distributed over a process layout (reference
// inc/layout.hpp:139-261 assign_ownership / simulated_parallel_apply; the
// reference only tallies messages, this runs the exchanges).
//
// Every process holds the full factor set (replication) and the
// full input.  Each stage entry (one output coefficient block) runs on the
// owner of the factor block it applies -- V leaf nu, W (l, tau, nu), centre
// core (tau, nu) on the V side; R and U leaf on the U side, keyed by the
// output block -- so the coefficient blocks a process needs from another
// process are exactly the inputs of its entries whose producer entry is owned
// elsewhere.  Those transfers are packed per (source, destination) into
// contiguous buffers: with a communicator they are grouped ncclSend/ncclRecv
// between stages, without one the p processes run in turn on this GPU and the
// packed buffer is unpacked into the destination's coefficient buffer, so the
// single-GPU test exercises the same plan, pack and unpack kernels.  The
// output blocks are disjoint across processes; multi-process runs assemble y
// with one sum all-reduce.
#include <algorithm>
#include <map>
#include <set>
#include <type_traits>

#include "butterfly.h"
#include "comm.h"
#include "layout.h"

namespace bfly {

namespace {

// rows [off_b, off_b + rows) x k columns of buf (ld) <-> out[b*rows + r + col*(nblk*rows)]
template <typename R>
__global__ void pack_blocks_kernel(const cx<R>* __restrict__ buf, int64_t ld, const int64_t* __restrict__ offs,
                                   int nblk, int rows, int k, cx<R>* __restrict__ out) {
  const int64_t per = (int64_t)nblk * rows, total = per * k;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = i / per, j = i - col * per, b = j / rows, r = j - b * rows;
    out[i] = buf[offs[b] + r + col * ld];
  }
}
template <typename R>
__global__ void unpack_blocks_kernel(cx<R>* __restrict__ buf, int64_t ld, const int64_t* __restrict__ offs,
                                     int nblk, int rows, int k, const cx<R>* __restrict__ in) {
  const int64_t per = (int64_t)nblk * rows, total = per * k;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = i / per, j = i - col * per, b = j / rows, r = j - b * rows;
    buf[offs[b] + r + col * ld] = in[i];
  }
}

unsigned grid_for(int64_t n) { return (unsigned)std::min<int64_t>(std::max<int64_t>(ceil_div(n, (int64_t)256), 1), 148 * 8); }

}  // namespace

template <typename R>
typename DevButterfly<R>::DistPlan& DevButterfly<R>::dist_plan(int trans, int kind, int p) {
  for (auto& d : dist_plans_)
    if (d->trans == trans && d->kind == kind && d->p == p) return *d;
  if (trans == OP_N && !have_n_) {
    build_plan_n();
    have_n_ = true;
  }
  if (trans != OP_N && !have_h_) {
    build_plan_h();
    have_h_ = true;
  }
  Plan& pl = trans == OP_N ? plan_n_ : plan_h_;
  auto dp = std::make_unique<DistPlan>();
  dp->trans = trans;
  dp->kind = kind;
  dp->p = p;
  const int g = layout_log_p(p);
  const int n = (int)pl.st.size();
  std::vector<std::vector<int>> owner(n);
  dp->h.assign(n, std::vector<std::vector<GemmEnt>>(p));
  for (int s = 0; s < n; ++s) {
    const StageDesc& d = pl.st[s];
    owner[s].resize(d.h.size());
    for (size_t e = 0; e < d.h.size(); ++e) {
      const int o = layout_owner(kind, L, g, d.own_side, d.own_level, d.own_tau[e], d.own_nu[e]);
      owner[s][e] = o;
      dp->h[s][o].push_back(d.h[e]);
    }
  }
  dp->d.resize(n);
  for (int s = 0; s < n; ++s)
    for (int r = 0; r < p; ++r) dp->d[s].push_back(to_device(ctx, dp->h[s][r]));
  // transfers feeding stage s: producer (stage s-1) blocks read by entries
  // owned by another process
  std::vector<double> recv(p, 0.0);
  dp->xfers.resize(n);
  for (int s = 1; s < n; ++s) {
    const StageDesc& P = pl.st[s - 1];
    const StageDesc& Q = pl.st[s];
    std::map<int64_t, int> start;  // producer output row -> producer entry
    for (size_t e = 0; e < P.h.size(); ++e) start[P.h[e].c] = (int)e;
    std::map<std::pair<int, int>, std::set<int64_t>> need;  // (src, dst) -> producer offsets
    for (size_t e = 0; e < Q.h.size(); ++e) {
      const int dst = owner[s][e];
      for (int si = 0; si < Q.S; ++si) {
        const int64_t b0 = si == 0 ? Q.h[e].b0 : Q.h[e].b1;
        const int64_t b1 = b0 + std::min(Q.K, Q.h[e].krows);
        auto it = start.upper_bound(b0);
        if (it == start.begin()) fail(PRECONDITION, "apply_layout: input rows without producer");
        --it;
        for (; it != start.end() && it->first < b1; ++it) {
          const int src = owner[s - 1][it->second];
          if (src != dst) need[{src, dst}].insert(it->first);
        }
      }
    }
    for (auto& kv : need) {
      DistXfer x;
      x.src = kv.first.first;
      x.dst = kv.first.second;
      x.offs.assign(kv.second.begin(), kv.second.end());
      x.d_offs = to_device(ctx, x.offs);
      recv[x.dst] += (double)x.offs.size() * P.M;
      dp->xfers[s].push_back(std::move(x));
    }
  }
  dp->report[4] = *std::max_element(recv.begin(), recv.end());
  for (double v : recv) dp->report[5] += v;
  // the reference's tallies from the ownership maps (layout.hpp:190-261)
  {
    auto vown = [&](int l, int64_t tau, int64_t nu) { return layout_owner(kind, L, g, 0, l, tau, nu); };
    auto uown = [&](int l, int64_t tau, int64_t nu) { return layout_owner(kind, L, g, 1, l, tau, nu); };
    auto state = [&](bool u, int l) {
      double sum = 0;
      for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
        for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu) sum += u ? u_rank(l, tau, nu) : v_rank(l, tau, nu);
      return sum;
    };
    CommReport rep;
    for (int l = 1; l <= lm; ++l) {
      bool moved = false;
      for (int64_t tau = 0; tau < (int64_t(1) << l) && !moved; ++tau)
        for (int64_t nu = 0; nu < (int64_t(1) << (L - l)) && !moved; ++nu) {
          const int c = vown(l, tau, nu);
          moved = vown(l - 1, tau / 2, 2 * nu) != c || vown(l - 1, tau / 2, 2 * nu + 1) != c;
        }
      if (moved) {
        rep.exchange_msgs += 1;
        rep.exchange_volume += state(false, l - 1) / p;
      }
    }
    for (int l = lm; l < L; ++l) {
      bool moved = false;
      for (int64_t tau = 0; tau < (int64_t(1) << (l + 1)) && !moved; ++tau)
        for (int64_t nu = 0; nu < (int64_t(1) << (L - l - 1)) && !moved; ++nu) {
          const int c = uown(l + 1, tau, nu);
          moved = uown(l, tau / 2, 2 * nu) != c || uown(l, tau / 2, 2 * nu + 1) != c;
        }
      if (moved) {
        rep.exchange_msgs += 1;
        rep.exchange_volume += state(true, l) / p;
      }
    }
    rep.alltoall_volume = kind == LAYOUT_COLUMN ? (double)this->n() / p
                          : kind == LAYOUT_ROW  ? (double)this->m() / p
                                                : state(true, lm) / p;
    rep.alltoall_msgs = std::min<int64_t>(nb() / p, p - 1);
    dp->report[0] = rep.exchange_volume;
    dp->report[1] = (double)rep.exchange_msgs;
    dp->report[2] = rep.alltoall_volume;
    dp->report[3] = (double)rep.alltoall_msgs;
  }
  dist_plans_.push_back(std::move(dp));
  return *dist_plans_.back();
}

template <typename R>
void DevButterfly<R>::apply_layout(int trans, int kind, int p, const cx<R>* x, int64_t ldx, cx<R>* y, int64_t ldy,
                                   int64_t k, double* report) {
  Ctx* c = ctx;
  if (trans != OP_N && trans != OP_H) fail(PRECONDITION, "apply_layout: trans must be N or H");
  if (!layout_valid(kind, L, 1, p)) fail(PRECONDITION, "apply_layout: invalid layout (kind, power-of-two p <= 2^L)");
  if (!rt.identity || !ct.identity) fail(PRECONDITION, "apply_layout: tree-ordered points required");
  const bool real = c->world > 1;
  if (real && p != c->world) fail(PRECONDITION, "apply_layout: p must equal the communicator size");
  if (k <= 0) return;
  DistPlan& dp = dist_plan(trans, kind, p);
  if (report)
    for (int i = 0; i < 6; ++i) report[i] = dp.report[i];
  Plan& pl = trans == OP_N ? plan_n_ : plan_h_;
  const int n = (int)pl.st.size();
  const int64_t NB = nb(), nout = trans == OP_N ? m() : this->n();
  const int nvr = real ? 1 : p;  // processes run by this call
  const size_t nbuf = (size_t)(NB * max_p() * k);
  std::vector<DBuf<cx<R>>> bufs(2 * nvr);
  for (auto& b : bufs) b.reset(c, nbuf);
  size_t stage_max = 0;
  for (int s = 1; s < n; ++s)
    for (const auto& xf : dp.xfers[s]) stage_max = std::max(stage_max, xf.offs.size() * (size_t)pl.st[s - 1].M);
  DBuf<cx<R>> sendb(c, stage_max * k), recvb;
  if (real) {
    // one packed buffer per peer and direction per stage
    size_t tot = 0;
    for (int s = 1; s < n; ++s) {
      size_t st = 0;
      for (const auto& xf : dp.xfers[s]) st += xf.offs.size() * (size_t)pl.st[s - 1].M;
      tot = std::max(tot, st);
    }
    sendb.reset(c, tot * k);
    recvb.reset(c, tot * k);
    if (ldy != nout) fail(PRECONDITION, "apply_layout: multi-process output needs ldy == rows");
    BFLY_CUDA(cudaMemsetAsync(y, 0, sizeof(cx<R>) * (size_t)(nout * k), c->stream));
  }
  const int me = c->rank;
  for (int s = 0; s < n; ++s) {
    const StageDesc& d = pl.st[s];
    if (s > 0) {
      const int rows = pl.st[s - 1].M;
      const int64_t ld = pl.st[s - 1].ld_out;
      if (!real) {
        for (const auto& xf : dp.xfers[s]) {
          const int nblk = (int)xf.offs.size();
          const int64_t cnt = (int64_t)nblk * rows * k;
          const cx<R>* src = bufs[2 * xf.src + (s - 1) % 2].p;
          cx<R>* dst = bufs[2 * xf.dst + (s - 1) % 2].p;
          pack_blocks_kernel<R><<<grid_for(cnt), 256, 0, c->stream>>>(src, ld, xf.d_offs.p, nblk, rows, (int)k,
                                                                      sendb.p);
          BFLY_LAUNCH_CHECK("pack_blocks");
          unpack_blocks_kernel<R><<<grid_for(cnt), 256, 0, c->stream>>>(dst, ld, xf.d_offs.p, nblk, rows, (int)k,
                                                                        sendb.p);
          BFLY_LAUNCH_CHECK("unpack_blocks");
        }
      } else {
        size_t so = 0, ro = 0;
        std::vector<std::pair<const DistXfer*, size_t>> ins;
        for (const auto& xf : dp.xfers[s]) {
          const int nblk = (int)xf.offs.size();
          const int64_t cnt = (int64_t)nblk * rows * k;
          if (xf.src == me) {
            pack_blocks_kernel<R><<<grid_for(cnt), 256, 0, c->stream>>>(bufs[(s - 1) % 2].p, ld, xf.d_offs.p, nblk,
                                                                        rows, (int)k, sendb.p + so);
            BFLY_LAUNCH_CHECK("pack_blocks");
            so += (size_t)cnt;
          }
        }
        comm_group_start(c);
        so = 0;
        for (const auto& xf : dp.xfers[s]) {
          const size_t cnt = xf.offs.size() * (size_t)rows * k;
          if (xf.src == me) {
            comm_send(c, sendb.p + so, cnt * sizeof(cx<R>), xf.dst);
            so += cnt;
          }
          if (xf.dst == me) {
            comm_recv(c, recvb.p + ro, cnt * sizeof(cx<R>), xf.src);
            ins.push_back({&xf, ro});
            ro += cnt;
          }
        }
        comm_group_end(c);
        for (const auto& in : ins) {
          const int nblk = (int)in.first->offs.size();
          const int64_t cnt = (int64_t)nblk * rows * k;
          unpack_blocks_kernel<R><<<grid_for(cnt), 256, 0, c->stream>>>(bufs[(s - 1) % 2].p, ld, in.first->d_offs.p,
                                                                        nblk, rows, (int)k, recvb.p + in.second);
          BFLY_LAUNCH_CHECK("unpack_blocks");
        }
      }
    }
    const bool final = s == n - 1;
    for (int v = 0; v < nvr; ++v) {
      const int r = real ? me : v;
      const int ne = (int)dp.h[s][r].size();
      if (ne == 0) continue;
      const cx<R>* in = s == 0 ? x : bufs[2 * v + (s - 1) % 2].p;
      const int64_t ldin = s == 0 ? ldx : pl.st[s - 1].ld_out;
      cx<R>* out = final ? y : bufs[2 * v + s % 2].p;
      const int64_t ldout = final ? ldy : d.ld_out;
      launch_bgemm<R>(c, d.op, d.M, d.K, d.S, d.A, d.lda, in, ldin, out, ldout, dp.d[s][r].p, ne, (int)k, false,
                      (int)k, true);
    }
  }
  if (real) {
    // disjoint output blocks: the sum assembles y on every process
    if constexpr (std::is_same<R, double>::value)
      comm_allreduce_sum_f64(c, reinterpret_cast<double*>(y), (size_t)(nout * k) * 2);
    else
      comm_allreduce_sum_f32(c, reinterpret_cast<float*>(y), (size_t)(nout * k) * 2);
  }
}

template void DevButterfly<double>::apply_layout(int, int, int, const double2*, int64_t, double2*, int64_t, int64_t,
                                                 double*);
template void DevButterfly<float>::apply_layout(int, int, int, const float2*, int64_t, float2*, int64_t, int64_t,
                                                double*);

}  // namespace bfly
