// comm.cu -- native row-band sharding over NCCL (SURVEY.md §8(b) "icl_comm_init /
// icl_*_sharded", §8(e) multi-GPU): one large image split into row bands across
// the ranks of one node, halo rows exchanged by one grouped ncclSend / ncclRecv
// per neighbour, overlapped with the rows that need no halo.
//
// Partition (identical to paper_1605_06399_b200/dist.py, which the CPU tests
// compare against): rank k owns global rows [r0, r1) = [k*ceil(H/N),
// min(r0 + ceil(H/N), H)) and its band buffer holds rows [s0, s1) =
// [max(0, r0 - up), min(H, r1 + down)); up/down are the stencil rows of the
// filter.  Filters run on the band through icl_band (boundary in GLOBAL
// coordinates), so stitched outputs equal the unsharded call -- bit for bit
// for sepconv, Harris and conv2d.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2", reusing the copy torch
// already mapped when present), so libicl.so has no link-time NCCL
// dependency and the rest of the library works without it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <cstdio>
#include <cstring>
#include <functional>
#include <mutex>

#include "../../include/icl.h"
#include "internal.h"

namespace icl {
namespace {

struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*);
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*commDestroy)(ncclComm_t);
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*groupStart)();
  ncclResult_t (*groupEnd)();
  const char* (*errorString)(ncclResult_t);
  // NCCL >= 2.28 symmetric memory (optional: nullptr with an older libnccl)
  ncclResult_t (*memAlloc)(void**, size_t);
  ncclResult_t (*memFree)(void*);
  ncclResult_t (*winRegister)(ncclComm_t, void*, size_t, void**, int);
  ncclResult_t (*winDeregister)(ncclComm_t, void*);
};

std::once_flag g_nccl_once;
NcclApi g_nccl;
bool g_nccl_ok = false;
char g_nccl_err[256] = "";

void load_nccl() {
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's copy, if mapped
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    snprintf(g_nccl_err, sizeof g_nccl_err, "libnccl.so.2 not loadable: %s", dlerror());
    return;
  }
#define ICL_SYM(field, name)                                                          \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name));            \
  if (!g_nccl.field) {                                                                \
    snprintf(g_nccl_err, sizeof g_nccl_err, "libnccl.so.2 lacks %s", name);           \
    return;                                                                           \
  }
  ICL_SYM(getUniqueId, "ncclGetUniqueId")
  ICL_SYM(commInitRank, "ncclCommInitRank")
  ICL_SYM(commDestroy, "ncclCommDestroy")
  ICL_SYM(send, "ncclSend")
  ICL_SYM(recv, "ncclRecv")
  ICL_SYM(groupStart, "ncclGroupStart")
  ICL_SYM(groupEnd, "ncclGroupEnd")
  ICL_SYM(errorString, "ncclGetErrorString")
#undef ICL_SYM
  g_nccl.memAlloc = reinterpret_cast<decltype(g_nccl.memAlloc)>(dlsym(h, "ncclMemAlloc"));
  g_nccl.memFree = reinterpret_cast<decltype(g_nccl.memFree)>(dlsym(h, "ncclMemFree"));
  g_nccl.winRegister = reinterpret_cast<decltype(g_nccl.winRegister)>(dlsym(h, "ncclCommWindowRegister"));
  g_nccl.winDeregister = reinterpret_cast<decltype(g_nccl.winDeregister)>(dlsym(h, "ncclCommWindowDeregister"));
  g_nccl_ok = true;
}

icl_status nccl(icl_status* st) {
  std::call_once(g_nccl_once, load_nccl);
  if (!g_nccl_ok) *st = report_error(ICL_ERR_NCCL, g_nccl_err);
  return g_nccl_ok ? ICL_OK : ICL_ERR_NCCL;
}

icl_status nccl_fail(ncclResult_t r, const char* what) {
  char buf[256];
  snprintf(buf, sizeof buf, "%s: %s", what, g_nccl.errorString ? g_nccl.errorString(r) : "nccl error");
  return report_error(ICL_ERR_NCCL, buf);
}

struct Band {
  int64_t H, r0, r1, s0, s1;
  int up, down, rank, N;
};

// dist.partition
bool partition(int64_t H, int N, int k, int up, int down, Band* b) {
  const int64_t per = (H + N - 1) / N;
  b->H = H;
  b->N = N;
  b->rank = k;
  b->up = up;
  b->down = down;
  b->r0 = std::min<int64_t>((int64_t)k * per, H);
  b->r1 = std::min<int64_t>(b->r0 + per, H);
  b->s0 = std::max<int64_t>(0, b->r0 - up);
  b->s1 = std::min<int64_t>(H, b->r1 + down);
  return !(N > 1 && b->r1 - b->r0 < std::max(up, down));
}

// The call is collective, so validity must be the same answer on every rank: reject the
// configuration when ANY rank's band is thinner than the halo (in practice the last one),
// not only when the calling rank's is -- otherwise a valid neighbour would post a send /
// recv that the rejecting rank never matches.
bool config_valid(int64_t H, int N, int up, int down) {
  Band t;
  for (int k = 0; k < N; ++k)
    if (!partition(H, N, k, up, down, &t)) return false;
  return true;
}

struct PlanEntry {
  int peer;
  int64_t send0, send1, recv0, recv1;
};

// dist.exchange_plan: symmetric by construction
int exchange_plan(const Band& b, PlanEntry out[2]) {
  int n = 0;
  if (b.r0 < b.r1 && b.rank > 0) {
    Band prev;
    if (partition(b.H, b.N, b.rank - 1, b.up, b.down, &prev)) {
      PlanEntry e{b.rank - 1, b.r0, prev.s1, b.s0, b.r0};
      if (e.send1 > e.send0 || e.recv1 > e.recv0) out[n++] = e;
    }
  }
  if (b.rank < b.N - 1) {
    Band nxt;
    if (partition(b.H, b.N, b.rank + 1, b.up, b.down, &nxt) && nxt.r0 < nxt.r1) {
      PlanEntry e{b.rank + 1, nxt.s0, b.r1, b.r1, b.s1};
      if (e.send1 > e.send0 || e.recv1 > e.recv0) out[n++] = e;
    }
  }
  return n;
}

icl_status halo_of(icl_filter f, int p0, int p1, int* up, int* down) {
  switch (f) {
    case ICL_FILTER_SEPCONV: *up = *down = p0; return ICL_OK;             // ry
    case ICL_FILTER_HARRIS: *up = p0 / 2 + 1; *down = p0 - 1 - p0 / 2 + 1; return ICL_OK;  // block
    case ICL_FILTER_NLM: *up = *down = p0 + p1; return ICL_OK;            // P + S
    case ICL_FILTER_CONV2D: *up = *down = p0; return ICL_OK;              // r
  }
  return report_error(ICL_ERR_INVALID_ARG, "unknown filter");
}

icl_image rows_of(const icl_image* im, int64_t row0, int64_t nrows) {
  icl_image v = *im;
  v.data = static_cast<char*>(im->data) + row0 * im->pitch_bytes;
  v.height = nrows;
  return v;
}

}  // namespace
}  // namespace icl

using namespace icl;

// In-process loopback transport (icl_comm_init_local): N communicators of ONE process, every
// rank driven by its own host thread, exchanging the packed halo rows by device copies through
// per-(src, dst) mailboxes instead of ncclSend / ncclRecv.  It keeps NCCL's matching and
// completion semantics -- a recv waits for the peer's matching send to be POSTED, copies after
// the sender's packed rows are ready (event), and a send completes (on the sender's comm
// stream) only after the receiver's copy -- so run_sharded's pack -> exchange -> unpack runs
// unchanged at N = 2..8 on one GPU (NCCL refuses two ranks on one device).  Test plumbing for
// the exchange path, not a product transport.
struct LocalMsg {
  const void* src = nullptr;
  size_t bytes = 0;
  cudaEvent_t ready = nullptr;  // sender's packed rows complete
  cudaEvent_t done = nullptr;   // receiver's copy complete
  bool acked = false;
};

struct LocalGroup {
  int n = 0, refs = 0;
  std::mutex mu;
  std::condition_variable cv;
  std::deque<LocalMsg*> box[ICL_LOCAL_MAX_RANKS][ICL_LOCAL_MAX_RANKS];  // [src][dst], FIFO per pair
};

struct icl_comm {
  LocalGroup* lg = nullptr;  // non-null: in-process loopback transport
  ncclComm_t nc = nullptr;
  int nranks = 1, rank = 0;
  cudaStream_t cs = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  char* stage = nullptr;  // packed halo rows: [send q0 | recv q0 | send q1 | recv q1]
  size_t stage_bytes = 0;
};

namespace {
using BandCall = std::function<icl_status(const icl_image* src, const icl_image* dst, const icl_image* mask,
                                          const icl_band* band, cudaStream_t s)>;

// The grouped send / recv of one run_sharded call over the loopback transport: post every
// send, then serve every recv (host-wait for the peer's post, device copy after its ready
// event), then wait for the receivers' copies of this rank's sends.  Every rank posts before
// it blocks, so the group cannot deadlock.
icl_status local_exchange(icl_comm* c, const PlanEntry* plan, int np, const size_t* off, int64_t row_bytes) {
  LocalGroup* g = c->lg;
  LocalMsg* sent[2] = {nullptr, nullptr};
  cudaError_t e;
  for (int q = 0; q < np; ++q) {
    const size_t sb = (size_t)((plan[q].send1 - plan[q].send0) * row_bytes);
    if (!sb) continue;
    LocalMsg* m = new LocalMsg();
    m->src = c->stage + off[2 * q];
    m->bytes = sb;
    if ((e = cudaEventCreateWithFlags(&m->ready, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&m->done, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventRecord(m->ready, c->cs)) != cudaSuccess) {
      delete m;
      return report_error(ICL_ERR_CUDA, cudaGetErrorString(e));
    }
    sent[q] = m;
    std::lock_guard<std::mutex> lk(g->mu);
    g->box[c->rank][plan[q].peer].push_back(m);
    g->cv.notify_all();
  }
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(120);
  for (int q = 0; q < np; ++q) {
    const size_t rb = (size_t)((plan[q].recv1 - plan[q].recv0) * row_bytes);
    if (!rb) continue;
    std::unique_lock<std::mutex> lk(g->mu);
    auto& bx = g->box[plan[q].peer][c->rank];
    if (!g->cv.wait_until(lk, deadline, [&] { return !bx.empty(); }))
      return report_error(ICL_ERR_NCCL, "local transport: the peer never posted its send (is every rank calling?)");
    LocalMsg* m = bx.front();
    bx.pop_front();
    lk.unlock();
    if (m->bytes != rb) return report_error(ICL_ERR_NCCL, "local transport: send / recv sizes differ");
    cudaStreamWaitEvent(c->cs, m->ready, 0);
    if ((e = cudaMemcpyAsync(c->stage + off[2 * q + 1], m->src, rb, cudaMemcpyDeviceToDevice, c->cs)) != cudaSuccess)
      return report_error(ICL_ERR_CUDA, cudaGetErrorString(e));
    cudaEventRecord(m->done, c->cs);
    lk.lock();
    m->acked = true;
    g->cv.notify_all();
  }
  for (int q = 0; q < np; ++q) {
    LocalMsg* m = sent[q];
    if (!m) continue;
    {
      std::unique_lock<std::mutex> lk(g->mu);
      if (!g->cv.wait_until(lk, deadline, [&] { return m->acked; }))
        return report_error(ICL_ERR_NCCL, "local transport: the peer never received this rank's send");
    }
    cudaStreamWaitEvent(c->cs, m->done, 0);  // the send completes once the peer's copy has run
    cudaEventDestroy(m->ready);  // released by the driver once the pending work completes
    cudaEventDestroy(m->done);
    delete m;
  }
  return ICL_OK;
}

// Exchange the halo rows of `buf` and run the filter on the rank's rows of `dst`.
icl_status run_sharded(icl_comm* c, const icl_image* buf, const icl_image* dst, const icl_image* mask, int64_t H,
                       int up, int down, int elem, const BandCall& call, cudaStream_t user) {
  if (!c) return report_error(ICL_ERR_INVALID_ARG, "null comm");
  if (!buf || !dst || !buf->data || !dst->data) return report_error(ICL_ERR_INVALID_ARG, "null image");
  Band b;
  if (!partition(H, c->nranks, c->rank, up, down, &b) || !config_valid(H, c->nranks, up, down))
    return report_error(ICL_ERR_INVALID_ARG, "a row band (this rank's or another's) is thinner than the halo");
  if (buf->height != b.s1 - b.s0 || dst->height != b.r1 - b.r0) {
    char m[200];
    snprintf(m, sizeof m, "rank %d: band buffer must hold rows [%lld, %lld) and dst rows [%lld, %lld)", c->rank,
             (long long)b.s0, (long long)b.s1, (long long)b.r0, (long long)b.r1);
    return report_error(ICL_ERR_INVALID_ARG, m);
  }
  if (b.r1 == b.r0) return ICL_OK;  // an empty rank (more ranks than rows)
  PlanEntry plan[2];
  const int np = c->nranks > 1 ? exchange_plan(b, plan) : 0;
  const icl_band whole{H, b.s0, b.r0};
  if (np == 0) return call(buf, dst, mask, &whole, user);

  // exchange on the comm stream, forked from the caller's stream (own rows are ready there)
  cudaError_t e;
  if ((e = cudaEventRecord(c->fork, user)) != cudaSuccess) return report_error(ICL_ERR_CUDA, cudaGetErrorString(e));
  cudaStreamWaitEvent(c->cs, c->fork, 0);
  // one ncclSend + one ncclRecv per neighbour of PACKED rows (all images of the batch), so the
  // message shapes never depend on either side's pitch; pack / unpack are 2-D copies on the
  // comm stream
  const int64_t rowb = buf->width * elem;
  const int64_t B = buf->batch, bstride = buf->batch > 1 ? buf->batch_stride_bytes : 0;
  size_t off[4], need = 0;
  for (int q = 0; q < np; ++q) {
    off[2 * q] = need;
    need += (size_t)((plan[q].send1 - plan[q].send0) * rowb * B + 255) / 256 * 256;
    off[2 * q + 1] = need;
    need += (size_t)((plan[q].recv1 - plan[q].recv0) * rowb * B + 255) / 256 * 256;
  }
  if (need > c->stage_bytes) {
    cudaStreamSynchronize(c->cs);
    if (c->stage) cudaFree(c->stage);
    c->stage = nullptr;
    c->stage_bytes = 0;
    if ((e = cudaMalloc(&c->stage, need)) != cudaSuccess) return report_error(ICL_ERR_CUDA, cudaGetErrorString(e));
    c->stage_bytes = need;
  }
  auto rows2d = [&](int64_t img, int64_t g0) {
    return static_cast<char*>(buf->data) + img * bstride + (g0 - b.s0) * buf->pitch_bytes;
  };
  for (int q = 0; q < np; ++q) {  // pack
    const int64_t n = plan[q].send1 - plan[q].send0;
    for (int64_t img = 0; img < B && n > 0; ++img)
      cudaMemcpy2DAsync(c->stage + off[2 * q] + img * n * rowb, rowb, rows2d(img, plan[q].send0), buf->pitch_bytes,
                        rowb, n, cudaMemcpyDeviceToDevice, c->cs);
  }
  if (c->lg) {
    icl_status xs = local_exchange(c, plan, np, off, rowb * B);
    if (xs != ICL_OK) return xs;
  } else {
    ncclResult_t r = g_nccl.groupStart();
    if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
    for (int q = 0; q < np && r == ncclSuccess; ++q) {
      const size_t sb = (size_t)((plan[q].send1 - plan[q].send0) * rowb * B);
      const size_t rb = (size_t)((plan[q].recv1 - plan[q].recv0) * rowb * B);
      if (sb) r = g_nccl.send(c->stage + off[2 * q], sb, ncclUint8, plan[q].peer, c->nc, c->cs);
      if (r == ncclSuccess && rb) r = g_nccl.recv(c->stage + off[2 * q + 1], rb, ncclUint8, plan[q].peer, c->nc, c->cs);
    }
    ncclResult_t r2 = g_nccl.groupEnd();
    if (r != ncclSuccess) return nccl_fail(r, "ncclSend/ncclRecv");
    if (r2 != ncclSuccess) return nccl_fail(r2, "ncclGroupEnd");
  }
  for (int q = 0; q < np; ++q) {  // unpack
    const int64_t n = plan[q].recv1 - plan[q].recv0;
    for (int64_t img = 0; img < B && n > 0; ++img)
      cudaMemcpy2DAsync(rows2d(img, plan[q].recv0), buf->pitch_bytes, c->stage + off[2 * q + 1] + img * n * rowb, rowb,
                        rowb, n, cudaMemcpyDeviceToDevice, c->cs);
  }
  cudaEventRecord(c->join, c->cs);

  // rows that need no halo run on the caller's stream during the exchange
  const int64_t i0 = b.r0 + (b.r0 > 0 ? up : 0), i1 = b.r1 - (b.r1 < H ? down : 0);
  icl_status st = ICL_OK;
  if (i1 > i0) {
    const icl_image dv = rows_of(dst, i0 - b.r0, i1 - i0);
    const icl_image mv = mask && mask->data ? rows_of(mask, i0 - b.r0, i1 - i0) : icl_image{};
    const icl_band bi{H, b.s0, i0};
    st = call(buf, &dv, mask && mask->data ? &mv : nullptr, &bi, user);
  }
  cudaStreamWaitEvent(user, c->join, 0);  // halo rows present from here on
  if (st != ICL_OK) return st;
  auto edge = [&](int64_t a0, int64_t a1) -> icl_status {
    if (a1 <= a0) return ICL_OK;
    const icl_image dv = rows_of(dst, a0 - b.r0, a1 - a0);
    const icl_image mv = mask && mask->data ? rows_of(mask, a0 - b.r0, a1 - a0) : icl_image{};
    const icl_band be{H, b.s0, a0};
    return call(buf, &dv, mask && mask->data ? &mv : nullptr, &be, user);
  };
  if ((st = edge(b.r0, std::min(i0, b.r1))) != ICL_OK) return st;
  return edge(std::max(i1, i0), b.r1);
}
}  // namespace

extern "C" {

icl_status icl_halo_rows(icl_filter filter, int p0, int p1, int* up, int* down) {
  if (!up || !down) return report_error(ICL_ERR_INVALID_ARG, "null output");
  return halo_of(filter, p0, p1, up, down);
}

icl_status icl_shard_band(int64_t global_height, int nranks, int rank, int up, int down, int64_t out[4]) {
  if (!out || global_height < 1 || nranks < 1 || rank < 0 || rank >= nranks || up < 0 || down < 0)
    return report_error(ICL_ERR_INVALID_ARG, "bad shard arguments");
  Band b;
  const bool ok = partition(global_height, nranks, rank, up, down, &b);
  out[0] = b.r0;
  out[1] = b.r1;
  out[2] = b.s0;
  out[3] = b.s1;
  return ok ? ICL_OK : report_error(ICL_ERR_INVALID_ARG, "row band thinner than the halo");
}

icl_status icl_shard_plan(int64_t global_height, int nranks, int rank, int up, int down, int64_t plan[10], int* n) {
  int64_t bb[4];
  icl_status st = icl_shard_band(global_height, nranks, rank, up, down, bb);
  if (st != ICL_OK) return st;
  if (!plan || !n) return report_error(ICL_ERR_INVALID_ARG, "null output");
  Band b;
  partition(global_height, nranks, rank, up, down, &b);
  PlanEntry pe[2];
  *n = exchange_plan(b, pe);
  for (int q = 0; q < *n; ++q) {
    plan[5 * q] = pe[q].peer;
    plan[5 * q + 1] = pe[q].send0;
    plan[5 * q + 2] = pe[q].send1;
    plan[5 * q + 3] = pe[q].recv0;
    plan[5 * q + 4] = pe[q].recv1;
  }
  return ICL_OK;
}

icl_status icl_comm_unique_id(void* id) {
  if (!id) return report_error(ICL_ERR_INVALID_ARG, "null id");
  icl_status st = ICL_OK;
  if (nccl(&st) != ICL_OK) return st;
  ncclUniqueId u;
  ncclResult_t r = g_nccl.getUniqueId(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(id, &u, sizeof u);
  return ICL_OK;
}

icl_status icl_comm_init(icl_comm** comm, int nranks, int rank, const void* id) {
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks)
    return report_error(ICL_ERR_INVALID_ARG, "bad comm arguments");
  icl_status st = ICL_OK;
  if (nccl(&st) != ICL_OK) return st;
  icl_comm* c = new icl_comm();
  c->nranks = nranks;
  c->rank = rank;
  ncclUniqueId u;
  memcpy(&u, id, sizeof u);
  ncclResult_t r = g_nccl.commInitRank(&c->nc, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming)) != cudaSuccess) {
    g_nccl.commDestroy(c->nc);
    delete c;
    return report_error(ICL_ERR_CUDA, cudaGetErrorString(e));
  }
  *comm = c;
  return ICL_OK;
}

icl_status icl_comm_init_local(icl_comm** comms, int nranks) {
  if (!comms || nranks < 1 || nranks > ICL_LOCAL_MAX_RANKS)
    return report_error(ICL_ERR_INVALID_ARG, "nranks must be in [1, ICL_LOCAL_MAX_RANKS]");
  LocalGroup* g = new LocalGroup();
  g->n = nranks;
  for (int k = 0; k < nranks; ++k) {
    icl_comm* c = new icl_comm();
    c->lg = g;
    c->nranks = nranks;
    c->rank = k;
    cudaError_t e;
    if ((e = cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming)) != cudaSuccess) {
      for (int j = 0; j < k; ++j) icl_comm_destroy(comms[j]);
      if (c->cs) cudaStreamDestroy(c->cs);
      delete c;
      if (k == 0) delete g;
      return report_error(ICL_ERR_CUDA, cudaGetErrorString(e));
    }
    g->refs++;
    comms[k] = c;
  }
  return ICL_OK;
}

icl_status icl_comm_destroy(icl_comm* comm) {
  if (!comm) return ICL_OK;
  if (comm->cs) cudaStreamSynchronize(comm->cs);
  if (comm->lg) {
    LocalGroup* g = comm->lg;
    bool last;
    {
      std::lock_guard<std::mutex> lk(g->mu);
      last = --g->refs == 0;
    }
    if (last) delete g;
  }
  ncclResult_t r = comm->nc ? g_nccl.commDestroy(comm->nc) : ncclSuccess;
  if (comm->fork) cudaEventDestroy(comm->fork);
  if (comm->join) cudaEventDestroy(comm->join);
  if (comm->stage) cudaFree(comm->stage);
  if (comm->cs) cudaStreamDestroy(comm->cs);
  delete comm;
  return r == ncclSuccess ? ICL_OK : nccl_fail(r, "ncclCommDestroy");
}

// ---------------------------------------------------------------- NCCL symmetric windows (§8(f) row 3)
static icl_status window_api(icl_comm* comm) {
  if (!comm) return report_error(ICL_ERR_INVALID_ARG, "null comm");
  if (comm->lg || !comm->nc) return report_error(ICL_ERR_UNSUPPORTED, "symmetric windows need an NCCL communicator");
  icl_status st = ICL_OK;
  if (nccl(&st) != ICL_OK) return st;
  if (!g_nccl.memAlloc || !g_nccl.memFree || !g_nccl.winRegister || !g_nccl.winDeregister)
    return report_error(ICL_ERR_UNSUPPORTED, "libnccl.so.2 has no symmetric-memory API (NCCL >= 2.28)");
  return ICL_OK;
}

icl_status icl_comm_mem_alloc(icl_comm* comm, size_t bytes, void** ptr) {
  icl_status st = window_api(comm);
  if (st != ICL_OK) return st;
  if (!ptr || !bytes) return report_error(ICL_ERR_INVALID_ARG, "null pointer or zero bytes");
  ncclResult_t r = g_nccl.memAlloc(ptr, bytes);
  return r == ncclSuccess ? ICL_OK : nccl_fail(r, "ncclMemAlloc");
}

icl_status icl_comm_mem_free(icl_comm* comm, void* ptr) {
  icl_status st = window_api(comm);
  if (st != ICL_OK || !ptr) return st;
  ncclResult_t r = g_nccl.memFree(ptr);
  return r == ncclSuccess ? ICL_OK : nccl_fail(r, "ncclMemFree");
}

icl_status icl_comm_window_register(icl_comm* comm, void* buf, size_t bytes, icl_window** win) {
  icl_status st = window_api(comm);
  if (st != ICL_OK) return st;
  if (!buf || !bytes || !win) return report_error(ICL_ERR_INVALID_ARG, "null buffer / size / output");
  void* w = nullptr;
  ncclResult_t r = g_nccl.winRegister(comm->nc, buf, bytes, &w, 0x01 /* NCCL_WIN_COLL_SYMMETRIC */);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommWindowRegister");
  icl_window* iw = new icl_window();
  iw->win = w;
  iw->buf = buf;
  iw->bytes = bytes;
  iw->rank = comm->rank;
  iw->nranks = comm->nranks;
  *win = iw;
  return ICL_OK;
}

icl_status icl_comm_window_deregister(icl_comm* comm, icl_window* win) {
  if (!win) return ICL_OK;
  icl_status st = window_api(comm);
  if (st != ICL_OK) return st;
  if (comm->cs) cudaStreamSynchronize(comm->cs);
  ncclResult_t r = g_nccl.winDeregister(comm->nc, win->win);
  delete win;
  return r == ncclSuccess ? ICL_OK : nccl_fail(r, "ncclCommWindowDeregister");
}

icl_status icl_sepconv_sharded(icl_comm* comm, const icl_image* buf, const icl_image* dst, int64_t global_height,
                               const float* taps_x, int rx, const float* taps_y, int ry, icl_border border,
                               float border_value, void* stream) {
  return run_sharded(comm, buf, dst, nullptr, global_height, ry, ry, 4,
                     [&](const icl_image* s, const icl_image* d, const icl_image*, const icl_band* b,
                         cudaStream_t cs) {
                       return icl_sepconv(s, d, taps_x, rx, taps_y, ry, border, border_value, b, nullptr, 0, cs);
                     },
                     static_cast<cudaStream_t>(stream));
}

icl_status icl_harris_sharded(icl_comm* comm, const icl_image* buf, const icl_image* response, int64_t global_height,
                              int block, float k, icl_border border, float border_value, const icl_image* mask,
                              float threshold, void* stream) {
  int up = 0, down = 0;
  halo_of(ICL_FILTER_HARRIS, block, 0, &up, &down);
  return run_sharded(comm, buf, response, mask, global_height, up, down, 4,
                     [&](const icl_image* s, const icl_image* d, const icl_image* m, const icl_band* b,
                         cudaStream_t cs) {
                       return icl_harris(s, d, block, k, border, border_value, m, threshold, b, cs);
                     },
                     static_cast<cudaStream_t>(stream));
}

icl_status icl_nlm_sharded(icl_comm* comm, const icl_image* buf, const icl_image* dst, int64_t global_height,
                           int patch_radius, int search_radius, float h, icl_border border, float border_value,
                           void* stream) {
  const int r = patch_radius + search_radius;
  return run_sharded(comm, buf, dst, nullptr, global_height, r, r, 4,
                     [&](const icl_image* s, const icl_image* d, const icl_image*, const icl_band* b,
                         cudaStream_t cs) {
                       return icl_nlm(s, d, patch_radius, search_radius, h, border, border_value, b, cs);
                     },
                     static_cast<cudaStream_t>(stream));
}

icl_status icl_conv2d_u8_sharded(icl_comm* comm, const icl_image* buf, const icl_image* dst, int64_t global_height,
                                 const float* filter, int radius, icl_border border, float border_value,
                                 void* stream) {
  return run_sharded(comm, buf, dst, nullptr, global_height, radius, radius, 1,
                     [&](const icl_image* s, const icl_image* d, const icl_image*, const icl_band* b,
                         cudaStream_t cs) {
                       return icl_conv2d_u8(s, d, filter, radius, border, border_value, b, cs);
                     },
                     static_cast<cudaStream_t>(stream));
}

}  // extern "C"
