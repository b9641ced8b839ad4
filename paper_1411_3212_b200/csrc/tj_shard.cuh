// Multi-GPU data plane of the sharded tick (the reference is
// single-process, so there is no reference counterpart).
//
// One process (or thread) per GPU, one context per rank.  A rank's tick:
//   1. the ranks' slice sizes are exchanged; every rank's slice of the
//      objects and queries is gathered into the full tick (NCCL broadcasts
//      from every root inside one group: variable-sized all-gather);
//   2. the full tick runs with the rank's contiguous Morton range of leaves
//      (k_shard_mark): its per-query lists are the results restricted to
//      those leaves, disjoint across ranks and each sorted by id;
//   3. each query's partial lists go to the query's home rank (the rank
//      whose slice issued it): the partial CSR restricted to a home rank's
//      query range is contiguous, so the exchange is an all-to-all of
//      per-query counts, then of id runs (NCCL send/recv in one group);
//   4. the home rank merges the G sorted partial lists of each of its queries
//      on the device (k_merge_partials) into its queries' complete CSR.
// Transports: NCCL (tj_comm_init; libnccl.so.2 is loaded at run time, so the
// library has no link-time NCCL dependency), or an in-process group of
// contexts driven from one thread each (tj_comm_init_local: the whole
// protocol on one device, for tests and single-GPU checks).
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <mutex>

namespace tj {

// per query: results in this rank's partial CSR
__global__ void __launch_bounds__(256) k_partial_counts(const int64_t* __restrict__ off, int32_t* __restrict__ cnt,
                                                        int64_t m) {
  TJ_GRID_STRIDE(q, m) cnt[q] = (int32_t)(off[q + 1] - off[q]);
}

// per own query: total over the G sources
struct SumIn {
  const int32_t* cnt;  // [G][M]
  int G;
  int64_t M;
  __device__ int64_t operator()(int64_t q) const {
    int64_t s = 0;
    for (int j = 0; j < G; ++j) s += cnt[(int64_t)j * M + q];
    return s;
  }
};

// The union of each own query's G disjoint, id-sorted partial lists (source
// j's run of query q starts at src[j] + start[j][q]).  A warp owns 32
// consecutive queries: lists with one non-empty source (most of them: a
// query's leaves usually lie in one rank's range) are copied by the whole
// warp, coalesced; lists from several sources are merged by heads, one lane
// per query.
__global__ void __launch_bounds__(256) k_merge_partials(int G, int64_t M, const int32_t* __restrict__ cnt,
                                                        const int64_t* __restrict__ start,
                                                        const int64_t* const* __restrict__ src,
                                                        const int64_t* __restrict__ moff, int64_t* __restrict__ mids) {
  constexpr int kMaxG = 64;
  const int lane = lane_id();
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; q0 < M; q0 += nwarp * 32) {
    const int64_t q = q0 + lane;
    int nz = 0, last = 0;
    if (q < M)
      for (int j = 0; j < G; ++j)
        if (cnt[(int64_t)j * M + q]) {
          ++nz;
          last = j;
        }
    // single-source lists: the warp copies them one after another
    unsigned single = __ballot_sync(0xffffffffu, nz == 1);
    while (single) {
      const int l = __ffs(single) - 1;
      single &= single - 1;
      const int64_t ql = q0 + l;
      const int j = __shfl_sync(0xffffffffu, last, l);
      const int c = cnt[(int64_t)j * M + ql];
      const int64_t* s_ = src[j] + start[(int64_t)j * M + ql];
      int64_t* dst = mids + moff[ql];
      for (int k = lane; k < c; k += 32) dst[k] = s_[k];
    }
    if (nz > 1) {
      const int64_t* pos[kMaxG];
      const int64_t* end[kMaxG];
      int total = 0;
      for (int j = 0; j < G; ++j) {
        const int c = cnt[(int64_t)j * M + q];
        pos[j] = src[j] + start[(int64_t)j * M + q];
        end[j] = pos[j] + c;
        total += c;
      }
      int64_t* dst = mids + moff[q];
      for (int o = 0; o < total; ++o) {
        int bj = -1;
        int64_t bv = 0;
        for (int j = 0; j < G; ++j)
          if (pos[j] < end[j] && (bj < 0 || *pos[j] < bv)) {
            bj = j;
            bv = *pos[j];
          }
        dst[o] = bv;
        ++pos[bj];
      }
    }
  }
}

}  // namespace tj

// ---------------------------------------------------------------------------
// Transports
// ---------------------------------------------------------------------------
struct Transport {
  int rank = 0, nranks = 1;
  virtual ~Transport() = default;
  virtual const char* name() const = 0;
  // all-gather of k int64 values per rank into all[nranks * k] (host memory)
  virtual int exchange_host(tj_ctx* c, const int64_t* mine, int k, int64_t* all) = 0;
  // variable-sized all-gather: rank j's counts[j] elements land at recv + displs[j] (elements)
  virtual int allgatherv(tj_ctx* c, const void* send, void* recv, const int64_t* counts, const int64_t* displs,
                         size_t elem) = 0;
  // all-to-all: scounts[j] elements from send + sdispls[j] go to rank j; rank j's rcounts[j] land at
  // recv + rdispls[j]
  virtual int alltoallv(tj_ctx* c, const void* send, const int64_t* scounts, const int64_t* sdispls, void* recv,
                        const int64_t* rcounts, const int64_t* rdispls, size_t elem) = 0;
};

namespace {

// ---- NCCL, resolved at run time ---------------------------------------------
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string err;
};

NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (tried) return api.h ? &api : nullptr;
  tried = true;
  // the process's NCCL if one is loaded (torch's), else the system's
  const char* env = std::getenv("TJ_NCCL_LIB");
  const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    if (!nm) continue;
    api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (api.h) break;
  }
  if (!api.h) {
    api.err = std::string("cannot load libnccl.so.2: ") + dlerror();
    return nullptr;
  }
#define TJ_SYM(f)                                                        \
  api.f = reinterpret_cast<decltype(api.f)>(dlsym(api.h, "nccl" #f));    \
  if (!api.f) {                                                          \
    api.err = "libnccl.so.2 lacks nccl" #f;                              \
    api.h = nullptr;                                                     \
    return nullptr;                                                      \
  }
  TJ_SYM(GetUniqueId) TJ_SYM(CommInitRank) TJ_SYM(CommDestroy) TJ_SYM(AllGather) TJ_SYM(Broadcast) TJ_SYM(Send)
  TJ_SYM(Recv) TJ_SYM(GroupStart) TJ_SYM(GroupEnd) TJ_SYM(GetErrorString)
#undef TJ_SYM
  return &api;
}

struct NcclTransport : Transport {
  NcclApi* api = nullptr;
  ncclComm_t comm = nullptr;
  DBuf scratch;  // exchange_host staging
  const char* name() const override { return "nccl"; }
  ~NcclTransport() override {
    if (comm) api->CommDestroy(comm);
    if (scratch.p) cudaFree(scratch.p);
  }
  int check(tj_ctx* c, ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return TJ_OK;
    return fail(c, TJ_E_NCCL, std::string(what) + ": " + api->GetErrorString(r));
  }
  int exchange_host(tj_ctx* c, const int64_t* mine, int k, int64_t* all) override {
    int rc;
    if ((rc = ensure(c, scratch, (size_t)(nranks + 1) * k * 8))) return rc;
    int64_t* d = P<int64_t>(scratch);
    TJ_CUDA(cudaMemcpyAsync(d + (size_t)nranks * k, mine, k * 8, cudaMemcpyHostToDevice, c->st));
    if ((rc = check(c, api->AllGather(d + (size_t)nranks * k, d, k, ncclInt64, comm, c->st), "ncclAllGather")))
      return rc;
    TJ_CUDA(cudaMemcpyAsync(all, d, (size_t)nranks * k * 8, cudaMemcpyDeviceToHost, c->st));
    TJ_CUDA(cudaStreamSynchronize(c->st));
    return TJ_OK;
  }
  int allgatherv(tj_ctx* c, const void* send, void* recv, const int64_t* counts, const int64_t* displs,
                 size_t elem) override {
    int rc;
    if ((rc = check(c, api->GroupStart(), "ncclGroupStart"))) return rc;
    for (int j = 0; j < nranks; ++j) {
      char* dst = static_cast<char*>(recv) + displs[j] * elem;
      const void* src = j == rank ? send : dst;
      if (counts[j] == 0) continue;
      if ((rc = check(c, api->Broadcast(src, dst, counts[j] * elem, ncclUint8, j, comm, c->st), "ncclBroadcast")))
        return rc;
    }
    return check(c, api->GroupEnd(), "ncclGroupEnd");
  }
  int alltoallv(tj_ctx* c, const void* send, const int64_t* scounts, const int64_t* sdispls, void* recv,
                const int64_t* rcounts, const int64_t* rdispls, size_t elem) override {
    int rc;
    if ((rc = check(c, api->GroupStart(), "ncclGroupStart"))) return rc;
    for (int j = 0; j < nranks; ++j) {
      if (scounts[j] &&
          (rc = check(c, api->Send(static_cast<const char*>(send) + sdispls[j] * elem, scounts[j] * elem, ncclUint8, j,
                                   comm, c->st), "ncclSend")))
        return rc;
      if (rcounts[j] &&
          (rc = check(c, api->Recv(static_cast<char*>(recv) + rdispls[j] * elem, rcounts[j] * elem, ncclUint8, j,
                                   comm, c->st), "ncclRecv")))
        return rc;
    }
    return check(c, api->GroupEnd(), "ncclGroupEnd");
  }
};

}  // namespace

// ---- in-process group: G contexts on threads of one process ------------------
struct tj_group {
  int n = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  std::vector<const void*> ptr;
  std::vector<const int64_t*> cnt, displ;
  std::vector<int64_t> vals;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

namespace {

struct LocalTransport : Transport {
  tj_group* g = nullptr;
  const char* name() const override { return "local"; }
  int exchange_host(tj_ctx* c, const int64_t* mine, int k, int64_t* all) override {
    (void)c;
    {
      std::lock_guard<std::mutex> lk(g->mu);
      if ((int64_t)g->vals.size() < (int64_t)nranks * k) g->vals.resize((size_t)nranks * k);
    }
    g->barrier();
    std::memcpy(g->vals.data() + (size_t)rank * k, mine, k * 8);
    g->barrier();
    std::memcpy(all, g->vals.data(), (size_t)nranks * k * 8);
    g->barrier();
    return TJ_OK;
  }
  int allgatherv(tj_ctx* c, const void* send, void* recv, const int64_t* counts, const int64_t* displs,
                 size_t elem) override {
    TJ_CUDA(cudaStreamSynchronize(c->st));  // this rank's slice is ready
    g->ptr[rank] = send;
    g->barrier();
    for (int j = 0; j < nranks; ++j) {
      char* dst = static_cast<char*>(recv) + displs[j] * elem;
      if (counts[j] && g->ptr[j] != dst)
        TJ_CUDA(cudaMemcpyAsync(dst, g->ptr[j], counts[j] * elem, cudaMemcpyDeviceToDevice, c->st));
    }
    TJ_CUDA(cudaStreamSynchronize(c->st));
    g->barrier();  // every peer has read this rank's slice
    return TJ_OK;
  }
  int alltoallv(tj_ctx* c, const void* send, const int64_t* scounts, const int64_t* sdispls, void* recv,
                const int64_t* rcounts, const int64_t* rdispls, size_t elem) override {
    TJ_CUDA(cudaStreamSynchronize(c->st));
    g->ptr[rank] = send;
    g->cnt[rank] = scounts;
    g->displ[rank] = sdispls;
    g->barrier();
    for (int j = 0; j < nranks; ++j) {
      const int64_t k = g->cnt[j][rank];
      if (k != rcounts[j]) return fail(c, TJ_E_NCCL, "all-to-all counts disagree across the group");
      if (k)
        TJ_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + rdispls[j] * elem,
                                static_cast<const char*>(g->ptr[j]) + g->displ[j][rank] * elem, k * elem,
                                cudaMemcpyDeviceToDevice, c->st));
    }
    TJ_CUDA(cudaStreamSynchronize(c->st));
    g->barrier();
    return TJ_OK;
  }
};

// the sharded tick: gather -> sharded device tick -> partials to home ranks -> device merge
int sharded_tick(tj_ctx* c, const tj_tick_in* in, tj_tick_out* out, tj_stats& S) {
  Transport& T = *c->comm;
  const int G = T.nranks, r = T.rank;
  int rc;
  const int64_t mine[2] = {in->n_obj, in->n_q};
  std::vector<int64_t> all(2 * G), N(G), M(G), nd(G + 1, 0), md(G + 1, 0);
  if ((rc = T.exchange_host(c, mine, 2, all.data()))) return rc;
  for (int j = 0; j < G; ++j) {
    N[j] = all[2 * j];
    M[j] = all[2 * j + 1];
    nd[j + 1] = nd[j] + N[j];
    md[j + 1] = md[j] + M[j];
  }
  const int64_t n = nd[G], m = md[G], Mr = M[r];
  if (n >= (int64_t(1) << 28) || m > INT32_MAX / 2)
    return fail(c, TJ_E_INVALID_ARG, "sharded tick too large for 32-bit rows");
  // 1. the full tick on every rank
  if ((rc = ensure(c, c->ids, n * 8)) || (rc = ensure(c, c->xs, n * 8)) || (rc = ensure(c, c->ys, n * 8)) ||
      (rc = ensure(c, c->qxa, m * 8)) || (rc = ensure(c, c->qya, m * 8)) || (rc = ensure(c, c->qxb, m * 8)) ||
      (rc = ensure(c, c->qyb, m * 8)))
    return rc;
  DBuf* full[7] = {&c->ids, &c->xs, &c->ys, &c->qxa, &c->qya, &c->qxb, &c->qyb};
  const void* src[7] = {in->obj_id, in->obj_x, in->obj_y, in->q_xa, in->q_ya, in->q_xb, in->q_yb};
  for (int a = 0; a < 7; ++a) {
    const bool obj = a < 3;
    const int64_t cnt = obj ? N[r] : Mr, off = obj ? nd[r] : md[r];
    char* slot = static_cast<char*>(full[a]->p) + off * 8;
    const void* send = src[a];
    if (in->mem == TJ_MEM_HOST) {  // this rank's slice lands in its place of the full array first
      if (cnt) TJ_CUDA(cudaMemcpyAsync(slot, src[a], cnt * 8, cudaMemcpyHostToDevice, c->st));
      send = slot;
    }
    if ((rc = T.allgatherv(c, send, full[a]->p, obj ? N.data() : M.data(), obj ? nd.data() : md.data(), 8)))
      return rc;
  }
  c->shard_rank = r;
  c->shard_n = G;
  int64_t R = 0;
  if ((rc = compute_tick(c, n, m, P<int64_t>(c->ids), P<double>(c->xs), P<double>(c->ys), P<double>(c->qxa),
                         P<double>(c->qya), P<double>(c->qxb), P<double>(c->qyb), S, R)))
    return rc;
  if (G == 1) {  // one rank: the tick's lists are already complete
    S.n_objects = n;
    S.n_queries = m;
    return deliver(c, in->out_mem, out, m, R, n > 0, c->outoff, c->outids, c->scratch, S);
  }
  // 2. partial lists to the home ranks: per-query counts, then the id runs
  if ((rc = ensure(c, c->pcnt, (size_t)std::max<int64_t>(m, 1) * 4)) ||
      (rc = ensure(c, c->rcnt, (size_t)std::max<int64_t>(G * Mr, 1) * 4)) ||
      (rc = ensure(c, c->sstart, (size_t)std::max<int64_t>(G * Mr, 1) * 8)) ||
      (rc = ensure(c, c->moff, (size_t)(Mr + 1) * 8)) || (rc = ensure(c, c->sconst, 64 * 8)))
    return rc;
  if (m) k_partial_counts<<<c->num_sms * 4, 256, 0, c->st>>>(P<int64_t>(c->outoff), P<int32_t>(c->pcnt), m);
  std::vector<int64_t> bound(G + 1), scnt(G), sdis(G), rqc(G, Mr), rqd(G);
  for (int j = 0; j <= G; ++j)
    TJ_CUDA(cudaMemcpyAsync(&bound[j], P<int64_t>(c->outoff) + md[j], 8, cudaMemcpyDeviceToHost, c->st));
  TJ_CUDA(cudaStreamSynchronize(c->st));
  for (int j = 0; j < G; ++j) {
    scnt[j] = bound[j + 1] - bound[j];
    sdis[j] = bound[j];
    rqd[j] = (int64_t)j * Mr;
  }
  if ((rc = T.alltoallv(c, c->pcnt.p, M.data(), md.data(), c->rcnt.p, rqc.data(), rqd.data(), 4))) return rc;
  std::vector<int64_t> mat((size_t)G * G), rc_ids(G), rd_ids(G + 1, 0);
  if ((rc = T.exchange_host(c, scnt.data(), G, mat.data()))) return rc;
  int64_t Rr = 0;
  for (int j = 0; j < G; ++j) {
    rc_ids[j] = j == r ? 0 : mat[(size_t)j * G + r];  // (this rank's own lists are not sent)
    rd_ids[j + 1] = rd_ids[j] + rc_ids[j];
    Rr += mat[(size_t)j * G + r];
  }
  if ((rc = ensure(c, c->rids, (size_t)std::max<int64_t>(rd_ids[G], 1) * 8)) ||
      (rc = ensure(c, c->mids, (size_t)std::max<int64_t>(Rr, 1) * 8)) ||
      (rc = ensure(c, c->mscratch, (size_t)std::max<int64_t>(Rr, 1) * 4)))
    return rc;
  // this rank's own partial lists stay where the tick wrote them (no self-copy)
  const int64_t self_cnt = scnt[r];
  scnt[r] = 0;
  rc_ids[r] = 0;
  if ((rc = T.alltoallv(c, c->outids.p, scnt.data(), sdis.data(), c->rids.p, rc_ids.data(), rd_ids.data(), 8)))
    return rc;
  // 3. merge on the device: per-source starts, query offsets, the union of the sorted runs
  (void)self_cnt;
  int64_t hconst[64] = {0};  // [0] = own queries, [1 + j] = where source j's runs are (device pointers)
  hconst[0] = Mr;
  if (G > 62) return fail(c, TJ_E_INVALID_ARG, "at most 62 ranks");
  for (int j = 0; j < G; ++j)
    hconst[1 + j] = j == r ? (int64_t)(uintptr_t)(P<int64_t>(c->outids) + bound[r])
                           : (int64_t)(uintptr_t)(P<int64_t>(c->rids) + rd_ids[j]);
  TJ_CUDA(cudaMemcpyAsync(c->sconst.p, hconst, sizeof(hconst), cudaMemcpyHostToDevice, c->st));
  int64_t* d_M = P<int64_t>(c->sconst);
  ScanPlan sp{std::min(1024, 4 * c->num_sms), P<int64_t>(c->partial), nullptr, c->scan_words};
  for (int j = 0; j < G; ++j)
    scan_launch(sp, ArrIn<int32_t>{P<int32_t>(c->rcnt) + (int64_t)j * Mr},
                ExclOut<int64_t>{P<int64_t>(c->sstart) + (int64_t)j * Mr}, d_M, c->d_hdr, (int64_t*)nullptr, c->st);
  scan_launch(sp, SumIn{P<int32_t>(c->rcnt), G, Mr}, ExclOut<int64_t>{P<int64_t>(c->moff)}, d_M, c->d_hdr,
              P<int64_t>(c->moff) + Mr, c->st);
  if (Mr)
    k_merge_partials<<<c->num_sms * 8, 256, 0, c->st>>>(G, Mr, P<int32_t>(c->rcnt), P<int64_t>(c->sstart),
                                                       reinterpret_cast<const int64_t* const*>(d_M + 1),
                                                       P<int64_t>(c->moff), P<int64_t>(c->mids));
  if ((rc = check_launch(c))) return rc;
  S.kernel_launches += (m ? 1 : 0) + 3 * (G + 1) + (Mr ? 1 : 0);
  S.n_objects = n;
  S.n_queries = Mr;
  S.results_total = Rr;
  return deliver(c, in->out_mem, out, Mr, Rr, true, c->moff, c->mids, c->mscratch, S);
}

}  // namespace
