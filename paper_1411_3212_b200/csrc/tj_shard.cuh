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

// Query routing (after the index build, which every rank builds identically):
// each own query goes to the owners of the leaves its window touches — the
// same clip, window and leaf enumeration the scatter does, with the owner of
// a leaf from the weight prefix k_shard_mark uses.  Its ORIGINAL rect is
// written into each destination's segment of the send buffers (segment j at
// j * mr, the place from a per-destination counter, kept in packpos for the
// merge); a query disjoint from the MBR goes nowhere (its list is empty).
__device__ __forceinline__ int leaf_owner(const Dev& d, uint32_t r, int G) {
  const DevHdr* h = d.h;
  const int64_t T = h->shard_total > 0 ? h->shard_total : 1;
  const int64_t mid = 2 * d.leaf_wpre[r] + (int64_t)d.leaf_nobj[r] + 1;
  const int64_t o = (mid * G) / (2 * T);
  return o < G ? (int)o : G - 1;
}
__global__ void __launch_bounds__(256) k_route(const Dev d, int64_t mr, int G, const double* __restrict__ qxa,
                                               const double* __restrict__ qya, const double* __restrict__ qxb,
                                               const double* __restrict__ qyb, double* sxa, double* sya,
                                               double* sxb, double* syb, int32_t* packpos,
                                               unsigned long long* dcnt, uint64_t* qmask) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const double xa = h->xa, ya = h->ya, xb = h->xb, yb = h->yb;
  const double sx = h->sx_deep, sy = h->sy_deep;
  const int wpos = h->wpos, hpos = h->hpos, ld = h->l_deep;
  const uint32_t side = h->side_deep;
  TJ_GRID_STRIDE(q, mr) {
    const double a = qxa[q], b = qya[q], c = qxb[q], e = qyb[q];
    double cxa = a < xa ? xa : a, cya = b < ya ? ya : b, cxb = c > xb ? xb : c, cyb = e > yb ? yb : e;
    uint64_t mask = 0;
    if (!(cxa > cxb || cya > cyb)) {
      int4 w;
      w.x = (int)cell_of(cxa, xa, sx, wpos, side);
      w.y = (int)cell_of(cxb, xa, sx, wpos, side);
      w.z = (int)cell_of(cya, ya, sy, hpos, side);
      w.w = (int)cell_of(cyb, ya, sy, hpos, side);
      if (is_small(w)) {
        uint32_t key[4], rank[4];
        const int ne = enum_small(w, ld, d.zmap, key, rank);
        for (int k = 0; k < ne; ++k) mask |= 1ull << leaf_owner(d, rank[k], G);
      } else {
        enum_window(w.x, w.y, w.z, w.w, ld, d.zmap,
                    [&](int, uint32_t, uint32_t rank) { mask |= 1ull << leaf_owner(d, rank, G); });
      }
    }
    qmask[q] = mask;
    for (uint64_t mm = mask; mm; mm &= mm - 1) {
      const int j = __ffsll((long long)mm) - 1;
      const int64_t pp = (int64_t)atomicAdd(&dcnt[j], 1ull);
      packpos[(int64_t)j * mr + q] = (int32_t)pp;
      const int64_t o = (int64_t)j * mr + pp;
      sxa[o] = a;
      sya[o] = b;
      sxb[o] = c;
      syb[o] = e;
    }
  }
}

// the returned partial lists of own query q, indexed like the merge wants them:
// cnt[j][q], start[j][q] (0 where q was not routed to j)
__global__ void __launch_bounds__(256) k_route_gather(int64_t mr, int G, const uint64_t* __restrict__ qmask,
                                                      const int32_t* __restrict__ packpos,
                                                      const int32_t* __restrict__ rcnt,
                                                      const int64_t* __restrict__ rstart, int32_t* gcnt,
                                                      int64_t* gstart) {
  TJ_GRID_STRIDE(q, mr) {
    const uint64_t mask = qmask[q];
    for (int j = 0; j < G; ++j) {
      const int64_t o = (int64_t)j * mr + q;
      if ((mask >> j) & 1ull) {
        const int64_t p = (int64_t)j * mr + packpos[o];
        gcnt[o] = rcnt[p];
        gstart[o] = rstart[p];
      } else {
        gcnt[o] = 0;
        gstart[o] = 0;
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

// the sharded tick: gather the objects -> index build -> route the queries to the owners of
// their leaves -> the rank's leaf range -> partial lists back to the home ranks -> device merge
int sharded_tick(tj_ctx* c, const tj_tick_in* in, tj_tick_out* out, tj_stats& S) {
  Transport& T = *c->comm;
  const int G = T.nranks, r = T.rank;
  int rc;
  if (G > 31) return fail(c, TJ_E_INVALID_ARG, "at most 31 ranks");
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
  // 1. every rank's objects gathered into the full set (the index is built on all of them)
  if ((rc = ensure(c, c->ids, n * 8)) || (rc = ensure(c, c->xs, n * 8)) || (rc = ensure(c, c->ys, n * 8))) return rc;
  DBuf* full[3] = {&c->ids, &c->xs, &c->ys};
  const void* osrc[3] = {in->obj_id, in->obj_x, in->obj_y};
  for (int a = 0; a < 3; ++a) {
    char* slot = static_cast<char*>(full[a]->p) + nd[r] * 8;
    const void* send = osrc[a];
    if (in->mem == TJ_MEM_HOST) {  // this rank's slice lands in its place of the full array first
      if (N[r]) TJ_CUDA(cudaMemcpyAsync(slot, osrc[a], N[r] * 8, cudaMemcpyHostToDevice, c->st));
      send = slot;
    }
    if ((rc = T.allgatherv(c, send, full[a]->p, N.data(), nd.data(), 8))) return rc;
  }
  // this rank's own queries on the device
  const double* oq[4] = {in->q_xa, in->q_ya, in->q_xb, in->q_yb};
  if (in->mem == TJ_MEM_HOST)
    for (int a = 0; a < 4; ++a) {
      if ((rc = ensure(c, c->oq[a], (size_t)Mr * 8 + 8))) return rc;
      if (Mr) TJ_CUDA(cudaMemcpyAsync(c->oq[a].p, oq[a], Mr * 8, cudaMemcpyHostToDevice, c->st));
      oq[a] = P<double>(c->oq[a]);
    }
  if (n == 0 || G == 1) {  // nothing to route: every list is complete on this rank (or empty)
    c->shard_rank = 0;
    c->shard_n = 1;
    int64_t R = 0;
    if ((rc = compute_tick(c, n, Mr, P<int64_t>(c->ids), P<double>(c->xs), P<double>(c->ys), oq[0], oq[1], oq[2],
                           oq[3], S, R)))
      return rc;
    S.n_objects = n;
    S.n_queries = Mr;
    return deliver(c, in->out_mem, out, Mr, R, n > 0, c->outoff, c->outids, c->scratch, S);
  }
  c->shard_rank = r;
  c->shard_n = G;
  // 2. the queries go to the owners of the leaves their windows touch, right after the index build
  //    (a rank receives at most every query of the tick once)
  for (int a = 0; a < 4; ++a)
    if ((rc = ensure(c, c->rq[a], (size_t)m * 8 + 8)) || (rc = ensure(c, c->sq[a], (size_t)G * Mr * 8 + 8)))
      return rc;
  if ((rc = ensure(c, c->packpos, (size_t)G * Mr * 4 + 4)) || (rc = ensure(c, c->qmask, (size_t)Mr * 8 + 8)) ||
      (rc = ensure(c, c->dcnt, (size_t)G * 8)) || (rc = ensure(c, c->sconst, 64 * 8)))
    return rc;
  std::vector<int64_t> dc(G), sdq(G), rcq(G), rdq(G + 1, 0), mat((size_t)G * G);
  for (int j = 0; j < G; ++j) sdq[j] = (int64_t)j * Mr;
  int64_t m_recv = 0;
  bool routed = false;
  c->after_build = [&]() -> int {
    // Collectives run once per tick on every rank: a capacity replay of one rank's tick (its own
    // queries' sizes) reuses the queries it received, and an index build that aborted (identical
    // on every rank: the index is) routes nothing — the replay that builds the index does.
    int32_t ab = 0;
    TJ_CUDA(cudaMemcpyAsync(&ab, &c->d_hdr->abort, sizeof(int32_t), cudaMemcpyDeviceToHost, c->st));
    TJ_CUDA(cudaStreamSynchronize(c->st));
    if (ab) return TJ_OK;
    if (routed) {
      TJ_CUDA(cudaMemcpyAsync(&c->d_hdr->m, &m_recv, sizeof(int64_t), cudaMemcpyHostToDevice, c->st));
      TJ_CUDA(cudaStreamSynchronize(c->st));
      return TJ_OK;
    }
    routed = true;
    TJ_CUDA(cudaMemsetAsync(c->dcnt.p, 0, G * 8, c->st));
    if (Mr)
      k_route<<<grid_for(c, Mr), 256, 0, c->st>>>(c->dv, Mr, G, oq[0], oq[1], oq[2], oq[3], P<double>(c->sq[0]),
                                                 P<double>(c->sq[1]), P<double>(c->sq[2]), P<double>(c->sq[3]),
                                                 P<int32_t>(c->packpos), P<unsigned long long>(c->dcnt),
                                                 P<uint64_t>(c->qmask));
    TJ_CUDA(cudaMemcpyAsync(dc.data(), c->dcnt.p, G * 8, cudaMemcpyDeviceToHost, c->st));
    TJ_CUDA(cudaStreamSynchronize(c->st));
    int rc2;
    if ((rc2 = T.exchange_host(c, dc.data(), G, mat.data()))) return rc2;
    rdq[0] = 0;
    for (int j = 0; j < G; ++j) {
      rcq[j] = mat[(size_t)j * G + r];
      rdq[j + 1] = rdq[j] + rcq[j];
    }
    m_recv = rdq[G];
    for (int a = 0; a < 4; ++a)
      if ((rc2 = T.alltoallv(c, c->sq[a].p, dc.data(), sdq.data(), c->rq[a].p, rcq.data(), rdq.data(), 8)))
        return rc2;
    // the rest of the tick runs on the received queries
    TJ_CUDA(cudaMemcpyAsync(&c->d_hdr->m, &m_recv, sizeof(int64_t), cudaMemcpyHostToDevice, c->st));
    TJ_CUDA(cudaStreamSynchronize(c->st));
    return TJ_OK;
  };
  int64_t R = 0;
  rc = compute_tick(c, n, m, P<int64_t>(c->ids), P<double>(c->xs), P<double>(c->ys), P<double>(c->rq[0]),
                    P<double>(c->rq[1]), P<double>(c->rq[2]), P<double>(c->rq[3]), S, R);
  c->after_build = nullptr;
  if (rc) return rc;
  // 3. each received query's partial list back to its home rank: counts, then the id runs
  if ((rc = ensure(c, c->pcnt, (size_t)std::max<int64_t>(m_recv, 1) * 4)) ||
      (rc = ensure(c, c->rcnt, (size_t)G * Mr * 4 + 4)) || (rc = ensure(c, c->sstart, (size_t)G * Mr * 8 + 8)) ||
      (rc = ensure(c, c->gcnt, (size_t)G * Mr * 4 + 4)) || (rc = ensure(c, c->gstart, (size_t)G * Mr * 8 + 8)) ||
      (rc = ensure(c, c->moff, (size_t)(Mr + 1) * 8)))
    return rc;
  if (m_recv)
    k_partial_counts<<<c->num_sms * 4, 256, 0, c->st>>>(P<int64_t>(c->outoff), P<int32_t>(c->pcnt), m_recv);
  std::vector<int64_t> bound(G + 1), sid(G), sdid(G), rid(G), rdid(G + 1, 0);
  for (int j = 0; j <= G; ++j)
    TJ_CUDA(cudaMemcpyAsync(&bound[j], P<int64_t>(c->outoff) + rdq[j], 8, cudaMemcpyDeviceToHost, c->st));
  TJ_CUDA(cudaStreamSynchronize(c->st));
  for (int j = 0; j < G; ++j) {
    sid[j] = bound[j + 1] - bound[j];
    sdid[j] = bound[j];
  }
  if ((rc = T.alltoallv(c, c->pcnt.p, rcq.data(), rdq.data(), c->rcnt.p, dc.data(), sdq.data(), 4))) return rc;
  if ((rc = T.exchange_host(c, sid.data(), G, mat.data()))) return rc;
  for (int j = 0; j < G; ++j) {
    rid[j] = mat[(size_t)j * G + r];
    rdid[j + 1] = rdid[j] + rid[j];
  }
  const int64_t Rr = rdid[G];
  if ((rc = ensure(c, c->rids, (size_t)std::max<int64_t>(Rr, 1) * 8)) ||
      (rc = ensure(c, c->mids, (size_t)std::max<int64_t>(Rr, 1) * 8)) ||
      (rc = ensure(c, c->mscratch, (size_t)std::max<int64_t>(Rr, 1) * 4)))
    return rc;
  if ((rc = T.alltoallv(c, c->outids.p, sid.data(), sdid.data(), c->rids.p, rid.data(), rdid.data(), 8))) return rc;
  // 4. merge on the device: run starts per destination, own queries' offsets, the union
  int64_t hconst[64] = {0};  // [0] own queries; [1 + j] source j's runs (device pointer); [32 + j] dc[j]
  hconst[0] = Mr;
  for (int j = 0; j < G; ++j) {
    hconst[1 + j] = (int64_t)(uintptr_t)(P<int64_t>(c->rids) + rdid[j]);
    hconst[32 + j] = dc[j];
  }
  TJ_CUDA(cudaMemcpyAsync(c->sconst.p, hconst, sizeof(hconst), cudaMemcpyHostToDevice, c->st));
  int64_t* dK = P<int64_t>(c->sconst);
  ScanPlan sp{std::min(1024, 4 * c->num_sms), P<int64_t>(c->partial), nullptr, c->scan_words};
  for (int j = 0; j < G; ++j)
    scan_launch(sp, ArrIn<int32_t>{P<int32_t>(c->rcnt) + (int64_t)j * Mr},
                ExclOut<int64_t>{P<int64_t>(c->sstart) + (int64_t)j * Mr}, dK + 32 + j, c->d_hdr, (int64_t*)nullptr,
                c->st);
  if (Mr)
    k_route_gather<<<grid_for(c, Mr), 256, 0, c->st>>>(Mr, G, P<uint64_t>(c->qmask), P<int32_t>(c->packpos),
                                                       P<int32_t>(c->rcnt), P<int64_t>(c->sstart),
                                                       P<int32_t>(c->gcnt), P<int64_t>(c->gstart));
  scan_launch(sp, SumIn{P<int32_t>(c->gcnt), G, Mr}, ExclOut<int64_t>{P<int64_t>(c->moff)}, dK, c->d_hdr,
              P<int64_t>(c->moff) + Mr, c->st);
  if (Mr)
    k_merge_partials<<<c->num_sms * 8, 256, 0, c->st>>>(G, Mr, P<int32_t>(c->gcnt), P<int64_t>(c->gstart),
                                                       reinterpret_cast<const int64_t* const*>(dK + 1),
                                                       P<int64_t>(c->moff), P<int64_t>(c->mids));
  if ((rc = check_launch(c))) return rc;
  S.kernel_launches += 2 + (m_recv ? 1 : 0) + 3 * (G + 1) + (Mr ? 2 : 0);
  S.n_objects = n;
  S.n_queries = Mr;
  S.results_total = Rr;
  return deliver(c, in->out_mem, out, Mr, Rr, true, c->moff, c->mids, c->mscratch, S);
}

}  // namespace
