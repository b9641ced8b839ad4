// C ABI of the B200 QUAD tick pipeline (include/tickjoin_b200.h).
//
// Host side of the native library: context + device arena management, the
// per-tick launch sequence (one stream, no host synchronisation between
// stages; sizes live in DevHdr), capacity-overflow replay, result delivery,
// and the reference-order introspection used by the parity tests.
#include "tickjoin_b200.h"
#include "tj_kernels.cuh"

#ifndef TJ_ZMAP_GENERIC
#define TJ_ZMAP_GENERIC 0  // 1: the zmap through the generic scan (ZFlagIn / ZOut) instead of k_zmap_count / k_zmap_rank
#endif

#include <algorithm>
#include <cstdio>
#include <functional>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

using namespace tj;

namespace {

std::string g_last_error;

struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

}  // namespace

struct Transport;  // multi-GPU exchange (tj_shard.cuh)

// One instantiated CUDA graph of the tick's launch sequence.  Every size
// after the index build lives on the device, so a graph is valid for any
// tick with the same host-side launch shape: input/arena pointers (all in
// `Dev`), n, m and the radix pass count.
struct TickGraph {
  Dev dv;
  int64_t n = 0, m = 0;
  int obj_passes = 0, shard_n = 0, launches[8] = {};
  bool reuse = false;
  bool key_req = false;
  const void* scan_state[2] = {nullptr, nullptr};  // host-side buffers baked into the graph
  int64_t scan_words = 0;
  cudaGraphExec_t exec[8] = {};
};

struct tj_ctx {
  tj_config cfg{};
  int device = 0;
  int num_sms = 148;
  int scatter_per_sm = 8;
  bool fused_pyr = true;  // TJ_FUSED_PYR=0: one launch per pyramid level
  int ug_sf = 0;  // method "ug": cells per side (cfg.l_max then holds ceil(log2) of it)
  int join_blocks = 4;  // resident k_join CTAs per SM (occupancy API)
  int decode_blocks = TJ_DQ_MINB;  // resident k_decode_query CTAs per SM (occupancy API)
  cudaStream_t st = nullptr;
  cudaStream_t side = nullptr;             // object sort, concurrent with the query scatter
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev[10] = {};
  DevHdr* d_hdr = nullptr;
  DevHdr* h_hdr = nullptr;  // pinned
  int64_t* d_consts = nullptr;
  std::string err;
  // inputs
  DBuf ids, xs, ys, qxa, qya, qxb, qyb;
  // objects
  DBuf code, okey0, okey1, oval0, oval1, sx, sy, tx, ty;
  DBuf loff, presence, prespre, order;  // keyed lists (ids that are not the rows)
  DBuf crow;                            // sharded ticks: compacted rows of own-leaf objects
  // index
  DBuf linfo, pyr, clev, zmap, lcode, lnobj, lobase, lnisq, lncov, lsbase, lwoff, lubase;
  // queries
  DBuf qpos, qwin, nsub, qsbase, biglist, leafcnt;
  // subqueries
  DBuf sqle, sqcount, ecount, erect, slotoff, leafcur, unitleaf;
  // join / outputs
  DBuf bitmap, outids, outoff, scratch, outoff32;
  // scan / radix scratch
  DBuf partial, partial2, rhist, roffs, sstate, sstate2;
  int64_t scan_words = 0;  // look-back scan state words (tile counter + tiles)
  bool lb_scan = false;       // single-pass look-back scan (measured slower here than reduce-then-scan)
  bool serial_sort = false;   // TJ_SERIAL_SORT=1: object sort on the main stream (for measuring K1 alone)
  bool check_tiling = false;  // TJ_CHECK_TILING=1: the build_zmap tiling check on the device (TilingGap)
  bool sort_xy = false;       // TJ_SORT_XY=1: coordinates carried through the radix passes (no gathers)
  // adaptive rebuild: the last built index (header fields + the buffers it lives in)
  bool have_index = false;
  bool reuse = false;  // this tick reuses it
  int32_t reuse_not_mono = 0, reuse_not_id = 0;  // id-order flags of this tick, from the reuse check pass
  unsigned long long reuse_id_kmin = 0, reuse_id_kmax = 0;
  // keyed lists (ids that are not the rows): the id-key kernels join the launch sequence when the
  // previous tick's ids qualified — a wrong guess costs speed, never results (k_key_decide checks on
  // the device; TJ_KEYED=0 turns them off)
  bool key_auto = true;
  bool key_req = false;
  bool dup_ids_seen = false;
  DevHdr idx{};
  // (the kept index lives in zmap, sized by l_max only, and in the leaf codes, which keep their
  // contents when n grows the leaf capacity: see prepare_static)
  // pinned host outputs
  void* h_off = nullptr;
  size_t h_off_bytes = 0;
  void* h_ids = nullptr;
  size_t h_ids_bytes = 0;
  // capacities of the dynamically sized arenas
  int64_t cap_S = 0, cap_W = 0, cap_R = 0, cap_L = 0, cap_U = 0;
  int64_t last_L = 0;
  // last tick, for introspection
  bool have = false;
  int64_t n = 0, m = 0;
  DevHdr last{};
  Dev dv{};
  int obj_passes = 0;
  int shard_rank = 0, shard_n = 1;
  bool use_graphs = true;
  std::vector<TickGraph> graphs;
  DBuf lactive, lwpre;
  // multi-GPU data plane (tj_comm_init / tj_comm_init_local, tj_tick_sharded)
  Transport* comm = nullptr;
  DBuf pcnt, rcnt, sstart, moff, sconst, rids, mids, mscratch;
  // query routing: own queries, their destination masks / places, send and receive rects
  DBuf oq[4], qmask, packpos, dcnt, sq[4], rq[4], gcnt, gstart;
  std::function<int()> after_build;  // run between the index build and the rest of a tick
};

namespace {

int fail(tj_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  g_last_error = msg;
  return code;
}

#define TJ_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(c, e_ == cudaErrorMemoryAllocation ? TJ_E_OOM : TJ_E_CUDA,            \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                  \
  } while (0)

// grow-only device buffer; `keep`: the old contents survive a reallocation
int ensure(tj_ctx* c, DBuf& b, size_t bytes, bool keep = false) {
  if (bytes == 0) bytes = 16;
  if (b.bytes >= bytes) return TJ_OK;
  void* np_ = nullptr;
  cudaError_t e = cudaMalloc(&np_, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(c, TJ_E_OOM, std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
  }
  if (b.p) {
    cudaStreamSynchronize(c->st);
    if (c->side) cudaStreamSynchronize(c->side);
    if (keep) cudaMemcpy(np_, b.p, b.bytes, cudaMemcpyDeviceToDevice);
    cudaFree(b.p);
  }
  b.p = np_;
  b.bytes = bytes;
  return TJ_OK;
}

int ensure_host(tj_ctx* c, void*& p, size_t& have, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (have >= bytes) return TJ_OK;
  if (p) cudaFreeHost(p);
  p = nullptr;
  have = 0;
  cudaError_t e = cudaMallocHost(&p, bytes);
  if (e != cudaSuccess) return fail(c, TJ_E_OOM, std::string("cudaMallocHost: ") + cudaGetErrorString(e));
  have = bytes;
  return TJ_OK;
}

template <typename T>
T* P(const DBuf& b) { return reinterpret_cast<T*>(b.p); }

int bits_for(int64_t v) {  // bits needed to represent values in [0, v]
  int b = 0;
  while (b < 63 && (v >> b) != 0) ++b;
  return b;
}

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline int grid_for(tj_ctx* c, int64_t items, int per_sm = 8) {
  int64_t g = ceil_div(items, 256);
  int64_t cap = (int64_t)c->num_sms * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// Allocate everything whose size depends only on n, m and the config.
int prepare_static(tj_ctx* c, int64_t n, int64_t m) {
  const int lmax = c->cfg.l_max;
  const int F = std::min(lmax, kDenseTop);
  const int64_t th = c->cfg.th_quad;
  int rc;
#define ENS(buf, bytes) \
  if ((rc = ensure(c, c->buf, (size_t)(bytes))) != TJ_OK) return rc
  // leaves: <= 4 + 3*(#split nodes); a level holds <= n/(th+1) split nodes
  const int64_t Zmax = int64_t(1) << (2 * lmax);
  int64_t lcap = 4 + 3 * (int64_t)(lmax > 1 ? lmax - 1 : 0) * (n / (th + 1) + 1);
  c->cap_L = c->ug_sf ? Zmax : std::min(lcap, Zmax);  // a uniform grid: every cell is a leaf
  ENS(code, n * 4);
  ENS(okey0, n * 4);
  ENS(okey1, n * 4);
  ENS(oval0, n * 4);
  ENS(oval1, n * 4);
  ENS(sx, n * 8 + 16);  // + slack: the join's bulk copies round a tile up to 16 bytes
  ENS(sy, n * 8 + 16);
  ENS(tx, n * 8);
  ENS(ty, n * 8);
  if (c->shard_n > 1) ENS(crow, n * 4);
  if (c->key_req) {
    ENS(loff, n * 4);
    ENS(presence, (int64_t(1) << (kKeyBits - 5)) * 4 + 64);
    ENS(prespre, (int64_t(1) << (kKeyBits - 5)) * 4 + 64);
    ENS(order, n * 4);
  }
  ENS(pyr, pyr_off(F + 1) * 4);
  ENS(clev, Zmax);
  ENS(zmap, Zmax * 4);
  // the adaptive policy's kept index: leaf codes survive growth (zmap is sized by l_max alone)
  if ((rc = ensure(c, c->lcode, (size_t)(c->cap_L * 4), true)) != TJ_OK) return rc;
  ENS(lnobj, c->cap_L * 4);
  ENS(lobase, c->cap_L * 4);
  ENS(lnisq, c->cap_L * 4);
  ENS(lncov, c->cap_L * 4);
  ENS(lsbase, c->cap_L * 4);
  ENS(lwoff, c->cap_L * 8);
  ENS(linfo, c->cap_L * 16);
  ENS(lubase, c->cap_L * 8);
  ENS(leafcur, c->cap_L * 2 * 4);
  ENS(lactive, c->cap_L);
  ENS(lwpre, c->cap_L * 8);
  ENS(leafcnt, c->cap_L * sizeof(int4));
  ENS(nsub, m * 4);
  ENS(qsbase, m * 4);
  ENS(qpos, m * sizeof(int4));
  ENS(qwin, m * sizeof(int4));
  ENS(biglist, m * 4);
  ENS(outoff, (m + 1) * 8);
  ENS(partial, 1024 * 8);
  ENS(partial2, 1024 * 8);
  const int Gr = 2 * c->num_sms;
  ENS(rhist, (int64_t)kRadixDigits * Gr * 4);
  ENS(roffs, (int64_t)kRadixDigits * Gr * 8);
  if (c->cap_S == 0) c->cap_S = 4 * m + 256;
  if (c->cap_W == 0) c->cap_W = 8 * c->cap_S + 4096;
  if (c->cap_R == 0) c->cap_R = 16 * m + 4096;
  if (c->cap_U == 0) c->cap_U = c->cap_S + c->cap_L;
#undef ENS
  return TJ_OK;
}

int prepare_dynamic(tj_ctx* c) {
  int rc;
#define ENS(buf, bytes) \
  if ((rc = ensure(c, c->buf, (size_t)(bytes))) != TJ_OK) return rc
  ENS(sqle, c->cap_S * 8);
  ENS(sqcount, c->cap_S * 4);
  ENS(erect, c->cap_S * sizeof(Rect4));
  ENS(ecount, c->cap_S * 4);
  ENS(slotoff, (c->cap_S + 1) * 8);
  ENS(bitmap, c->cap_W * 4);
  {  // look-back scan state: enough tiles for the longest scanned array
    const int64_t Zmax = int64_t(1) << (2 * c->cfg.l_max);
    const int64_t longest = std::max({c->cap_S + 1, c->m + 1, c->n + 1, Zmax, c->cap_L,
                                      (int64_t)kRadixDigits * 2 * c->num_sms});
    c->scan_words = (longest + kScanTile - 1) / kScanTile + 2;
    ENS(sstate, c->scan_words * 8);
    ENS(sstate2, c->scan_words * 8);
  }
  ENS(unitleaf, c->cap_U * 4);
  ENS(scratch, c->cap_R * 8);
  ENS(outids, c->cap_R * 8);
#undef ENS
  return TJ_OK;
}

void fill_dev(tj_ctx* c, const int64_t* ids, const double* xs, const double* ys, const double* qxa,
              const double* qya, const double* qxb, const double* qyb) {
  Dev& d = c->dv;
  const int lmax = c->cfg.l_max;
  const int F = std::min(lmax, kDenseTop);
  d.h = c->d_hdr;
  d.ids = ids;
  d.xs = xs;
  d.ys = ys;
  d.qxa = qxa;
  d.qya = qya;
  d.qxb = qxb;
  d.qyb = qyb;
  d.code = P<uint32_t>(c->code);
  d.okey[0] = P<uint32_t>(c->okey0);
  d.okey[1] = P<uint32_t>(c->okey1);
  d.oval[0] = P<int32_t>(c->oval0);
  d.oval[1] = P<int32_t>(c->oval1);
  d.sx = P<double>(c->sx);
  d.sy = P<double>(c->sy);
  d.pyr = P<uint32_t>(c->pyr);
  d.clev = P<uint8_t>(c->clev);
  d.zmap = P<uint32_t>(c->zmap);
  d.leaf_code = P<uint32_t>(c->lcode);
  d.leaf_nobj = P<int32_t>(c->lnobj);
  d.leaf_obase = P<int32_t>(c->lobase);
  d.leaf_nisq = P<int32_t>(c->lnisq);
  d.leaf_ncov = P<int32_t>(c->lncov);
  d.leaf_sbase = P<int32_t>(c->lsbase);
  d.leaf_woff = P<int64_t>(c->lwoff);
  d.leaf_ubase = P<int64_t>(c->lubase);
  d.nsub = P<int32_t>(c->nsub);
  d.qsbase = P<int32_t>(c->qsbase);
  d.qpos = P<int4>(c->qpos);
  d.qwin = P<int4>(c->qwin);
  d.sq_le = P<int2>(c->sqle);
  d.sq_count = P<int32_t>(c->sqcount);
  d.erect = P<Rect4>(c->erect);
  d.ecount = P<int32_t>(c->ecount);
  d.linfo = P<int4>(c->linfo);
  d.slot_off = P<int64_t>(c->slotoff);
  d.bitmap = P<uint32_t>(c->bitmap);
  d.out_ids = P<int64_t>(c->outids);
  d.out_off = P<int64_t>(c->outoff);
  d.sidx = d.oval[c->obj_passes & 1];
  d.loff = P<uint32_t>(c->loff);
  d.presence = P<uint32_t>(c->presence);
  d.pres_pre = P<int32_t>(c->prespre);
  d.order = P<int32_t>(c->order);
  d.crow = P<int32_t>(c->crow);
  d.leaf_cur = P<int32_t>(c->leafcur);
  d.leaf_cnt = P<int4>(c->leafcnt);
  d.unit_leaf = P<int32_t>(c->unitleaf);
  d.big_list = P<int32_t>(c->biglist);
  d.leaf_active = c->shard_n > 1 ? P<uint8_t>(c->lactive) : nullptr;
  d.leaf_wpre = P<int64_t>(c->lwpre);
  d.scratch = P<int64_t>(c->scratch);
}

// one pass of the stable LSD radix sort: digit histograms, their scan, the
// rank-and-scatter (with the (x, y) payload when XY)
template <bool XY, typename KeySrc>
void radix_pass(tj_ctx* c, cudaStream_t st, const ScanPlan& sp, KeySrc keys, const int32_t* vin, uint32_t* kout,
                int32_t* vout, const double* xin, const double* yin, double* xout, double* yout,
                const int64_t* n_ptr, int shift, int gate = 0) {
  const int Gr = 2 * c->num_sms;
  k_radix_upsweep<<<Gr, kRadixThreads, 0, st>>>(keys, n_ptr, c->d_hdr, shift, P<uint32_t>(c->rhist));
  scan_launch(sp, ArrIn<uint32_t>{P<uint32_t>(c->rhist)}, ExclOut<int64_t>{P<int64_t>(c->roffs)}, c->d_consts,
              c->d_hdr, (int64_t*)nullptr, st);
  k_radix_downsweep<KeySrc, XY><<<Gr, kRadixThreads, radix_smem_bytes<XY>(), st>>>(
      keys, vin, kout, vout, xin, yin, xout, yout, n_ptr, c->d_hdr, shift, P<int64_t>(c->roffs), gate);
}

// Objects into leaf order: stable LSD radix sort of (leaf rank, input row)
// over `passes` 8-bit digits (keys from k_obj_keys, rows implicit in the
// first pass; the last pass writes no keys), then the coordinates gathered
// into leaf order.  TJ_SORT_XY=1: the coordinates ride along through every
// pass instead (sequential reads and staged writes; measured slower here).
int sort_objects(tj_ctx* c, cudaStream_t st, const ScanPlan& sp) {
  Dev& d = c->dv;
  DevHdr* h = c->d_hdr;
  const int P_ = c->obj_passes;
  const int Gn = grid_for(c, c->n);
  int launched = 0;
  if (c->key_req) {  // keyed lists: eligibility, duplicate ids, id ranks (idle kernels when the device declines)
    k_key_decide<<<1, 1, 0, st>>>(h);
    k_key_zero<<<c->num_sms * 8, 256, 0, st>>>(d);
    k_key_presence<<<Gn, 256, 0, st>>>(d);
    scan_launch(sp, PopIn{d.presence}, ExclOut<int32_t>{d.pres_pre}, &h->pres_words, h, &h->pres_total, st);
    k_key_close<<<1, 1, 0, st>>>(h);
    k_key_order<<<Gn, 256, 0, st>>>(d);
    launched += 8;
  }
  const bool compact = c->shard_n > 1 && !c->sort_xy;
  if (compact) {  // sharded: own-leaf objects only, compacted in order (keys + rows)
    scan_launch(sp, OwnObjIn{d}, OwnObjOut{d}, &h->n, h, &h->n_sort, st);
    launched += 3;
  } else {
    k_obj_keys<<<Gn, 256, 0, st>>>(d);
    launched += 1;
  }
  double* bx[2] = {P<double>(c->sx), P<double>(c->tx)};
  double* by[2] = {P<double>(c->sy), P<double>(c->ty)};
  const double *xin = d.xs, *yin = d.ys;
  for (int p = 0; p < P_; ++p) {
    const int src = p & 1, dst = src ^ 1;
    const bool last = p == P_ - 1;
    const int ob = (P_ - 1 - p) & 1;  // the last pass lands in (sx, sy)
    uint32_t* kout = last ? nullptr : d.okey[dst];
    // first pass: the input rows, or (keyed lists, ids not increasing) the rows in id order
    const int32_t* vin = p == 0 ? (compact ? (const int32_t*)d.crow : (c->key_req ? (const int32_t*)d.order : nullptr))
                                : d.oval[src];
    const int gate = p == 0 && c->key_req && !compact ? 1 : 0;
    if (c->sort_xy) {
      radix_pass<true>(c, st, sp, ArrKey{d.okey[src]}, vin, kout, d.oval[dst], xin, yin, bx[ob], by[ob], &h->n,
                       kRadixBits * p, gate);
      xin = bx[ob];
      yin = by[ob];
    } else {
      radix_pass<false>(c, st, sp, ArrKey{d.okey[src]}, vin, kout, d.oval[dst], nullptr, nullptr, nullptr, nullptr,
                        &h->n_sort, kRadixBits * p, gate);
    }
  }
  if (c->key_req) {  // keyed lists: every leaf position's id offset
    k_key_loff<<<Gn, 256, 0, st>>>(d);
    launched += 1;
  }
  int gathers = 0;
  if (!c->sort_xy) {  // (x and y gathered by one kernel measured 8% slower on this branch)
    k_gather<double><<<Gn, 256, 0, st>>>(d, d.xs, d.sx);
    k_gather<double><<<Gn, 256, 0, st>>>(d, d.ys, d.sy);
    gathers = 2;
  }
  // 5 launches per radix pass (upsweep + 3-kernel scan + downsweep)
  return launched + 5 * P_ + gathers;
}

// The per-tick launch sequence, in stages (index build, query scatter, join
// preparation, join, decode, merge); no host synchronisation inside.  Stage
// boundaries carry the timing events.  Returns the kernels launched.
constexpr int kStages = 7;
constexpr int kSortStage = 7;  // the object sort: its own graph, on the side stream

int launch_stage(tj_ctx* c, int stage) {
  cudaStream_t st = c->st;
  Dev& d = c->dv;
  DevHdr* h = c->d_hdr;
  const int lmax = c->cfg.l_max;
  const int F = std::min(lmax, kDenseTop);
  const int64_t n = c->n, m = c->m;
  const int Gn = grid_for(c, n), Gm = grid_for(c, m);
  const int Gs = grid_for(c, m, c->scatter_per_sm);  // the query scatter shares the GPU with the object sort
  const int Gbig = c->num_sms * 8;
  ScanPlan sp{std::min(1024, 4 * c->num_sms), P<int64_t>(c->partial),
              c->lb_scan ? P<unsigned long long>(c->sstate) : nullptr, c->scan_words};
  switch (stage) {
    case 0:  // ---- K0 / K1: index build ------------------------------------
      cudaMemsetAsync(d.leaf_cur, 0, c->cap_L * 2 * 4, st);
      cudaMemsetAsync(d.leaf_cnt, 0, c->cap_L * sizeof(int4), st);
      if (c->reuse) {  // adaptive: the old tree, leaf counts recounted by the check pass
        if (c->shard_n > 1) {  // own leaves first: their blocks are the only ones sorted
          scan_launch(sp, LeafWeightIn{d.leaf_nobj}, PrefOut{d.leaf_wpre}, &h->L, h, &h->shard_total, st);
          k_shard_mark<<<Gbig, 256, 0, st>>>(d);
          scan_launch(sp, OwnNobjIn{d.leaf_nobj, d.leaf_active}, ExclOut<int32_t>{d.leaf_obase}, &h->L, h,
                      (int64_t*)nullptr, st);
        } else {
          scan_launch(sp, ArrIn<int32_t>{d.leaf_nobj}, ExclOut<int32_t>{d.leaf_obase}, &h->L, h, (int64_t*)nullptr,
                      st);
        }
        return 3 + (c->shard_n > 1 ? 4 : 0);
      }
      cudaMemsetAsync(d.pyr + pyr_off(F), 0, (pyr_off(F + 1) - pyr_off(F)) * 4, st);  // the histogram level
      k_mbr<<<Gn, 256, 0, st>>>(d);
      k_finalize_mbr<<<1, 1, 0, st>>>(h);
      k_codes<<<Gn, 256, 0, st>>>(d);
      if (c->ug_sf) {  // uniform grid: every cell of the l_max grid is a leaf (no tree to build)
        k_finalize_index<<<1, 1, 0, st>>>(h);
        cudaMemsetAsync(d.clev, lmax, int64_t(1) << (2 * lmax), st);
      } else {
        if (c->fused_pyr) {  // levels F-1 .. 0 in spans of kPyrSpan (k_pyr_fused)
          for (int hi = F; hi > 0; hi -= kPyrSpan) {
            const int lo = std::max(0, hi - kPyrSpan);
            k_pyr_fused<<<(int)(int64_t(1) << (2 * lo)), 256, 0, st>>>(d, lo, hi);
          }
        } else {
          for (int l = F - 1; l >= 0; --l) k_pyr_level<<<grid_for(c, int64_t(1) << (2 * l)), 256, 0, st>>>(d, l);
        }
        k_finalize_index<<<1, 1, 0, st>>>(h);
#if TJ_ZMAP_GENERIC
        k_cell_level<<<Gbig, 256, 0, st>>>(d);
#endif
      }
#if TJ_ZMAP_GENERIC
      scan_launch(sp, ZFlagIn{d.clev, h}, ZOut{d}, &h->Z, h, &h->L, st);
#else
      if (c->ug_sf) k_zmap_count<false><<<sp.G, 256, 0, st>>>(d, sp.partial);
      else k_zmap_count<true><<<sp.G, 256, 0, st>>>(d, sp.partial);  // leaf levels computed here (k_cell_level fused)
      k_scan_partials<<<1, 1024, 0, st>>>(sp.partial, sp.G, &h->L, h);
      k_zmap_rank<<<sp.G, 256, 0, st>>>(d, sp.partial);
#endif
      k_check_caps<<<1, 1, 0, st>>>(h, 0, kRadixBits * c->obj_passes, 32);
      if (c->check_tiling) k_check_tiling<<<Gbig, 256, 0, st>>>(d);
      if (c->shard_n > 1) {  // leaf-range sharding: this rank's contiguous Morton range, before the scatter,
                             // and block bases over its own leaves (only their objects are sorted)
        scan_launch(sp, LeafWeightIn{d.leaf_nobj}, PrefOut{d.leaf_wpre}, &h->L, h, &h->shard_total, st);
        k_shard_mark<<<Gbig, 256, 0, st>>>(d);
        scan_launch(sp, OwnNobjIn{d.leaf_nobj, d.leaf_active}, ExclOut<int32_t>{d.leaf_obase}, &h->L, h,
                    (int64_t*)nullptr, st);
      } else {
        scan_launch(sp, ArrIn<int32_t>{d.leaf_nobj}, ExclOut<int32_t>{d.leaf_obase}, &h->L, h, (int64_t*)nullptr,
                    st);
      }
      // 3 launches per scan
      return (c->ug_sf ? 11 : 12 - (TJ_ZMAP_GENERIC ? 0 : 1) + (c->fused_pyr ? (F + kPyrSpan - 1) / kPyrSpan : F)) + (c->shard_n > 1 ? 4 : 0) +
             (c->check_tiling ? 1 : 0);
    case kSortStage: {  // ---- K1's last part: objects into leaf order (side stream) ----
      cudaStream_t ss = c->serial_sort ? c->st : c->side;
      ScanPlan sp2{std::min(1024, 4 * c->num_sms), P<int64_t>(c->partial2),
                   c->lb_scan ? P<unsigned long long>(c->sstate2) : nullptr, c->scan_words};
      return sort_objects(c, ss, sp2);
    }
    case 1: {  // ---- K2: query -> leaf scatter (concurrent with the object sort) ----
      k_query_count<<<Gs, 256, 0, st>>>(d);
      scan_launch(sp, ArrIn<int32_t>{d.nsub}, ExclOut<int32_t>{d.qsbase}, &h->m, h, &h->S, st);
      k_check_caps<<<1, 1, 0, st>>>(h, 1, 0, 0);
      scan_launch(sp, LeafSqIn{d.leaf_cnt}, ExclOut<int32_t>{d.leaf_sbase}, &h->L, h,
                  (int64_t*)nullptr, st);
      k_query_fill<<<Gs, 256, 0, st>>>(d);
      k_leaf_stats<<<Gbig, 256, 0, st>>>(d);
      return 10;
    }
    case 2: {  // ---- join preparation -----------------------------------
      const int extra = 0;
      scan_launch(sp, WordsIn{d.leaf_nobj, d.leaf_nisq, d.leaf_active}, ExclOut<int64_t>{d.leaf_woff}, &h->L, h,
                  &h->W, st);
      scan_launch(sp, UnitsIn{d.leaf_nobj, d.leaf_nisq, d.leaf_active}, ExclOut<int64_t>{d.leaf_ubase}, &h->L, h,
                  &h->U, st);
      k_check_caps<<<1, 1, 0, st>>>(h, 2, 0, 0);
      k_unit_map<<<Gbig, 256, 0, st>>>(d);
      k_zero_counts<<<Gbig, 256, 0, st>>>(d);
      return 9 + extra;
    }
    case 3:  // ---- K3: join ---------------------------------------------
      k_join<<<c->num_sms * c->join_blocks, kJT, sizeof(JoinSmem), st>>>(d);
      return 1;
    case 4:  // ---- K4: result offsets ---------------------------------------
      k_cov_counts<<<Gbig, 256, 0, st>>>(d);
      k_slot_counts<<<Gbig, 256, 0, st>>>(d);
      scan_launch(sp, ArrIn<int32_t>{d.sq_count}, ExclOut<int64_t>{d.slot_off}, &h->S, h, &h->R, st);
      k_check_caps<<<1, 1, 0, st>>>(h, 3, 0, 0);
      k_close_offsets<<<1, 1, 0, st>>>(d);
      return 7;
    case 5:  // ---- K4: decode + canonical lists (its own stage: timed alone) ----
      // the CTAs its register budget lets reside; the instantiations for the other id modes return at once
      k_decode_query<kIdsRows><<<c->num_sms * c->decode_blocks, kDQThreads, 0, st>>>(d);
      k_decode_query<kIdsKeyed><<<c->num_sms * c->decode_blocks, kDQThreads, 0, st>>>(d);
      k_decode_query<kIdsLookup><<<c->num_sms * c->decode_blocks, kDQThreads, 0, st>>>(d);
      return 3;
    default:  // ---- lists that need a sort by id ----------------------------
      k_merge_big<<<c->num_sms * 2, 256, 0, st>>>(d);
      return 1;
  }
}

// timing event recorded after each stage: build, scatter, prep, join, decode, merge
constexpr int kStageEvent[kStages] = {6, 1, 2, 3, 9, 4, 5};

void init_hdr(tj_ctx* c, int64_t n, int64_t m) {
  DevHdr& H = *c->h_hdr;
  std::memset(&H, 0, sizeof(DevHdr));
  H.n = n;
  H.m = m;
  H.th = c->cfg.th_quad;
  H.l_max = c->cfg.l_max;
  H.F = std::min(c->cfg.l_max, kDenseTop);
  H.covering = c->cfg.covering_optimization ? 1 : 0;
  H.cap_S = c->cap_S;
  H.cap_W = c->cap_W;
  H.cap_R = c->cap_R;
  H.cap_U = c->cap_U;
  H.cap_L = c->cap_L;
  H.kmin_x = H.kmin_y = ~0ull;
  H.kmax_x = H.kmax_y = 0ull;
  H.l_deep = c->ug_sf ? c->cfg.l_max : 1;  // a uniform grid has all its cells at one level
  H.grid_sf = c->ug_sf;
  H.shard_rank = c->shard_rank;
  H.shard_n = c->shard_n;
  H.n_sort = n;  // (sharded: the own-leaf compaction overwrites it)
  H.id_kmin = ~0ull;
  H.id_kmax = 0ull;
  H.key_req = c->key_req ? 1 : 0;
  if (c->reuse) {  // adaptive reuse: the index's MBR, scales, depth and leaves
    const DevHdr& I = c->idx;
    H.xa = I.xa; H.ya = I.ya; H.xb = I.xb; H.yb = I.yb;
    H.width = I.width; H.height = I.height;
    H.wpos = I.wpos; H.hpos = I.hpos;
    H.sx_max = I.sx_max; H.sy_max = I.sy_max; H.sx_deep = I.sx_deep; H.sy_deep = I.sy_deep;
    H.side_deep = I.side_deep;
    for (int l = 0; l <= kMaxLevel; ++l) {
      H.lw[l] = I.lw[l];
      H.lh[l] = I.lh[l];
    }
    H.l_deep = I.l_deep;
    H.Z = I.Z;
    H.L = I.L;
    H.reuse_index = 1;
    // the reuse branch of stage 0 skips k_mbr: the check pass measured this tick's id order
    H.not_monotone = c->reuse_not_mono;
    H.not_identity = c->reuse_not_id;
    H.id_kmin = c->reuse_id_kmin;
    H.id_kmax = c->reuse_id_kmax;
  }
  const char* dbg = std::getenv("TJ_DEBUG");
  H.dbg = dbg ? std::atoi(dbg) : 0;
}

int passes_for(int64_t maxkey) { return std::max(1, (bits_for(maxkey) + kRadixBits - 1) / kRadixBits); }

int check_launch(tj_ctx* c) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, TJ_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return TJ_OK;
}

bool same_shape(const TickGraph& g, const tj_ctx* c) {
  return g.n == c->n && g.m == c->m && g.obj_passes == c->obj_passes && g.shard_n == c->shard_n &&
         g.reuse == c->reuse && g.key_req == c->key_req &&
         g.scan_state[0] == c->sstate.p && g.scan_state[1] == c->sstate2.p && g.scan_words == c->scan_words &&
         std::memcmp(&g.dv, &c->dv, sizeof(Dev)) == 0;
}

void drop_graphs(tj_ctx* c) {
  for (auto& g : c->graphs)
    for (auto& e : g.exec)
      if (e) cudaGraphExecDestroy(e);
  c->graphs.clear();
}

// Capture every stage of the launch sequence as its own CUDA graph (the
// timing events sit between the stage graphs, on the stream).
bool capture_tick(tj_ctx* c, TickGraph& g) {
  for (int s = 0; s <= kSortStage; ++s) {
    cudaStream_t cs = (s == kSortStage && !c->serial_sort) ? c->side : c->st;
    cudaGraph_t graph = nullptr;
    if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return false;
    g.launches[s] = launch_stage(c, s);
    cudaError_t e = cudaStreamEndCapture(cs, &graph);
    if (e == cudaSuccess) e = cudaGraphInstantiate(&g.exec[s], graph, cudaGraphInstantiateFlagUseNodePriority);
    if (graph) cudaGraphDestroy(graph);
    if (e != cudaSuccess) return false;
  }
  return true;
}

// Launch one tick: replay the cached stage graphs of this launch shape (the
// tick's ~80 kernels become six graph launches), capturing them on first use.
int run_tick(tj_ctx* c, int64_t* launches) {
  TickGraph* g = nullptr;
  if (c->use_graphs) {
    for (auto& x : c->graphs)
      if (same_shape(x, c)) g = &x;
    if (!g) {
      TickGraph ng;
      std::memcpy(&ng.dv, &c->dv, sizeof(Dev));
      ng.n = c->n;
      ng.m = c->m;
      ng.obj_passes = c->obj_passes;
      ng.shard_n = c->shard_n;
      ng.reuse = c->reuse;
      ng.key_req = c->key_req;
      ng.scan_state[0] = c->sstate.p;
      ng.scan_state[1] = c->sstate2.p;
      ng.scan_words = c->scan_words;
      if (capture_tick(c, ng)) {
        if (c->graphs.size() >= 4) {
          for (auto& e : c->graphs.front().exec)
            if (e) cudaGraphExecDestroy(e);
          c->graphs.erase(c->graphs.begin());
        }
        c->graphs.push_back(ng);
        g = &c->graphs.back();
      } else {  // capture unsupported here: launch directly from now on
        for (auto& e : ng.exec)
          if (e) cudaGraphExecDestroy(e);
        cudaGetLastError();
        c->use_graphs = false;
      }
    }
  }
  auto stage = [&](int s, cudaStream_t cs) -> int {
    if (g) {
      *launches += g->launches[s];
      cudaError_t e = cudaGraphLaunch(g->exec[s], cs);
      if (e != cudaSuccess) return fail(c, TJ_E_CUDA, std::string("cudaGraphLaunch: ") + cudaGetErrorString(e));
    } else {
      *launches += launch_stage(c, s);
    }
    return TJ_OK;
  };
  int rc;
  cudaEventRecord(c->ev[0], c->st);
  for (int s = 0; s < kStages; ++s) {
    if (s == 1) {  // fork: the object sort on the side stream, concurrent with the query scatter
      cudaStream_t ss = c->serial_sort ? c->st : c->side;
      cudaStreamWaitEvent(ss, c->ev[kStageEvent[0]], 0);
      cudaEventRecord(c->ev[7], ss);
      if ((rc = stage(kSortStage, ss))) return rc;
      cudaEventRecord(c->ev[8], ss);
    }
    // the join needs the sorted objects; its preparation (stage 2: word / unit offsets from the
    // directory) does not, so it runs while the sort finishes.  Stage 2's event is recorded once
    // the sort has joined, so it marks the join's start.
    if (s == 3) {
      cudaStreamWaitEvent(c->st, c->ev[8], 0);
      cudaEventRecord(c->ev[kStageEvent[2]], c->st);
    }
    if ((rc = stage(s, c->st))) return rc;
    if (s != 2) cudaEventRecord(c->ev[kStageEvent[s]], c->st);
    if (s == 0 && c->after_build && (rc = c->after_build())) return rc;  // sharded: route the queries
  }
  return check_launch(c);
}

// The device tick on device-resident inputs: leaves the query-order CSR in c->outoff / c->outids
// and the tick's statistics in S.
int compute_tick(tj_ctx* c, int64_t n, int64_t m, const int64_t* ids, const double* xs, const double* ys,
                 const double* qxa, const double* qya, const double* qxb, const double* qyb, tj_stats& S,
                 int64_t& R) {
  int rc;
  R = 0;
  if ((rc = ensure(c, c->outoff, (m + 1) * 8))) return rc;
  if (n == 0) {  // engine.py:188-190: every issued query gets []
    TJ_CUDA(cudaMemsetAsync(c->outoff.p, 0, (m + 1) * 8, c->st));
    TJ_CUDA(cudaStreamSynchronize(c->st));
  } else {
    c->n = n;
    c->m = m;
    if ((rc = prepare_static(c, n, m))) return rc;
    // first tick: assume < 2^16 leaves (two radix passes); a larger tree aborts and replays the
    // tick with more passes once.  Starting from the capacity bound instead would capture the first
    // tick's graphs with a pass count later ticks no longer use (a re-capture when its inputs recur).
    if (c->last_L == 0) c->last_L = std::min<int64_t>(c->cap_L, int64_t(1) << 16);
    c->obj_passes = passes_for(std::max<int64_t>(c->last_L, 1) - 1);  // grows (tick replay) if L crosses a digit
    // adaptive rebuild (engine.py:163-174): check the previous index against this tick's objects
    c->reuse = false;
    if (c->cfg.rebuild == TJ_REBUILD_ADAPTIVE && c->have_index) {
      if ((rc = prepare_dynamic(c))) return rc;
      fill_dev(c, ids, xs, ys, qxa, qya, qxb, qyb);
      c->reuse = true;
      init_hdr(c, n, m);
      TJ_CUDA(cudaMemcpyAsync(c->d_hdr, c->h_hdr, sizeof(DevHdr), cudaMemcpyHostToDevice, c->st));
      const int lmax = c->cfg.l_max, F = std::min(lmax, kDenseTop);
      const int Gn = grid_for(c, n);
      Dev& d = c->dv;
      cudaMemsetAsync(d.pyr + pyr_off(F), 0, (pyr_off(F + 1) - pyr_off(F)) * 4, c->st);
      k_mbr<<<Gn, 256, 0, c->st>>>(d);
      k_reuse_oob<<<1, 1, 0, c->st>>>(c->d_hdr);
      k_codes<<<Gn, 256, 0, c->st>>>(d);  // at the old index's scale
      for (int l = F - 1; l >= 0; --l)
        k_pyr_level<<<grid_for(c, int64_t(1) << (2 * l)), 256, 0, c->st>>>(d, l);
      k_leaf_recount<<<c->num_sms * 8, 256, 0, c->st>>>(d);
      S.kernel_launches += 4 + F;
      if ((rc = check_launch(c))) return rc;
      TJ_CUDA(cudaMemcpyAsync(c->h_hdr, c->d_hdr, sizeof(DevHdr), cudaMemcpyDeviceToHost, c->st));
      TJ_CUDA(cudaStreamSynchronize(c->st));
      const DevHdr& H = *c->h_hdr;
      // needs_rebuild (quadtree.py:250-270): escaped objects, a leaf over 8 x th, or > 5% over 2 x th
      const bool rebuild = H.oob || H.overfull8 > 0 || (double)H.overfull2 / (double)std::max<int64_t>(H.L, 1) > 0.05;
      c->reuse = !rebuild;
      c->reuse_not_mono = H.not_monotone;
      c->reuse_not_id = H.not_identity;
      c->reuse_id_kmin = H.id_kmin;
      c->reuse_id_kmax = H.id_kmax;
    }
    bool done = false;
    for (int attempt = 0; attempt < 8 && !done; ++attempt) {
      if ((rc = prepare_dynamic(c))) return rc;
      fill_dev(c, ids, xs, ys, qxa, qya, qxb, qyb);
      init_hdr(c, n, m);
      TJ_CUDA(cudaMemcpyAsync(c->d_hdr, c->h_hdr, sizeof(DevHdr), cudaMemcpyHostToDevice, c->st));
      if ((rc = run_tick(c, &S.kernel_launches))) return rc;
      TJ_CUDA(cudaMemcpyAsync(c->h_hdr, c->d_hdr, sizeof(DevHdr), cudaMemcpyDeviceToHost, c->st));
      TJ_CUDA(cudaStreamSynchronize(c->st));
      const DevHdr& H = *c->h_hdr;
      if (!H.abort) {
        done = true;
        break;
      }
      S.retries++;
      if (H.abort & (8 | 16)) return fail(c, TJ_E_CUDA, "internal capacity bound violated (leaves)");
      if (H.abort & 64) return fail(c, TJ_E_INVALID_ARG, "tick too large: 2^32 or more bitmap words");
      if (H.abort & 32) {
        c->obj_passes = passes_for(H.L - 1);
      }
      if (H.abort & 1) c->cap_S = std::max<int64_t>(2 * c->cap_S, H.S + H.S / 4 + 256);
      if (H.abort & 2) {
        c->cap_W = std::max<int64_t>(c->cap_W, H.W + H.W / 4 + 4096);
        c->cap_U = std::max<int64_t>(c->cap_U, H.U + H.U / 4 + 1024);
      }
      if (H.abort & 4) c->cap_R = std::max<int64_t>(2 * c->cap_R, H.R + H.R / 4 + 4096);
    }
    if (!done) return fail(c, TJ_E_CUDA, "tick did not converge after capacity growth");
    const DevHdr& H = *c->h_hdr;
    c->last = H;
    c->last_L = H.L;
    if (!c->reuse) {  // this tick built the index: keep it for the adaptive policy
      c->idx = H;
      c->have_index = true;
    }
    // keyed lists for the next tick, predicted from this one's ids
    if (H.dup_ids) c->dup_ids_seen = true;
    c->key_req = c->key_auto && !c->sort_xy && !c->dup_ids_seen && H.not_identity &&
                 ((H.id_kmax - H.id_kmin) >> kKeyBits) == 0;
    S.id_order = H.key_mode ? TJ_IDS_KEYED : (!H.not_monotone ? TJ_IDS_MONOTONE : TJ_IDS_SORTED);
    if (H.tiling_gap) return fail(c, TJ_E_TILING_GAP, "leaves do not tile the deepest-level grid");
    if (H.dup) return fail(c, TJ_E_DUPLICATE_RESULT, "a (query, object) pair was produced twice");
    if (H.count_mismatch) return fail(c, TJ_E_COUNT_MISMATCH, "decoded counts disagree with popcounts");
    R = H.R;
    c->have = true;
    float ms[5] = {0, 0, 0, 0, 0}, tot = 0;
    cudaEventElapsedTime(&ms[0], c->ev[0], c->ev[1]);
    cudaEventElapsedTime(&ms[1], c->ev[1], c->ev[3]);
    cudaEventElapsedTime(&ms[2], c->ev[3], c->ev[4]);
    cudaEventElapsedTime(&ms[3], c->ev[4], c->ev[5]);
    cudaEventElapsedTime(&ms[4], c->ev[2], c->ev[3]);
    cudaEventElapsedTime(&tot, c->ev[0], c->ev[5]);
    S.t_index_ms = ms[0];
    S.t_filter_ms = ms[1];
    S.t_decode_ms = ms[2];
    S.t_merge_ms = ms[3];
    S.t_join_ms = ms[4];
    float kb = 0;
    cudaEventElapsedTime(&kb, c->ev[0], c->ev[6]);
    S.t_build_ms = kb;
    S.t_scatter_ms = ms[0] - kb;
    float ks = 0;
    cudaEventElapsedTime(&ks, c->ev[7], c->ev[8]);
    S.t_sort_ms = ks;
    float kd = 0;
    cudaEventElapsedTime(&kd, c->ev[9], c->ev[4]);
    S.t_decode_kernel_ms = kd;
    S.t_total_ms = tot;
    S.task_objects = (int64_t)H.task_obj;
    S.task_subqueries = (int64_t)H.task_isq;
    S.containment_tests = (int64_t)H.tests;
    S.decoded_bits = (int64_t)H.W_ref * 32;
    S.subq_intersecting = (int64_t)H.sum_isq;
    S.subq_covering = (int64_t)H.sum_cov;
    S.covering_results = (int64_t)H.cov_results;
    S.active_cells = (int64_t)H.active_cells;
    S.results_total = H.R;
    S.occ_sum = (int64_t)H.occ_sum;
    S.occ_sumsq = (int64_t)H.occ_sumsq;
    S.n_leaves = H.L;
    S.l_deep = H.l_deep;
    S.n_tasks = H.n_tasks;
    S.bitmap_words = (int64_t)H.W_ref;
    S.n_subqueries = H.S;
    S.work_units = H.U;
    S.rebuilt = c->reuse ? 0 : 1;
    S.mbr[0] = H.xa;
    S.mbr[1] = H.ya;
    S.mbr[2] = H.xb;
    S.mbr[3] = H.yb;
  }

  return TJ_OK;
}

// Result delivery (device pointers or pinned host copies; TJ_OUT_IDS32 narrows ids and offsets on the
// device when they fit) of a query-order CSR: offsets (m + 1, int64) and ids (R, int64); `scratch`
// holds the narrowed ids.
int deliver(tj_ctx* c, int out_mem, tj_tick_out* out, int64_t m, int64_t R, bool have_ids, const DBuf& offbuf,
            const DBuf& idsbuf, DBuf& scratch, tj_stats& S) {
  int rc;
  const bool want32 = (out_mem & TJ_OUT_IDS32) != 0;
  const int out_space = out_mem & ~TJ_OUT_IDS32;
  out->n_q = m;
  out->n_results = R;
  // TJ_OUT_IDS32: narrow the ids on the device (into the idle merge scratch) when they all fit
  bool use32 = false;
  if (want32) {
    use32 = true;
    if (R > 0) {
      k_narrow_ids<<<c->num_sms * 4, 256, 0, c->st>>>(P<int64_t>(idsbuf), P<int32_t>(scratch), R, c->d_hdr);
      ++S.kernel_launches;
      TJ_CUDA(cudaMemcpyAsync(&c->h_hdr->ids_wide, &c->d_hdr->ids_wide, sizeof(int32_t), cudaMemcpyDeviceToHost,
                              c->st));
      TJ_CUDA(cudaStreamSynchronize(c->st));
      use32 = c->h_hdr->ids_wide == 0;
    }
  }
  const int64_t idb = use32 ? 4 : 8;
  const bool off32 = want32 && R < (int64_t(1) << 31);
  const int64_t ob = off32 ? 4 : 8;
  if (off32) {
    if ((rc = ensure(c, c->outoff32, (size_t)(m + 1) * 4))) return rc;
    k_narrow_offsets<<<c->num_sms * 4, 256, 0, c->st>>>(P<int64_t>(offbuf), P<int32_t>(c->outoff32), m + 1);
    ++S.kernel_launches;
  }
  out->id_bytes = (int32_t)idb;
  out->offset_bytes = (int32_t)ob;
  out->ids = nullptr;
  out->ids32 = nullptr;
  out->offsets = nullptr;
  out->offsets32 = nullptr;
  if (out_space == TJ_MEM_DEVICE) {
    if (off32) out->offsets32 = P<int32_t>(c->outoff32);
    else out->offsets = P<int64_t>(offbuf);
    if (use32) out->ids32 = R ? P<int32_t>(scratch) : nullptr;
    else out->ids = have_ids ? P<int64_t>(idsbuf) : nullptr;
    out->mem = TJ_MEM_DEVICE;
  } else {
    if ((rc = ensure_host(c, c->h_off, c->h_off_bytes, (m + 1) * ob))) return rc;
    if ((rc = ensure_host(c, c->h_ids, c->h_ids_bytes, R * idb))) return rc;
    TJ_CUDA(cudaMemcpyAsync(c->h_off, off32 ? c->outoff32.p : offbuf.p, (m + 1) * ob, cudaMemcpyDeviceToHost,
                            c->st));
    if (R) TJ_CUDA(cudaMemcpyAsync(c->h_ids, use32 ? scratch.p : idsbuf.p, R * idb, cudaMemcpyDeviceToHost,
                                   c->st));
    TJ_CUDA(cudaStreamSynchronize(c->st));
    if (off32) out->offsets32 = (const int32_t*)c->h_off;
    else out->offsets = (const int64_t*)c->h_off;
    if (use32) out->ids32 = (const int32_t*)c->h_ids;
    else out->ids = (const int64_t*)c->h_ids;
    out->mem = TJ_MEM_HOST;
  }
  return TJ_OK;
}


}  // namespace

#include "tj_shard.cuh"

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int tj_abi_version(void) { return TJ_ABI_VERSION; }

int tj_device_count(int* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  if (count) *count = n;
  return TJ_OK;
}

const char* tj_last_error(const tj_ctx* ctx) { return ctx ? ctx->err.c_str() : g_last_error.c_str(); }

int tj_create(const tj_config* cfg, tj_ctx** out) {
  tj_ctx* c = nullptr;
  if (!cfg || !out) return fail(c, TJ_E_INVALID_ARG, "null argument");
  // MethodConfig.validate (engine.py:73-88)
  if (cfg->split_factor < 0) return fail(c, TJ_E_BAD_CONFIG, "split_factor must be >= 1");
  if (cfg->split_factor > (1 << kMaxLevel))
    return fail(c, TJ_E_BAD_CONFIG, "split factors above 4096 are not supported on the device path");
  if (cfg->split_factor == 0) {
    if (cfg->th_quad < 1) return fail(c, TJ_E_BAD_CONFIG, "th_quad must be >= 1");
    if (cfg->l_max < 1 || cfg->l_max > kMaxLevel) return fail(c, TJ_E_BAD_CONFIG, "l_max must be in [1, 12]");
  }
  if (cfg->rebuild != TJ_REBUILD_EVERY_TICK && cfg->rebuild != TJ_REBUILD_ADAPTIVE)
    return fail(c, TJ_E_BAD_CONFIG, "unknown rebuild policy");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(c, TJ_E_NO_DEVICE, "no CUDA device visible");
  }
  if (cfg->device < 0 || cfg->device >= ndev) return fail(c, TJ_E_NO_DEVICE, "device ordinal out of range");
  c = new tj_ctx();
  c->cfg = *cfg;
  if (cfg->split_factor > 0) {  // method "ug": the grid as the leaf level of a 2^L x 2^L cell map
    c->ug_sf = cfg->split_factor;
    int L = 1;
    while ((1 << L) < cfg->split_factor) ++L;
    c->cfg.l_max = L;
    c->cfg.th_quad = 1;
    c->cfg.rebuild = TJ_REBUILD_EVERY_TICK;
  }
  c->device = cfg->device;
  if (const char* ng = std::getenv("TJ_NO_GRAPH")) c->use_graphs = std::atoi(ng) == 0;
  if (const char* lb = std::getenv("TJ_SCAN_LB")) c->lb_scan = std::atoi(lb) != 0;
  if (const char* ss = std::getenv("TJ_SERIAL_SORT")) c->serial_sort = std::atoi(ss) != 0;
  if (const char* sx = std::getenv("TJ_SORT_XY")) c->sort_xy = std::atoi(sx) != 0;
  if (const char* sp = std::getenv("TJ_SCATTER_PER_SM")) c->scatter_per_sm = std::max(1, std::atoi(sp));
  if (const char* fp = std::getenv("TJ_FUSED_PYR")) c->fused_pyr = std::atoi(fp) != 0;
  if (const char* ky = std::getenv("TJ_KEYED")) c->key_auto = std::atoi(ky) != 0;
  if (const char* ct = std::getenv("TJ_CHECK_TILING")) c->check_tiling = std::atoi(ct) != 0;
  cudaSetDevice(c->device);
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device);
  // side-stream priority (TJ_SIDE_PRIO=1: the object sort's blocks go first) measured no gain:
  // the sort branch is latency-bound, not starved of SMs; default priority
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  int side_prio = prio_lo;
  if (const char* sp = std::getenv("TJ_SIDE_PRIO")) side_prio = std::atoi(sp) ? prio_hi : prio_lo;
  if (cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, side_prio) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaMalloc(&c->d_hdr, sizeof(DevHdr)) != cudaSuccess ||
      cudaMallocHost(&c->h_hdr, sizeof(DevHdr)) != cudaSuccess ||
      cudaMalloc(&c->d_consts, 8 * sizeof(int64_t)) != cudaSuccess) {
    std::string msg = std::string("context setup: ") + cudaGetErrorString(cudaGetLastError());
    tj_destroy(c);
    return fail(nullptr, TJ_E_CUDA, msg);
  }
  for (auto& e : c->ev) cudaEventCreate(&e);
  cudaFuncSetAttribute(k_join, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(JoinSmem));
  cudaFuncSetAttribute(k_radix_downsweep<ArrKey, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)radix_smem_bytes<true>());
  cudaFuncSetAttribute(k_radix_downsweep<ArrKey, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)radix_smem_bytes<false>());
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->join_blocks, k_join, kJT, sizeof(JoinSmem));
  if (c->join_blocks < 1) c->join_blocks = 1;
  // the decode's grid: exactly its resident CTAs (a persistent grid-stride kernel)
  // (no shared-memory carveout preference: asking for the maximum shrank L1, which the decode's
  // leaf-position lookups live in — 40% slower at C5)
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->decode_blocks, k_decode_query<kIdsRows>, kDQThreads, 0);
  if (c->decode_blocks < 1) c->decode_blocks = 1;

  int64_t consts[8] = {(int64_t)kRadixDigits * 2 * c->num_sms, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpy(c->d_consts, consts, sizeof(consts), cudaMemcpyHostToDevice);
  *out = c;
  return TJ_OK;
}

int tj_destroy(tj_ctx* c) {
  if (!c) return TJ_OK;
  cudaSetDevice(c->device);
  if (c->st) cudaStreamSynchronize(c->st);
  drop_graphs(c);
  DBuf* all[] = {&c->ids, &c->xs, &c->ys, &c->qxa, &c->qya, &c->qxb, &c->qyb, &c->code, &c->okey0, &c->okey1,
                 &c->oval0, &c->oval1, &c->sx, &c->sy, &c->tx, &c->ty, &c->loff, &c->presence, &c->prespre, &c->order, &c->crow, &c->pyr, &c->clev,
                 &c->zmap, &c->lcode, &c->lnobj, &c->lobase, &c->lnisq, &c->lncov, &c->lsbase, &c->lwoff,
                 &c->lubase, &c->leafcnt, &c->nsub, &c->qsbase, &c->qpos, &c->qwin, &c->biglist, &c->sqle,
                 &c->sqcount, &c->ecount, &c->erect, &c->slotoff, &c->linfo, &c->leafcur, &c->unitleaf, &c->lactive, &c->lwpre, &c->bitmap,
                 &c->outids, &c->outoff, &c->scratch, &c->outoff32, &c->partial, &c->partial2, &c->rhist, &c->roffs, &c->sstate, &c->sstate2,
                 &c->pcnt, &c->rcnt, &c->sstart, &c->moff, &c->sconst, &c->rids, &c->mids, &c->mscratch,
                 &c->oq[0], &c->oq[1], &c->oq[2], &c->oq[3], &c->qmask, &c->packpos, &c->dcnt, &c->sq[0], &c->sq[1],
                 &c->sq[2], &c->sq[3], &c->rq[0], &c->rq[1], &c->rq[2], &c->rq[3], &c->gcnt, &c->gstart};
  delete c->comm;
  c->comm = nullptr;
  for (DBuf* b : all)
    if (b->p) cudaFree(b->p);
  if (c->h_off) cudaFreeHost(c->h_off);
  if (c->h_ids) cudaFreeHost(c->h_ids);
  if (c->d_hdr) cudaFree(c->d_hdr);
  if (c->h_hdr) cudaFreeHost(c->h_hdr);
  if (c->d_consts) cudaFree(c->d_consts);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->st) cudaStreamDestroy(c->st);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  delete c;
  return TJ_OK;
}

int tj_tick(tj_ctx* c, const tj_tick_in* in, tj_tick_out* out, tj_stats* stats) {
  if (!c || !in || !out) return fail(c, TJ_E_INVALID_ARG, "null argument");
  const int64_t n = in->n_obj, m = in->n_q;
  const int out_space = in->out_mem & ~TJ_OUT_IDS32;
  if (out_space != TJ_MEM_HOST && out_space != TJ_MEM_DEVICE)
    return fail(c, TJ_E_INVALID_ARG, "unknown output memory space");
  if (n < 0 || m < 0) return fail(c, TJ_E_INVALID_ARG, "negative size");
  if (n > INT32_MAX / 2 || m > INT32_MAX / 2) return fail(c, TJ_E_INVALID_ARG, "tick too large for 32-bit rows");
  if (n >= (int64_t(1) << 28)) return fail(c, TJ_E_INVALID_ARG, "more than 2^28 objects per tick is not supported");
  if ((n && (!in->obj_id || !in->obj_x || !in->obj_y)) ||
      (m && (!in->q_issuer || !in->q_xa || !in->q_ya || !in->q_xb || !in->q_yb)))
    return fail(c, TJ_E_INVALID_ARG, "null input array");
  TJ_CUDA(cudaSetDevice(c->device));
  c->have = false;
  tj_stats S{};
  S.n_objects = n;
  S.n_queries = m;
  int rc;

  // ---- inputs to device ---------------------------------------------------
  const int64_t* ids = in->obj_id;
  const double *xs = in->obj_x, *ys = in->obj_y;
  const double *qxa = in->q_xa, *qya = in->q_ya, *qxb = in->q_xb, *qyb = in->q_yb;
  if (in->mem == TJ_MEM_HOST) {
    if ((rc = ensure(c, c->ids, n * 8)) || (rc = ensure(c, c->xs, n * 8)) || (rc = ensure(c, c->ys, n * 8)) ||
        (rc = ensure(c, c->qxa, m * 8)) || (rc = ensure(c, c->qya, m * 8)) || (rc = ensure(c, c->qxb, m * 8)) ||
        (rc = ensure(c, c->qyb, m * 8)))
      return rc;
    TJ_CUDA(cudaMemcpyAsync(c->ids.p, ids, n * 8, cudaMemcpyHostToDevice, c->st));
    TJ_CUDA(cudaMemcpyAsync(c->xs.p, xs, n * 8, cudaMemcpyHostToDevice, c->st));
    TJ_CUDA(cudaMemcpyAsync(c->ys.p, ys, n * 8, cudaMemcpyHostToDevice, c->st));
    TJ_CUDA(cudaMemcpyAsync(c->qxa.p, qxa, m * 8, cudaMemcpyHostToDevice, c->st));
    TJ_CUDA(cudaMemcpyAsync(c->qya.p, qya, m * 8, cudaMemcpyHostToDevice, c->st));
    TJ_CUDA(cudaMemcpyAsync(c->qxb.p, qxb, m * 8, cudaMemcpyHostToDevice, c->st));
    TJ_CUDA(cudaMemcpyAsync(c->qyb.p, qyb, m * 8, cudaMemcpyHostToDevice, c->st));
    ids = P<int64_t>(c->ids);
    xs = P<double>(c->xs);
    ys = P<double>(c->ys);
    qxa = P<double>(c->qxa);
    qya = P<double>(c->qya);
    qxb = P<double>(c->qxb);
    qyb = P<double>(c->qyb);
  } else if (in->mem != TJ_MEM_DEVICE) {
    return fail(c, TJ_E_INVALID_ARG, "unknown memory space");
  }

  int64_t R = 0;
  if ((rc = compute_tick(c, n, m, ids, xs, ys, qxa, qya, qxb, qyb, S, R))) return rc;
  if ((rc = deliver(c, in->out_mem, out, m, R, n > 0, c->outoff, c->outids, c->scratch, S))) return rc;
  if (stats) *stats = S;
  return TJ_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Introspection (host copies in the reference's order)
// ---------------------------------------------------------------------------
namespace {

template <typename T>
int d2h(tj_ctx* c, std::vector<T>& v, const void* src, int64_t count) {
  v.resize((size_t)std::max<int64_t>(count, 0));
  if (count > 0) TJ_CUDA(cudaMemcpy(v.data(), src, count * sizeof(T), cudaMemcpyDeviceToHost));
  return TJ_OK;
}

struct LeafView {
  std::vector<uint32_t> code;
  std::vector<int32_t> nobj, obase, nisq, ncov, sbase;
  std::vector<int64_t> woff;
  std::vector<int64_t> packed;  // reference packing per leaf rank
  std::vector<int64_t> order;   // leaf ranks in ascending packed order
};

int load_leaves(tj_ctx* c, LeafView& lv) {
  const int64_t L = c->last.L;
  int rc;
  if ((rc = d2h(c, lv.code, c->lcode.p, L)) || (rc = d2h(c, lv.nobj, c->lnobj.p, L)) ||
      (rc = d2h(c, lv.obase, c->lobase.p, L)) || (rc = d2h(c, lv.nisq, c->lnisq.p, L)) ||
      (rc = d2h(c, lv.ncov, c->lncov.p, L)) || (rc = d2h(c, lv.sbase, c->lsbase.p, L)) ||
      (rc = d2h(c, lv.woff, c->lwoff.p, L)))
    return rc;
  lv.packed.resize(L);
  const int sh = 2 * c->cfg.l_max;
  for (int64_t r = 0; r < L; ++r) {
    const int64_t lev = lv.code[r] >> kLevelShift;
    const int64_t z = lv.code[r] & kPayloadMask;
    lv.packed[r] = c->ug_sf ? z : (lev << sh) | z;  // ug: cell id = Morton(i, j) (grid.py:68)
  }
  lv.order.resize(L);
  for (int64_t r = 0; r < L; ++r) lv.order[r] = r;
  std::sort(lv.order.begin(), lv.order.end(), [&](int64_t a, int64_t b) { return lv.packed[a] < lv.packed[b]; });
  return TJ_OK;
}

// Directory entries of leaf r's block [e0, e0 + cnt) in the reference's
// order (ascending slot = query input order, directory.py:131): the device
// keeps fill order inside a block; entry -> slot inverts the slots' entries.
// Method "ug": a query's subqueries are listed row-major over its window
// (grid.py:91-97), the device keeps them in Morton order; pos[slot] = the
// slot's index in the reference's list (identity for the quadtree).
int ug_ref_pos(tj_ctx* c, const std::vector<int2>& le, std::vector<int64_t>& pos) {
  pos.resize(le.size());
  for (size_t s = 0; s < le.size(); ++s) pos[s] = (int64_t)s;
  if (!c->ug_sf) return TJ_OK;
  std::vector<int32_t> nsub;
  std::vector<uint32_t> code;
  int rc;
  if ((rc = d2h(c, nsub, c->nsub.p, c->m)) || (rc = d2h(c, code, c->lcode.p, c->last.L))) return rc;
  auto rowmajor = [&](int64_t s) {
    const uint32_t z = code[le[s].x] & kPayloadMask;
    return (uint64_t(compact2(z >> 1)) << 32) | compact2(z);  // (j, i)
  };
  std::vector<int64_t> tmp;
  int64_t s0 = 0;
  for (int64_t q = 0; q < c->m; ++q) {
    const int k = nsub[q];
    tmp.resize(k);
    for (int j = 0; j < k; ++j) tmp[j] = s0 + j;
    std::sort(tmp.begin(), tmp.end(), [&](int64_t a, int64_t b) { return rowmajor(a) < rowmajor(b); });
    for (int j = 0; j < k; ++j) pos[tmp[j]] = s0 + j;
    s0 += k;
  }
  return TJ_OK;
}

int entry_slots(tj_ctx* c, std::vector<int32_t>& eslot) {
  std::vector<int2> le;
  std::vector<int64_t> pos;
  int rc;
  if ((rc = d2h(c, le, c->sqle.p, c->last.S)) || (rc = ug_ref_pos(c, le, pos))) return rc;
  eslot.assign(le.size(), -1);
  for (size_t s = 0; s < le.size(); ++s) eslot[le[s].y] = (int32_t)pos[s];
  return TJ_OK;
}
std::vector<int32_t> block_in_ref_order(const std::vector<int32_t>& eslot, int64_t e0, int64_t cnt) {
  std::vector<int32_t> es((size_t)cnt);
  for (int64_t j = 0; j < cnt; ++j) es[j] = (int32_t)(e0 + j);
  std::sort(es.begin(), es.end(), [&](int32_t x, int32_t y) { return eslot[x] < eslot[y]; });
  return es;
}

// Objects of the last tick in device leaf order: rows[k] = input row at leaf position k, refpos[k] =
// its place in the reference's leaf block (input order, directory.py:128).  Keyed lists put each
// leaf block in id order on the device, so refpos is a permutation there; the identity otherwise.
int leaf_order(tj_ctx* c, const LeafView& lv, std::vector<int32_t>& rows, std::vector<int32_t>& refpos) {
  int rc;
  if ((rc = d2h(c, rows, c->dv.sidx, c->n))) return rc;
  refpos.resize(rows.size());
  for (size_t k = 0; k < refpos.size(); ++k) refpos[k] = (int32_t)k;
  if (!c->last.key_mode) return TJ_OK;
  std::vector<int32_t> ord;
  for (size_t r = 0; r < lv.nobj.size(); ++r) {
    const int32_t b = lv.obase[r], no = lv.nobj[r];
    ord.resize(no);
    for (int32_t j = 0; j < no; ++j) ord[j] = j;
    std::sort(ord.begin(), ord.end(), [&](int32_t a, int32_t x) { return rows[b + a] < rows[b + x]; });
    for (int32_t j = 0; j < no; ++j) refpos[b + ord[j]] = b + j;
  }
  return TJ_OK;
}

int need_tick(tj_ctx* c) {
  if (!c) return TJ_E_INVALID_ARG;
  if (!c->have) return fail(c, TJ_E_INVALID_ARG, "no completed tick with objects to introspect");
  cudaSetDevice(c->device);
  return TJ_OK;
}

}  // namespace

extern "C" {

int tj_get_index(tj_ctx* c, tj_index_info* info, int64_t* leaves, int64_t leaves_cap, int64_t* zmap,
                 int64_t zmap_cap) {
  int rc;
  if ((rc = need_tick(c))) return rc;
  const DevHdr& H = c->last;
  if (info) {
    info->mbr[0] = H.xa;
    info->mbr[1] = H.ya;
    info->mbr[2] = H.xb;
    info->mbr[3] = H.yb;
    info->th_quad = c->cfg.th_quad;
    info->l_max = c->cfg.l_max;
    info->l_deep = H.l_deep;
    info->n_leaves = H.L;
    info->n_cells = H.Z;
  }
  if (!leaves && !zmap) return TJ_OK;
  LeafView lv;
  if ((rc = load_leaves(c, lv))) return rc;
  if (leaves) {
    if (leaves_cap < H.L) return fail(c, TJ_E_INVALID_ARG, "leaves buffer too small");
    for (int64_t k = 0; k < H.L; ++k) leaves[k] = lv.packed[lv.order[k]];
  }
  if (zmap) {
    if (zmap_cap < H.Z) return fail(c, TJ_E_INVALID_ARG, "zmap buffer too small");
    std::vector<uint32_t> z;
    if ((rc = d2h(c, z, c->zmap.p, H.Z))) return rc;
    for (int64_t k = 0; k < H.Z; ++k) zmap[k] = lv.packed[z[k] & kPayloadMask];
  }
  return TJ_OK;
}

int tj_get_object_cells(tj_ctx* c, int64_t* cells, int64_t cap) {
  int rc;
  if ((rc = need_tick(c))) return rc;
  if (!cells || cap < c->n) return fail(c, TJ_E_INVALID_ARG, "cells buffer too small");
  LeafView lv;
  if ((rc = load_leaves(c, lv))) return rc;
  std::vector<uint32_t> code, z;
  if ((rc = d2h(c, code, c->code.p, c->n)) || (rc = d2h(c, z, c->zmap.p, c->last.Z))) return rc;
  const int sh = 2 * (c->cfg.l_max - c->last.l_deep);
  for (int64_t i = 0; i < c->n; ++i) cells[i] = lv.packed[z[code[i] >> sh] & kPayloadMask];
  return TJ_OK;
}

int tj_get_subqueries(tj_ctx* c, int64_t* count, int64_t* q_row, int64_t* cell, uint8_t* covering,
                      int64_t cap) {
  int rc;
  if ((rc = need_tick(c))) return rc;
  const int64_t S = c->last.S;
  if (count) *count = S;
  if (!q_row && !cell && !covering) return TJ_OK;
  if (cap < S) return fail(c, TJ_E_INVALID_ARG, "subquery buffers too small");
  LeafView lv;
  if ((rc = load_leaves(c, lv))) return rc;
  std::vector<int2> le;
  std::vector<int32_t> nsub;
  if ((rc = d2h(c, le, c->sqle.p, S)) || (rc = d2h(c, nsub, c->nsub.p, c->m))) return rc;
  std::vector<int64_t> pos;
  if ((rc = ug_ref_pos(c, le, pos))) return rc;
  int64_t s = 0;  // slots are grouped per query in input order (nsub each)
  for (int64_t q = 0; q < c->m; ++q)
    for (int32_t j = 0; j < nsub[q]; ++j, ++s) {
      const int32_t leaf = le[s].x;
      const int64_t p = pos[s];
      if (q_row) q_row[p] = q;
      if (cell) cell[p] = lv.packed[leaf];
      if (covering) covering[p] = (uint8_t)(le[s].y - lv.sbase[leaf] >= lv.nisq[leaf]);
    }
  return TJ_OK;
}

int tj_get_directory(tj_ctx* c, int64_t* obj_rows, int64_t obj_cap, int64_t* isq, int64_t* n_isq, int64_t* cov,
                     int64_t* n_cov, int64_t sq_cap) {
  int rc;
  if ((rc = need_tick(c))) return rc;
  const DevHdr& H = c->last;
  if (n_isq) *n_isq = (int64_t)H.sum_isq;
  if (n_cov) *n_cov = (int64_t)H.sum_cov;
  if (!obj_rows && !isq && !cov) return TJ_OK;
  LeafView lv;
  if ((rc = load_leaves(c, lv))) return rc;
  if (obj_rows) {
    if (obj_cap < c->n) return fail(c, TJ_E_INVALID_ARG, "obj_rows buffer too small");
    std::vector<int32_t> rows, refpos, byref(c->n);
    if ((rc = leaf_order(c, lv, rows, refpos))) return rc;
    for (int64_t k = 0; k < c->n; ++k) byref[refpos[k]] = rows[k];
    int64_t k = 0;
    for (int64_t r : lv.order)
      for (int32_t j = 0; j < lv.nobj[r]; ++j) obj_rows[k++] = byref[lv.obase[r] + j];
  }
  if (isq || cov) {
    if (sq_cap < (int64_t)std::max(H.sum_isq, H.sum_cov)) return fail(c, TJ_E_INVALID_ARG, "sq buffers too small");
    std::vector<int32_t> eslot;
    if ((rc = entry_slots(c, eslot))) return rc;
    int64_t ki = 0, kc = 0;
    for (int64_t r : lv.order) {
      if (isq)
        for (int32_t e : block_in_ref_order(eslot, lv.sbase[r], lv.nisq[r])) isq[ki++] = eslot[e];
      if (cov)
        for (int32_t e : block_in_ref_order(eslot, lv.sbase[r] + lv.nisq[r], lv.ncov[r])) cov[kc++] = eslot[e];
    }
  }
  return TJ_OK;
}

int tj_get_bitmaps(tj_ctx* c, int64_t* n_tasks, int64_t* n_words, int64_t* task_cell, int64_t* task_nobj,
                   int64_t* task_nisq, int64_t* task_woff, uint32_t* words, int64_t* counts, int64_t task_cap,
                   int64_t word_cap, int64_t count_cap) {
  int rc;
  if ((rc = need_tick(c))) return rc;
  const DevHdr& H = c->last;
  if (n_tasks) *n_tasks = H.n_tasks;
  if (n_words) *n_words = (int64_t)H.W_ref;
  if (!task_cell && !words && !counts) return TJ_OK;
  if (task_cap < H.n_tasks || word_cap < (int64_t)H.W_ref) return fail(c, TJ_E_INVALID_ARG, "bitmap buffers too small");
  LeafView lv;
  if ((rc = load_leaves(c, lv))) return rc;
  std::vector<uint32_t> bm;
  std::vector<int32_t> info, eslot;
  if ((rc = d2h(c, bm, c->bitmap.p, H.W)) || (rc = d2h(c, info, c->ecount.p, H.S)) ||
      (rc = entry_slots(c, eslot)))
    return rc;
  std::vector<int32_t> orows, refpos;
  if (c->last.key_mode && words && (rc = leaf_order(c, lv, orows, refpos))) return rc;
  int64_t t = 0, w = 0, k = 0;
  if (task_woff) task_woff[0] = 0;
  for (int64_t r : lv.order) {
    const int64_t no = lv.nobj[r], ni = lv.nisq[r];
    if (!(no > 0 && ni > 0)) continue;
    const int64_t nw = ni * ((no + 31) / 32);
    if (task_cell) task_cell[t] = lv.packed[r];
    if (task_nobj) task_nobj[t] = no;
    if (task_nisq) task_nisq[t] = ni;
    const int64_t nb = (no + 31) / 32;
    const std::vector<int32_t> rows = block_in_ref_order(eslot, lv.sbase[r], ni);
    if (words && !c->last.key_mode)
      for (int64_t j = 0; j < ni; ++j)
        std::memcpy(words + w + j * nb, bm.data() + lv.woff[r] + (rows[j] - lv.sbase[r]) * row_words((int)nb), nb * 4);
    if (words && c->last.key_mode)  // device bit k of the leaf block -> the reference's bit refpos[k]
      for (int64_t j = 0; j < ni; ++j) {
        const uint32_t* src = bm.data() + lv.woff[r] + (rows[j] - lv.sbase[r]) * row_words((int)nb);
        uint32_t* dst = words + w + j * nb;
        std::memset(dst, 0, nb * 4);
        for (int64_t p = 0; p < no; ++p)
          if ((src[p >> 5] >> (p & 31)) & 1u) {
            const int64_t q = refpos[lv.obase[r] + p] - lv.obase[r];
            dst[q >> 5] |= 1u << (q & 31);
          }
      }
    if (counts) {
      if (k + ni > count_cap) return fail(c, TJ_E_INVALID_ARG, "counts buffer too small");
      for (int64_t j = 0; j < ni; ++j) counts[k + j] = (int64_t)info[rows[j]];
    }
    w += nw;
    k += ni;
    ++t;
    if (task_woff) task_woff[t] = w;
  }
  return TJ_OK;
}

int tj_get_imbalance(tj_ctx* c, int32_t sim_processors, int32_t heaviest_first, double* imbalance) {
  int rc;
  if ((rc = need_tick(c))) return rc;
  if (sim_processors < 1 || !imbalance) return fail(c, TJ_E_INVALID_ARG, "bad arguments");
  LeafView lv;
  if ((rc = load_leaves(c, lv))) return rc;
  std::vector<std::pair<int64_t, int64_t>> tasks;  // (weight, packed cell), directory order
  for (int64_t r : lv.order)
    if (lv.nobj[r] > 0 && lv.nisq[r] > 0) tasks.emplace_back((int64_t)lv.nobj[r] * lv.nisq[r], lv.packed[r]);
  if (heaviest_first)  // scheduler.py:31-38: (-weight, cell_id)
    std::stable_sort(tasks.begin(), tasks.end(), [](const auto& a, const auto& b) {
      return a.first != b.first ? a.first > b.first : a.second < b.second;
    });
  std::vector<int64_t> tot(sim_processors, 0);  // scheduler.py:41-54
  for (const auto& t : tasks) {
    int best = 0;
    for (int p = 1; p < sim_processors; ++p)
      if (tot[p] < tot[best]) best = p;
    tot[best] += t.first;
  }
  const int64_t top = *std::max_element(tot.begin(), tot.end());
  const int64_t low = *std::min_element(tot.begin(), tot.end());
  *imbalance = top == 0 ? 0.0 : (double)(top - low) / (double)top;
  return TJ_OK;
}

int tj_get_occupancy(tj_ctx* c, int64_t* counts, int64_t cap, int64_t* n_active) {
  int rc;
  if ((rc = need_tick(c))) return rc;
  if (!n_active) return fail(c, TJ_E_INVALID_ARG, "bad arguments");
  std::vector<int32_t> nobj;
  std::vector<uint32_t> code;
  if ((rc = d2h(c, nobj, c->lnobj.p, c->last.L)) || (rc = d2h(c, code, c->lcode.p, c->last.L))) return rc;
  std::vector<std::pair<int64_t, int32_t>> occ;  // (packed cell, count) of the non-empty leaves
  const int sh = 2 * c->cfg.l_max;
  for (int64_t r = 0; r < c->last.L; ++r)
    if (nobj[r] > 0) {
      const int64_t lev = code[r] >> kLevelShift, z = code[r] & kPayloadMask;
      occ.emplace_back(c->ug_sf ? z : (lev << sh) | z, nobj[r]);
    }
  std::sort(occ.begin(), occ.end());
  *n_active = (int64_t)occ.size();
  if (!counts) return TJ_OK;
  if (cap < (int64_t)occ.size()) return fail(c, TJ_E_INVALID_ARG, "counts buffer too small");
  for (size_t k = 0; k < occ.size(); ++k) counts[k] = occ[k].second;
  return TJ_OK;
}

int tj_get_staging_flushes(tj_ctx* c, int32_t staging_capacity, int64_t* flushes) {
  int rc;
  if ((rc = need_tick(c))) return rc;
  if (staging_capacity < 1 || !flushes) return fail(c, TJ_E_INVALID_ARG, "bad arguments");
  unsigned long long* dcnt = reinterpret_cast<unsigned long long*>(c->d_consts + 7);  // scratch slot
  TJ_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(*dcnt), c->st));
  k_staging_flushes<<<c->num_sms * 8, 256, 0, c->st>>>(c->dv, staging_capacity, dcnt);
  unsigned long long v = 0;
  TJ_CUDA(cudaMemcpyAsync(&v, dcnt, sizeof(v), cudaMemcpyDeviceToHost, c->st));
  TJ_CUDA(cudaStreamSynchronize(c->st));
  *flushes = (int64_t)v;
  return TJ_OK;
}

int tj_set_shard(tj_ctx* c, int32_t rank, int32_t nranks) {
  if (!c || nranks < 1 || rank < 0 || rank >= nranks) return fail(c, TJ_E_INVALID_ARG, "bad shard");
  c->shard_rank = rank;
  c->shard_n = nranks;
  c->have = false;
  return TJ_OK;
}

int tj_nccl_unique_id(void* id, int32_t bytes) {
  if (!id || bytes < (int32_t)sizeof(ncclUniqueId)) return fail(nullptr, TJ_E_INVALID_ARG, "need 128 bytes");
  NcclApi* api = nccl_api();
  if (!api) return fail(nullptr, TJ_E_NCCL, "NCCL unavailable");
  ncclResult_t r = api->GetUniqueId(static_cast<ncclUniqueId*>(id));
  if (r != ncclSuccess) return fail(nullptr, TJ_E_NCCL, std::string("ncclGetUniqueId: ") + api->GetErrorString(r));
  return TJ_OK;
}

int tj_comm_init(tj_ctx* c, const void* unique_id, int32_t rank, int32_t nranks) {
  if (!c || !unique_id || nranks < 1 || rank < 0 || rank >= nranks) return fail(c, TJ_E_INVALID_ARG, "bad comm");
  NcclApi* api = nccl_api();
  if (!api) return fail(c, TJ_E_NCCL, "NCCL unavailable");
  TJ_CUDA(cudaSetDevice(c->device));
  auto* t = new NcclTransport();
  t->api = api;
  t->rank = rank;
  t->nranks = nranks;
  ncclUniqueId uid;
  std::memcpy(&uid, unique_id, sizeof(uid));
  ncclResult_t r = api->CommInitRank(&t->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    t->comm = nullptr;
    delete t;
    return fail(c, TJ_E_NCCL, std::string("ncclCommInitRank: ") + api->GetErrorString(r));
  }
  delete c->comm;
  c->comm = t;
  return TJ_OK;
}

int tj_group_create(int32_t nranks, tj_group** out) {
  if (nranks < 1 || !out) return fail(nullptr, TJ_E_INVALID_ARG, "bad group");
  auto* g = new tj_group();
  g->n = nranks;
  g->ptr.assign(nranks, nullptr);
  g->cnt.assign(nranks, nullptr);
  g->displ.assign(nranks, nullptr);
  *out = g;
  return TJ_OK;
}

int tj_group_destroy(tj_group* g) {
  delete g;
  return TJ_OK;
}

int tj_comm_init_local(tj_ctx* c, tj_group* g, int32_t rank) {
  if (!c || !g || rank < 0 || rank >= g->n) return fail(c, TJ_E_INVALID_ARG, "bad local comm");
  auto* t = new LocalTransport();
  t->g = g;
  t->rank = rank;
  t->nranks = g->n;
  delete c->comm;
  c->comm = t;
  return TJ_OK;
}

int tj_tick_sharded(tj_ctx* c, const tj_tick_in* in, tj_tick_out* out, tj_stats* stats) {
  if (!c || !in || !out) return fail(c, TJ_E_INVALID_ARG, "null argument");
  if (!c->comm) return fail(c, TJ_E_INVALID_ARG, "no communicator: tj_comm_init / tj_comm_init_local first");
  const int64_t n = in->n_obj, m = in->n_q;
  const int out_space = in->out_mem & ~TJ_OUT_IDS32;
  if (out_space != TJ_MEM_HOST && out_space != TJ_MEM_DEVICE)
    return fail(c, TJ_E_INVALID_ARG, "unknown output memory space");
  if (in->mem != TJ_MEM_HOST && in->mem != TJ_MEM_DEVICE) return fail(c, TJ_E_INVALID_ARG, "unknown memory space");
  if (n < 0 || m < 0) return fail(c, TJ_E_INVALID_ARG, "negative size");
  if ((n && (!in->obj_id || !in->obj_x || !in->obj_y)) || (m && (!in->q_xa || !in->q_ya || !in->q_xb || !in->q_yb)))
    return fail(c, TJ_E_INVALID_ARG, "null input array");
  TJ_CUDA(cudaSetDevice(c->device));
  c->have = false;
  tj_stats S{};
  int rc = sharded_tick(c, in, out, S);
  if (rc) return rc;
  if (stats) *stats = S;
  return TJ_OK;
}

int tj_get_stream(tj_ctx* c, void** stream) {
  if (!c || !stream) return TJ_E_INVALID_ARG;
  *stream = (void*)c->st;
  return TJ_OK;
}

int tj_host_alloc(int64_t bytes, void** ptr) {
  if (!ptr || bytes < 0) return TJ_E_INVALID_ARG;
  cudaError_t e = cudaMallocHost(ptr, (size_t)std::max<int64_t>(bytes, 16));
  if (e != cudaSuccess) {
    g_last_error = cudaGetErrorString(e);
    return TJ_E_OOM;
  }
  return TJ_OK;
}

int tj_host_free(void* ptr) {
  if (ptr) cudaFreeHost(ptr);
  return TJ_OK;
}

}  // extern "C"
