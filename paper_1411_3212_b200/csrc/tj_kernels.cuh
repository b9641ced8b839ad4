// QUAD tick kernels for sm_100a.  One persistent-grid launch sequence per
// tick; every size after the index build lives in DevHdr on the device.
//
//   K0  mbr / finalize           geometry.py:72-77, morton.py:100-104
//   K1  codes + level-l_max histogram, dense count pyramid,
//       leaf level per deepest cell, zmap + leaf table (scan), object keys,
//       stable radix sort of objects by leaf, payload gather
//                                 quadtree.py:74-165, directory.py:128
//   K2  query clip + window + leaf enumeration (count / fill), subquery keys,
//       stable radix sort of subqueries by (leaf, covering)
//                                 grid.py:115-122, quadtree.py:168-240, directory.py:131-142
//   K3  per-leaf join into linear 32-bit-word bitmaps + popcounts
//                                 bitmap.py:70-119, engine.py:269-303
//   K4  result offsets, bitmap decode, covering expansion, per-query merge
//                                 decode.py:40-123, engine.py:306-329
#pragma once

#include "tj_common.cuh"
#include "tj_scan.cuh"

namespace tj {

struct __align__(32) Rect4 {
  double xa, ya, xb, yb;
};

struct Dev {
  DevHdr* h;
  // inputs (device)
  const int64_t* ids;
  const double* xs;
  const double* ys;
  const double* qxa;
  const double* qya;
  const double* qxb;
  const double* qyb;
  // objects
  uint32_t* code;
  uint32_t* okey[2];
  int32_t* oval[2];
  const int32_t* sidx;  // objects in leaf order: input rows (points into oval[])
  // keyed lists (DevHdr::key_mode): per leaf position, id - id_min (< 2^28); leaf blocks in id order
  uint32_t* loff;
  uint32_t* presence;   // one bit per id offset (2^28 bits): duplicate detection and id ranks
  int32_t* pres_pre;    // exclusive prefix of the presence words' popcounts
  int32_t* order;       // id rank -> input row (key_sorted ticks)
  int32_t* crow;        // sharded ticks: the rows of the objects in own leaves, compacted in sort order
  double* sx;
  double* sy;
  // index
  uint32_t* pyr;
  uint8_t* clev;
  uint32_t* zmap;
  uint32_t* leaf_code;
  int32_t* leaf_nobj;
  int32_t* leaf_obase;
  int32_t* leaf_nisq;
  int32_t* leaf_ncov;
  int32_t* leaf_sbase;
  int64_t* leaf_woff;
  int64_t* leaf_ubase;
  // queries
  int32_t* nsub;
  int32_t* qsbase;
  // subqueries
  int2* sq_le;              // per subquery slot: (leaf rank, directory entry); query and covering flag are
                            // implied (slot ranges per query; entry row >= the leaf's intersecting count)
  int32_t* sq_count;        // result count per subquery slot (popcount, or block size if covering)
  int32_t* ecount;          // result count per directory entry (entry order)
  Rect4* erect;             // clipped rect per directory entry (entry order, the join's input)
  int4* linfo;              // per leaf: object base, object count, entry base, intersecting count
  int64_t* slot_off;        // per slot (S + 1): start of its run in the output CSR
  int32_t* leaf_cur;       // per leaf x {intersecting, covering}: fill cursor of large-window pairs
  int4* leaf_cnt;          // per leaf: intersecting / covering pairs of small windows, of large windows
  int4* qpos;              // per small-window query: each pair's place in its leaf block
  int4* qwin;              // per query: deepest-cell window of its clipped rect (count pass -> fill pass)
  int32_t* unit_leaf;      // join work unit -> leaf
  uint8_t* leaf_active;    // multi-GPU leaf-range sharding: leaf owned by this rank (nullptr: all)
  int64_t* leaf_wpre;      // exclusive prefix of the per-leaf work weight (sharding)
  int32_t* big_list;       // queries whose lists need the CTA-wide merge
  int64_t* scratch;        // R entries: merge-pass scratch for k_merge_big
  // join + outputs
  uint32_t* bitmap;
  int64_t* out_ids;
  int64_t* out_off;
};

// multi-GPU leaf-range sharding: leaf r belongs to this rank (always, unsharded)
__device__ __forceinline__ bool leaf_on(const uint8_t* active, int64_t r) { return !active || active[r]; }

#define TJ_GRID_STRIDE(i, n) \
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// ===========================================================================
// K0: MBR
// ===========================================================================
__device__ __forceinline__ unsigned long long shfl_min64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u < v ? u : v;
  }
  return v;
}
__device__ __forceinline__ unsigned long long shfl_max64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u > v ? u : v;
  }
  return v;
}

// Exact MBR (order-preserving u64 keys, warp-reduced atomics) and, in the
// same pass, whether object ids strictly increase in input order (then
// per-leaf blocks are id-sorted and per-query merges are merges of sorted
// runs) and whether id == input row (the generator's arange ids: then the
// final lists need no id lookup).  Four items per thread in flight.
__global__ void __launch_bounds__(256) k_mbr(const Dev d) {  // (capped at 64 registers: 2% slower)
  DevHdr* h = d.h;
  const int64_t n = h->n;
  unsigned long long mnx = ~0ull, mny = ~0ull, mxx = 0ull, mxy = 0ull;
  unsigned long long imn = ~0ull, imx = 0ull;  // id range (keyed lists)
  int bad = 0, notid = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // warp-uniform trip count (the next-id shuffle below needs every lane of the warp)
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 - lane_id() < n; i0 += 4 * stride) {
    double x[4], y[4];
    int64_t v[4], nx[4];
    const bool last_lane = lane_id() == 31;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * stride;
      const bool ok = i < n;
      x[u] = ok ? d.xs[i] : 0.0;
      y[u] = ok ? d.ys[i] : 0.0;
      v[u] = ok ? d.ids[i] : 0;
      // the next row's id: the next lane's (consecutive rows per warp); the warp's last lane loads it
      nx[u] = (last_lane && i + 1 < n) ? d.ids[i + 1] : 0x7fffffffffffffffll;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t nb = __shfl_down_sync(0xffffffffu, v[u], 1);
      if (!last_lane) nx[u] = nb;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) {
        const unsigned long long kx = dkey(x[u]), ky = dkey(y[u]);
        mnx = kx < mnx ? kx : mnx;
        mny = ky < mny ? ky : mny;
        mxx = kx > mxx ? kx : mxx;
        mxy = ky > mxy ? ky : mxy;
        notid |= (v[u] != i);
        bad |= (i + 1 < n) && (v[u] >= nx[u]);
        const unsigned long long ik = (unsigned long long)v[u] ^ 0x8000000000000000ull;
        imn = ik < imn ? ik : imn;
        imx = ik > imx ? ik : imx;
      }
    }
  }
  mnx = shfl_min64(mnx);
  mny = shfl_min64(mny);
  mxx = shfl_max64(mxx);
  mxy = shfl_max64(mxy);
  imn = shfl_min64(imn);
  imx = shfl_max64(imx);
  if (lane_id() == 0) {
    atomicMin(&h->kmin_x, mnx);
    atomicMin(&h->kmin_y, mny);
    atomicMax(&h->kmax_x, mxx);
    atomicMax(&h->kmax_y, mxy);
    atomicMin(&h->id_kmin, imn);
    atomicMax(&h->id_kmax, imx);
  }
  if (__any_sync(0xffffffffu, bad) && lane_id() == 0) atomicOr(&h->not_monotone, 1);
  if (__any_sync(0xffffffffu, notid) && lane_id() == 0) atomicOr(&h->not_identity, 1);
}

__global__ void k_finalize_mbr(DevHdr* h) {
  // geometry.py:72-77 (exact min/max) and morton.py:100-104 scale factors
  if (h->reuse_index) return;  // adaptive reuse keeps the index MBR
  h->xa = dunkey(h->kmin_x);
  h->ya = dunkey(h->kmin_y);
  h->xb = dunkey(h->kmax_x);
  h->yb = dunkey(h->kmax_y);
  h->width = __dsub_rn(h->xb, h->xa);
  h->height = __dsub_rn(h->yb, h->ya);
  h->wpos = h->width > 0.0;
  h->hpos = h->height > 0.0;
  // quadtree: 2^l_max cells per side; uniform grid: split_factor (grid.py:39-46)
  const double side = h->grid_sf ? (double)h->grid_sf : (double)(1u << h->l_max);
  h->sx_max = h->wpos ? __ddiv_rn(side, h->width) : 0.0;
  h->sy_max = h->hpos ? __ddiv_rn(side, h->height) : 0.0;
  for (int l = 0; l <= kMaxLevel; ++l) {
    h->lw[l] = __ddiv_rn(h->width, (double)(1u << l));
    h->lh[l] = __ddiv_rn(h->height, (double)(1u << l));
  }
  if (h->grid_sf) {  // the grid's cells are the leaves of level l_max: cell_w = width / split_factor
    h->lw[h->l_max] = __ddiv_rn(h->width, (double)h->grid_sf);
    h->lh[h->l_max] = __ddiv_rn(h->height, (double)h->grid_sf);
  }
}

// ===========================================================================
// K1: index build
// ===========================================================================
// l_max codes (morton.py:90-109 + interleave) and the level-F histogram with
// warp-aggregated atomics (one atomic per distinct bin per warp).
__global__ void __launch_bounds__(256) k_codes(const Dev d) {
  DevHdr* h = d.h;
  const int64_t n = h->n;
  const int lmax = h->l_max, F = h->F;
  const uint32_t side = h->grid_sf ? (uint32_t)h->grid_sf : 1u << lmax;
  const double xa = h->xa, ya = h->ya, sx = h->sx_max, sy = h->sy_max;
  const int wpos = h->wpos, hpos = h->hpos;
  const int sh = 2 * (lmax - F);
  uint32_t* hist = d.pyr + pyr_off(F);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += 4 * stride) {
    double x[4], y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * stride;
      x[u] = i < n ? d.xs[i] : 0.0;
      y[u] = i < n ? d.ys[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) {
        const uint32_t z = morton2(cell_of(x[u], xa, sx, wpos, side), cell_of(y[u], ya, sy, hpos, side));
        d.code[i] = z;
        if (!(h->dbg & 4)) atomicAdd(&hist[z >> sh], 1u);  // level-F histogram (fire-and-forget reductions)
      }
    }
  }
}

__device__ __forceinline__ void note_split(DevHdr* h, bool split, int next_level) {
  const unsigned any = __ballot_sync(0xffffffffu, split);
  if (any && lane_id() == (__ffs(any) - 1)) atomicMax(&h->l_deep, next_level);
}

// dense level l from level l+1 (quadtree.py:111-116: a node at level l splits
// iff count > th_quad and l < l_max; l_deep = deepest level with leaves)
__global__ void __launch_bounds__(256) k_pyr_level(const Dev d, int l) {
  DevHdr* h = d.h;
  const int64_t cnt = int64_t(1) << (2 * l);
  const uint32_t* child = d.pyr + pyr_off(l + 1);
  uint32_t* self = d.pyr + pyr_off(l);
  const uint32_t th = (uint32_t)h->th;
  const bool can_split = l >= 1 && l < h->l_max;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x; b < cnt; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = b + threadIdx.x;
    bool split = false;
    if (z < cnt) {
      const uint4 c = *reinterpret_cast<const uint4*>(child + 4 * z);
      const uint32_t s = c.x + c.y + c.z + c.w;
      self[z] = s;
      split = can_split && s > th;
    }
    note_split(h, split, l + 1);
  }
}

// Levels hi-1 .. lo of the dense pyramid in one launch: CTA b owns node b of
// level lo and sums its subtree upward from level hi (4^(hi-lo) <= 4096
// children staged through shared memory), writing every level it computes and
// noting splits like k_pyr_level (12 launches become 2 at l_max 12).
constexpr int kPyrSpan = 6;  // levels per fused launch
__global__ void __launch_bounds__(256) k_pyr_fused(const Dev d, int lo, int hi) {
  DevHdr* h = d.h;
  __shared__ uint32_t buf[2][1024];
  const uint32_t th = (uint32_t)h->th;
  const int64_t node = blockIdx.x;  // at level lo
  int deep = 0;  // deepest level a split of this thread's nodes creates (one atomic per warp at the end)
  // level hi-1 from the global level hi: every child load issued before any is used
  {
    constexpr int kIt = 4;  // level-(hi-1) nodes per thread: 4^(kPyrSpan-1) <= 4 * 256
    const int l = hi - 1;
    const int per = 1 << (2 * (l - lo));  // level-l nodes under this CTA's node
    const uint32_t* child = d.pyr + pyr_off(hi);
    uint32_t* self = d.pyr + pyr_off(l);
    const bool can_split = l >= 1 && l < h->l_max;
    uint4 c[kIt];
#pragma unroll
    for (int it = 0; it < kIt; ++it) {
      const int k = it * 256 + threadIdx.x;
      c[it] = k < per ? *reinterpret_cast<const uint4*>(child + 4 * (node * per + k)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int it = 0; it < kIt; ++it) {
      const int k = it * 256 + threadIdx.x;
      if (k < per) {
        const uint32_t sum = c[it].x + c[it].y + c[it].z + c[it].w;
        self[node * per + k] = sum;
        buf[(hi - 1 - lo) & 1][k] = sum;
        if (can_split && sum > th) deep = max(deep, l + 1);
      }
    }
  }
  __syncthreads();
  for (int l = hi - 2; l >= lo; --l) {
    const int64_t per = int64_t(1) << (2 * (l - lo));
    const uint32_t* src = buf[(l + 1 - lo) & 1];
    uint32_t* dst = buf[(l - lo) & 1];
    uint32_t* self = d.pyr + pyr_off(l);
    const bool can_split = l >= 1 && l < h->l_max;
    for (int64_t k = threadIdx.x; k < per; k += blockDim.x) {
      const uint32_t sum = src[4 * k] + src[4 * k + 1] + src[4 * k + 2] + src[4 * k + 3];
      self[node * per + k] = sum;
      dst[k] = sum;
      if (can_split && sum > th) deep = max(deep, l + 1);
    }
    __syncthreads();
  }
  deep = __reduce_max_sync(0xffffffffu, deep);
  if (lane_id() == 0 && deep > *(volatile int*)&h->l_deep) atomicMax(&h->l_deep, deep);
}

__global__ void k_finalize_index(DevHdr* h) {
  if (h->abort) return;
  h->Z = int64_t(1) << (2 * h->l_deep);
  h->side_deep = h->grid_sf ? (uint32_t)h->grid_sf : 1u << h->l_deep;
  const double side = (double)h->side_deep;
  h->sx_deep = h->wpos ? __ddiv_rn(side, h->width) : 0.0;
  h->sy_deep = h->hpos ? __ddiv_rn(side, h->height) : 0.0;
}

// object count of node (l, z); l >= 1
__device__ __forceinline__ uint32_t node_count(const Dev& d, int F, int l, uint32_t z) {
  (void)F;  // F == l_max: the dense pyramid covers every level
  return d.pyr[pyr_off(l) + z];
}

// Level of the leaf containing deepest cell c: the first level whose ancestor
// does not split (count <= th, or l_max).  Equivalent to the reference's
// level-wise construction (quadtree.py:106-127): a quadrant exists iff its
// parent split, and counts are monotone along the root path.
__global__ void __launch_bounds__(256) k_cell_level(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t Z = h->Z;
  const int ld = h->l_deep, lmax = h->l_max, F = h->F;
  const uint32_t th = (uint32_t)h->th;
  TJ_GRID_STRIDE(c, Z) {
    // (loading every ancestor's count at once measured slower: most cells stop well above l_deep)
    int lev = ld;
    for (int l = 1; l <= ld; ++l) {
      const uint32_t cnt = node_count(d, F, l, (uint32_t)(c >> (2 * (ld - l))));
      if (cnt <= th || l == lmax) {
        lev = l;
        break;
      }
    }
    d.clev[c] = (uint8_t)lev;
  }
}

// ---- adaptive rebuild (rebuild="adaptive": quadtree.py:243-270, engine.py:163-174)
// The previous tick's index is reused unless needs_rebuild: an object outside
// the old MBR (OutOfBounds, morton.py:98-99), any leaf holding more than
// 8 x th_quad objects, or more than 5% of the leaves holding more than
// 2 x th_quad.  The check recounts the old leaves from the dense pyramid of
// this tick's codes, taken at the old index's scale.
__global__ void k_reuse_oob(DevHdr* h) {
  const bool out = dunkey(h->kmin_x) < h->xa || dunkey(h->kmax_x) > h->xb || dunkey(h->kmin_y) < h->ya ||
                   dunkey(h->kmax_y) > h->yb;
  if (out) h->oob = 1;
}

__global__ void __launch_bounds__(256) k_leaf_recount(const Dev d) {
  DevHdr* h = d.h;
  const uint32_t th = (uint32_t)h->th;
  unsigned long long o2 = 0, o8 = 0;
  TJ_GRID_STRIDE(r, h->L) {
    const uint32_t code = d.leaf_code[r];
    const uint32_t cnt = node_count(d, h->F, (int)(code >> kLevelShift), code & kPayloadMask);
    d.leaf_nobj[r] = (int32_t)cnt;
    o2 += cnt > 2u * th;
    o8 += cnt > 8u * th;
  }
  o2 = warp_sum(o2);
  o8 = warp_sum(o8);
  if (lane_id() == 0) {
    if (o2) atomicAdd(&h->overfull2, o2);
    if (o8) atomicAdd(&h->overfull8, o8);
  }
}

struct ZFlagIn {
  const uint8_t* clev;
  const DevHdr* h;
  __device__ int64_t operator()(int64_t c) const {
    const int lev = clev[c];
    const int64_t span_mask = (int64_t(1) << (2 * (h->l_deep - lev))) - 1;
    return (c & span_mask) == 0 ? 1 : 0;
  }
};

// zmap entry: (leaf level << 24) | leaf rank (leaves ranked in Morton order);
// leaf table: code (level << 24 | z) and object count.  quadtree.py:142-158
struct ZOut {
  Dev d;
  __device__ void operator()(int64_t c, int64_t ex, int64_t v) const {
    const DevHdr* h = d.h;
    const int lev = d.clev[c];
    const int64_t rank = ex + v - 1;
    d.zmap[c] = ((uint32_t)lev << kLevelShift) | (uint32_t)rank;
    if (v && rank < h->cap_L) {
      const uint32_t z = (uint32_t)(c >> (2 * (h->l_deep - lev)));
      d.leaf_code[rank] = ((uint32_t)lev << kLevelShift) | z;
      d.leaf_nobj[rank] = (int32_t)node_count(d, h->F, lev, z);
    }
  }
};

// The zmap scan specialised (the generic scan moves 8-byte values through a
// shared-memory tile per cell): 16 consecutive cells per thread, their levels in
// one 16-byte load, leaf starts as a 16-bit mask, int32 block scan of the
// masks' popcounts, the 16 zmap entries as four 16-byte stores.  Two passes
// (starts per block, then ranks) around k_scan_partials; blocks own contiguous
// chunks of whole 4096-cell tiles.
constexpr int kZPer = 16, kZTile = 256 * kZPer;
__device__ __forceinline__ void zmap_chunk(int64_t Z, int64_t* b, int64_t* e) {
  const int64_t chunk = ((Z + gridDim.x - 1) / gridDim.x + kZTile - 1) / kZTile * kZTile;
  *b = (int64_t)blockIdx.x * chunk;
  *e = *b + chunk < Z ? *b + chunk : Z;
}
// leaf-start mask of cells c0 .. c0+15 (bit k: cell c0+k is the first deepest cell of its leaf) and their levels
__device__ __forceinline__ uint32_t zmap_starts(const uint8_t* clev, int64_t c0, int64_t e, int ld, uint8_t lv[kZPer]) {
  if (c0 + kZPer <= e) {
    const uint4 q = *reinterpret_cast<const uint4*>(clev + c0);
    const uint32_t wds[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int k = 0; k < kZPer; ++k) lv[k] = (uint8_t)(wds[k >> 2] >> (8 * (k & 3)));
  } else {
#pragma unroll
    for (int k = 0; k < kZPer; ++k) lv[k] = c0 + k < e ? clev[c0 + k] : (uint8_t)ld;
  }
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < kZPer; ++k) {
    const int64_t span_mask = (int64_t(1) << (2 * (ld - lv[k]))) - 1;
    m |= (c0 + k < e && ((c0 + k) & span_mask) == 0) ? (1u << k) : 0u;
  }
  return m;
}

// k_cell_level for an aligned group of 16 deepest cells (l_deep >= 2): they share
// every ancestor down to level l_deep - 2, so that part of the walk is done once;
// level l_deep - 1 has four ancestors; at l_deep the walk ends anyway.
__device__ __forceinline__ void group_levels(const Dev& d, int64_t c0, int ld, int lmax, uint32_t th,
                                             uint8_t lv[kZPer]) {
  int lev = 0;
  for (int l = 1; l <= ld - 2; ++l) {
    const uint32_t cnt = node_count(d, 0, l, (uint32_t)(c0 >> (2 * (ld - l))));
    if (cnt <= th || l == lmax) {
      lev = l;
      break;
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int lj = lev;
    if (!lev) {
      const uint32_t cnt = node_count(d, 0, ld - 1, (uint32_t)(c0 >> 2) + j);
      lj = (cnt <= th || ld - 1 == lmax) ? ld - 1 : ld;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) lv[4 * j + i] = (uint8_t)lj;
  }
}

// kLevels: compute the cells' leaf levels from the pyramid and store them (the
// quadtree; fused k_cell_level); otherwise read them (the uniform grid's).
template <bool kLevels>
__global__ void __launch_bounds__(256) k_zmap_count(const Dev d, int64_t* partial) {
  DevHdr* h = d.h;
  if (h->abort) return;
  __shared__ int64_t sh[33];
  int64_t b, e;
  zmap_chunk(h->Z, &b, &e);
  const int ld = h->l_deep, lmax = h->l_max;
  const uint32_t th = (uint32_t)h->th;
  int64_t cnt = 0;
  for (int64_t base = b; base < e; base += kZTile) {
    const int64_t c0 = base + threadIdx.x * kZPer;
    if (kLevels && c0 < e) {
      uint8_t lv[kZPer];
      if (ld >= 2) {  // Z = 4^ld is a multiple of 16: whole groups
        group_levels(d, c0, ld, lmax, th, lv);
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          w[k] = (uint32_t)lv[4 * k] | ((uint32_t)lv[4 * k + 1] << 8) | ((uint32_t)lv[4 * k + 2] << 16) |
                 ((uint32_t)lv[4 * k + 3] << 24);
        *reinterpret_cast<uint4*>(d.clev + c0) = make_uint4(w[0], w[1], w[2], w[3]);
      } else {  // a single-level tree: the per-cell walk
        for (int64_t c = c0; c < c0 + kZPer && c < e; ++c) {
          int lev = ld;
          for (int l = 1; l <= ld; ++l) {
            const uint32_t n = node_count(d, 0, l, (uint32_t)(c >> (2 * (ld - l))));
            if (n <= th || l == lmax) {
              lev = l;
              break;
            }
          }
          d.clev[c] = (uint8_t)lev;
        }
      }
    }
    uint8_t lv[kZPer];
    cnt += __popc(zmap_starts(d.clev, c0, e, ld, lv));
  }
  cnt = warp_sum(cnt);
  if (lane_id() == 0) sh[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x < 32) {
    int64_t v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0;
    v = warp_sum(v);
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
  }
}

__global__ void __launch_bounds__(256) k_zmap_rank(const Dev d, const int64_t* partial) {
  DevHdr* h = d.h;
  if (h->abort) return;
  __shared__ int32_t sh[33];
  int64_t b, e;
  zmap_chunk(h->Z, &b, &e);
  const int ld = h->l_deep;
  int64_t carry = partial[blockIdx.x];
  for (int64_t base = b; base < e; base += kZTile) {
    const int64_t c0 = base + threadIdx.x * kZPer;
    uint8_t lv[kZPer];
    const uint32_t m = zmap_starts(d.clev, c0, e, ld, lv);
    int32_t tot;
    const int64_t ex = carry + block_excl_scan((int32_t)__popc(m), sh, &tot);
    uint32_t z[kZPer];
#pragma unroll
    for (int k = 0; k < kZPer; ++k) {
      const int64_t rank = ex + __popc(m & ((2u << k) - 1u)) - 1;  // leaf starts at or before the cell, less one
      z[k] = ((uint32_t)lv[k] << kLevelShift) | (uint32_t)rank;
      if (((m >> k) & 1u) && rank < h->cap_L) {
        const uint32_t zc = (uint32_t)((c0 + k) >> (2 * (ld - lv[k])));
        d.leaf_code[rank] = ((uint32_t)lv[k] << kLevelShift) | zc;
        d.leaf_nobj[rank] = (int32_t)node_count(d, h->F, lv[k], zc);
      }
    }
    if (c0 + kZPer <= e) {
      uint4* dst = reinterpret_cast<uint4*>(d.zmap + c0);
#pragma unroll
      for (int k = 0; k < kZPer / 4; ++k) dst[k] = make_uint4(z[4 * k], z[4 * k + 1], z[4 * k + 2], z[4 * k + 3]);
    } else {
#pragma unroll
      for (int k = 0; k < kZPer; ++k)
        if (c0 + k < e) d.zmap[c0 + k] = z[k];
    }
    carry += tot;
  }
}

// TJ_CHECK_TILING=1: the reference's internal check of build_zmap (quadtree.py:153-157) on the
// device — leaves in Morton order must tile the 4^l_deep deepest cells without gaps or overlaps
// (each leaf at level l spans 4^(l_deep - l) cells starting at z * span).  Holds by construction;
// a debug check, off by default.
__global__ void __launch_bounds__(256) k_check_tiling(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t L = h->L, Z = h->Z;
  const int ld = h->l_deep;
  int gap = L == 0;
  TJ_GRID_STRIDE(r, L) {
    const uint32_t code = d.leaf_code[r];
    const int lev = (int)(code >> kLevelShift);
    const int64_t span = int64_t(1) << (2 * (ld - lev));
    const int64_t start = (int64_t)(code & kPayloadMask) * span;
    if (r == 0 && start != 0) gap = 1;
    if (r + 1 < L) {
      const uint32_t nc = d.leaf_code[r + 1];
      const int nl = (int)(nc >> kLevelShift);
      if ((int64_t)(nc & kPayloadMask) * (int64_t(1) << (2 * (ld - nl))) != start + span) gap = 1;
    } else if (start + span != Z) {
      gap = 1;
    }
  }
  if (__any_sync(0xffffffffu, gap) && lane_id() == 0) atomicOr(&h->tiling_gap, 1);
}

// object -> leaf rank (quadtree.py:161-165) as the radix key; the value of
// the first radix pass is the input row itself (implicit)
__global__ void __launch_bounds__(256) k_obj_keys(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t n = h->n;
  const int sh = 2 * (h->l_max - h->l_deep);
  const bool keyed = h->key_sorted;  // keyed lists: the objects enter the stable leaf sort in id order
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j0 < n; j0 += 4 * stride) {
    uint32_t cd[4];  // four code -> zmap chains in flight
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = j0 + u * stride;
      cd[u] = j < n ? d.code[keyed ? d.order[j] : j] : 0u;
    }
    uint32_t z[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) z[u] = j0 + u * stride < n ? d.zmap[cd[u] >> sh] : 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j0 + u * stride < n) d.okey[0][j0 + u * stride] = z[u] & kPayloadMask;
  }
}

// Sharded ticks (§8e): only the objects in this rank's leaves are sorted.  A
// scan over the objects (in input order, or id order for keyed lists) flags
// those whose leaf is owned and compacts their leaf keys and rows, in order, so
// the stable sort sees them as the unsharded sort would.
struct OwnObjIn {
  Dev d;
  __device__ int64_t operator()(int64_t j) const {
    const DevHdr* h = d.h;
    const int32_t row = h->key_sorted ? d.order[j] : (int32_t)j;
    const uint32_t leaf = d.zmap[d.code[row] >> (2 * (h->l_max - h->l_deep))] & kPayloadMask;
    return d.leaf_active[leaf] ? 1 : 0;
  }
};
struct OwnObjOut {
  Dev d;
  __device__ void operator()(int64_t j, int64_t ex, int64_t v) const {
    if (!v) return;
    const DevHdr* h = d.h;
    const int32_t row = h->key_sorted ? d.order[j] : (int32_t)j;
    d.okey[0][ex] = d.zmap[d.code[row] >> (2 * (h->l_max - h->l_deep))] & kPayloadMask;
    d.crow[ex] = row;
  }
};
// leaf object counts of own leaves only (the compacted blocks' bases)
struct OwnNobjIn {
  const int32_t* nobj;
  const uint8_t* active;
  __device__ int64_t operator()(int64_t r) const { return active[r] ? nobj[r] : 0; }
};

// ---- keyed lists (object ids that are not the input rows) ------------------
// The reference sorts every result list by id (decode.py:117, np.sort in
// merge_results).  When ids are not the rows, the device instead keeps every
// leaf block in id order and stores each block position's id as a 32-bit
// offset from the smallest id (loff): every run of a query is then id-sorted,
// and the decode merges runs of offsets exactly like the monotone path merges
// runs of rows, reading them leaf-locally.  Ids that do not increase with the
// row are put in id order by a counting sort over a presence bitmap of the
// offsets (one bit per possible id: rank = popcounts below it), and the stable
// leaf sort then takes the objects in that order.  Eligible when the ids'
// range is below 2^28 (the bitmap; the decode's packed merge heads) and, for
// non-increasing ids, no two objects share an id (set bits == n); otherwise
// lists are sorted per query (k_merge_big, which raises DuplicateResult).
// Within a leaf the reference keeps input order (directory.py:128); the
// introspection entry points restore it.
constexpr int kKeyBits = 28;
__global__ void k_key_decide(DevHdr* h) {
  h->key_mode = 0;
  h->key_sorted = 0;
  h->pres_words = 0;
  if (h->abort || !h->key_req || !h->not_identity || h->n == 0) return;
  if (((h->id_kmax - h->id_kmin) >> kKeyBits) != 0) return;
  h->id_min = (int64_t)(h->id_kmin ^ 0x8000000000000000ull);
  h->key_mode = 1;
  if (h->not_monotone) h->pres_words = (int64_t)((h->id_kmax - h->id_kmin) >> 5) + 1;
}

__global__ void __launch_bounds__(256) k_key_zero(const Dev d) {
  DevHdr* h = d.h;
  TJ_GRID_STRIDE(w, h->pres_words) d.presence[w] = 0u;
}
__global__ void __launch_bounds__(256) k_key_presence(const Dev d) {
  DevHdr* h = d.h;
  if (!h->pres_words) return;
  const int64_t id_min = h->id_min;
  TJ_GRID_STRIDE(i, h->n) {
    const uint32_t off = (uint32_t)(d.ids[i] - id_min);
    atomicOr(&d.presence[off >> 5], 1u << (off & 31));  // no return value: reductions
  }
}
struct PopIn {
  const uint32_t* w;
  __device__ int64_t operator()(int64_t i) const { return __popc(w[i]); }
};
__global__ void k_key_close(DevHdr* h) {
  if (!h->pres_words) return;
  if (h->pres_total != h->n) {  // a shared id: per-list sorts (and DuplicateResult where a list has both)
    h->dup_ids = 1;
    h->key_mode = 0;
    return;
  }
  h->key_sorted = 1;
}
// id rank of every object (popcounts of the presence bits below its id): order[rank] = row
__global__ void __launch_bounds__(256) k_key_order(const Dev d) {
  DevHdr* h = d.h;
  if (!h->key_sorted) return;
  const int64_t id_min = h->id_min;
  TJ_GRID_STRIDE(i, h->n) {
    const uint32_t off = (uint32_t)(d.ids[i] - id_min);
    const uint32_t w = off >> 5;
    const int32_t rank = d.pres_pre[w] + __popc(d.presence[w] & ((1u << (off & 31)) - 1u));
    d.order[rank] = (int32_t)i;
  }
}
// every leaf position's id offset, after the leaf sort
__global__ void __launch_bounds__(256) k_key_loff(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort || !h->key_mode) return;
  const int64_t n = h->n_sort, id_min = h->id_min;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < n; p0 += 4 * stride) {
    int32_t r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) r[u] = p0 + u * stride < n ? d.sidx[p0 + u * stride] : 0;
    int64_t v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = p0 + u * stride < n ? __ldcg(reinterpret_cast<const long long*>(d.ids) + r[u]) : 0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (p0 + u * stride < n) d.loff[p0 + u * stride] = (uint32_t)(v[u] - id_min);
  }
}

// Payload gather into leaf order, one array per launch: each launch's random
// reads hit one 80 MB array (at 10M objects) that can stay L2-resident,
// instead of two arrays (160 MB) thrashing the 126 MB L2 together.
template <typename T>
__global__ void __launch_bounds__(256) k_gather(const Dev d, const T* __restrict__ src, T* __restrict__ dst) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t n = h->n_sort;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < n; p0 += 4 * stride) {
    int32_t r[4];  // four independent gathers in flight per thread
#pragma unroll
    for (int u = 0; u < 4; ++u) r[u] = p0 + u * stride < n ? d.sidx[p0 + u * stride] : 0;
    T v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = p0 + u * stride < n ? __ldcg(src + r[u]) : T(0);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (p0 + u * stride < n) __stcs(dst + p0 + u * stride, v[u]);
  }
}

// checks after a size became known: abort bits make the rest of the tick a no-op
__global__ void k_check_caps(DevHdr* h, int stage, int radix_bits_obj, int radix_bits_sq) {
  if (stage == 0) {  // after leaves
    if (h->L > h->cap_L) atomicOr(&h->abort, 16);
    if (radix_bits_obj < 32 && (h->L - 1) >> radix_bits_obj) atomicOr(&h->abort, 32);
    if (radix_bits_sq < 32 && (2 * h->L - 1) >> radix_bits_sq) atomicOr(&h->abort, 32);
  } else if (stage == 1) {
    if (h->S > h->cap_S) atomicOr(&h->abort, 1);
  } else if (stage == 2) {
    if (h->W > h->cap_W || h->U > h->cap_U) atomicOr(&h->abort, 2);
    if (h->W >= (int64_t)0xffffffffll) atomicOr(&h->abort, 64);  // the decode's 32-bit word offsets
  } else if (stage == 3) {
    if (h->R > h->cap_R) atomicOr(&h->abort, 4);
  }
}

// ===========================================================================
// K2: query -> leaf scatter
// ===========================================================================
// Enumerate every leaf intersecting the deepest-cell window exactly once:
// depth-first from the smallest quadrant containing the window, stopping at a
// quadrant whose first deepest cell belongs to a leaf no deeper than it
// (the emission rule of quadtree.py:204-208).
template <typename Emit>
__device__ __forceinline__ int enum_window(int i0, int i1, int j0, int j1, int ld, const uint32_t* zmap,
                                           Emit emit) {
  const uint32_t diff = (uint32_t)((i0 ^ i1) | (j0 ^ j1));
  const int lc = ld - (diff ? 32 - __clz(diff) : 0);
  uint32_t stk[3 * kMaxLevel + 4];
  int sp = 0;
  stk[sp++] = ((uint32_t)lc << 24) | ((uint32_t)(i0 >> (ld - lc)) << 12) | (uint32_t)(j0 >> (ld - lc));
  int cnt = 0;
  while (sp) {
    const uint32_t e = stk[--sp];
    const int l = (int)(e >> 24);
    const uint32_t ni = (e >> 12) & 0xFFFu, nj = e & 0xFFFu;
    const int s = ld - l;
    const uint32_t c0 = morton2(ni << s, nj << s);
    const uint32_t zz = zmap[c0];
    const int lev = (int)(zz >> kLevelShift);
    if (lev <= l) {
      emit(lev, c0 >> (2 * (ld - lev)), zz & kPayloadMask);
      ++cnt;
      continue;
    }
    const int cs = s - 1;
#pragma unroll
    for (int c = 3; c >= 0; --c) {
      const int ci = (int)((ni << 1) | (uint32_t)(c & 1)), cj = (int)((nj << 1) | (uint32_t)(c >> 1));
      const int lo_i = ci << cs, hi_i = ((ci + 1) << cs) - 1;
      const int lo_j = cj << cs, hi_j = ((cj + 1) << cs) - 1;
      if (lo_i <= i1 && hi_i >= i0 && lo_j <= j1 && hi_j >= j0)
        stk[sp++] = ((uint32_t)(l + 1) << 24) | ((uint32_t)ci << 12) | (uint32_t)cj;
    }
  }
  return cnt;
}

// Windows of at most 2x2 deepest cells (every query of configs A-C): probe
// the cells directly — four independent zmap loads instead of a walk.  A leaf
// is emitted at its first cell inside the window, so each intersected leaf
// appears once; entries come back sorted by packed (level, z).
__device__ __forceinline__ bool is_small(const int4 w) { return w.y - w.x <= 1 && w.w - w.z <= 1; }

#define TJ_CSWAP(a, b)                                  \
  if (key[b] < key[a]) {                                \
    uint32_t tk = key[a]; key[a] = key[b]; key[b] = tk; \
    uint32_t tr = rank[a]; rank[a] = rank[b]; rank[b] = tr; \
  }

__device__ __forceinline__ int enum_small(const int4 w, int ld, const uint32_t* zmap, uint32_t key[4],
                                          uint32_t rank[4]) {
  uint32_t e[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int ci = w.x + (k & 1), cj = w.z + (k >> 1);
    e[k] = (ci <= w.y && cj <= w.w) ? zmap[morton2(ci, cj)] : 0xFFFFFFFFu;
  }
  int n = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int ci = w.x + (k & 1), cj = w.z + (k >> 1);
    key[k] = 0xFFFFFFFFu;
    rank[k] = 0;
    if (e[k] != 0xFFFFFFFFu) {
      const int lev = (int)(e[k] >> kLevelShift), sh = ld - lev;
      const int li0 = (ci >> sh) << sh, lj0 = (cj >> sh) << sh;
      if (max(li0, w.x) == ci && max(lj0, w.z) == cj) {
        key[k] = ((uint32_t)lev << kLevelShift) | (morton2(ci, cj) >> (2 * sh));
        rank[k] = e[k] & kPayloadMask;
        ++n;
      }
    }
  }
  TJ_CSWAP(0, 1) TJ_CSWAP(2, 3) TJ_CSWAP(0, 2) TJ_CSWAP(1, 3) TJ_CSWAP(1, 2)
  return n;
}
#undef TJ_CSWAP

// Covering flag with the reference's exact op order (quadtree.py:219-231):
// w = width / 2^level; lxa = xa + li*w; covering iff qxa <= lxa and
// qxb >= min(lxa + w, mbr.xb), likewise in y.
__device__ __forceinline__ bool covers(const Rect4& q, int lev, uint32_t z, const DevHdr* h) {
  const double w = h->lw[lev];
  const double hh = h->lh[lev];
  const double li = (double)compact2(z), lj = (double)compact2(z >> 1);
  const double lxa = __dadd_rn(h->xa, __dmul_rn(li, w));
  const double lya = __dadd_rn(h->ya, __dmul_rn(lj, hh));
  double ux = __dadd_rn(lxa, w);
  ux = ux < h->xb ? ux : h->xb;
  double uy = __dadd_rn(lya, hh);
  uy = uy < h->yb ? uy : h->yb;
  return (q.xa <= lxa) && (q.xb >= ux) && (q.ya <= lya) && (q.yb >= uy);
}

// Clip (geometry.py:80-88: max/min against the index MBR) and the deepest-
// cell window of the clipped rect (quadtree.py:182-183).  Both scatter passes
// recompute it from the input rect (cheaper than storing and re-reading it).
// Returns false for a query disjoint from the MBR.
__device__ __forceinline__ bool clip_window(const Dev& d, int64_t q, double xa, double ya, double xb, double yb,
                                            double sx, double sy, int wpos, int hpos, uint32_t side, Rect4& r,
                                            int4& w) {
  double cxa = d.qxa[q], cya = d.qya[q], cxb = d.qxb[q], cyb = d.qyb[q];
  cxa = cxa < xa ? xa : cxa;  // max(q.xa, mbr.xa)
  cya = cya < ya ? ya : cya;
  cxb = cxb > xb ? xb : cxb;  // min(q.xb, mbr.xb)
  cyb = cyb > yb ? yb : cyb;
  r.xa = cxa; r.ya = cya; r.xb = cxb; r.yb = cyb;
  w = make_int4(-1, -1, -1, -1);
  if (cxa > cxb || cya > cyb) return false;
  w.x = (int)cell_of(cxa, xa, sx, wpos, side);
  w.y = (int)cell_of(cxb, xa, sx, wpos, side);
  w.z = (int)cell_of(cya, ya, sy, hpos, side);
  w.w = (int)cell_of(cyb, ya, sy, hpos, side);
  return true;
}

// Counting sort of the (query, leaf) pairs into per-leaf directory blocks
// (directory.py:119-158), two passes over the queries:
//  count: every pair bumps its leaf's intersecting or covering counter.  A
//    small window (<= 2x2 deepest cells, every query of configs A-C keeps
//    the counter's old value — its place in the block — for the fill;
//  fill: (after a scan of the block sizes) a small-window pair lands at that
//    place with no further atomics; pairs of larger windows take places after
//    the small ones from a cursor.
// Within a block, entries are in this (unordered) fill order; the join and
// the decode are invariant to it and the introspection entry points return
// the reference's query order (directory.py:131).
__device__ __forceinline__ bool pair_cov(const Dev& d, int lev, uint32_t z, const Rect4& r, int cov_on) {
  return cov_on && covers(r, lev, z, d.h);
}

// clip (geometry.py:80-88), window (quadtree.py:182-183), count subqueries
// per query and (query, leaf) pairs per leaf block
__global__ void __launch_bounds__(256) k_query_count(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t m = h->m;
  const double xa = h->xa, ya = h->ya, xb = h->xb, yb = h->yb;
  const double sx = h->sx_deep, sy = h->sy_deep;
  const int wpos = h->wpos, hpos = h->hpos, ld = h->l_deep;
  const uint32_t side = h->side_deep;
  const int cov_on = h->covering;
  TJ_GRID_STRIDE(q, m) {
    Rect4 r;
    int4 w;
    int cnt = 0;
    if (clip_window(d, q, xa, ya, xb, yb, sx, sy, wpos, hpos, side, r, w)) {
      if (is_small(w)) {
        uint32_t key[4], rank[4];
        const int ne = enum_small(w, ld, d.zmap, key, rank);
        int pos[4] = {0, 0, 0, 0};
        uint32_t rc[4] = {0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k < ne && leaf_on(d.leaf_active, rank[k])) {
            const bool cv = pair_cov(d, (int)(key[k] >> kLevelShift), key[k] & kPayloadMask, r, cov_on);
            int4* c = d.leaf_cnt + rank[k];
            const int v = atomicAdd(cv ? &c->y : &c->x, 1);  // owned pairs, in order
            const uint32_t packed = rank[k] | (cv ? 0x80000000u : 0u);
#pragma unroll
            for (int j = 0; j < 4; ++j) {  // (no local-memory indexing)
              pos[j] = (j == cnt) ? v : pos[j];
              rc[j] = (j == cnt) ? packed : rc[j];
            }
            ++cnt;
          }
        // the fill needs no window walk for these: their leaves (covering flag in bit 31) and places
        d.qpos[q] = make_int4(pos[0], pos[1], pos[2], pos[3]);
        w = make_int4((int)rc[0], (int)rc[1], (int)rc[2], (int)rc[3]);
      } else {
        d.qpos[q] = make_int4(-1, 0, 0, 0);  // a window the fill walks again
        enum_window(w.x, w.y, w.z, w.w, ld, d.zmap, [&](int lev, uint32_t z, uint32_t rank) {
          if (!leaf_on(d.leaf_active, rank)) return;
          int4* c = d.leaf_cnt + rank;
          atomicAdd(pair_cov(d, lev, z, r, cov_on) ? &c->w : &c->z, 1);
          ++cnt;
        });
      }
    }
    d.nsub[q] = cnt;
    d.qwin[q] = w;
  }
}


__device__ __forceinline__ void emit_subquery(const Dev& d, int32_t slot, uint32_t rank, int32_t e, const Rect4& r) {
  d.sq_le[slot] = make_int2((int32_t)rank, e);  // one 8-byte store
  d.erect[e] = r;  // the join's input, in entry order
}

// Fill: per query, subqueries in ascending packed (level, z) order — the
// depth-first walk yields z-ascending order within each level, so a per-level
// counting placement gives the reference's order (quadtree.py:194-217).
__global__ void __launch_bounds__(256) k_query_fill(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t m = h->m;
  const int ld = h->l_deep;
  const int cov_on = h->covering;
  const double xa = h->xa, ya = h->ya, xb = h->xb, yb = h->yb;
  TJ_GRID_STRIDE(q, m) {
    const int n = d.nsub[q];
    if (n == 0) continue;
    // the clip again (geometry.py:80-88): re-reading the query costs what reading a stored clip
    // would, and the count pass then writes no per-query rect.  (Prefetching the next query's
    // count, rect and handoff while placing this one's pairs measured 6% slower: 64 registers.)
    Rect4 r;
    r.xa = d.qxa[q];
    r.ya = d.qya[q];
    r.xb = d.qxb[q];
    r.yb = d.qyb[q];
    r.xa = r.xa < xa ? xa : r.xa;  // exactly clip_window's max / min
    r.ya = r.ya < ya ? ya : r.ya;
    r.xb = r.xb > xb ? xb : r.xb;
    r.yb = r.yb > yb ? yb : r.yb;
    const int4 p4 = d.qpos[q];
    const int4 w = d.qwin[q];  // small window: its leaves as found by the count pass; else the window
    const int32_t base = d.qsbase[q];
    if (p4.x >= 0) {
      const uint32_t rc[4] = {(uint32_t)w.x, (uint32_t)w.y, (uint32_t)w.z, (uint32_t)w.w};
      const int pos[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < n) {
          const uint32_t rank = rc[k] & 0x7fffffffu;
          const bool cv = (rc[k] >> 31) != 0;
          const int4 c = d.leaf_cnt[rank];
          const int32_t e = d.leaf_sbase[rank] + (cv ? c.x + c.z : 0) + pos[k];
          emit_subquery(d, base + k, rank, e, r);
        }
      continue;
    }
    int cur[kMaxLevel + 1];
#pragma unroll
    for (int l = 0; l <= kMaxLevel; ++l) cur[l] = 0;
    if (n > 1) {
      enum_window(w.x, w.y, w.z, w.w, ld, d.zmap, [&](int lev, uint32_t, uint32_t rank) {
        if (leaf_on(d.leaf_active, rank)) cur[lev]++;
      });
      int run = 0;
#pragma unroll
      for (int l = 0; l <= kMaxLevel; ++l) {
        const int c = cur[l];
        cur[l] = run;
        run += c;
      }
    }
    enum_window(w.x, w.y, w.z, w.w, ld, d.zmap, [&](int lev, uint32_t z, uint32_t rank) {
      if (!leaf_on(d.leaf_active, rank)) return;
      const bool cv = pair_cov(d, lev, z, r, cov_on);
      const int4 c = d.leaf_cnt[rank];
      const int32_t e = d.leaf_sbase[rank] + (cv ? c.x + c.z + c.y : c.x) +
                        atomicAdd(&d.leaf_cur[2 * rank + (cv ? 1 : 0)], 1);
      emit_subquery(d, base + cur[lev]++, rank, e, r);
    });
  }
}

// per-leaf occupancy / task statistics (engine.py:212-225,261-267)
__global__ void __launch_bounds__(256) k_leaf_stats(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t L = h->L;
  unsigned long long act = 0, s1 = 0, s2 = 0, tasks = 0, tests = 0, si = 0, sc = 0, pa = 0, sa = 0, wr = 0;
  TJ_GRID_STRIDE(r, L) {
    const int4 c = d.leaf_cnt[r];
    const int32_t nisq = c.x + c.z, ncov = c.y + c.w;
    d.leaf_nisq[r] = nisq;
    d.leaf_ncov[r] = ncov;
    d.linfo[r] = make_int4(d.leaf_obase[r], d.leaf_nobj[r], d.leaf_sbase[r], nisq);
    const unsigned long long no = (unsigned long long)d.leaf_nobj[r];
    const unsigned long long ni = (unsigned long long)nisq;
    si += ni;
    sc += (unsigned long long)ncov;
    if (no) {
      act += 1;
      s1 += no;
      s2 += no * no;
      if (ni) {
        tasks += 1;
        tests += no * ni;
        pa += no;
        sa += ni;
        if (leaf_on(d.leaf_active, r)) wr += ni * ((no + 31) / 32);
      }
    }
  }
  act = warp_sum(act);
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  tasks = warp_sum(tasks);
  tests = warp_sum(tests);
  si = warp_sum(si);
  sc = warp_sum(sc);
  pa = warp_sum(pa);
  sa = warp_sum(sa);
  wr = warp_sum(wr);
  if (lane_id() == 0) {
    if (wr) atomicAdd(&h->W_ref, wr);
    if (pa) atomicAdd(&h->task_obj, pa);
    if (sa) atomicAdd(&h->task_isq, sa);
    if (si) atomicAdd(&h->sum_isq, si);
    if (sc) atomicAdd(&h->sum_cov, sc);
    if (act) atomicAdd(&h->active_cells, act);
    if (s1) atomicAdd(&h->occ_sum, s1);
    if (s2) atomicAdd(&h->occ_sumsq, s2);
    if (tasks) atomicAdd((unsigned long long*)&h->n_tasks, tasks);
    if (tests) atomicAdd(&h->tests, tests);
  }
}

// ===========================================================================
// K3: per-leaf join (Alg. 2) into linear bitmaps
// ===========================================================================
// Work unit = (task leaf, object tile of up to 16 blocks = 512 objects); one
// CTA per unit.  The tile's (x, y) are staged in shared memory once and
// tested against every intersecting subquery of the leaf.  The output is the
// paper's bitmap: bit k of word b of subquery s is the closed fp64 test
// xa <= x <= xb and ya <= y <= yb of object 32b + k of the leaf's block
// (bitmap.py:89-97), stored in the linear layout linear[s*blocks + b]
// (bitmap.py:105-111), plus per-subquery popcounts (bitmap.py:114-119).
//
// Testing every (subquery, object) pair costs four fp64 compares on the
// 64-lane/clk FP64 pipe.  Leaves with enough subqueries instead bucket each
// axis of the tile into 256 equal buckets with one monotone map
// k(v) = floor(fl(fl(v - min) * 256 / (max - min))), and build, per axis and
// per 32-object block, the prefix tables Pre_k = {objects with bucket < k}
// (shared-memory atomicOr scatter + a warp OR-scan per column).  Because k is
// monotone, an object whose bucket lies strictly between the buckets of a
// subquery's two bounds passes that axis' test, and one outside them fails
// it; so a whole result word is
//   D = (Pre_kb & ~Pre_ka+1)_x & (Pre_kb & ~Pre_ka+1)_y      (certain bits)
// from eight table loads, and only the few objects that share a bucket with
// a bound (A = (Pre_kb+1 & ~Pre_ka)_x & (...)_y & ~D) get the exact fp64
// test.  Bit-identical to the direct test by construction.
#ifndef TJ_JT
#define TJ_JT 128
#endif
constexpr int kJT = TJ_JT;                    // join CTA threads
constexpr int kJW = kJT / 32;
constexpr int kTileBlocks = 12;               // object tile: 12 blocks = 384 objects (th_quad)
constexpr int kTileObj = kTileBlocks * 32;
#ifndef TJ_NK
#define TJ_NK 128
#endif
constexpr int kNK = TJ_NK;                    // buckets per axis
constexpr int kRows = kNK + 2;                // prefix rows k = 0 .. kNK + 1
#ifndef TJ_QC
#define TJ_QC 256
#endif
constexpr int kQC = TJ_QC;                    // subqueries per chunk
#ifndef TJ_TMQ
#define TJ_TMQ 12
#endif
constexpr int kTableMinQ = TJ_TMQ;            // table path from this many subqueries
#ifndef TJ_JOIN_TPS
#define TJ_JOIN_TPS 1
#endif
constexpr bool kJoinTPS = TJ_JOIN_TPS != 0;   // table path: one thread per subquery (0: per (subquery, block))
#ifndef TJ_JOIN_ODD
#define TJ_JOIN_ODD 1
#endif
constexpr bool kJoinOdd = TJ_JOIN_ODD != 0;   // odd pair stride of the table rows (bank spread)


// Optional row padding (TJ_ROW_PAD=8: bitmap rows padded to whole 32-byte
// sectors, pad words written as zeros by the join): the decode reads each
// subquery's row at a random place, and an unaligned 28-byte row spans two
// sectors.  Measured at config C5: the decode is unchanged (it is not bound
// by those sectors) and the join 18% slower, so rows are unpadded by default.
// Statistics and the introspection always use the reference's unpadded word
// counts (bitmap.py:105-111).
#ifndef TJ_ROW_PAD
#define TJ_ROW_PAD 1  // 8: sector-padded rows (measured: the decode unchanged, the join 18% slower)
#endif
constexpr int kRowPad = TJ_ROW_PAD;
__host__ __device__ __forceinline__ int row_words(int nb) { return (nb + kRowPad - 1) / kRowPad * kRowPad; }

struct WordsIn {
  const int32_t* nobj;
  const int32_t* nisq;
  const uint8_t* active;
  __device__ int64_t operator()(int64_t r) const {
    const int64_t no = nobj[r], ni = nisq[r];
    return (no > 0 && ni > 0 && leaf_on(active, r)) ? ni * row_words((int)((no + 31) / 32)) : 0;
  }
};
struct UnitsIn {
  const int32_t* nobj;
  const int32_t* nisq;
  const uint8_t* active;
  __device__ int64_t operator()(int64_t r) const {
    const int64_t no = nobj[r], ni = nisq[r];
    if (!(no > 0 && ni > 0 && leaf_on(active, r))) return 0;
    const int64_t nb = (no + 31) / 32;
    return (nb + kTileBlocks - 1) / kTileBlocks;
  }
};

// directory blocks: per leaf, intersecting entries then covering entries
struct LeafSqIn {
  const int4* cnt;
  __device__ int64_t operator()(int64_t r) const {
    const int4 c = cnt[r];
    return (int64_t)c.x + c.y + c.z + c.w;
  }
};

// Multi-GPU leaf-range sharding: every rank builds the same
// index; right after it, leaves are cut into contiguous Morton ranges balanced
// by their object counts (queries are issued where objects are), and a rank
// scatters, joins, decodes and assembles only the (query, leaf) pairs of its
// own leaves — its per-query lists are the restriction of the full lists to
// its leaves (disjoint across ranks).
struct LeafWeightIn {
  const int32_t* nobj;
  __device__ int64_t operator()(int64_t r) const { return (int64_t)nobj[r] + 1; }
};
struct PrefOut {
  int64_t* a;
  __device__ void operator()(int64_t i, int64_t ex, int64_t) const { a[i] = ex; }
};
__global__ void __launch_bounds__(256) k_shard_mark(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t T = h->shard_total > 0 ? h->shard_total : 1;
  const LeafWeightIn wt{d.leaf_nobj};
  TJ_GRID_STRIDE(r, h->L) {
    const int64_t mid = 2 * d.leaf_wpre[r] + wt(r);  // 2 x midpoint of the leaf's weight interval
    const int64_t owner = (mid * h->shard_n) / (2 * T);
    d.leaf_active[r] = (owner == h->shard_rank) || (owner >= h->shard_n && h->shard_rank == h->shard_n - 1);
  }
}

// work unit -> leaf (so a join CTA finds its leaf with one load)
__global__ void __launch_bounds__(256) k_unit_map(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const UnitsIn units{d.leaf_nobj, d.leaf_nisq, d.leaf_active};
  TJ_GRID_STRIDE(r, h->L) {
    const int64_t nu = units(r), b = d.leaf_ubase[r];
    for (int64_t k = 0; k < nu; ++k) d.unit_leaf[b + k] = (int32_t)r;
  }
}

__global__ void __launch_bounds__(256) k_zero_counts(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  TJ_GRID_STRIDE(e, h->S) d.ecount[e] = 0;
}

// Tile objects arrive by bulk copy (cp.async.bulk, the TMA engine's 1-D
// copy), double-buffered: while a CTA joins unit u, the copy engine stages
// unit u + gridDim's x / y into the other buffer, completion tracked by an
// mbarrier per buffer.  A bulk copy needs 16-byte aligned addresses and sizes,
// so a tile is copied from the 16-byte boundary at or below its first object
// (lead = 0 or 1 doubles) and rounded up (the coordinate arrays carry 16
// bytes of slack); objects past the tile's end are never read unmasked.
constexpr int kTileBuf = kTileObj + 4;    // lead + round-up
struct JoinSmem {
  double ox[2][kTileBuf];                 // tile objects, two stages
  double oy[2][kTileBuf];
  unsigned long long bar[2];              // mbarriers of the two stages
  uint32_t tab[2 * kRows * (kTileBlocks + 2)];  // [axis][k][b], row stride >= tile blocks
  ushort4 kb[kQC];                        // bucket of xa, xb, ya, yb
  int32_t cnt[kQC];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "TJ_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra TJ_WAIT_%=;\n}"
      ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

// The tile of unit u: first object (global index), object count, 16-byte lead
struct TileRef {
  int32_t ob;
  int P;
};
__device__ __forceinline__ TileRef tile_of(const Dev& d, int64_t u) {
  const int64_t r = d.unit_leaf[u];
  const int4 li = d.linfo[r];
  const int nb = (li.y + 31) >> 5;
  const int b0 = (int)(u - d.leaf_ubase[r]) * kTileBlocks, nbt = min(kTileBlocks, nb - b0);
  return TileRef{li.x + b0 * 32, min(li.y - b0 * 32, nbt * 32)};
}
// issue the bulk copies of a tile's x / y into stage buffers (one thread)
__device__ __forceinline__ void stage_tile(const Dev& d, JoinSmem& S, int st, TileRef t) {
  const int lead = t.ob & 1;  // doubles before the tile in its 16-byte line
  const uint32_t bytes = (uint32_t)(((t.P + lead) * 8 + 15) & ~15);
  mbar_expect_tx(&S.bar[st], 2 * bytes);
  bulk_g2s(S.ox[st], d.sx + (t.ob - lead), bytes, &S.bar[st]);
  bulk_g2s(S.oy[st], d.sy + (t.ob - lead), bytes, &S.bar[st]);
}

// Monotone bucket map of one axis of a leaf.  Any base and positive scale
// keep it monotone (fl(v - base), the product, the clamps and the
// truncation are all non-decreasing in v); the leaf's own extent makes the
// buckets even.  Objects and bounds use the same map.
// (evaluated in fp32: rounding to float, subtracting a constant and scaling by
// a positive constant are each monotone, and monotonicity is all the bucket
// tables need — the exact fp64 test settles every bit they cannot prove)
__device__ __forceinline__ int bucket(double v, float base, float scale) {
  float t = __fmul_rn(__fsub_rn(__double2float_rn(v), base), scale);
  t = fmaxf(t, 0.0f);
  t = fminf(t, (float)(kNK - 1));
  return 1 + __float2int_rz(t);
}

__device__ __forceinline__ bool in_rect(double x, double y, const Rect4& R) {
  return x >= R.xa && x <= R.xb && y >= R.ya && y <= R.yb;  // bitmap.py:89-94
}

__global__ void __launch_bounds__(kJT) k_join(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  extern __shared__ __align__(16) unsigned char join_smem[];
  JoinSmem& S = *reinterpret_cast<JoinSmem*>(join_smem);
  const int tid = threadIdx.x, lane = lane_id(), wp = tid >> 5;
  const int64_t U = h->U;
  const double gxa = h->xa, gya = h->ya, gw = h->width, gh = h->height;
  const double sxm = h->sx_max, sym = h->sy_max;  // 2^l_max / extent (0 for an empty extent)
  const int lmax = h->l_max;
  if (tid == 0) {
    mbar_init(&S.bar[0]);
    mbar_init(&S.bar[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (blockIdx.x < U) stage_tile(d, S, 0, tile_of(d, blockIdx.x));
  }
  __syncthreads();
  int iter = 0;
  for (int64_t u = blockIdx.x; u < U; u += gridDim.x, ++iter) {
    const int stg = iter & 1;
    // the next unit's objects into the other stage (free: the previous unit ended with a barrier)
    if (tid == 0 && u + gridDim.x < U) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the stage's generic reads before the copy
      stage_tile(d, S, stg ^ 1, tile_of(d, u + gridDim.x));
    }
    const int64_t r = d.unit_leaf[u];
    const int4 li = d.linfo[r];  // object base, object count, entry base, intersecting count
    const int nobj = li.y, nisq = li.w;
    const int nb = (nobj + 31) >> 5;
    const int ot = (int)(u - d.leaf_ubase[r]);
    const int n_ot = (nb + kTileBlocks - 1) / kTileBlocks;
    const int b0 = ot * kTileBlocks, nbt = min(kTileBlocks, nb - b0);
    const int P = min(nobj - b0 * 32, nbt * 32);
    const int32_t ob = li.x + b0 * 32;
    const int64_t woff = d.leaf_woff[r];
    const int nbp = row_words(nb);  // row stride (sector-padded)
    const int32_t sbase = li.z;
    const bool table = nisq >= kTableMinQ;
    // table row stride in words: even for paired 8-byte lookups; with one thread per subquery its
    // pairs per row are odd, so the random rows of a warp's subqueries spread over the banks
    // (4 pairs per row put every row start on one of 4 bank pairs: 8-way conflicts)
    const int nbs = (kJoinTPS && n_ot == 1) ? (kJoinOdd ? 2 * (((nbt + 1) >> 1) | 1) : (nbt + 1) & ~1) : nbt;
    // ---- this unit's objects (bulk-copied into stage stg) ----------------------
    mbar_wait(&S.bar[stg], (uint32_t)((iter >> 1) & 1));
    const double* ox = S.ox[stg] + (ob & 1);
    const double* oy = S.oy[stg] + (ob & 1);
    float bx = 0.0f, by = 0.0f, scx = 0.0f, scy = 0.0f;
    if (table) {
      const uint32_t code = d.leaf_code[r];
      const int lev = (int)(code >> kLevelShift);
      const uint32_t z = code & kPayloadMask;
      const double inv = 1.0 / (h->grid_sf ? (double)h->grid_sf : (double)(1u << lev));
      bx = gxa + (double)compact2(z) * inv * gw;
      by = gya + (double)compact2(z >> 1) * inv * gh;
      // kNK buckets across the leaf: sx_max = 2^l_max / width
      const double f = (double)kNK / (double)(1u << (lmax - lev));
      scx = sxm * f;
      scy = sym * f;
      static_assert((2 * kRows) % 4 == 0, "table rows must allow 16-byte zeroing");
      for (int i = tid; i < 2 * kRows * nbs / 4; i += kJT) reinterpret_cast<uint4*>(S.tab)[i] = make_uint4(0u, 0u, 0u, 0u);
      __syncthreads();
      // bucket scatter: Bk[axis][k][b] |= bit of each object
      for (int i = tid; i < P; i += kJT) {
        const int kx = bucket(ox[i], bx, scx), ky = bucket(oy[i], by, scy);
        const uint32_t bit = 1u << (i & 31);
        atomicOr(&S.tab[kx * nbs + (i >> 5)], bit);
        atomicOr(&S.tab[(kRows + ky) * nbs + (i >> 5)], bit);
      }
      __syncthreads();
      // exclusive prefix-OR down every (axis, block) column: Pre_k = OR_{k' < k} Bk_k'
      constexpr int kPer = (kRows + 31) / 32;
      for (int task = wp; task < 2 * nbt; task += kJW) {
        const int ax = task >= nbt ? 1 : 0, b = task - ax * nbt;
        uint32_t* col = S.tab + ax * kRows * nbs + b;
        uint32_t v[kPer];
        uint32_t acc = 0;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
          const int k = lane * kPer + j;
          v[j] = k < kRows ? col[k * nbs] : 0u;
          acc |= v[j];
        }
        uint32_t pre = acc;  // inclusive OR-scan of the lane totals
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(0xffffffffu, pre, o);
          if (lane >= o) pre |= t;
        }
        uint32_t run = __shfl_up_sync(0xffffffffu, pre, 1);
        if (lane == 0) run = 0u;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
          const int k = lane * kPer + j;
          if (k < kRows) col[k * nbs] = run;
          run |= v[j];
        }
      }
    }
    __syncthreads();
    const uint32_t divm = (65536u + (uint32_t)nbt - 1u) / (uint32_t)nbt;  // it / nbt for it < 65536 / 16
    const Rect4* erect = d.erect + sbase;
    // (multi-tile leaves — objects pinned at l_max, many per bucket — keep one thread per (subquery,
    // block) item: their many ambiguous bits serialise a subquery's fix-ups in one lane; at config E
    // the per-subquery mapping made the join 2x slower)
    if (kJoinTPS && table && n_ot == 1) {
      // ---- one thread per subquery: its row of the tile, two blocks per step (paired 8-byte table
      // lookups of rows k and k + 1), its popcount in a register; no shared-memory staging, no atomics
      const uint2* TX = reinterpret_cast<const uint2*>(S.tab);
      const uint2* TY = reinterpret_cast<const uint2*>(S.tab + kRows * nbs);
      const int hs = nbs >> 1;
      const bool last_tile = b0 + nbt == nb;
      Rect4 Rn;
      if (tid < nisq) Rn = erect[tid];
      for (int t = tid; t < nisq; t += kJT) {
        const Rect4 R = Rn;
        if (t + kJT < nisq) Rn = erect[t + kJT];  // the next subquery's rect in flight
        const int kxa = bucket(R.xa, bx, scx) * hs, kxb = bucket(R.xb, bx, scx) * hs;
        const int kya = bucket(R.ya, by, scy) * hs, kyb = bucket(R.yb, by, scy) * hs;
        uint32_t* orow = d.bitmap + woff + (int64_t)t * nbp + b0;
        int cnt = 0;
        for (int b2 = 0; b2 < hs; ++b2) {
          const uint2 xa0 = TX[kxa + b2], xa1 = TX[kxa + hs + b2], xb0 = TX[kxb + b2], xb1 = TX[kxb + hs + b2];
          const uint2 ya0 = TY[kya + b2], ya1 = TY[kya + hs + b2], yb0 = TY[kyb + b2], yb1 = TY[kyb + hs + b2];
          uint32_t D[2], A[2];
          D[0] = (xb0.x & ~xa1.x) & (yb0.x & ~ya1.x);
          D[1] = (xb0.y & ~xa1.y) & (yb0.y & ~ya1.y);
          A[0] = (xb1.x & ~xa0.x) & (yb1.x & ~ya0.x) & ~D[0];
          A[1] = (xb1.y & ~xa0.y) & (yb1.y & ~ya0.y) & ~D[1];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int b = 2 * b2 + e;
            uint32_t a = A[e];
            while (a) {
              const int bit = __ffs(a) - 1;
              a &= a - 1;
              const int o = (b << 5) + bit;
              if (in_rect(ox[o], oy[o], R)) D[e] |= 1u << bit;
            }
            if (b < nbt) {  // (pairs as one 8-byte store into even-padded rows: no faster)
              orow[b] = D[e];
              cnt += __popc(D[e]);
            }
          }
        }
        if (kRowPad > 1 && last_tile)  // the row's pad words: whole-sector stores
          for (int b = nb - b0; b < nbp - b0; ++b) orow[b] = 0u;
        int32_t* ec = d.ecount + sbase + t;
        if (n_ot == 1) *ec = cnt;
        else if (cnt) atomicAdd(ec, cnt);
      }
      __syncthreads();  // the tile's shared memory is reused by the next unit
      continue;
    }
    // ---- subquery chunks ------------------------------------------------------
    for (int c0 = 0; c0 < nisq; c0 += kQC) {
      const int nq = min(kQC, nisq - c0);
      for (int t = tid; t < nq; t += kJT) {
        S.cnt[t] = 0;
        if (table) {
          const Rect4 R = erect[c0 + t];
          S.kb[t] = make_ushort4((unsigned short)bucket(R.xa, bx, scx), (unsigned short)bucket(R.xb, bx, scx),
                                 (unsigned short)bucket(R.ya, by, scy), (unsigned short)bucket(R.yb, by, scy));
        }
      }
      __syncthreads();
      uint32_t* out = d.bitmap + woff + (int64_t)c0 * nbp + b0;
      if (table) {
        const uint32_t* TX = S.tab;
        const uint32_t* TY = S.tab + kRows * nbs;
        const int items = nq * nbt;
        for (int it = tid; it < items; it += kJT) {
          const int s = (int)(((uint32_t)it * divm) >> 16), b = it - s * nbt;
          const ushort4 k4 = S.kb[s];
          const uint32_t xa0 = TX[k4.x * nbs + b], xa1 = TX[(k4.x + 1) * nbs + b];
          const uint32_t xb0 = TX[k4.y * nbs + b], xb1 = TX[(k4.y + 1) * nbs + b];
          const uint32_t ya0 = TY[k4.z * nbs + b], ya1 = TY[(k4.z + 1) * nbs + b];
          const uint32_t yb0 = TY[k4.w * nbs + b], yb1 = TY[(k4.w + 1) * nbs + b];
          uint32_t D = (xb0 & ~xa1) & (yb0 & ~ya1);
          uint32_t A = (xb1 & ~xa0) & (yb1 & ~ya0) & ~D;
          if (A) {
            const Rect4 R = erect[c0 + s];
            do {
              const int bit = __ffs(A) - 1;
              A &= A - 1;
              const int o = (b << 5) + bit;
              if (in_rect(ox[o], oy[o], R)) D |= 1u << bit;
            } while (A);
          }
          out[(int64_t)s * nbp + b] = D;
          if (D) atomicAdd(&S.cnt[s], __popc(D));
        }
      } else {
        // direct: lane = subquery, 32 objects of one block per step
        const int nsc = (nq + 31) >> 5;
        for (int it = wp; it < nsc * nbt; it += kJW) {
          const int sc = it / nbt, b = it - sc * nbt;
          const int s = sc * 32 + lane;
          Rect4 R;
          R.xa = R.ya = __longlong_as_double(0x7ff0000000000000ll);  // +inf: empty rect
          R.xb = R.yb = __longlong_as_double((long long)0xfff0000000000000ull);
          if (s < nq) R = erect[c0 + s];
          uint32_t w = 0;
#pragma unroll 8
          for (int k = 0; k < 32; ++k) {
            const int o = (b << 5) + k;
            if (in_rect(ox[o], oy[o], R)) w |= 1u << k;
          }
          const int valid = P - (b << 5);  // objects past the tile hold other leaves' coordinates
          if (valid < 32) w &= (1u << valid) - 1u;
          if (s < nq) {
            out[(int64_t)s * nbp + b] = w;
            if (w) atomicAdd(&S.cnt[s], __popc(w));
          }
        }
      }
      if (kRowPad > 1 && b0 + nbt == nb && nbp > nb) {  // the row's pad words: whole-sector stores
        const int np = nbp - nb;
        for (int it = tid; it < nq * np; it += kJT) {
          const int s = it / np;
          out[(int64_t)s * nbp + (nb - b0) + (it - s * np)] = 0u;
        }
      }
      __syncthreads();
      for (int t = tid; t < nq; t += kJT) {
        int32_t* ec = d.ecount + sbase + c0 + t;
        if (n_ot == 1) *ec = S.cnt[t];
        else atomicAdd(ec, S.cnt[t]);
      }
    }
  }
}

// ===========================================================================
// K4: result offsets, decode straight into the canonical per-query lists
// ===========================================================================
// Subquery slots are grouped per query in query input order (k_query_fill),
// so one exclusive scan of the per-slot result counts in slot order gives
// every run's position in the output CSR, and at a query's first slot the
// query's CSR offset: a query's list is its runs, merged (decode.py:102-123).
// Result counts: an intersecting subquery contributes its popcount (written
// per slot by the join), a covering one its leaf's whole block
// (decode.py:83-99).
__global__ void __launch_bounds__(256) k_cov_counts(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int lane = lane_id();
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long covres = 0;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < h->L; r += nwarp) {
    const int nc = d.leaf_ncov[r];
    if (nc == 0 || !leaf_on(d.leaf_active, r)) continue;
    const int32_t base = d.leaf_sbase[r] + d.leaf_nisq[r];
    const int32_t nobj = d.leaf_nobj[r];
    for (int c = lane; c < nc; c += 32) d.ecount[base + c] = nobj;
    if (lane == 0) covres += (unsigned long long)nobj * nc;
  }
  if (lane == 0 && covres) atomicAdd(&h->cov_results, covres);
}

// per-slot result counts in slot (= output) order.  (Reading them straight inside the slot-offset
// scan instead — its reduce and down-sweep passes each doing the random entry lookups — measured
// 0.11 ms slower per tick at C5.)
__global__ void __launch_bounds__(256) k_slot_counts(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t S = h->S;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s0 < S; s0 += 4 * stride) {
    int32_t e[4];  // four slot -> entry -> count chains in flight
#pragma unroll
    for (int u = 0; u < 4; ++u) e[u] = s0 + u * stride < S ? d.sq_le[s0 + u * stride].y : 0;
    int32_t c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) c[u] = s0 + u * stride < S ? d.ecount[e[u]] : 0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (s0 + u * stride < S) d.sq_count[s0 + u * stride] = c[u];
  }
}

__global__ void k_close_offsets(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  d.slot_off[h->S] = h->R;
  d.out_off[h->m] = h->R;
}

// result ids are written once and never re-read on the device: streaming stores
__device__ __forceinline__ void st_out(int64_t* p, int64_t v) { __stcs(reinterpret_cast<long long*>(p), (long long)v); }

constexpr int32_t kRowEnd = 0x7fffffff;
constexpr uint32_t kNoRow = 0xffffffffu;  // a covering slot: its run is the whole leaf block

#ifndef TJ_DQ_WPL
#define TJ_DQ_WPL 4  // decode phase A: bitmap words in flight per lane
#endif
#ifndef TJ_DQ_RPL
#define TJ_DQ_RPL 4  // decode phase B: row lookups in flight per lane
#endif
#ifndef TJ_DQ_TWGUARD
#define TJ_DQ_TWGUARD 1  // decode phase A: skip the word batches past a chunk's last word (warp-uniform; C5 decode -1.2%)
#endif
#ifndef TJ_DQ_MINB
#define TJ_DQ_MINB 10  // resident decode CTAs per SM the register budget is cut for
#endif
#ifndef TJ_DQ_SMEM_TMP
#define TJ_DQ_SMEM_TMP 0  // 1: the warp merge's second buffer in shared memory (16 KB more per CTA: fewer resident CTAs; measured no faster at C20)
#endif
constexpr int kDQThreads = 128;
constexpr int kDQWarps = kDQThreads / 32;
#ifndef TJ_DQ_STAGE
#define TJ_DQ_STAGE 896  // 1024 measured 3% slower: ten CTAs' windows then need the 196 KB shared-memory
                         // carveout, leaving 60 KB of L1 for the leaf-position lookups instead of 92 KB
#endif
constexpr int kDQStage = TJ_DQ_STAGE;   // results staged per warp window
constexpr int kLaneRuns = 4;     // lane-per-query k-way merge up to this many runs

constexpr int kRankRuns = 32;  // oversized lists (> one window) of 2..32 runs: warp rank merge; more: k_merge_big
constexpr int kLaneList = 128; // longer lists are sorted by the whole warp (warp_bitonic), not one lane

// Warp bitonic sort of one list a[0, cnt) in shared memory, cnt <= 32 * E,
// back in place (values distinct int32 input rows; padding INT_MAX).
// Lane-major layout — lane L holds elements L*E .. L*E+E-1 — so the stages
// with partner distance j < E are register compare-exchanges and only those
// with j >= E cross lanes (one shuffle per element).  For lists of many runs
// this costs O(n log^2 n / 32) register ops per lane with no dependent
// shared-memory searches, against k binary searches per element for the
// rank merge.
template <int E>
__device__ __forceinline__ void warp_bitonic(int32_t* a, int cnt) {
  constexpr int P = 32 * E;
  const int lane = lane_id();
  int32_t v[E];
#pragma unroll
  for (int u = 0; u < E; ++u) {
    const int i = lane * E + u;
    v[u] = i < cnt ? a[i] : 0x7fffffff;
  }
  // phases k < E: directions per slot (compile-time); the whole lane's block is one run
#pragma unroll
  for (int k = 2; k < E; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int u = 0; u < E; ++u) {
        if ((u & j) == 0) {
          const int32_t x = v[u], y = v[u + j];
          v[u] = (u & k) == 0 ? min(x, y) : max(x, y);
          v[u + j] = (u & k) == 0 ? max(x, y) : min(x, y);
        }
      }
    }
  }
  // phases k >= E: the direction is per lane.  Descending lanes hold ~v
  // (order-reversing on int32), so every exchange below is ascending.
  int32_t flip = 0;
#pragma unroll
  for (int k = E; k <= P; k <<= 1) {
    const int32_t nf = ((lane * E) & k) ? -1 : 0;
#pragma unroll
    for (int u = 0; u < E; ++u) v[u] ^= flip ^ nf;
    flip = nf;
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= E) {
        const int lj = j / E;
        const bool upper = (lane & lj) != 0;  // the upper partner keeps the max
#pragma unroll
        for (int u = 0; u < E; ++u) {
          const int32_t y = __shfl_xor_sync(0xffffffffu, v[u], lj);
          v[u] = ((v[u] < y) != upper) ? v[u] : y;
        }
      } else {
#pragma unroll
        for (int u = 0; u < E; ++u) {
          if ((u & j) == 0) {
            const int32_t x = v[u], y = v[u + j];
            v[u] = min(x, y);
            v[u + j] = max(x, y);
          }
        }
      }
    }
  }
  // the last phase (k = P) is ascending everywhere: flip == 0
  __syncwarp();
#pragma unroll
  for (int u = 0; u < E; ++u) {
    const int i = lane * E + u;
    if (i < cnt) a[i] = v[u];
  }
  __syncwarp();
}

// Warp merge of one list's k sorted runs (k <= 32; rs[j] = start of run j in
// the list `a` of cq elements, rs[k] = cq): pairwise rounds, each a segmented
// merge path — lane L produces outputs [L*cq/32, (L+1)*cq/32) of the round,
// finding its place by a binary search on the merge diagonal of the pair it
// starts in, then merging serially (one load per output, continuing into the
// next pairs).  A merged pair occupies exactly its two inputs' range, so runs
// only change their starts.  Rounds ping-pong between `a` and `tmp`; the last
// one stores the ids to `out`.  O(n log k) work against O(n log^2 n) for a
// bitonic sort of the concatenation (config C @20u: lists of 129..1024
// results with ~6.5 runs, where the bitonic sort was 78% of the decode).
template <typename IdOf>
__device__ __forceinline__ void warp_merge_runs(int32_t* a, int32_t* tmp, int32_t* rs, int cq, int k,
                                                int64_t* out, IdOf idof) {
  const int lane = lane_id();
  int32_t* src = a;
  int32_t* dst = tmp;
  int nr = k;
  auto run_start = [&](int j) -> int { return j < nr ? rs[j] : cq; };
  while (nr > 1) {
    const int np = (nr + 1) >> 1;
    const bool last = np == 1;
    const int lo = (int)(((int64_t)lane * cq) >> 5), hi = (int)(((int64_t)(lane + 1) * cq) >> 5);
    if (lo < hi) {
      // the pair holding output lo: the last pair starting at or before it
      int q = 0;
      for (int step = 16; step > 0; step >>= 1)
        if (q + step < np && rs[2 * (q + step)] <= lo) q += step;
      int sA = rs[2 * q], eA = run_start(2 * q + 1), eB = run_start(2 * q + 2);
      // merge path: l outputs from A among the first d of the pair
      const int d = lo - sA, nA = eA - sA, nB = eB - eA;
      int l = d > nB ? d - nB : 0, r = d < nA ? d : nA;
      while (l < r) {
        const int mid = (l + r) >> 1;
        if (src[sA + mid] < src[eA + d - 1 - mid]) l = mid + 1;
        else r = mid;
      }
      int ia = sA + l, ib = eA + (d - l);
      int32_t ha = ia < eA ? src[ia] : 0x7fffffff, hb = ib < eB ? src[ib] : 0x7fffffff;
      for (int p = lo; p < hi; ++p) {
        while (p == eB) {  // into the next (non-empty) pair: both its runs start at their heads
          ++q;
          sA = eB;
          eA = run_start(2 * q + 1);
          eB = run_start(2 * q + 2);
          ia = sA;
          ib = eA;
          ha = ia < eA ? src[ia] : 0x7fffffff;
          hb = ib < eB ? src[ib] : 0x7fffffff;
        }
        const bool ta = ha < hb;
        const int32_t v = ta ? ha : hb;
        if (last) st_out(out + p, idof(v));
        else dst[p] = v;
        if (ta) ha = ++ia < eA ? src[ia] : 0x7fffffff;
        else hb = ++ib < eB ? src[ib] : 0x7fffffff;
      }
    }
    // the merged pairs' starts: run q of the next round starts where run 2q did
    const int ns = 2 * lane < nr ? rs[2 * lane] : cq;
    __syncwarp();
    if (lane <= 32 - 1) rs[lane] = lane < np ? ns : cq;
    __syncwarp();
    nr = np;
    int32_t* t = src;
    src = dst;
    dst = t;
  }
}

template <typename T, typename Emit>
__device__ __forceinline__ void warp_rank_merge(const T* src, int cnt, int k, int c, Emit emit) {
  const int lane = lane_id();
  const int inc = warp_incl_scan(c);
  const int st = inc - c;  // lane j < k: start of run j
  for (int i0 = 0; i0 < cnt; i0 += 32) {
    const int i = i0 + lane;
    const bool ok = i < cnt;
    const T v = ok ? src[i] : T(0);
    int j = 0;  // own run: the last run starting at or before i
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const int sj = __shfl_sync(0xffffffffu, st, (j + step) & 31);
      if (j + step < k && sj <= i) j += step;
    }
    int rank = i - __shfl_sync(0xffffffffu, st, j);
    for (int jj = 0; jj < k; ++jj) {
      const int a0 = __shfl_sync(0xffffffffu, st, jj);
      const int nx = __shfl_sync(0xffffffffu, st, (jj + 1) & 31);
      const int a1 = jj + 1 < k ? nx : cnt;
      if (ok && jj != j) {
        int first = a0, len = a1 - a0;  // lower_bound(v) in run jj
        while (len > 0) {
          const int half = len >> 1;
          if (src[first + half] < v) {
            first += half + 1;
            len -= half + 1;
          } else {
            len = half;
          }
        }
        rank += first - a0;
      }
    }
    if (ok) emit(rank, v);
  }
}

// Per-query decode + merge (Alg. 4 and merge_results, decode.py:40-123).
// A warp owns 32 consecutive queries; their lists are adjacent in the output
// (and so are their subquery slots), so it cuts them into windows of at most
// kDQStage results and, per window:
//  A. decodes every slot's run into shared memory at its final position:
//     the words of all the window's runs are flattened across the lanes
//     (independent loads), and one running popcount prefix over them is the
//     output position of every bit — runs are concatenated in slot order,
//     which is output order;
//  B. turns leaf positions into input rows with batched independent loads;
//  C. stores the window (runs concatenated) with coalesced writes, ids
//     looked up there;
//  D. re-sorts the lists of several runs (object ids increase with the input
//     row): one lane per query merges 2..4 runs of <= 128 results by head;
//     longer lists or more runs are sorted by the whole warp, one list at a
//     time, in registers (warp_bitonic; > 512 results: two sorted halves and
//     one rank merge).
// Lists of one query larger than a window are concatenated in global memory
// by the whole warp and rank-merged there (<= 32 runs); lists that need a
// sort by id (ids not monotone) or oversized lists of more than 32 runs go to
// the CTA-wide k_merge_big.
// Id modes of the decode (one instantiation each; the two that do not match
// the tick's ids return at once): merge keys and ids of a leaf position are
//  kIdsRows:   key = input row, id = the row (ids are the rows);
//  kIdsKeyed:  key = the block's id offset (keyed lists), id = id_min + key;
//  kIdsLookup: key = input row, id = ids[row] (lists sorted per query by
//              k_merge_big unless the ids increase with the row).
enum { kIdsRows = 0, kIdsKeyed = 1, kIdsLookup = 2 };
__device__ __forceinline__ int id_mode_of(const DevHdr* h) {
  return !h->not_identity ? kIdsRows : (h->key_mode ? kIdsKeyed : kIdsLookup);
}

template <int kMode>
__global__ void __launch_bounds__(kDQThreads, TJ_DQ_MINB) k_decode_query(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort || id_mode_of(h) != kMode) return;
  __shared__ int32_t sbuf[kDQWarps][kDQStage];
  __shared__ int32_t rsb[kDQWarps][33];  // run starts of the list a warp merges
#if TJ_DQ_SMEM_TMP
  __shared__ int32_t tmpb[kDQWarps][kDQStage];  // the merge rounds' second buffer
#endif
  const bool mono = kMode != kIdsLookup || !h->not_monotone;
  const int64_t m = h->m;
  const int lane = lane_id(), wp = threadIdx.x >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // leaf position -> merge key
  const int32_t* __restrict__ sidx = kMode == kIdsKeyed ? reinterpret_cast<const int32_t*>(d.loff) : d.sidx;
  int32_t* sa = sbuf[wp];
  int bad = 0;
  auto idof = [&](int32_t v) -> int64_t {
    if constexpr (kMode == kIdsRows) return (int64_t)v;
    else if constexpr (kMode == kIdsKeyed) return h->id_min + (int64_t)(uint32_t)v;
    else return d.ids[v];
  };
  for (int64_t q0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; q0 < m; q0 += nwarp * 32) {
    const int64_t ql = q0 + lane;
    int k = 0;
    int32_t s0 = 0;
    int64_t qo = 0, cnt = 0;
    if (ql < m) {
      k = d.nsub[ql];
      s0 = d.qsbase[ql];
      qo = d.slot_off[s0];
      cnt = d.slot_off[s0 + k] - qo;
      d.out_off[ql] = qo;
    }
    const int nq = (int)min((int64_t)32, m - q0);
    int l0 = 0;
    while (l0 < nq) {
      const int64_t base = __shfl_sync(0xffffffffu, qo, l0);
      // window = lanes [l0, l1): the longest run of queries whose lists fit the stage
      const unsigned fit = __ballot_sync(0xffffffffu, lane >= l0 && lane < nq && qo + cnt - base <= kDQStage);
      int l1 = l0 + __popc(fit);
      if (l1 == l0) {
        // ---- one oversized list: the warp concatenates its runs in global memory
        const int kq = __shfl_sync(0xffffffffu, k, l0);
        const int32_t sq0 = __shfl_sync(0xffffffffu, s0, l0);
        const int64_t cq = __shfl_sync(0xffffffffu, cnt, l0);
        const bool rmerge = mono && kq > 1 && kq <= kRankRuns && cq < (int64_t(1) << 30);
        int64_t* cat = rmerge ? d.scratch : d.out_ids;  // runs concatenated here
        int64_t pos = base;
        for (int j = 0; j < kq; ++j) {
          const int32_t s = sq0 + j;
          const int64_t cj = d.sq_count[s];
          if (cj == 0) continue;
          const int2 le = d.sq_le[s];
          const int32_t leaf = le.x;
          const int4 li = d.linfo[leaf];
          const int nobj = li.y;
          const int32_t obase = li.x;
          const int nbw = (nobj + 31) >> 5;
          const int row = le.y - li.z;
          const bool cov = row >= li.w;
          const uint32_t* wpt = cov ? nullptr : d.bitmap + d.leaf_woff[leaf] + (int64_t)row * row_words(nbw);
          const uint32_t tail = (nobj & 31) ? ((1u << (nobj & 31)) - 1u) : 0xffffffffu;
          int64_t got = 0;
          for (int b0 = 0; b0 < nbw; b0 += 32) {
            const int b = b0 + lane;
            uint32_t w = b < nbw ? (cov ? (b == nbw - 1 ? tail : 0xffffffffu) : wpt[b]) : 0u;
            const int c = __popc(w);
            const int inc = warp_incl_scan(c);
            int64_t p = pos + got + (inc - c);
            while (w) {
              const int bit = __ffs(w) - 1;
              w &= w - 1;
              cat[p++] = idof(sidx[obase + (b << 5) + bit]);
            }
            got += __shfl_sync(0xffffffffu, inc, 31);
          }
          bad |= (lane == 0) && (got != cj);  // CountMismatch (bitmap.py:131-132)
          pos += cj;
        }
        if (rmerge) {
          __syncwarp();
          int64_t* out = d.out_ids + base;
          warp_rank_merge(d.scratch + base, (int)cq, kq, lane < kq ? d.sq_count[sq0 + lane] : 0,
                          [&](int r, int64_t v) { out[r] = v; });
        } else if (lane == 0 && cq > 1 && (kq > 1 || !mono)) {
          const int idx = atomicAdd(&h->n_big, 1);
          d.big_list[idx] = (int32_t)(q0 + l0);
        }
        l0 += 1;
        continue;
      }
      const bool act = lane >= l0 && lane < l1;
      const int32_t slo = __shfl_sync(0xffffffffu, s0, l0);
      const int32_t shi = __shfl_sync(0xffffffffu, s0 + k, l1 - 1);
      const int64_t T = __shfl_sync(0xffffffffu, qo + cnt, l1 - 1) - base;
      // ---- A: bits -> leaf positions, at their output positions in sa
      for (int32_t c0 = slo; c0 < shi; c0 += 32) {
        const int32_t s = c0 + lane;
        int nbw = 0, obase = 0, cs = 0;
        uint32_t wof = kNoRow;  // the row's first word (32 bits: the tick's bitmap is < 2^32 words)
        uint32_t tail = 0;
        int2 le = make_int2(0, 0);
        if (s < shi) {  // count and slot loaded together (no dependent round trip)
          cs = d.sq_count[s];
          le = d.sq_le[s];
        }
        if (cs > 0) {
          const int32_t leaf = le.x;
          const int4 li = d.linfo[leaf];
          const int nobj = li.y;
          const int row = le.y - li.z;
          obase = li.x;
          nbw = (nobj + 31) >> 5;
          tail = (nobj & 31) ? ((1u << (nobj & 31)) - 1u) : 0xffffffffu;
          wof = row >= li.w ? kNoRow : (uint32_t)(d.leaf_woff[leaf] + (int64_t)row * row_words(nbw));
        }
        const int pos0 = (int)(d.slot_off[c0] - base);  // output offset of the chunk's first run
        const int winc = warp_incl_scan(nbw);
        const int wexc = winc - nbw;
        const int TW = __shfl_sync(0xffffffffu, winc, 31);
        int pos = 0;  // prefix of the flattened popcounts
        for (int t0 = 0; t0 < TW; t0 += 32 * TJ_DQ_WPL) {
          // TJ_DQ_WPL words per lane per step: independent loads in flight (8 measured slower: registers)
          uint32_t w[TJ_DQ_WPL];
          int wo[TJ_DQ_WPL];
#pragma unroll
          for (int u = 0; u < TJ_DQ_WPL; ++u) {
            const int t = t0 + u * 32 + lane;
            w[u] = 0;
            wo[u] = 0;
#if TJ_DQ_TWGUARD
            if (t0 + u * 32 >= TW) continue;  // warp-uniform: no search for batches past the chunk's words
#endif
            int j = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
              const int v = __shfl_sync(0xffffffffu, wexc, j + step);
              if (v <= t) j += step;
            }
            const int jx = __shfl_sync(0xffffffffu, wexc, j);
            const int jn = __shfl_sync(0xffffffffu, nbw, j);
            const int jo = __shfl_sync(0xffffffffu, obase, j);
            const uint32_t jw = __shfl_sync(0xffffffffu, wof, j);
            const uint32_t jt = __shfl_sync(0xffffffffu, tail, j);
            const int wb = t - jx;
            if (t < TW) w[u] = jw != kNoRow ? __ldcs(d.bitmap + jw + wb) : (wb == jn - 1 ? jt : 0xffffffffu);  // read once: evict first
            wo[u] = jo + (wb << 5);
          }
#pragma unroll
          for (int u = 0; u < TJ_DQ_WPL; ++u) {
#if TJ_DQ_TWGUARD
            if (t0 + u * 32 >= TW) break;
#endif
            uint32_t x = w[u];
            const int c = __popc(x);
            const int inc = warp_incl_scan(c);
            int p = pos0 + pos + (inc - c);
            while (x) {
              const int bit = __ffs(x) - 1;
              x &= x - 1;
              sa[p++] = wo[u] + bit;
            }
            pos += __shfl_sync(0xffffffffu, inc, 31);
          }
        }
        // the runs' popcounts must add up to the counts the offsets came from
        const int32_t cend = c0 + 32 < shi ? c0 + 32 : shi;
        bad |= (lane == 0) && (pos0 + pos != d.slot_off[cend] - base);  // CountMismatch (bitmap.py:131-132)
      }
      __syncwarp();
      // ---- B: leaf positions -> input rows (independent loads, 4 in flight per lane)
      for (int i0 = 0; i0 < (int)T; i0 += 32 * TJ_DQ_RPL) {
        int32_t v[TJ_DQ_RPL];
#pragma unroll
        for (int u = 0; u < TJ_DQ_RPL; ++u) {
          const int i = i0 + u * 32 + lane;
          v[u] = i < (int)T ? sidx[sa[i]] : 0;
        }
#pragma unroll
        for (int u = 0; u < TJ_DQ_RPL; ++u) {
          const int i = i0 + u * 32 + lane;
          if (i < (int)T) sa[i] = v[u];
        }
      }
      __syncwarp();
      // ---- C: store the window (runs concatenated; ids looked up here)
      for (int i = lane; i < (int)T; i += 32) st_out(d.out_ids + base + i, idof(sa[i]));
      __syncwarp();
      // ---- D: per query with 2..4 runs and <= 128 results, merge the runs by head (one lane per query)
      // (TJ_DEBUG bit 8: skip the merges — wrong lists, for timing the other phases only)
      const bool merge_on = !(h->dbg & 8);
      if (act && cnt > 1 && merge_on) {
        const int qs = (int)(qo - base);
        if (!mono) {  // ids not increasing with the input row: sorted by id in k_merge_big
          const int idx = atomicAdd(&h->n_big, 1);
          d.big_list[idx] = (int32_t)ql;
        } else if (k > 1 && k <= kLaneRuns && cnt <= kLaneList) {
          // heads packed as (row << 2 | run) (rows < 2^28): the minimum names its run
          static_assert(kLaneRuns == 4, "the packed-head minimum below is written for four runs");
          constexpr uint32_t kEnd = 0x7ffffffcu;
          int pos[kLaneRuns], end[kLaneRuns];
          uint32_t hk[kLaneRuns];
          int acc = qs;
#pragma unroll
          for (int j = 0; j < kLaneRuns; ++j) {
            const int c = j < k ? d.sq_count[s0 + j] : 0;
            pos[j] = acc;
            end[j] = acc + c;
            acc += c;
            hk[j] = (c > 0 ? ((uint32_t)sa[pos[j]] << 2) : kEnd) | (uint32_t)j;
          }
          int64_t* dst = d.out_ids + qo;
          for (int o = 0; o < (int)cnt; ++o) {
            const uint32_t mn = min(min(hk[0], hk[1]), min(hk[2], hk[3]));
            const int bj = (int)(mn & 3u);
            st_out(dst + o, idof((int32_t)(mn >> 2)));
            // advance the winning run: select its cursor, one shared-memory load, select back
            int np = pos[0], ne = end[0];
#pragma unroll
            for (int j = 1; j < kLaneRuns; ++j) {
              np = j == bj ? pos[j] : np;
              ne = j == bj ? end[j] : ne;
            }
            ++np;
            const uint32_t nk = (np < ne ? ((uint32_t)sa[np] << 2) : kEnd) | (uint32_t)bj;
#pragma unroll
            for (int j = 0; j < kLaneRuns; ++j) {
              pos[j] = j == bj ? np : pos[j];
              hk[j] = j == bj ? nk : hk[j];
            }
          }
        }
      }
      // other multi-run lists: the warp sorts them one at a time
      unsigned rq = __ballot_sync(0xffffffffu, merge_on && act && cnt > 1 && mono && k > 1 &&
                                                   (k > kLaneRuns || cnt > kLaneList));
      while (rq) {
        const int src = __ffs(rq) - 1;
        rq &= rq - 1;
        const int64_t qoq = __shfl_sync(0xffffffffu, qo, src);
        const int cq = (int)__shfl_sync(0xffffffffu, cnt, src);
        int64_t* out = d.out_ids + qoq;
        int32_t* lst = sa + (qoq - base);
        const int kq = __shfl_sync(0xffffffffu, k, src);
        if (kq <= 32) {  // merge the runs (starts from the slot counts; empty runs are harmless)
          const int32_t sq0 = __shfl_sync(0xffffffffu, s0, src);
          const int c = lane < kq ? d.sq_count[sq0 + lane] : 0;
          const int inc = warp_incl_scan(c);
          int32_t* rs = rsb[wp];
          rs[lane] = lane < kq ? inc - c : cq;
          __syncwarp();
#if TJ_DQ_SMEM_TMP
          warp_merge_runs(lst, tmpb[wp], rs, cq, kq, out, idof);
#else
          warp_merge_runs(lst, reinterpret_cast<int32_t*>(d.scratch + qoq), rs, cq, kq, out, idof);
#endif
        } else if (cq <= 512) {  // sort in registers, then store
          if (cq <= 64) warp_bitonic<2>(lst, cq);
          else if (cq <= 128) warp_bitonic<4>(lst, cq);
          else if (cq <= 256) warp_bitonic<8>(lst, cq);
          else warp_bitonic<16>(lst, cq);
          for (int i = lane; i < cq; i += 32) st_out(out + i, idof(lst[i]));
        } else {  // two sorted halves, then one rank merge of the pair
          warp_bitonic<16>(lst, 512);
          warp_bitonic<16>(lst + 512, cq - 512);
          warp_rank_merge(lst, cq, 2, lane == 0 ? 512 : cq - 512, [&](int r, int32_t v) { st_out(out + r, idof(v)); });
        }
      }
      __syncwarp();
      l0 = l1;
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) h->count_mismatch = 1;
}

// ug_baseline's contention counters (baseline.py:64-121): each task cell
// flushes its private stage of `cap` pairs whenever full and once for the
// remainder, so flushes = sum over task cells of ceil(intersecting pairs / cap).
__global__ void __launch_bounds__(256) k_staging_flushes(const Dev d, int32_t cap, unsigned long long* out) {
  DevHdr* h = d.h;
  const int lane = lane_id();
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long acc = 0;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < h->L; r += nwarp) {
    const int nisq = d.leaf_nisq[r];
    if (nisq == 0 || d.leaf_nobj[r] == 0 || !leaf_on(d.leaf_active, r)) continue;
    const int32_t base = d.leaf_sbase[r];
    long long p = 0;
    for (int k = lane; k < nisq; k += 32) p += d.ecount[base + k];
    p = warp_sum(p);
    if (lane == 0) acc += (unsigned long long)((p + cap - 1) / cap);
  }
  if (lane == 0 && acc) atomicAdd(out, acc);
}

// TJ_OUT_IDS32 delivery: result ids narrowed to int32 (flag if one does not fit)
__global__ void __launch_bounds__(256) k_narrow_ids(const int64_t* __restrict__ src, int32_t* __restrict__ dst,
                                                    int64_t R, DevHdr* h) {
  int wide = 0;
  TJ_GRID_STRIDE(i, R) {
    const long long v = __ldcs(reinterpret_cast<const long long*>(src) + i);
    wide |= v != (long long)(int32_t)v;
    __stcs(dst + i, (int32_t)v);
  }
  if (__any_sync(0xffffffffu, wide) && lane_id() == 0) h->ids_wide = 1;
}

// TJ_OUT_IDS32 delivery of the CSR offsets (the caller checked R < 2^31)
__global__ void __launch_bounds__(256) k_narrow_offsets(const int64_t* __restrict__ src, int32_t* __restrict__ dst,
                                                        int64_t cnt) {
  TJ_GRID_STRIDE(i, cnt) __stcs(dst + i, (int32_t)__ldcs(reinterpret_cast<const long long*>(src) + i));
}

// ---------------------------------------------------------------------------
// CTA-wide sort of one segment (used only when object ids are not increasing
// in input order: then lists must be sorted by id, decode.py:117).
// Bitonic in shared memory for short segments; longer ones: shared-memory
// sorted chunks + merge-path passes through a same-sized scratch range.
// ---------------------------------------------------------------------------
constexpr int kSortSmem = 2048;

template <typename T>
__device__ void cta_bitonic(T* a, int n, T* sm, T sentinel) {
  int P = 32;
  while (P < n) P <<= 1;
  for (int i = threadIdx.x; i < P; i += blockDim.x) sm[i] = i < n ? a[i] : sentinel;
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          const T x = sm[i], y = sm[ixj];
          if ((x > y) == up) {
            sm[i] = y;
            sm[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = sm[i];
  __syncthreads();
}

template <typename T>
__device__ void cta_sort(T* a, int64_t n, T* scratch, T* sm, T sentinel) {
  if (n <= 1) return;
  for (int64_t c0 = 0; c0 < n; c0 += kSortSmem)
    cta_bitonic(a + c0, (int)((n - c0) < kSortSmem ? (n - c0) : kSortSmem), sm, sentinel);
  T* src = a;
  T* dst = scratch;
  for (int64_t w = kSortSmem; w < n; w <<= 1) {
    for (int64_t lo = 0; lo < n; lo += 2 * w) {
      const int64_t mid = (lo + w < n) ? lo + w : n;
      const int64_t hi = (lo + 2 * w < n) ? lo + 2 * w : n;
      const int64_t la = mid - lo, lb = hi - mid;
      const T* A = src + lo;
      const T* B = src + mid;
      for (int64_t p = threadIdx.x; p < la + lb; p += blockDim.x) {
        int64_t l0 = p - lb > 0 ? p - lb : 0, h0 = p < la ? p : la;
        while (l0 < h0) {
          const int64_t md = (l0 + h0) >> 1;
          if (A[md] <= B[p - md - 1]) l0 = md + 1; else h0 = md;
        }
        const int64_t i = l0, j = p - l0;
        dst[lo + p] = (j >= lb || (i < la && A[i] <= B[j])) ? A[i] : B[j];
      }
    }
    __syncthreads();
    T* tmp = src;
    src = dst;
    dst = tmp;
  }
  if (src != a) {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a[i] = src[i];
    __syncthreads();
  }
}

// Long lists queued by k_merge_runs: CTA-wide sort (bitonic chunks in shared
// memory + merge-path passes through the stage range as scratch).
__global__ void __launch_bounds__(256) k_merge_big(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  __shared__ int64_t sm[kSortSmem];
  const int nbig = h->n_big;
  for (int i = blockIdx.x; i < nbig; i += gridDim.x) {
    const int32_t q = d.big_list[i];
    const int64_t qo = d.out_off[q], qe = d.out_off[q + 1];
    const int64_t len = qe - qo;
    int64_t* a = d.out_ids + qo;  // runs already concatenated here by k_assemble
    cta_sort<int64_t>(a, len, d.scratch + qo, sm, (int64_t)0x7fffffffffffffffll);
    int dup = 0;
    for (int64_t k = threadIdx.x; k + 1 < len; k += blockDim.x) dup |= (a[k] == a[k + 1]);
    if (__syncthreads_or(dup) && threadIdx.x == 0) h->dup = 1;
  }
}

}  // namespace tj
