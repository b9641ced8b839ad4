// QUAD tick kernels for sm_100a.  One persistent-grid launch sequence per
// tick; every size after the index build lives in DevHdr on the device.
//
//   K0  mbr / finalize           geometry.py:72-77, morton.py:100-104
//   K1  codes + level-F histogram, dense pyramid, heavy-node sub-pyramids,
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
  const int32_t* sidx;  // sorted input rows (points into oval[])
  double* sx;
  double* sy;
  int64_t* sid;
  // index
  uint32_t* pyr;
  int32_t* heavy_map;
  uint32_t* sub;
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
  Rect4* crect;
  int4* qwin;
  int32_t* nsub;
  int32_t* qsbase;
  // subqueries
  int32_t* sq_leaf;
  int32_t* sq_q;
  uint8_t* sq_cov;
  int32_t* sq_count;
  int32_t* ecount;          // result count per decode entry e (entry order of ssorted)
  Rect4* srect;             // clipped rect per subquery slot (query order)
  uint64_t* run_info;       // per slot: (start of its decoded run in stage) << 28 | result count
  int64_t* slot_out;       // per decode row e: start of its list in `stage`
  uint32_t* skey[2];
  int32_t* sval[2];
  const int32_t* ssorted;  // per leaf [isq slots asc][cov slots asc]
  const uint32_t* skey_sorted;
  int32_t* run_start;      // per subquery key (2*leaf + covering): first sorted position
  int32_t* run_end;        // one past the last
  int32_t* unit_leaf;      // join work unit -> leaf
  uint8_t* leaf_active;    // multi-GPU leaf-range sharding: leaf owned by this rank (nullptr: all)
  int64_t* leaf_wpre;      // exclusive prefix of the per-leaf work weight (sharding)
  int32_t* big_list;       // queries whose lists need the CTA-wide merge
  int64_t* run_off;        // per subquery slot: start of its decoded run in `stage`
  int64_t* scratch;        // R entries: merge-pass scratch for k_merge_big
  // join + outputs
  uint32_t* bitmap;
  int32_t* stage;          // decoded runs (input rows), decode order
  int64_t* out_ids;
  int64_t* out_off;
  // config
  int64_t SUB;  // sub-pyramid entries per heavy node
  int D;        // l_max - F
};

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

__global__ void __launch_bounds__(256) k_mbr(const Dev d) {
  DevHdr* h = d.h;
  const int64_t n = h->n;
  unsigned long long mnx = ~0ull, mny = ~0ull, mxx = 0ull, mxy = 0ull;
  TJ_GRID_STRIDE(i, n) {
    const unsigned long long kx = dkey(d.xs[i]), ky = dkey(d.ys[i]);
    mnx = kx < mnx ? kx : mnx;
    mny = ky < mny ? ky : mny;
    mxx = kx > mxx ? kx : mxx;
    mxy = ky > mxy ? ky : mxy;
  }
  mnx = shfl_min64(mnx);
  mny = shfl_min64(mny);
  mxx = shfl_max64(mxx);
  mxy = shfl_max64(mxy);
  if (lane_id() == 0) {
    atomicMin(&h->kmin_x, mnx);
    atomicMin(&h->kmin_y, mny);
    atomicMax(&h->kmax_x, mxx);
    atomicMax(&h->kmax_y, mxy);
  }
}

// Also detects whether object ids strictly increase in input order: then
// per-leaf blocks (input order) are id-sorted and per-query merges are merges
// of sorted runs.
// (and whether id == input row, the generator's arange ids: then the final
// lists need no id lookup at all)
__global__ void __launch_bounds__(256) k_monotone(const Dev d) {
  DevHdr* h = d.h;
  const int64_t n = h->n;
  int bad = 0, notid = 0;
  TJ_GRID_STRIDE(i, n) {
    const int64_t v = d.ids[i];
    notid |= (v != i);
    if (i + 1 < n) bad |= (v >= d.ids[i + 1]);
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
  const double side = (double)(1u << h->l_max);
  h->sx_max = h->wpos ? __ddiv_rn(side, h->width) : 0.0;
  h->sy_max = h->hpos ? __ddiv_rn(side, h->height) : 0.0;
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
  const uint32_t side = 1u << lmax;
  const double xa = h->xa, ya = h->ya, sx = h->sx_max, sy = h->sy_max;
  const int wpos = h->wpos, hpos = h->hpos;
  const int sh = 2 * (lmax - F);
  uint32_t* hist = d.pyr + pyr_off(F);
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x; b < n; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = b + threadIdx.x;
    uint32_t bin = 0xFFFFFFFFu;
    if (i < n) {
      const uint32_t ci = cell_of(d.xs[i], xa, sx, wpos, side);
      const uint32_t cj = cell_of(d.ys[i], ya, sy, hpos, side);
      const uint32_t z = morton2(ci, cj);
      d.code[i] = z;
      bin = z >> sh;
    }
    const uint32_t peers = __match_any_sync(0xffffffffu, bin);
    if (i < n && (int)(__ffs(peers) - 1) == lane_id()) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
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

// level-F nodes over the threshold get a dense sub-pyramid slot
__global__ void __launch_bounds__(256) k_heavy(const Dev d) {
  DevHdr* h = d.h;
  const int F = h->F;
  const int64_t cnt = int64_t(1) << (2 * F);
  const uint32_t* hist = d.pyr + pyr_off(F);
  const uint32_t th = (uint32_t)h->th;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x; b < cnt; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = b + threadIdx.x;
    bool split = false;
    if (z < cnt) {
      split = hist[z] > th;  // F < l_max here
      int slot = -1;
      if (split) {
        slot = atomicAdd(&h->n_heavy, 1);
        if (slot >= h->cap_heavy) {
          atomicOr(&h->abort, 8);
          slot = -1;
        }
      }
      d.heavy_map[z] = slot;
    }
    note_split(h, split, F + 1);
  }
}

__global__ void __launch_bounds__(256) k_zero_sub(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t cnt = (int64_t)h->n_heavy * d.SUB;
  TJ_GRID_STRIDE(i, cnt) d.sub[i] = 0u;
}

__global__ void __launch_bounds__(256) k_sub_hist(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t n = h->n;
  const int D = d.D;
  const uint32_t lowmask = (1u << (2 * D)) - 1u;
  const int64_t off = sub_off(D);
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x; b < n; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = b + threadIdx.x;
    int64_t bin = -1;
    if (i < n) {
      const uint32_t z = d.code[i];
      const int slot = d.heavy_map[z >> (2 * D)];
      if (slot >= 0) bin = (int64_t)slot * d.SUB + off + (z & lowmask);
    }
    const uint32_t peers = __match_any_sync(0xffffffffu, (unsigned long long)bin);
    if (bin >= 0 && (int)(__ffs(peers) - 1) == lane_id()) atomicAdd(&d.sub[bin], (uint32_t)__popc(peers));
  }
}

// relative level r (absolute F + r) from r + 1 inside each heavy node
__global__ void __launch_bounds__(256) k_sub_level(const Dev d, int r) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t per = int64_t(1) << (2 * r);
  const int64_t cnt = (int64_t)h->n_heavy * per;
  const uint32_t th = (uint32_t)h->th;
  const int l = h->F + r;
  const bool can_split = l < h->l_max;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x; b < cnt; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = b + threadIdx.x;
    bool split = false;
    if (e < cnt) {
      const int64_t slot = e >> (2 * r), loc = e & (per - 1);
      uint32_t* base = d.sub + slot * d.SUB;
      const uint4 c = *reinterpret_cast<const uint4*>(base + sub_off(r + 1) + 4 * loc);
      const uint32_t s = c.x + c.y + c.z + c.w;
      base[sub_off(r) + loc] = s;
      split = can_split && s > th;
    }
    note_split(h, split, l + 1);
  }
}

__global__ void k_finalize_index(DevHdr* h) {
  if (h->abort) return;
  h->Z = int64_t(1) << (2 * h->l_deep);
  const double side = (double)(1u << h->l_deep);
  h->sx_deep = h->wpos ? __ddiv_rn(side, h->width) : 0.0;
  h->sy_deep = h->hpos ? __ddiv_rn(side, h->height) : 0.0;
}

// object count of node (l, z); l >= 1
__device__ __forceinline__ uint32_t node_count(const Dev& d, int F, int l, uint32_t z) {
  if (l <= F) return d.pyr[pyr_off(l) + z];
  const int r = l - F;
  const int slot = d.heavy_map[z >> (2 * r)];
  if (slot < 0) return 0u;
  return d.sub[(int64_t)slot * d.SUB + sub_off(r) + (z & ((1u << (2 * r)) - 1u))];
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

// object -> leaf rank (quadtree.py:161-165) as the radix key, input row as value
__global__ void __launch_bounds__(256) k_obj_keys(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t n = h->n;
  const int sh = 2 * (h->l_max - h->l_deep);
  TJ_GRID_STRIDE(i, n) {
    d.okey[0][i] = d.zmap[d.code[i] >> sh] & kPayloadMask;
    d.oval[0][i] = (int32_t)i;
  }
}

// Payload gather into leaf order, one array per launch: each launch's random
// reads hit one 80 MB array (at 10M objects) that stays L2-resident, instead
// of three arrays (240 MB) thrashing the 126 MB L2 together.
template <typename T>
__global__ void __launch_bounds__(256) k_gather(const Dev d, const T* __restrict__ src, T* __restrict__ dst) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t n = h->n;
  TJ_GRID_STRIDE(p, n) dst[p] = src[d.sidx[p]];
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

// clip (geometry.py:80-88), window (quadtree.py:182-183), count subqueries
__global__ void __launch_bounds__(256) k_query_count(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t m = h->m;
  const double xa = h->xa, ya = h->ya, xb = h->xb, yb = h->yb;
  const double sx = h->sx_deep, sy = h->sy_deep;
  const int wpos = h->wpos, hpos = h->hpos, ld = h->l_deep;
  const uint32_t side = 1u << ld;
  TJ_GRID_STRIDE(q, m) {
    double cxa = d.qxa[q], cya = d.qya[q], cxb = d.qxb[q], cyb = d.qyb[q];
    cxa = cxa < xa ? xa : cxa;  // max(q.xa, mbr.xa)
    cya = cya < ya ? ya : cya;
    cxb = cxb > xb ? xb : cxb;  // min(q.xb, mbr.xb)
    cyb = cyb > yb ? yb : cyb;
    Rect4 r;
    r.xa = cxa; r.ya = cya; r.xb = cxb; r.yb = cyb;
    d.crect[q] = r;
    int cnt = 0;
    int4 w = make_int4(-1, -1, -1, -1);
    if (!(cxa > cxb || cya > cyb)) {
      w.x = (int)cell_of(cxa, xa, sx, wpos, side);
      w.y = (int)cell_of(cxb, xa, sx, wpos, side);
      w.z = (int)cell_of(cya, ya, sy, hpos, side);
      w.w = (int)cell_of(cyb, ya, sy, hpos, side);
      if (is_small(w)) {
        uint32_t key[4], rank[4];
        cnt = enum_small(w, ld, d.zmap, key, rank);
      } else {
        cnt = enum_window(w.x, w.y, w.z, w.w, ld, d.zmap, [](int, uint32_t, uint32_t) {});
      }
    }
    d.qwin[q] = w;
    d.nsub[q] = cnt;
  }
}

// Covering flag with the reference's exact op order (quadtree.py:219-231):
// w = width / 2^level; lxa = xa + li*w; covering iff qxa <= lxa and
// qxb >= min(lxa + w, mbr.xb), likewise in y.
__device__ __forceinline__ bool covers(const Rect4& q, int lev, uint32_t z, const DevHdr* h) {
  const double side = (double)(1u << lev);
  const double w = __ddiv_rn(h->width, side);
  const double hh = __ddiv_rn(h->height, side);
  const double li = (double)compact2(z), lj = (double)compact2(z >> 1);
  const double lxa = __dadd_rn(h->xa, __dmul_rn(li, w));
  const double lya = __dadd_rn(h->ya, __dmul_rn(lj, hh));
  double ux = __dadd_rn(lxa, w);
  ux = ux < h->xb ? ux : h->xb;
  double uy = __dadd_rn(lya, hh);
  uy = uy < h->yb ? uy : h->yb;
  return (q.xa <= lxa) && (q.xb >= ux) && (q.ya <= lya) && (q.yb >= uy);
}

// Subquery flags: bit 0 covering, bit 1 the query has a single subquery
// (its list needs no merge and is decoded straight into the output).
constexpr uint8_t kFlagCov = 1, kFlagSingle = 2;

__device__ __forceinline__ void emit_subquery(const Dev& d, int32_t slot, int64_t q, int n, int lev, uint32_t z,
                                              uint32_t rank, const Rect4& r, int cov_on) {
  const bool cv = cov_on && covers(r, lev, z, d.h);
  d.sq_leaf[slot] = (int32_t)rank;
  d.sq_q[slot] = (int32_t)q;
  d.srect[slot] = r;  // clipped rect per subquery slot (query order: sequential writes)
  d.sq_cov[slot] = (uint8_t)((cv ? kFlagCov : 0) | (n == 1 ? kFlagSingle : 0));
  // radix key = 2*leaf + covering: per leaf, intersecting subqueries then
  // covering ones, each in slot (= query input) order — directory.py:131
  d.skey[0][slot] = 2u * rank + (cv ? 1u : 0u);
  d.sval[0][slot] = slot;
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
  TJ_GRID_STRIDE(q, m) {
    const int n = d.nsub[q];
    if (n == 0) continue;
    const int4 w = d.qwin[q];
    const int32_t base = d.qsbase[q];
    const Rect4 r = d.crect[q];
    if (is_small(w)) {
      uint32_t key[4], rank[4];
      enum_small(w, ld, d.zmap, key, rank);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < n) emit_subquery(d, base + k, q, n, (int)(key[k] >> kLevelShift), key[k] & kPayloadMask, rank[k], r, cov_on);
      continue;
    }
    int cur[kMaxLevel + 1];
#pragma unroll
    for (int l = 0; l <= kMaxLevel; ++l) cur[l] = 0;
    if (n > 1) {
      enum_window(w.x, w.y, w.z, w.w, ld, d.zmap, [&](int lev, uint32_t, uint32_t) { cur[lev]++; });
      int run = 0;
#pragma unroll
      for (int l = 0; l <= kMaxLevel; ++l) {
        const int c = cur[l];
        cur[l] = run;
        run += c;
      }
    }
    enum_window(w.x, w.y, w.z, w.w, ld, d.zmap, [&](int lev, uint32_t z, uint32_t rank) {
      emit_subquery(d, base + cur[lev]++, q, n, lev, z, rank, r, cov_on);
    });
  }
}

// Run boundaries of the sorted subquery keys give every leaf's intersecting
// and covering block (directory.py:137-142) without atomics.
__global__ void __launch_bounds__(256) k_sq_runs(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t S = h->S;
  const uint32_t* ks = d.skey_sorted;
  TJ_GRID_STRIDE(e, S) {
    const uint32_t k = ks[e];
    if (e == 0 || ks[e - 1] != k) d.run_start[k] = (int32_t)e;
    if (e == S - 1 || ks[e + 1] != k) d.run_end[k] = (int32_t)(e + 1);
  }
}

// per-leaf occupancy / task statistics (engine.py:212-225,261-267)
__global__ void __launch_bounds__(256) k_leaf_stats(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t L = h->L;
  unsigned long long act = 0, s1 = 0, s2 = 0, tasks = 0, tests = 0, si = 0, sc = 0, pa = 0, sa = 0;
  TJ_GRID_STRIDE(r, L) {
    const int32_t a0 = d.run_start[2 * r], a1 = d.run_end[2 * r];
    const int32_t c0 = d.run_start[2 * r + 1], c1 = d.run_end[2 * r + 1];
    d.leaf_nisq[r] = a1 - a0;
    d.leaf_ncov[r] = c1 - c0;
    d.leaf_sbase[r] = (a1 > a0) ? a0 : c0;
    const unsigned long long no = (unsigned long long)d.leaf_nobj[r];
    const unsigned long long ni = (unsigned long long)(a1 - a0);
    si += ni;
    sc += (unsigned long long)(c1 - c0);
    if (no) {
      act += 1;
      s1 += no;
      s2 += no * no;
      if (ni) {
        tasks += 1;
        tests += no * ni;
        pa += no;
        sa += ni;
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
  if (lane_id() == 0) {
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
constexpr int kJoinThreads = 256;
constexpr int kJoinWarps = kJoinThreads / 32;
constexpr int kST = 32;   // subqueries per work unit (one warp, lane = subquery)
constexpr int kOTB = 32;  // 32-object blocks per work unit (1024 objects)

__device__ __forceinline__ bool leaf_on(const uint8_t* active, int64_t r) { return !active || active[r]; }

struct WordsIn {
  const int32_t* nobj;
  const int32_t* nisq;
  const uint8_t* active;
  __device__ int64_t operator()(int64_t r) const {
    const int64_t no = nobj[r], ni = nisq[r];
    return (no > 0 && ni > 0 && leaf_on(active, r)) ? ni * ((no + 31) / 32) : 0;
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
    return ((ni + kST - 1) / kST) * ((nb + kOTB - 1) / kOTB);
  }
};

// Multi-GPU leaf-range sharding: every rank builds the same
// index and subquery directory; leaves are cut into contiguous Morton ranges
// balanced by a work weight (objects x subqueries + both), and a rank joins,
// decodes and assembles only its own leaves — its per-query lists are the
// restriction of the full lists to its leaves (disjoint across ranks).
struct LeafWeightIn {
  const int32_t* nobj;
  const int32_t* nisq;
  const int32_t* ncov;
  __device__ int64_t operator()(int64_t r) const {
    const int64_t no = nobj[r], sq = (int64_t)nisq[r] + ncov[r];
    return no * sq + no + sq;
  }
};
struct PrefOut {
  int64_t* a;
  __device__ void operator()(int64_t i, int64_t ex, int64_t) const { a[i] = ex; }
};
__global__ void __launch_bounds__(256) k_shard_mark(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t T = h->shard_total > 0 ? h->shard_total : 1;
  const LeafWeightIn wt{d.leaf_nobj, d.leaf_nisq, d.leaf_ncov};
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
  TJ_GRID_STRIDE(s, h->S) d.ecount[s] = 0;
}

// Warp-level work units: (leaf, 32 intersecting subqueries, up to 1024
// objects), lane = subquery.  The lane keeps its clipped rect in registers;
// for each 32-object block of the leaf, the warp stages the block's (x, y)
// pairs in its shared-memory slice (prefetching the next block), and every
// lane walks the 32 objects (broadcast loads) with four chained closed fp64
// comparisons + one predicated OR per object (bitmap.py:89-94) — bit k of the
// lane's word is object 32b+k of the leaf's block (bitmap.py:95-97), i.e. the
// paper's bitmap word lands directly in the subquery's lane, no ballot or
// transpose.  Words are staged per warp and stored in the linear layout
// linear[s*blocks + b] (bitmap.py:105-111) with coalesced rows; popcounts
// (bitmap.py:114-119) stay in registers.  Warps never wait on each other.
struct __align__(16) XY {
  double x, y;
};

__device__ __forceinline__ XY load_obj(const Dev& d, int32_t ob, int k, int nobj) {
  XY o;
  if (k < nobj) {
    o.x = d.sx[ob + k];
    o.y = d.sy[ob + k];
  } else {  // padding objects never match (NaN compares false): padding bits stay zero
    o.x = __longlong_as_double(0x7ff8000000000000ll);
    o.y = o.x;
  }
  return o;
}

__global__ void __launch_bounds__(kJoinThreads, 4) k_join(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  __shared__ XY sobj[kJoinWarps][32];
  __shared__ uint32_t stile[kJoinWarps][32][kOTB + 1];
  const int64_t U = h->U;
  const int lane = lane_id(), wp = threadIdx.x >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  XY* so = sobj[wp];
  for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < U; u += nwarp) {
    const int64_t r = d.unit_leaf[u];
    const int nobj = d.leaf_nobj[r], nisq = d.leaf_nisq[r];
    const int nb = (nobj + 31) >> 5;
    const int n_ot = (nb + kOTB - 1) / kOTB;
    const int lu = (int)(u - d.leaf_ubase[r]);
    const int st = lu / n_ot, ot = lu - st * n_ot;
    const int s0 = st * kST, ns = min(kST, nisq - s0);
    const int b0 = ot * kOTB, nbt = min(kOTB, nb - b0);
    const int32_t ob = d.leaf_obase[r];
    const bool live = lane < ns;
    const int64_t e = (int64_t)d.leaf_sbase[r] + s0 + lane;  // decode entry of this lane's subquery
    Rect4 R;
    R.xa = R.ya = __longlong_as_double(0x7ff0000000000000ll);   // +inf: empty rect
    R.xb = R.yb = __longlong_as_double((long long)0xfff0000000000000ull);  // -inf
    if (live) R = d.srect[d.ssorted[e]];  // the one random access per subquery of the regrouping
    uint32_t cnt = 0;
    XY nxt = load_obj(d, ob, b0 * 32 + lane, nobj);
    for (int bl = 0; bl < nbt; ++bl) {
      so[lane] = nxt;
      __syncwarp();
      if (bl + 1 < nbt) nxt = load_obj(d, ob, (b0 + bl + 1) * 32 + lane, nobj);
      uint32_t w = 0;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const XY o = so[k];
        // closed test, chained predicates: 4 DSETP + 1 predicated OR per object
        asm("{\n\t.reg .pred p;\n\t"
            "setp.ge.f64 p, %1, %2;\n\t"
            "setp.le.and.f64 p, %1, %3, p;\n\t"
            "setp.ge.and.f64 p, %4, %5, p;\n\t"
            "setp.le.and.f64 p, %4, %6, p;\n\t"
            "@p or.b32 %0, %0, %7;\n\t}"
            : "+r"(w)
            : "d"(o.x), "d"(R.xa), "d"(R.xb), "d"(o.y), "d"(R.ya), "d"(R.yb), "r"(1u << k));
      }
      stile[wp][lane][bl] = w;
      cnt += __popc(w);
      __syncwarp();
    }
    uint32_t* out = d.bitmap + d.leaf_woff[r] + (int64_t)s0 * nb + b0;
    if (nbt == nb) {
      const int tot = ns * nb;
      for (int e = lane; e < tot; e += 32) {
        const int s = e / nb;
        out[e] = stile[wp][s][e - s * nb];
      }
    } else {
      const int tot = ns * nbt;
      for (int e = lane; e < tot; e += 32) {
        const int s = e / nbt, c = e - s * nbt;
        out[(int64_t)s * nb + c] = stile[wp][s][c];
      }
    }
    if (live) {
      if (n_ot == 1) d.ecount[e] = (int32_t)cnt;
      else atomicAdd(&d.ecount[e], (int32_t)cnt);
    }
    __syncwarp();
  }
}

// covering subqueries' counts = their leaf's whole block
__global__ void __launch_bounds__(256) k_cov_counts(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int lane = lane_id();
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < h->L; r += nwarp) {
    const int nc = d.leaf_ncov[r];
    if (nc == 0 || !leaf_on(d.leaf_active, r)) continue;
    const int32_t base = d.leaf_sbase[r] + d.leaf_nisq[r];
    const int32_t nobj = d.leaf_nobj[r];
    for (int c = lane; c < nc; c += 32) d.ecount[base + c] = nobj;
  }
}

// ===========================================================================
// K4: decode, covering expansion, canonical per-query lists
// ===========================================================================
// Result counts: an intersecting subquery contributes its popcount, a
// covering one its leaf's whole block (decode.py:83-99).
// (run_info is filled per slot by the decode-order scan, RowOut: one packed
// random write per subquery instead of two)
constexpr int kRunCountBits = 28;
__device__ __forceinline__ int64_t slot_count(const Dev& d, int32_t slot) {
  return (int64_t)(d.run_info[slot] & ((1ull << kRunCountBits) - 1));
}
__device__ __forceinline__ int64_t slot_off(const Dev& d, int32_t slot) {
  return (int64_t)(d.run_info[slot] >> kRunCountBits);
}

// decode order: entries e of `ssorted` (leaf by leaf, intersecting then
// covering) — every leaf's decoded lists form one contiguous chunk of `stage`
struct RowCntIn {
  Dev d;
  __device__ int64_t operator()(int64_t e) const { return (int64_t)d.ecount[e]; }
};
struct RowOut {
  Dev d;
  __device__ void operator()(int64_t e, int64_t ex, int64_t v) const {
    d.slot_out[e] = ex;  // row e's list starts at stage[ex] ...
    d.run_info[d.ssorted[e]] = ((uint64_t)ex << kRunCountBits) | (uint64_t)v;  // ... = slot's run
  }
};
// output order: queries in input order, lists concatenated (ResultSet CSR)
struct QueryCntIn {
  Dev d;
  __device__ int64_t operator()(int64_t q) const {
    const int k = d.nsub[q];
    const int32_t s0 = d.qsbase[q];
    int64_t c = 0;
    for (int j = 0; j < k; ++j) c += slot_count(d, s0 + j);
    return c;
  }
};

__global__ void k_close_offsets(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  d.out_off[h->m] = h->R;
  if (h->R != h->R_check) h->count_mismatch = 1;  // CountMismatch (bitmap.py:131-132)
  if (h->R >= (int64_t(1) << (64 - kRunCountBits))) h->count_mismatch = 1;  // run_info packing bound
}

constexpr int kDecodeThreads = 256;
constexpr int kDecodeBatch = 512;  // per-warp staging of 32 rows' decoded rows

// Alg. 4 (decode.py:40-99, bitmap.py:122-133, engine.py:306-326) as warp
// tasks over the join's work units (leaf, 32 intersecting subquery rows):
// lane = row; the lane walks its row's words and, for every set bit
// (ascending = block order), puts the object's input row at the row's next
// position.  The 32 rows' lists are adjacent in `stage` (decode order), so
// they are assembled in a per-warp shared-memory buffer and stored with
// full-width coalesced writes.  No block barriers: warps are independent.
__global__ void __launch_bounds__(kDecodeThreads) k_decode_rows(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  __shared__ int32_t sbatch[kDecodeThreads / 32][kDecodeBatch];
  const int64_t U = h->U, S = h->S, R = h->R;
  const int lane = lane_id(), wp = threadIdx.x >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int32_t* wbuf = sbatch[wp];
  for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < U; u += nwarp) {
    const int64_t r = d.unit_leaf[u];
    const int nobj = d.leaf_nobj[r], ni = d.leaf_nisq[r];
    const int nb = (nobj + 31) >> 5;
    const int n_ot = (nb + kOTB - 1) / kOTB;
    const int lu = (int)(u - d.leaf_ubase[r]);
    const int st = lu / n_ot, ot = lu - st * n_ot;
    if (ot != 0) continue;  // one decode task per 32-row chunk (all object tiles at once)
    const int r0 = st * kST, nrow = min(32, ni - r0);
    const int32_t sb = d.leaf_sbase[r];
    const int32_t* ids = d.sidx + d.leaf_obase[r];  // input rows of the leaf's objects (block order)
    const bool live = lane < nrow;
    const int64_t e = (int64_t)sb + r0 + lane;
    const int64_t off = live ? d.slot_out[e] : 0;
    const int64_t base = __shfl_sync(0xffffffffu, off, 0);
    const int64_t e_end = (int64_t)sb + r0 + nrow;
    const int64_t end = e_end < S ? d.slot_out[e_end] : R;
    const int64_t total = end - base;
    const bool buffered = total <= kDecodeBatch;
    if (live) {
      const uint32_t* words = d.bitmap + d.leaf_woff[r] + (int64_t)(r0 + lane) * nb;
      if (buffered) {
        int32_t* dst = wbuf + (off - base);  // shared memory
        for (int b = 0; b < nb; ++b) {
          uint32_t w = words[b];
          while (w) {
            const int bit = __ffs(w) - 1;
            w &= w - 1;
            *dst++ = ids[b * 32 + bit];
          }
        }
      } else {
        int32_t* dst = d.stage + off;  // global
        for (int b = 0; b < nb; ++b) {
          uint32_t w = words[b];
          while (w) {
            const int bit = __ffs(w) - 1;
            w &= w - 1;
            *dst++ = ids[b * 32 + bit];
          }
        }
      }
    }
    __syncwarp();
    if (buffered)
      for (int k = lane; k < (int)total; k += 32) d.stage[base + k] = wbuf[k];
    __syncwarp();
  }
}

// covering subqueries copy the whole block (decode.py:83-99), a warp per leaf
__global__ void __launch_bounds__(256) k_decode_cov(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int lane = lane_id();
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long covres = 0;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < h->L; r += nwarp) {
    const int nc = d.leaf_ncov[r];
    if (nc == 0 || !leaf_on(d.leaf_active, r)) continue;
    const int nobj = d.leaf_nobj[r];
    if (nobj == 0) continue;
    const int32_t* ids = d.sidx + d.leaf_obase[r];
    const int32_t e0 = d.leaf_sbase[r] + d.leaf_nisq[r];
    for (int c = 0; c < nc; ++c) {
      int32_t* dst = d.stage + d.slot_out[e0 + c];
      for (int k = lane; k < nobj; k += 32) dst[k] = ids[k];
    }
    if (lane == 0) covres += (unsigned long long)nobj * nc;
  }
  if (lane == 0 && covres) atomicAdd(&h->cov_results, covres);
}


// Per-query canonical lists (decode.py:102-123: concatenate, sort, reject
// duplicates), assembled from the decoded runs (input rows, int32) into the
// output CSR (object ids, int64), written in query order.  Monotone ids (ids
// increase with input row — every generated workload): each run is sorted by
// row, so sorting by row sorts by id; one run is a copy, two runs a merge-path
// merge in registers, more runs a register bitonic sort; ids are looked up
// (ids[row]) at the final store.  Otherwise rows are turned into ids first and
// sorted by id, with a duplicate check.  Lists longer than 64 (or > 32 runs)
// are concatenated into the output and queued for the CTA-wide k_merge_big.
template <typename T>
__device__ __forceinline__ T bitonic_step(T v, int i, int j, int k) {
  const T o = __shfl_xor_sync(0xffffffffu, v, j);
  const bool up = (i & k) == 0, low = (i & j) == 0;
  return (low == up) ? (o < v ? o : v) : (o > v ? o : v);
}
// ascending bitonic sort of 32 (r = 1) or 64 (r = 2, index = reg*32 + lane) keys in registers
template <typename T, int NR>
__device__ __forceinline__ void warp_sort(T (&v)[2]) {
  const int lane = lane_id();
#pragma unroll
  for (int k = 2; k <= 32 * NR; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j == 32) {  // partner is the other register of the same lane (k == 64: ascending)
        const T lo = v[0] < v[1] ? v[0] : v[1], hi = v[0] < v[1] ? v[1] : v[0];
        v[0] = lo;
        v[1] = hi;
      } else {
#pragma unroll
        for (int r = 0; r < NR; ++r) v[r] = bitonic_step(v[r], r * 32 + lane, j, k);
      }
    }
}

// value at concatenated index t (reg t/32, lane t%32)
template <int NR>
__device__ __forceinline__ int32_t vget(const int32_t (&v)[2], int t) {
  const int32_t a = __shfl_sync(0xffffffffu, v[0], t & 31);
  if (NR == 1) return a;
  const int32_t b = __shfl_sync(0xffffffffu, v[1], t & 31);
  return t < 32 ? a : b;
}

// merge path of two sorted runs A = [0, na), B = [na, cnt) held in registers:
// output position p takes min(A[i], B[p-i]) at the split i found by binary search
template <int NR>
__device__ __forceinline__ void warp_merge2(const int32_t (&v)[2], int na, int cnt, int32_t (&o)[2]) {
  const int lane = lane_id();
  const int nb = cnt - na;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int p = r * 32 + lane;
    int lo = p - nb > 0 ? p - nb : 0, hi = p < na ? p : na;
    if (p >= cnt) lo = hi = 0;
    while (__any_sync(0xffffffffu, lo < hi)) {
      const int mid = (lo + hi) >> 1;
      const int ia = mid, ib = na + p - mid - 1;
      const int32_t va = vget<NR>(v, ia < 63 ? ia : 63);
      const int32_t vb = vget<NR>(v, ib > 0 ? (ib < 63 ? ib : 63) : 0);
      if (lo < hi) {
        if (va < vb) lo = mid + 1; else hi = mid;
      }
    }
    const int i = lo, j = p - lo;
    const int32_t ai = vget<NR>(v, i < na ? i : 0);
    const int32_t bj = vget<NR>(v, j < nb ? na + j : 0);
    o[r] = (j >= nb || (i < na && ai < bj)) ? ai : bj;
  }
}

__global__ void __launch_bounds__(256) k_assemble(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const bool mono = !h->not_monotone;
  const int64_t m = h->m;
  const int lane = lane_id();
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t* __restrict__ ids = d.ids;
  const int32_t* __restrict__ stage = d.stage;
  const bool ident = !h->not_identity;
  auto idof = [&](int32_t row) -> int64_t { return ident ? (int64_t)row : ids[row]; };
  for (int64_t q0 = gw * 32; q0 < m; q0 += nwarp * 32) {
    const int64_t ql = q0 + lane;
    int kl = 0;
    int32_t s0l = 0;
    int64_t qol = 0, cntl = 0;
    if (ql < m) {
      kl = d.nsub[ql];
      s0l = d.qsbase[ql];
      qol = d.out_off[ql];
      cntl = d.out_off[ql + 1] - qol;
    }
    // single-run lists (sorted already when ids are monotone; length <= 1
    // otherwise): flattened copy of the warp's output range — independent
    // loads, coalesced stores
    const bool single = kl == 1 && (mono || cntl <= 1);
    const int64_t srcl = (single && cntl > 0) ? slot_off(d, s0l) : -1;
    const bool done = kl == 0 || cntl == 0 || single;
    {
      const int64_t lo = __shfl_sync(0xffffffffu, qol, 0);
      const int64_t hi = __shfl_sync(0xffffffffu, qol + cntl, 31);
      const int64_t hi2 = q0 + 32 <= m ? hi : d.out_off[m];
      const int nvalid = (int)min((int64_t)32, m - q0);
      const uint32_t rel = lane < nvalid ? (uint32_t)(qol - lo) : 0xffffffffu;
      constexpr int U = 4;  // 4 x 32 outputs per step: 4 independent loads in flight per lane
      for (int64_t p0 = lo; p0 < hi2; p0 += 32 * U) {
        int64_t src[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t pr = (uint32_t)(p0 - lo) + u * 32 + lane;
          int j = 0;
#pragma unroll
          for (int step = 16; step > 0; step >>= 1) {
            const uint32_t v = __shfl_sync(0xffffffffu, rel, j + step);
            if (v <= pr) j += step;
          }
          const uint32_t relj = __shfl_sync(0xffffffffu, rel, j);
          const int64_t srcj = __shfl_sync(0xffffffffu, srcl, j);
          src[u] = (p0 + u * 32 + lane < hi2 && srcj >= 0) ? srcj + (pr - relj) : -1;
        }
        int32_t val[U];
#pragma unroll
        for (int u = 0; u < U; ++u) val[u] = src[u] >= 0 ? stage[src[u]] : 0;
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (src[u] >= 0) d.out_ids[p0 + u * 32 + lane] = idof(val[u]);
      }
    }
    // monotone ids, 2..4 runs: lane-per-query k-way merge straight from the
    // decoded runs (heads in registers, one-element lookahead per run); the
    // 32 queries of the warp merge concurrently
    const bool lanemerge = mono && !done && kl >= 2 && kl <= 4 && cntl <= 512;
    if (__any_sync(0xffffffffu, lanemerge) && lanemerge) {
      int64_t pos[4], end[4];
      int32_t head[4];
      int64_t acc = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        pos[j] = 0;
        end[j] = 0;
        head[j] = 0x7fffffff;
        if (j < kl) {
          const int64_t c = slot_count(d, s0l + j);
          pos[j] = slot_off(d, s0l + j);
          end[j] = pos[j] + c;
          acc += c;
          if (c > 0) head[j] = stage[pos[j]];
        }
      }
      int64_t* out = d.out_ids + qol;
      for (int64_t o = 0; o < cntl; ++o) {
        int bj = 0;
        int32_t bv = head[0];
#pragma unroll
        for (int j = 1; j < 4; ++j)
          if (head[j] < bv) {
            bv = head[j];
            bj = j;
          }
        out[o] = idof(bv);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j == bj) {
            ++pos[j];
            head[j] = pos[j] < end[j] ? stage[pos[j]] : 0x7fffffff;
            if (((pos[j] & 7) == 0) && pos[j] + 16 < end[j])  // pull the sector two ahead into L1
              asm volatile("prefetch.global.L1 [%0];" ::"l"(stage + pos[j] + 16));
          }
      }
    }
    // short multi-run lists (<= 64 entries, <= 32 runs): one query at a
    // time, the next query's run metadata in flight meanwhile
    const bool smallq = !done && !lanemerge && cntl <= 64 && kl <= 32;
    unsigned pend = __ballot_sync(0xffffffffu, smallq);
    {
      auto meta = [&](int src, int64_t& c, int64_t& o) {
        const int kk = __shfl_sync(0xffffffffu, kl, src);
        const int32_t ss = __shfl_sync(0xffffffffu, s0l, src);
        c = 0;
        o = 0;
        if (lane < kk) {
          c = slot_count(d, ss + lane);
          o = slot_off(d, ss + lane);
        }
      };
      int cur = pend ? __ffs(pend) - 1 : -1;
      pend &= pend - 1;
      int64_t c_cur = 0, o_cur = 0;
      if (cur >= 0) meta(cur, c_cur, o_cur);
      while (cur >= 0) {
        const int nxt = pend ? __ffs(pend) - 1 : -1;
        pend &= pend - 1;
        int64_t c_nxt = 0, o_nxt = 0;
        if (nxt >= 0) meta(nxt, c_nxt, o_nxt);
        const int k = __shfl_sync(0xffffffffu, kl, cur);
        const int64_t qo = __shfl_sync(0xffffffffu, qol, cur);
        const int cnt = (int)__shfl_sync(0xffffffffu, cntl, cur);
        const int cinc = warp_incl_scan((int)c_cur);
        const int cexc = cinc - (int)c_cur;
        int32_t v[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int x = r * 32 + lane;
          int jj = 0;
#pragma unroll
          for (int step = 16; step > 0; step >>= 1) {
            const int st = __shfl_sync(0xffffffffu, cexc, jj + step);
            if (jj + step < k && st <= x) jj += step;
          }
          const int stj = __shfl_sync(0xffffffffu, cexc, jj);
          const int64_t ofj = __shfl_sync(0xffffffffu, o_cur, jj);
          v[r] = x < cnt ? stage[ofj + (x - stj)] : 0x7fffffff;
        }
        if (mono) {
          int32_t o[2];
          if (k == 2) {
            const int na = __shfl_sync(0xffffffffu, (int)c_cur, 0);
            if (cnt <= 32) warp_merge2<1>(v, na, cnt, o); else warp_merge2<2>(v, na, cnt, o);
          } else {
            if (cnt <= 32) warp_sort<int32_t, 1>(v); else warp_sort<int32_t, 2>(v);
            o[0] = v[0];
            o[1] = v[1];
          }
#pragma unroll
          for (int r = 0; r < 2; ++r)
            if (r * 32 + lane < cnt) d.out_ids[qo + r * 32 + lane] = idof(o[r]);
        } else {
          int64_t w[2];
#pragma unroll
          for (int r = 0; r < 2; ++r) w[r] = r * 32 + lane < cnt ? idof(v[r]) : (int64_t)0x7fffffffffffffffll;
          if (cnt <= 32) warp_sort<int64_t, 1>(w); else warp_sort<int64_t, 2>(w);
          int dup = 0;
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int x = r * 32 + lane;
            if (x < cnt) d.out_ids[qo + x] = w[r];
            // neighbour of x is x+1: next lane, or register 1 lane 0
            const int64_t nb0 = __shfl_down_sync(0xffffffffu, w[r], 1);
            const int64_t wrap = __shfl_sync(0xffffffffu, w[1], 0);
            const int64_t nbv = lane < 31 ? nb0 : (r == 0 ? wrap : (int64_t)0x7fffffffffffffffll);
            dup |= (x + 1 < cnt) && nbv == w[r];
          }
          if (__any_sync(0xffffffffu, dup) && lane == 0) h->dup = 1;
        }
        cur = nxt;
        c_cur = c_nxt;
        o_cur = o_nxt;
      }
    }
    // long lists / many runs: concatenate the runs (as ids) into the output
    // and queue the query for the CTA-wide sort
    unsigned todo = __ballot_sync(0xffffffffu, !done && !smallq && !lanemerge);
    while (todo) {
      const int src_lane = __ffs(todo) - 1;
      todo &= todo - 1;
      const int k = __shfl_sync(0xffffffffu, kl, src_lane);
      const int32_t s0 = __shfl_sync(0xffffffffu, s0l, src_lane);
      const int64_t qo = __shfl_sync(0xffffffffu, qol, src_lane);
      int64_t pre = 0;
      for (int j0 = 0; j0 < k; j0 += 32) {
        const int j = j0 + lane;
        int64_t cj = 0, oj = 0;
        if (j < k) {
          cj = slot_count(d, s0 + j);
          oj = slot_off(d, s0 + j);
        }
        const int64_t inc = warp_incl_scan(cj);
        const int64_t seg = __shfl_sync(0xffffffffu, inc, 31);
        for (int64_t x0 = 0; x0 < seg; x0 += 32) {  // flattened copy of these <= 32 runs
          const int64_t x = x0 + lane;
          int jj = 0;
#pragma unroll
          for (int step = 16; step > 0; step >>= 1) {
            const int64_t v = __shfl_sync(0xffffffffu, inc - cj, jj + step);  // exclusive starts
            if (v <= x && j0 + jj + step < k) jj += step;
          }
          const int64_t st_j = __shfl_sync(0xffffffffu, inc - cj, jj);
          const int64_t of_j = __shfl_sync(0xffffffffu, oj, jj);
          if (x < seg) d.out_ids[qo + pre + x] = idof(stage[of_j + (x - st_j)]);
        }
        pre += seg;
      }
      if (lane == 0) {
        const int idx = atomicAdd(&h->n_big, 1);
        d.big_list[idx] = (int32_t)(q0 + src_lane);
      }
    }
  }
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
