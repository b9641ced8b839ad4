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
  int64_t* slot_out;
  uint32_t* skey[2];
  int32_t* sval[2];
  const int32_t* ssorted;  // per leaf [isq slots asc][cov slots asc]
  // join + outputs
  uint32_t* bitmap;
  int64_t* stage;
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
__global__ void __launch_bounds__(256) k_monotone(const Dev d) {
  DevHdr* h = d.h;
  const int64_t n = h->n;
  int bad = 0;
  TJ_GRID_STRIDE(i, n - 1) { bad |= (d.ids[i] >= d.ids[i + 1]); }
  if (__any_sync(0xffffffffu, bad) && lane_id() == 0) atomicOr(&h->not_monotone, 1);
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

__global__ void __launch_bounds__(256) k_gather(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t n = h->n;
  TJ_GRID_STRIDE(p, n) {
    const int32_t i = d.sidx[p];
    d.sx[p] = d.xs[i];
    d.sy[p] = d.ys[i];
    d.sid[p] = d.ids[i];
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
      cnt = enum_window(w.x, w.y, w.z, w.w, ld, d.zmap, [](int, uint32_t, uint32_t) {});
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
      const int32_t slot = base + cur[lev]++;
      const bool cv = cov_on && covers(r, lev, z, h);
      d.sq_leaf[slot] = (int32_t)rank;
      d.sq_q[slot] = (int32_t)q;
      d.sq_cov[slot] = cv ? 1 : 0;
      atomicAdd(cv ? &d.leaf_ncov[rank] : &d.leaf_nisq[rank], 1);
    });
  }
}

// key = 2*leaf + covering: per leaf, intersecting subqueries then covering
// ones, each in slot (= query input) order — directory.py:131 lexsort
__global__ void __launch_bounds__(256) k_sq_keys(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t S = h->S;
  TJ_GRID_STRIDE(s, S) {
    d.skey[0][s] = 2u * (uint32_t)d.sq_leaf[s] + (uint32_t)d.sq_cov[s];
    d.sval[0][s] = (int32_t)s;
  }
}

struct LeafSubIn {
  const int32_t* nisq;
  const int32_t* ncov;
  __device__ int64_t operator()(int64_t r) const { return (int64_t)nisq[r] + ncov[r]; }
};

// per-leaf occupancy / task statistics (engine.py:212-225,261-267)
__global__ void __launch_bounds__(256) k_leaf_stats(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t L = h->L;
  unsigned long long act = 0, s1 = 0, s2 = 0, tasks = 0, tests = 0, si = 0, sc = 0, pa = 0, sa = 0;
  TJ_GRID_STRIDE(r, L) {
    const unsigned long long no = (unsigned long long)d.leaf_nobj[r];
    const unsigned long long ni = (unsigned long long)d.leaf_nisq[r];
    si += ni;
    sc += (unsigned long long)d.leaf_ncov[r];
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
constexpr int kST = 64;   // subqueries per work unit
constexpr int kOTB = 32;  // 32-object blocks per work unit (1024 objects)

struct WordsIn {
  const int32_t* nobj;
  const int32_t* nisq;
  __device__ int64_t operator()(int64_t r) const {
    const int64_t no = nobj[r], ni = nisq[r];
    return (no > 0 && ni > 0) ? ni * ((no + 31) / 32) : 0;
  }
};
struct UnitsIn {
  const int32_t* nobj;
  const int32_t* nisq;
  __device__ int64_t operator()(int64_t r) const {
    const int64_t no = nobj[r], ni = nisq[r];
    if (!(no > 0 && ni > 0)) return 0;
    const int64_t nb = (no + 31) / 32;
    return ((ni + kST - 1) / kST) * ((nb + kOTB - 1) / kOTB);
  }
};

__global__ void __launch_bounds__(256) k_zero_counts(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  TJ_GRID_STRIDE(s, h->S) d.sq_count[s] = 0;
}

// One CTA per work unit (leaf, 64-subquery tile, 1024-object tile).  Each warp
// holds one 32-object block in registers (lane = object), walks 32
// subqueries whose clipped rects sit in shared memory, and turns the four
// closed fp64 comparisons (bitmap.py:89-94) into one bitmap word per
// subquery with a ballot: bit k of word (s, b) = object 32b+k of the leaf's
// block (bitmap.py:95-97).  Words are staged per tile and stored in the
// linear layout linear[s*blocks + b] (bitmap.py:105-111) with coalesced rows;
// popcounts (bitmap.py:114-119) accumulate in shared memory.
__global__ void __launch_bounds__(kJoinThreads) k_join(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  __shared__ Rect4 rect[kST];
  __shared__ uint32_t tile[kST][kOTB + 1];
  __shared__ uint32_t cnt[kST];
  __shared__ int32_t slots[kST];
  const int64_t U = h->U, L = h->L;
  const int t = threadIdx.x, wp = t >> 5, lane = t & 31;
  for (int64_t u = blockIdx.x; u < U; u += gridDim.x) {
    // leaf owning unit u: last r with ubase[r] <= u
    int64_t lo = 0, hi = L;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (d.leaf_ubase[mid] <= u) lo = mid; else hi = mid;
    }
    const int64_t r = lo;
    const int nobj = d.leaf_nobj[r], nisq = d.leaf_nisq[r];
    const int nb = (nobj + 31) >> 5;
    const int n_ot = (nb + kOTB - 1) / kOTB;
    const int lu = (int)(u - d.leaf_ubase[r]);
    const int st = lu / n_ot, ot = lu - st * n_ot;
    const int s0 = st * kST, ns = min(kST, nisq - s0);
    const int b0 = ot * kOTB, nbt = min(kOTB, nb - b0);
    const int32_t sb = d.leaf_sbase[r];
    const int32_t ob = d.leaf_obase[r];
    if (t < ns) {
      const int32_t slot = d.ssorted[sb + s0 + t];
      slots[t] = slot;
      rect[t] = d.crect[d.sq_q[slot]];
      cnt[t] = 0;
    }
    __syncthreads();
    const int nchunk = (ns + 31) >> 5;
    const int npairs = nchunk * nbt;
    for (int p = wp; p < npairs; p += kJoinWarps) {
      const int sc = p / nbt, bl = p - sc * nbt;
      const int k = (b0 + bl) * 32 + lane;
      const bool valid = k < nobj;
      const double x = valid ? d.sx[ob + k] : 0.0;
      const double y = valid ? d.sy[ob + k] : 0.0;
      const int smax = min(32, ns - sc * 32);
      uint32_t mine = 0;
      for (int q = 0; q < smax; ++q) {
        const Rect4 R = rect[sc * 32 + q];
        const bool in = valid && (x >= R.xa) && (x <= R.xb) && (y >= R.ya) && (y <= R.yb);
        const uint32_t wrd = __ballot_sync(0xffffffffu, in);
        if (lane == q) mine = wrd;
      }
      if (lane < smax) {
        tile[sc * 32 + lane][bl] = mine;
        atomicAdd(&cnt[sc * 32 + lane], (uint32_t)__popc(mine));
      }
    }
    __syncthreads();
    uint32_t* out = d.bitmap + d.leaf_woff[r] + (int64_t)s0 * nb + b0;
    if (nbt == nb) {
      const int tot = ns * nb;
      for (int e = t; e < tot; e += kJoinThreads) {
        const int s = e / nb;
        out[e] = tile[s][e - s * nb];
      }
    } else {
      const int tot = ns * nbt;
      for (int e = t; e < tot; e += kJoinThreads) {
        const int s = e / nbt, c = e - s * nbt;
        out[(int64_t)s * nb + c] = tile[s][c];
      }
    }
    if (t < ns) {
      if (n_ot == 1) d.sq_count[slots[t]] = (int32_t)cnt[t];
      else atomicAdd(&d.sq_count[slots[t]], (int32_t)cnt[t]);
    }
    __syncthreads();
  }
}

// ===========================================================================
// K4: decode, covering expansion, canonical per-query lists
// ===========================================================================
struct SlotCntIn {
  const uint8_t* cov;
  const int32_t* leaf;
  const int32_t* nobj;
  const int32_t* count;
  __device__ int64_t operator()(int64_t s) const {
    return cov[s] ? (int64_t)nobj[leaf[s]] : (int64_t)count[s];
  }
};

__global__ void __launch_bounds__(256) k_query_offsets(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t m = h->m, S = h->S;
  TJ_GRID_STRIDE(q, m + 1) {
    const int64_t sb = q < m ? d.qsbase[q] : S;
    d.out_off[q] = sb < S ? d.slot_out[sb] : h->R;
  }
}

// a query's lists go straight to the output when they need no merge
__device__ __forceinline__ int64_t* dst_of(const Dev& d, int32_t q, int not_mono) {
  return (d.nsub[q] == 1 && !not_mono) ? d.out_ids : d.stage;
}

// Alg. 4: one warp per intersecting subquery row; lanes take words, popcount,
// warp-scan, then write the ids of set bits (block order) at the prefix
// offsets (decode.py:40-49, bitmap.py:122-133, engine.py:306-326).
__global__ void __launch_bounds__(256) k_decode(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int64_t L = h->L;
  const int not_mono = h->not_monotone;
  const int lane = lane_id();
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  // walk tasks' rows: row index e over the concatenation of all leaves' isq blocks
  const int64_t S = h->S;
  for (int64_t e = gw; e < S; e += nwarp) {
    const int32_t slot = d.ssorted[e];
    if (d.sq_cov[slot]) continue;
    const int32_t r = d.sq_leaf[slot];
    const int nobj = d.leaf_nobj[r];
    if (nobj == 0) continue;
    const int row = (int)(e - d.leaf_sbase[r]);
    const int nb = (nobj + 31) >> 5;
    const uint32_t* words = d.bitmap + d.leaf_woff[r] + (int64_t)row * nb;
    int64_t* dst = dst_of(d, d.sq_q[slot], not_mono) + d.slot_out[slot];
    const int64_t* ids = d.sid + d.leaf_obase[r];
    int64_t base = 0;
    for (int c0 = 0; c0 < nb; c0 += 32) {
      const int b = c0 + lane;
      uint32_t w = b < nb ? words[b] : 0u;
      const int pc = __popc(w);
      const int inc = warp_incl_scan(pc);
      int64_t pos = base + inc - pc;
      while (w) {
        const int bit = __ffs(w) - 1;
        w &= w - 1;
        dst[pos++] = ids[b * 32 + bit];
      }
      base += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
  (void)L;
}

// covering subqueries copy the whole leaf block (decode.py:83-99)
__global__ void __launch_bounds__(256) k_cover(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort) return;
  const int not_mono = h->not_monotone;
  const int lane = lane_id();
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t S = h->S;
  unsigned long long covres = 0;
  for (int64_t s = gw; s < S; s += nwarp) {
    if (!d.sq_cov[s]) continue;
    const int32_t r = d.sq_leaf[s];
    const int nobj = d.leaf_nobj[r];
    if (nobj == 0) continue;
    int64_t* dst = dst_of(d, d.sq_q[s], not_mono) + d.slot_out[s];
    const int64_t* ids = d.sid + d.leaf_obase[r];
    for (int k = lane; k < nobj; k += 32) dst[k] = ids[k];
    covres += (unsigned long long)nobj;
  }
  if (lane == 0 && covres) atomicAdd(&h->cov_results, covres);
}

// Per-query merge of sorted runs (one run per subquery; runs are disjoint by
// the space partition) by rank: an element's output index is its index in its
// own run plus the number of smaller elements in every other run
// (decode.py:102-123 concatenate+sort, done without a sort).
__global__ void __launch_bounds__(256) k_merge_runs(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort || h->not_monotone) return;
  const int64_t m = h->m;
  const int lane = lane_id();
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int64_t q = gw; q < m; q += nwarp) {
    const int k = d.nsub[q];
    if (k <= 1) continue;
    const int32_t s0 = d.qsbase[q];
    const int64_t qo = d.out_off[q], qe = d.out_off[q + 1];
    const int64_t* src = d.stage;
    for (int64_t p = qo + lane; p < qe; p += 32) {
      const int64_t key = src[p];
      int64_t rank = 0;
      for (int j = 0; j < k; ++j) {
        const int64_t a = d.slot_out[s0 + j];
        const int64_t b = (j + 1 < k) ? d.slot_out[s0 + j + 1] : qe;
        if (p >= a && p < b) {
          rank += p - a;
        } else {
          int64_t lo = a, hi = b;  // lower_bound(key) in run j
          while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (src[mid] < key) lo = mid + 1; else hi = mid;
          }
          rank += lo - a;
        }
      }
      d.out_ids[qo + rank] = key;
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

// non-monotone ids: every query list with >= 2 entries is sorted by id and
// checked for duplicates (decode.py:117-121)
__global__ void __launch_bounds__(256) k_sort_queries(const Dev d) {
  DevHdr* h = d.h;
  if (h->abort || !h->not_monotone) return;
  __shared__ int64_t sm[kSortSmem];
  const int64_t m = h->m;
  for (int64_t q = blockIdx.x; q < m; q += gridDim.x) {
    const int64_t qo = d.out_off[q], qe = d.out_off[q + 1];
    const int64_t len = qe - qo;
    if (len == 0) continue;
    // lists of multi-run or (for non-monotone ids) any query sit in `stage`
    int64_t* a = d.out_ids + qo;
    if (d.nsub[q] != 1 || h->not_monotone) {
      for (int64_t i = threadIdx.x; i < len; i += blockDim.x) a[i] = d.stage[qo + i];
      __syncthreads();
    }
    cta_sort<int64_t>(a, len, d.stage + qo, sm, (int64_t)0x7fffffffffffffffll);
    int dup = 0;
    for (int64_t i = threadIdx.x; i + 1 < len; i += blockDim.x) dup |= (a[i] == a[i + 1]);
    if (__syncthreads_or(dup) && threadIdx.x == 0) h->dup = 1;
  }
}

}  // namespace tj
