// Shared device-side definitions for the B200 QUAD tick pipeline.
//
// Exactness contract: every float operation that the
// reference performs with NumPy binary64 is performed here with an explicit
// round-to-nearest intrinsic (__dadd_rn/__dsub_rn/__dmul_rn/__ddiv_rn), in the
// same order, and the whole library is compiled with --fmad=false, so no
// multiply-add is ever contracted.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tj {

constexpr int kWarp = 32;
constexpr int kMaxLevel = 12;        // morton.py:20 L_MAX
constexpr int kDenseTop = 12;        // dense pyramid levels 0..l_max (l_max <= 12): the histogram is
                                     // taken at l_max (fine bins: little atomic contention in hotspots)
constexpr int kLevelShift = 24;      // zmap / leaf code: (level << 24) | payload
constexpr uint32_t kPayloadMask = (1u << kLevelShift) - 1u;
static_assert(kDenseTop >= kMaxLevel, "node_count reads every level from the dense pyramid");

// Per-tick device header: sizes that only the device knows, reduction
// targets, and the abort flag that makes every later kernel a no-op when a
// capacity was exceeded (the host then grows buffers and replays the tick).
struct DevHdr {
  // host-written each tick
  int64_t n, m;
  int32_t th, l_max, F, covering;
  int64_t cap_S, cap_W, cap_R, cap_U, cap_L;
  // MBR reduction (order-preserving keys) and derived scalars
  unsigned long long kmin_x, kmin_y, kmax_x, kmax_y;
  double xa, ya, xb, yb, width, height;
  double sx_max, sy_max, sx_deep, sy_deep;
  double lw[13], lh[13];    // leaf extent per level: width / 2^level, height / 2^level (quadtree.py:219-231)
  int32_t wpos, hpos;       // width > 0, height > 0
  int32_t l_deep;
  int32_t pad0;
  int32_t reuse_index;      // adaptive policy: this tick reuses the previous index
  int64_t Z, L;             // deepest cells, leaves
  int64_t S, S_i, S_c;      // subqueries: all / intersecting / covering
  int64_t n_tasks, W, U;    // join tasks, bitmap words (rows sector-padded), work units
  unsigned long long W_ref; // bitmap words without the row padding (the reference's count)
  int64_t R;                // results
  int64_t R_check;          // results counted in query order (must equal R)
  // statistics (engine.py:212-258)
  unsigned long long tests, cov_results, active_cells, occ_sum, occ_sumsq, sum_isq, sum_cov;
  unsigned long long task_obj, task_isq;  // P_a, S_a: objects / subqueries inside join tasks
  // flags
  int32_t abort;            // bit0 S, bit1 W/U, bit2 R, bit4 L
  int32_t not_monotone;     // object ids not strictly increasing in input order
  int32_t not_identity;     // some object id differs from its input row
  int32_t pad1;
  int32_t dup;              // DuplicateResult detected
  int32_t oob;              // OutOfBounds (adaptive reuse: object outside old MBR)
  int32_t count_mismatch;   // CountMismatch
  int32_t ids_wide;         // TJ_OUT_IDS32: some result id does not fit in int32
  int32_t grid_sf;          // uniform grid (method "ug"): cells per side; 0 = quadtree
  uint32_t side_deep;       // cells per side of the l_deep grid (2^l_deep, or grid_sf)
  int32_t n_big;            // queries queued for k_merge_big
  int32_t dbg;              // experiment switches (TJ_DEBUG env), 0 in production
  unsigned long long overfull2, overfull8;  // needs_rebuild counters
  int32_t shard_rank, shard_n;              // leaf-range sharding (n == 1: off)
  int64_t shard_total;                      // total leaf work weight
  int64_t n_sort;                           // objects the leaf sort orders: n, or (sharded) those in own leaves
  int32_t tiling_gap;                       // TJ_CHECK_TILING: the leaves do not tile the deepest grid
  int32_t pad2;
  // object ids that are not the input rows ("keyed" lists): every leaf block is put in id order on
  // the device and carries its ids as 32-bit offsets from id_min (Dev::loff), so the decode merges
  // runs and emits ids with leaf-local loads (no per-result random id lookups, no per-list sorts)
  unsigned long long id_kmin, id_kmax;      // order-preserving keys (id ^ 2^63) of the smallest / largest id
  int64_t id_min;
  int64_t pres_words;                       // presence bitmap words in use (0: no id counting sort)
  int64_t pres_total;                       // set bits: n when the ids are distinct
  int32_t key_req;                          // host: this tick's sequence carries the id-key kernels
  int32_t key_mode;                         // device: keyed lists (ids not the rows, range < 2^28, distinct)
  int32_t key_sorted;                       // keyed and not increasing: objects enter the leaf sort in id order
  int32_t dup_ids;                          // two objects share an id (keyed lists off: k_merge_big sorts)
};

// dense pyramid layout: level 0 (root) padded to 4 entries, level l >= 1 at
// 4 + (4^l - 4)/3 — every level starts on a 16-byte boundary (uint4 loads)
__host__ __device__ inline int64_t pyr_off(int l) {
  return l == 0 ? 0 : ((int64_t(1) << (2 * l)) - 4) / 3 + 4;
}

// order-preserving map double -> uint64 (for atomic min/max)
__device__ __forceinline__ unsigned long long dkey(double v) {
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dunkey(unsigned long long k) {
  unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// Morton spread / compact of 12..16-bit coordinates; x on even bits (morton.py:45-66)
__host__ __device__ __forceinline__ uint32_t spread2(uint32_t v) {
  v &= 0xFFFFu;
  v = (v | (v << 8)) & 0x00FF00FFu;
  v = (v | (v << 4)) & 0x0F0F0F0Fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}
__host__ __device__ __forceinline__ uint32_t compact2(uint32_t v) {
  v &= 0x55555555u;
  v = (v | (v >> 1)) & 0x33333333u;
  v = (v | (v >> 2)) & 0x0F0F0F0Fu;
  v = (v | (v >> 4)) & 0x00FF00FFu;
  v = (v | (v >> 8)) & 0x0000FFFFu;
  return v;
}
__host__ __device__ __forceinline__ uint32_t morton2(uint32_t i, uint32_t j) {
  return spread2(i) | (spread2(j) << 1);
}

// Cell coordinate of one value: int(min((v - lo) * scale, side - 1)), 0 when
// the extent is empty (morton.py:100-108).  No FMA: separate rn ops.
__device__ __forceinline__ uint32_t cell_of(double v, double lo, double scale, int pos, uint32_t side) {
  if (!pos) return 0u;
  double t = __dmul_rn(__dsub_rn(v, lo), scale);
  double lim = (double)(side - 1u);
  t = (t < lim) ? t : lim;  // np.minimum (no NaNs on this path)
  t = (t > 0.0) ? t : 0.0;  // a no-op for points inside the MBR; keeps the adaptive check's
                            // out-of-MBR points (discarded by the rebuild) inside the grid
  return (uint32_t)__double2int_rz(t);
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane_id() >= o) v += u;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive
// prefix, and the block total via *total.  `sh` needs blockDim/32 + 1 slots.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* sh, T* total) {
  const int lane = lane_id(), wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) sh[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T s = lane < nw ? sh[lane] : T(0);
    T si = warp_incl_scan(s);
    if (lane < nw) sh[lane] = si - s;
    if (lane == 31) sh[32] = si;
  }
  __syncthreads();
  T r = inc - v + sh[wid];
  *total = sh[32];
  __syncthreads();
  return r;
}

}  // namespace tj
