// Device-wide exclusive scan and stable radix sort with device-resident sizes.
//
// Every size in the tick after the index build (leaves, subqueries, words,
// results) is known only on the device.  These primitives read their length
// from a device pointer so the whole tick is a fixed launch sequence (CUDA
// graph capturable) with no host round trip between stages.
#pragma once

#include "tj_common.cuh"

namespace tj {

constexpr int kScanThreads = 256;

// ---------------------------------------------------------------------------
// Exclusive scan: three launches (chunk reduce, partial scan, chunk scan).
// `In`  : int64_t operator()(int64_t i) const        — value of item i
// `Out` : void operator()(int64_t i, int64_t excl, int64_t v) const
// ---------------------------------------------------------------------------
constexpr int kScanItems = 8;  // items per thread per step: 8 independent loads in flight (ILP)
constexpr int kScanTile = kScanThreads * kScanItems;
// 8-byte tile entries padded by one slot per 16: the blocked accesses (thread t,
// items 8t..8t+7, a 64-byte stride) and the striped ones both hit distinct
// bank pairs within each half-warp instead of 16-way conflicts
__device__ __forceinline__ int scan_pad(int i) { return i + (i >> 4); }
constexpr int kScanTilePadded = kScanTile + kScanTile / 16;

__device__ __forceinline__ void scan_chunk(int64_t n, int64_t G, int64_t blk, int64_t* b, int64_t* e) {
  const int64_t chunk = ((n + G - 1) / G + kScanTile - 1) / kScanTile * kScanTile;
  *b = blk * chunk;
  *e = (*b + chunk < n) ? *b + chunk : n;
}

template <typename In>
__global__ void __launch_bounds__(kScanThreads)
k_scan_reduce(In in, const int64_t* n_ptr, const DevHdr* h, int64_t* partial) {
  if (h->abort) return;
  __shared__ int64_t sh[33];
  int64_t b, e;
  scan_chunk(*n_ptr, gridDim.x, blockIdx.x, &b, &e);
  int64_t s = 0;
  for (int64_t base = b; base < e; base += kScanTile) {
    int64_t v[kScanItems];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      const int64_t i = base + k * kScanThreads + threadIdx.x;  // striped: coalesced
      v[k] = i < e ? in(i) : 0;
    }
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) s += v[k];
  }
  s = warp_sum(s);
  if (lane_id() == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    int64_t v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0;
    v = warp_sum(v);
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
  }
}

// single block of 1024 threads; G <= 1024
__global__ void __launch_bounds__(1024)
k_scan_partials(int64_t* partial, int G, int64_t* total_out, DevHdr* h) {
  if (h->abort) return;
  __shared__ int64_t sh[33];
  int64_t v = threadIdx.x < G ? partial[threadIdx.x] : 0;
  int64_t tot;
  int64_t ex = block_excl_scan(v, sh, &tot);
  if (threadIdx.x < G) partial[threadIdx.x] = ex;
  if (threadIdx.x == 0 && total_out) *total_out = tot;
}

// Items are loaded striped (coalesced; 8 independent loads per thread),
// transposed through shared memory to a blocked arrangement for the scan, and
// the exclusive prefixes transposed back so `Out` writes are coalesced too.
template <typename In, typename Out>
__global__ void __launch_bounds__(kScanThreads)
k_scan_down(In in, Out out, const int64_t* n_ptr, const DevHdr* h, const int64_t* partial) {
  if (h->abort) return;
  __shared__ int64_t sh[33];
  __shared__ int64_t tile[kScanTilePadded];
  int64_t b, e;
  scan_chunk(*n_ptr, gridDim.x, blockIdx.x, &b, &e);
  int64_t carry = partial[blockIdx.x];
  const int t = threadIdx.x;
  for (int64_t base = b; base < e; base += kScanTile) {  // uniform trip count per block
    int64_t v[kScanItems];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      const int64_t i = base + k * kScanThreads + t;
      v[k] = i < e ? in(i) : 0;
      tile[scan_pad(k * kScanThreads + t)] = v[k];
    }
    __syncthreads();
    int64_t blk[kScanItems];
    int64_t loc = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      blk[k] = tile[scan_pad(t * kScanItems + k)];
      loc += blk[k];
    }
    int64_t tot;
    int64_t ex = carry + block_excl_scan(loc, sh, &tot);  // (contains __syncthreads)
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      tile[scan_pad(t * kScanItems + k)] = ex;
      ex += blk[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      const int64_t i = base + k * kScanThreads + t;
      if (i < e) out(i, tile[scan_pad(k * kScanThreads + t)], v[k]);
    }
    carry += tot;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Single-pass exclusive scan with decoupled look-back: tiles are claimed in
// order from an atomic counter; a tile publishes its aggregate, walks back
// over its predecessors' published aggregates / inclusive prefixes to get its
// exclusive prefix, publishes its inclusive prefix, and writes its outputs.
// Reads the input once (the three-kernel scan reads it twice).  state[0] is
// the tile counter, state[1 + t] tile t's (flag << 62 | value); the state is
// cleared (one memset) before every scan.
// ---------------------------------------------------------------------------
constexpr unsigned long long kLbAgg = 1ull << 62, kLbInc = 2ull << 62, kLbVal = (1ull << 62) - 1;

template <typename In, typename Out>
__global__ void __launch_bounds__(kScanThreads)
k_scan_lb(In in, Out out, const int64_t* n_ptr, DevHdr* h, int64_t* total_out, unsigned long long* state) {
  if (h->abort) return;
  __shared__ int64_t sh[33];
  __shared__ int64_t tile[kScanTilePadded];
  __shared__ int64_t s_tile, s_excl;
  const int64_t n = *n_ptr;
  const int64_t ntiles = (n + kScanTile - 1) / kScanTile;
  if (ntiles == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && total_out) *total_out = 0;
    return;
  }
  const int t = threadIdx.x;
  unsigned long long* st = state + 1;
  for (;;) {
    if (t == 0) s_tile = (int64_t)atomicAdd(&state[0], 1ull);
    __syncthreads();
    const int64_t tl = s_tile;
    if (tl >= ntiles) break;
    const int64_t base = tl * kScanTile;
    int64_t v[kScanItems];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      const int64_t i = base + k * kScanThreads + t;
      v[k] = i < n ? in(i) : 0;
      tile[scan_pad(k * kScanThreads + t)] = v[k];
    }
    __syncthreads();
    int64_t blk[kScanItems];
    int64_t loc = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      blk[k] = tile[scan_pad(t * kScanItems + k)];
      loc += blk[k];
    }
    int64_t tot;
    int64_t ex = block_excl_scan(loc, sh, &tot);  // (contains __syncthreads)
    if (t == 0) {
      int64_t excl = 0;
      if (tl == 0) {
        atomicExch(&st[0], kLbInc | (unsigned long long)tot);
      } else {
        atomicExch(&st[tl], kLbAgg | (unsigned long long)tot);
        for (int64_t pp = tl - 1;;) {
          const unsigned long long sv = *(volatile unsigned long long*)&st[pp];
          if (sv == 0) continue;  // predecessor not published yet
          excl += (int64_t)(sv & kLbVal);
          if (sv & kLbInc) break;
          --pp;
        }
        atomicExch(&st[tl], kLbInc | (unsigned long long)(excl + tot));
      }
      s_excl = excl;
      if (tl == ntiles - 1 && total_out) *total_out = excl + tot;
    }
    __syncthreads();
    ex += s_excl;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      tile[scan_pad(t * kScanItems + k)] = ex;
      ex += blk[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      const int64_t i = base + k * kScanThreads + t;
      if (i < n) out(i, tile[scan_pad(k * kScanThreads + t)], v[k]);
    }
    __syncthreads();
  }
}

struct ScanPlan {
  int G;
  int64_t* partial;             // G entries (three-kernel scan)
  unsigned long long* state;    // look-back scan: counter + tile states
  int64_t state_words;
};

template <typename In, typename Out>
inline void scan_launch(const ScanPlan& p, In in, Out out, const int64_t* n_ptr, DevHdr* h,
                        int64_t* total_out, cudaStream_t st) {
  if (p.state) {
    cudaMemsetAsync(p.state, 0, (size_t)p.state_words * 8, st);
    k_scan_lb<In, Out><<<p.G, kScanThreads, 0, st>>>(in, out, n_ptr, h, total_out, p.state);
    return;
  }
  k_scan_reduce<In><<<p.G, kScanThreads, 0, st>>>(in, n_ptr, h, p.partial);
  k_scan_partials<<<1, 1024, 0, st>>>(p.partial, p.G, total_out, h);
  k_scan_down<In, Out><<<p.G, kScanThreads, 0, st>>>(in, out, n_ptr, h, p.partial);
}

// Generic functors ----------------------------------------------------------
template <typename T>
struct ArrIn {
  const T* a;
  __device__ int64_t operator()(int64_t i) const { return (int64_t)a[i]; }
};
template <typename T>
struct ExclOut {
  T* a;
  __device__ void operator()(int64_t i, int64_t ex, int64_t) const { a[i] = (T)ex; }
};

// ---------------------------------------------------------------------------
// Stable LSD radix sort of (u32 key, i32 value) pairs, kRadixBits-bit digits.
// Upsweep: per-chunk digit histograms; scan over (digit, chunk); downsweep:
// each CTA walks its chunk in input order, ranks items per digit with warp
// ballots (stable: warp w / round k / lane order), stages the tile by digit in
// shared memory and writes digit runs coalesced.
// ---------------------------------------------------------------------------
#ifndef TJ_RADIX_MINB
#define TJ_RADIX_MINB 2  // resident downsweep CTAs per SM the register budget is cut for (2: -9% vs 3; 1 and 4 slower)
#endif
#ifndef TJ_RADIX_BITS
#define TJ_RADIX_BITS 8
#endif
constexpr int kRadixBits = TJ_RADIX_BITS;           // 8: 2 passes cover 16-bit keys (leaf ranks)
constexpr int kRadixDigits = 1 << kRadixBits;       // 256 digits per pass
constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixDPT = kRadixDigits > kRadixThreads ? kRadixDigits / kRadixThreads : 1;  // digits per thread
constexpr int kRadixIPT = 16;                       // items per thread per tile
constexpr int kRadixTile = kRadixThreads * kRadixIPT;  // 4096

// key sources: a key array, or computed on the fly (first pass)
struct ArrKey {
  const uint32_t* k;
  __device__ uint32_t operator()(int64_t i) const { return k[i]; }
};

__device__ __forceinline__ int64_t radix_chunk(int64_t n, int64_t G) {
  return ((n + G - 1) / G + kRadixTile - 1) / kRadixTile * kRadixTile;
}

template <typename KeySrc>
__global__ void __launch_bounds__(kRadixThreads)
k_radix_upsweep(KeySrc keys, const int64_t* n_ptr, const DevHdr* h, int shift,
                uint32_t* hist /* [digits][G] */) {
  if (h->abort) return;
  __shared__ uint32_t cnt[kRadixWarps][kRadixDigits];
  const int64_t n = *n_ptr, G = gridDim.x;
  const int64_t chunk = radix_chunk(n, G);
  const int64_t b = blockIdx.x * chunk;
  const int64_t e = (b + chunk < n) ? b + chunk : n;
  const int w = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < kRadixWarps * kRadixDigits; k += kRadixThreads) (&cnt[0][0])[k] = 0;
  __syncthreads();
  for (int64_t i = b + threadIdx.x; i < e; i += kRadixThreads)
    atomicAdd(&cnt[w][(keys(i) >> shift) & (kRadixDigits - 1)], 1u);
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kRadixDPT; ++j) {
    const int dgt = threadIdx.x + j * kRadixThreads;
    if (dgt < kRadixDigits) {
      uint32_t s = 0;
#pragma unroll
      for (int ww = 0; ww < kRadixWarps; ++ww) s += cnt[ww][dgt];
      hist[(int64_t)dgt * G + blockIdx.x] = s;
    }
  }
}

// vals_in == nullptr: the value of item i is i (first pass over input rows);
// gate: vals_in is used only when the tick's objects enter in id order
// (DevHdr::key_sorted), else item i's value is i.
// keys_out == nullptr: the keys are not written (last pass).
// Payload (x, y) doubles (xin != nullptr): item i's payload is xin[i], yin[i]
// (the input arrays on the first pass, the previous pass's output after);
// it moves with the item through the same shared-memory staging, so every
// pass reads and writes it coalesced instead of a random gather afterwards.
struct RadixSmem {
  uint32_t wcnt[kRadixWarps][kRadixDigits];
  uint32_t base[kRadixDigits];     // running global offset per digit (this chunk)
  uint32_t tprefix[kRadixDigits];  // tile-local exclusive prefix per digit
  uint32_t skey[kRadixTile];
  int32_t sval[kRadixTile];
  int64_t shs[33];
};
struct RadixSmemXY {
  RadixSmem r;
  double sx[kRadixTile];
  double sy[kRadixTile];
};

template <typename KeySrc, bool XY>
__global__ void __launch_bounds__(kRadixThreads, TJ_RADIX_MINB)
k_radix_downsweep(KeySrc keys_in, const int32_t* vals_in, uint32_t* keys_out, int32_t* vals_out,
                  const double* __restrict__ xin, const double* __restrict__ yin, double* __restrict__ xout,
                  double* __restrict__ yout, const int64_t* n_ptr, const DevHdr* h, int shift,
                  const int64_t* offs /* [digits][G] exclusive */, int gate) {
  if (h->abort) return;
  if (gate && !h->key_sorted) vals_in = nullptr;
  extern __shared__ __align__(16) unsigned char radix_smem[];
  RadixSmem& S = *reinterpret_cast<RadixSmem*>(radix_smem);
  double* sx = XY ? reinterpret_cast<RadixSmemXY*>(radix_smem)->sx : nullptr;
  double* sy = XY ? reinterpret_cast<RadixSmemXY*>(radix_smem)->sy : nullptr;
  const int64_t n = *n_ptr, G = gridDim.x;
  const int64_t chunk = radix_chunk(n, G);
  const int64_t b = blockIdx.x * chunk;
  const int64_t e = (b + chunk < n) ? b + chunk : n;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
#pragma unroll
  for (int j = 0; j < kRadixDPT; ++j)
    if (t + j * kRadixThreads < kRadixDigits)
      S.base[t + j * kRadixThreads] = (uint32_t)offs[(int64_t)(t + j * kRadixThreads) * G + blockIdx.x];
  const uint32_t lt = (1u << lane) - 1u;
  // keys/values of the current tile are loaded one tile ahead (all IPT loads in flight)
  uint32_t key[kRadixIPT];
  int32_t val[kRadixIPT];
  auto load_tile = [&](int64_t tb) {
#pragma unroll
    for (int r = 0; r < kRadixIPT; ++r) {
      const int64_t i = tb + (int64_t)w * 32 * kRadixIPT + r * 32 + lane;
      const bool ok = i < e;
      key[r] = ok ? keys_in(i) : 0u;
      val[r] = ok ? (vals_in ? vals_in[i] : (int32_t)i) : 0;
    }
  };
  if (b < e) load_tile(b);
  for (int64_t tb = b; tb < e; tb += kRadixTile) {
    for (int k = t; k < kRadixWarps * kRadixDigits; k += kRadixThreads) (&S.wcnt[0][0])[k] = 0;
    __syncthreads();
    uint32_t dig[kRadixIPT], rk[kRadixIPT];
    // warp w owns items [tb + w*32*IPT, ...), processed in rounds of 32 in order
#pragma unroll
    for (int r = 0; r < kRadixIPT; ++r) {
      const int64_t i = tb + (int64_t)w * 32 * kRadixIPT + r * 32 + lane;
      const bool ok = i < e;
      // invalid lanes get digit kRadixDigits (the extra bit below)
      dig[r] = ok ? ((key[r] >> shift) & (kRadixDigits - 1)) : (uint32_t)kRadixDigits;
      // the lanes with this digit: 9 ballots (one match.any instead measured 4% slower per pass)
      uint32_t peers = 0xffffffffu;
#pragma unroll
      for (int bit = 0; bit <= kRadixBits; ++bit) {
        const bool on = (dig[r] >> bit) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, on);
        peers &= on ? bal : ~bal;
      }
      const int leader = __ffs(peers) - 1;
      uint32_t old = 0;
      if (ok && lane == leader) {
        old = S.wcnt[w][dig[r]];
        S.wcnt[w][dig[r]] = old + __popc(peers);
      }
      old = __shfl_sync(0xffffffffu, old, leader);
      rk[r] = old + __popc(peers & lt);
      __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive prefix across warps, tile total, tile-local digit offsets
    uint32_t run[kRadixDPT];
    int64_t carry = 0;
#pragma unroll
    for (int j = 0; j < kRadixDPT; ++j) {
      const int dgt = t + j * kRadixThreads;
      uint32_t acc = 0;
      if (dgt < kRadixDigits) {
#pragma unroll
        for (int ww = 0; ww < kRadixWarps; ++ww) {
          const uint32_t c = S.wcnt[ww][dgt];
          S.wcnt[ww][dgt] = acc;
          acc += c;
        }
      }
      run[j] = acc;
      int64_t tot;
      const int64_t ex = block_excl_scan((int64_t)acc, S.shs, &tot);
      if (dgt < kRadixDigits) S.tprefix[dgt] = (uint32_t)(ex + carry);
      carry += tot;
    }
    __syncthreads();
    uint32_t pos[kRadixIPT];
#pragma unroll
    for (int r = 0; r < kRadixIPT; ++r) {
      pos[r] = 0xffffffffu;
      if (dig[r] < (uint32_t)kRadixDigits) {
        pos[r] = S.tprefix[dig[r]] + S.wcnt[w][dig[r]] + rk[r];
        S.skey[pos[r]] = key[r];
        S.sval[pos[r]] = val[r];
      }
    }
    if constexpr (XY) {  // payload: coalesced loads straight into the staged order, 4 in flight per lane
#pragma unroll
      for (int r0 = 0; r0 < kRadixIPT; r0 += 4) {
        double xv[4], yv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t i = tb + (int64_t)w * 32 * kRadixIPT + (r0 + u) * 32 + lane;
          xv[u] = pos[r0 + u] != 0xffffffffu ? __ldcs(xin + i) : 0.0;
          yv[u] = pos[r0 + u] != 0xffffffffu ? __ldcs(yin + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (pos[r0 + u] != 0xffffffffu) {
            sx[pos[r0 + u]] = xv[u];
            sy[pos[r0 + u]] = yv[u];
          }
      }
    }
    if (tb + kRadixTile < e) load_tile(tb + kRadixTile);  // next tile in flight during the scatter
    __syncthreads();
    const int tile_n = (int)((e - tb) < kRadixTile ? (e - tb) : kRadixTile);
    for (int p = t; p < tile_n; p += kRadixThreads) {
      const uint32_t k = S.skey[p];
      const uint32_t d = (k >> shift) & (kRadixDigits - 1);
      const int64_t dst = (int64_t)S.base[d] + (p - S.tprefix[d]);
      if (keys_out) keys_out[dst] = k;
      vals_out[dst] = S.sval[p];
      if constexpr (XY) {
        xout[dst] = sx[p];
        yout[dst] = sy[p];
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kRadixDPT; ++j)
      if (t + j * kRadixThreads < kRadixDigits) S.base[t + j * kRadixThreads] += run[j];
    __syncthreads();
  }
}

template <bool XY>
constexpr size_t radix_smem_bytes() { return XY ? sizeof(RadixSmemXY) : sizeof(RadixSmem); }

}  // namespace tj
