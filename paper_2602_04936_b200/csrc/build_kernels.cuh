// build_kernels.cuh — index construction on sm_100a.
//
// Replaces, from the reference (pkg/src/lcpsearch/):
//   core.lexicographic_order (core.py:162-174)  -> k_pack + stable LSD radix sort
//   core.adjacent_lcp        (core.py:177-184)  -> k_adjacent_lcp
//   trie.build level loop    (trie.py:409-419)  -> k_adj_hist + k_trie_* (lazy export)
//   TalEngine directory      (tal.py:76-82)     -> k_directory
// plus the k-ary search levels that stand in for the trie descent
// (trie.py:229-256): k_gather_level.
#pragma once

#include "common.cuh"

// ---------------------------------------------------------------------------
// pack: uint16 rows (n, L) -> packed keys (n, W); ids = 0..n-1
// ---------------------------------------------------------------------------
__global__ void k_pack(const uint16_t* __restrict__ rows, long long n, int L, int W, int b,
                       int spw, int sigma, u64* __restrict__ keys, u32* __restrict__ ids,
                       int* __restrict__ err) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long total = n * W;
  if (t >= total) return;
  long long row = t / W;
  int w = (int)(t - row * W);
  int j0 = w * spw;
  int j1 = min(L, j0 + spw);
  const uint16_t* r = rows + row * (long long)L;
  u64 acc = 0;
  bool bad = false;
  for (int j = j0; j < j1; ++j) {
    u32 s = r[j];
    bad |= (int)s >= sigma;
    acc |= (u64)s << (64 - b * (j - j0 + 1));
  }
  if (bad) raise_flag(err);
  keys[t] = acc;
  if (ids != nullptr && w == 0) ids[row] = (u32)row;
}

// ---------------------------------------------------------------------------
// pack, streaming form (L % 8 == 0, the rows 16-byte aligned): the (n, L)
// uint16 corpus is read as a flat stream of 16-byte chunks (8 symbols), one
// `ld.global.nc.v4` per lane, so a warp reads 512 contiguous bytes.  A chunk
// never straddles a key word (spw is a multiple of 8 for b <= 8; for b = 16 a
// chunk is exactly two words), so each lane packs its 8 symbols in place and
// the lanes of one word OR their parts with a segmented shuffle reduction;
// the first lane of the word stores it.  A warp "unit" is whole rows
// (cpr = L/8 <= 32 chunks per row: 32/cpr rows) or a 32-chunk piece of one
// row (cpr > 32), so no word is split across units.  4 units per lane are in
// flight.  Replaces the big-endian byte view of core.py:172-173.
// ---------------------------------------------------------------------------
constexpr int PK_THREADS = 256;
constexpr int PK_UNROLL = 4;

__global__ void __launch_bounds__(PK_THREADS) k_pack_stream(
    const uint16_t* __restrict__ rows, long long n, int L, int W, int b, int spw, int sigma,
    u64* __restrict__ keys, u32* __restrict__ ids, int* __restrict__ err) {
  const int lane = lane_id();
  const int cpr = L >> 3;                          // 16-byte chunks per row
  const int rpu = cpr <= 32 ? 32 / cpr : 1;        // rows per unit
  const int ppr = cpr <= 32 ? 1 : (cpr + 31) >> 5; // units per row
  const long long units = cpr <= 32 ? (n + rpu - 1) / rpu : n * ppr;
  const int gsize = b == 16 ? 1 : spw >> 3;        // chunks per key word
  const long long warp0 = ((long long)blockIdx.x * PK_THREADS + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * PK_THREADS) >> 5;
  bool bad = false;
  for (long long u0 = warp0; u0 < units; u0 += nwarps * PK_UNROLL) {
    uint4 v[PK_UNROLL];
    long long row[PK_UNROLL];
    int j[PK_UNROLL];
    bool ok[PK_UNROLL];
#pragma unroll
    for (int t = 0; t < PK_UNROLL; ++t) {
      const long long u = u0 + (long long)t * nwarps;
      if (cpr <= 32) {
        row[t] = u * rpu + lane / cpr;
        j[t] = lane % cpr;
        ok[t] = u < units && lane < rpu * cpr && row[t] < n;
      } else {
        row[t] = u / ppr;
        j[t] = (int)(u - row[t] * ppr) * 32 + lane;
        ok[t] = u < units && j[t] < cpr;
      }
      v[t] = ok[t] ? ld_stream16(rows + row[t] * L + j[t] * 8) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int t = 0; t < PK_UNROLL; ++t) {
      const u32 w32[4] = {v[t].x, v[t].y, v[t].z, v[t].w};
      u32 sym[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        sym[2 * i] = w32[i] & 0xffffu;  // little-endian: symbol 2i is the low half
        sym[2 * i + 1] = w32[i] >> 16;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) bad |= ok[t] && (int)sym[i] >= sigma;
      if (b == 16) {  // the chunk is words 2j and 2j+1 of the row
        u64 a = 0, c = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          a |= (u64)sym[i] << (48 - 16 * i);
          c |= (u64)sym[4 + i] << (48 - 16 * i);
        }
        if (ok[t]) {
          u64* dst = keys + row[t] * W + 2 * j[t];
          if (2 * j[t] + 1 < W) *reinterpret_cast<ulonglong2*>(dst) = make_ulonglong2(a, c);
          else dst[0] = a;
        }
      } else {
        const int w = (8 * j[t]) / spw;        // key word of this chunk
        const int p0 = (8 * j[t]) - w * spw;   // first symbol's slot in the word
        u64 part = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) part |= (u64)sym[i] << (64 - b * (p0 + i + 1));
        // segmented OR over the gsize lanes of one word (contiguous lanes;
        // a word's group never crosses a unit)
        const long long key = ok[t] ? row[t] * W + w : -1 - lane;
        for (int o = 1; o < gsize; o <<= 1) {
          const u64 po = __shfl_down_sync(LCP_FULL_MASK, part, o);
          const long long ko = __shfl_down_sync(LCP_FULL_MASK, key, o);
          if (lane + o < 32 && ko == key) part |= po;
        }
        const long long kprev = __shfl_up_sync(LCP_FULL_MASK, key, 1);
        if (ok[t] && (lane == 0 || kprev != key)) keys[key] = part;
      }
      if (ids != nullptr && ok[t] && j[t] == 0) ids[row[t]] = (u32)row[t];
    }
  }
  if (__any_sync(LCP_FULL_MASK, bad) && lane == 0) raise_flag(err);
}

// Aligned streaming pack, the common shapes (B = bits per symbol as a
// template constant; L a multiple of the 64/B symbols of a key word and
// L/8 dividing 32, e.g. L = 16, 32, 64 at sigma <= 256): a warp unit is 32/cpr
// whole rows, every lane owns a fixed (row-in-unit, chunk) slot, the 8-symbol
// chunk is packed with constant shifts into its 8*B-bit field, and the lanes of
// one word sit in an aligned group of 8/B lanes, so the word is OR-reduced
// with xor shuffles on its 32-bit halves.  ~50 lane instructions per 16-byte
// chunk instead of ~240 in the general form (ncu: k_pack_stream issue-bound
// at 70 % issue-slot use, 20 % of HBM).
template <int B>
__global__ void __launch_bounds__(PK_THREADS) k_pack_aligned(
    const uint16_t* __restrict__ rows, long long n, int L, int W, int sigma,
    u64* __restrict__ keys, u32* __restrict__ ids, int* __restrict__ err) {
  constexpr int GS = B >= 8 ? 1 : 8 / B;  // lanes per key word
  const int lane = lane_id();
  const int cpr = L >> 3;
  const int rpu = 32 / cpr;
  const int rr = lane / cpr, j = lane - rr * cpr;  // loop invariants
  const int g = j & (GS - 1);                       // chunk slot inside the word
  const int w = B == 16 ? 2 * j : j / GS;           // (first) key word of the chunk
  const int fshift = B >= 8 ? 0 : 64 - 8 * B * (g + 1);
  const long long units = (n + rpu - 1) / rpu;
  const long long warp0 = ((long long)blockIdx.x * PK_THREADS + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * PK_THREADS) >> 5;
  u32 vmax = 0;
  for (long long u0 = warp0; u0 < units; u0 += nwarps * PK_UNROLL) {
    uint4 v[PK_UNROLL];
#pragma unroll
    for (int t = 0; t < PK_UNROLL; ++t) {
      const long long row = (u0 + (long long)t * nwarps) * rpu + rr;
      v[t] = row < n ? ld_stream16(rows + row * L + j * 8) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int t = 0; t < PK_UNROLL; ++t) {
      const long long row = (u0 + (long long)t * nwarps) * rpu + rr;
      const bool ok = row < n;
      vmax = __vmaxu2(vmax, __vmaxu2(__vmaxu2(v[t].x, v[t].y), __vmaxu2(v[t].z, v[t].w)));
      // symbol 2i is the low half of word i (little-endian rows)
      const u32 sy[8] = {v[t].x & 0xffffu, v[t].x >> 16, v[t].y & 0xffffu, v[t].y >> 16,
                         v[t].z & 0xffffu, v[t].z >> 16, v[t].w & 0xffffu, v[t].w >> 16};
      if constexpr (B == 16) {
        const u64 a = ((u64)sy[0] << 48) | ((u64)sy[1] << 32) | ((u64)sy[2] << 16) | sy[3];
        const u64 c = ((u64)sy[4] << 48) | ((u64)sy[5] << 32) | ((u64)sy[6] << 16) | sy[7];
        if (ok) *reinterpret_cast<ulonglong2*>(keys + row * W + w) = make_ulonglong2(a, c);
      } else if constexpr (B == 8) {
        const u32 hi = (sy[0] << 24) | (sy[1] << 16) | (sy[2] << 8) | sy[3];
        const u32 lo = (sy[4] << 24) | (sy[5] << 16) | (sy[6] << 8) | sy[7];
        if (ok) keys[row * W + w] = ((u64)hi << 32) | lo;
      } else {
        u32 c = 0;  // the chunk's 8*B-bit field, most significant symbol first
#pragma unroll
        for (int i = 0; i < 8; ++i) c |= sy[i] << (8 * B - B * (i + 1));
        const u64 part = (u64)c << fshift;
        u32 hi = (u32)(part >> 32), lo = (u32)part;
#pragma unroll
        for (int o = 1; o < GS; o <<= 1) {
          hi |= __shfl_xor_sync(LCP_FULL_MASK, hi, o);
          lo |= __shfl_xor_sync(LCP_FULL_MASK, lo, o);
        }
        if (ok && g == 0) keys[row * W + w] = ((u64)hi << 32) | lo;
      }
      if (ids != nullptr && ok && j == 0) ids[row] = (u32)row;
    }
  }
  const u32 m = max(vmax & 0xffffu, vmax >> 16);
  if (__any_sync(LCP_FULL_MASK, (int)m >= sigma) && lane == 0) raise_flag(err);
}

// hi / lo 32-bit planes of each key's first word (full-scan layout)
__global__ void k_split_words(const u64* __restrict__ keys, long long n, int W,
                              u32* __restrict__ hi, u32* __restrict__ lo) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const u64 k = keys[i * W];
    hi[i] = (u32)(k >> 32);
    lo[i] = (u32)k;
  }
}

// first word of each W-word key (the W > 1 TAL sweep plane)
__global__ void k_first_word(const u64* __restrict__ keys, long long n, int W, u64* __restrict__ w0) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) w0[i] = keys[i * W];
}

__global__ void k_iota(u32* __restrict__ v, long long n) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (u32)i;
}

// kw[i] = keys[perm[i]*W + w]
__global__ void k_gather_word(const u64* __restrict__ keys, const u32* __restrict__ perm,
                              long long n, int W, int w, u64* __restrict__ kw) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) kw[i] = keys[(long long)perm[i] * W + w];
}

// out[i*W + w] = keys[perm[i]*W + w]
__global__ void k_gather_keys(const u64* __restrict__ keys, const u32* __restrict__ perm,
                              long long n, int W, u64* __restrict__ out) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * W) return;
  long long i = t / W;
  int w = (int)(t - i * W);
  out[t] = keys[(long long)perm[i] * W + w];
}

// ---------------------------------------------------------------------------
// Stable LSD radix sort of (u64 key, u32 value), 8-bit digits: the digit
// histograms of every pass (k_digit_hist8), per-tile digit counts (upsweep,
// digit-major [256][ntiles], for the count + scan + scatter form) and the
// scatter kernel k_onesweep below.
// Stability: a tile is split into 8 contiguous warp segments; a warp walks
// its segment 32 items at a time in index order, so rank = items of the
// same digit in earlier tiles + earlier warps + earlier steps + lower lanes.
// ---------------------------------------------------------------------------
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
#ifndef LCP_OS_ITEMS
#define LCP_OS_ITEMS 8  // keys per lane of a sort tile: 2048-key tiles keep 4 tiles
                        // resident per SM (16 per lane: 43 -> 31 us per pass at 2M
                        // vs 8: 23.5 us; A/B with -DLCP_OS_ITEMS=16)
#endif
constexpr int RS_ITEMS = LCP_OS_ITEMS;           // per lane (== the scatter's tile)
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;   // keys per tile
constexpr int RS_WARP_SEG = 32 * RS_ITEMS;       // 512 keys

// all eight digit histograms of one word in one pass (pass-skip detection)
__global__ void k_digit_hist8(const u64* __restrict__ k, long long n, u32* __restrict__ hist) {
  __shared__ u32 h[8 * 256];
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    u64 v = k[i];
#pragma unroll
    for (int p = 0; p < 8; ++p) atomicAdd(&h[p * 256 + (int)((v >> (8 * p)) & 255)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

__global__ void __launch_bounds__(RS_THREADS) k_rs_upsweep(const u64* __restrict__ keys, long long n,
                                                           int shift, int ntiles,
                                                           u32* __restrict__ counts) {
  __shared__ u32 h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  long long base = (long long)blockIdx.x * RS_TILE;
#pragma unroll 4
  for (int j = 0; j < RS_ITEMS; ++j) {
    long long i = base + j * RS_THREADS + threadIdx.x;
    if (i < n) atomicAdd(&h[(int)((keys[i] >> shift) & 255)], 1u);
  }
  __syncthreads();
  counts[(long long)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// ---------------------------------------------------------------------------
// Exclusive scan (in place), recursive over tiles.  T = u32 or u64.
// ---------------------------------------------------------------------------
constexpr int SC_THREADS = 512;
constexpr int SC_ITEMS = 8;
constexpr int SC_TILE = SC_THREADS * SC_ITEMS;

template <typename T>
__device__ T block_excl_scan(T v, T* total, T* sh /* >= 32 */) {
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(LCP_FULL_MASK, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int nw = blockDim.x >> 5;
    T s = lane < nw ? sh[lane] : (T)0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(LCP_FULL_MASK, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) sh[lane] = s;
  }
  __syncthreads();
  T wprefix = warp ? sh[warp - 1] : (T)0;
  *total = sh[(blockDim.x >> 5) - 1];
  __syncthreads();
  return wprefix + x - v;
}

template <typename T>
__global__ void __launch_bounds__(SC_THREADS) k_scan_tiles(T* __restrict__ data, long long m,
                                                           T* __restrict__ tile_sums) {
  __shared__ T sh[32];
  long long base = (long long)blockIdx.x * SC_TILE + (long long)threadIdx.x * SC_ITEMS;
  T v[SC_ITEMS];
  T s = 0;
#pragma unroll
  for (int j = 0; j < SC_ITEMS; ++j) {
    v[j] = (base + j < m) ? data[base + j] : (T)0;
    s += v[j];
  }
  T total;
  T ex = block_excl_scan<T>(s, &total, sh);
#pragma unroll
  for (int j = 0; j < SC_ITEMS; ++j) {
    if (base + j < m) data[base + j] = ex;
    ex += v[j];
  }
  if (threadIdx.x == 0 && tile_sums) tile_sums[blockIdx.x] = total;
}

template <typename T>
__global__ void k_scan_add(T* __restrict__ data, long long m, const T* __restrict__ tile_prefix) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) data[i] += tile_prefix[i / SC_TILE];
}

// ---------------------------------------------------------------------------
// Onesweep stable LSD radix pass (8-bit digit): ONE kernel per pass.
//   - every digit histogram comes from one upfront k_digit_hist8 read, so a
//     pass needs no upsweep: bucket starts = exclusive scan of its histogram;
//   - tiles take ids from an atomic counter in start order, count their
//     digits (warp match_any multisplit, index order => stable), publish
//     per-digit aggregates and resolve their exclusive prefix over earlier
//     tiles by decoupled look-back (status word = 2-bit flag | 62-bit count);
//   - the tile is reordered by digit in shared memory and written out in that
//     order, so each digit's run is a contiguous, coalesced store.
// Traffic per pass: read key + value, write key + value (24 B per pair at
// W=1 with u32 values).  Replaces the stable argsort of core.py:174.
// ---------------------------------------------------------------------------
constexpr int OS_THREADS = 256;
constexpr int OS_WARPS = OS_THREADS / 32;
constexpr int OS_ITEMS = LCP_OS_ITEMS;
constexpr int OS_TILE = OS_THREADS * OS_ITEMS;  // 2048 pairs (8 per lane)
constexpr int OS_MIN_CTAS = OS_ITEMS <= 8 ? 4 : 3;  // resident tiles per SM the registers allow
constexpr int OS_WARP_SEG = 32 * OS_ITEMS;
constexpr u64 OS_FLAG_AGG = 1ull << 62;
constexpr u64 OS_FLAG_PREFIX = 2ull << 62;
constexpr u64 OS_COUNT_MASK = (1ull << 62) - 1;
constexpr int OS_LB_WIN = 16;  // look-back statuses loaded per round trip (first hop: 8)
constexpr size_t OS_SMEM = (size_t)OS_TILE * 12 + (size_t)OS_WARPS * 256 * 4 + 3 * 256 * 4 + 64;

// lanes holding the same 8-bit digit as this lane (valid lanes only), from
// eight ballots: MATCH.ANY was the onesweep tile's slowest instruction
__device__ __forceinline__ unsigned match_digit8(u32 d, bool ok) {
  unsigned m = __ballot_sync(LCP_FULL_MASK, ok);
#pragma unroll
  for (int bit = 0; bit < 8; ++bit) {
    const unsigned b = __ballot_sync(LCP_FULL_MASK, (d >> bit) & 1u);
    m &= ((d >> bit) & 1u) ? b : ~b;
  }
  return ok ? m : 0u;
}

__device__ __forceinline__ u64 ld_relaxed_u64(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// LOOKBACK = false: the tile offsets come from a separate count + scan
// (k_rs_upsweep + scan_exclusive: offsets[d * ntiles + tile] already include
// the bucket start), tile = blockIdx.x, no status traffic; one more read of
// the keys (8 B per pair) instead of the look-back chain, whose first wave is
// serial (every co-resident tile waits for its predecessors' prefixes).
template <bool LOOKBACK>
__global__ void __launch_bounds__(OS_THREADS, OS_MIN_CTAS) k_onesweep(
    const u64* __restrict__ kin, const u32* __restrict__ vin, u64* __restrict__ kout,
    u32* __restrict__ vout, long long n, int shift, const u32* __restrict__ hist,
    u64* __restrict__ status, unsigned* __restrict__ tile_counter, const u32* __restrict__ offsets,
    int ntiles) {
  extern __shared__ __align__(16) unsigned char os_smem[];
  u64* sk = reinterpret_cast<u64*>(os_smem);                       // OS_TILE keys
  u32* sv = reinterpret_cast<u32*>(sk + OS_TILE);                  // OS_TILE values
  u32* wcnt = sv + OS_TILE;                                        // [OS_WARPS][256]
  u32* gstart = wcnt + OS_WARPS * 256;                             // bucket start + tile prefix
  u32* tstart = gstart + 256;                                      // digit start inside the tile
  u32* scratch = tstart + 256;                                     // 32 for block scans + tile id
  const int lane = lane_id();
  const int warp = threadIdx.x >> 5;
  const int d0 = threadIdx.x;  // the digit this thread owns in per-digit phases

  if (LOOKBACK && threadIdx.x == 0) scratch[32] = atomicAdd(tile_counter, 1u);
  for (int i = threadIdx.x; i < OS_WARPS * 256; i += OS_THREADS) wcnt[i] = 0;
  __syncthreads();
  const long long tile = LOOKBACK ? (long long)scratch[32] : (long long)blockIdx.x;
  // count + scan form: this digit's output base, loaded now so the scattered
  // read overlaps the key loads (ncu: it was the longest stall when read late)
  const u32 off_pref = LOOKBACK ? 0u : __ldg(offsets + (long long)d0 * ntiles + tile);
  const long long seg = tile * OS_TILE + (long long)warp * OS_WARP_SEG;

  u64 key[OS_ITEMS];
  u32 val[OS_ITEMS];
  u32 rank[OS_ITEMS];
#pragma unroll
  for (int j = 0; j < OS_ITEMS; ++j) {
    const long long i = seg + j * 32 + lane;
    const bool ok = i < n;
    key[j] = ok ? kin[i] : 0;
    val[j] = ok ? vin[i] : 0;
  }
  // stable in-warp ranks: rank = same-digit items of earlier rows of the
  // warp's segment + lower lanes of this row.  The 16 MATCH.ANY are
  // independent; each row's leader adds the row's count with one shared
  // atomic whose old value is that row's base (a warp's shared atomics to one
  // address apply in instruction order, so rows stay in index order)
#pragma unroll
  for (int j = 0; j < OS_ITEMS; ++j) {
    const bool ok = seg + j * 32 + lane < n;
    const u32 d = ok ? (u32)((key[j] >> shift) & 255) : 256u;
    const unsigned peers = match_digit8(d, ok);
    const unsigned lower = peers & ((1u << lane) - 1u);
    const int leader = __ffs(peers) - 1;
    u32 before = 0;
    if (ok && lower == 0) before = atomicAdd(&wcnt[warp * 256 + d], (u32)__popc(peers));
    before = __shfl_sync(LCP_FULL_MASK, before, leader);
    rank[j] = before + __popc(lower);
  }
  __syncthreads();
  // per digit: exclusive over warps, and the tile's count
  u32 cnt = 0;
#pragma unroll
  for (int w = 0; w < OS_WARPS; ++w) {
    const u32 c = wcnt[w * 256 + d0];
    wcnt[w * 256 + d0] = cnt;
    cnt += c;
  }
  // publish the aggregate (tile 0: its inclusive prefix) as early as possible
  u64* my = LOOKBACK ? status + tile * 256 + d0 : nullptr;
  if (LOOKBACK) st_relaxed_u64(my, (tile == 0 ? OS_FLAG_PREFIX : OS_FLAG_AGG) | (u64)cnt);
  // bucket start of this digit (exclusive scan of the pass histogram) and the
  // digit's start inside the tile
  u32 total;
  const u32 bstart = block_excl_scan<u32>(hist[d0], &total, scratch);
  const u32 tst = block_excl_scan<u32>(cnt, &total, scratch);
  tstart[d0] = tst;
  __syncthreads();
  // reorder the tile by (digit, stable rank) in shared memory: this needs only
  // tile-local counts, so it runs before the look-back and frees the registers
#pragma unroll
  for (int j = 0; j < OS_ITEMS; ++j) {
    const long long i = seg + j * 32 + lane;
    if (i < n) {
      const u32 d = (u32)((key[j] >> shift) & 255);
      const u32 pos = tstart[d] + wcnt[warp * 256 + d] + rank[j];
      sk[pos] = key[j];
      sv[pos] = val[j];
    }
  }
  // decoupled look-back over earlier tiles, OS_LB_WIN statuses per round trip
  // (independent loads): a tile with no resolved predecessor in reach would
  // otherwise walk back one dependent L2 round trip per tile, which is what
  // bounds the first wave (ncu: ~16 hops per tile at 2M, 47 us per pass)
  u64 excl = 0;
  long long p = LOOKBACK ? tile - 1 : -1;
  int win = 8;
  while (p >= 0) {
    u64 v[OS_LB_WIN];
#pragma unroll
    for (int i = 0; i < OS_LB_WIN; ++i)
      v[i] = (i < win && p - i >= 0) ? ld_relaxed_u64(status + (p - i) * 256 + d0) : OS_FLAG_PREFIX;
    int used = 0;
    bool resolved = false;
#pragma unroll
    for (int i = 0; i < OS_LB_WIN; ++i) {
      if (i < win && !resolved && used == i) {
        const u64 f = v[i] >> 62;
        if (f != 0) {
          excl += v[i] & OS_COUNT_MASK;
          resolved = f == 2;
          used = i + 1;
        }
      }
    }
    if (resolved) break;
    p -= used;  // used < win: tile p was not ready yet; poll it again
    win = OS_LB_WIN;
  }
  if (LOOKBACK) {
    if (tile > 0) st_relaxed_u64(my, OS_FLAG_PREFIX | (excl + cnt));
    gstart[d0] = bstart + (u32)excl;
  } else {
    gstart[d0] = off_pref;
  }
  __syncthreads();
  const long long rem = n - tile * OS_TILE;
  const int tile_n = rem < OS_TILE ? (int)rem : OS_TILE;
#pragma unroll 4
  for (int i = threadIdx.x; i < tile_n; i += OS_THREADS) {
    const u64 k = sk[i];
    const u32 d = (u32)((k >> shift) & 255);
    const long long g = (long long)gstart[d] + (i - (long long)tstart[d]);
    kout[g] = k;
    vout[g] = sv[i];
  }
}

// ---------------------------------------------------------------------------
// adjacent LCP of sorted keys: adj[i] = lcp(keys[i], keys[i+1])
// ---------------------------------------------------------------------------
template <int WMAX>
__global__ void k_adjacent_lcp(DevIndex ix, uint16_t* __restrict__ adj) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i + 1 >= ix.n) return;
  adj[i] = (uint16_t)key_lcp<WMAX>(ix.keys + i * ix.W, ix.keys + (i + 1) * ix.W, ix);
}

// search level: out[e*W + w] = keys[(e*stride)*W + w]
__global__ void k_gather_level(const u64* __restrict__ keys, long long cnt, long long stride,
                               int W, u64* __restrict__ out) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt * W) return;
  long long e = t / W;
  int w = (int)(t - e * W);
  out[t] = keys[e * stride * W + w];
}

// ---------------------------------------------------------------------------
// id sketch level: block b of the output holds the LCP_SK_LIST smallest of
// src[b*GROUP, (b+1)*GROUP) ascending.  Level 0 reads `order` (GROUP = 256
// sorted positions); level j+1 reads level j's lists (GROUP = 32 lists x 32).
// One warp per output block: sort the first 32 values across the lanes, then
// merge each further 32 into the running 32 smallest (warp_merge32) — no
// shared memory, no block barriers (the former CTA-wide bitonic sort of the
// whole group took 41 us per build at 2M rows).
// ---------------------------------------------------------------------------
constexpr int SK_THREADS = 256;
// Levels above 0 (GROUP = 1024 = 32 sorted lists): one CTA per output block,
// 8 warps each merging 4 lists, then a tree over the warps (a single warp per
// block serialised 31 merges: 33 us at 2M rows, against 19.5 us for the
// former bitonic sort and 14.8 us for the level-0 warp form).
template <int GROUP>
__global__ void __launch_bounds__(SK_THREADS) k_id_sketch_cta(const u32* __restrict__ src,
                                                              long long src_len,
                                                              u32* __restrict__ dst) {
  static_assert(GROUP % (32 * (SK_THREADS / 32)) == 0, "whole 32-entry chunks per warp");
  __shared__ u32 wl[SK_THREADS];  // one 32-entry list per warp
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const long long base = (long long)blockIdx.x * GROUP;
  constexpr int PER_WARP = GROUP / (SK_THREADS / 32);
  u32 slot = 0xffffffffu;
#pragma unroll 1
  for (int j = 0; j < PER_WARP; j += 32) {
    const long long i = base + warp * PER_WARP + j + lane;
    const u32 v = i < src_len ? __ldg(src + i) : 0xffffffffu;
    slot = j == 0 ? warp_sort32(v) : warp_merge32(slot, v);
  }
  wl[threadIdx.x] = slot;
  __syncthreads();
  for (int half = SK_THREADS / 64; half >= 1; half >>= 1) {
    if (warp < half) wl[threadIdx.x] = warp_merge32(wl[threadIdx.x], wl[(warp + half) * 32 + lane]);
    __syncthreads();
  }
  if (warp == 0) dst[(long long)blockIdx.x * LCP_SK_LIST + lane] = wl[lane];
}

template <int GROUP>
__global__ void __launch_bounds__(SK_THREADS) k_id_sketch(const u32* __restrict__ src,
                                                          long long src_len, long long nblocks,
                                                          u32* __restrict__ dst) {
  static_assert(GROUP % 32 == 0 && LCP_SK_LIST == 32, "one 32-entry list per warp");
  const int lane = lane_id();
  const long long b = ((long long)blockIdx.x * SK_THREADS + threadIdx.x) >> 5;
  if (b >= nblocks) return;
  const long long base = b * GROUP;
  u32 slot = 0xffffffffu;
#pragma unroll 1
  for (int j = 0; j < GROUP; j += 32) {
    const long long i = base + j + lane;
    const u32 v = i < src_len ? __ldg(src + i) : 0xffffffffu;
    slot = j == 0 ? warp_sort32(v) : warp_merge32(slot, v);
  }
  dst[b * LCP_SK_LIST + lane] = slot;
}

// ---------------------------------------------------------------------------
// TAL dense directory: dir[c] = #items whose d-prefix code < c
// (== np.searchsorted(codes, arange(sigma**d + 1)), tal.py:76-82).
// The d-prefix fits word 0 whenever sigma**d <= 2**24.
// ---------------------------------------------------------------------------
__global__ void k_directory(DevIndex ix, int d, long long buckets, long long* __restrict__ dir) {
  long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c > buckets) return;
  if (c == buckets) {
    dir[c] = ix.n;
    return;
  }
  // decode base-sigma code into d symbols, pack into a word-0 prefix
  u64 pre = 0;
  long long rem = c;
  for (int j = d - 1; j >= 0; --j) {
    u64 s = (u64)(rem % ix.sigma);
    rem /= ix.sigma;
    pre |= s << (64 - ix.b * (j + 1));
  }
  int keep = d * ix.b;
  u64 mask = keep >= 64 ? ~0ull : (~0ull << (64 - keep));
  long long lo = 0, hi = ix.n;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if ((ix.keys[mid * ix.W] & mask) < pre) lo = mid + 1;
    else hi = mid;
  }
  dir[c] = lo;
}

// ---------------------------------------------------------------------------
// Per-depth trie tables (TrieIndex.row_lo / edge_symbol / level_offset).
// Level d (1..L) starts a node at row 0 and at every row i with adj[i-1] < d.
// ---------------------------------------------------------------------------
__global__ void k_adj_hist(const uint16_t* __restrict__ adj, long long m,
                           unsigned long long* __restrict__ hist) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) atomicAdd(&hist[adj[i]], 1ull);
}

constexpr int TT_THREADS = 256;
// counts[(d-1)*nblk + blk] = #{i in block : adj[i-1] < d}, rows i in [1, n)
__global__ void __launch_bounds__(TT_THREADS) k_trie_count(const uint16_t* __restrict__ adj, long long n,
                                                           int nblk, unsigned long long* __restrict__ counts) {
  int d = blockIdx.y + 1;
  long long i = 1 + (long long)blockIdx.x * TT_THREADS + threadIdx.x;
  bool f = i < n && (int)adj[i - 1] < d;
  int c = __syncthreads_count(f);
  if (threadIdx.x == 0) counts[(long long)(d - 1) * nblk + blockIdx.x] = (unsigned long long)c;
}

__global__ void __launch_bounds__(TT_THREADS) k_trie_scatter(DevIndex ix, const uint16_t* __restrict__ adj,
                                                             int nblk, const unsigned long long* __restrict__ scan,
                                                             const long long* __restrict__ level_offset,
                                                             int* __restrict__ row_lo,
                                                             uint16_t* __restrict__ edge) {
  __shared__ int wsum[TT_THREADS / 32];
  int d = blockIdx.y + 1;
  long long n = ix.n;
  long long i = 1 + (long long)blockIdx.x * TT_THREADS + threadIdx.x;
  bool f = i < n && (int)adj[i - 1] < d;
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  unsigned m = __ballot_sync(LCP_FULL_MASK, f);
  if (lane == 0) wsum[warp] = __popc(m);
  __syncthreads();
  int before = 0;
  for (int w = 0; w < warp; ++w) before += wsum[w];
  before += __popc(m & ((1u << lane) - 1u));
  // flat scan covers levels 1..d-1 non-root starts; roots of levels 0..d
  // take d+1 slots ahead of this level's first non-root start.
  unsigned long long pos = scan[(long long)(d - 1) * nblk + blockIdx.x] + before + d + 1;
  if (f) {
    row_lo[pos] = (int)i;
    edge[pos] = (uint16_t)key_symbol(ix.keys + i * ix.W, d - 1, ix);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    long long r = level_offset[d];
    row_lo[r] = 0;
    edge[r] = (uint16_t)key_symbol(ix.keys, d - 1, ix);
  }
}

// ---------------------------------------------------------------------------
// LCPI index snapshot (storage.py:12-27, 155-210), generated on the GPU from
// the per-depth arena.  Record of node v at depth d, in node-id order:
//   u16 depth | u32 posting_len | (d == L: u32 ids[posting_len]) | u16 child_count |
//   (d < L: child_count x (u16 symbol, u32 child_id))
// Children of a depth-d node covering rows [lo, hi) are the depth-(d+1) nodes
// whose first row falls in [lo, hi); a leaf's posting is order[lo, hi).
// ---------------------------------------------------------------------------
__device__ __forceinline__ long long lower_i32(const int* a, long long m, long long v) {
  long long lo = 0, hi = m;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if ((long long)a[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int node_depth(const long long* off, int L, long long v) {
  int lo = 0, hi = L + 1;  // largest d with off[d] <= v
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= v) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ void put_u16(unsigned char* p, unsigned v) {
  p[0] = (unsigned char)v;
  p[1] = (unsigned char)(v >> 8);
}
__device__ __forceinline__ void put_u32(unsigned char* p, unsigned v) {
  p[0] = (unsigned char)v;
  p[1] = (unsigned char)(v >> 8);
  p[2] = (unsigned char)(v >> 16);
  p[3] = (unsigned char)(v >> 24);
}

// record sizes (bytes) of every node
__global__ void k_snap_sizes(const int* __restrict__ row_lo, const long long* __restrict__ off,
                             long long nodes, long long n, int L,
                             unsigned long long* __restrict__ size) {
  long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nodes) return;
  const int d = node_depth(off, L, v);
  const long long lo = row_lo[v];
  const long long hi = v + 1 < off[d + 1] ? row_lo[v + 1] : n;
  if (d == L) {
    size[v] = 8ull + 4ull * (unsigned long long)(hi - lo);
  } else {
    const int* nxt = row_lo + off[d + 1];
    const long long m = off[d + 2] - off[d + 1];
    const long long cc = lower_i32(nxt, m, hi) - lower_i32(nxt, m, lo);
    size[v] = 8ull + 6ull * (unsigned long long)cc;
  }
}

// node headers: depth, posting_len, child_count
__global__ void k_snap_headers(const int* __restrict__ row_lo, const long long* __restrict__ off,
                               const unsigned long long* __restrict__ start, long long nodes,
                               long long n, int L, unsigned char* __restrict__ out) {
  long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nodes) return;
  const int d = node_depth(off, L, v);
  const long long lo = row_lo[v];
  const long long hi = v + 1 < off[d + 1] ? row_lo[v + 1] : n;
  unsigned char* p = out + start[v];
  put_u16(p, (unsigned)d);
  if (d == L) {
    const unsigned plen = (unsigned)(hi - lo);
    put_u32(p + 2, plen);
    put_u16(p + 6 + 4ull * plen, 0u);
  } else {
    const int* nxt = row_lo + off[d + 1];
    const long long m = off[d + 2] - off[d + 1];
    const long long cc = lower_i32(nxt, m, hi) - lower_i32(nxt, m, lo);
    put_u32(p + 2, 0u);
    put_u16(p + 6, (unsigned)cc);
  }
}

// child entries: node c (depth >= 1) is entry rank of its parent's list
__global__ void k_snap_children(const int* __restrict__ row_lo, const uint16_t* __restrict__ edge,
                                const long long* __restrict__ off,
                                const unsigned long long* __restrict__ start, long long nodes,
                                int L, unsigned char* __restrict__ out) {
  long long c = 1 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nodes) return;
  const int d = node_depth(off, L, c);  // >= 1
  const long long row = row_lo[c];
  const int* par = row_lo + off[d - 1];
  const long long pm = off[d] - off[d - 1];
  // parent: last depth-(d-1) node starting at or before row
  long long lo = 0, hi = pm;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if ((long long)par[mid] <= row) lo = mid + 1;
    else hi = mid;
  }
  const long long p = off[d - 1] + lo - 1;
  const long long first = off[d] + lower_i32(row_lo + off[d], off[d + 1] - off[d], row_lo[p]);
  unsigned char* q = out + start[p] + 8 + 6ull * (unsigned long long)(c - first);
  put_u16(q, edge[c]);
  put_u32(q + 2, (unsigned)c);
}

// postings: row i lands in the leaf covering it, in row order
__global__ void k_snap_postings(const int* __restrict__ row_lo, const long long* __restrict__ off,
                                const unsigned long long* __restrict__ start,
                                const u32* __restrict__ order, long long n, int L,
                                unsigned char* __restrict__ out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int* leaf = row_lo + off[L];
  const long long m = off[L + 1] - off[L];
  long long lo = 0, hi = m;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if ((long long)leaf[mid] <= i) lo = mid + 1;
    else hi = mid;
  }
  const long long v = off[L] + lo - 1;
  put_u32(out + start[v] + 6 + 4ull * (unsigned long long)(i - leaf[lo - 1]), order[i]);
}

// rank[order[i]] = i: original id -> sorted position
__global__ void k_invert(const u32* __restrict__ order, long long n, u32* __restrict__ rank) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    rank[order[i]] = (u32)i;
}
