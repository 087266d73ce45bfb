// common.cuh — shared types and device helpers for the sm_100a LCP kernels.
//
// Packed-key layout (replaces the big-endian void-key view of
// core.lexicographic_order, core.py:172-173):
//   b   = bits per symbol = next power of two >= ceil(log2 sigma)  (1,2,4,8,16)
//   spw = 64 / b symbols per u64 word (symbols never straddle words)
//   W   = ceil(L / spw) words per key, row-major keys[i*W + w]
//   symbol j lives in word j / spw at shift 64 - b*(j % spw + 1), MSB first,
//   unused low bits are zero.  Unsigned comparison of the word sequence is
//   exactly the lexicographic order of the uint16 symbol rows, and
//   lcp(a, b) = w*spw + clz(a[w]^b[w]) / b for the first differing word w.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

typedef unsigned long long u64;
typedef unsigned int u32;

#define LCP_FULL_MASK 0xffffffffu
#define LCP_MAX_LEVELS 12
#define LCP_SEARCH_FANOUT 64  // k-ary search: 32 lanes x 2 separators

struct DevIndex {
  const u64* keys;        // sorted packed keys, n*W
  const u32* order;       // sorted position -> original item id
  const u64* keys_orig;   // packed keys in original row order, n*W (full scan)
  const u64* levels;      // concatenated search-level tables (W words per entry)
  const long long* directory;  // TAL dense directory (sigma**d + 1) or null
  long long n;
  long long level_off[LCP_MAX_LEVELS];  // entry offset of level j in `levels`
  long long level_cnt[LCP_MAX_LEVELS];  // entries of level j
  int nlevels;       // levels above the leaf (the leaf is `keys` itself)
  int smem_levels;   // top levels staged into shared memory
  int smem_entries;  // entries in those staged levels
  int L, W, b, lb, spw, sigma;
  int tal_depth;           // -1 when no TAL structure
  long long tal_buckets;   // sigma**tal_depth
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// ---- key helpers ---------------------------------------------------------

// Position-j symbol shift inside its word.
__device__ __forceinline__ int sym_shift(int j, const DevIndex& ix) {
  return 64 - ix.b * ((j & (ix.spw - 1)) + 1);
}

__device__ __forceinline__ u32 key_symbol(const u64* key, int j, const DevIndex& ix) {
  u64 w = key[j >> (6 - ix.lb)];
  return (u32)((w >> sym_shift(j, ix)) & ((1ull << ix.b) - 1ull));
}

// lcp of two packed keys of W words.  WMAX > 0: compile-time upper bound on
// W (fully unrolled); WMAX == 0: any W.
template <int WMAX>
__device__ __forceinline__ int key_lcp(const u64* a, const u64* q, const DevIndex& ix) {
  if constexpr (WMAX == 1) {
    u64 x = a[0] ^ q[0];
    return x ? (__clzll((long long)x) >> ix.lb) : ix.L;
  } else if constexpr (WMAX > 1) {
#pragma unroll
    for (int w = 0; w < WMAX; ++w) {
      if (w < ix.W) {
        u64 x = a[w] ^ q[w];
        if (x) return w * ix.spw + (__clzll((long long)x) >> ix.lb);
      }
    }
    return ix.L;
  } else {
    for (int w = 0; w < ix.W; ++w) {
      u64 x = a[w] ^ q[w];
      if (x) return w * ix.spw + (__clzll((long long)x) >> ix.lb);
    }
    return ix.L;
  }
}

// lexicographic a < q over W words
template <int WMAX>
__device__ __forceinline__ bool key_less(const u64* a, const u64* q, const DevIndex& ix) {
  if constexpr (WMAX == 1) {
    return a[0] < q[0];
  } else if constexpr (WMAX > 1) {
#pragma unroll
    for (int w = 0; w < WMAX; ++w) {
      if (w < ix.W && a[w] != q[w]) return a[w] < q[w];
    }
    return false;
  } else {
    for (int w = 0; w < ix.W; ++w)
      if (a[w] != q[w]) return a[w] < q[w];
    return false;
  }
}

// Compare the first d symbols of key a against q: -1 a<q, 0 equal, 1 a>q.
__device__ __forceinline__ int prefix_cmp(const u64* a, const u64* q, int d, const DevIndex& ix) {
  int full = d >> (6 - ix.lb);        // whole words covered
  for (int w = 0; w < full; ++w) {
    if (a[w] != q[w]) return a[w] < q[w] ? -1 : 1;
  }
  int rem = d & (ix.spw - 1);
  if (rem) {
    int keep = rem * ix.b;                       // 1..63 bits
    u64 m = ~0ull << (64 - keep);
    u64 x = a[full] & m, y = q[full] & m;
    if (x != y) return x < y ? -1 : 1;
  }
  return 0;
}

// (L - lcp) << 32 | id : the k smallest of these are the top-k by
// (lcp desc, id asc) — trie.py:90-94 + tal.py:183 + oracle.py:58 in one key.
__device__ __forceinline__ u64 make_composite(int lcp, u32 id, int L) {
  return ((u64)(u32)(L - lcp) << 32) | (u64)id;
}

// ---- warp top-k (slot i on lane i holds the i-th smallest) ---------------

__device__ __forceinline__ void warp_insert(u64& slot, u64 c) {
  const int lane = lane_id();
  unsigned lt = __ballot_sync(LCP_FULL_MASK, slot < c);
  int p = __popc(lt);
  u64 up = __shfl_up_sync(LCP_FULL_MASK, slot, 1);
  if (lane > p) slot = up;
  else if (lane == p) slot = c;
}

// Offer one candidate per lane (UINT64_MAX = none); keeps the `need`
// smallest.  thr caches slot[need-1].
__device__ __forceinline__ void warp_offer(u64& slot, u64& thr, u64 comp, int need) {
  unsigned m = __ballot_sync(LCP_FULL_MASK, comp < thr);
  while (m) {
    int src = __ffs(m) - 1;
    m &= m - 1;
    u64 c = __shfl_sync(LCP_FULL_MASK, comp, src);
    if (c < thr) {
      warp_insert(slot, c);
      thr = __shfl_sync(LCP_FULL_MASK, slot, need - 1);
    }
  }
}

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(LCP_FULL_MASK, v, o);
  return v;
}

__device__ __forceinline__ u64 warp_or64(u64 v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v |= __shfl_xor_sync(LCP_FULL_MASK, v, o);
  return v;
}

// ---- TMA bulk copy + mbarrier (sm_90+/sm_100a) ---------------------------

__device__ __forceinline__ u32 smem_u32(const void* p) {
  return (u32)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// 1-D bulk copy global -> shared, completion signalled on the mbarrier.
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(u64* bar, u32 phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LCP_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LCP_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// streaming read-only load (keys are immutable after build)
__device__ __forceinline__ u64 ldg64(const u64* p) { return __ldg(p); }
