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
#define LCP_LEAF_KEYS 16      // the last search table resolves a 16-key leaf block
#define LCP_SK_BLOCK 256      // id sketch: level-0 block of sorted positions
#define LCP_SK_FANOUT 32      // id sketch: child blocks per block above level 0
#define LCP_SK_LIST 32        // id sketch: smallest ids kept per block (ascending)

struct DevIndex {
  const u64* keys;        // sorted packed keys, n*W
  const u32* order;       // sorted position -> original item id
  const u64* keys_orig;   // packed keys in original row order, n*W (full scan)
  const u32* keys_hi;     // W == 1: high 32 bits of keys_orig (SoA plane for the scan)
  const u32* keys_lo;     // W == 1: low 32 bits of keys_orig
  const u64* levels;      // concatenated search-level tables (W words per entry)
  const u64* keys_w0;     // W > 1: first word of each sorted key (coalesced compares, TAL sweep)
  const u64* levels_w0;   // first word of each search-table entry (== levels when W == 1)
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
  int idbits;              // id bits of the compact u32 composite (32: use u64)
  // id sketch: for every block of LCP_SK_BLOCK * LCP_SK_FANOUT**j sorted
  // positions, its LCP_SK_LIST smallest ids ascending (0xffffffff padded).
  // Serves "smallest ids in a long sorted range" when R(d*) is huge.
  const u32* sketch;
  const u32* rank;  // original id -> sorted position (inverse of order)
  long long sk_off[LCP_MAX_LEVELS];  // block offset of level j (lists of LCP_SK_LIST)
  long long sk_cnt[LCP_MAX_LEVELS];  // blocks at level j
  int sk_levels;
  // per launch, normally null: a device int capping `count` (a batch whose size
  // is only known on the device, e.g. the queries a range shard owns)
  const int* dcount;
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// raise an invalid-input flag: every writer stores 1, so a plain store is
// enough — and it is valid on mapped host memory (a result block the kernel
// writes directly), where device atomics are not guaranteed
__device__ __forceinline__ void raise_flag(int* f) { *reinterpret_cast<volatile int*>(f) = 1; }

// 16-byte streaming load of read-only data that is used once (no L1 allocation)
__device__ __forceinline__ uint4 ld_stream16(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

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

// Compact composite: (L - lcp) << idbits | id in 32 bits when
// n < 2**idbits and L < 2**(32 - idbits) (config 3: 6 + 26 bits); the
// order is the same as the u64 form, so it is used for selection only.
// n < 2**idbits (not <=) keeps the largest real composite, (lcp 0, id n-1)
// at L = 2**(32-idbits) - 1, strictly below the all-ones empty sentinel.
template <typename C>
__device__ __forceinline__ C make_comp(int lcp, u32 id, int L, int idbits) {
  return ((C)(u32)(L - lcp) << idbits) | (C)id;
}

template <typename C>
__device__ __forceinline__ u64 widen_comp(C c, int idbits) {
  if constexpr (sizeof(C) == 8) {
    return c;
  } else {
    if (c == ~C(0)) return ~0ull;
    return ((u64)(c >> idbits) << 32) | (u64)(c & ((1u << idbits) - 1u));
  }
}

// ---- warp top-k (slot i on lane i holds the i-th smallest) ---------------

template <typename C>
__device__ __forceinline__ C cmin(C a, C b) { return a < b ? a : b; }
template <typename C>
__device__ __forceinline__ C cmax(C a, C b) { return a < b ? b : a; }

template <typename C>
__device__ __forceinline__ void warp_insert(C& slot, C c) {
  const int lane = lane_id();
  unsigned lt = __ballot_sync(LCP_FULL_MASK, slot < c);
  int p = __popc(lt);
  C up = __shfl_up_sync(LCP_FULL_MASK, slot, 1);
  if (lane > p) slot = up;
  else if (lane == p) slot = c;
}

// Offer one candidate per lane (all-ones = none); keeps the `need`
// smallest.  thr caches slot[need-1].
template <typename C>
__device__ __forceinline__ C warp_sort32(C v);

// Batch merge for warp_offer: sort the batch, reverse it against the sorted
// list, keep the lane-wise minima (the 32 smallest of both, a bitonic
// sequence) and finish with a bitonic merge.  Out of line so the callers'
// hot loops keep their register budget (it runs on extension paths only).
template <typename C>
__device__ __noinline__ C warp_merge32(C slot, C batch) {
  const int lane = lane_id();
  C v = warp_sort32(batch);
  v = cmin(slot, __shfl_sync(LCP_FULL_MASK, v, 31 - lane));
#pragma unroll
  for (int j = 16; j > 0; j >>= 1) {
    const C p = __shfl_xor_sync(LCP_FULL_MASK, v, j);
    v = (lane & j) == 0 ? cmin(v, p) : cmax(v, p);
  }
  return v;
}

// BATCH: merge more than six candidates at once (warp_merge32).  Off in the
// 32-register query kernels and their out-of-line helpers: the extra call
// level made k_query_w1 spill and cost 1 % of headline throughput.
template <typename C, bool BATCH = false>
__device__ __forceinline__ void warp_offer(C& slot, C& thr, C comp, int need) {
  unsigned m = __ballot_sync(LCP_FULL_MASK, comp < thr);
  if (BATCH && __popc(m) > 6) {
    slot = warp_merge32(slot, comp < thr ? comp : ~C(0));
    thr = __shfl_sync(LCP_FULL_MASK, slot, need - 1);
    return;
  }
  while (m) {
    int src = __ffs(m) - 1;
    m &= m - 1;
    C c = __shfl_sync(LCP_FULL_MASK, comp, src);
    if (c < thr) {
      warp_insert(slot, c);
      thr = __shfl_sync(LCP_FULL_MASK, slot, need - 1);
    }
  }
}

// Bitonic sort of 32 values, one per lane: lane i ends with the i-th smallest.
template <typename C>
__device__ __forceinline__ C warp_sort32(C v) {
  const int lane = lane_id();
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      C p = __shfl_xor_sync(LCP_FULL_MASK, v, j);
      bool keep_min = ((lane & k) == 0) == ((lane & j) == 0);
      v = keep_min ? cmin(v, p) : cmax(v, p);
    }
  }
  return v;
}

// Bitonic sort of 64 values a[lane] = v0, a[lane + 32] = v1 (ascending).
template <typename C>
__device__ __forceinline__ void warp_sort64(C& v0, C& v1) {
  const int lane = lane_id();
#pragma unroll
  for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j == 32) {
        C lo = cmin(v0, v1), hi = cmax(v0, v1);
        v0 = lo;
        v1 = hi;
      } else {
        C p0 = __shfl_xor_sync(LCP_FULL_MASK, v0, j);
        C p1 = __shfl_xor_sync(LCP_FULL_MASK, v1, j);
        const bool lower = (lane & j) == 0;
        const bool up0 = (lane & k) == 0;
        const bool up1 = ((lane + 32) & k) == 0;
        v0 = (up0 == lower) ? cmin(v0, p0) : cmax(v0, p0);
        v1 = (up1 == lower) ? cmin(v1, p1) : cmax(v1, p1);
      }
    }
  }
}

template <typename C, int T>
__device__ __forceinline__ C pick_slot(const C (&v)[T], int t) {
  C r = ~C(0);
#pragma unroll
  for (int i = 0; i < T; ++i)
    if (i == t) r = v[i];
  return r;
}

// Candidates form one contiguous run [r0, r0 + c) of a warp-strided array
// (item index t*32 + lane lives in comp[t] of `lane`).  Returns the run
// sorted ascending in slot layout (lane i = i-th smallest) for c <= 64;
// beyond that it keeps the `need` smallest via serial warp insertion.
template <typename C, int T>
__device__ __forceinline__ C sort_run(const C (&comp)[T], int r0, int c, int need) {
  const int lane = lane_id();
  const int t0 = r0 >> 5;
  if (c <= 32) {
    const int e = r0 + lane;
    C a = __shfl_sync(LCP_FULL_MASK, pick_slot<C, T>(comp, t0), e & 31);
    C b = __shfl_sync(LCP_FULL_MASK, pick_slot<C, T>(comp, t0 + 1), e & 31);
    C v = lane < c ? (((e >> 5) == t0) ? a : b) : ~C(0);
    return warp_sort32(v);
  }
  if (c <= 64) {
    const int e0 = r0 + lane, e1 = r0 + 32 + lane;
    C a = __shfl_sync(LCP_FULL_MASK, pick_slot<C, T>(comp, t0), e0 & 31);
    C b = __shfl_sync(LCP_FULL_MASK, pick_slot<C, T>(comp, t0 + 1), e0 & 31);
    C cc = __shfl_sync(LCP_FULL_MASK, pick_slot<C, T>(comp, t0 + 2), e0 & 31);
    C v0 = ((e0 >> 5) == t0) ? a : b;
    C v1 = ((e1 >> 5) == t0 + 1) ? b : cc;
    if (32 + lane >= c) v1 = ~C(0);
    warp_sort64(v0, v1);
    return v0;
  }
  C slot = ~C(0), thr = ~C(0);
#pragma unroll
  for (int t = 0; t < T; ++t) warp_offer(slot, thr, comp[t], need);
  return slot;
}

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(LCP_FULL_MASK, v, o);
  return v;
}

__device__ __forceinline__ u64 warp_or64(u64 v) {  // two REDUX.OR instead of ten shuffles
  return ((u64)__reduce_or_sync(LCP_FULL_MASK, (u32)(v >> 32)) << 32) |
         (u64)__reduce_or_sync(LCP_FULL_MASK, (u32)v);
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

// ascending bitonic sort of buf[0, P) (P a power of two) by the whole CTA
// (blockDim a multiple of 32); callers synchronize before it, it ends
// synchronized.  Threads walk pair indices t (i = t with a zero inserted at
// bit j), so every lane does a compare-exchange at every stage.  A warp's pair
// indices [32w, 32w + 32) + r * blockDim touch only its own 64-element
// segments when j <= 32, so those stages need only a warp barrier; a CTA
// barrier precedes every stage with j >= 64 and follows each merge's last stage.
__device__ __forceinline__ void bitonic_sort_smem(u64* buf, int P) {
  const int half = P >> 1;
  for (int k2 = 2; k2 <= P; k2 <<= 1) {
    for (int j = k2 >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < half; t += blockDim.x) {
        const int i = 2 * t - (t & (j - 1));
        const u64 a = buf[i], b = buf[i + j];
        if ((a > b) == ((i & k2) == 0)) {
          buf[i] = b;
          buf[i + j] = a;
        }
      }
      if (j > 32 || j == 1) __syncthreads();
      else __syncwarp();
    }
  }
}
