// query_kernels.cuh — batched top-k LCP queries on sm_100a.
//
// Replaces (pkg/src/lcpsearch/):
//   TrieIndex._descend          trie.py:229-256  -> warp k-ary lower_bound over packed keys
//   TrieIndex.query strict/complete trie.py:290-342 -> window d* + bounded range scan + warp top-k
//   TalEngine.bucket_range/query tal.py:116-194   -> directory lookup + CTA bucket scan
//
// Complete mode without backtracking: with need = min(k, n),
// d* = max{d : |R(d)| >= need}; the answer is the `need` smallest
// (L-lcp)<<32|id over the contiguous sorted range R(d*).  Because lcp is
// non-decreasing before pos = lower_bound(q) and non-increasing after it,
// d* is the need-th largest lcp inside the window [pos-need, pos+need),
// and R(d*) is found by extending that window outward (long runs: run-edge
// search + id sketch).
// The reference's ancestor walk visits exactly d_max - d* ancestors, which
// is how the host rebuilds WorkReport.nodes_visited.
#pragma once

#include "common.cuh"

constexpr int QW_MAX_THREADS = 1024;            // one CTA per SM, one query per warp

#ifdef LCP_TRACE
// Debug-only per-query stage timestamps (SM clock), compiled into the trace
// build of tools/trace_query.py, never into the shipped library.
__device__ unsigned long long lcp_trace_buf[65536 * 8];
#define LCP_STAMP(qi, slot)                                                      \
  do {                                                                          \
    if (lane_id() == 0 && (qi) < 65536) lcp_trace_buf[(qi) * 8 + (slot)] = clock64(); \
  } while (0)
#else
#define LCP_STAMP(qi, slot) \
  do {                      \
  } while (0)
#endif
constexpr int FAST_KMAX = 32;                   // warp top-k capacity

// pack one query row into W words held by every lane; returns false if a
// symbol is >= sigma (reference: trie.py:223-226 / tal.py:104-107)
template <int WMAX>
__device__ __forceinline__ bool warp_pack_query(const uint16_t* __restrict__ qrow,
                                                const DevIndex& ix, u64 (&qk)[WMAX]) {
  const int lane = lane_id();
  if (ix.L <= 32) {  // warp-uniform: one symbol per lane, selected into its word
    const bool has = lane < ix.L;
    const u32 s = has ? qrow[lane] : 0u;
    const u64 v = has ? (u64)s << sym_shift(lane, ix) : 0ull;
    const int wj = lane >> (6 - ix.lb);
#pragma unroll
    for (int w = 0; w < WMAX; ++w) qk[w] = warp_or64(w == wj ? v : 0ull);
    return !__any_sync(LCP_FULL_MASK, has && (int)s >= ix.sigma);
  }
#pragma unroll
  for (int w = 0; w < WMAX; ++w) qk[w] = 0;
  bool bad = false;
  for (int j = lane; j < ix.L; j += 32) {
    u32 s = qrow[j];
    bad |= (int)s >= ix.sigma;
    int wj = j >> (6 - ix.lb);
    u64 v = (u64)s << sym_shift(j, ix);
#pragma unroll
    for (int w = 0; w < WMAX; ++w)
      if (w == wj) qk[w] |= v;
  }
#pragma unroll
  for (int w = 0; w < WMAX; ++w) qk[w] = warp_or64(qk[w]);
  return !__any_sync(LCP_FULL_MASK, bad);
}

// W == 1: every lane packs its symbols, two REDUX.OR combine the halves.
__device__ __forceinline__ bool warp_pack_w1(const uint16_t* __restrict__ qrow, const DevIndex& ix,
                                             u64& q) {
  u64 v = 0;
  bool bad = false;
  for (int j = lane_id(); j < ix.L; j += 32) {
    u32 s = qrow[j];
    bad |= (int)s >= ix.sigma;
    v |= (u64)s << sym_shift(j, ix);
  }
  const u32 lo = __reduce_or_sync(LCP_FULL_MASK, (u32)v);
  const u32 hi = __reduce_or_sync(LCP_FULL_MASK, (u32)(v >> 32));
  q = ((u64)hi << 32) | lo;
  return !__any_sync(LCP_FULL_MASK, bad);
}

// key i (sorted) < q for W > 1: first word from its plane, the rest on a tie
template <int WMAX>
__device__ __forceinline__ bool w0_less(u64 a0, const u64* key, const u64 (&qk)[WMAX],
                                        const DevIndex& ix) {
  if (a0 != qk[0]) return a0 < qk[0];
#pragma unroll
  for (int w = 1; w < WMAX; ++w) {
    if (w < ix.W && key[w] != qk[w]) return key[w] < qk[w];
  }
  return false;
}

// lower_bound(keys, q) by a 64-ary search: every level is one coalesced
// 64-separator read per warp (2 per lane) + 2 ballots.  Top levels come
// from shared memory (staged by TMA bulk copy), the rest from L2/HBM.
template <int WMAX>
__device__ __forceinline__ long long warp_lower_bound(const DevIndex& ix, const u64* staged,
                                                      const u64 (&qk)[WMAX]) {
  // 32-bit positions (n < 2**31 by contract): the 64-bit index arithmetic
  // was a large share of the W > 1 kernels' instructions
  const int lane = lane_id();
  const int W = ix.W;
  const int n = (int)ix.n;
  int blk = 0;
  for (int j = 0;; ++j) {
    const int off = (int)ix.level_off[j];
    const int cnt = (int)ix.level_cnt[j];
    const u64* tab = (j < ix.smem_levels && WMAX == 1) ? staged + off : ix.levels + (size_t)off * W;
    if (j == ix.nlevels) {  // leaf block: 16 keys, one per lane
      const int base = blk * LCP_LEAF_KEYS;
      const int i = base + lane;
      bool lt = false;
      if (lane < LCP_LEAF_KEYS && i < n) {
        if constexpr (WMAX == 1) lt = key_less<WMAX>(ix.keys + (size_t)i * W, qk, ix);
        else lt = w0_less<WMAX>(__ldg(ix.keys_w0 + i), ix.keys + (size_t)i * W, qk, ix);
      }
      return base + (int)__reduce_add_sync(LCP_FULL_MASK, (u32)lt);
    }
    const int base = blk * LCP_SEARCH_FANOUT;
    const int i0 = base + 2 * lane;
    bool lt0 = false, lt1 = false;
    if constexpr (WMAX == 1) {
      if (i0 + 1 < cnt) {
        ulonglong2 v = *reinterpret_cast<const ulonglong2*>(tab + i0);
        lt0 = v.x < qk[0];
        lt1 = v.y < qk[0];
      } else if (i0 < cnt) {
        lt0 = tab[i0] < qk[0];
      }
    } else {  // first words (staged, or the global plane) in one 16-byte load;
              // the whole entry from the global table only on a tie
      const bool sm = j < ix.smem_levels;
      const u64* w0 = (sm ? staged : ix.levels_w0) + off;
      if (i0 + 1 < cnt) {  // plain loads from shared memory, __ldg from global
        const ulonglong2 v = sm ? *reinterpret_cast<const ulonglong2*>(w0 + i0)
                                : __ldg(reinterpret_cast<const ulonglong2*>(w0 + i0));
        lt0 = w0_less<WMAX>(v.x, tab + (size_t)i0 * W, qk, ix);
        lt1 = w0_less<WMAX>(v.y, tab + (size_t)(i0 + 1) * W, qk, ix);
      } else if (i0 < cnt) {
        lt0 = w0_less<WMAX>(sm ? w0[i0] : __ldg(w0 + i0), tab + (size_t)i0 * W, qk, ix);
      }
    }
    const int c = (int)__reduce_add_sync(LCP_FULL_MASK, (u32)lt0 + (u32)lt1);
    if (c == 0) return 0;  // only reachable at the root level
    blk = base + c - 1;
  }
}

template <int WMAX>
__device__ __forceinline__ int lcp_at(const DevIndex& ix, long long i, const u64 (&qk)[WMAX]) {
  if constexpr (WMAX == 1) {
    u64 x = ix.keys[i] ^ qk[0];
    return x ? (__clzll((long long)x) >> ix.lb) : ix.L;
  } else {
    // the first word from its plane (coalesced across lanes); the rest of
    // the key only when it equals q's
    const u64 x = __ldg(ix.keys_w0 + i) ^ qk[0];
    if (x) return __clzll((long long)x) >> ix.lb;
    const u64* key = ix.keys + i * ix.W;
#pragma unroll
    for (int w = 1; w < WMAX; ++w) {
      if (w < ix.W) {
        const u64 y = key[w] ^ qk[w];
        if (y) return w * ix.spw + (__clzll((long long)y) >> ix.lb);
      }
    }
    return ix.L;
  }
}



// Leaf-region loads for the W > 1 kernels: every lane issues its T first-word
// and T id loads (clamped index) before using any of them, so the region is
// one round trip; a conditional load (`ok ? lcp_at(...) : -1`) was compiled
// into one branch per row, serialising T round trips.  The remaining words
// are read only for rows equal to q in the first word.  lcp -1 outside [0, n).
template <int WMAX>
__device__ __forceinline__ int lcp_rest(const DevIndex& ix, long long i, const u64 (&qk)[WMAX]) {
  const u64* key = ix.keys + i * ix.W;
#pragma unroll
  for (int w = 1; w < WMAX; ++w) {
    if (w < ix.W) {
      const u64 y = key[w] ^ qk[w];
      if (y) return w * ix.spw + (__clzll((long long)y) >> ix.lb);
    }
  }
  return ix.L;
}

template <int WMAX, int T>
__device__ __forceinline__ int region_lcps(const DevIndex& ix, long long s, const u64 (&qk)[WMAX],
                                           int (&l)[T], u32 (&id)[T]) {
  const long long n = ix.n;
  const u64* w0 = WMAX == 1 ? ix.keys : ix.keys_w0;
  u64 x0[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const long long ic = min(max(s + t * 32 + lane_id(), 0ll), n - 1);
    x0[t] = __ldg(w0 + ic) ^ qk[0];
    id[t] = __ldg(ix.order + ic);
  }
  int dmax = -1;
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const long long i = s + t * 32 + lane_id();
    int lv;
    if (x0[t]) lv = __clzll((long long)x0[t]) >> ix.lb;
    else lv = WMAX == 1 ? ix.L : lcp_rest<WMAX>(ix, min(max(i, 0ll), n - 1), qk);
    l[t] = lv | ((i >= 0 && i < n) ? 0 : -1);
    dmax = max(dmax, l[t]);
  }
  return dmax;
}

// lcp of sorted row i (0 <= i < n) against q, with the row's id loaded in the
// same round trip (the id is needed only when the row qualifies, but loading
// it after the lcp would cost a second dependent round trip)
template <int WMAX>
__device__ __forceinline__ int lcp_id_at(const DevIndex& ix, long long i, const u64 (&qk)[WMAX], u32& id) {
  const u64 x = __ldg((WMAX == 1 ? ix.keys : ix.keys_w0) + i) ^ qk[0];
  id = __ldg(ix.order + i);
  if (x) return __clzll((long long)x) >> ix.lb;
  return WMAX == 1 ? ix.L : lcp_rest<WMAX>(ix, i, qk);
}

// Stage the top search levels into shared memory with one TMA bulk copy.
// stage_issue starts the copy; stage_wait blocks on its mbarrier (phase 0),
// so warps can load and pack their first query while the copy is in flight.
__device__ __forceinline__ void stage_issue(const DevIndex& ix, u64* bar, u64* staged) {
  if (ix.smem_levels <= 0) return;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // the first-word plane (== levels when W == 1): 8 B per entry
    u32 bytes = (u32)ix.smem_entries * 8u;
    mbar_arrive_expect_tx(bar, bytes);
    bulk_g2s(staged, ix.levels_w0, bytes, bar);
  }
}

__device__ __forceinline__ void stage_wait(const DevIndex& ix, u64* bar) {
  if (ix.smem_levels > 0) mbar_wait(bar, 0);
}

__device__ __forceinline__ void stage_levels(const DevIndex& ix, u64* bar, u64* staged) {
  stage_issue(ix, bar, staged);
  stage_wait(ix, bar);
}

// ---------------------------------------------------------------------------
// Long runs.  Outside the loaded region every item of R(d*) has lcp exactly
// d* (R(d*+1) has < need items and surrounds pos, so it lies inside the
// region), so the tail of the answer is "the smallest ids in a sorted-position
// range".  run_edge finds where the run ends; tier_offer reads the smallest
// ids of that range from the id sketch instead of scanning it.
// ---------------------------------------------------------------------------
constexpr int EXT_SCAN_CHUNKS = 4;  // 32-key chunks scanned per side before the sketch path

// Last position of the run {lcp >= d} walking from `in` (inside the run)
// toward `out` (outside it, or the sentinel -1 / n): 32-ary warp search,
// ceil(log32 |in - out|) rounds of one scattered probe per lane.
template <int WMAX>
__device__ __forceinline__ long long run_edge(const DevIndex& ix, const u64 (&qk)[WMAX], int d,
                                              long long in, long long out) {
  const long long dir = out > in ? 1 : -1;
  for (;;) {
    const long long span = (out - in) * dir;
    if (span <= 1) return in;
    const long long step = (span + 31) >> 5;
    const long long off = step * (lane_id() + 1);
    const bool inside = off < span && lcp_at<WMAX>(ix, in + dir * off, qk) >= d;
    const long long c = __popc(__ballot_sync(LCP_FULL_MASK, inside));
    if (step * (c + 1) < span) out = in + dir * step * (c + 1);
    in += dir * step * c;
  }
}

// offer tier|order[i] for i in [x, y)
template <typename C>
__device__ __forceinline__ void offer_positions(const DevIndex& ix, long long x, long long y,
                                                C tier, C& slot, C& thr, int need) {
  for (long long base = x; base < y; base += 32) {
    const long long i = base + lane_id();
    warp_offer(slot, thr, i < y ? (tier | (C)__ldg(ix.order + i)) : ~C(0), need);
  }
}

// offer the id lists of sketch blocks [x, y) of one level; a block whose
// smallest id cannot enter the top-need is skipped after one load
template <typename C>
__device__ __forceinline__ void offer_lists(const u32* __restrict__ lists, long long x, long long y,
                                            C tier, C& slot, C& thr, int need) {
  for (long long base = x; base < y; base += 32) {
    const long long blk = base + lane_id();
    const u32 mn = blk < y ? __ldg(lists + blk * LCP_SK_LIST) : 0xffffffffu;
    const C cm = mn == 0xffffffffu ? ~C(0) : (tier | (C)mn);
    unsigned m = __ballot_sync(LCP_FULL_MASK, cm < thr);
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      if (__shfl_sync(LCP_FULL_MASK, cm, src) < thr) {
        const u32 v = __ldg(lists + (base + src) * LCP_SK_LIST + lane_id());
        warp_offer(slot, thr, v == 0xffffffffu ? ~C(0) : (tier | (C)v), need);
      }
    }
  }
}

// the `need` smallest of tier|id over sorted positions [a, b): the partial
// level-0 blocks at either end position by position, then at each sketch
// level the blocks not covered by a whole block of the level above
template <typename C>
__device__ __noinline__ C tier_offer(const DevIndex& ix, long long a, long long b, C tier,
                                     C slot, int need) {
  // out of line: keeps the cold path's registers off the hot loop's budget
  C thr = __shfl_sync(LCP_FULL_MASK, slot, need - 1);
  long long A = (a + LCP_SK_BLOCK - 1) / LCP_SK_BLOCK, B = b / LCP_SK_BLOCK;
  if (A >= B) {
    offer_positions<C>(ix, a, b, tier, slot, thr, need);
    return slot;
  }
  offer_positions<C>(ix, a, A * LCP_SK_BLOCK, tier, slot, thr, need);
  offer_positions<C>(ix, B * LCP_SK_BLOCK, b, tier, slot, thr, need);
  for (int j = 0;; ++j) {
    const u32* lists = ix.sketch + ix.sk_off[j] * LCP_SK_LIST;
    const long long A2 = (A + LCP_SK_FANOUT - 1) / LCP_SK_FANOUT, B2 = B / LCP_SK_FANOUT;
    if (j + 1 >= ix.sk_levels || A2 >= B2) {
      offer_lists<C>(lists, A, B, tier, slot, thr, need);
      return slot;
    }
    offer_lists<C>(lists, A, A2 * LCP_SK_FANOUT, tier, slot, thr, need);
    offer_lists<C>(lists, B2 * LCP_SK_FANOUT, B, tier, slot, thr, need);
    A = A2;
    B = B2;
  }
}

// ---------------------------------------------------------------------------
// Shared tail of the warp query kernels: R(d*) may continue past the loaded
// region on either side.  Scan outward 32 keys at a time; a run still going
// after EXT_SCAN_CHUNKS chunks is finished by run_edge + tier_offer.
// ---------------------------------------------------------------------------
template <typename C, int WMAX>
__device__ __forceinline__ void extend_range(const DevIndex& ix, const u64 (&qk)[WMAX], int dstar,
                                             int need, bool left, long long lo_edge, bool right,
                                             long long hi_edge, int idbits, C& slot,
                                             long long& rsize, long long& rlo) {
  const int lane = lane_id();
  const long long n = ix.n;
  const int L = ix.L;
  if (!(left || right)) return;
  C thr = __shfl_sync(LCP_FULL_MASK, slot, need - 1);
  const C tier = make_comp<C>(dstar, 0u, L, idbits);
  long long e = lo_edge;  // [e, ...) is known to lie in R(d*)
  bool go = left;
  for (int chunk = 0; go; ++chunk) {
    if (chunk == EXT_SCAN_CHUNKS) {
      const long long r = dstar ? run_edge<WMAX>(ix, qk, dstar, e, -1) : 0;
      slot = tier_offer<C>(ix, r, e, tier, slot, need);
      thr = __shfl_sync(LCP_FULL_MASK, slot, need - 1);
      rsize += e - r;
      rlo = r;
      break;
    }
    long long i = e - 32 + lane;
    u32 oid;
    const int l = lcp_id_at<WMAX>(ix, max(i, 0ll), qk, oid) | (i >= 0 ? 0 : -1);
    bool c = l >= dstar;
    warp_offer(slot, thr, c ? make_comp<C>(l, oid, L, idbits) : ~C(0), need);
    unsigned m = __ballot_sync(LCP_FULL_MASK, c);
    rsize += __popc(m);
    if (m) rlo = e - 32 + (__ffs(m) - 1);
    e -= 32;
    go = m == LCP_FULL_MASK && e > 0;
  }
  e = hi_edge;  // [..., e) is known to lie in R(d*)
  go = right;
  for (int chunk = 0; go; ++chunk) {
    if (chunk == EXT_SCAN_CHUNKS) {
      const long long r = dstar ? run_edge<WMAX>(ix, qk, dstar, e - 1, n) + 1 : n;
      slot = tier_offer<C>(ix, e, r, tier, slot, need);
      rsize += r - e;
      break;
    }
    long long i = e + lane;
    u32 oid;
    const int l = lcp_id_at<WMAX>(ix, min(i, n - 1), qk, oid) | (i < n ? 0 : -1);
    bool c = l >= dstar;
    warp_offer(slot, thr, c ? make_comp<C>(l, oid, L, idbits) : ~C(0), need);
    unsigned m = __ballot_sync(LCP_FULL_MASK, c);
    rsize += __popc(m);
    e += 32;
    go = m == LCP_FULL_MASK && e < n;
  }
}

template <typename C>
__device__ __forceinline__ void write_result(long long qi, int stride, int take, int L, C slot,
                                             int idbits, int dmax, int dstar, long long rsize,
                                             long long rlo, u32* out_ids, uint16_t* out_lcps,
                                             int* out_hits, uint16_t* out_md, u64* out_aux) {
  const int lane = lane_id();
  if (lane < take) {
    const u64 w = widen_comp<C>(slot, idbits);
    out_ids[qi * stride + lane] = (u32)(w & 0xffffffffull);
    out_lcps[qi * stride + lane] = (uint16_t)(L - (int)(w >> 32));
  }
  if (lane == 0) {
    out_hits[qi] = take;
    out_md[qi] = (uint16_t)dmax;
    out_aux[2 * qi] = (u64)(u32)dmax | ((u64)(u32)dstar << 32);
    out_aux[2 * qi + 1] = (u64)rsize | ((u64)rlo << 32);
  }
}

// d* = max{d : #{window items with lcp >= d} >= need}.  One REDUX counts the
// four levels d_max .. d_max-3 at once (8-bit fields; a window holds <= 96
// items), which settles most queries; the rest binary-search below them.
template <int T>
__device__ __forceinline__ int window_dstar(const int (&l)[T], int dmax, int need) {
  if (dmax <= 0) return 0;
  // counts <= 32*T: four 8-bit fields while they fit, else two 16-bit fields
  constexpr int FB = 32 * T < 256 ? 8 : 16;
  constexpr int NL = 32 / FB;
  constexpr u32 FM = (1u << FB) - 1u;
  u32 mine = 0;
#pragma unroll
  for (int t = 0; t < T; ++t) {
#pragma unroll
    for (int c = 0; c < NL; ++c) mine += (u32)(l[t] >= dmax - c) << (FB * c);
  }
  const u32 tot = __reduce_add_sync(LCP_FULL_MASK, mine);
#pragma unroll
  for (int c = 0; c < NL; ++c) {
    if (dmax - c < 0) return 0;
    if ((int)((tot >> (FB * c)) & FM) >= need) return dmax - c;
  }
  int lo = 0, hi = dmax - NL;  // every level above failed
  if (hi <= 0) return 0;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    u32 mine = 0;
#pragma unroll
    for (int t = 0; t < T; ++t) mine += l[t] >= mid;
    const int c = (int)__reduce_add_sync(LCP_FULL_MASK, mine);
    if (c >= need) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// strict / complete / TAL, k <= 32, W == 1 (the config-3 hot path): one warp
// per query.  The 64-ary search tables narrow lower_bound(q) to a 16-key
// leaf block [B, B+16); the warp then loads a 64-key (need <= 16) or 96-key
// region around it with its ids in one coalesced round trip.  That region
// contains the window [pos-need, pos+need) for any pos in (B, B+16], so it
// serves d* and the candidate scan at once.  Candidates (lcp >= d*) form one
// run; it is compacted to one per lane and ranked by all-pairs comparison of
// (L-lcp)<<idbits|id.
// ---------------------------------------------------------------------------
__device__ __forceinline__ long long prefix_bound(const DevIndex& ix, const u64* q, int d,
                                                  bool upper);

// One 64-ary search step over a level table: number of entries < q among
// the 64 separators [blk*64, blk*64+64) (two per lane).  Tables are padded
// to whole blocks with all-ones keys, which never compare below q.
__device__ __forceinline__ int level_count(const u64* tab, int blk, u64 q) {
  const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(tab + blk * LCP_SEARCH_FANOUT + 2 * lane_id());
  return (int)__reduce_add_sync(LCP_FULL_MASK, (u32)(v.x < q) + (u32)(v.y < q));
}
__device__ __forceinline__ int level_count_g(const u64* __restrict__ tab, int blk, u64 q) {
  const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(tab + blk * LCP_SEARCH_FANOUT) + lane_id());
  return (int)__reduce_add_sync(LCP_FULL_MASK, (u32)(v.x < q) + (u32)(v.y < q));
}

// strict / complete: <= 32 regs, so two batches share an SM; TAL: 64 regs
// for the unrolled bucket sweep
// TAL bucket [blo, bhi) of the packed W == 1 query q (tal.py:116-143): the
// dense directory when built, else the two prefix bounds
__device__ __forceinline__ void tal_bucket_w1(const DevIndex& ix, u64 q, int& blo, int& bhi) {
  const int d = ix.tal_depth, b = ix.b;
  if (d > 0) {
    if (ix.directory) {
      long long code = 0;
      for (int j = 0; j < d; ++j)
        code = code * ix.sigma + (long long)((q >> (64 - b * (j + 1))) & ((1ull << b) - 1));
      blo = (int)__ldg(ix.directory + code);
      bhi = (int)__ldg(ix.directory + code + 1);
    } else {
      u64 qk1[1] = {q};
      blo = (int)prefix_bound(ix, qk1, d, false);
      bhi = (int)prefix_bound(ix, qk1, d, true);
    }
  }
}

// TAL symbols_compared (tal.py:173-177) = sum over the bucket B of
// min(lcp_i + 1, L) = sum_{d=0}^{L-1} #{i in B : lcp_i >= d}
//   = |B| * (1 + min(dB, L-1)) + sum_{d=dB+1}^{L-1} |R(d)|,
// because B = R(dB) (every bucket item matches q's first dB symbols) and, for
// d > dB, {i in B : lcp_i >= d} = R(d), the run of sorted rows sharing q's
// d-prefix.  R(d) within the leaf region is read off the region's lcps (one
// ballot per depth, depths dB+1..dmax, R(d) empty beyond dmax).  A run that
// reaches a region edge continues to its true edge: left of the region the
// lcps are non-decreasing towards q's position, right of it non-increasing,
// so each edge is the boundary of a monotone predicate.  All those searches
// (one per (depth, side), at most 32) run together: the warp splits into
// groups of G = 32 / #searches lanes, each group probes G points of its
// interval per round, so an interval shrinks (G+1)-fold per dependent L2 round
// trip (the former lane-per-search binary search took log2|B| round trips).
// So the count costs a few dependent probes instead of a sweep over the whole
// bucket (the former tal_sym_w1 read every bucket item: 128 MB of L2 traffic
// per 4096-query batch at config 3, B = 256).  W == 1 keys.
template <int T>
__device__ __forceinline__ unsigned long long tal_sym_region(const DevIndex& ix, u64 q, int blo, int bhi,
                                                             const int (&l)[T], int s, int dmax) {
  const int lane = lane_id();
  const int L = ix.L, dB = ix.tal_depth, lb = ix.lb;
  unsigned long long sym = (unsigned long long)(bhi - blo) * (unsigned long long)(1 + min(dB, L - 1));
  const int l0 = __shfl_sync(LCP_FULL_MASK, l[0], 0);        // position s
  const int lz = __shfl_sync(LCP_FULL_MASK, l[T - 1], 31);   // position s + 32T - 1
  const int e = s + 32 * T;                                  // first position after the region
  const int dtop = min(dmax, L - 1);
  for (int d = dB + 1; d <= dtop; ++d) {
    int c = 0;
#pragma unroll
    for (int t = 0; t < T; ++t) c += __popc(__ballot_sync(LCP_FULL_MASK, l[t] >= d));
    if (c == 0) break;  // R(d) is nested: nothing deeper either
    sym += (unsigned long long)c;
  }
  // runs leaving the region: depths dB+1..Dl on the left (R(d) contains
  // position s iff l0 >= d), dB+1..Dr on the right
  const int nl = s > blo ? max(0, min(l0, dtop) - dB) : 0;
  const int nr = e < bhi ? max(0, min(lz, dtop) - dB) : 0;
  const int K = nl + nr;
  if (K == 0) return sym;
  unsigned long long extra = 0;
  for (int k0 = 0; k0 < K; k0 += 32) {  // K <= L - 1 < 64: at most two passes
    const int kn = min(32, K - k0);
    // lanes per search G = 2^j - 1 <= 32 / kn: the G probes split an interval
    // into 2^j parts with shifts (no division)
    const int j = 31 - __clz(32 / kn + 1);
    const int G = (1 << j) - 1;
    const int g = lane / G, r = lane - g * G;
    const int k = k0 + g;                  // this lane's search (valid iff g < kn)
    const bool live = g < kn;
    const bool left = k < nl;
    const int d = dB + 1 + (left ? k : k - nl);
    // left: first i in [blo, s) with lcp_i >= d; right: first i in [e, bhi)
    // with lcp_i < d.  The answer lies in [lo, hi].
    int lo = left ? blo : e, hi = left ? s : bhi;
    const unsigned gmask = live ? (G == 32 ? LCP_FULL_MASK : (((1u << G) - 1u) << (g * G))) : 0u;
    while (__any_sync(LCP_FULL_MASK, live && lo < hi)) {
      const int span = hi - lo;  // lo < hi: probe G interior points of [lo, hi)
      const int p = lo + (int)(((long long)(r + 1) * span) >> j);
      bool pred = false;
      if (live && lo < hi) {
        const u64 x = __ldg(ix.keys + p) ^ q;
        const int lp = x ? min(__clzll((long long)x) >> lb, L) : L;
        pred = left ? lp >= d : lp < d;
      }
      const unsigned m = __ballot_sync(LCP_FULL_MASK, pred) & gmask;
      if (live && lo < hi) {
        if (m) {  // first true probe r*: answer in (p_{r*-1}, p_{r*}]
          const int rs = __ffs(m) - 1 - g * G;
          hi = lo + (int)(((long long)(rs + 1) * span) >> j);
          if (rs > 0) lo = lo + (int)(((long long)rs * span) >> j) + 1;
        } else {  // every probe false: answer in (p_{G-1}, hi]
          lo = lo + (int)(((long long)G * span) >> j) + 1;
        }
      }
    }
    if (live && r == 0) extra += left ? (unsigned long long)(s - lo) : (unsigned long long)(lo - e);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) extra += __shfl_xor_sync(LCP_FULL_MASK, extra, o);
  return sym + extra;
}

// One query of k_query_w1 (below) for the warp: row `qrow`, output slot qi.
// Shared by the batch kernel and the persistent single-query server.
template <typename C, int T, int MODE>
__device__ __forceinline__ void query_w1_one(const DevIndex& ix, const uint16_t* __restrict__ qrow, int qi,
                                             int k, int stride, u32* __restrict__ out_ids,
                                             uint16_t* __restrict__ out_lcps, int* __restrict__ out_hits,
                                             uint16_t* __restrict__ out_md, u64* __restrict__ out_aux,
                                             int* __restrict__ err, u64* bar, const u64* staged) {
  // MODE: 0 strict, 1 complete, 2 tal (trie.MODE_CODES)
  const int lane = lane_id();
  const int n = (int)ix.n;  // < 2**31 by contract
  const int L = ix.L;
  const int b = ix.b, lb = ix.lb;
  const int idbits = ix.idbits;
  // complete: min(k, n) hits; strict: up to k; tal: the top-k of the bucket,
  // which is the complete-mode answer with need = k whenever |bucket| >= k
  const int need = MODE == 1 ? min(k, n) : k;
  const u64* __restrict__ keys = ix.keys;
  const u32* __restrict__ order = ix.order;
  // W == 1  =>  L <= 64: lane packs symbols lane and lane + 32
  const bool has0 = lane < L, has1 = lane + 32 < L;
  const int sh0 = 64 - b * (lane + 1), sh1 = 64 - b * (lane + 33);

  LCP_STAMP(qi, 0);
  const u32 s0 = has0 ? qrow[lane] : 0u;
  bool bad = has0 && (int)s0 >= ix.sigma;
  u64 v = has0 ? (u64)s0 << sh0 : 0ull;
  if (L > 32) {  // warp-uniform: only sigma = 2 keys hold more than 32 symbols
    const u32 s1 = has1 ? qrow[lane + 32] : 0u;
    bad |= has1 && (int)s1 >= ix.sigma;
    v |= has1 ? (u64)s1 << sh1 : 0ull;
  }
  const u64 q = ((u64)__reduce_or_sync(LCP_FULL_MASK, (u32)(v >> 32)) << 32) |
                (u64)__reduce_or_sync(LCP_FULL_MASK, (u32)v);
  const bool any_bad = __any_sync(LCP_FULL_MASK, bad);
  if (any_bad) {
    stage_wait(ix, bar);
    if (lane == 0) {
      raise_flag(err);
      out_hits[qi] = 0;
      out_md[qi] = 0;
      out_aux[2 * qi] = 0;
      out_aux[2 * qi + 1] = 0;
    }
    return;
  }
  // TAL: the query's d-prefix bucket [blo, bhi) (tal.py:116-143), looked up
  // before the search so the directory read overlaps it
  int blo = 0, bhi = n;
  if constexpr (MODE == 2) tal_bucket_w1(ix, q, blo, bhi);
  stage_wait(ix, bar);  // first iteration: the query load overlaps the copy
  LCP_STAMP(qi, 1);
  // 64-ary search down to the 16-key leaf block holding lower_bound(q).
  // Only the root can count 0 separators below q (q <= every key: pos = 0);
  // below it, a child block starts with its parent's separator, which is < q.
  int blk = 0;
  if (ix.nlevels > 0) {
    const int c0 = ix.smem_levels > 0 ? level_count(staged, 0, q) : level_count_g(ix.levels, 0, q);
    if (c0 > 0) {
      blk = c0 - 1;
      int j = 1;
#pragma unroll 1
      for (; j < ix.smem_levels; ++j)
        blk = blk * LCP_SEARCH_FANOUT + level_count(staged + (int)ix.level_off[j], blk, q) - 1;
#pragma unroll 1
      for (; j < ix.nlevels; ++j)
        blk = blk * LCP_SEARCH_FANOUT + level_count_g(ix.levels + (int)ix.level_off[j], blk, q) - 1;
    }
  }
  LCP_STAMP(qi, 2);
  // Leaf block [B, B+16) holds pos = lower_bound(q) in (B, B+16] (or
  // pos = 0); the region is warp-strided (item t*32 + lane) and pos is
  // never materialised.
  static_assert(LCP_LEAF_KEYS == 16, "region offsets below assume 16-key leaf blocks");
  // pos in (B, B + 16]: the region [B - (16T - 8), ...) of 32T keys holds
  // [pos - need, pos + need) for need <= 16 (T=2) / 32 (T=3) with the
  // slack split evenly around the leaf block
  const int s = blk * LCP_LEAF_KEYS - (16 * T - 8);
  int l[T];
  u32 id[T];
  int dmax = -1;
  // unconditional loads at a clamped index (n >= 1), masked afterwards;
  // lcp = min(clz64(key ^ q) >> lb, L) is exact for W == 1 (clz64(0) = 64)
  u64 key[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int ic = min(max(s + t * 32 + lane, 0), n - 1);
    key[t] = __ldg(keys + ic);
    id[t] = __ldg(order + ic);
  }
#pragma unroll
  for (int t = 0; t < T; ++t) {
    // branch-free (-1 outside [0, n)): a branch here let the compiler sink
    // the key load behind it
    const int ok_mask = (unsigned)(s + t * 32 + lane) < (unsigned)n ? 0 : -1;
    l[t] = min(__clzll((long long)(key[t] ^ q)) >> lb, L) | ok_mask;
    dmax = max(dmax, l[t]);
  }
  dmax = (int)__reduce_max_sync(LCP_FULL_MASK, (unsigned)(dmax + 1)) - 1;
  LCP_STAMP(qi, 3);

  int md = dmax;
  u64 aux0 = 0, aux1 = 0;
  bool tal_small = false;  // bucket smaller than k: answer = the whole bucket
  if constexpr (MODE == 2) {
    const unsigned long long sym = tal_sym_region<T>(ix, q, blo, bhi, l, s, dmax);
    md = ix.tal_depth;
    aux0 = (u64)(bhi - blo);
    aux1 = sym;
    tal_small = bhi - blo < k;
    if (bhi == blo) {  // empty bucket: no hits, nothing scanned (tal.py:168-171)
      if (lane == 0) {
        out_hits[qi] = 0;
        out_md[qi] = (uint16_t)md;
        out_aux[2 * qi] = 0;
        out_aux[2 * qi + 1] = 0;
      }
      return;
    }
  }
  if (tal_small) {
    // |bucket| < k <= 32: rank the whole bucket, one item per lane
    const int bs = bhi - blo;
    C cv = ~C(0);
    if (lane < bs) {
      const u64 x = __ldg(keys + blo + lane) ^ q;
      const int ll = x ? (__clzll((long long)x) >> lb) : L;
      cv = make_comp<C>(ll, __ldg(order + blo + lane), L, idbits);
    }
    int rank = 0;
    for (int jj = 0; jj < bs; ++jj) rank += __shfl_sync(LCP_FULL_MASK, cv, jj) < cv;
    if (lane < bs) {
      const u64 w = widen_comp<C>(cv, idbits);
      out_ids[(size_t)qi * stride + rank] = (u32)(w & 0xffffffffull);
      out_lcps[(size_t)qi * stride + rank] = (uint16_t)(L - (int)(w >> 32));
    }
    if (lane == 0) {
      out_hits[qi] = bs;
      out_md[qi] = (uint16_t)md;
      out_aux[2 * qi] = aux0;
      out_aux[2 * qi + 1] = aux1;
    }
    return;
  }

  const int dstar = MODE == 0 ? dmax : window_dstar<T>(l, dmax, need);
  if constexpr (MODE != 2) {
    aux0 = (u64)(u32)dmax | ((u64)(u32)dstar << 32);
  }
  C comp[T];
  int cnt = 0, r0 = 32 * T;
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const bool c = l[t] >= dstar;
    comp[t] = c ? make_comp<C>(l[t], id[t], L, idbits) : ~C(0);
    const unsigned m = __ballot_sync(LCP_FULL_MASK, c);
    cnt += __popc(m);
    if (m && r0 == 32 * T) r0 = t * 32 + __ffs(m) - 1;
  }
  const int first_valid = s < 0 ? -s : 0;
  const int end = min(s + 32 * T, n);
  const bool left = s > 0 && r0 == first_valid;
  const bool right = end < n && s + r0 + cnt == end;
  LCP_STAMP(qi, 4);
  if (!left && !right && cnt <= 32) {
    // R(d*) lies inside the region: compact the run to one candidate per
    // lane and rank it by all-pairs comparison (independent shuffles, no
    // sorting network); the lane of rank r writes output slot r.
    const int t0 = r0 >> 5, e = r0 + lane;
    const C a = __shfl_sync(LCP_FULL_MASK, pick_slot<C, T>(comp, t0), e & 31);
    const C bb = __shfl_sync(LCP_FULL_MASK, pick_slot<C, T>(comp, t0 + 1), e & 31);
    const C cv = lane < cnt ? (((e >> 5) == t0) ? a : bb) : ~C(0);
    // all-pairs rank in blocks of 8 with immediate shuffle lanes; lanes >= cnt
    // hold all-ones and never count, so only the block guard is needed
    int rank = 0;
#pragma unroll
    for (int blk8 = 0; blk8 < 32; blk8 += 8) {
      if (blk8 >= cnt) break;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) rank += __shfl_sync(LCP_FULL_MASK, cv, blk8 + jj) < cv;
    }
    LCP_STAMP(qi, 5);
    const int take = min(need, cnt);
    if (lane < cnt && rank < take) {
      const u64 w = widen_comp<C>(cv, idbits);
      out_ids[(size_t)qi * stride + rank] = (u32)(w & 0xffffffffull);
      out_lcps[(size_t)qi * stride + rank] = (uint16_t)(L - (int)(w >> 32));
    }
    if (lane == 0) {
      out_hits[qi] = take;
      out_md[qi] = (uint16_t)md;
      out_aux[2 * qi] = aux0;
      out_aux[2 * qi + 1] = MODE == 2 ? aux1 : ((u64)(u32)cnt | ((u64)(u32)(s + r0) << 32));
    }
    LCP_STAMP(qi, 6);
    LCP_STAMP(qi, 7);
    return;
  }
  C slot = sort_run<C, T>(comp, r0, cnt, need);
  LCP_STAMP(qi, 5);
  u64 qk[1] = {q};
  long long rsize = cnt, rlo = s + r0;
  extend_range<C, 1>(ix, qk, dstar, need, left, s, right, end, idbits, slot, rsize, rlo);
  LCP_STAMP(qi, 6);
  const int take = (int)min((long long)need, rsize);
  if (lane < take) {
    const u64 w = widen_comp<C>(slot, idbits);
    out_ids[(size_t)qi * stride + lane] = (u32)(w & 0xffffffffull);
    out_lcps[(size_t)qi * stride + lane] = (uint16_t)(L - (int)(w >> 32));
  }
  if (lane == 0) {
    out_hits[qi] = take;
    out_md[qi] = (uint16_t)md;
    out_aux[2 * qi] = aux0;
    out_aux[2 * qi + 1] = MODE == 2 ? aux1 : ((u64)rsize | ((u64)rlo << 32));
  }
  LCP_STAMP(qi, 7);
}

template <typename C, int T, int MODE>
__global__ void __launch_bounds__(QW_MAX_THREADS, MODE == 2 ? 1 : 2)
    k_query_w1(const __grid_constant__ DevIndex ix, const uint16_t* __restrict__ queries, int count, int k,
               int stride, u32* __restrict__ out_ids, uint16_t* __restrict__ out_lcps,
               int* __restrict__ out_hits, uint16_t* __restrict__ out_md,
               u64* __restrict__ out_aux, int* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  u64* bar = reinterpret_cast<u64*>(smem_raw);
  u64* staged = reinterpret_cast<u64*>(smem_raw + 16);
  stage_issue(ix, bar, staged);
  const int warp = threadIdx.x >> 5;
  const int warps = blockDim.x >> 5;
  if (ix.dcount) count = min(count, *ix.dcount);  // device-resident batch size (lcp_query_counted)
  for (int qi = blockIdx.x * warps + warp; qi < count; qi += gridDim.x * warps)
    query_w1_one<C, T, MODE>(ix, queries + (size_t)qi * ix.L, qi, k, stride, out_ids, out_lcps, out_hits,
                             out_md, out_aux, err, bar, staged);
}

// ---------------------------------------------------------------------------
// strict / complete, 32 < need <= 32 * NS (NS = 2 or 4), W == 1: one warp
// per query with an NS-slot top-k list (lane i holds ranks i, i + 32, ...).
// Same search as k_query_w1; the region [B - 32 NS, B + 32 + 32 NS) contains
// [pos - 32 NS, pos + 32 NS).
// ---------------------------------------------------------------------------
template <typename C, int NS>
struct TopKN {
  static constexpr int M = 32 * NS;
  C s[NS];  // s[j] on lane i holds rank 32 * j + i
  C thr;
  C* sc;    // the warp's M-entry shared buffer (batch merges)
  __device__ __forceinline__ void init(C* buf) {
#pragma unroll
    for (int j = 0; j < NS; ++j) s[j] = ~C(0);
    thr = ~C(0);
    sc = buf;
  }
  __device__ __forceinline__ void set_thr(int need) {
    const int r = need - 1;
    C sel = s[0];
#pragma unroll
    for (int j = 1; j < NS; ++j)
      if ((r >> 5) == j) sel = s[j];
    thr = __shfl_sync(LCP_FULL_MASK, sel, r & 31);
  }
  // Merges one candidate per lane at once: the batch is sorted across lanes
  // (bitonic), list entry (lane, j) moves to rank 32 j + lane + #{batch < it}
  // and batch entry q to q + #{list <= it} (ties list-first, so the ranks are
  // a bijection onto [0, M + 32)); ranks below M are scattered through sc.
  __device__ __forceinline__ void merge_batch(C x, int need) {
    const int lane = lane_id();
#pragma unroll
    for (int k2 = 2; k2 <= 32; k2 <<= 1) {
#pragma unroll
      for (int j = k2 >> 1; j > 0; j >>= 1) {
        const C y = __shfl_xor_sync(LCP_FULL_MASK, x, j);
        x = (((lane & j) == 0) == ((lane & k2) == 0)) ? cmin(x, y) : cmax(x, y);
      }
    }
#pragma unroll
    for (int j = 0; j < NS; ++j) sc[32 * j + lane] = s[j];
    __syncwarp();
    int nl = 0;
#pragma unroll
    for (int step = M / 2; step; step >>= 1)
      if (sc[nl + step - 1] <= x) nl += step;
    if (sc[nl] <= x) ++nl;
    int nb[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      int p = 0;
#pragma unroll
      for (int step = 16; step; step >>= 1)
        if (__shfl_sync(LCP_FULL_MASK, x, p + step - 1) < s[j]) p += step;
      if (__shfl_sync(LCP_FULL_MASK, x, p) < s[j]) ++p;
      nb[j] = p;
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      const int r = 32 * j + lane + nb[j];
      if (r < M) sc[r] = s[j];
    }
    if (lane + nl < M) sc[lane + nl] = x;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < NS; ++j) s[j] = sc[32 * j + lane];
    __syncwarp();
    set_thr(need);
  }
  __device__ __forceinline__ void insert(C c, int need) {
    const int lane = lane_id();
    int p = 0;
#pragma unroll
    for (int j = 0; j < NS; ++j) p += __popc(__ballot_sync(LCP_FULL_MASK, s[j] < c));
    C top[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) top[j] = __shfl_sync(LCP_FULL_MASK, s[j], 31);
#pragma unroll
    for (int j = NS - 1; j >= 0; --j) {
      const C up = __shfl_up_sync(LCP_FULL_MASK, s[j], 1);
      const int h = lane + 32 * j;
      const C prev = lane == 0 ? (j > 0 ? top[j > 0 ? j - 1 : 0] : s[j]) : up;
      s[j] = h > p ? prev : (h == p ? c : s[j]);
    }
    set_thr(need);
  }
  // one candidate per lane (all-ones = none): a few by single insertions,
  // more by one batch merge
  __device__ __forceinline__ void offer(C comp, int need) {
    unsigned m = __ballot_sync(LCP_FULL_MASK, comp < thr);
    if (__popc(m) > 4) {
      merge_batch(comp < thr ? comp : ~C(0), need);
      return;
    }
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      const C c = __shfl_sync(LCP_FULL_MASK, comp, src);
      if (c < thr) insert(c, need);
    }
  }
};

// tier|id over sorted positions [a, b) through the id sketch (see tier_offer);
// valid while the tier contributes at most 32 items (one sketch list each)
template <typename C, int NS>
__device__ __noinline__ TopKN<C, NS> tier_offer_n(const DevIndex& ix, long long a, long long b, C tier,
                                                 TopKN<C, NS> lst, int need) {
  auto positions = [&](long long x, long long y) {
    for (long long base = x; base < y; base += 32) {
      const long long i = base + lane_id();
      lst.offer(i < y ? (tier | (C)__ldg(ix.order + i)) : ~C(0), need);
    }
  };
  auto lists = [&](const u32* __restrict__ ls, long long x, long long y) {
    for (long long base = x; base < y; base += 32) {
      const long long blk = base + lane_id();
      const u32 mn = blk < y ? __ldg(ls + blk * LCP_SK_LIST) : 0xffffffffu;
      const C cm = mn == 0xffffffffu ? ~C(0) : (tier | (C)mn);
      unsigned m = __ballot_sync(LCP_FULL_MASK, cm < lst.thr);
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        if (__shfl_sync(LCP_FULL_MASK, cm, src) < lst.thr) {
          const u32 v = __ldg(ls + (base + src) * LCP_SK_LIST + lane_id());
          lst.offer(v == 0xffffffffu ? ~C(0) : (tier | (C)v), need);
        }
      }
    }
  };
  long long A = (a + LCP_SK_BLOCK - 1) / LCP_SK_BLOCK, B = b / LCP_SK_BLOCK;
  if (A >= B) {
    positions(a, b);
    return lst;
  }
  positions(a, A * LCP_SK_BLOCK);
  positions(B * LCP_SK_BLOCK, b);
  for (int j = 0;; ++j) {
    const u32* ls = ix.sketch + ix.sk_off[j] * LCP_SK_LIST;
    const long long A2 = (A + LCP_SK_FANOUT - 1) / LCP_SK_FANOUT, B2 = B / LCP_SK_FANOUT;
    if (j + 1 >= ix.sk_levels || A2 >= B2) {
      lists(ls, A, B);
      return lst;
    }
    lists(ls, A, A2 * LCP_SK_FANOUT);
    lists(ls, B2 * LCP_SK_FANOUT, B);
    A = A2;
    B = B2;
  }
}

template <typename C, int MODE, int NS>
__global__ void __launch_bounds__(NS > 2 ? QW_MAX_THREADS / 2 : QW_MAX_THREADS, 1)  // NS=4: 128 regs
    k_query_w1_kn(const __grid_constant__ DevIndex ix, const uint16_t* __restrict__ queries,
                   int count, int k, int stride, u32* __restrict__ out_ids,
                   uint16_t* __restrict__ out_lcps, int* __restrict__ out_hits,
                   uint16_t* __restrict__ out_md, u64* __restrict__ out_aux, int* __restrict__ err) {
  // MODE: 0 strict, 1 complete, 2 tal; need <= 32 * NS; region 32 * (2 NS + 1)
  // keys.  TAL (k > 32 here): the complete answer with need = k when the
  // bucket holds >= k items, else the whole bucket ranked; symbols_compared by
  // the bucket sweep (see k_query_w1)
  constexpr int T = 2 * NS + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  u64* bar = reinterpret_cast<u64*>(smem_raw);
  u64* staged = reinterpret_cast<u64*>(smem_raw + 16);
  stage_issue(ix, bar, staged);
  const int lane = lane_id();
  const int warp = threadIdx.x >> 5;
  const int warps = blockDim.x >> 5;
  const int n = (int)ix.n;
  const int L = ix.L;
  const int b = ix.b, lb = ix.lb;
  const int idbits = ix.idbits;
  const int need = MODE == 1 ? min(k, n) : k;
  const u64* __restrict__ keys = ix.keys;
  const u32* __restrict__ order = ix.order;
  const bool has0 = lane < L, has1 = lane + 32 < L;
  const int sh0 = 64 - b * (lane + 1), sh1 = 64 - b * (lane + 33);

  if (ix.dcount) count = min(count, *ix.dcount);  // device-resident batch size (lcp_query_counted)
  for (int qi = blockIdx.x * warps + warp; qi < count; qi += gridDim.x * warps) {
    const uint16_t* qrow = queries + (size_t)qi * L;
    const u32 s0 = has0 ? qrow[lane] : 0u;
    const u32 s1 = has1 ? qrow[lane + 32] : 0u;
    const bool bad = (has0 && (int)s0 >= ix.sigma) || (has1 && (int)s1 >= ix.sigma);
    const u64 v = (has0 ? (u64)s0 << sh0 : 0ull) | (has1 ? (u64)s1 << sh1 : 0ull);
    const u64 q = ((u64)__reduce_or_sync(LCP_FULL_MASK, (u32)(v >> 32)) << 32) |
                  (u64)__reduce_or_sync(LCP_FULL_MASK, (u32)v);
    stage_wait(ix, bar);
    if (__any_sync(LCP_FULL_MASK, bad)) {
      if (lane == 0) {
        raise_flag(err);
        out_hits[qi] = 0;
        out_md[qi] = 0;
        out_aux[2 * qi] = 0;
        out_aux[2 * qi + 1] = 0;
      }
      continue;
    }
    int blo = 0, bhi = n;
    if constexpr (MODE == 2) tal_bucket_w1(ix, q, blo, bhi);
    int blk = 0;
    if (ix.nlevels > 0) {
      const int c0 = ix.smem_levels > 0 ? level_count(staged, 0, q) : level_count_g(ix.levels, 0, q);
      if (c0 > 0) {
        blk = c0 - 1;
        int j = 1;
#pragma unroll 1
        for (; j < ix.smem_levels; ++j)
          blk = blk * LCP_SEARCH_FANOUT + level_count(staged + (int)ix.level_off[j], blk, q) - 1;
#pragma unroll 1
        for (; j < ix.nlevels; ++j)
          blk = blk * LCP_SEARCH_FANOUT + level_count_g(ix.levels + (int)ix.level_off[j], blk, q) - 1;
      }
    }
    const int s = blk * LCP_LEAF_KEYS - 32 * NS;
    int l[T];
    u32 id[T];
    int dmax = -1;
    u64 key[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int ic = min(max(s + t * 32 + lane, 0), n - 1);
      key[t] = __ldg(keys + ic);
      id[t] = __ldg(order + ic);
    }
#pragma unroll
    for (int t = 0; t < T; ++t) {
      // branch-free (-1 outside [0, n)): a branch here let the compiler sink
      // the key load behind it
      const int ok_mask = (unsigned)(s + t * 32 + lane) < (unsigned)n ? 0 : -1;
      l[t] = min(__clzll((long long)(key[t] ^ q)) >> lb, L) | ok_mask;
      dmax = max(dmax, l[t]);
    }
    dmax = (int)__reduce_max_sync(LCP_FULL_MASK, (unsigned)(dmax + 1)) - 1;
    TopKN<C, NS> lst;
    lst.init(reinterpret_cast<C*>(smem_raw + 16 + (size_t)ix.smem_entries * 8) + warp * (32 * NS));
    unsigned long long tsym = 0;
    if constexpr (MODE == 2) {
      tsym = tal_sym_region<T>(ix, q, blo, bhi, l, s, dmax);
      const int bs = bhi - blo;
      if (bs < k) {  // the whole bucket, ranked (an empty one included)
        for (int base = blo; base < bhi; base += 32) {
          const int i = base + lane;
          C cv = ~C(0);
          if (i < bhi) {
            const u64 x = __ldg(keys + i) ^ q;
            cv = make_comp<C>(x ? (__clzll((long long)x) >> lb) : L, __ldg(order + i), L, idbits);
          }
          lst.offer(cv, k);
        }
#pragma unroll
        for (int j = 0; j < NS; ++j) {
          if (lane + 32 * j < bs) {
            const u64 w = widen_comp<C>(lst.s[j], idbits);
            out_ids[(size_t)qi * stride + lane + 32 * j] = (u32)(w & 0xffffffffull);
            out_lcps[(size_t)qi * stride + lane + 32 * j] = (uint16_t)(L - (int)(w >> 32));
          }
        }
        if (lane == 0) {
          out_hits[qi] = bs;
          out_md[qi] = (uint16_t)ix.tal_depth;
          out_aux[2 * qi] = (u64)bs;
          out_aux[2 * qi + 1] = tsym;
        }
        continue;
      }
    }
    const int dstar = MODE == 0 ? dmax : window_dstar<T>(l, dmax, need);
    int cnt = 0, r0 = 32 * T, above = 0;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const bool c = l[t] >= dstar;
      const unsigned m = __ballot_sync(LCP_FULL_MASK, c);
      cnt += __popc(m);
      above += __popc(__ballot_sync(LCP_FULL_MASK, l[t] > dstar));
      if (m && r0 == 32 * T) r0 = t * 32 + __ffs(m) - 1;
      lst.offer(c ? make_comp<C>(l[t], id[t], L, idbits) : ~C(0), need);
    }
    const int first_valid = s < 0 ? -s : 0;
    const int end = min(s + 32 * T, n);
    long long rsize = cnt, rlo = s + r0;
    // R(d*) past the region: outside it every item has lcp == d*
    const C tier = make_comp<C>(dstar, 0u, L, idbits);
    const bool sketch_ok = need - above <= LCP_SK_LIST;  // tier supplies <= 32 items
    // up to EXT_SCAN_CHUNKS chunks outward on each side
    bool goL = s > 0 && r0 == first_valid, goR = end < n && s + r0 + cnt == end;
    long long eL = s, eR = end;  // [eL, eR) is scanned
    // d* = 0: the run is the whole corpus, so no chunk can end it
    const int ext_chunks = dstar ? EXT_SCAN_CHUNKS : 0;
    for (int chunk = 0; goL && chunk < ext_chunks; ++chunk) {
      const long long i = eL - 32 + lane;
      const int li = i >= 0 ? min(__clzll((long long)(__ldg(keys + i) ^ q)) >> lb, L) : -1;
      const bool c = li >= dstar;
      lst.offer(c ? make_comp<C>(li, __ldg(order + i), L, idbits) : ~C(0), need);
      const unsigned m = __ballot_sync(LCP_FULL_MASK, c);
      rsize += __popc(m);
      if (m) rlo = eL - 32 + (__ffs(m) - 1);
      eL -= 32;
      goL = m == LCP_FULL_MASK && eL > 0;
    }
    for (int chunk = 0; goR && chunk < ext_chunks; ++chunk) {
      const long long i = eR + lane;
      const int li = i < n ? min(__clzll((long long)(__ldg(keys + i) ^ q)) >> lb, L) : -1;
      const bool c = li >= dstar;
      lst.offer(c ? make_comp<C>(li, __ldg(order + i), L, idbits) : ~C(0), need);
      const unsigned m = __ballot_sync(LCP_FULL_MASK, c);
      rsize += __popc(m);
      eR += 32;
      goR = m == LCP_FULL_MASK && eR < n;
    }
    if (goL || goR) {
      // the run goes on: its ends by run_edge; every item past the scanned
      // span has lcp == d* (R(d*+1) lies in the region), so only ids matter
      u64 qk1[1] = {q};
      const long long rl = goL ? (dstar ? run_edge<1>(ix, qk1, dstar, eL, -1) : 0) : eL;
      const long long rr = goR ? (dstar ? run_edge<1>(ix, qk1, dstar, eR - 1, n) + 1 : n) : eR;
      const long long rest = (eL - rl) + (rr - eR);
      rsize += rest;
      if (goL) rlo = rl;
      if (sketch_ok) {  // the id sketch: 32 smallest ids per block
        if (goL) lst = tier_offer_n<C, NS>(ix, rl, eL, tier, lst, need);
        if (goR) lst = tier_offer_n<C, NS>(ix, eR, rr, tier, lst, need);
      } else if (16 * rest >= n) {
        // most of the corpus: ids in ascending order through rank[], until
        // the list is full and no later id can enter
        for (long long base = 0; base < n && (tier | (C)base) < lst.thr; base += 32) {
          const long long id = base + lane;
          C cv = ~C(0);
          if (id < n) {
            const long long p = __ldg(ix.rank + id);
            if ((p >= rl && p < eL) || (p >= eR && p < rr)) cv = tier | (C)id;
          }
          lst.offer(cv, need);
        }
      } else {  // position by position, ids only
        for (long long base = rl; base < eL; base += 32) {
          const long long i = base + lane;
          lst.offer(i < eL ? (tier | (C)__ldg(order + i)) : ~C(0), need);
        }
        for (long long base = eR; base < rr; base += 32) {
          const long long i = base + lane;
          lst.offer(i < rr ? (tier | (C)__ldg(order + i)) : ~C(0), need);
        }
      }
    }
    const int take = (int)min((long long)need, rsize);
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      if (lane + 32 * j < take) {
        const u64 w = widen_comp<C>(lst.s[j], idbits);
        out_ids[(size_t)qi * stride + lane + 32 * j] = (u32)(w & 0xffffffffull);
        out_lcps[(size_t)qi * stride + lane + 32 * j] = (uint16_t)(L - (int)(w >> 32));
      }
    }
    if (lane == 0) {
      out_hits[qi] = take;
      if constexpr (MODE == 2) {
        out_md[qi] = (uint16_t)ix.tal_depth;
        out_aux[2 * qi] = (u64)(bhi - blo);
        out_aux[2 * qi + 1] = tsym;
      } else {
        out_md[qi] = (uint16_t)dmax;
        out_aux[2 * qi] = (u64)(u32)dmax | ((u64)(u32)dstar << 32);
        out_aux[2 * qi + 1] = (u64)rsize | ((u64)rlo << 32);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// strict / complete, k <= 32, 2 <= W <= WMAX <= 8: one warp per query;
// 64-ary search to pos, then the 64-key window [pos-32, pos+32).
// ---------------------------------------------------------------------------
template <int WMAX>
__global__ void __launch_bounds__(QW_MAX_THREADS, 1)
    k_query_warp(const __grid_constant__ DevIndex ix, const uint16_t* __restrict__ queries, int count, int k, int mode,
                 int stride, u32* __restrict__ out_ids, uint16_t* __restrict__ out_lcps,
                 int* __restrict__ out_hits, uint16_t* __restrict__ out_md,
                 u64* __restrict__ out_aux, int* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  u64* bar = reinterpret_cast<u64*>(smem_raw);
  u64* staged = reinterpret_cast<u64*>(smem_raw + 16);
  stage_levels(ix, bar, staged);

  const int lane = lane_id();
  const int warp = threadIdx.x >> 5;
  const long long n = ix.n;
  const int L = ix.L;
  const bool complete = mode == 1;

  const int warps = blockDim.x >> 5;
  if (ix.dcount) count = min(count, *ix.dcount);  // device-resident batch size (lcp_query_counted)
  for (long long qi = (long long)blockIdx.x * warps + warp; qi < count;
       qi += (long long)gridDim.x * warps) {
    u64 qk[WMAX];
    if (!warp_pack_query<WMAX>(queries + qi * L, ix, qk)) {
      if (lane == 0) {
        raise_flag(err);
        out_hits[qi] = 0;
        out_md[qi] = 0;
        out_aux[2 * qi] = 0;
        out_aux[2 * qi + 1] = 0;
      }
      continue;
    }
    const long long pos = warp_lower_bound<WMAX>(ix, staged, qk);
    const long long s = pos - 32;  // window [s, s+64), warp-strided
    int l[2];
    u32 id[2];
    int dmax = region_lcps<WMAX, 2>(ix, s, qk, l, id);
#pragma unroll
    for (int o = 16; o; o >>= 1) dmax = max(dmax, __shfl_xor_sync(LCP_FULL_MASK, dmax, o));
    const int need = complete ? (int)min((long long)k, n) : k;
    const int dstar = complete ? window_dstar<2>(l, dmax, need) : dmax;
    u64 comp[2];
    int cnt = 0, r0 = 64;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const bool c = l[t] >= dstar;
      comp[t] = c ? make_comp<u64>(l[t], id[t], L, 32) : ~0ull;
      const unsigned m = __ballot_sync(LCP_FULL_MASK, c);
      cnt += __popc(m);
      if (m && r0 == 64) r0 = t * 32 + __ffs(m) - 1;
    }
    u64 slot = sort_run<u64, 2>(comp, r0, cnt, need);
    long long rsize = cnt, rlo = s + r0;
    const long long first_valid = s < 0 ? -s : 0;
    const long long end = min(s + 64, n);
    const bool left = s > 0 && r0 == first_valid;
    const bool right = end < n && s + r0 + cnt == end;
    extend_range<u64, WMAX>(ix, qk, dstar, need, left, s, right, end, 32, slot, rsize, rlo);
    const int take = (int)min((long long)need, rsize);
    write_result<u64>(qi, stride, take, L, slot, 32, dmax, dstar, rsize, rlo, out_ids, out_lcps,
                      out_hits, out_md, out_aux);
  }
}

// bucket [lo, hi) of the query's d-prefix: dense directory (tal.py:138-143)
// or binary search on the packed d-prefixes (tal.py:124-136)
__device__ __forceinline__ void tal_bucket(const DevIndex& ix, const u64* qk,
                                           const uint16_t* qrow, long long& lo,
                                           long long& hi) {
  const int d = ix.tal_depth;
  if (d == 0) {
    lo = 0;
    hi = ix.n;
    return;
  }
  if (ix.directory) {
    long long code = 0;
    for (int j = 0; j < d; ++j) code = code * ix.sigma + qrow[j];
    lo = ix.directory[code];
    hi = ix.directory[code + 1];
    return;
  }
  long long a = 0, b = ix.n;
  while (a < b) {
    long long m = (a + b) >> 1;
    if (prefix_cmp(ix.keys + m * ix.W, qk, d, ix) < 0) a = m + 1;
    else b = m;
  }
  lo = a;
  b = ix.n;
  while (a < b) {
    long long m = (a + b) >> 1;
    if (prefix_cmp(ix.keys + m * ix.W, qk, d, ix) <= 0) a = m + 1;
    else b = m;
  }
  hi = a;
}

// symbols_compared = sum over the bucket [blo, bhi) of min(lcp + 1, L)
// (tal.py:173-177) for W > 1: a coalesced sweep of the sorted first-word
// plane, 4 loads in flight per lane; only keys equal to q in the whole first
// word compare further words.  The warp total on every lane.
template <int WMAX>
__device__ __forceinline__ unsigned long long tal_sym_warp(const DevIndex& ix, const u64 (&qk)[WMAX],
                                                           long long blo, long long bhi) {
  const int lane = lane_id();
  const int L = ix.L, lb = ix.lb;
  unsigned long long sym = 0;
  for (long long i0 = blo + lane; i0 < bhi; i0 += 128) {
    u64 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + 32 * u;
      x[u] = i < bhi ? __ldg(ix.keys_w0 + i) ^ qk[0] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + 32 * u;
      if (i < bhi) {
        const int li = x[u] ? (__clzll((long long)x[u]) >> lb) : lcp_at<WMAX>(ix, i, qk);
        sym += (unsigned)min(li + 1, L);
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sym += __shfl_xor_sync(LCP_FULL_MASK, sym, o);
  return sym;
}

// ---------------------------------------------------------------------------
// TAL, k <= 32, 2 <= W <= WMAX <= 8 (tal.py:116-194): one warp per query.
// The answer is the complete-mode answer with need = k whenever the bucket
// holds >= k items (then d* >= depth, so R(d*) lies inside the bucket);
// smaller buckets are ranked whole.  symbols_compared = sum over the bucket of
// min(lcp + 1, L) comes from a coalesced sweep of the sorted first-word plane;
// only keys equal to q in the whole first word compare further words.
// ---------------------------------------------------------------------------
template <int WMAX>
__global__ void __launch_bounds__(QW_MAX_THREADS, 1)
    k_query_warp_tal(const __grid_constant__ DevIndex ix, const uint16_t* __restrict__ queries,
                     int count, int k, int stride, u32* __restrict__ out_ids,
                     uint16_t* __restrict__ out_lcps, int* __restrict__ out_hits,
                     uint16_t* __restrict__ out_md, u64* __restrict__ out_aux,
                     int* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  u64* bar = reinterpret_cast<u64*>(smem_raw);
  u64* staged = reinterpret_cast<u64*>(smem_raw + 16);
  stage_levels(ix, bar, staged);
  const int lane = lane_id();
  const int warp = threadIdx.x >> 5;
  const int warps = blockDim.x >> 5;
  const long long n = ix.n;
  const int L = ix.L;
  const int depth = ix.tal_depth;
  if (ix.dcount) count = min(count, *ix.dcount);  // device-resident batch size (lcp_query_counted)
  for (long long qi = (long long)blockIdx.x * warps + warp; qi < count;
       qi += (long long)gridDim.x * warps) {
    u64 qk[WMAX];
    if (!warp_pack_query<WMAX>(queries + qi * L, ix, qk)) {
      if (lane == 0) {
        raise_flag(err);
        out_hits[qi] = 0;
        out_md[qi] = 0;
        out_aux[2 * qi] = 0;
        out_aux[2 * qi + 1] = 0;
      }
      continue;
    }
    long long blo, bhi;
    tal_bucket(ix, qk, queries + qi * L, blo, bhi);
    const unsigned long long sym = tal_sym_warp<WMAX>(ix, qk, blo, bhi);
    const long long bs = bhi - blo;
    if (bs < k) {  // the whole bucket (empty: no hits, nothing scanned, tal.py:168-171)
      u64 cv = ~0ull;
      if (lane < bs) cv = make_comp<u64>(lcp_at<WMAX>(ix, blo + lane, qk), ix.order[blo + lane], L, 32);
      int rank = 0;
      for (int jj = 0; jj < (int)bs; ++jj) rank += __shfl_sync(LCP_FULL_MASK, cv, jj) < cv;
      if (lane < bs) {
        out_ids[qi * stride + rank] = (u32)(cv & 0xffffffffull);
        out_lcps[qi * stride + rank] = (uint16_t)(L - (int)(cv >> 32));
      }
      if (lane == 0) {
        out_hits[qi] = (int)bs;
        out_md[qi] = (uint16_t)depth;
        out_aux[2 * qi] = (u64)bs;
        out_aux[2 * qi + 1] = bs ? sym : 0ull;
      }
      continue;
    }
    // complete-mode answer with need = k (as k_query_warp)
    const long long pos = warp_lower_bound<WMAX>(ix, staged, qk);
    const long long s = pos - 32;
    int l[2];
    u32 id[2];
    int dmax = region_lcps<WMAX, 2>(ix, s, qk, l, id);
#pragma unroll
    for (int o = 16; o; o >>= 1) dmax = max(dmax, __shfl_xor_sync(LCP_FULL_MASK, dmax, o));
    const int dstar = window_dstar<2>(l, dmax, k);
    u64 comp[2];
    int cnt = 0, r0 = 64;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const bool c = l[t] >= dstar;
      comp[t] = c ? make_comp<u64>(l[t], id[t], L, 32) : ~0ull;
      const unsigned m = __ballot_sync(LCP_FULL_MASK, c);
      cnt += __popc(m);
      if (m && r0 == 64) r0 = t * 32 + __ffs(m) - 1;
    }
    u64 slot = sort_run<u64, 2>(comp, r0, cnt, k);
    long long rsize = cnt, rlo = s + r0;
    const long long first_valid = s < 0 ? -s : 0;
    const long long end = min(s + 64, n);
    extend_range<u64, WMAX>(ix, qk, dstar, k, s > 0 && r0 == first_valid, s, end < n && s + r0 + cnt == end,
                            end, 32, slot, rsize, rlo);
    if (lane < k) {
      out_ids[qi * stride + lane] = (u32)(slot & 0xffffffffull);
      out_lcps[qi * stride + lane] = (uint16_t)(L - (int)(slot >> 32));
    }
    if (lane == 0) {
      out_hits[qi] = k;
      out_md[qi] = (uint16_t)depth;
      out_aux[2 * qi] = (u64)bs;
      out_aux[2 * qi + 1] = sym;
    }
  }
}


// ---------------------------------------------------------------------------
// strict / complete / TAL, 32 < need <= 32 * NS <= 128, 2 <= W <= WMAX <= 8:
// one warp per query with an NS-slot top-k list.  Window [pos - 32 NS,
// pos + 32 NS) after the 64-ary search; extension as in k_query_w1_kn (chunks,
// then the run's ends by run_edge and ids only: sketch, rank walk or
// positions).  TAL as in k_query_warp_tal: the whole bucket when it holds
// fewer than k items, else the complete answer with need = k.
// ---------------------------------------------------------------------------
template <int WMAX, int NS, bool TAL>
__global__ void __launch_bounds__(NS > 2 ? QW_MAX_THREADS / 2 : QW_MAX_THREADS, 1)
    k_query_warp_kn(const __grid_constant__ DevIndex ix, const uint16_t* __restrict__ queries,
                    int count, int k, int mode, int stride, u32* __restrict__ out_ids,
                    uint16_t* __restrict__ out_lcps, int* __restrict__ out_hits,
                    uint16_t* __restrict__ out_md, u64* __restrict__ out_aux,
                    int* __restrict__ err) {
  constexpr int T = 2 * NS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  u64* bar = reinterpret_cast<u64*>(smem_raw);
  u64* staged = reinterpret_cast<u64*>(smem_raw + 16);
  stage_levels(ix, bar, staged);
  const int lane = lane_id();
  const int warp = threadIdx.x >> 5;
  const int warps = blockDim.x >> 5;
  const long long n = ix.n;
  const int L = ix.L;
  const bool complete = TAL || mode == 1;  // TAL: the complete answer with need = k
  u64* scb = reinterpret_cast<u64*>(smem_raw + 16 + (size_t)ix.smem_entries * 8) +
             warp * (32 * NS);

  if (ix.dcount) count = min(count, *ix.dcount);  // device-resident batch size (lcp_query_counted)
  for (long long qi = (long long)blockIdx.x * warps + warp; qi < count;
       qi += (long long)gridDim.x * warps) {
    u64 qk[WMAX];
    if (!warp_pack_query<WMAX>(queries + qi * L, ix, qk)) {
      if (lane == 0) {
        raise_flag(err);
        out_hits[qi] = 0;
        out_md[qi] = 0;
        out_aux[2 * qi] = 0;
        out_aux[2 * qi + 1] = 0;
      }
      continue;
    }
    TopKN<u64, NS> lst;
    lst.init(scb);
    long long blo = 0, bhi = n;
    unsigned long long tsym = 0;
    if constexpr (TAL) {
      tal_bucket(ix, qk, queries + qi * L, blo, bhi);
      tsym = tal_sym_warp<WMAX>(ix, qk, blo, bhi);
      const long long bs = bhi - blo;
      if (bs < k) {  // the whole bucket, ranked (an empty one included)
        for (long long base = blo; base < bhi; base += 32) {
          const long long i = base + lane;
          lst.offer(i < bhi ? make_comp<u64>(lcp_at<WMAX>(ix, i, qk), __ldg(ix.order + i), L, 32)
                            : ~0ull, k);
        }
#pragma unroll
        for (int j = 0; j < NS; ++j) {
          if (lane + 32 * j < bs) {
            const u64 w = lst.s[j];
            out_ids[(size_t)qi * stride + lane + 32 * j] = (u32)(w & 0xffffffffull);
            out_lcps[(size_t)qi * stride + lane + 32 * j] = (uint16_t)(L - (int)(w >> 32));
          }
        }
        if (lane == 0) {
          out_hits[qi] = (int)bs;
          out_md[qi] = (uint16_t)ix.tal_depth;
          out_aux[2 * qi] = (u64)bs;
          out_aux[2 * qi + 1] = tsym;
        }
        continue;
      }
    }
    const long long pos = warp_lower_bound<WMAX>(ix, staged, qk);
    const long long s = pos - 32 * NS;  // window [s, s + 32 T), warp-strided
    int l[T];
    u32 id[T];
    int dmax = region_lcps<WMAX, T>(ix, s, qk, l, id);
    dmax = (int)__reduce_max_sync(LCP_FULL_MASK, (unsigned)(dmax + 1)) - 1;
    const int need = complete ? (int)min((long long)k, n) : k;
    const int dstar = complete ? window_dstar<T>(l, dmax, need) : dmax;
    int cnt = 0, r0 = 32 * T, above = 0;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const bool c = l[t] >= dstar;
      const unsigned m = __ballot_sync(LCP_FULL_MASK, c);
      cnt += __popc(m);
      above += __popc(__ballot_sync(LCP_FULL_MASK, l[t] > dstar));
      if (m && r0 == 32 * T) r0 = t * 32 + __ffs(m) - 1;
      lst.offer(c ? make_comp<u64>(l[t], id[t], L, 32) : ~0ull, need);
    }
    const long long first_valid = s < 0 ? -s : 0;
    const long long end = min(s + 32 * T, n);
    long long rsize = cnt, rlo = s + r0;
    const u64 tier = make_comp<u64>(dstar, 0u, L, 32);
    const bool sketch_ok = need - above <= LCP_SK_LIST;
    bool goL = s > 0 && r0 == first_valid, goR = end < n && s + r0 + cnt == end;
    long long eL = s, eR = end;
    // d* = 0: the run is the whole corpus, so no chunk can end it
    const int ext_chunks = dstar ? EXT_SCAN_CHUNKS : 0;
    for (int chunk = 0; goL && chunk < ext_chunks; ++chunk) {
      const long long i = eL - 32 + lane;
      const int li = i >= 0 ? lcp_at<WMAX>(ix, i, qk) : -1;
      const bool c = li >= dstar;
      lst.offer(c ? make_comp<u64>(li, __ldg(ix.order + i), L, 32) : ~0ull, need);
      const unsigned m = __ballot_sync(LCP_FULL_MASK, c);
      rsize += __popc(m);
      if (m) rlo = eL - 32 + (__ffs(m) - 1);
      eL -= 32;
      goL = m == LCP_FULL_MASK && eL > 0;
    }
    for (int chunk = 0; goR && chunk < ext_chunks; ++chunk) {
      const long long i = eR + lane;
      const int li = i < n ? lcp_at<WMAX>(ix, i, qk) : -1;
      const bool c = li >= dstar;
      lst.offer(c ? make_comp<u64>(li, __ldg(ix.order + i), L, 32) : ~0ull, need);
      const unsigned m = __ballot_sync(LCP_FULL_MASK, c);
      rsize += __popc(m);
      eR += 32;
      goR = m == LCP_FULL_MASK && eR < n;
    }
    if (goL || goR) {
      const long long rl = goL ? (dstar ? run_edge<WMAX>(ix, qk, dstar, eL, -1) : 0) : eL;
      const long long rr = goR ? (dstar ? run_edge<WMAX>(ix, qk, dstar, eR - 1, n) + 1 : n) : eR;
      const long long rest = (eL - rl) + (rr - eR);
      rsize += rest;
      if (goL) rlo = rl;
      if (sketch_ok) {
        if (goL) lst = tier_offer_n<u64, NS>(ix, rl, eL, tier, lst, need);
        if (goR) lst = tier_offer_n<u64, NS>(ix, eR, rr, tier, lst, need);
      } else if (16 * rest >= n) {
        for (long long base = 0; base < n && (tier | (u64)base) < lst.thr; base += 32) {
          const long long idv = base + lane;
          u64 cv = ~0ull;
          if (idv < n) {
            const long long p = __ldg(ix.rank + idv);
            if ((p >= rl && p < eL) || (p >= eR && p < rr)) cv = tier | (u64)idv;
          }
          lst.offer(cv, need);
        }
      } else {
        for (long long base = rl; base < eL; base += 32) {
          const long long i = base + lane;
          lst.offer(i < eL ? (tier | (u64)__ldg(ix.order + i)) : ~0ull, need);
        }
        for (long long base = eR; base < rr; base += 32) {
          const long long i = base + lane;
          lst.offer(i < rr ? (tier | (u64)__ldg(ix.order + i)) : ~0ull, need);
        }
      }
    }
    const int take = (int)min((long long)need, rsize);
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      if (lane + 32 * j < take) {
        const u64 w = lst.s[j];
        out_ids[(size_t)qi * stride + lane + 32 * j] = (u32)(w & 0xffffffffull);
        out_lcps[(size_t)qi * stride + lane + 32 * j] = (uint16_t)(L - (int)(w >> 32));
      }
    }
    if (lane == 0) {
      out_hits[qi] = take;
      if constexpr (TAL) {
        out_md[qi] = (uint16_t)ix.tal_depth;
        out_aux[2 * qi] = (u64)(bhi - blo);
        out_aux[2 * qi + 1] = tsym;
      } else {
        out_md[qi] = (uint16_t)dmax;
        out_aux[2 * qi] = (u64)(u32)dmax | ((u64)(u32)dstar << 32);
        out_aux[2 * qi + 1] = (u64)rsize | ((u64)rlo << 32);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// General path: any k, any W, all modes + full scan.  One CTA per query;
// the query's range [lo, hi) is emitted as its `take` smallest composites in
// ascending order, in rounds of GEN_CAP (8-pass radix select + smem bitonic
// sort).  Queries are pre-packed by k_pack into qkeys.
// ---------------------------------------------------------------------------
constexpr int GEN_THREADS = 128;
constexpr int GEN_CAP = 2048;

// block-wide AND / OR of per-thread values (all threads call; ends synchronized)
__device__ __forceinline__ void block_and_or(u64& a, u64& o, u64 (*s_red)[2]) {
  const int lane = lane_id(), warp = threadIdx.x >> 5;
#pragma unroll
  for (int s = 16; s; s >>= 1) {
    a &= __shfl_xor_sync(LCP_FULL_MASK, a, s);
    o |= __shfl_xor_sync(LCP_FULL_MASK, o, s);
  }
  if (lane == 0) {
    s_red[warp][0] = a;
    s_red[warp][1] = o;
  }
  __syncthreads();
  a = s_red[0][0];
  o = s_red[0][1];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
    a &= s_red[w][0];
    o |= s_red[w][1];
  }
  __syncthreads();
}

// appends c to dst when pred (one shared atomic per warp); all lanes call
__device__ __forceinline__ void warp_append(bool pred, u64 c, u64* dst, u32* cnt, u32 cap) {
  const unsigned m = __ballot_sync(LCP_FULL_MASK, pred);
  if (!m) return;
  const int lane = lane_id(), leader = __ffs(m) - 1;
  u32 base = 0;
  if (lane == leader) base = atomicAdd(cnt, (u32)__popc(m));
  base = __shfl_sync(LCP_FULL_MASK, base, leader);
  const u32 slot = base + __popc(m & ((1u << lane) - 1u));
  if (pred && slot < cap) dst[slot] = c;
}

// The want-th smallest value among {get(i) : i in [lo, hi), first || get(i) > last},
// by 8-bit digits from the top.  Digits constant over the whole range
// (vdiff = AND ^ OR of its values is zero there) come from vand without a pass;
// histogram updates are aggregated per warp (__match_any_sync), so the few
// distinct digits of the lcp field cost one shared atomic per warp each.
// All threads call; the result is uniform.
template <typename Get>
__device__ __forceinline__ u64 radix_select(const Get& get, long long lo, long long hi, bool first,
                                            u64 last, u32 want, u64 vand, u64 vdiff, u32* hist,
                                            u64* s_prefix, u32* s_rank) {
  const int lane = lane_id();
  u64 prefix = 0, hmask = 0;
  u32 rank = want;
  for (int shift = 56; shift >= 0; shift -= 8) {
    const u64 dmask = 255ull << shift;
    if (!(vdiff & dmask)) {
      prefix |= vand & dmask;
      hmask |= dmask;
      continue;
    }
    for (int t = threadIdx.x; t < 256; t += blockDim.x) hist[t] = 0;
    __syncthreads();
    for (long long b = lo; b < hi; b += blockDim.x) {
      const long long i = b + threadIdx.x;
      u32 dg = 256;
      if (i < hi) {
        const u64 c = get(i);
        if ((first || c > last) && (c & hmask) == prefix) dg = (u32)((c >> shift) & 255);
      }
      const unsigned peers = __match_any_sync(LCP_FULL_MASK, dg);
      if (dg < 256 && lane == __ffs(peers) - 1) atomicAdd(&hist[dg], (u32)__popc(peers));
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // warp 0: the bin holding the rank-th value
      u32 v[8], s = 0;
#pragma unroll
      for (int r = 0; r < 8; ++r) s += (v[r] = hist[lane * 8 + r]);
      u32 inc = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(LCP_FULL_MASK, inc, o);
        if (lane >= o) inc += t;
      }
      u32 cum = inc - s;
      if (cum < rank && inc >= rank) {
        int r = 0;
        for (; r < 7 && cum + v[r] < rank; ++r) cum += v[r];
        *s_prefix = prefix | ((u64)(lane * 8 + r) << shift);
        *s_rank = rank - cum;
      }
    }
    __syncthreads();
    prefix = *s_prefix;
    rank = *s_rank;
    hmask |= dmask;
  }
  __syncthreads();  // s_prefix / s_rank reads done before any reuse
  return prefix;
}

// first index in [0, n) whose d-prefix compares >= q (strict=false) or > q (strict=true)
__device__ __forceinline__ long long prefix_bound(const DevIndex& ix, const u64* q, int d,
                                                  bool upper) {
  long long a = 0, b = ix.n;
  while (a < b) {
    long long m = (a + b) >> 1;
    int c = prefix_cmp(ix.keys + m * ix.W, q, d, ix);
    if (c < 0 || (upper && c == 0)) a = m + 1;
    else b = m;
  }
  return a;
}

// Any-W helpers for the general path: the first word from the sorted
// first-word plane (keys_w0 / levels_w0; the keys / levels themselves when
// W == 1), the rest of the key only when the first words are equal.
__device__ __forceinline__ int lcp_any(const DevIndex& ix, long long i, const u64* q) {
  const u64 x = __ldg(ix.keys_w0 + i) ^ q[0];
  if (x) return __clzll((long long)x) >> ix.lb;
  const u64* key = ix.keys + i * ix.W;
  for (int w = 1; w < ix.W; ++w) {
    const u64 y = key[w] ^ q[w];
    if (y) return w * ix.spw + (__clzll((long long)y) >> ix.lb);
  }
  return ix.L;
}

__device__ __forceinline__ bool less_any(const DevIndex& ix, u64 a0, const u64* key, const u64* q) {
  if (a0 != q[0]) return a0 < q[0];
  for (int w = 1; w < ix.W; ++w)
    if (key[w] != q[w]) return key[w] < q[w];
  return false;
}

// lower_bound(keys, q) for any W by one warp: 64-ary over the global search
// tables (two separators per lane per level), then the 16-key leaf block
__device__ __forceinline__ long long warp_lower_bound_any(const DevIndex& ix, const u64* q) {
  const int lane = lane_id();
  const int W = ix.W;
  long long blk = 0;
  for (int j = 0; j < ix.nlevels; ++j) {
    const u64* tab = ix.levels + ix.level_off[j] * W;
    const long long cnt = ix.level_cnt[j];
    const long long i0 = blk * LCP_SEARCH_FANOUT + 2 * lane;
    const u64* w0 = ix.levels_w0 + ix.level_off[j];
    const bool lt0 = i0 < cnt && less_any(ix, __ldg(w0 + i0), tab + i0 * W, q);
    const bool lt1 = i0 + 1 < cnt && less_any(ix, __ldg(w0 + i0 + 1), tab + (i0 + 1) * W, q);
    const int c = __popc(__ballot_sync(LCP_FULL_MASK, lt0)) + __popc(__ballot_sync(LCP_FULL_MASK, lt1));
    if (c == 0) return 0;  // only at the root: q <= every key
    blk = blk * LCP_SEARCH_FANOUT + c - 1;
  }
  const long long base = blk * LCP_LEAF_KEYS;
  const long long i = base + lane;
  const bool lt = lane < LCP_LEAF_KEYS && i < ix.n && less_any(ix, __ldg(ix.keys_w0 + i), ix.keys + i * W, q);
  return base + __popc(__ballot_sync(LCP_FULL_MASK, lt));
}

// run_edge for any W (see run_edge): last position of {lcp >= d} from `in` toward `out`
__device__ __forceinline__ long long run_edge_any(const DevIndex& ix, const u64* q, int d,
                                                  long long in, long long out) {
  const long long dir = out > in ? 1 : -1;
  for (;;) {
    const long long span = (out - in) * dir;
    if (span <= 1) return in;
    const long long step = (span + 31) >> 5;
    const long long off = step * (lane_id() + 1);
    const bool inside = off < span && lcp_any(ix, in + dir * off, q) >= d;
    const long long c = __popc(__ballot_sync(LCP_FULL_MASK, inside));
    if (step * (c + 1) < span) out = in + dir * step * (c + 1);
    in += dir * step * c;
  }
}

// ---------------------------------------------------------------------------
// strict / complete, k <= 32, W > 8 (long keys): one warp per query like
// k_query_warp, with the packed query read from qkeys (k_pack) instead of
// registers, so any W works: the any-W search, a 64-key window [pos - 32,
// pos + 32), rank selection, extension by chunks and then run_edge_any + the
// id sketch.  Compares read the first-word planes (lcp_any).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(QW_MAX_THREADS, 1)
    k_query_warp_any(const __grid_constant__ DevIndex ix, const u64* __restrict__ qkeys, int count,
                     int k, int mode, int stride, u32* __restrict__ out_ids,
                     uint16_t* __restrict__ out_lcps, int* __restrict__ out_hits,
                     uint16_t* __restrict__ out_md, u64* __restrict__ out_aux) {
  const int lane = lane_id();
  const int warp = threadIdx.x >> 5;
  const int warps = blockDim.x >> 5;
  const long long n = ix.n;
  const int L = ix.L;
  const bool complete = mode == 1;
  if (ix.dcount) count = min(count, *ix.dcount);  // device-resident batch size (lcp_query_counted)
  for (long long qi = (long long)blockIdx.x * warps + warp; qi < count;
       qi += (long long)gridDim.x * warps) {
    const u64* q = qkeys + qi * ix.W;
    const long long pos = warp_lower_bound_any(ix, q);
    const long long s = pos - 32;  // window [s, s + 64), warp-strided
    int l[2];
    u32 id[2];
    int dmax = -1;
    u64 x0[2];  // both rows' first words and ids in flight together (see region_lcps)
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const long long ic = min(max(s + t * 32 + lane, 0ll), n - 1);
      x0[t] = __ldg(ix.keys_w0 + ic) ^ q[0];
      id[t] = __ldg(ix.order + ic);
    }
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const long long i = s + t * 32 + lane;
      const int lv = x0[t] ? (__clzll((long long)x0[t]) >> ix.lb) : lcp_any(ix, min(max(i, 0ll), n - 1), q);
      l[t] = lv | ((i >= 0 && i < n) ? 0 : -1);
      dmax = max(dmax, l[t]);
    }
    dmax = (int)__reduce_max_sync(LCP_FULL_MASK, (unsigned)(dmax + 1)) - 1;
    const int need = complete ? (int)min((long long)k, n) : k;
    const int dstar = complete ? window_dstar<2>(l, dmax, need) : dmax;
    u64 comp[2];
    int cnt = 0, r0 = 64;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const bool c = l[t] >= dstar;
      comp[t] = c ? make_comp<u64>(l[t], id[t], L, 32) : ~0ull;
      const unsigned m = __ballot_sync(LCP_FULL_MASK, c);
      cnt += __popc(m);
      if (m && r0 == 64) r0 = t * 32 + __ffs(m) - 1;
    }
    u64 slot = sort_run<u64, 2>(comp, r0, cnt, need);
    u64 thr = __shfl_sync(LCP_FULL_MASK, slot, need - 1);
    long long rsize = cnt, rlo = s + r0;
    const long long first_valid = s < 0 ? -s : 0;
    const long long end = min(s + 64, n);
    const u64 tier = make_comp<u64>(dstar, 0u, L, 32);
    bool goL = s > 0 && r0 == first_valid, goR = end < n && s + r0 + cnt == end;
    long long eL = s, eR = end;  // [eL, eR) is scanned
    const int ext_chunks = dstar ? EXT_SCAN_CHUNKS : 0;
    for (int chunk = 0; goL && chunk < ext_chunks; ++chunk) {
      const long long i = eL - 32 + lane;
      const int li = i >= 0 ? lcp_any(ix, i, q) : -1;
      const bool c = li >= dstar;
      warp_offer(slot, thr, c ? make_comp<u64>(li, __ldg(ix.order + i), L, 32) : ~0ull, need);
      const unsigned m = __ballot_sync(LCP_FULL_MASK, c);
      rsize += __popc(m);
      if (m) rlo = eL - 32 + (__ffs(m) - 1);
      eL -= 32;
      goL = m == LCP_FULL_MASK && eL > 0;
    }
    for (int chunk = 0; goR && chunk < ext_chunks; ++chunk) {
      const long long i = eR + lane;
      const int li = i < n ? lcp_any(ix, i, q) : -1;
      const bool c = li >= dstar;
      warp_offer(slot, thr, c ? make_comp<u64>(li, __ldg(ix.order + i), L, 32) : ~0ull, need);
      const unsigned m = __ballot_sync(LCP_FULL_MASK, c);
      rsize += __popc(m);
      eR += 32;
      goR = m == LCP_FULL_MASK && eR < n;
    }
    if (goL || goR) {  // past the scanned span every item has lcp == d*: the id sketch
      const long long rl = goL ? (dstar ? run_edge_any(ix, q, dstar, eL, -1) : 0) : eL;
      const long long rr = goR ? (dstar ? run_edge_any(ix, q, dstar, eR - 1, n) + 1 : n) : eR;
      rsize += (eL - rl) + (rr - eR);
      if (goL) {
        rlo = rl;
        slot = tier_offer<u64>(ix, rl, eL, tier, slot, need);
      }
      if (goR) slot = tier_offer<u64>(ix, eR, rr, tier, slot, need);
    }
    const int take = (int)min((long long)need, rsize);
    write_result<u64>(qi, stride, take, L, slot, 32, dmax, dstar, rsize, rlo, out_ids, out_lcps,
                      out_hits, out_md, out_aux);
  }
}

// ---------------------------------------------------------------------------
// strict / complete, 32 < need <= 32 * NS <= 128, W > 8: k_query_warp_kn on
// the packed-query buffer with the any-W helpers (see k_query_warp_any).
// ---------------------------------------------------------------------------
template <int NS>
__global__ void __launch_bounds__(NS > 2 ? QW_MAX_THREADS / 2 : QW_MAX_THREADS, 1)
    k_query_warp_any_kn(const __grid_constant__ DevIndex ix, const u64* __restrict__ qkeys,
                        int count, int k, int mode, int stride, u32* __restrict__ out_ids,
                        uint16_t* __restrict__ out_lcps, int* __restrict__ out_hits,
                        uint16_t* __restrict__ out_md, u64* __restrict__ out_aux) {
  constexpr int T = 2 * NS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = lane_id();
  const int warp = threadIdx.x >> 5;
  const int warps = blockDim.x >> 5;
  const long long n = ix.n;
  const int L = ix.L;
  const bool complete = mode == 1;
  u64* scb = reinterpret_cast<u64*>(smem_raw) + warp * (32 * NS);
  if (ix.dcount) count = min(count, *ix.dcount);  // device-resident batch size (lcp_query_counted)
  for (long long qi = (long long)blockIdx.x * warps + warp; qi < count;
       qi += (long long)gridDim.x * warps) {
    const u64* q = qkeys + qi * ix.W;
    const long long pos = warp_lower_bound_any(ix, q);
    const long long s = pos - 32 * NS;
    int l[T];
    u32 id[T];
    int dmax = -1;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const long long i = s + t * 32 + lane;
      const bool ok = i >= 0 && i < n;
      l[t] = ok ? lcp_any(ix, i, q) : -1;
      id[t] = ok ? __ldg(ix.order + i) : 0u;
      dmax = max(dmax, l[t]);
    }
    dmax = (int)__reduce_max_sync(LCP_FULL_MASK, (unsigned)(dmax + 1)) - 1;
    const int need = complete ? (int)min((long long)k, n) : k;
    const int dstar = complete ? window_dstar<T>(l, dmax, need) : dmax;
    TopKN<u64, NS> lst;
    lst.init(scb);
    int cnt = 0, r0 = 32 * T, above = 0;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const bool c = l[t] >= dstar;
      const unsigned m = __ballot_sync(LCP_FULL_MASK, c);
      cnt += __popc(m);
      above += __popc(__ballot_sync(LCP_FULL_MASK, l[t] > dstar));
      if (m && r0 == 32 * T) r0 = t * 32 + __ffs(m) - 1;
      lst.offer(c ? make_comp<u64>(l[t], id[t], L, 32) : ~0ull, need);
    }
    const long long first_valid = s < 0 ? -s : 0;
    const long long end = min(s + 32 * T, n);
    long long rsize = cnt, rlo = s + r0;
    const u64 tier = make_comp<u64>(dstar, 0u, L, 32);
    const bool sketch_ok = need - above <= LCP_SK_LIST;
    bool goL = s > 0 && r0 == first_valid, goR = end < n && s + r0 + cnt == end;
    long long eL = s, eR = end;
    const int ext_chunks = dstar ? EXT_SCAN_CHUNKS : 0;
    for (int chunk = 0; goL && chunk < ext_chunks; ++chunk) {
      const long long i = eL - 32 + lane;
      const int li = i >= 0 ? lcp_any(ix, i, q) : -1;
      const bool c = li >= dstar;
      lst.offer(c ? make_comp<u64>(li, __ldg(ix.order + i), L, 32) : ~0ull, need);
      const unsigned m = __ballot_sync(LCP_FULL_MASK, c);
      rsize += __popc(m);
      if (m) rlo = eL - 32 + (__ffs(m) - 1);
      eL -= 32;
      goL = m == LCP_FULL_MASK && eL > 0;
    }
    for (int chunk = 0; goR && chunk < ext_chunks; ++chunk) {
      const long long i = eR + lane;
      const int li = i < n ? lcp_any(ix, i, q) : -1;
      const bool c = li >= dstar;
      lst.offer(c ? make_comp<u64>(li, __ldg(ix.order + i), L, 32) : ~0ull, need);
      const unsigned m = __ballot_sync(LCP_FULL_MASK, c);
      rsize += __popc(m);
      eR += 32;
      goR = m == LCP_FULL_MASK && eR < n;
    }
    if (goL || goR) {
      const long long rl = goL ? (dstar ? run_edge_any(ix, q, dstar, eL, -1) : 0) : eL;
      const long long rr = goR ? (dstar ? run_edge_any(ix, q, dstar, eR - 1, n) + 1 : n) : eR;
      const long long rest = (eL - rl) + (rr - eR);
      rsize += rest;
      if (goL) rlo = rl;
      if (sketch_ok) {
        if (goL) lst = tier_offer_n<u64, NS>(ix, rl, eL, tier, lst, need);
        if (goR) lst = tier_offer_n<u64, NS>(ix, eR, rr, tier, lst, need);
      } else if (16 * rest >= n) {
        for (long long base = 0; base < n && (tier | (u64)base) < lst.thr; base += 32) {
          const long long idv = base + lane;
          u64 cv = ~0ull;
          if (idv < n) {
            const long long p = __ldg(ix.rank + idv);
            if ((p >= rl && p < eL) || (p >= eR && p < rr)) cv = tier | (u64)idv;
          }
          lst.offer(cv, need);
        }
      } else {
        for (long long base = rl; base < eL; base += 32) {
          const long long i = base + lane;
          lst.offer(i < eL ? (tier | (u64)__ldg(ix.order + i)) : ~0ull, need);
        }
        for (long long base = eR; base < rr; base += 32) {
          const long long i = base + lane;
          lst.offer(i < rr ? (tier | (u64)__ldg(ix.order + i)) : ~0ull, need);
        }
      }
    }
    const int take = (int)min((long long)need, rsize);
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      if (lane + 32 * j < take) {
        const u64 w = lst.s[j];
        out_ids[(size_t)qi * stride + lane + 32 * j] = (u32)(w & 0xffffffffull);
        out_lcps[(size_t)qi * stride + lane + 32 * j] = (uint16_t)(L - (int)(w >> 32));
      }
    }
    if (lane == 0) {
      out_hits[qi] = take;
      out_md[qi] = (uint16_t)dmax;
      out_aux[2 * qi] = (u64)(u32)dmax | ((u64)(u32)dstar << 32);
      out_aux[2 * qi + 1] = (u64)rsize | ((u64)rlo << 32);
    }
  }
}

struct GenItem {
  const DevIndex* ix;
  const u64* q;
  bool fullscan;
  __device__ __forceinline__ u64 comp(long long i, int* lcp_out) const {
    int l = fullscan ? key_lcp<0>(ix->keys_orig + i * ix->W, q, *ix) : lcp_any(*ix, i, q);
    *lcp_out = l;
    u32 id = fullscan ? (u32)i : ix->order[i];
    return make_composite(l, id, ix->L);
  }
};

__global__ void __launch_bounds__(GEN_THREADS)
    k_query_general(DevIndex ix, const u64* __restrict__ qkeys, const uint16_t* __restrict__ queries,
                    int count, int k, int mode, int fullscan, int stride,
                    u32* __restrict__ out_ids, uint16_t* __restrict__ out_lcps,
                    int* __restrict__ out_hits, uint16_t* __restrict__ out_md,
                    u64* __restrict__ out_aux) {
  __shared__ u64 buf[GEN_CAP];
  __shared__ u32 hist[256];
  __shared__ long long s_lo, s_hi, s_take;
  __shared__ int s_dmax, s_dstar, s_md;
  __shared__ u32 s_cnt;
  __shared__ u64 s_prefix;
  __shared__ u32 s_rank;
  __shared__ unsigned long long s_sym;
  __shared__ long long s_pos;
  __shared__ long long s_p0;    // a position with lcp = d_max (strict / complete)
  __shared__ long long s_a, s_b;  // R(d* + 1) for the split selection
  __shared__ int s_wc[GEN_THREADS / 32];
  __shared__ long long s_part[GEN_THREADS / 32][2];
  __shared__ u64 s_red[GEN_THREADS / 32][2];
  const int L = ix.L;
  const int lane = lane_id(), warp = threadIdx.x >> 5;

  if (ix.dcount) count = min(count, *ix.dcount);  // device-resident batch size (lcp_query_counted)
  for (long long qi = blockIdx.x; qi < count; qi += gridDim.x) {
    const u64* q = qkeys + qi * ix.W;
    // strict / complete with need <= GEN_CAP / 2: CTA-cooperative setup.
    // pos by warp 0's 64-ary search; d* from the window [pos - need,
    // pos + need) (R(d*+1) lies inside it); R(d*) from the window, extended by
    // run_edge_any when the run reaches a window edge.
    if (!fullscan && mode != 2 && ix.n > 0 && (long long)k <= GEN_CAP / 2) {
      if (warp == 0) {
        const long long pos = warp_lower_bound_any(ix, q);
        if (lane == 0) s_pos = pos;
      }
      __syncthreads();
      const long long pos = s_pos;
      const long long need = mode == 1 ? min((long long)k, ix.n) : (long long)k;
      const long long wlo = max(0ll, pos - need), whi = min(ix.n, pos + need);
      const int wn = (int)(whi - wlo);
      int* wl = reinterpret_cast<int*>(buf);  // window lcps (<= GEN_CAP ints)
      int mymax = -1;
      for (int i = threadIdx.x; i < wn; i += GEN_THREADS) {
        const int l = lcp_any(ix, wlo + i, q);
        wl[i] = l;
        mymax = max(mymax, l);
      }
      auto block_pair = [&](long long a, long long b, bool is_min) {
        // block-wide (min|max, max) of per-thread pairs via s_part
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const long long oa = __shfl_xor_sync(LCP_FULL_MASK, a, o);
          a = is_min ? min(a, oa) : a + oa;
          b = max(b, __shfl_xor_sync(LCP_FULL_MASK, b, o));
        }
        if (lane == 0) {
          s_part[warp][0] = a;
          s_part[warp][1] = b;
        }
        __syncthreads();
        long long ra = s_part[0][0], rb = s_part[0][1];
        for (int w = 1; w < GEN_THREADS / 32; ++w) {
          ra = is_min ? min(ra, s_part[w][0]) : ra + s_part[w][0];
          rb = max(rb, s_part[w][1]);
        }
        __syncthreads();
        return make_longlong2(ra, rb);
      };
      const int dmax = (int)block_pair(0, mymax, false).y;
      int dstar = dmax;
      if (mode == 1) {
        int dl = 0, dh = dmax;
        while (dl < dh) {
          const int mid = (dl + dh + 1) >> 1;
          long long c = 0;
          for (int i = threadIdx.x; i < wn; i += GEN_THREADS) c += wl[i] >= mid;
          if (block_pair(c, 0, false).x >= need) dl = mid;
          else dh = mid - 1;
        }
        dstar = dl;
      }
      long long first = LLONG_MAX, last = -1;
      for (int i = threadIdx.x; i < wn; i += GEN_THREADS)
        if (wl[i] >= dstar) {
          first = min(first, (long long)i);
          last = max(last, (long long)i);
        }
      const longlong2 fl = block_pair(first, last, true);
      long long lo = wlo + fl.x, hi = wlo + fl.y + 1;
      if (warp == 0) {
        if (lo == wlo && wlo > 0) lo = dstar ? run_edge_any(ix, q, dstar, lo, -1) : 0;
        if (hi == whi && whi < ix.n) hi = dstar ? run_edge_any(ix, q, dstar, hi - 1, ix.n) + 1 : ix.n;
        if (lane == 0) {
          s_lo = lo;
          s_hi = hi;
          s_take = mode == 1 ? need : min((long long)k, hi - lo);
          s_dmax = dmax;
          s_dstar = dstar;
          s_md = dmax;
          s_sym = 0;
          s_p0 = pos < ix.n && wl[pos - wlo] == dmax ? pos : pos - 1;
        }
      }
    } else if (!fullscan && mode != 2 && ix.n > 0) {
      // need beyond the window: warp 0 finds R(d) for any d by run_edge_any on
      // both sides of the deepest match p0, and d* by binary search over depths
      if (warp == 0) {
        const long long pos = warp_lower_bound_any(ix, q);
        const int lp = pos > 0 ? lcp_any(ix, pos - 1, q) : -1;
        const int lq = pos < ix.n ? lcp_any(ix, pos, q) : -1;
        const int dmax = max(lp, lq);
        const long long p0 = lq == dmax ? pos : pos - 1;
        auto range = [&](int d, long long& a, long long& b) {
          a = d ? run_edge_any(ix, q, d, p0, -1) : 0;
          b = d ? run_edge_any(ix, q, d, p0, ix.n) + 1 : ix.n;
        };
        long long lo, hi;
        int dstar = dmax;
        range(dmax, lo, hi);
        const long long need = mode == 1 ? min((long long)k, ix.n) : (long long)k;
        if (mode == 1 && hi - lo < need) {
          int dl = 0, dh = dmax - 1;  // |R(0)| = n >= need
          while (dl < dh) {
            const int mid = (dl + dh + 1) >> 1;
            long long a, b;
            range(mid, a, b);
            if (b - a >= need) dl = mid;
            else dh = mid - 1;
          }
          dstar = dl;
          range(dstar, lo, hi);
        }
        if (lane == 0) {
          s_lo = lo;
          s_hi = hi;
          s_take = mode == 1 ? need : min((long long)k, hi - lo);
          s_dmax = dmax;
          s_dstar = dstar;
          s_md = dmax;
          s_sym = 0;
          s_p0 = p0;
        }
      }
    } else if (threadIdx.x == 0) {
      long long lo = 0, hi = ix.n, take = 0;
      int dmax = 0, dstar = 0, md = 0;
      if (fullscan) {
        take = min((long long)k, ix.n);
      } else if (mode == 2) {
        tal_bucket(ix, q, queries + qi * L, lo, hi);
        take = min((long long)k, hi - lo);
        md = ix.tal_depth;
      } else {
        hi = 0;  // strict / complete over an empty index
      }
      s_lo = lo;
      s_hi = hi;
      s_take = take;
      s_dmax = dmax;
      s_dstar = dstar;
      s_md = md;
      s_sym = 0;
    }
    __syncthreads();
    const long long lo = s_lo, hi = s_hi, take = s_take;
    const long long size = hi - lo;
    GenItem it{&ix, q, fullscan != 0};
    unsigned long long sym = 0;
    u64 vand = ~0ull, vor = 0;
    auto emit = [&](const u64* src, long long at, int n) {
      for (int t = threadIdx.x; t < n; t += GEN_THREADS) {
        const u64 c = src[t];
        out_ids[qi * stride + at + t] = (u32)(c & 0xffffffffull);
        out_lcps[qi * stride + at + t] = (uint16_t)(L - (int)(c >> 32));
      }
    };
    // the take smallest composites of sorted positions (full scan: original
    // rows) [lo, hi), ascending, written from output slot `at`
    // the take smallest composites of sorted positions (full scan: original
    // rows) [lo, hi), ascending, written from output slot `at`
    auto select_range = [&](const long long lo, const long long hi, const long long take,
                            const long long at) {
      const long long size = hi - lo;
      if (size <= GEN_CAP) {
        int P = 1, Pt = 1;
        while (P < size) P <<= 1;
        while (Pt < take) Pt <<= 1;
        constexpr int PER = GEN_CAP / GEN_THREADS;
        u64 v[PER];
  #pragma unroll
        for (int r = 0; r < PER; ++r) {
          const int t = threadIdx.x + r * GEN_THREADS;
          v[r] = ~0ull;
          if (t < size) {
            int l;
            v[r] = it.comp(lo + t, &l);
            sym += (unsigned long long)min(l + 1, L);
            vand &= v[r];
            vor |= v[r];
          }
          if (t < P) buf[t] = v[r];
        }
        if (take > 0 && 2 * Pt <= P) {
          // select, then sort only the take smallest (a power of two at least
          // half as large): threshold by radix select over the staged values,
          // compaction through registers back into buf
          block_and_or(vand, vor, s_red);
          const u64 T = radix_select([&](long long i) { return buf[i]; }, 0, size, true, 0ull,
                                     (u32)take, vand, vand ^ vor, hist, &s_prefix, &s_rank);
          if (threadIdx.x == 0) s_cnt = 0;
          __syncthreads();
  #pragma unroll
          for (int r = 0; r < PER; ++r) warp_append(v[r] <= T, v[r], buf, &s_cnt, (u32)Pt);
          __syncthreads();
          for (int t = (int)take + threadIdx.x; t < Pt; t += GEN_THREADS) buf[t] = ~0ull;
          P = Pt;
        }
        __syncthreads();
        bitonic_sort_smem(buf, P);
        emit(buf, at, (int)take);
      } else {
        // one pass for symbols_compared and the value span, then rounds of
        // GEN_CAP: radix select of the round's last value, collect (last, T], sort
        for (long long i = lo + threadIdx.x; i < hi; i += GEN_THREADS) {
          int l;
          const u64 c = it.comp(i, &l);
          sym += (unsigned long long)min(l + 1, L);
          vand &= c;
          vor |= c;
        }
        block_and_or(vand, vor, s_red);
        long long emitted = 0;
        u64 last = 0;
        bool first = true;
        auto get = [&](long long i) {
          int l;
          return it.comp(i, &l);
        };
        while (emitted < take) {
          const u32 want = (u32)min((long long)GEN_CAP, take - emitted);
          const u64 T = radix_select(get, lo, hi, first, last, want, vand, vand ^ vor, hist,
                                     &s_prefix, &s_rank);
          if (threadIdx.x == 0) s_cnt = 0;
          __syncthreads();
          for (long long b = lo; b < hi; b += GEN_THREADS) {
            const long long i = b + threadIdx.x;
            u64 c = 0;
            bool in = false;
            if (i < hi) {
              c = get(i);
              in = (first || c > last) && c <= T;
            }
            warp_append(in, c, buf, &s_cnt, GEN_CAP);
          }
          __syncthreads();
          int P = 1;
          while (P < (int)want) P <<= 1;
          for (int t = (int)want + threadIdx.x; t < P; t += GEN_THREADS) buf[t] = ~0ull;
          __syncthreads();
          bitonic_sort_smem(buf, P);
          emit(buf, at + emitted, (int)want);
          __syncthreads();
          last = T;
          first = false;
          emitted += want;
        }
      }
    };
    // Strict / complete over a range beyond GEN_CAP whose lcp = d* tier
    // (R(d*) minus R(d*+1)) covers at least n/16 items, e.g. d* = 0: sorted
    // R(d*+1) (fewer than need items), then the tier's m smallest ids taken in
    // id order through rank[] (about n / |tier| <= 16 probes per id taken),
    // which is already the output order.  (A sparse tier stays on the plain
    // selection: routing it through an id-only selection too cost 7 -> 5
    // resident CTAs per SM, a net loss.)
    bool split = false;
    if (!fullscan && mode != 2 && size > GEN_CAP) {
      if (warp == 0) {
        long long a = lo, b = lo;  // R(d* + 1), empty when d* = d_max
        const int d1 = s_dstar + 1;
        if (d1 <= s_dmax) {
          a = run_edge_any(ix, q, d1, s_p0, -1);
          b = run_edge_any(ix, q, d1, s_p0, ix.n) + 1;
        }
        if (lane == 0) {
          s_a = a;
          s_b = b;
        }
      }
      __syncthreads();
      split = 16 * (size - (s_b - s_a)) >= ix.n;
    }
    if (split) {
      const long long sa = s_a, sb = s_b, c1 = sb - sa, m = take - c1;
      select_range(sa, sb, c1, 0);
      const uint16_t dl = (uint16_t)s_dstar;
      long long got = 0;
      for (long long base = 0; got < m && base < ix.n; base += GEN_THREADS) {
        const long long id = base + threadIdx.x;
        bool in = false;
        if (id < ix.n) {
          const long long p = __ldg(ix.rank + id);
          in = p >= lo && p < hi && (p < sa || p >= sb);
        }
        const unsigned bal = __ballot_sync(LCP_FULL_MASK, in);
        if (lane == 0) s_wc[warp] = __popc(bal);
        __syncthreads();
        long long slot = got + __popc(bal & ((1u << lane) - 1u));
        int tot = 0;
        for (int w = 0; w < GEN_THREADS / 32; ++w) {
          if (w < warp) slot += s_wc[w];
          tot += s_wc[w];
        }
        if (in && slot < m) {
          out_ids[qi * stride + c1 + slot] = (u32)id;
          out_lcps[qi * stride + c1 + slot] = dl;
        }
        got += tot;
        __syncthreads();
      }
    } else {
      select_range(lo, hi, take, 0);
    }
    // reduce symbols_compared (TAL accounting)
#pragma unroll
    for (int o = 16; o; o >>= 1) sym += __shfl_xor_sync(LCP_FULL_MASK, sym, o);
    if ((threadIdx.x & 31) == 0 && sym) atomicAdd(&s_sym, sym);
    __syncthreads();
    if (threadIdx.x == 0) {
      out_hits[qi] = (int)take;
      if (!fullscan) {
        out_md[qi] = (uint16_t)s_md;
        if (mode == 2) {
          out_aux[2 * qi] = (u64)size;
          out_aux[2 * qi + 1] = s_sym;
        } else {
          out_aux[2 * qi] = (u64)(u32)s_dmax | ((u64)(u32)s_dstar << 32);
          out_aux[2 * qi + 1] = (u64)size | ((u64)lo << 32);
        }
      }
    }
    __syncthreads();
  }
}
