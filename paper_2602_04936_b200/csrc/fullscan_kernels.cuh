// fullscan_kernels.cuh — brute-force streaming scan + candidate merges.
//
// Replaces oracle._lcp_profile + oracle.oracle_top_k (oracle.py:38-59): every
// item, in original row order, against every query; top-min(k,n) by
// (lcp desc, id asc).
//
// Layout: one thread owns one query (packed key in registers and a private
// sorted top-k list); a CTA of FS_THREADS queries streams a chunk of the
// packed keys through shared memory in 16 KB stages (TMA bulk copies,
// double-buffered on mbarriers), so each key read from HBM/L2 is broadcast
// to FS_THREADS queries.  Keys arrive in ascending id order, so a key only
// enters a full list if its lcp strictly beats the list's worst lcp: for
// W == 1 that test is one 64-bit compare  (key ^ q) <= limm1.
// Per-(query, chunk) lists go to scratch and are merged by k_merge (take <=
// 32) or k_merge_sort (lists of up to FS_KMAX_* entries, chunks * take <= 8192).
#pragma once

#include "common.cuh"

constexpr int FS_THREADS = 256;
constexpr int FS_KMAX_U32 = 128;  // register list capacity, 32-bit composites
constexpr int FS_KMAX_U64 = 64;   // 64-bit composites
constexpr int FS1_STAGE_KEYS = 2048;  // keys per shared-memory stage (hi + lo planes: 16 KB)

template <int KCAP>
__device__ __forceinline__ void list_insert(u64 (&list)[KCAP], u64 c) {
#pragma unroll
  for (int i = KCAP - 1; i > 0; --i) {
    u64 prev = list[i - 1];
    list[i] = (c < prev) ? prev : ((c < list[i]) ? c : list[i]);
  }
  list[0] = c < list[0] ? c : list[0];
}

template <int KCAP>
__device__ __forceinline__ u64 list_get(const u64 (&list)[KCAP], int idx) {
  u64 v = ~0ull;
#pragma unroll
  for (int i = 0; i < KCAP; ++i)
    if (i == idx) v = list[i];
  return v;
}

template <typename C, int KCAP>
__device__ __forceinline__ void list_insert_mm(C (&list)[KCAP], C c) {
#pragma unroll
  for (int i = KCAP - 1; i > 0; --i) list[i] = cmax(list[i - 1], cmin(list[i], c));
  list[0] = cmin(list[0], c);
}

template <typename C, int KCAP>
__device__ __forceinline__ C list_at(const C (&list)[KCAP], int idx) {
  if (idx == KCAP - 1) return list[KCAP - 1];
  C v = ~C(0);
#pragma unroll
  for (int i = 0; i < KCAP; ++i)
    if (i == idx) v = list[i];
  return v;
}

template <typename C, int KCAP>
__global__ void __launch_bounds__(FS_THREADS)
    k_fullscan_w1(DevIndex ix, const uint16_t* __restrict__ queries, const u64* __restrict__ qkeys,
                  int count, int need, long long chunk, int nchunks, u64* __restrict__ partial,
                  int* __restrict__ hint, int* __restrict__ err) {
  // Any W: the filter and the first-word lcp run on the hi / lo planes of each
  // key's first word; only keys equal to q in the whole first word (lcp >= spw)
  // read their remaining words (keys_orig) against the packed query (qkeys).
  extern __shared__ __align__(16) unsigned char smem_raw[];
  u64* bars = reinterpret_cast<u64*>(smem_raw);
  u32* stage = reinterpret_cast<u32*>(smem_raw + 16);  // [2][hi | lo] x FS1_STAGE_KEYS
  const int L = ix.L;
  const int idbits = sizeof(C) == 8 ? 32 : ix.idbits;
  const long long n = ix.n;
  const long long qi = (long long)blockIdx.x * FS_THREADS + threadIdx.x;
  const bool active = qi < count;

  // the batch was packed by the streaming pack kernel (coalesced row reads,
  // symbol check): one 8-byte load per query here
  const u64 q0 = active ? qkeys[qi * ix.W] : 0ull;
  const u32 qh = (u32)(q0 >> 32), ql = (u32)q0;
  const int W = ix.W;

  C list[KCAP];
#pragma unroll
  for (int i = 0; i < KCAP; ++i) list[i] = ~C(0);
  int filled = 0;
  C thr = ~C(0);      // list[need-1] once full
  int a_own = 0;      // own bound: worst kept lcp + 1 once full
  int a = 0;          // effective bound max(a_own, hint)
  u64 limm1 = ~0ull;  // survive iff (key ^ q) <= limm1  <=>  lcp >= a
  u32 lim_hi = ~0u;
  bool done = !active;
  int* my_hint = active ? hint + qi : nullptr;

  auto set_bound = [&](int na) {
    a = na;
    if (a > L) {
      done = true;
      return;
    }
    const int bits = a * ix.b;
    limm1 = bits >= 64 ? 0ull : (~0ull >> bits);
    lim_hi = (u32)(limm1 >> 32);
  };

  const long long c0 = (long long)blockIdx.y * chunk;
  const long long c1 = min(n, c0 + chunk);
  const long long nst = c1 > c0 ? (c1 - c0 + FS1_STAGE_KEYS - 1) / FS1_STAGE_KEYS : 0;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](long long s) {
    const long long base = c0 + s * FS1_STAGE_KEYS;
    const long long rows = min((long long)FS1_STAGE_KEYS, c1 - base);
    const u32 bytes = (u32)(((rows * 4) + 15) & ~15ll);
    u32* dst = stage + (s & 1) * (2 * FS1_STAGE_KEYS);
    mbar_arrive_expect_tx(&bars[s & 1], 2 * bytes);
    bulk_g2s(dst, ix.keys_hi + base, bytes, &bars[s & 1]);
    bulk_g2s(dst + FS1_STAGE_KEYS, ix.keys_lo + base, bytes, &bars[s & 1]);
  };
  if (threadIdx.x == 0) {
    if (nst > 0) issue(0);
    if (nst > 1) issue(1);
  }

  for (long long s = 0; s < nst; ++s) {
    if (!done) {
      const int g = *(volatile int*)my_hint;  // other chunks' bound for this query
      if (g > a) set_bound(g);
    }
    mbar_wait(&bars[s & 1], (u32)((s >> 1) & 1));
    const u32* hb = stage + (s & 1) * (2 * FS1_STAGE_KEYS);
    const u32* lb = hb + FS1_STAGE_KEYS;
    const long long base = c0 + s * FS1_STAGE_KEYS;
    const int rows = (int)min((long long)FS1_STAGE_KEYS, c1 - base);
    auto offer = [&](int r) {
      const u64 x = ((u64)(hb[r] ^ qh) << 32) | (u64)(lb[r] ^ ql);
      if (x > limm1) return;
      int l = x ? (__clzll((long long)x) >> ix.lb) : L;
      if (!x && W > 1) {  // first word equal: finish on the remaining words
        const u64* key = ix.keys_orig + (base + r) * W;
        const u64* qk = qkeys + qi * W;
        l = L;
        for (int w = 1; w < W; ++w) {
          const u64 y = key[w] ^ qk[w];
          if (y) {
            l = w * ix.spw + (__clzll((long long)y) >> ix.lb);
            break;
          }
        }
        if (l < a) return;
      }
      const C c = make_comp<C>(l, (u32)(base + r), L, idbits);
      if (c >= thr) return;
      list_insert_mm<C, KCAP>(list, c);
      if (++filled >= need) {
        thr = list_at<C, KCAP>(list, need - 1);
        const int t = L - (int)(widen_comp<C>(thr, idbits) >> 32);  // worst kept lcp
        if (t + 1 > a_own) {
          a_own = t + 1;
          atomicMax(my_hint, t);
        }
        if (a_own > a) set_bound(a_own);
      }
    };
    if (!done) {
      int r = 0;
      for (; r + 15 < rows; r += 16) {
        u32 x[16];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const uint4 h = *reinterpret_cast<const uint4*>(hb + r + 4 * v);
          x[4 * v + 0] = h.x ^ qh;
          x[4 * v + 1] = h.y ^ qh;
          x[4 * v + 2] = h.z ^ qh;
          x[4 * v + 3] = h.w ^ qh;
        }
        const u32 m0 = min(min(min(x[0], x[1]), min(x[2], x[3])),
                           min(min(x[4], x[5]), min(x[6], x[7])));
        const u32 m1 = min(min(min(x[8], x[9]), min(x[10], x[11])),
                           min(min(x[12], x[13]), min(x[14], x[15])));
        if (min(m0, m1) <= lim_hi) {  // rare once the bound has tightened
          u32 live = 0;
#pragma unroll
          for (int e = 0; e < 16; ++e) live |= (u32)(x[e] <= lim_hi) << e;
          while (live && !done) {
            const int e = __ffs(live) - 1;
            live &= live - 1;
            offer(r + e);
          }
          if (done) break;
        }
      }
      for (; r < rows && !done; ++r)
        if ((hb[r] ^ qh) <= lim_hi) offer(r);
    }
    __syncthreads();  // everyone done with this buffer
    if (threadIdx.x == 0 && s + 2 < nst) issue(s + 2);
  }

  // chunk-major, query-fastest layout: adjacent threads store adjacent words
  if (active) {
    u64* out = partial + (long long)blockIdx.y * need * count + qi;
#pragma unroll
    for (int j = 0; j < KCAP; ++j)
      if (j < need) out[(long long)j * count] = widen_comp<C>(list[j], idbits);
  }
}

// ---------------------------------------------------------------------------
// Small query batches (count <= FSQ_QMAX, need <= 32): HBM-streaming scan.
//
// With a handful of queries the corpus pass is bandwidth-, not issue-bound
// (~2 lane instructions per (key, query) against 4 B per key), so the layout
// flips: every lane holds ALL the batch's query words, one CTA per SM of 16
// warps streams the hi plane of the keys' first words with 16-byte
// `ld.global.nc` loads (4 keys per load, FSQ_UNROLL loads in flight per lane),
// each warp over its own contiguous id segment.  Per (key, query) the fast
// path is xor + min on the hi word against the query's bound; the lo word
// (and further words for W > 1) is read only for the rare survivors, whose
// exact composites go into a warp top-k list.  Bounds tighten from the warp's
// own full list (worst kept lcp + 1: ids only grow along a segment) and from a
// per-query global hint (atomicMax of every full list's worst kept lcp).
// Each CTA tree-merges its warps' lists in shared memory; the last CTA to
// finish merges the CTAs' lists with all its warps, writes the outputs and
// resets the hint / counter, so one launch is the whole query.
// Replaces oracle._lcp_profile + oracle_top_k (oracle.py:38-59) for the
// single-query / small-batch calls of the reference API.
// ---------------------------------------------------------------------------
constexpr int FSQ_THREADS = 512;
constexpr int FSQ_WARPS = FSQ_THREADS / 32;
constexpr int FSQ_QMAX = 8;
constexpr int FSQ_STEP = 1024;  // segment granularity (keys); >= one warp step for every Q
constexpr int FSQ_SEG_MIN = 4096;  // keys per warp at least (small corpora: fewer CTAs)
constexpr int FSQ_SEED_STEPS = 1;  // 256-key seed sub-steps (4 measured slower: 30 -> 37 us at 2M, Q=1)
// 16-byte hi-plane loads per lane per step: fewer with more queries (registers)
template <int Q>
__host__ __device__ constexpr int fsq_unroll() { return Q <= 2 ? 8 : (Q <= 4 ? 4 : 2); }
// resident CTAs per SM (one query fits 64 registers: two CTAs, 32 warps)
template <int Q>
__host__ __device__ constexpr int fsq_ctas_per_sm() { return Q == 1 ? 2 : 1; }

// merge the sorted 32-slot warp lists buf[0..n) (one per 32 entries) into
// buf[0]: a tree over the CTA's warps, `groups` independent trees side by side
// (tree g: lists g*n .. g*n+n-1); all threads of the CTA call it
template <typename C>
__device__ void cta_tree_merge(C* buf, int n, int groups) {
  const int lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int half = (n + 1) >> 1, width = n; width > 1; width = half, half = (half + 1) >> 1) {
    const int pairs = width - half;  // list i < pairs absorbs list i + half
    for (int t = warp; t < pairs * groups; t += nw) {
      const int g = t / pairs, i = t - g * pairs;
      C* dst = buf + (g * n + i) * 32;
      const C* src = buf + (g * n + i + half) * 32;
      dst[lane] = warp_merge32(dst[lane], src[lane]);
    }
    __syncthreads();
  }
}

// exact composite of key i against query q (first word from the hi / lo
// planes, further words for W > 1), or all-ones if its lcp is below the bound
template <typename C>
__device__ __noinline__ C fsq_candidate(const u32* __restrict__ keys_hi, const u32* __restrict__ keys_lo,
                                        const u64* __restrict__ keys_orig, int spw,
                                        const u64* __restrict__ qkeys, int q, u32 qh, u32 ql, int a,
                                        long long i, int L, int W, int lb, int idbits) {
  const u64 x = ((u64)(__ldg(keys_hi + i) ^ qh) << 32) | (u64)(__ldg(keys_lo + i) ^ ql);
  int l = x ? (__clzll((long long)x) >> lb) : L;
  if (!x && W > 1) {  // first word equal: finish on the remaining words
    const u64* key = keys_orig + i * W;
    const u64* qk = qkeys + (long long)q * W;
    for (int w = 1; w < W; ++w) {
      const u64 y = key[w] ^ qk[w];
      if (y) {
        l = w * spw + (__clzll((long long)y) >> lb);
        break;
      }
    }
  }
  l = min(l, L);
  return l >= a ? make_comp<C>(l, (u32)i, L, idbits) : ~C(0);
}

template <typename C, int Q>
__global__ void __launch_bounds__(FSQ_THREADS, fsq_ctas_per_sm<Q>())
    k_fullscan_smallq(DevIndex ix, const u64* __restrict__ qkeys, int count, int need, long long seg,
                      C* __restrict__ partial, int* __restrict__ hint, unsigned* __restrict__ done_ctr,
                      u32* __restrict__ out_ids, uint16_t* __restrict__ out_lcps,
                      int* __restrict__ out_hits, int out_stride) {
  constexpr int U = fsq_unroll<Q>();
  extern __shared__ __align__(16) unsigned char fsq_smem[];
  C* wl = reinterpret_cast<C*>(fsq_smem);  // [Q][FSQ_WARPS][32] warp lists
  __shared__ int s_last;
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const int L = ix.L, W = ix.W, lb = ix.lb, b = ix.b;
  const int idbits = sizeof(C) == 8 ? 32 : ix.idbits;
  const long long n = ix.n;

  u32 qh[Q], ql[Q], limh[Q];
  C slot[Q], thr[Q];
  int a[Q], a_own[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const u64 q0 = q < count ? qkeys[(long long)q * W] : 0ull;
    qh[q] = (u32)(q0 >> 32);
    ql[q] = (u32)q0;
    slot[q] = ~C(0);
    thr[q] = ~C(0);
    a[q] = q < count ? 0 : L + 1;  // absent queries never admit a key
    a_own[q] = 0;
    limh[q] = q < count ? ~0u : 0u;
  }
  // survive iff lcp >= na; on the hi word: (hi ^ qh) <= limh is necessary
  auto set_bound = [&](int q, int na) {
    a[q] = na;
    const int bits = na * b;
    limh[q] = na > L ? 0u : (bits >= 32 ? 0u : (~0u >> bits));
  };

  const long long gw = (long long)blockIdx.x * FSQ_WARPS + warp;
  const long long k0 = gw * seg;
  const long long k1 = min(n, k0 + seg);
#pragma unroll 1
  for (int sb = 0; sb < FSQ_SEED_STEPS && k0 + sb * 256 < k1; ++sb) {
    constexpr int US = 2;  // 256 keys: few registers beyond the main loop's
    const long long base = k0 + sb * 256;
    uint4 h[US];
#pragma unroll
    for (int u = 0; u < US; ++u) h[u] = ld_stream16(ix.keys_hi + base + u * 128 + lane * 4);
    // seed: the lists are empty, so every key of the first 256 is a candidate;
    // read their lo words with vector loads and offer only the step's top
    // lcp tier (the compact exact path below would re-read each key with its
    // own round trip)
      uint4 lo[US];
#pragma unroll
      for (int u = 0; u < US; ++u) lo[u] = ld_stream16(ix.keys_lo + base + u * 128 + lane * 4);
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        if (q >= count) continue;
        // t* = the largest first-word lcp that at least `need` of the step's
        // keys reach (binary search on warp-wide counts); only keys with
        // lcp >= t* can be among the step's top-need, and they are few
        const int T = min(L, ix.spw);
        auto n_at_least = [&](int t) {
          const int bits = t * b;
          const u64 lim = bits >= 64 ? 0ull : (~0ull >> bits);
          int c = 0;
#pragma unroll
          for (int u = 0; u < US; ++u) {
            const u32 hh[4] = {h[u].x, h[u].y, h[u].z, h[u].w};
            const u32 ll[4] = {lo[u].x, lo[u].y, lo[u].z, lo[u].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const u64 x = ((u64)(hh[j] ^ qh[q]) << 32) | (u64)(ll[j] ^ ql[q]);
              c += (base + u * 128 + lane * 4 + j < k1) && x <= lim;
            }
          }
          return __reduce_add_sync(LCP_FULL_MASK, (unsigned)c);
        };
        // keys below the list's bound cannot enter; keys below the sub-step's
        // own need-th lcp are beaten by need keys offered here
        int lo_t = min(a[q], T), hi_t = T;
        while (lo_t < hi_t) {
          const int mid = (lo_t + hi_t + 1) >> 1;
          if ((int)n_at_least(mid) >= need) lo_t = mid;
          else hi_t = mid - 1;
        }
        const int bits = lo_t * b;
        const u64 lim = bits >= 64 ? 0ull : (~0ull >> bits);
#pragma unroll
        for (int u = 0; u < US; ++u) {
          const u32 hh[4] = {h[u].x, h[u].y, h[u].z, h[u].w};
          const u32 ll[4] = {lo[u].x, lo[u].y, lo[u].z, lo[u].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const long long i = base + u * 128 + lane * 4 + j;
            const u64 x = ((u64)(hh[j] ^ qh[q]) << 32) | (u64)(ll[j] ^ ql[q]);
            const bool pass = i < k1 && x <= lim;
            if (!__any_sync(LCP_FULL_MASK, pass)) continue;
            C c = ~C(0);
            if (pass)
              c = (!x && W > 1) ? fsq_candidate<C>(ix.keys_hi, ix.keys_lo, ix.keys_orig, ix.spw, qkeys, q,
                                                   qh[q], ql[q], 0, i, L, W, lb, idbits)
                                : make_comp<C>(x ? min(L, __clzll((long long)x) >> lb) : L, (u32)i, L, idbits);
            warp_offer<C, true>(slot[q], thr[q], c, need);
          }
        }
        if (thr[q] != ~C(0)) {
          const int t = L - (int)(widen_comp<C>(thr[q], idbits) >> 32);
          a_own[q] = t + 1;
          if (lane == 0) atomicMax(hint + q, t);
          if (a_own[q] > a[q]) set_bound(q, a_own[q]);
        }
      }
  }
  int step = 0;
  for (long long base = k0 + 256 * FSQ_SEED_STEPS; base < k1; base += 128 * U, ++step) {
    if ((step & 1) == 0) {  // other warps' bounds (global hint)
      const int hv = lane < Q && lane < count ? *(volatile int*)(hint + lane) : 0;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int g = __shfl_sync(LCP_FULL_MASK, hv, q);
        if (g > a[q]) set_bound(q, g);
      }
    }
    uint4 h[U];
#pragma unroll
    for (int u = 0; u < U; ++u) h[u] = ld_stream16(ix.keys_hi + base + u * 128 + lane * 4);  // padded past n
    unsigned surv = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      u32 m = ~0u;
#pragma unroll
      for (int u = 0; u < U; ++u)
        m = min(m, min(min(h[u].x ^ qh[q], h[u].y ^ qh[q]), min(h[u].z ^ qh[q], h[u].w ^ qh[q])));
      surv |= (u32)(m <= limh[q]) << q;
    }
    surv = __reduce_or_sync(LCP_FULL_MASK, surv);
    if (!surv) continue;
    // exact path, compact on purpose (the unrolled form thrashed the
    // instruction cache: ncu "no instruction" was the top stall): each lane
    // marks its surviving key slots, then the warp offers one survivor per
    // lane per round, re-reading its words (L2) by index
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      if (!((surv >> q) & 1)) continue;
      u32 pm = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        pm |= (u32)((h[u].x ^ qh[q]) <= limh[q]) << (4 * u);
        pm |= (u32)((h[u].y ^ qh[q]) <= limh[q]) << (4 * u + 1);
        pm |= (u32)((h[u].z ^ qh[q]) <= limh[q]) << (4 * u + 2);
        pm |= (u32)((h[u].w ^ qh[q]) <= limh[q]) << (4 * u + 3);
      }
      while (__any_sync(LCP_FULL_MASK, pm != 0)) {
        C c = ~C(0);
        if (pm) {
          const int sl = __ffs(pm) - 1;
          pm &= pm - 1;
          const long long i = base + (sl >> 2) * 128 + lane * 4 + (sl & 3);
          if (i < k1)
            c = fsq_candidate<C>(ix.keys_hi, ix.keys_lo, ix.keys_orig, ix.spw, qkeys, q, qh[q], ql[q],
                                 a[q], i, L, W, lb, idbits);
        }
        warp_offer<C, true>(slot[q], thr[q], c, need);
      }
      if (thr[q] != ~C(0)) {  // full: later keys of this segment have larger ids
        const int t = L - (int)(widen_comp<C>(thr[q], idbits) >> 32);
        if (t + 1 > a_own[q]) {
          a_own[q] = t + 1;
          if (lane == 0) atomicMax(hint + q, t);
        }
        if (a_own[q] > a[q]) set_bound(q, a_own[q]);
      }
    }
  }
  // CTA merge: 16 warp lists per query -> one (tree of warp merges)
#pragma unroll
  for (int q = 0; q < Q; ++q) wl[(q * FSQ_WARPS + warp) * 32 + lane] = slot[q];
  __syncthreads();
  cta_tree_merge<C>(wl, FSQ_WARPS, min(Q, count));
  for (int t = threadIdx.x; t < count * need; t += FSQ_THREADS) {
    const int q = t / need, j = t - q * need;
    partial[((long long)blockIdx.x * count + q) * need + j] = wl[(q * FSQ_WARPS) * 32 + j];
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(done_ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // last CTA: the grid's lists per query, spread over all warps (warp w takes
  // CTA lists w', w' + P, ... of query w % Q), then a tree merge per query
  const int qn = min(Q, count);
  const int P = FSQ_WARPS / qn;  // warps per query
  if (warp < qn * P) {
    const int q = warp % qn, part = warp / qn;
    C sl = ~C(0), th = ~C(0);
    // lane l takes CTA list part + (r + l) * P; the lists' entries are offered
    // row by row (each list is sorted, so late rows rarely beat the threshold)
    for (long long r = 0; part + r * P < (long long)gridDim.x; r += 32) {
      const long long li = part + (r + lane) * P;
      for (int j = 0; j < need; ++j) {
        C c = ~C(0);
        if (li < gridDim.x) c = *(volatile C*)(partial + (li * count + q) * need + j);
        warp_offer<C, true>(sl, th, c, need);
      }
    }
    wl[(q * P + part) * 32 + lane] = sl;
  }
  __syncthreads();
  cta_tree_merge<C>(wl, P, qn);
  for (int t = threadIdx.x; t < count * need; t += FSQ_THREADS) {
    const int q = t / need, j = t - q * need;
    const u64 w64 = widen_comp<C>(wl[(q * P) * 32 + j], idbits);
    out_ids[(long long)q * out_stride + j] = (u32)(w64 & 0xffffffffull);
    out_lcps[(long long)q * out_stride + j] = (uint16_t)(L - (int)(w64 >> 32));
  }
  for (int q = threadIdx.x; q < count; q += FSQ_THREADS) {
    out_hits[q] = need;
    hint[q] = 0;  // ready for the next launch (graph replays)
  }
  if (threadIdx.x == 0) *done_ctr = 0;
}

// ---------------------------------------------------------------------------
// merge: per query, the `take` smallest of `shards` candidate lists of `kin`
// entries each (UINT64_MAX = empty).  cand index = s*s_stride + q*q_stride + j*j_stride.
// strict: keep only candidates whose lcp equals the best lcp over all lists
// (global strict mode = R(d_max) over the union).
// One warp per query; take <= 32.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    k_merge(const u64* __restrict__ cand, int shards, int count, int kin, long long s_stride,
            long long q_stride, long long j_stride, int take, int L, int strict, u32* __restrict__ out_ids,
            uint16_t* __restrict__ out_lcps, int* __restrict__ out_hits, int out_stride) {
  const int lane = lane_id();
  const long long qi = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (qi >= count) return;
  u64 best = ~0ull;
  if (strict) {
    for (int s = 0; s < shards; ++s)
      for (int j = lane; j < kin; j += 32) {
        u64 c = cand[s * s_stride + qi * q_stride + j * j_stride];
        best = c < best ? c : best;
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      u64 y = __shfl_xor_sync(LCP_FULL_MASK, best, o);
      best = y < best ? y : best;
    }
  }
  const u64 tier = best >> 32;
  u64 slot = ~0ull, thr = ~0ull;
  int valid = 0;
  for (int s = 0; s < shards; ++s) {
    for (int j0 = 0; j0 < kin; j0 += 32) {
      int j = j0 + lane;
      u64 c = j < kin ? cand[s * s_stride + qi * q_stride + j * j_stride] : ~0ull;
      if (strict && (c >> 32) != tier) c = ~0ull;
      valid += __popc(__ballot_sync(LCP_FULL_MASK, c != ~0ull));
      warp_offer<u64, true>(slot, thr, c, take);
    }
  }
  const int hits = min(take, valid);
  if (lane < hits) {
    out_ids[qi * out_stride + lane] = (u32)(slot & 0xffffffffull);
    out_lcps[qi * out_stride + lane] = (uint16_t)(L - (int)(slot >> 32));
  }
  if (lane == 0) out_hits[qi] = hits;
}

// merge for take > 32: one CTA per query sorts all shards' candidates
// (shards * kin <= MERGE_SORT_CAP, padded to a power of two) in shared memory
constexpr int MERGE_SORT_THREADS = 256;
constexpr int MERGE_SORT_CAP = 8192;

__global__ void __launch_bounds__(MERGE_SORT_THREADS)
    k_merge_sort(const u64* __restrict__ cand, int shards, int count, int kin, long long s_stride,
                 long long q_stride, long long j_stride, int take, int L, int strict, u32* __restrict__ out_ids,
                 uint16_t* __restrict__ out_lcps, int* __restrict__ out_hits, int out_stride) {
  extern __shared__ __align__(16) u64 sbuf[];
  __shared__ u64 s_best[MERGE_SORT_THREADS / 32];
  __shared__ int s_valid;
  const int m = shards * kin;
  int P = 1;
  while (P < m) P <<= 1;
  for (long long qi = blockIdx.x; qi < count; qi += gridDim.x) {
    u64 best = ~0ull;
    for (int t = threadIdx.x; t < P; t += MERGE_SORT_THREADS) {
      const u64 c = t < m ? cand[(t / kin) * s_stride + qi * q_stride + (t % kin) * j_stride] : ~0ull;
      sbuf[t] = c;
      best = c < best ? c : best;
    }
    if (threadIdx.x == 0) s_valid = 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const u64 y = __shfl_xor_sync(LCP_FULL_MASK, best, o);
      best = y < best ? y : best;
    }
    if (lane_id() == 0) s_best[threadIdx.x >> 5] = best;
    __syncthreads();
    for (int w = 0; w < MERGE_SORT_THREADS / 32; ++w) best = s_best[w] < best ? s_best[w] : best;
    int valid = 0;
    for (int t = threadIdx.x; t < P; t += MERGE_SORT_THREADS) {
      u64 c = sbuf[t];
      if (strict && (c >> 32) != (best >> 32)) c = ~0ull;  // strict: the best lcp tier only
      sbuf[t] = c;
      valid += c != ~0ull;
    }
    atomicAdd(&s_valid, valid);
    __syncthreads();
    bitonic_sort_smem(sbuf, P);
    const int hits = min(take, s_valid);
    for (int t = threadIdx.x; t < hits; t += MERGE_SORT_THREADS) {
      const u64 c = sbuf[t];
      out_ids[qi * out_stride + t] = (u32)(c & 0xffffffffull);
      out_lcps[qi * out_stride + t] = (uint16_t)(L - (int)(c >> 32));
    }
    if (threadIdx.x == 0) out_hits[qi] = hits;
    __syncthreads();
  }
}

__global__ void k_encode(const u32* __restrict__ ids, const uint16_t* __restrict__ lcps,
                         const int* __restrict__ hits, int count, int k, int in_stride, int L,
                         long long id_offset, u64* __restrict__ cand) {
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)count * k) return;
  long long q = t / k;
  int j = (int)(t - q * k);
  u64 c = ~0ull;
  if (j < hits[q])
    c = make_composite(lcps[q * in_stride + j], (u32)(ids[q * in_stride + j] + id_offset), L);
  cand[t] = c;
}
