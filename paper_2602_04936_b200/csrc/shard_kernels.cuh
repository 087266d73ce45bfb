// shard_kernels.cuh — device-side query routing for the multi-GPU paths.
//
// No reference counterpart: the paper is single-GPU; the
// north star shards the corpus over the GPUs of one box by lexicographic range
// or row block.  These kernels keep a sharded query step free of
// host round trips, so the whole step (route -> local top-k -> threshold
// exchange -> consult -> candidate exchange -> merge) is one stream-ordered
// sequence that a CUDA graph can capture:
//
//   k_route_queries   owner(q) = #splitters <= q (lexicographic, packed keys);
//                     phase 0 selects the queries this rank owns, phase 1 the
//                     queries another rank owns whose answer may reach into
//                     this rank's range: max(lcp(q, first), lcp(q, last)) >= t(q)
//                     (q lies outside the range, so those two rows bound every
//                     item's lcp).  The selected rows are compacted (ballot +
//                     one atomic per warp) into a dense batch plus their
//                     positions; the count stays on the device.
//   k_shard_threshold t(q) of the owner's answer: the lcp of its need-th hit
//                     (complete) or its d_max (strict), -1 when it holds fewer
//                     than need items — then every shard may contribute.
//   k_encode_sel      local answers -> (L - lcp) << 32 | global id candidates
//                     at the queries' batch positions (UINT64_MAX elsewhere).
#pragma once

#include "common.cuh"

// lexicographic compare of two W-word packed keys
__device__ __forceinline__ int cmp_words(const u64* a, const u64* b, int W) {
  for (int w = 0; w < W; ++w) {
    if (a[w] != b[w]) return a[w] < b[w] ? -1 : 1;
  }
  return 0;
}

__device__ __forceinline__ int lcp_words(const u64* a, const u64* b, int W, int L, int spw, int lb) {
  for (int w = 0; w < W; ++w) {
    const u64 x = a[w] ^ b[w];
    if (x) return min(L, w * spw + (__clzll((long long)x) >> lb));
  }
  return L;
}

constexpr int RT_THREADS = 256;

// consult == 0: select the owned queries and (optionally) reset the step's
// per-query state, thresholds[q] = -1 and cand[q][0..cand_k) = UINT64_MAX, so a
// step needs no separate fill launches; consult == 1: select by the consult rule
__global__ void __launch_bounds__(RT_THREADS)
    k_route_queries(const u64* __restrict__ qkeys, const uint16_t* __restrict__ queries, int count,
                    int L, int W, int spw, int lb, const u64* __restrict__ splitters, int nsplit,
                    const u64* __restrict__ first, const u64* __restrict__ last,
                    const int* __restrict__ nonempty, int rank, int* __restrict__ thresholds,
                    int consult, uint16_t* __restrict__ out_rows, int* __restrict__ out_sel,
                    int* __restrict__ d_count, u64* __restrict__ reset_cand, int cand_k) {
  const int q = blockIdx.x * RT_THREADS + threadIdx.x;
  const int lane = lane_id();
  bool take = false;
  if (q < count) {
    const u64* qk = qkeys + (long long)q * W;
    int owner = 0;
    for (int s = 0; s < nsplit; ++s) owner += cmp_words(splitters + (long long)s * W, qk, W) <= 0;
    if (!consult) {
      take = owner == rank;
      if (thresholds) thresholds[q] = -1;
      if (reset_cand)
        for (int j = 0; j < cand_k; ++j) reset_cand[(long long)q * cand_k + j] = ~0ull;
    } else if (owner != rank && nonempty[rank]) {
      const int best = max(lcp_words(qk, first + (long long)rank * W, W, L, spw, lb),
                           lcp_words(qk, last + (long long)rank * W, W, L, spw, lb));
      take = best >= thresholds[q];
    }
  }
  const unsigned m = __ballot_sync(LCP_FULL_MASK, take);
  int base = 0;
  if (lane == 0 && m) base = atomicAdd(d_count, __popc(m));
  base = __shfl_sync(LCP_FULL_MASK, base, 0);
  if (take) {
    const int pos = base + __popc(m & ((1u << lane) - 1u));
    out_sel[pos] = q;
    const uint16_t* src = queries + (long long)q * L;
    uint16_t* dst = out_rows + (long long)pos * L;
    for (int j = 0; j < L; ++j) dst[j] = src[j];
  }
}

__global__ void k_shard_threshold(const uint16_t* __restrict__ lcps, const int* __restrict__ hits,
                                  const uint16_t* __restrict__ md, const int* __restrict__ sel,
                                  const int* __restrict__ d_count, int stride, int need, int strict,
                                  int* __restrict__ thresholds) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *d_count) return;
  int t;
  if (strict) t = hits[i] > 0 ? (int)md[i] : -1;
  else t = (need > 0 && hits[i] >= need) ? (int)lcps[(long long)i * stride + need - 1] : -1;
  thresholds[sel[i]] = t;
}

__global__ void k_encode_sel(const u32* __restrict__ ids, const uint16_t* __restrict__ lcps,
                             const int* __restrict__ hits, const int* __restrict__ sel,
                             const int* __restrict__ d_count, int capacity, int k, int in_stride,
                             int L, const long long* __restrict__ gids, long long id_offset,
                             u64* __restrict__ cand) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)capacity * k) return;
  const int i = (int)(t / k), j = (int)(t - (long long)i * k);
  if (i >= *d_count) return;
  const long long q = sel[i];
  u64 c = ~0ull;
  if (j < hits[i]) {
    const u32 lid = ids[(long long)i * in_stride + j];
    const long long gid = (gids ? gids[lid] : (long long)lid) + id_offset;
    c = make_composite(lcps[(long long)i * in_stride + j], (u32)gid, L);
  }
  cand[q * k + j] = c;
}

// ---------------------------------------------------------------------------
// Candidate exchange over NVLink peer memory (replaces the NCCL all-to-all +
// merge of a sharded step).  Every rank's candidate buffer (batch rows x k
// u64) and a per-rank signal array (world u32) live in symmetric memory (one
// allocation per rank, mapped into every peer), so:
//   k_signal_peers   after a rank's candidates are final: bump its step epoch
//                    and, behind a system-scope fence, store the epoch into
//                    slot [rank] of every peer's signal array (NVLink stores);
//   k_merge_peers    rank r waits until every slot of its own signal array
//                    holds the current epoch, then merges its own clients'
//                    rows [r*m, (r+1)*m) by READING each peer's candidates
//                    directly (NVLink loads) — the exchange and the merge are
//                    one kernel, and no receive buffer or collective call is
//                    needed.
// Reuse is safe without a second barrier: a step's candidates are written
// only after that step's query all-gather, which no rank completes before
// every rank has finished the previous step's merge (stream order).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void st_release_sys_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void k_signal_peers(unsigned* const* __restrict__ peer_signals, int world, int rank,
                               unsigned* __restrict__ epoch) {
  // one thread: the candidates were written by earlier kernels of this stream
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const unsigned e = *epoch + 1u;
  *epoch = e;
  __threadfence_system();
  for (int s = 0; s < world; ++s) st_release_sys_u32(peer_signals[s] + rank, e);
}

// One warp per query row of this rank's clients (k <= 32: warp top-k, as
// k_merge); candidate c of shard s for local row q is peer_cand[s][(rank*m + q)*k + c]
__global__ void __launch_bounds__(256)
    k_merge_peers(const u64* const* __restrict__ peer_cand, int world, int rank, int m, int k, int take,
                  int L, int strict, const unsigned* __restrict__ my_signals,
                  const unsigned* __restrict__ epoch, u32* __restrict__ out_ids,
                  uint16_t* __restrict__ out_lcps, int* __restrict__ out_hits, int out_stride) {
  if (threadIdx.x == 0) {  // one thread waits; the barrier releases the CTA
    const unsigned e = *epoch;
    for (int s = 0; s < world; ++s)
      while (ld_acquire_sys_u32(my_signals + s) < e) {
      }
  }
  __syncthreads();
  const int lane = lane_id();
  const long long qi = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (qi >= m) return;
  const long long row = (long long)rank * m + qi;
  u64 best = ~0ull;
  if (strict) {
    for (int s = 0; s < world; ++s)
      for (int j = lane; j < k; j += 32) {
        const u64 c = __ldcv(peer_cand[s] + row * k + j);
        best = c < best ? c : best;
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const u64 y = __shfl_xor_sync(LCP_FULL_MASK, best, o);
      best = y < best ? y : best;
    }
  }
  const u64 tier = best >> 32;
  u64 slot = ~0ull, thr = ~0ull;
  int valid = 0;
  for (int s = 0; s < world; ++s) {
    for (int j0 = 0; j0 < k; j0 += 32) {
      const int j = j0 + lane;
      u64 c = j < k ? __ldcv(peer_cand[s] + row * k + j) : ~0ull;  // not cached: peers rewrite it per step
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
