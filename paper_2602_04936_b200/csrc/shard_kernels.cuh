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
