// serve_kernels.cuh — persistent single-query server (latency mode).
//
// The reference answers one query per call (trie.py:290-342; the GNC loop of
// bench.py:353 calls it back to back).  Through the launch path a single
// query costs a graph launch, the kernel, and the host's wait on an event
// (≈13 µs round trip with direct host I/O).  The server removes the launch,
// the event and every dependent PCIe round trip but one: one warp stays
// resident and talks to the host through two mailboxes in page-locked host
// memory, each a run of 32-byte sectors whose last word is a tag:
//   request   sector j = 14 query symbols + tag.  The host writes a sector's
//             symbols, then its tag (x86 stores become visible in order), so
//             a sector read showing the new tag carries the new symbols; the
//             warp polls all request sectors with one load per lane (one
//             PCIe read per sector) until every tag holds the same new value;
//   response  sector j = 28 bytes of the packed answer + tag.  The per-query
//             code (query_w1_one) writes its outputs into shared memory laid
//             out as that payload; one store per word sends every sector with
//             the request's tag.  The host waits until every response sector
//             shows the tag, then unpacks the payload.
// No fence or second round trip is needed: each sector is self-validating.
// The warp exits on a stop tag (SERVE_STOP) or after SERVE_IDLE_NS without a
// request, so a stray device-wide synchronisation never waits on it for long;
// the host relaunches it on demand.
#pragma once

#include "query_kernels.cuh"

constexpr unsigned SERVE_STOP = 0x80000000u;
constexpr unsigned long long SERVE_IDLE_NS = 100ull * 1000 * 1000;  // 100 ms
constexpr int SERVE_SECTORS = 8;        // per mailbox: 8 x 32 B
constexpr int SERVE_SYMS_PER_SECTOR = 14;
constexpr int SERVE_PAYLOAD_PER_SECTOR = 28;
// response payload (bytes): hits i32 @0, matched_depth u16 @4, aux u64[2] @8,
// err i32 @24, ids u32[stride] @28, lcps u16[stride] @28 + 4 stride
constexpr int SERVE_P_HITS = 0, SERVE_P_MD = 4, SERVE_P_AUX = 8, SERVE_P_ERR = 24, SERVE_P_IDS = 28;

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned ld_sys_u32(const unsigned* p) {  // uncached, from host memory
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_sys_u32(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename C, int T, int MODE>
__global__ void __launch_bounds__(32, 1)
    k_serve_w1(const __grid_constant__ DevIndex ix, const unsigned* req, unsigned* resp, unsigned last, int k,
               int stride) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  u64* bar = reinterpret_cast<u64*>(smem_raw);
  u64* staged = reinterpret_cast<u64*>(smem_raw + 16);
  unsigned* row = reinterpret_cast<unsigned*>(staged + ix.smem_entries);  // query symbols, 2 per word
  unsigned* pay = row + SERVE_SECTORS * 8;                               // response payload
  unsigned char* pb = reinterpret_cast<unsigned char*>(pay);
  stage_issue(ix, bar, staged);
  const int lane = lane_id();
  const int nq = (ix.L + SERVE_SYMS_PER_SECTOR - 1) / SERVE_SYMS_PER_SECTOR;
  const int nr = (SERVE_P_IDS + 6 * stride + SERVE_PAYLOAD_PER_SECTOR - 1) / SERVE_PAYLOAD_PER_SECTOR;
  const bool tag_lane = (lane & 7) == 7;
  for (;;) {
    // poll: every request sector read once per round (words lane and
    // lane + 32: up to 8 sectors), all tags must agree
    unsigned w0 = 0, w1 = 0, tag = last;
    const unsigned long long t0 = global_ns();
    for (;;) {
      if (lane < nq * 8) w0 = ld_sys_u32(req + lane);
      if (lane + 32 < nq * 8) w1 = ld_sys_u32(req + lane + 32);
      tag = __shfl_sync(LCP_FULL_MASK, w0, 7);
      const bool stale = tag_lane && ((lane < nq * 8 && w0 != tag) || (lane + 32 < nq * 8 && w1 != tag));
      if (tag != last && !__any_sync(LCP_FULL_MASK, stale)) break;
      if (global_ns() - t0 > SERVE_IDLE_NS) {
        tag = SERVE_STOP;
        break;
      }
    }
    if (tag & SERVE_STOP) return;
    if (!tag_lane) {
      if (lane < nq * 8) row[(lane >> 3) * 7 + (lane & 7)] = w0;
      if (lane + 32 < nq * 8) row[((lane + 32) >> 3) * 7 + (lane & 7)] = w1;
    }
    if (lane < 8) pay[lane] = 0;  // header words: hits, md, aux, err
    __syncwarp();
    query_w1_one<C, T, MODE>(ix, reinterpret_cast<const uint16_t*>(row), 0, k, stride,
                             reinterpret_cast<u32*>(pb + SERVE_P_IDS),
                             reinterpret_cast<uint16_t*>(pb + SERVE_P_IDS + 4 * stride),
                             reinterpret_cast<int*>(pb + SERVE_P_HITS), reinterpret_cast<uint16_t*>(pb + SERVE_P_MD),
                             reinterpret_cast<u64*>(pb + SERVE_P_AUX), reinterpret_cast<int*>(pb + SERVE_P_ERR),
                             bar, staged);
    __syncwarp();
    for (int i = lane; i < nr * 8; i += 32) st_sys_u32(resp + i, tag_lane ? tag : pay[(i >> 3) * 7 + (i & 7)]);
    last = tag;
  }
}
