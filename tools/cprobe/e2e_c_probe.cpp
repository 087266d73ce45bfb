// C-level end-to-end probe: the packed async ABI driven from a C++ loop (no
// Python), plus raw pinned H2D / D2H bandwidth for the same byte counts.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <chrono>
#include <vector>

#include "../../include/lcp_b200.h"

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  const int64_t n = 2000000;
  const int L = 32, B = 4096, K = 10;
  std::vector<uint16_t> rows((size_t)n * L);
  uint64_t s = 88172645463325252ull;
  for (auto& v : rows) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; v = (uint16_t)(s & 3); }
  lcp_index* ix = nullptr;
  if (lcp_index_build(rows.data(), n, L, 4, -1, &ix)) { printf("build: %s\n", lcp_last_error()); return 1; }
  uint16_t* q = nullptr;
  cudaMallocHost((void**)&q, (size_t)8 * B * L * 2);
  for (int i = 0; i < 8 * B; ++i)
    for (int j = 0; j < L; ++j) q[(size_t)i * L + j] = rows[(size_t)((i * 7919) % n) * L + j];
  lcp_packed_layout lay;
  lcp_packed_layout_for(B, K, &lay);
  for (int depth : {1, 2, 4, 8}) {
    std::vector<lcp_workspace*> ws(depth);
    std::vector<void*> out(depth);
    for (int d = 0; d < depth; ++d) {
      lcp_workspace_create(&ws[d]);
      cudaMallocHost(&out[d], lay.total);
    }
    const int steps = 4000;
    double sub = 0;
    double t0 = 0;
    for (int i = -100; i < steps; ++i) {
      if (i == 0) t0 = now_us();
      const int d = (i + 100) % depth;
      lcp_workspace_wait(ws[d]);
      double a = now_us();
      lcp_query_host_packed_async(ix, ws[d], q + (size_t)((i + 800) % 8) * B * L, B, K, 1, K, out[d],
                                  LCP_PACKED_NO_WORK);
      if (i >= 0) sub += now_us() - a;
    }
    for (int d = 0; d < depth; ++d) lcp_workspace_wait(ws[d]);
    double el = now_us() - t0;
    printf("C loop depth %d: %.2f us/batch (submit %.2f) -> %.1f M q/s\n", depth, el / steps, sub / steps,
           B * steps / el);
    for (int d = 0; d < depth; ++d) { lcp_workspace_free(ws[d]); cudaFreeHost(out[d]); }
  }
  // raw PCIe: events around 1000 copies
  void *hbuf, *dbuf;
  cudaMallocHost(&hbuf, 1 << 20);
  cudaMalloc(&dbuf, 1 << 20);
  cudaStream_t st1, st2;
  cudaStreamCreate(&st1);
  cudaStreamCreate(&st2);
  for (size_t bytes : {(size_t)262144, (size_t)270336, (size_t)1048576}) {
    for (int dir = 0; dir < 2; ++dir) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, st1);
      for (int i = 0; i < 1000; ++i)
        cudaMemcpyAsync(dir ? hbuf : dbuf, dir ? dbuf : hbuf, bytes,
                        dir ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice, st1);
      cudaEventRecord(b, st1);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("%s %zu B: %.2f us/copy, %.1f GB/s\n", dir ? "D2H" : "H2D", bytes, ms, bytes / (ms * 1e-3 / 1000) / 1e9);
    }
  }
  {  // concurrent H2D (st1) and D2H (st2)
    void *h2, *d2;
    cudaMallocHost(&h2, 1 << 20);
    cudaMalloc(&d2, 1 << 20);
    cudaEvent_t a, b1, b2;
    cudaEventCreate(&a);
    cudaEventCreate(&b1);
    cudaEventCreate(&b2);
    cudaDeviceSynchronize();
    cudaEventRecord(a, st1);
    cudaStreamWaitEvent(st2, a, 0);
    for (int i = 0; i < 1000; ++i) {
      cudaMemcpyAsync(dbuf, hbuf, 262144, cudaMemcpyHostToDevice, st1);
      cudaMemcpyAsync(h2, d2, 270336, cudaMemcpyDeviceToHost, st2);
    }
    cudaEventRecord(b1, st1);
    cudaEventRecord(b2, st2);
    cudaEventSynchronize(b1);
    cudaEventSynchronize(b2);
    float m1, m2;
    cudaEventElapsedTime(&m1, a, b1);
    cudaEventElapsedTime(&m2, a, b2);
    printf("concurrent H2D 256K + D2H 264K: %.2f / %.2f us per pair\n", m1, m2);
  }
  // aggregate PCIe with S streams, each doing H2D 256 KB + D2H 264 KB per step
  for (int S : {1, 2, 4, 8}) {
    std::vector<cudaStream_t> ss(S);
    std::vector<void*> hs(S), ds(S), ho(S), dout(S);
    for (int i = 0; i < S; ++i) {
      cudaStreamCreateWithFlags(&ss[i], cudaStreamNonBlocking);
      cudaMallocHost(&hs[i], 262144);
      cudaMallocHost(&ho[i], 270336);
      cudaMalloc(&ds[i], 262144);
      cudaMalloc(&dout[i], 270336);
    }
    cudaDeviceSynchronize();
    const int steps = 2000;
    double t0 = now_us();
    for (int i = 0; i < steps; ++i) {
      const int j = i % S;
      cudaMemcpyAsync(ds[j], hs[j], 262144, cudaMemcpyHostToDevice, ss[j]);
      cudaMemcpyAsync(ho[j], dout[j], 270336, cudaMemcpyDeviceToHost, ss[j]);
    }
    cudaDeviceSynchronize();
    double el = now_us() - t0;
    printf("%d streams: %.2f us per (H2D 256K + D2H 264K) step, %.1f GB/s combined\n", S, el / steps,
           (262144.0 + 270336.0) * steps / (el * 1e3));
  }
  // the same pipeline without graphs: per batch on stream j, H2D -> lcp_query -> D2H
  for (int depth : {4, 6, 8}) {
    std::vector<lcp_workspace*> ws(depth);
    std::vector<cudaStream_t> ss(depth);
    std::vector<uint16_t*> dq(depth);
    std::vector<char*> dout(depth), hout(depth);
    const size_t ob = (size_t)B * K * 6 + (size_t)B * 4;
    for (int d = 0; d < depth; ++d) {
      lcp_workspace_create(&ws[d]);
      cudaStreamCreateWithFlags(&ss[d], cudaStreamNonBlocking);
      cudaMalloc((void**)&dq[d], (size_t)B * L * 2);
      cudaMalloc((void**)&dout[d], ob);
      cudaMallocHost((void**)&hout[d], ob);
    }
    const int steps = 4000;
    double t0 = 0;
    for (int i = -100; i < steps; ++i) {
      if (i == 0) t0 = now_us();
      const int d = (i + 100) % depth;
      cudaStreamSynchronize(ss[d]);
      cudaMemcpyAsync(dq[d], q + (size_t)((i + 800) % 8) * B * L, (size_t)B * L * 2, cudaMemcpyHostToDevice, ss[d]);
      lcp_query(ix, ws[d], dq[d], B, K, 1, K, (uint32_t*)dout[d], (uint16_t*)(dout[d] + (size_t)B * K * 4),
                (int32_t*)(dout[d] + (size_t)B * K * 6), nullptr, nullptr, ss[d]);
      cudaMemcpyAsync(hout[d], dout[d], ob, cudaMemcpyDeviceToHost, ss[d]);
    }
    for (int d = 0; d < depth; ++d) cudaStreamSynchronize(ss[d]);
    const double el = now_us() - t0;
    printf("no-graph pipeline depth %d: %.2f us/batch -> %.1f M q/s\n", depth, el / steps, B * steps / el);
  }
  // zero-copy: the query kernel reads pinned host queries and writes pinned host results
  for (int depth : {1, 2, 4, 8}) {
    std::vector<lcp_workspace*> ws(depth);
    std::vector<uint32_t*> ids(depth);
    std::vector<uint16_t*> lc(depth);
    std::vector<int32_t*> hits(depth);
    std::vector<cudaStream_t> sts(depth);
    for (int d = 0; d < depth; ++d) {
      lcp_workspace_create(&ws[d]);
      cudaMallocHost((void**)&ids[d], (size_t)B * K * 4);
      cudaMallocHost((void**)&lc[d], (size_t)B * K * 2);
      cudaMallocHost((void**)&hits[d], (size_t)B * 4);
      cudaStreamCreateWithFlags(&sts[d], cudaStreamNonBlocking);
    }
    const int steps = 4000;
    double t0 = 0;
    for (int i = -100; i < steps; ++i) {
      if (i == 0) t0 = now_us();
      const int d = (i + 100) % depth;
      cudaStreamSynchronize(sts[d]);
      int r = lcp_query(ix, ws[d], q + (size_t)((i + 800) % 8) * B * L, B, K, 1, K, ids[d], lc[d], hits[d],
                        nullptr, nullptr, sts[d]);
      if (r) { printf("zc query: %s\n", lcp_last_error()); return 1; }
    }
    for (int d = 0; d < depth; ++d) cudaStreamSynchronize(sts[d]);
    double el = now_us() - t0;
    printf("zero-copy depth %d: %.2f us/batch -> %.1f M q/s (hits[0]=%d ids[0]=%u)\n", depth, el / steps,
           B * steps / el, hits[0][0], ids[0][0]);
  }
  lcp_index_free(ix);
  return 0;
}
