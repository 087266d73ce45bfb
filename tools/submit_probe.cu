// Host cost of one pipelined e2e submission (256 KB H2D, a small kernel,
// 256 KB D2H, completion event) in three forms:
//   A: cudaMemcpyAsync + cudaGraphLaunch(kernel) + cudaMemcpyAsync + cudaEventRecord
//   B: one graph holding H2D + kernel + D2H nodes, + cudaEventRecord
//   C: B with the event record as a graph node (one API call per batch)
// Depth-8 ring of streams as in the library's async path.
// nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/submit_probe.cu -o /tmp/submit_probe
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void k_touch(const unsigned* in, unsigned* out, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = in[i] + 1;
}

int main() {
  const int D = 8, STEPS = 20000;
  const size_t B = 256 << 10;
  std::vector<cudaStream_t> st(D);
  std::vector<cudaEvent_t> ev(D);
  std::vector<void*> hin(D), hout(D), din(D), dout(D);
  for (int i = 0; i < D; ++i) {
    CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    CK(cudaHostAlloc(&hin[i], B, 0));
    CK(cudaHostAlloc(&hout[i], B, 0));
    CK(cudaMalloc(&din[i], B));
    CK(cudaMalloc(&dout[i], B));
  }
  const int n = (int)(B / 4);
  // form 0: copies + 1-kernel graph; 1: all in the graph; 2: copies + memset+kernel graph;
  // 3: copies + direct kernel launch (no graph); 4: copies + memset + direct launch
  for (int form = 0; form < 5; ++form) {
    std::vector<cudaGraphExec_t> ge(D);
    for (int i = 0; i < D; ++i) {
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(st[i], cudaStreamCaptureModeThreadLocal));
      if (form == 1) CK(cudaMemcpyAsync(din[i], hin[i], B, cudaMemcpyHostToDevice, st[i]));
      if (form == 2) CK(cudaMemsetAsync(dout[i], 0, 8, st[i]));
      k_touch<<<148, 256, 0, st[i]>>>((const unsigned*)din[i], (unsigned*)dout[i], n);
      if (form == 1) CK(cudaMemcpyAsync(hout[i], dout[i], B, cudaMemcpyDeviceToHost, st[i]));
      CK(cudaStreamEndCapture(st[i], &g));
      CK(cudaGraphInstantiate(&ge[i], g, 0));
      CK(cudaGraphDestroy(g));
    }
    double t_sub = 0, t_wait = 0;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
    CK(cudaDeviceSynchronize());
    const auto t0 = now();
    for (int s = 0; s < STEPS; ++s) {
      const int i = s % D;
      auto a = now();
      if (s >= D) CK(cudaEventSynchronize(ev[i]));
      auto b = now();
      if (form != 1) CK(cudaMemcpyAsync(din[i], hin[i], B, cudaMemcpyHostToDevice, st[i]));
      if (form == 4) CK(cudaMemsetAsync(dout[i], 0, 8, st[i]));
      if (form >= 3) k_touch<<<148, 256, 0, st[i]>>>((const unsigned*)din[i], (unsigned*)dout[i], n);
      else CK(cudaGraphLaunch(ge[i], st[i]));
      if (form != 1) CK(cudaMemcpyAsync(hout[i], dout[i], B, cudaMemcpyDeviceToHost, st[i]));
      CK(cudaEventRecord(ev[i], st[i]));
      auto c = now();
      t_wait += sec(a, b);
      t_sub += sec(b, c);
    }
    CK(cudaDeviceSynchronize());
    const double el = sec(t0, now());
    printf("form %d: %.2f us/batch; submit %.2f us, blocked %.2f us\n", form, 1e6 * el / STEPS,
           1e6 * t_sub / STEPS, 1e6 * t_wait / STEPS);
    for (auto x : ge) CK(cudaGraphExecDestroy(x));
  }
  // host allocation flags: default, mapped|portable (lcp_pinned_alloc),
  // write-combined (source of H2D only)
  const unsigned flag_sets[3] = {cudaHostAllocDefault, cudaHostAllocMapped | cudaHostAllocPortable,
                                 cudaHostAllocWriteCombined | cudaHostAllocMapped | cudaHostAllocPortable};
  for (int fs = 0; fs < 3; ++fs) {
    for (int i = 0; i < D; ++i) {
      CK(cudaFreeHost(hin[i]));
      CK(cudaHostAlloc(&hin[i], B, flag_sets[fs]));
      if (fs < 2) {
        CK(cudaFreeHost(hout[i]));
        CK(cudaHostAlloc(&hout[i], B, flag_sets[fs]));
      }
    }
  // copy-engine duplex: H2D only, D2H only, and both at once on separate
  // streams (no dependencies), 256 KB each, depth 8
  printf("host flags %s\n", fs == 0 ? "default" : fs == 1 ? "mapped|portable" : "write-combined (H2D source)");
  for (int mode = 0; mode < 3; ++mode) {
    CK(cudaDeviceSynchronize());
    const auto t0 = std::chrono::steady_clock::now();
    for (int s = 0; s < STEPS; ++s) {
      const int i = s % D;
      if (s >= D) CK(cudaEventSynchronize(ev[i]));
      if (mode == 0 || (mode == 2 && i < D / 2))
        CK(cudaMemcpyAsync(din[i], hin[i], B, cudaMemcpyHostToDevice, st[i]));
      else
        CK(cudaMemcpyAsync(hout[i], dout[i], B, cudaMemcpyDeviceToHost, st[i]));
      CK(cudaEventRecord(ev[i], st[i]));
    }
    CK(cudaDeviceSynchronize());
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("%s: %.2f us per 256 KB copy\n", mode == 0 ? "H2D only" : mode == 1 ? "D2H only" : "H2D and D2H mixed",
           1e6 * el / STEPS);
  }
  }
  return 0;
}
