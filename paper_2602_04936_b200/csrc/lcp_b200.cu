// lcp_b200.cu — C-ABI implementation (include/lcp_b200.h).
//
// Host orchestration of the sm_100a kernels.  No torch types cross this
// boundary; device memory is owned by the index / workspace objects.
// There is no CPU compute path: every query, scan, sort and merge below is
// a kernel launch.

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <map>
#include <mutex>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/lcp_b200.h"
#include "build_kernels.cuh"
#include "common.cuh"
#include "fullscan_kernels.cuh"
#include "query_kernels.cuh"
#include "shard_kernels.cuh"
#include "serve_kernels.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define LCP_CK(call)                                                                  \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail(LCP_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));  \
  } while (0)

#define LCP_CK_LAUNCH()                                                               \
  do {                                                                                \
    cudaError_t e_ = cudaGetLastError();                                              \
    if (e_ != cudaSuccess)                                                            \
      return fail(LCP_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

#define LCP_TRY(expr)        \
  do {                       \
    int r_ = (expr);         \
    if (r_ != LCP_OK) return r_; \
  } while (0)

constexpr int kSmemStageCap = 32768;    // bytes of search levels staged per CTA
constexpr long long kMaxDirectory = 1ll << 24;  // tal.py:26 MAX_DIRECTORY_ENTRIES

bool is_device_ptr(const void* p) {
  if (p == nullptr) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

unsigned blocks_for(long long work, int threads) {
  long long b = (work + threads - 1) / threads;
  return (unsigned)std::max(1ll, b);
}

// Index memory comes from the device's stream-ordered pool, which keeps up to
// min(8 GB, 10 % of HBM) of freed memory mapped: rebuilding an index reuses it
// instead of unmapping and remapping hundreds of MB through the driver, while
// larger frees still return memory for other allocators (e.g. PyTorch's).
void keep_pool_mapped() {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::lock_guard<std::mutex> lock(mu);
  if (std::find(done.begin(), done.end(), dev) != done.end()) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    unsigned long long thr = std::min<unsigned long long>(8ull << 30, total_b / 10);
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  done.push_back(dev);
}

template <typename T>
int dalloc(T** p, long long count, long long* acct, cudaStream_t st) {
  size_t bytes = (size_t)std::max(1ll, count) * sizeof(T);
  cudaError_t e = cudaMallocAsync((void**)p, bytes, st);
  if (e != cudaSuccess)
    return fail(LCP_ERR_CUDA, std::string("cudaMalloc(") + std::to_string(bytes) +
                                  " bytes): " + cudaGetErrorString(e));
  if (acct) *acct += (long long)bytes;
  return LCP_OK;
}

// grow-only device buffer; `moves` counts reallocations so cached graphs that
// baked in the old pointer can be told apart (lcp_workspace::epoch)
struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  unsigned long long moves = 0;
  int ensure(size_t bytes) {
    if (bytes <= cap) return LCP_OK;
    ++moves;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 4096);
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess)
      return fail(LCP_ERR_CUDA, std::string("workspace cudaMalloc: ") + cudaGetErrorString(e));
    cap = want;
    return LCP_OK;
  }
  template <typename T>
  T* as() const { return reinterpret_cast<T*>(p); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

int num_sms() {
  static const int sms = [] {  // thread-safe one-time initialisation
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    return v;
  }();
  return sms;
}

// k_query_general grid: every resident CTA slot (the kernel strides over queries)
long long gen_grid(long long count) {
  static const int per_sm = [] {  // thread-safe one-time initialisation
    int v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_query_general, GEN_THREADS, 0) !=
            cudaSuccess || v <= 0)
      v = 8;
    return v;
  }();
  return std::min<long long>(count, (long long)per_sm * num_sms());
}

// ---- exclusive scan ------------------------------------------------------
template <typename T>
int scan_exclusive(T* data, long long m, cudaStream_t st) {
  if (m <= 0) return LCP_OK;
  long long ntiles = (m + SC_TILE - 1) / SC_TILE;
  if (ntiles == 1) {
    k_scan_tiles<T><<<1, SC_THREADS, 0, st>>>(data, m, (T*)nullptr);
    LCP_CK_LAUNCH();
    return LCP_OK;
  }
  T* sums = nullptr;
  LCP_CK(cudaMallocAsync((void**)&sums, (size_t)ntiles * sizeof(T), st));
  k_scan_tiles<T><<<(unsigned)ntiles, SC_THREADS, 0, st>>>(data, m, sums);
  LCP_CK_LAUNCH();
  int r = scan_exclusive<T>(sums, ntiles, st);
  if (r != LCP_OK) return r;
  k_scan_add<T><<<blocks_for(m, 256), 256, 0, st>>>(data, m, sums);
  LCP_CK_LAUNCH();
  LCP_CK(cudaFreeAsync(sums, st));
  return LCP_OK;
}

// ---- stable LSD radix sort of (u64 key, u32 val) ---------------------------
// Sorts in place semantically: on return (*k, *v) point at the sorted data
// (buffers may have been swapped with the alternates).  One upfront read
// builds all eight digit histograms (k_digit_hist8); the host reads them once
// to skip passes whose digit is constant (e.g. the low bits when L*b < 64);
// every remaining pass is one onesweep kernel (k_onesweep).
int radix_sort_pairs(u64** k, u32** v, u64** k_alt, u32** v_alt, long long n, cudaStream_t st) {
  if (n <= 1) return LCP_OK;
  u32* hist = nullptr;
  LCP_CK(cudaMallocAsync((void**)&hist, 8 * 256 * sizeof(u32), st));
  LCP_CK(cudaMemsetAsync(hist, 0, 8 * 256 * sizeof(u32), st));
  unsigned hb = (unsigned)std::min<long long>(blocks_for(n, 256), 4ll * num_sms());
  k_digit_hist8<<<hb, 256, 0, st>>>(*k, n, hist);
  LCP_CK_LAUNCH();
  std::vector<u32> h(8 * 256);
  LCP_CK(cudaMemcpyAsync(h.data(), hist, h.size() * sizeof(u32), cudaMemcpyDeviceToHost, st));
  LCP_CK(cudaStreamSynchronize(st));

  const long long ntiles = (n + OS_TILE - 1) / OS_TILE;
  u64* status = nullptr;
  unsigned* counters = nullptr;
  LCP_CK(cudaMallocAsync((void**)&status, (size_t)ntiles * 256 * sizeof(u64), st));
  LCP_CK(cudaMallocAsync((void**)&counters, 8 * sizeof(unsigned), st));
  LCP_CK(cudaMemsetAsync(counters, 0, 8 * sizeof(unsigned), st));
  static const cudaError_t attr = [] {  // thread-safe one-time initialisation
    cudaError_t e = cudaFuncSetAttribute(k_onesweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)OS_SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_onesweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)OS_SMEM);
    return e;
  }();
  LCP_CK(attr);
  // count + scan + scatter (three kernels, one more read of the keys, no
  // serial chain) or decoupled look-back (one kernel per pass).  Measured at
  // 2M / 25M rows (2048-key tiles): 0.735 / 4.37 ms whole build against
  // 0.79 / 4.79 ms with the look-back, whose first wave is a serial prefix
  // chain; LCP_SORT_LOOKBACK=1 selects it (A/B hook)
  static const bool lookback = [] {
    const char* e = getenv("LCP_SORT_LOOKBACK");
    return e && atoi(e) != 0;
  }();
  u32* offs = nullptr;
  if (!lookback) LCP_CK(cudaMallocAsync((void**)&offs, (size_t)ntiles * 256 * sizeof(u32), st));
  for (int p = 0; p < 8; ++p) {
    bool trivial = false;
    for (int d = 0; d < 256; ++d)
      if ((long long)h[p * 256 + d] == n) trivial = true;
    if (trivial) continue;  // every key has the same digit: pass is the identity
    if (lookback) {
      LCP_CK(cudaMemsetAsync(status, 0, (size_t)ntiles * 256 * sizeof(u64), st));
    } else {
      k_rs_upsweep<<<(unsigned)ntiles, RS_THREADS, 0, st>>>(*k, n, 8 * p, (int)ntiles, offs);
      LCP_CK_LAUNCH();
      LCP_TRY(scan_exclusive<u32>(offs, ntiles * 256, st));
    }
    if (lookback)
      k_onesweep<true><<<(unsigned)ntiles, OS_THREADS, OS_SMEM, st>>>(
          *k, *v, *k_alt, *v_alt, n, 8 * p, hist + p * 256, status, counters + p, nullptr, (int)ntiles);
    else
      k_onesweep<false><<<(unsigned)ntiles, OS_THREADS, OS_SMEM, st>>>(
          *k, *v, *k_alt, *v_alt, n, 8 * p, hist + p * 256, status, counters + p, offs, (int)ntiles);
    LCP_CK_LAUNCH();
    std::swap(*k, *k_alt);
    std::swap(*v, *v_alt);
  }
  if (offs) LCP_CK(cudaFreeAsync(offs, st));
  LCP_CK(cudaFreeAsync(status, st));
  LCP_CK(cudaFreeAsync(counters, st));
  LCP_CK(cudaFreeAsync(hist, st));
  return LCP_OK;
}

// pack n rows into keys (+ ids): the streaming kernel when every row is a
// whole number of 16-byte chunks, the per-word kernel otherwise
int pack_rows(const uint16_t* rows, long long n, const DevIndex& dv, u64* keys, u32* ids, int* err,
              cudaStream_t st) {
  if (n <= 0) return LCP_OK;
  const int cpr = dv.L / 8;
  if (dv.L % 8 == 0 && ((uintptr_t)rows & 15) == 0 && dv.L % dv.spw == 0 && cpr <= 32 &&
      32 % cpr == 0) {
    const long long units = (n + 32 / cpr - 1) / (32 / cpr);
    const long long want = (units + (PK_THREADS / 32) * PK_UNROLL - 1) / ((PK_THREADS / 32) * PK_UNROLL);
    const unsigned grid = (unsigned)std::max(1ll, std::min<long long>(want, 8ll * num_sms()));
#define LCP_PKA(BB) k_pack_aligned<BB><<<grid, PK_THREADS, 0, st>>>(rows, n, dv.L, dv.W, dv.sigma, keys, ids, err)
    switch (dv.b) {
      case 1: LCP_PKA(1); break;
      case 2: LCP_PKA(2); break;
      case 4: LCP_PKA(4); break;
      case 8: LCP_PKA(8); break;
      default: LCP_PKA(16); break;
    }
#undef LCP_PKA
  } else if (dv.L % 8 == 0 && ((uintptr_t)rows & 15) == 0) {
    const long long units = cpr <= 32 ? (n + 32 / cpr - 1) / (32 / cpr) : n * ((cpr + 31) / 32);
    const long long want = (units + (PK_THREADS / 32) * PK_UNROLL - 1) / ((PK_THREADS / 32) * PK_UNROLL);
    const unsigned grid = (unsigned)std::max(1ll, std::min<long long>(want, 8ll * num_sms()));
    k_pack_stream<<<grid, PK_THREADS, 0, st>>>(rows, n, dv.L, dv.W, dv.b, dv.spw, dv.sigma, keys, ids, err);
  } else {
    k_pack<<<blocks_for(n * dv.W, 256), 256, 0, st>>>(rows, n, dv.L, dv.W, dv.b, dv.spw, dv.sigma, keys,
                                                      ids, err);
  }
  LCP_CK_LAUNCH();
  return LCP_OK;
}

int pow2_bits(int sigma) {
  int need = 0;
  while ((1 << need) < sigma) ++need;  // ceil(log2 sigma)
  int b = 1;
  while (b < need) b <<= 1;
  return b;
}

int ilog2(int v) {
  int r = 0;
  while ((1 << r) < v) ++r;
  return r;
}

}  // namespace

// ===========================================================================
struct lcp_index {
  DevIndex dv{};
  unsigned long long generation = 0;  // unique per build: keys cached graphs
  int tal_depth = -1;
  long long tal_buckets = 0;  // -1: overflow (> 2^62)
  long long device_bytes = 0;
  u64* keys = nullptr;
  u64* keys_orig = nullptr;
  u32* order = nullptr;
  u32* keys_hi = nullptr;
  u32* keys_lo = nullptr;
  uint16_t* adj = nullptr;
  u64* levels = nullptr;
  long long* directory = nullptr;
  u32* sketch = nullptr;
  u32* rank = nullptr;  // original id -> sorted position
  u64* keys_w0 = nullptr;
  u64* levels_w0 = nullptr;  // W > 1: first word of each search-table entry
  std::vector<long long> level_offset;  // cached trie level offsets
};

// One captured async submission (H2D -> query kernel -> D2H -> error word),
// replayed with a single cudaGraphLaunch when the same buffers come back.
// `epoch` is the workspace's scratch epoch at capture: a graph bakes in the
// device scratch pointers, so once any scratch buffer moved it must not replay.
// A graph holds device work only (the flag reset and the query kernels over
// workspace scratch); the host<->device copies are issued around it per call,
// so no graph ever references caller memory (a freed and reallocated host
// block at the same address crashed cuGraphLaunch when the copies were nodes).
struct GraphKey {
  unsigned long long gen, epoch;
  int count, k, mode, stride;
  // direct host I/O (small batches): the page-locked query / result blocks the
  // kernels read and write; null when the submission copies through scratch
  const void* hq;
  const void* ho;
  bool operator==(const GraphKey& o) const {
    return gen == o.gen && epoch == o.epoch && count == o.count && k == o.k && mode == o.mode &&
           stride == o.stride && hq == o.hq && ho == o.ho;
  }
};
struct CachedGraph {
  GraphKey key;
  cudaGraphExec_t exec;
  unsigned long long last_use;
};
constexpr int kGraphCache = 16;

// Live lcp_pinned_alloc blocks: base -> (bytes, device alias).  Direct host I/O
// is used only for ranges inside one of them, so a kernel never dereferences
// host memory that is not page-locked and mapped.
struct PinnedBlock {
  size_t bytes;
  void* dev;
};
static std::mutex g_pinned_mu;
static std::map<uintptr_t, PinnedBlock> g_pinned;

static char* pinned_device_alias(const void* p, size_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  std::lock_guard<std::mutex> g(g_pinned_mu);
  auto it = g_pinned.upper_bound(a);
  if (it == g_pinned.begin()) return nullptr;
  --it;
  if (!it->second.dev || a + bytes > it->first + it->second.bytes) return nullptr;
  return static_cast<char*>(it->second.dev) + (a - it->first);
}

struct lcp_workspace {
  cudaStream_t stream = nullptr;
  std::vector<CachedGraph> graphs;
  unsigned long long tick = 0;
  cudaEvent_t done = nullptr;  // completion of the in-flight async batch
  bool pending = false;
  int pending_sigma = 0;
  const int* pending_err = nullptr;  // host flag inside the in-flight packed block
  int* d_err = nullptr;
  int* h_err = nullptr;  // pinned
  DBuf qkeys, partial, hint, q_in, ids, lcps, hits, md, aux;
  // changes whenever a scratch buffer is reallocated (its old memory freed)
  unsigned long long epoch() const {
    return qkeys.moves + partial.moves + hint.moves + q_in.moves + ids.moves + lcps.moves +
           hits.moves + md.moves + aux.moves;
  }
  // drop cached graphs captured against scratch that has since moved
  void prune_stale_graphs() {
    const unsigned long long e = epoch();
    for (size_t i = 0; i < graphs.size();) {
      if (graphs[i].key.epoch != e) {
        cudaGraphExecDestroy(graphs[i].exec);
        graphs.erase(graphs.begin() + i);
      } else {
        ++i;
      }
    }
  }
};

extern "C" {

int lcp_abi_version(void) { return LCP_ABI_VERSION; }

const char* lcp_last_error(void) { return g_err.c_str(); }

int lcp_index_free(lcp_index* ix) {
  if (!ix) return LCP_OK;
  // like cudaFree: nothing may still use the index; the memory returns to the
  // (mapped) stream-ordered pool
  cudaDeviceSynchronize();
  if (ix->keys) cudaFreeAsync(ix->keys, 0);
  if (ix->keys_orig) cudaFreeAsync(ix->keys_orig, 0);
  if (ix->order) cudaFreeAsync(ix->order, 0);
  if (ix->keys_hi) cudaFreeAsync(ix->keys_hi, 0);
  if (ix->keys_lo) cudaFreeAsync(ix->keys_lo, 0);
  if (ix->adj) cudaFreeAsync(ix->adj, 0);
  if (ix->levels) cudaFreeAsync(ix->levels, 0);
  if (ix->directory) cudaFreeAsync(ix->directory, 0);
  if (ix->sketch) cudaFreeAsync(ix->sketch, 0);
  if (ix->rank) cudaFreeAsync(ix->rank, 0);
  if (ix->keys_w0) cudaFreeAsync(ix->keys_w0, 0);
  if (ix->levels_w0) cudaFreeAsync(ix->levels_w0, 0);
  cudaStreamSynchronize(0);
  delete ix;
  return LCP_OK;
}

static int build_impl(lcp_index* ix, const uint16_t* rows, long long n, int L, int sigma,
                      int tal_depth, cudaStream_t st) {
  DevIndex& dv = ix->dv;
  const int W = dv.W;
  long long* acct = &ix->device_bytes;
  // LCP_BUILD_TRACE=1: per-phase wall times on stderr (diagnostics only)
  static const bool trace = getenv("LCP_BUILD_TRACE") != nullptr;
  auto t_start = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!trace) return;
    cudaStreamSynchronize(st);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    fprintf(stderr, "[build] %-10s %8.2f ms\n", what, ms);
  };

  // rows -> device
  const uint16_t* d_rows = rows;
  uint16_t* owned_rows = nullptr;
  if (!is_device_ptr(rows)) {
    LCP_CK(cudaMallocAsync((void**)&owned_rows, (size_t)n * L * sizeof(uint16_t), st));
    LCP_CK(cudaMemcpyAsync(owned_rows, rows, (size_t)n * L * sizeof(uint16_t),
                           cudaMemcpyHostToDevice, st));
    d_rows = owned_rows;
  }
  struct RowsGuard {
    uint16_t* p;
    cudaStream_t st;
    ~RowsGuard() { if (p) cudaFreeAsync(p, st); }
  } rows_guard{owned_rows, st};

  phase("rows");
  const long long pad = 64;
  LCP_TRY(dalloc(&ix->keys_orig, (n + pad) * W, acct, st));
  LCP_CK(cudaMemsetAsync(ix->keys_orig, 0, (size_t)(n + pad) * W * 8, st));
  u32* perm = nullptr;
  u32* perm_alt = nullptr;
  u64* kw = nullptr;
  u64* kw_alt = nullptr;
  int* d_err = nullptr;
  LCP_CK(cudaMallocAsync((void**)&perm, (size_t)(n + pad) * 4, st));
  LCP_CK(cudaMallocAsync((void**)&perm_alt, (size_t)(n + pad) * 4, st));
  LCP_CK(cudaMallocAsync((void**)&kw, (size_t)(n + pad) * 8, st));
  LCP_CK(cudaMallocAsync((void**)&kw_alt, (size_t)(n + pad) * 8, st));
  LCP_CK(cudaMallocAsync((void**)&d_err, sizeof(int), st));
  struct TmpGuard {
    std::vector<void*> ps;
    cudaStream_t st;
    ~TmpGuard() { for (void* p : ps) if (p) cudaFreeAsync(p, st); }
  } tmp{{perm_alt, kw_alt, d_err}, st};
  LCP_CK(cudaMemsetAsync(d_err, 0, sizeof(int), st));

  LCP_TRY(pack_rows(d_rows, n, dv, ix->keys_orig, perm, d_err, st));
  int h_err = 0;
  LCP_CK(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
  LCP_CK(cudaStreamSynchronize(st));
  if (h_err) {
    cudaFreeAsync(perm, st);
    cudaFreeAsync(kw, st);
    return fail(LCP_ERR_INVALID_INPUT,
                "symbol out of range for alphabet of size " + std::to_string(sigma));
  }

  phase("pack");
  // stable LSD over words (least significant word first) — core.py:162-174
  for (int w = W - 1; w >= 0; --w) {
    if (W == 1) {
      LCP_CK(cudaMemcpyAsync(kw, ix->keys_orig, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
    } else {
      k_gather_word<<<blocks_for(n, 256), 256, 0, st>>>(ix->keys_orig, perm, n, W, w, kw);
      LCP_CK_LAUNCH();
    }
    u64* kb = kw;
    u32* vb = perm;
    u64* ka = kw_alt;
    u32* va = perm_alt;
    LCP_TRY(radix_sort_pairs(&kb, &vb, &ka, &va, n, st));
    kw = kb;
    perm = vb;
    kw_alt = ka;
    perm_alt = va;
  }
  phase("sort");
  tmp.ps = {perm_alt, kw_alt, d_err};
  ix->order = perm;
  *acct += (n + pad) * 4;
  if (W == 1) {
    ix->keys = kw;
    *acct += (n + pad) * 8;
  } else {
    tmp.ps.push_back(kw);
    LCP_TRY(dalloc(&ix->keys, (n + pad) * W, acct, st));
    LCP_CK(cudaMemsetAsync(ix->keys, 0, (size_t)(n + pad) * W * 8, st));
    k_gather_keys<<<blocks_for(n * W, 256), 256, 0, st>>>(ix->keys_orig, perm, n, W, ix->keys);
    LCP_CK_LAUNCH();
  }
  dv.keys = ix->keys;
  dv.keys_orig = ix->keys_orig;
  dv.order = ix->order;
  {  // hi / lo planes of the original-order keys' first word, for the full scan
    // whole 16 KB stages, plus slack for the small-batch scan's last step
    const long long pn = (n + 4095) / 4096 * 4096 + 2048;
    LCP_TRY(dalloc(&ix->keys_hi, pn, acct, st));
    LCP_TRY(dalloc(&ix->keys_lo, pn, acct, st));
    LCP_CK(cudaMemsetAsync(ix->keys_hi, 0, (size_t)pn * 4, st));
    LCP_CK(cudaMemsetAsync(ix->keys_lo, 0, (size_t)pn * 4, st));
    k_split_words<<<blocks_for(n, 256), 256, 0, st>>>(ix->keys_orig, n, W, ix->keys_hi, ix->keys_lo);
    LCP_CK_LAUNCH();
  }
  dv.keys_hi = ix->keys_hi;
  dv.keys_lo = ix->keys_lo;

  phase("planes");
  // adjacent lcp — core.py:177-184
  LCP_TRY(dalloc(&ix->adj, std::max(1ll, n - 1), acct, st));
  if (n > 1) {
    if (W == 1) k_adjacent_lcp<1><<<blocks_for(n - 1, 256), 256, 0, st>>>(dv, ix->adj);
    else k_adjacent_lcp<0><<<blocks_for(n - 1, 256), 256, 0, st>>>(dv, ix->adj);
    LCP_CK_LAUNCH();
  }

  phase("adj");
  // k-ary search levels (stand-in for the trie descent, trie.py:229-256)
  // Tables j = 0..h-1 sample every LCP_LEAF_KEYS * 64**(h-1-j)-th key; the
  // last one resolves lower_bound(q) to a leaf block of LCP_LEAF_KEYS keys.
  int h = 0;
  {
    long long cap = LCP_LEAF_KEYS;
    while (n > cap && h < LCP_MAX_LEVELS - 1) {
      cap *= 64;
      ++h;
    }
  }
  dv.nlevels = h;
  long long total = 0;
  std::vector<long long> strides(h);
  for (int j = 0; j < h; ++j) {
    long long s = LCP_LEAF_KEYS;
    for (int t = 0; t < h - 1 - j; ++t) s *= 64;
    strides[j] = s;
    long long cnt = (n + s - 1) / s;
    dv.level_cnt[j] = cnt;
    dv.level_off[j] = total;
    // whole 64-entry blocks, padded with all-ones keys (never < q): the
    // W == 1 search reads a full block per level with no bounds checks
    total += (cnt + LCP_SEARCH_FANOUT - 1) / LCP_SEARCH_FANOUT * LCP_SEARCH_FANOUT;
  }
  LCP_TRY(dalloc(&ix->levels, std::max(2ll, total) * W, acct, st));
  LCP_CK(cudaMemsetAsync(ix->levels, 0xFF, (size_t)std::max(2ll, total) * W * 8, st));
  for (int j = 0; j < h; ++j) {
    k_gather_level<<<blocks_for(dv.level_cnt[j] * W, 256), 256, 0, st>>>(
        ix->keys, dv.level_cnt[j], strides[j], W, ix->levels + dv.level_off[j] * W);
    LCP_CK_LAUNCH();
  }
  dv.levels = ix->levels;
  dv.levels_w0 = ix->levels;  // W == 1: the keys / levels are their own first-word planes
  dv.keys_w0 = ix->keys;
  if (W > 1) {  // first-word planes: W > 1 comparisons read 8 B per entry / key
    // (coalesced) and the whole key only when the first words are equal
    const long long lt = std::max(2ll, total);
    LCP_TRY(dalloc(&ix->levels_w0, lt, acct, st));
    k_first_word<<<blocks_for(lt, 256), 256, 0, st>>>(ix->levels, lt, W, ix->levels_w0);
    LCP_CK_LAUNCH();
    dv.levels_w0 = ix->levels_w0;
    LCP_TRY(dalloc(&ix->keys_w0, std::max(1ll, n), acct, st));
    k_first_word<<<blocks_for(n, 256), 256, 0, st>>>(ix->keys, n, W, ix->keys_w0);
    LCP_CK_LAUNCH();
    dv.keys_w0 = ix->keys_w0;
  }
  dv.smem_levels = 0;
  dv.smem_entries = 0;
  static const long long smem_cap = [] {  // LCP_SMEM_STAGE_CAP: A/B hook (bytes)
    const char* e = getenv("LCP_SMEM_STAGE_CAP");
    return e ? atoll(e) : (long long)kSmemStageCap;
  }();
  for (int j = 0; j < h; ++j) {
    long long end = dv.level_off[j] +
                    (dv.level_cnt[j] + LCP_SEARCH_FANOUT - 1) / LCP_SEARCH_FANOUT * LCP_SEARCH_FANOUT;
    if (end * 8 > smem_cap) break;  // the first-word plane is staged
    dv.smem_levels = j + 1;
    dv.smem_entries = (int)end;
  }

  phase("levels");
  // id sketch (smallest ids per block of sorted positions): bounds the work
  // of a query whose R(d*) spans far more than the loaded region
  {
    long long cnt = (n + LCP_SK_BLOCK - 1) / LCP_SK_BLOCK, tot = 0;
    int lv = 0;
    for (;;) {
      dv.sk_off[lv] = tot;
      dv.sk_cnt[lv] = cnt;
      tot += cnt;
      ++lv;
      if (cnt <= LCP_SK_FANOUT || lv == LCP_MAX_LEVELS) break;
      cnt = (cnt + LCP_SK_FANOUT - 1) / LCP_SK_FANOUT;
    }
    dv.sk_levels = lv;
    LCP_TRY(dalloc(&ix->sketch, tot * LCP_SK_LIST, acct, st));
    const auto sk_grid = [](long long blocks) { return (unsigned)((blocks * 32 + SK_THREADS - 1) / SK_THREADS); };
    k_id_sketch<LCP_SK_BLOCK><<<sk_grid(dv.sk_cnt[0]), SK_THREADS, 0, st>>>(ix->order, n, dv.sk_cnt[0],
                                                                            ix->sketch);
    LCP_CK_LAUNCH();
    for (int j = 1; j < lv; ++j) {
      k_id_sketch_cta<LCP_SK_FANOUT * LCP_SK_LIST><<<(unsigned)dv.sk_cnt[j], SK_THREADS, 0, st>>>(
          ix->sketch + dv.sk_off[j - 1] * LCP_SK_LIST, dv.sk_cnt[j - 1] * LCP_SK_LIST,
          ix->sketch + dv.sk_off[j] * LCP_SK_LIST);
      LCP_CK_LAUNCH();
    }
    dv.sketch = ix->sketch;
  }
  // inverse permutation (id -> sorted position): lets the general path take
  // the smallest ids of a tier that spans most of the corpus in id order
  LCP_TRY(dalloc(&ix->rank, std::max(1ll, n), acct, st));
  k_invert<<<blocks_for(n, 256), 256, 0, st>>>(ix->order, n, ix->rank);
  LCP_CK_LAUNCH();
  dv.rank = ix->rank;

  phase("sketch");
  // TAL bucket structure — tal.py:42-82
  if (tal_depth >= 0) {
    // (W == 1 TAL counts symbols from the region and the run edges,
    // tal_sym_region; W > 1 sweeps the first-word plane built with the levels)
    ix->tal_depth = tal_depth;
    long long buckets = 1;
    bool overflow = false;
    for (int j = 0; j < tal_depth; ++j) {
      if (buckets > (1ll << 62) / sigma) {
        overflow = true;
        break;
      }
      buckets *= sigma;
    }
    ix->tal_buckets = overflow ? -1 : buckets;
    if (tal_depth > 0 && !overflow && buckets <= kMaxDirectory) {
      LCP_TRY(dalloc(&ix->directory, buckets + 1, acct, st));
      k_directory<<<blocks_for(buckets + 1, 256), 256, 0, st>>>(dv, tal_depth, buckets,
                                                               ix->directory);
      LCP_CK_LAUNCH();
    }
  }
  dv.tal_depth = ix->tal_depth;
  dv.tal_buckets = ix->tal_buckets;
  dv.directory = ix->directory;
  LCP_CK(cudaStreamSynchronize(st));
  phase("done");
  return LCP_OK;
}

int lcp_index_build(const uint16_t* rows, int64_t n, int32_t length, int32_t sigma,
                    int32_t tal_depth, lcp_index** out) {
  if (!out) return fail(LCP_ERR_INVALID_INPUT, "out must not be null");
  *out = nullptr;
  if (sigma < 2 || sigma > 65536)
    return fail(LCP_ERR_INVALID_INPUT,
                "alphabet size must be in [2, 65536], got " + std::to_string(sigma));
  if (length < 1 || length > 65535)
    return fail(LCP_ERR_INVALID_INPUT,
                "sequence length must be in [1, 65535], got " + std::to_string(length));
  if (n < 0 || n >= (1ll << 31))
    return fail(LCP_ERR_INVALID_INPUT, "n must be in [0, 2**31), got " + std::to_string(n));
  if (tal_depth > length)
    return fail(LCP_ERR_INVALID_INPUT, "tal depth exceeds the sequence length");
  if (n > 0 && !rows) return fail(LCP_ERR_INVALID_INPUT, "rows must not be null");

  lcp_index* ix = new lcp_index();
  {
    static unsigned long long next_gen = 1;
    static std::mutex gen_mu;
    std::lock_guard<std::mutex> lock(gen_mu);
    ix->generation = next_gen++;
  }
  DevIndex& dv = ix->dv;
  dv.n = n;
  dv.L = length;
  dv.sigma = sigma;
  dv.b = pow2_bits(sigma);
  dv.lb = ilog2(dv.b);
  dv.spw = 64 / dv.b;
  dv.W = (length + dv.spw - 1) / dv.spw;
  dv.tal_depth = -1;
  {
    // compact u32 composite: (L - lcp) needs ceil(log2(L + 1)) bits, ids the rest
    int lbits = 0;
    while ((1 << lbits) < length + 1) ++lbits;
    const int idb = 32 - lbits;
    // ids < n <= 2^idb - 1: the largest composite (lcp 0, id n-1) then
    // stays below the all-ones empty sentinel even when L = 2^lbits - 1
    dv.idbits = (idb >= 1 && n < (1ll << idb)) ? idb : 32;
    // test hook: exercise the u64 selection path on small inputs
    const char* wide = getenv("LCP_FORCE_WIDE_COMPOSITE");
    if (wide && wide[0] == '1') dv.idbits = 32;
  }
  if (n == 0) {
    if (tal_depth >= 0) {
      ix->tal_depth = tal_depth;
      long long buckets = 1;
      for (int j = 0; j < tal_depth && buckets <= (1ll << 40); ++j) buckets *= sigma;
      ix->tal_buckets = buckets;
      dv.tal_depth = tal_depth;
      dv.tal_buckets = buckets;
      if (tal_depth > 0 && buckets <= kMaxDirectory) {
        int r = dalloc(&ix->directory, buckets + 1, &ix->device_bytes, (cudaStream_t)0);
        if (r != LCP_OK) {
          lcp_index_free(ix);
          return r;
        }
        cudaMemset(ix->directory, 0, (size_t)(buckets + 1) * 8);
        dv.directory = ix->directory;
      }
    }
    *out = ix;
    return LCP_OK;
  }
  keep_pool_mapped();
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
    delete ix;
    return fail(LCP_ERR_CUDA, "cudaStreamCreate failed");
  }
  int r = build_impl(ix, rows, n, length, sigma, tal_depth, st);
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (r != LCP_OK) {
    std::string keep = g_err;
    lcp_index_free(ix);
    g_err = keep;
    return r;
  }
  *out = ix;
  return LCP_OK;
}

int lcp_index_get_info(const lcp_index* ix, lcp_index_info* info) {
  if (!ix || !info) return fail(LCP_ERR_INVALID_INPUT, "null argument");
  const DevIndex& dv = ix->dv;
  info->n = dv.n;
  info->length = dv.L;
  info->sigma = dv.sigma;
  info->bits = dv.b;
  info->syms_per_word = dv.spw;
  info->words = dv.W;
  info->search_levels = dv.nlevels + 1;
  info->tal_depth = ix->tal_depth;
  info->has_directory = ix->directory != nullptr;
  info->tal_buckets = ix->tal_buckets;
  info->device_bytes = ix->device_bytes;
  return LCP_OK;
}

static int copy_out(void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return LCP_OK;
  if (!dst) return fail(LCP_ERR_INVALID_INPUT, "destination must not be null");
  LCP_CK(cudaMemcpy(dst, src, bytes, cudaMemcpyDefault));
  return LCP_OK;
}

int lcp_index_export_order(const lcp_index* ix, int32_t* order) {
  if (!ix) return fail(LCP_ERR_INVALID_INPUT, "null index");
  return copy_out(order, ix->order, (size_t)ix->dv.n * 4);
}

int lcp_index_export_sorted_keys(const lcp_index* ix, uint64_t* keys) {
  if (!ix) return fail(LCP_ERR_INVALID_INPUT, "null index");
  return copy_out(keys, ix->keys, (size_t)ix->dv.n * ix->dv.W * 8);
}

int lcp_index_export_sorted_key_range(const lcp_index* ix, int64_t first, int64_t count,
                                      uint64_t* keys) {
  if (!ix) return fail(LCP_ERR_INVALID_INPUT, "null index");
  if (first < 0 || count < 0 || first + count > ix->dv.n)
    return fail(LCP_ERR_INVALID_INPUT, "sorted key range out of bounds");
  return copy_out(keys, ix->keys + first * ix->dv.W, (size_t)count * ix->dv.W * 8);
}

int lcp_index_export_adjacent_lcp(const lcp_index* ix, uint16_t* adj) {
  if (!ix) return fail(LCP_ERR_INVALID_INPUT, "null index");
  if (ix->dv.n <= 1) return LCP_OK;
  return copy_out(adj, ix->adj, (size_t)(ix->dv.n - 1) * 2);
}

int lcp_index_export_directory(const lcp_index* ix, int64_t* directory) {
  if (!ix) return fail(LCP_ERR_INVALID_INPUT, "null index");
  if (!ix->directory) return fail(LCP_ERR_STATE, "no dense TAL directory was built");
  return copy_out(directory, ix->directory, (size_t)(ix->tal_buckets + 1) * 8);
}

static int level_offsets(lcp_index* ix) {
  if (!ix->level_offset.empty()) return LCP_OK;
  const long long n = ix->dv.n;
  const int L = ix->dv.L;
  std::vector<long long> off(L + 2, 0);
  if (n == 0) {
    for (int d = 1; d < L + 2; ++d) off[d] = 1;  // trie.py:421 level_offset[1:] = 1
    ix->level_offset = off;
    return LCP_OK;
  }
  std::vector<unsigned long long> hist(L + 1, 0);
  if (n > 1) {
    unsigned long long* d_hist = nullptr;
    LCP_CK(cudaMalloc((void**)&d_hist, (L + 1) * sizeof(unsigned long long)));
    LCP_CK(cudaMemset(d_hist, 0, (L + 1) * sizeof(unsigned long long)));
    k_adj_hist<<<blocks_for(n - 1, 256), 256>>>(ix->adj, n - 1, d_hist);
    LCP_CK_LAUNCH();
    LCP_CK(cudaMemcpy(hist.data(), d_hist, (L + 1) * sizeof(unsigned long long),
                      cudaMemcpyDeviceToHost));
    cudaFree(d_hist);
  }
  off[0] = 0;
  off[1] = 1;
  unsigned long long below = 0;  // #adj < d
  for (int d = 1; d <= L; ++d) {
    below += hist[d - 1];
    off[d + 1] = off[d] + 1 + (long long)below;
  }
  ix->level_offset = off;
  return LCP_OK;
}

int lcp_index_trie_level_offsets(const lcp_index* cix, int64_t* level_offset) {
  if (!cix || !level_offset) return fail(LCP_ERR_INVALID_INPUT, "null argument");
  lcp_index* ix = const_cast<lcp_index*>(cix);
  LCP_TRY(level_offsets(ix));
  for (size_t i = 0; i < ix->level_offset.size(); ++i) level_offset[i] = ix->level_offset[i];
  return LCP_OK;
}

// Per-depth arena (row_lo, edge_symbol, level_offset) materialised on the
// device; the caller frees the three buffers.  n > 0.
static int arena_device(lcp_index* ix, int** d_row, uint16_t** d_edge, long long** d_off) {
  LCP_TRY(level_offsets(ix));
  const long long n = ix->dv.n;
  const int L = ix->dv.L;
  const long long nodes = ix->level_offset[L + 1];
  unsigned long long* d_cnt = nullptr;
  const int nblk = (int)blocks_for(n - 1 > 0 ? n - 1 : 1, TT_THREADS);
  LCP_CK(cudaMalloc((void**)d_row, (size_t)nodes * 4));
  LCP_CK(cudaMalloc((void**)d_edge, (size_t)nodes * 2));
  LCP_CK(cudaMalloc((void**)d_off, (size_t)(L + 2) * 8));
  LCP_CK(cudaMalloc((void**)&d_cnt, (size_t)nblk * L * 8));
  LCP_CK(cudaMemcpy(*d_off, ix->level_offset.data(), (size_t)(L + 2) * 8, cudaMemcpyHostToDevice));
  int root_row = 0;
  uint16_t root_sym = 0;
  LCP_CK(cudaMemcpy(*d_row, &root_row, 4, cudaMemcpyHostToDevice));
  LCP_CK(cudaMemcpy(*d_edge, &root_sym, 2, cudaMemcpyHostToDevice));
  dim3 grid(nblk, L);
  k_trie_count<<<grid, TT_THREADS>>>(ix->adj, n, nblk, d_cnt);
  LCP_CK_LAUNCH();
  LCP_TRY(scan_exclusive<unsigned long long>(d_cnt, (long long)nblk * L, 0));
  k_trie_scatter<<<grid, TT_THREADS>>>(ix->dv, ix->adj, nblk, d_cnt, *d_off, *d_row, *d_edge);
  LCP_CK_LAUNCH();
  LCP_CK(cudaDeviceSynchronize());
  cudaFree(d_cnt);
  return LCP_OK;
}

int lcp_index_export_trie(const lcp_index* cix, int32_t* row_lo, uint16_t* edge_symbol) {
  if (!cix) return fail(LCP_ERR_INVALID_INPUT, "null index");
  lcp_index* ix = const_cast<lcp_index*>(cix);
  LCP_TRY(level_offsets(ix));
  const long long n = ix->dv.n;
  const int L = ix->dv.L;
  const long long nodes = ix->level_offset[L + 1];
  if (n == 0) {
    int32_t z = 0;
    uint16_t zs = 0;
    LCP_TRY(copy_out(row_lo, &z, 4));
    LCP_TRY(copy_out(edge_symbol, &zs, 2));
    return LCP_OK;
  }
  int* d_row = nullptr;
  uint16_t* d_edge = nullptr;
  long long* d_off = nullptr;
  int r = arena_device(ix, &d_row, &d_edge, &d_off);
  if (r == LCP_OK) r = copy_out(row_lo, d_row, (size_t)nodes * 4);
  if (r == LCP_OK) r = copy_out(edge_symbol, d_edge, (size_t)nodes * 2);
  cudaFree(d_row);
  cudaFree(d_edge);
  cudaFree(d_off);
  return r;
}

int lcp_index_snapshot(const lcp_index* cix, uint8_t* out, int64_t* size) {
  if (!cix || !size) return fail(LCP_ERR_INVALID_INPUT, "null argument");
  lcp_index* ix = const_cast<lcp_index*>(cix);
  LCP_TRY(level_offsets(ix));
  const long long n = ix->dv.n;
  const int L = ix->dv.L;
  const long long nodes = ix->level_offset[L + 1];
  // header (storage.py:44, "<4sH6BQIIQ"): magic version widths[6] n length sigma node_count
  unsigned char header[36];
  memcpy(header, "LCPI", 4);
  const uint16_t version = 1;
  memcpy(header + 4, &version, 2);
  const unsigned char widths[6] = {2, 4, 4, 2, 4, 2};  // storage.py:45
  memcpy(header + 6, widths, 6);
  const uint64_t n64 = (uint64_t)n, nodes64 = (uint64_t)nodes;
  const uint32_t len32 = (uint32_t)L, sig32 = (uint32_t)ix->dv.sigma;
  memcpy(header + 12, &n64, 8);
  memcpy(header + 20, &len32, 4);
  memcpy(header + 24, &sig32, 4);
  memcpy(header + 28, &nodes64, 8);
  if (n == 0) {  // a bare root: depth 0, no posting, no children
    const long long total = 36 + 8;
    if (!out) {
      *size = total;
      return LCP_OK;
    }
    if (*size < total) return fail(LCP_ERR_INVALID_INPUT, "snapshot buffer too small");
    unsigned char rec[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    LCP_TRY(copy_out(out, header, 36));
    LCP_TRY(copy_out(out + 36, rec, 8));
    *size = total;
    return LCP_OK;
  }
  int* d_row = nullptr;
  uint16_t* d_edge = nullptr;
  long long* d_off = nullptr;
  LCP_TRY(arena_device(ix, &d_row, &d_edge, &d_off));
  unsigned long long* d_start = nullptr;
  LCP_CK(cudaMalloc((void**)&d_start, (size_t)(nodes + 1) * 8));
  LCP_CK(cudaMemset(d_start + nodes, 0, 8));
  k_snap_sizes<<<blocks_for(nodes, 256), 256>>>(d_row, d_off, nodes, n, L, d_start);
  LCP_CK_LAUNCH();
  LCP_TRY(scan_exclusive<unsigned long long>(d_start, nodes + 1, 0));
  unsigned long long body = 0;
  LCP_CK(cudaMemcpy(&body, d_start + nodes, 8, cudaMemcpyDeviceToHost));
  const long long total = 36 + (long long)body;
  int r = LCP_OK;
  if (!out) {
    *size = total;
  } else if (*size < total) {
    r = fail(LCP_ERR_INVALID_INPUT, "snapshot buffer too small");
  } else {
    unsigned char* d_out = nullptr;
    if (cudaMalloc((void**)&d_out, (size_t)total) != cudaSuccess) {
      r = fail(LCP_ERR_CUDA, "cudaMalloc for the snapshot failed");
    } else {
      cudaMemcpy(d_out, header, 36, cudaMemcpyHostToDevice);
      k_snap_headers<<<blocks_for(nodes, 256), 256>>>(d_row, d_off, d_start, nodes, n, L, d_out + 36);
      if (nodes > 1)
        k_snap_children<<<blocks_for(nodes - 1, 256), 256>>>(d_row, d_edge, d_off, d_start, nodes, L,
                                                             d_out + 36);
      k_snap_postings<<<blocks_for(n, 256), 256>>>(d_row, d_off, d_start, ix->order, n, L, d_out + 36);
      if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
        r = fail(LCP_ERR_CUDA, "snapshot kernels failed");
      if (r == LCP_OK) r = copy_out(out, d_out, (size_t)total);
      cudaFree(d_out);
      *size = total;
    }
  }
  cudaFree(d_start);
  cudaFree(d_row);
  cudaFree(d_edge);
  cudaFree(d_off);
  return r;
}

}  // extern "C"

// Host-side reader of an LCPI snapshot (storage.py:226-389): validates the
// stream like the reference, recovers the dataset rows from the arena (each
// depth-d node's edge symbol is symbol d-1 of every row it covers), rebuilds
// the index on the GPU and checks the rebuilt snapshot is byte-identical.
int lcp_index_from_snapshot(const uint8_t* raw, int64_t size, lcp_index** out) {
  if (!raw || !out) return fail(LCP_ERR_INVALID_INPUT, "null argument");
  *out = nullptr;
  auto rd16 = [&](long long p) { return (unsigned)raw[p] | ((unsigned)raw[p + 1] << 8); };
  auto rd32 = [&](long long p) {
    return (unsigned long long)raw[p] | ((unsigned long long)raw[p + 1] << 8) |
           ((unsigned long long)raw[p + 2] << 16) | ((unsigned long long)raw[p + 3] << 24);
  };
  if (size < 36) return fail(LCP_ERR_INVALID_INPUT, "truncated index header");
  if (memcmp(raw, "LCPI", 4) != 0) return fail(LCP_ERR_INVALID_INPUT, "not an index snapshot (bad magic)");
  if (rd16(4) != 1) return fail(LCP_ERR_INVALID_INPUT, "unsupported snapshot version " + std::to_string(rd16(4)));
  const unsigned char widths[6] = {2, 4, 4, 2, 4, 2};
  if (memcmp(raw + 6, widths, 6) != 0) return fail(LCP_ERR_INVALID_INPUT, "unsupported field widths");
  unsigned long long n64, nodes64;
  uint32_t L32, sig32;
  memcpy(&n64, raw + 12, 8);
  memcpy(&L32, raw + 20, 4);
  memcpy(&sig32, raw + 24, 4);
  memcpy(&nodes64, raw + 28, 8);
  const long long n = (long long)n64, nodes = (long long)nodes64;
  const int L = (int)L32;
  if (n < 0 || n >= (1ll << 31) || L < 1 || L > 65535 || sig32 < 2 || sig32 > 65536)
    return fail(LCP_ERR_INVALID_INPUT, "snapshot header out of range");
  // walk the records level by level
  std::vector<long long> lvl_count, rec_start;
  std::vector<unsigned> ccs, plens;
  std::vector<uint16_t> edge(std::max(1ll, nodes), 0);
  long long pos = 36, parsed = 0, expected = 1, next_id = 1;
  while (parsed < nodes) {
    const int d = (int)lvl_count.size();
    for (long long i = 0; i < expected; ++i) {
      if (pos + 8 > size) return fail(LCP_ERR_INVALID_INPUT, "truncated node record at byte " + std::to_string(pos));
      const unsigned depth = rd16(pos);
      const unsigned long long plen = rd32(pos + 2);
      const long long cc_at = pos + 6 + 4 * (long long)plen;
      if (cc_at + 2 > size) return fail(LCP_ERR_INVALID_INPUT, "truncated posting list at byte " + std::to_string(pos));
      const unsigned cc = rd16(cc_at);
      if ((int)depth != d) return fail(LCP_ERR_INVALID_INPUT, "expected depth " + std::to_string(d) + ", found " + std::to_string(depth));
      if (cc_at + 2 + 6ll * cc > size) return fail(LCP_ERR_INVALID_INPUT, "truncated child list at byte " + std::to_string(pos));
      for (unsigned c = 0; c < cc; ++c) {
        const long long e = cc_at + 2 + 6ll * c;
        const unsigned long long cid = rd32(e + 2);
        if ((long long)cid != next_id || next_id >= nodes)
          return fail(LCP_ERR_INVALID_INPUT, "child ids at depth " + std::to_string(d) + " are not the next level");
        edge[next_id++] = (uint16_t)rd16(e);
      }
      rec_start.push_back(pos);
      plens.push_back((unsigned)plen);
      ccs.push_back(cc);
      pos = cc_at + 2 + 6ll * cc;
    }
    lvl_count.push_back(expected);
    parsed += expected;
    long long nxt = 0;
    for (long long i = parsed - expected; i < parsed; ++i) nxt += ccs[i];
    expected = nxt;
    if (expected == 0) break;
  }
  if (parsed != nodes)
    return fail(LCP_ERR_INVALID_INPUT, "header claims " + std::to_string(nodes) + " nodes, file holds " + std::to_string(parsed));
  if (pos != size) return fail(LCP_ERR_INVALID_INPUT, std::to_string(size - pos) + " trailing bytes");
  const int depths = (int)lvl_count.size() - 1;
  if (depths > L) return fail(LCP_ERR_INVALID_INPUT, "node depth exceeds declared length");
  if (n > 0 && depths != L) return fail(LCP_ERR_INVALID_INPUT, "leaf level is not at full depth");
  // postings of the last level form the sort permutation
  std::vector<long long> lvl_off(lvl_count.size() + 1, 0);
  for (size_t d = 0; d < lvl_count.size(); ++d) lvl_off[d + 1] = lvl_off[d] + lvl_count[d];
  std::vector<uint32_t> order;
  order.reserve(n);
  const size_t leaf0 = lvl_off[depths];
  for (size_t v = leaf0; v < (size_t)parsed; ++v)
    for (unsigned j = 0; j < plens[v]; ++j) order.push_back((uint32_t)rd32(rec_start[v] + 6 + 4ll * j));
  if ((long long)order.size() != n)
    return fail(LCP_ERR_INVALID_INPUT, "posting lists hold " + std::to_string(order.size()) + " items, header claims " + std::to_string(n));
  std::vector<char> seen(std::max(1ll, n), 0);
  for (uint32_t id : order) {
    if ((long long)id >= n || seen[id]) return fail(LCP_ERR_INVALID_INPUT, "posting ids are not a permutation");
    seen[id] = 1;
  }
  if (n == 0) return lcp_index_build(nullptr, 0, L, (int)sig32, -1, out);
  // subtree sizes bottom-up -> each node's row range; rows from the paths
  std::vector<long long> sz(parsed, 0);
  for (size_t v = leaf0; v < (size_t)parsed; ++v) sz[v] = plens[v];
  for (int d = depths - 1; d >= 0; --d) {
    long long child = lvl_off[d + 1];
    for (long long v = lvl_off[d]; v < lvl_off[d + 1]; ++v) {
      if (ccs[v] < 1) return fail(LCP_ERR_INVALID_INPUT, "childless interior node at depth " + std::to_string(d));
      long long t = 0;
      for (unsigned c = 0; c < ccs[v]; ++c) t += sz[child++];
      sz[v] = t;
    }
  }
  std::vector<uint16_t> items((size_t)n * L);
  for (int d = 1; d <= depths; ++d) {
    long long row = 0;
    for (long long v = lvl_off[d]; v < lvl_off[d + 1]; ++v) {
      if (edge[v] >= sig32) return fail(LCP_ERR_INVALID_INPUT, "edge symbol out of range for the alphabet");
      for (long long r = row; r < row + sz[v]; ++r) items[(size_t)order[r] * L + d - 1] = edge[v];
      row += sz[v];
    }
  }
  lcp_index* ix = nullptr;
  LCP_TRY(lcp_index_build(items.data(), n, L, (int)sig32, -1, &ix));
  // integrity: the rebuilt index must serialise to exactly these bytes
  int64_t rsize = 0;
  int r = lcp_index_snapshot(ix, nullptr, &rsize);
  if (r == LCP_OK && rsize != size) r = fail(LCP_ERR_INVALID_INPUT, "snapshot is not canonical (size mismatch)");
  if (r == LCP_OK) {
    std::vector<uint8_t> again((size_t)rsize);
    r = lcp_index_snapshot(ix, again.data(), &rsize);
    if (r == LCP_OK && memcmp(again.data(), raw, (size_t)size) != 0)
      r = fail(LCP_ERR_INVALID_INPUT, "snapshot is not canonical (rebuilt bytes differ)");
  }
  if (r != LCP_OK) {
    std::string keep = g_err;
    lcp_index_free(ix);
    g_err = keep;
    return r;
  }
  *out = ix;
  return LCP_OK;
}

__global__ void k_bucket_search(DevIndex ix, const u64* __restrict__ qkeys, int count,
                                long long* __restrict__ lo, long long* __restrict__ hi) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= count) return;
  const u64* qk = qkeys + (long long)q * ix.W;
  int d = ix.tal_depth;
  lo[q] = d ? prefix_bound(ix, qk, d, false) : 0;
  hi[q] = d ? prefix_bound(ix, qk, d, true) : ix.n;
}

extern "C" {

int lcp_index_bucket_range_search(const lcp_index* ix, const uint16_t* queries, int32_t count,
                                  int64_t* lo, int64_t* hi) {
  if (!ix) return fail(LCP_ERR_INVALID_INPUT, "null index");
  if (ix->tal_depth < 0) return fail(LCP_ERR_STATE, "index has no TAL bucket structure");
  if (count <= 0) return LCP_OK;
  const DevIndex& dv = ix->dv;
  if (dv.n == 0) {
    for (int i = 0; i < count; ++i) lo[i] = hi[i] = 0;
    return LCP_OK;
  }
  uint16_t* d_q = nullptr;
  u64* d_k = nullptr;
  long long *d_lo = nullptr, *d_hi = nullptr;
  int* d_err = nullptr;
  LCP_CK(cudaMalloc((void**)&d_q, (size_t)count * dv.L * 2));
  LCP_CK(cudaMalloc((void**)&d_k, (size_t)count * dv.W * 8));
  LCP_CK(cudaMalloc((void**)&d_lo, (size_t)count * 8));
  LCP_CK(cudaMalloc((void**)&d_hi, (size_t)count * 8));
  LCP_CK(cudaMalloc((void**)&d_err, 4));
  LCP_CK(cudaMemset(d_err, 0, 4));
  LCP_CK(cudaMemcpy(d_q, queries, (size_t)count * dv.L * 2, cudaMemcpyDefault));
  LCP_TRY(pack_rows(d_q, count, dv, d_k, nullptr, d_err, (cudaStream_t)0));
  k_bucket_search<<<blocks_for(count, 128), 128>>>(dv, d_k, count, d_lo, d_hi);
  LCP_CK_LAUNCH();
  int h_err = 0;
  LCP_CK(cudaMemcpy(&h_err, d_err, 4, cudaMemcpyDeviceToHost));
  int r = LCP_OK;
  if (h_err)
    r = fail(LCP_ERR_INVALID_INPUT,
             "query symbol out of range for alphabet of size " + std::to_string(dv.sigma));
  if (r == LCP_OK) r = copy_out(lo, d_lo, (size_t)count * 8);
  if (r == LCP_OK) r = copy_out(hi, d_hi, (size_t)count * 8);
  cudaFree(d_q);
  cudaFree(d_k);
  cudaFree(d_lo);
  cudaFree(d_hi);
  cudaFree(d_err);
  return r;
}

// ---- workspace --------------------------------------------------------------
int lcp_workspace_create(lcp_workspace** out) {
  if (!out) return fail(LCP_ERR_INVALID_INPUT, "out must not be null");
  lcp_workspace* ws = new lcp_workspace();
  cudaError_t e = cudaStreamCreateWithFlags(&ws->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc((void**)&ws->d_err, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(ws->d_err, 0, sizeof(int));
  if (e == cudaSuccess) e = cudaHostAlloc((void**)&ws->h_err, sizeof(int), cudaHostAllocDefault);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ws->done, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    delete ws;
    return fail(LCP_ERR_CUDA, std::string("workspace: ") + cudaGetErrorString(e));
  }
  *ws->h_err = 0;
  *out = ws;
  return LCP_OK;
}

int lcp_workspace_free(lcp_workspace* ws) {
  if (!ws) return LCP_OK;
  if (ws->stream) cudaStreamSynchronize(ws->stream);
  for (auto& g : ws->graphs) cudaGraphExecDestroy(g.exec);
  ws->graphs.clear();
  for (DBuf* b : {&ws->qkeys, &ws->partial, &ws->hint, &ws->q_in, &ws->ids, &ws->lcps, &ws->hits,
                  &ws->md, &ws->aux})
    b->release();
  cudaFree(ws->d_err);
  cudaFreeHost(ws->h_err);
  if (ws->done) cudaEventDestroy(ws->done);
  if (ws->stream) cudaStreamDestroy(ws->stream);
  delete ws;
  return LCP_OK;
}

void* lcp_workspace_stream(lcp_workspace* ws) { return ws ? (void*)ws->stream : nullptr; }

int lcp_workspace_check(lcp_workspace* ws, void* stream) {
  if (!ws) return fail(LCP_ERR_INVALID_INPUT, "null workspace");
  cudaStream_t st = (cudaStream_t)stream;
  LCP_CK(cudaMemcpyAsync(ws->h_err, ws->d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
  LCP_CK(cudaStreamSynchronize(st));
  if (*ws->h_err) {
    *ws->h_err = 0;
    LCP_CK(cudaMemsetAsync(ws->d_err, 0, sizeof(int), st));
    LCP_CK(cudaStreamSynchronize(st));
    return fail(LCP_ERR_INVALID_INPUT, "query symbol out of range for alphabet");
  }
  return LCP_OK;
}

}  // extern "C"

__global__ void k_fill_empty(int count, int md, int* hits, uint16_t* out_md, u64* aux) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  hits[i] = 0;
  if (out_md) out_md[i] = (uint16_t)md;
  if (aux) {
    aux[2 * i] = 0;
    aux[2 * i + 1] = 0;
  }
}

// Reserve enough shared memory that two query CTAs (two batches in flight)
// fit on one SM; the default carve-out for a 4 KB-smem kernel admits one.
// preferred L1 / shared split, set once per kernel (the static is per kernel)
template <auto Kernel>
static void prefer_carveout(int pct) {
  static const bool done = [pct] {  // thread-safe one-time initialisation
    cudaFuncSetAttribute(Kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaGetLastError();
    return true;
  }();
  (void)done;
}

// opt in to more than 48 KB of dynamic shared memory, once per kernel
template <auto Kernel>
static void allow_dyn_smem() {
  static const bool done = [] {  // thread-safe one-time initialisation
    cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaGetLastError();
    return true;
  }();
  (void)done;
}

template <typename C, int T>
static void launch_w1(const DevIndex& dv, int mode, unsigned grid, unsigned block, size_t smem,
                      cudaStream_t st, const uint16_t* q, int count, int k, int stride, u32* ids,
                      uint16_t* lcps, int* hits, uint16_t* md, u64* aux, int* err) {
  // strict / complete keep 25 % shared memory (two 1024-thread batches per SM);
  // TAL wants the largest L1 for the grouped bucket sweep
  prefer_carveout<k_query_w1<C, T, 0>>(25);
  prefer_carveout<k_query_w1<C, T, 1>>(25);
  prefer_carveout<k_query_w1<C, T, 2>>(0);
  if (mode == LCP_MODE_STRICT)
    k_query_w1<C, T, 0><<<grid, block, smem, st>>>(dv, q, count, k, stride, ids, lcps, hits, md, aux, err);
  else if (mode == LCP_MODE_COMPLETE)
    k_query_w1<C, T, 1><<<grid, block, smem, st>>>(dv, q, count, k, stride, ids, lcps, hits, md, aux, err);
  else
    k_query_w1<C, T, 2><<<grid, block, smem, st>>>(dv, q, count, k, stride, ids, lcps, hits, md, aux, err);
}

template <int WMAX>
static void launch_fast(const DevIndex& dv, const uint16_t* q, int count, int gcount, int k, int mode,
                        int stride, u32* ids, uint16_t* lcps, int* hits, uint16_t* md, u64* aux,
                        int* err, cudaStream_t st, lcp_workspace* ws) {
  if (mode == LCP_MODE_TAL && WMAX > 1) {
    const long long sms = num_sms();
    const long long wpc = std::min<long long>(32, std::max<long long>(1, (gcount + sms - 1) / sms));
    const unsigned block = (unsigned)(wpc * 32);
    const unsigned grid = (unsigned)std::min<long long>((gcount + wpc - 1) / wpc, 4ll * sms);
    const size_t smem = 16 + (size_t)dv.smem_entries * 8;
    k_query_warp_tal<WMAX><<<grid, block, smem, st>>>(dv, q, count, k, stride, ids, lcps, hits, md,
                                                      aux, err);
  } else {
    // One query per warp; spread the batch evenly over the SMs with one CTA
    // per SM (so each SM stages the search levels once), up to 1024 threads;
    // larger batches get more CTAs (2 x 1024 threads fit an SM).
    const long long sms = num_sms();
    static const long long wpc_min = [] {  // LCP_WPC_MIN: A/B hook (warps per CTA floor)
      const char* e = getenv("LCP_WPC_MIN");
      return e ? std::max(1ll, std::min(32ll, atoll(e))) : 1ll;
    }();
    static const long long qpw = [] {  // LCP_QPW: A/B hook (queries per warp)
      const char* e = getenv("LCP_QPW");
      return e ? std::max(1ll, std::min(16ll, atoll(e))) : 1ll;
    }();
    const long long units = (gcount + qpw - 1) / qpw;
    static const long long wpc_max = [] {  // LCP_WPC_MAX: A/B hook (warps per CTA cap)
      const char* e = getenv("LCP_WPC_MAX");
      return e ? std::max(1ll, std::min(32ll, atoll(e))) : 32ll;
    }();
    long long wpc = std::min<long long>(wpc_max, std::max<long long>(wpc_min, (units + sms - 1) / sms));
    const unsigned block = (unsigned)(wpc * 32);
    unsigned grid = (unsigned)std::min<long long>((units + wpc - 1) / wpc, 4ll * sms);
    size_t smem = 16 + (size_t)dv.smem_entries * 8;
    if constexpr (WMAX == 1) {
      // leaf region: 64 keys cover the +-need window for need <= 16, 96 keys for <= 32
      const long long need = mode == LCP_MODE_COMPLETE ? std::min<long long>(k, dv.n) : k;
      if (dv.idbits < 32) {
        if (need <= 16) launch_w1<u32, 2>(dv, mode, grid, block, smem, st, q, count, k, stride, ids, lcps, hits, md, aux, err);
        else launch_w1<u32, 3>(dv, mode, grid, block, smem, st, q, count, k, stride, ids, lcps, hits, md, aux, err);
      } else {
        if (need <= 16) launch_w1<u64, 2>(dv, mode, grid, block, smem, st, q, count, k, stride, ids, lcps, hits, md, aux, err);
        else launch_w1<u64, 3>(dv, mode, grid, block, smem, st, q, count, k, stride, ids, lcps, hits, md, aux, err);
      }
    }
    else
      k_query_warp<WMAX><<<grid, block, smem, st>>>(dv, q, count, k, mode, stride, ids,
                                                         lcps, hits, md, aux, err);
  }
}

extern "C" {

}  // extern "C"

// lcp_query's body; `errp` is the device int the kernels raise on an invalid
// query symbol (the workspace's flag, or a slot of a packed output block)
// `dcount` (device int, may be null) caps the batch on the device: `count` is
// then the capacity of the buffers and `gcount` the expected size the grids
// are sized for (the kernels' grid-stride loops cover any count up to capacity)
static int query_impl(const lcp_index* ix, lcp_workspace* ws, const uint16_t* queries,
                      int32_t count, int32_t k, int32_t mode, int32_t out_stride, uint32_t* ids,
                      uint16_t* lcps, int32_t* hits, uint16_t* matched_depth, uint64_t* aux,
                      void* stream, int* errp, const int* dcount = nullptr, int gcount = -1) {
  if (!ix || !ws) return fail(LCP_ERR_INVALID_INPUT, "null index or workspace");
  if (k < 1) return fail(LCP_ERR_INVALID_INPUT, "k must be >= 1, got " + std::to_string(k));
  if (mode < 0 || mode > 2)
    return fail(LCP_ERR_INVALID_INPUT, "mode must be 'strict', 'complete' or 'tal', got " +
                                           std::to_string(mode));
  if (mode == LCP_MODE_TAL && ix->tal_depth < 0)
    return fail(LCP_ERR_STATE, "index was built without a TAL bucket structure");
  DevIndex dvl = ix->dv;
  dvl.dcount = dcount;
  const DevIndex& dv = dvl;
  if (count < 0) return fail(LCP_ERR_INVALID_INPUT, "count must be >= 0");
  if (!dcount || gcount < 1 || gcount > count) gcount = count;
  if (count == 0) return LCP_OK;
  const long long need_stride = std::min<long long>(k, std::max(1ll, dv.n));
  if (out_stride < need_stride)
    return fail(LCP_ERR_INVALID_INPUT, "out_stride must be >= min(k, n)");
  if (!queries || !hits) return fail(LCP_ERR_INVALID_INPUT, "null query or output buffer");
  cudaStream_t st = (cudaStream_t)stream;
  if (dv.n == 0) {
    k_fill_empty<<<blocks_for(count, 256), 256, 0, st>>>(
        count, mode == LCP_MODE_TAL ? ix->tal_depth : 0, hits, matched_depth, reinterpret_cast<u64*>(aux));
    LCP_CK_LAUNCH();
    return LCP_OK;
  }
  // matched_depth / aux are optional for callers; route to scratch if absent
  uint16_t* md = matched_depth;
  u64* ax = reinterpret_cast<u64*>(aux);
  if (!md) {
    LCP_TRY(ws->md.ensure((size_t)count * 2));
    md = ws->md.as<uint16_t>();
  }
  if (!ax) {
    LCP_TRY(ws->aux.ensure((size_t)count * 16));
    ax = ws->aux.as<u64>();
  }
  const long long needk = mode == LCP_MODE_COMPLETE ? std::min<long long>(k, dv.n) : k;
  static const int kn_min = [] {  // A/B hook: smallest need on the list kernel (default 17)
    const char* e = getenv("LCP_KN_MIN");
    return e ? std::max(1, atoi(e)) : 17;
  }();
  const bool kn_ok = needk >= kn_min;
  if (dv.W == 1 && kn_ok && needk <= 128) {
    // 16 < need <= 128 (strict, complete, TAL): warp per query with a 1-, 2-
    // or 4-slot top-k list.  At need 17..32 it beats the T=3 rank kernel
    // (complete 11.1 vs 14.3-15.6 us, TAL 28.6 vs 33.3 us per 4096 batch),
    // which now runs only when LCP_KN_MIN raises the threshold
    const long long sms = num_sms();
    const long long wmax = needk <= 64 ? 32 : 16;  // 4-slot lists: 512-thread CTAs
    const long long wpc = std::min<long long>(wmax, std::max<long long>(1, (gcount + sms - 1) / sms));
    const unsigned block = (unsigned)(wpc * 32);
    const unsigned grid = (unsigned)std::min<long long>((gcount + wpc - 1) / wpc, 8ll * sms);
    // staged levels, then one 32 * NS-entry merge buffer per warp
    const size_t smem0 = 16 + (size_t)dv.smem_entries * 8;
#define LCP_KN(C, M, NS)                                                                         \
  do {                                                                                           \
    allow_dyn_smem<k_query_w1_kn<C, M, NS>>();                                                   \
    k_query_w1_kn<C, M, NS><<<grid, block, smem0 + (size_t)wpc * 32 * NS * sizeof(C), st>>>(    \
        dv, queries, count, k, out_stride, ids, lcps, hits, md, ax, errp);                       \
  } while (0)
    const bool strict = mode == LCP_MODE_STRICT, tal = mode == LCP_MODE_TAL;
    if (dv.idbits < 32) {
      if (needk <= 32) { if (tal) LCP_KN(u32, 2, 1); else if (strict) LCP_KN(u32, 0, 1); else LCP_KN(u32, 1, 1); }
      else if (needk <= 64) { if (tal) LCP_KN(u32, 2, 2); else if (strict) LCP_KN(u32, 0, 2); else LCP_KN(u32, 1, 2); }
      else { if (tal) LCP_KN(u32, 2, 4); else if (strict) LCP_KN(u32, 0, 4); else LCP_KN(u32, 1, 4); }
    } else {
      if (needk <= 32) { if (tal) LCP_KN(u64, 2, 1); else if (strict) LCP_KN(u64, 0, 1); else LCP_KN(u64, 1, 1); }
      else if (needk <= 64) { if (tal) LCP_KN(u64, 2, 2); else if (strict) LCP_KN(u64, 0, 2); else LCP_KN(u64, 1, 2); }
      else { if (tal) LCP_KN(u64, 2, 4); else if (strict) LCP_KN(u64, 0, 4); else LCP_KN(u64, 1, 4); }
    }
#undef LCP_KN
    LCP_CK_LAUNCH();
    return LCP_OK;
  }
  if (dv.W > 1 && dv.W <= 8 && needk > FAST_KMAX && needk <= 128) {
    // 32 < need <= 128, W > 1 (strict, complete, TAL): warp per query with a
    // 2- or 4-slot list
    const long long sms = num_sms();
    const long long wmax = needk <= 64 ? 32 : 16;  // 4-slot lists: 512-thread CTAs
    const long long wpc = std::min<long long>(wmax, std::max<long long>(1, (gcount + sms - 1) / sms));
    const unsigned block = (unsigned)(wpc * 32);
    const unsigned grid = (unsigned)std::min<long long>((gcount + wpc - 1) / wpc, 8ll * sms);
    const size_t smem0 = 16 + (size_t)dv.smem_entries * 8;
#define LCP_WKN1(WM, NS, TL)                                                                     \
  do {                                                                                           \
    allow_dyn_smem<k_query_warp_kn<WM, NS, TL>>();                                               \
    k_query_warp_kn<WM, NS, TL><<<grid, block, smem0 + (size_t)wpc * 32 * NS * 8, st>>>(        \
        dv, queries, count, k, mode, out_stride, ids, lcps, hits, md, ax, errp);                 \
  } while (0)
#define LCP_WKN(WM, NS) \
  do { if (mode == LCP_MODE_TAL) LCP_WKN1(WM, NS, true); else LCP_WKN1(WM, NS, false); } while (0)
    if (needk <= 64) {
      if (dv.W == 2) LCP_WKN(2, 2); else if (dv.W <= 4) LCP_WKN(4, 2); else LCP_WKN(8, 2);
    } else {
      if (dv.W == 2) LCP_WKN(2, 4); else if (dv.W <= 4) LCP_WKN(4, 4); else LCP_WKN(8, 4);
    }
#undef LCP_WKN
#undef LCP_WKN1
    LCP_CK_LAUNCH();
    return LCP_OK;
  }
  if (dv.W <= 8 && k <= FAST_KMAX) {
    if (dv.W == 1) launch_fast<1>(dv, queries, count, gcount, k, mode, out_stride, ids, lcps, hits, md, ax, errp, st, ws);
    else if (dv.W == 2) launch_fast<2>(dv, queries, count, gcount, k, mode, out_stride, ids, lcps, hits, md, ax, errp, st, ws);
    else if (dv.W <= 4) launch_fast<4>(dv, queries, count, gcount, k, mode, out_stride, ids, lcps, hits, md, ax, errp, st, ws);
    else launch_fast<8>(dv, queries, count, gcount, k, mode, out_stride, ids, lcps, hits, md, ax, errp, st, ws);
    LCP_CK_LAUNCH();
    return LCP_OK;
  }
  LCP_TRY(ws->qkeys.ensure((size_t)count * dv.W * 8));
  LCP_TRY(pack_rows(queries, count, dv, ws->qkeys.as<u64>(), nullptr, errp, st));
  if (dv.W > 8 && mode != LCP_MODE_TAL && k <= FAST_KMAX) {  // long keys: warp per query
    const long long sms = num_sms();
    const long long wpc = std::min<long long>(32, std::max<long long>(1, (gcount + sms - 1) / sms));
    const unsigned grid = (unsigned)std::min<long long>((gcount + wpc - 1) / wpc, 8ll * sms);
    k_query_warp_any<<<grid, (unsigned)(wpc * 32), 0, st>>>(dv, ws->qkeys.as<u64>(), count, k, mode,
                                                            out_stride, ids, lcps, hits, md, ax);
    LCP_CK_LAUNCH();
    return LCP_OK;
  }
  if (dv.W > 8 && mode != LCP_MODE_TAL && needk > FAST_KMAX && needk <= 128) {  // long keys, lists
    const long long sms = num_sms();
    const long long wmax = needk <= 64 ? 32 : 16;  // 4-slot lists: 512-thread CTAs
    const long long wpc = std::min<long long>(wmax, std::max<long long>(1, (gcount + sms - 1) / sms));
    const unsigned grid = (unsigned)std::min<long long>((gcount + wpc - 1) / wpc, 8ll * sms);
    if (needk <= 64) {
      allow_dyn_smem<k_query_warp_any_kn<2>>();
      k_query_warp_any_kn<2><<<grid, (unsigned)(wpc * 32), (size_t)wpc * 64 * 8, st>>>(
          dv, ws->qkeys.as<u64>(), count, k, mode, out_stride, ids, lcps, hits, md, ax);
    } else {
      allow_dyn_smem<k_query_warp_any_kn<4>>();
      k_query_warp_any_kn<4><<<grid, (unsigned)(wpc * 32), (size_t)wpc * 128 * 8, st>>>(
          dv, ws->qkeys.as<u64>(), count, k, mode, out_stride, ids, lcps, hits, md, ax);
    }
    LCP_CK_LAUNCH();
    return LCP_OK;
  }
  unsigned grid = (unsigned)gen_grid(gcount);
  k_query_general<<<grid, GEN_THREADS, 0, st>>>(dv, ws->qkeys.as<u64>(), queries, count, k, mode,
                                                0, out_stride, ids, lcps, hits, md, ax);
  LCP_CK_LAUNCH();
  return LCP_OK;
}

extern "C" {

int lcp_query(const lcp_index* ix, lcp_workspace* ws, const uint16_t* queries, int32_t count,
              int32_t k, int32_t mode, int32_t out_stride, uint32_t* ids, uint16_t* lcps,
              int32_t* hits, uint16_t* matched_depth, uint64_t* aux, void* stream) {
  if (!ws) return fail(LCP_ERR_INVALID_INPUT, "null index or workspace");
  return query_impl(ix, ws, queries, count, k, mode, out_stride, ids, lcps, hits, matched_depth,
                    aux, stream, ws->d_err);
}

static int host_finish(lcp_workspace* ws) {
  LCP_CK(cudaMemcpyAsync(ws->h_err, ws->d_err, sizeof(int), cudaMemcpyDeviceToHost, ws->stream));
  LCP_CK(cudaStreamSynchronize(ws->stream));
  if (*ws->h_err) {
    *ws->h_err = 0;
    LCP_CK(cudaMemsetAsync(ws->d_err, 0, sizeof(int), ws->stream));
    LCP_CK(cudaStreamSynchronize(ws->stream));
    return LCP_ERR_INVALID_INPUT;
  }
  return LCP_OK;
}

int lcp_query_host(const lcp_index* ix, lcp_workspace* ws, const uint16_t* queries, int32_t count,
                   int32_t k, int32_t mode, int32_t out_stride, uint32_t* ids, uint16_t* lcps,
                   int32_t* hits, uint16_t* matched_depth, uint64_t* aux) {
  if (!ix || !ws) return fail(LCP_ERR_INVALID_INPUT, "null index or workspace");
  if (count <= 0) return lcp_query(ix, ws, queries, count, k, mode, out_stride, ids, lcps, hits,
                                   matched_depth, aux, ws->stream);
  const DevIndex& dv = ix->dv;
  cudaStream_t st = ws->stream;
  const size_t qb = (size_t)count * dv.L * 2;
  const size_t ob = (size_t)count * std::max(1, out_stride);
  LCP_TRY(ws->q_in.ensure(qb));
  LCP_TRY(ws->ids.ensure(ob * 4));
  LCP_TRY(ws->lcps.ensure(ob * 2));
  LCP_TRY(ws->hits.ensure((size_t)count * 4));
  LCP_TRY(ws->md.ensure((size_t)count * 2));
  LCP_TRY(ws->aux.ensure((size_t)count * 16));
  LCP_CK(cudaMemcpyAsync(ws->q_in.p, queries, qb, cudaMemcpyHostToDevice, st));
  LCP_TRY(lcp_query(ix, ws, ws->q_in.as<uint16_t>(), count, k, mode, out_stride,
                    ws->ids.as<u32>(), ws->lcps.as<uint16_t>(), ws->hits.as<int>(),
                    ws->md.as<uint16_t>(), reinterpret_cast<uint64_t*>(ws->aux.as<u64>()), st));
  if (ids) LCP_CK(cudaMemcpyAsync(ids, ws->ids.p, ob * 4, cudaMemcpyDeviceToHost, st));
  if (lcps) LCP_CK(cudaMemcpyAsync(lcps, ws->lcps.p, ob * 2, cudaMemcpyDeviceToHost, st));
  LCP_CK(cudaMemcpyAsync(hits, ws->hits.p, (size_t)count * 4, cudaMemcpyDeviceToHost, st));
  if (matched_depth)
    LCP_CK(cudaMemcpyAsync(matched_depth, ws->md.p, (size_t)count * 2, cudaMemcpyDeviceToHost, st));
  if (aux) LCP_CK(cudaMemcpyAsync(aux, ws->aux.p, (size_t)count * 16, cudaMemcpyDeviceToHost, st));
  if (host_finish(ws) != LCP_OK)
    return fail(LCP_ERR_INVALID_INPUT,
                "query symbol out of range for alphabet of size " + std::to_string(dv.sigma));
  return LCP_OK;
}

static lcp_packed_layout packed_layout(long long count, long long stride) {
  auto up8 = [](long long v) { return (v + 7) & ~7ll; };
  lcp_packed_layout l;
  l.ids = 0;
  l.lcps = up8(count * stride * 4);
  l.hits = up8(l.lcps + count * stride * 2);
  l.err = up8(l.hits + count * 4);  // rides in the same D2H copy as the results
  l.matched_depth = l.err + 8;
  l.aux = up8(l.matched_depth + count * 2);
  l.total = l.aux + count * 16;
  return l;
}

int lcp_packed_layout_for(int32_t count, int32_t out_stride, lcp_packed_layout* layout) {
  if (!layout || count < 0 || out_stride < 1) return fail(LCP_ERR_INVALID_INPUT, "bad layout request");
  *layout = packed_layout(count, out_stride);
  return LCP_OK;
}

int lcp_query_host_packed(const lcp_index* ix, lcp_workspace* ws, const uint16_t* queries,
                          int32_t count, int32_t k, int32_t mode, int32_t out_stride,
                          void* out_block) {
  // the asynchronous submission (graph-cached device work; direct host I/O for
  // small batches in lcp_pinned_alloc blocks) followed by its wait
  LCP_TRY(lcp_query_host_packed_async(ix, ws, queries, count, k, mode, out_stride, out_block, 0));
  return lcp_workspace_wait(ws);
}

int lcp_query_host_packed_async(const lcp_index* ix, lcp_workspace* ws, const uint16_t* queries,
                                int32_t count, int32_t k, int32_t mode, int32_t out_stride,
                                void* out_block, int32_t flags) {
  if (!ix || !ws) return fail(LCP_ERR_INVALID_INPUT, "null index or workspace");
  if (ws->pending) return fail(LCP_ERR_STATE, "workspace already has a batch in flight");
  if (count <= 0) return LCP_OK;
  if (out_stride < 1 || !out_block || !queries)
    return fail(LCP_ERR_INVALID_INPUT, "bad output block or queries");
  const DevIndex& dv = ix->dv;
  cudaStream_t st = ws->stream;
  const lcp_packed_layout lay = packed_layout(count, out_stride);
  const size_t qb = (size_t)count * dv.L * 2;
  const size_t d2h = (flags & LCP_PACKED_NO_WORK) ? (size_t)lay.matched_depth : (size_t)lay.total;
  static const bool no_graphs = getenv("LCP_NO_GRAPH_CACHE") != nullptr;  // A/B switch
  ++ws->tick;
  // every buffer the submission touches exists before the lookup / capture (no
  // allocation inside a capture); a reallocation bumps the epoch, so graphs
  // holding the freed pointers can no longer match and are destroyed
  LCP_TRY(ws->q_in.ensure(qb));
  LCP_TRY(ws->ids.ensure((size_t)lay.total));
  LCP_TRY(ws->qkeys.ensure((size_t)count * dv.W * 8));
  ws->prune_stale_graphs();
  char* d = static_cast<char*>(ws->ids.p);
  // Small batches whose query and result blocks come from lcp_pinned_alloc:
  // the kernel reads the queries from, and writes the results into, host
  // memory directly (mapped page-locked memory over PCIe).  A round trip then
  // has no copy-engine work at all — the two copies' setup and the
  // copy -> kernel -> copy hand-offs were most of a single query's latency.
  // Large batches keep the copies: thousands of small PCIe transactions per
  // batch cost more than two bulk copies.
  static const int zc_max = [] {
    const char* e = getenv("LCP_DIRECT_IO_MAX");
    return e ? atoi(e) : 1024;  // tools/e2e_probe.py, tools/latency_probe.py
  }();
  char* zq = nullptr;
  char* zo = nullptr;
  if (count <= zc_max && dv.n > 0 && dv.W <= 8 && k <= FAST_KMAX) {  // kernels that read rows / write slots directly
    zq = pinned_device_alias(queries, qb);
    zo = zq ? pinned_device_alias(out_block, d2h) : nullptr;
  }
  const bool direct = zq && zo;
  const GraphKey key{ix->generation, ws->epoch(), count, k, mode | (flags << 8), out_stride,
                     direct ? queries : nullptr, direct ? out_block : nullptr};
  if (direct) {
    // the kernels only ever set the flag, so the host clears it
    *reinterpret_cast<volatile int*>(static_cast<char*>(out_block) + lay.err) = 0;
  } else {
    // one H2D, the device work (graph-cached), one D2H: the invalid-query flag
    // lives in the block (lay.err), cleared on the device, so no separate small
    // copy is needed
    LCP_CK(cudaMemcpyAsync(ws->q_in.p, queries, qb, cudaMemcpyHostToDevice, st));
  }
  char* o = direct ? zo : d;
  // without work counters the block ends before matched_depth: those go to scratch
  char* ow = direct && !(flags & LCP_PACKED_NO_WORK) ? zo : d;
  auto device_work = [&]() -> int {
    if (!direct) LCP_CK(cudaMemsetAsync(d + lay.err, 0, 8, st));
    return query_impl(ix, ws, direct ? reinterpret_cast<const uint16_t*>(zq) : ws->q_in.as<uint16_t>(),
                      count, k, mode, out_stride, reinterpret_cast<uint32_t*>(o + lay.ids),
                      reinterpret_cast<uint16_t*>(o + lay.lcps), reinterpret_cast<int32_t*>(o + lay.hits),
                      reinterpret_cast<uint16_t*>(ow + lay.matched_depth),
                      reinterpret_cast<uint64_t*>(ow + lay.aux), st, reinterpret_cast<int*>(o + lay.err));
  };
  CachedGraph* hit = nullptr;
  for (auto& g : ws->graphs)
    if (g.key == key) hit = &g;
  if (hit) {  // replay: one launch for the device work
    hit->last_use = ws->tick;
    LCP_CK(cudaGraphLaunch(hit->exec, st));
  } else {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    bool captured = false;
    if (!no_graphs && cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
      const int r = device_work();
      const cudaError_t e = cudaStreamEndCapture(st, &graph);
      if (r == LCP_OK && e == cudaSuccess && graph &&
          cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess)
        captured = true;
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();  // a failed capture leaves nothing enqueued
    }
    if (captured) {
      if ((int)ws->graphs.size() >= kGraphCache) {
        auto old = std::min_element(ws->graphs.begin(), ws->graphs.end(),
                                    [](const CachedGraph& a, const CachedGraph& b) {
                                      return a.last_use < b.last_use;
                                    });
        cudaGraphExecDestroy(old->exec);
        ws->graphs.erase(old);
      }
      ws->graphs.push_back({key, exec, ws->tick});
      LCP_CK(cudaGraphLaunch(exec, st));
    } else {
      LCP_TRY(device_work());
    }
  }
  if (!direct) LCP_CK(cudaMemcpyAsync(out_block, d, d2h, cudaMemcpyDeviceToHost, st));
  LCP_CK(cudaEventRecord(ws->done, st));
  ws->pending = true;
  ws->pending_sigma = dv.sigma;
  ws->pending_err = reinterpret_cast<const int*>(static_cast<const char*>(out_block) + lay.err);
  return LCP_OK;
}

int lcp_workspace_wait(lcp_workspace* ws) {
  if (!ws) return fail(LCP_ERR_INVALID_INPUT, "null workspace");
  if (!ws->pending) return LCP_OK;
  ws->pending = false;
  LCP_CK(cudaEventSynchronize(ws->done));
  const int* e = ws->pending_err;
  ws->pending_err = nullptr;
  if (e && *e)
    return fail(LCP_ERR_INVALID_INPUT, "query symbol out of range for alphabet of size " +
                                           std::to_string(ws->pending_sigma));
  return LCP_OK;
}

// ---- full scan ----------------------------------------------------------------
}  // extern "C"

template <typename C, int KCAP>
static int launch_fullscan_w1_k(const DevIndex& dv, const uint16_t* q, const u64* qkeys, int count,
                                int need, long long chunk, int nchunks, u64* partial, int* hint,
                                int* err, cudaStream_t st) {
  const size_t smem = 16 + 2 * 2 * FS1_STAGE_KEYS * 4;  // 2 stages x (hi + lo) planes
  static const cudaError_t attr = cudaFuncSetAttribute(  // thread-safe one-time initialisation
      k_fullscan_w1<C, KCAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  LCP_CK(attr);
  dim3 grid((count + FS_THREADS - 1) / FS_THREADS, nchunks);
  k_fullscan_w1<C, KCAP><<<grid, FS_THREADS, smem, st>>>(dv, q, qkeys, count, need, chunk, nchunks,
                                                         partial, hint, err);
  return LCP_OK;
}

// list length = need exactly for the common k, else the next size up
template <typename C>
static int launch_fullscan_w1_c(const DevIndex& dv, const uint16_t* q, const u64* qkeys, int count,
                                int need, long long chunk, int nchunks, u64* partial, int* hint,
                                int* err, cudaStream_t st) {
#define LCP_FS_CASE(K) \
  if (need <= K) return launch_fullscan_w1_k<C, K>(dv, q, qkeys, count, need, chunk, nchunks, partial, hint, err, st);
  LCP_FS_CASE(1) LCP_FS_CASE(2) LCP_FS_CASE(3) LCP_FS_CASE(4) LCP_FS_CASE(5) LCP_FS_CASE(6)
  LCP_FS_CASE(8) LCP_FS_CASE(10) LCP_FS_CASE(12) LCP_FS_CASE(16) LCP_FS_CASE(20)
  LCP_FS_CASE(24) LCP_FS_CASE(32) LCP_FS_CASE(48) LCP_FS_CASE(64)
  if constexpr (sizeof(C) == 4) {  // 32-bit composites: up to 128 list registers
    LCP_FS_CASE(96) LCP_FS_CASE(128)
  }
#undef LCP_FS_CASE
  return fail(LCP_ERR_INTERNAL, "full scan: need beyond the register lists");
}

static int launch_fullscan_w1(const DevIndex& dv, const uint16_t* q, const u64* qkeys, int count,
                              int need, long long chunk, int nchunks, u64* partial, int* hint,
                              int* err, cudaStream_t st) {
  if (dv.idbits < 32)
    return launch_fullscan_w1_c<u32>(dv, q, qkeys, count, need, chunk, nchunks, partial, hint, err, st);
  return launch_fullscan_w1_c<u64>(dv, q, qkeys, count, need, chunk, nchunks, partial, hint, err, st);
}


// per query, the take smallest of `shards` candidate lists of kin entries
// (cand index = s * s_stride + q * q_stride + j * j_stride): a warp per query for
// take <= 32, else a CTA sorting all shards * kin <= MERGE_SORT_CAP candidates
static int launch_merge(const u64* cand, int shards, int count, int kin, long long s_stride,
                        long long q_stride, long long j_stride, int take, int L, int strict, u32* ids, uint16_t* lcps,
                        int* hits, int out_stride, cudaStream_t st) {
  if (take <= FAST_KMAX) {
    k_merge<<<blocks_for((long long)count * 32, 256), 256, 0, st>>>(
        cand, shards, count, kin, s_stride, q_stride, j_stride, take, L, strict, ids, lcps, hits, out_stride);
  } else {
    if ((long long)shards * kin > MERGE_SORT_CAP)
      return fail(LCP_ERR_INVALID_INPUT, "merge supports shards * k <= " + std::to_string(MERGE_SORT_CAP));
    int P = 1;
    while (P < shards * kin) P <<= 1;
    static const cudaError_t attr = cudaFuncSetAttribute(  // thread-safe one-time initialisation
        k_merge_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, MERGE_SORT_CAP * 8);
    LCP_CK(attr);
    const unsigned grid = (unsigned)std::min<long long>(count, 8ll * num_sms());
    k_merge_sort<<<grid, MERGE_SORT_THREADS, (size_t)P * 8, st>>>(
        cand, shards, count, kin, s_stride, q_stride, j_stride, take, L, strict, ids, lcps, hits, out_stride);
  }
  LCP_CK_LAUNCH();
  return LCP_OK;
}

extern "C" {

int lcp_fullscan(const lcp_index* ix, lcp_workspace* ws, const uint16_t* queries, int32_t count,
                 int32_t k, int32_t out_stride, uint32_t* ids, uint16_t* lcps, int32_t* hits,
                 void* stream) {
  if (!ix || !ws) return fail(LCP_ERR_INVALID_INPUT, "null index or workspace");
  if (k < 1) return fail(LCP_ERR_INVALID_INPUT, "k must be >= 1, got " + std::to_string(k));
  const DevIndex& dv = ix->dv;
  if (count <= 0) return LCP_OK;
  if (out_stride < std::min<long long>(k, std::max(1ll, dv.n)))
    return fail(LCP_ERR_INVALID_INPUT, "out_stride must be >= min(k, n)");
  cudaStream_t st = (cudaStream_t)stream;
  if (dv.n == 0) {
    k_fill_empty<<<blocks_for(count, 256), 256, 0, st>>>(count, 0, hits, nullptr, nullptr);
    LCP_CK_LAUNCH();
    return LCP_OK;
  }
  const int take = (int)std::min<long long>(k, dv.n);
  static const bool smallq_off = getenv("LCP_FULLSCAN_NO_SMALLQ") != nullptr;  // A/B hook
  if (count <= FSQ_QMAX && take <= FAST_KMAX && !smallq_off) {
    // a few queries: one HBM-streaming pass with every query in every lane
    LCP_TRY(ws->qkeys.ensure((size_t)count * dv.W * 8));
    LCP_TRY(pack_rows(queries, count, dv, ws->qkeys.as<u64>(), nullptr, ws->d_err, st));
    int Q = 1;
    while (Q < count) Q <<= 1;
    // one or two CTAs per SM, but at least FSQ_SEG_MIN keys per warp: a small
    // corpus gets fewer, longer segments (the per-warp seed and the merge of
    // the CTA lists, not the key stream, dominate there)
    const long long G = std::max(1ll, std::min<long long>(
        num_sms() * (Q == 1 ? fsq_ctas_per_sm<1>() : 1),
        (dv.n + (long long)FSQ_WARPS * FSQ_SEG_MIN - 1) / ((long long)FSQ_WARPS * FSQ_SEG_MIN)));
    const long long warps = G * FSQ_WARPS;
    long long seg = (dv.n + warps - 1) / warps;
    seg = (seg + FSQ_STEP - 1) / FSQ_STEP * FSQ_STEP;
    const size_t csz = dv.idbits < 32 ? 4 : 8;
    LCP_TRY(ws->partial.ensure((size_t)G * count * take * csz));
    LCP_TRY(ws->hint.ensure((size_t)(count + 1) * 4));
    LCP_CK(cudaMemsetAsync(ws->hint.p, 0, (size_t)(count + 1) * 4, st));
    int* hint = ws->hint.as<int>();
    unsigned* ctr = reinterpret_cast<unsigned*>(hint + count);
#define LCP_FSQ(C, QQ)                                                                           \
  k_fullscan_smallq<C, QQ><<<(unsigned)G, FSQ_THREADS, (size_t)FSQ_WARPS * QQ * 32 * sizeof(C), \
                             st>>>(dv, ws->qkeys.as<u64>(), count, take, seg,                    \
                                   ws->partial.as<C>(), hint, ctr, ids, lcps, hits, out_stride)
    if (dv.idbits < 32) {
      if (Q == 1) LCP_FSQ(u32, 1); else if (Q == 2) LCP_FSQ(u32, 2); else if (Q == 4) LCP_FSQ(u32, 4); else LCP_FSQ(u32, 8);
    } else {
      if (Q == 1) LCP_FSQ(u64, 1); else if (Q == 2) LCP_FSQ(u64, 2); else if (Q == 4) LCP_FSQ(u64, 4); else LCP_FSQ(u64, 8);
    }
#undef LCP_FSQ
    LCP_CK_LAUNCH();
    return LCP_OK;
  }
  if (take <= (dv.idbits < 32 ? FS_KMAX_U32 : FS_KMAX_U64)) {
    const int per_stage = FS1_STAGE_KEYS;
    const long long qtiles = (count + FS_THREADS - 1) / FS_THREADS;
    const long long max_chunks = (dv.n + per_stage - 1) / per_stage;
    long long want = std::max(1ll, (4ll * num_sms() + qtiles - 1) / qtiles);
    if (const char* fc = getenv("LCP_FULLSCAN_CHUNKS")) want = std::max(1ll, atoll(fc));  // tuning hook
    want = std::min(want, max_chunks);
    if (take > FAST_KMAX) want = std::min<long long>(want, MERGE_SORT_CAP / take);  // CTA merge capacity
    long long chunk = (dv.n + want - 1) / want;
    chunk = (chunk + per_stage - 1) / per_stage * per_stage;
    const int nchunks = (int)((dv.n + chunk - 1) / chunk);
    LCP_TRY(ws->partial.ensure((size_t)count * nchunks * take * 8));
    u64* partial = ws->partial.as<u64>();
    // W > 1: the kernel filters on the first word and reads the rest of the
    // packed query for keys that match it entirely
    LCP_TRY(ws->qkeys.ensure((size_t)count * dv.W * 8));
    LCP_TRY(pack_rows(queries, count, dv, ws->qkeys.as<u64>(), nullptr, ws->d_err, st));
    const u64* qk = ws->qkeys.as<u64>();
    LCP_TRY(ws->hint.ensure((size_t)count * 4));
    LCP_CK(cudaMemsetAsync(ws->hint.p, 0, (size_t)count * 4, st));
    LCP_TRY(launch_fullscan_w1(dv, queries, qk, count, take, chunk, nchunks, partial,
                               ws->hint.as<int>(), ws->d_err, st));
    LCP_CK_LAUNCH();
    // partial lists are chunk-major, query-fastest: [chunk][j][query]
    return launch_merge(partial, nchunks, count, take, (long long)take * count, 1, count, take, dv.L,
                        0, ids, lcps, hits, out_stride, st);
  }
  LCP_TRY(ws->qkeys.ensure((size_t)count * dv.W * 8));
  LCP_TRY(pack_rows(queries, count, dv, ws->qkeys.as<u64>(), nullptr, ws->d_err, st));
  unsigned grid = (unsigned)gen_grid(count);
  k_query_general<<<grid, GEN_THREADS, 0, st>>>(dv, ws->qkeys.as<u64>(), queries, count, k, 1, 1,
                                                out_stride, ids, lcps, hits, nullptr, nullptr);
  LCP_CK_LAUNCH();
  return LCP_OK;
}

int lcp_fullscan_host(const lcp_index* ix, lcp_workspace* ws, const uint16_t* queries,
                      int32_t count, int32_t k, int32_t out_stride, uint32_t* ids, uint16_t* lcps,
                      int32_t* hits) {
  if (!ix || !ws) return fail(LCP_ERR_INVALID_INPUT, "null index or workspace");
  if (count <= 0) return LCP_OK;
  const DevIndex& dv = ix->dv;
  cudaStream_t st = ws->stream;
  const size_t qb = (size_t)count * dv.L * 2;
  const size_t ob = (size_t)count * std::max(1, out_stride);
  LCP_TRY(ws->q_in.ensure(qb));
  LCP_TRY(ws->ids.ensure(ob * 4));
  LCP_TRY(ws->lcps.ensure(ob * 2));
  LCP_TRY(ws->hits.ensure((size_t)count * 4));
  LCP_CK(cudaMemcpyAsync(ws->q_in.p, queries, qb, cudaMemcpyHostToDevice, st));
  LCP_TRY(lcp_fullscan(ix, ws, ws->q_in.as<uint16_t>(), count, k, out_stride, ws->ids.as<u32>(),
                       ws->lcps.as<uint16_t>(), ws->hits.as<int>(), st));
  if (ids) LCP_CK(cudaMemcpyAsync(ids, ws->ids.p, ob * 4, cudaMemcpyDeviceToHost, st));
  if (lcps) LCP_CK(cudaMemcpyAsync(lcps, ws->lcps.p, ob * 2, cudaMemcpyDeviceToHost, st));
  LCP_CK(cudaMemcpyAsync(hits, ws->hits.p, (size_t)count * 4, cudaMemcpyDeviceToHost, st));
  if (host_finish(ws) != LCP_OK)
    return fail(LCP_ERR_INVALID_INPUT,
                "query symbol out of range for alphabet of size " + std::to_string(dv.sigma));
  return LCP_OK;
}

// ---- shard candidates ------------------------------------------------------------
int lcp_encode_candidates(const uint32_t* ids, const uint16_t* lcps, const int32_t* hits,
                          int32_t count, int32_t k, int32_t in_stride, int32_t length,
                          int64_t id_offset, uint64_t* cand, void* stream) {
  if (count <= 0) return LCP_OK;
  if (k < 1 || in_stride < 1) return fail(LCP_ERR_INVALID_INPUT, "k and in_stride must be >= 1");
  k_encode<<<blocks_for((long long)count * k, 256), 256, 0, (cudaStream_t)stream>>>(
      ids, lcps, hits, count, k, in_stride, length, id_offset, (u64*)cand);
  LCP_CK_LAUNCH();
  return LCP_OK;
}

int lcp_merge_candidates(const uint64_t* cand, int32_t shards, int32_t count, int32_t k,
                         int32_t take, int32_t length, int32_t strict, uint32_t* ids,
                         uint16_t* lcps, int32_t* hits, void* stream) {
  if (count <= 0) return LCP_OK;
  if (shards < 1 || k < 1) return fail(LCP_ERR_INVALID_INPUT, "shards and k must be >= 1");
  if (take < 0 || take > k)
    return fail(LCP_ERR_INVALID_INPUT, "merge needs 0 <= take <= k");
  return launch_merge((const u64*)cand, shards, count, k, (long long)count * k, k, 1, take, length,
                      strict, ids, lcps, hits, std::max(1, take), (cudaStream_t)stream);
}

// ---- device-side routing for sharded steps (shard_kernels.cuh) ----------------
int lcp_pack_queries(const lcp_index* ix, lcp_workspace* ws, const uint16_t* rows, int32_t count,
                     uint64_t* keys, void* stream) {
  if (!ix || !ws) return fail(LCP_ERR_INVALID_INPUT, "null index or workspace");
  if (count <= 0) return LCP_OK;
  if (!rows || !keys) return fail(LCP_ERR_INVALID_INPUT, "null rows or keys");
  return pack_rows(rows, count, ix->dv, reinterpret_cast<u64*>(keys), nullptr, ws->d_err,
                   (cudaStream_t)stream);
}

int lcp_route_queries(const lcp_index* ix, lcp_workspace* ws, const uint16_t* queries,
                      const uint64_t* qkeys, int32_t count, const uint64_t* splitters, int32_t nsplit,
                      const uint64_t* first, const uint64_t* last, const int32_t* nonempty,
                      int32_t rank, int32_t* thresholds, int32_t consult, uint16_t* out_rows,
                      int32_t* out_sel, int32_t* d_count, uint64_t* reset_cand, int32_t cand_k,
                      void* stream) {
  if (!ix || !ws) return fail(LCP_ERR_INVALID_INPUT, "null index or workspace");
  if (!d_count || !out_sel || !out_rows) return fail(LCP_ERR_INVALID_INPUT, "null route output");
  if (nsplit < 0 || rank < 0 || rank > nsplit) return fail(LCP_ERR_INVALID_INPUT, "bad rank / splitter count");
  if (consult && (!thresholds || !first || !last || !nonempty))
    return fail(LCP_ERR_INVALID_INPUT, "consult routing needs thresholds, first / last rows and nonempty flags");
  if (reset_cand && cand_k < 1) return fail(LCP_ERR_INVALID_INPUT, "cand_k must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  LCP_CK(cudaMemsetAsync(d_count, 0, sizeof(int32_t), st));
  if (count <= 0) return LCP_OK;
  const DevIndex& dv = ix->dv;
  const u64* keys = reinterpret_cast<const u64*>(qkeys);
  if (!keys) {  // pack here (pass pre-packed keys to route one batch twice)
    LCP_TRY(ws->qkeys.ensure((size_t)count * dv.W * 8));
    LCP_TRY(pack_rows(queries, count, dv, ws->qkeys.as<u64>(), nullptr, ws->d_err, st));
    keys = ws->qkeys.as<u64>();
  }
  k_route_queries<<<blocks_for(count, RT_THREADS), RT_THREADS, 0, st>>>(
      keys, queries, count, dv.L, dv.W, dv.spw, dv.lb, reinterpret_cast<const u64*>(splitters), nsplit,
      reinterpret_cast<const u64*>(first), reinterpret_cast<const u64*>(last), nonempty, rank,
      thresholds, consult ? 1 : 0, out_rows, out_sel, d_count, reinterpret_cast<u64*>(reset_cand),
      cand_k);
  LCP_CK_LAUNCH();
  return LCP_OK;
}

int lcp_query_counted(const lcp_index* ix, lcp_workspace* ws, const uint16_t* queries,
                      int32_t capacity, const int32_t* d_count, int32_t expected, int32_t k,
                      int32_t mode, int32_t out_stride, uint32_t* ids, uint16_t* lcps, int32_t* hits,
                      uint16_t* matched_depth, uint64_t* aux, void* stream) {
  if (!ws) return fail(LCP_ERR_INVALID_INPUT, "null index or workspace");
  if (!d_count) return fail(LCP_ERR_INVALID_INPUT, "null device count");
  return query_impl(ix, ws, queries, capacity, k, mode, out_stride, ids, lcps, hits, matched_depth,
                    aux, stream, ws->d_err, d_count, expected);
}

int lcp_shard_thresholds(const uint16_t* lcps, const int32_t* hits, const uint16_t* matched_depth,
                         const int32_t* sel, const int32_t* d_count, int32_t capacity, int32_t stride,
                         int32_t need, int32_t strict, int32_t* thresholds, void* stream) {
  if (capacity <= 0) return LCP_OK;
  if (!lcps || !hits || !sel || !d_count || !thresholds || (strict && !matched_depth))
    return fail(LCP_ERR_INVALID_INPUT, "null threshold argument");
  k_shard_threshold<<<blocks_for(capacity, 256), 256, 0, (cudaStream_t)stream>>>(
      lcps, hits, matched_depth, sel, d_count, stride, need, strict, thresholds);
  LCP_CK_LAUNCH();
  return LCP_OK;
}

int lcp_encode_candidates_sel(const uint32_t* ids, const uint16_t* lcps, const int32_t* hits,
                              const int32_t* sel, const int32_t* d_count, int32_t capacity, int32_t k,
                              int32_t in_stride, int32_t length, const int64_t* gids,
                              int64_t id_offset, uint64_t* cand, void* stream) {
  if (capacity <= 0) return LCP_OK;
  if (k < 1 || in_stride < 1) return fail(LCP_ERR_INVALID_INPUT, "k and in_stride must be >= 1");
  k_encode_sel<<<blocks_for((long long)capacity * k, 256), 256, 0, (cudaStream_t)stream>>>(
      ids, lcps, hits, sel, d_count, capacity, k, in_stride, length,
      reinterpret_cast<const long long*>(gids), id_offset, reinterpret_cast<u64*>(cand));
  LCP_CK_LAUNCH();
  return LCP_OK;
}

int lcp_signal_peers(uint32_t* const* peer_signals, int32_t world, int32_t rank, uint32_t* epoch,
                     void* stream) {
  if (!peer_signals || !epoch || world < 1 || rank < 0 || rank >= world)
    return fail(LCP_ERR_INVALID_INPUT, "bad peer signal arguments");
  k_signal_peers<<<1, 32, 0, (cudaStream_t)stream>>>(reinterpret_cast<unsigned* const*>(peer_signals),
                                                     world, rank, epoch);
  LCP_CK_LAUNCH();
  return LCP_OK;
}

int lcp_merge_candidates_peers(const uint64_t* const* peer_cand, int32_t world, int32_t rank, int32_t m,
                               int32_t k, int32_t take, int32_t length, int32_t strict,
                               const uint32_t* my_signals, const uint32_t* epoch, uint32_t* ids,
                               uint16_t* lcps, int32_t* hits, int32_t out_stride, void* stream) {
  if (m <= 0) return LCP_OK;
  if (!peer_cand || !my_signals || !epoch || world < 1 || rank < 0 || rank >= world)
    return fail(LCP_ERR_INVALID_INPUT, "bad peer merge arguments");
  if (k < 1 || take < 0 || take > k || take > FAST_KMAX)
    return fail(LCP_ERR_INVALID_INPUT, "peer merge needs 0 <= take <= k and take <= 32");
  k_merge_peers<<<blocks_for((long long)m * 32, 256), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const u64* const*>(peer_cand), world, rank, m, k, take, length, strict,
      my_signals, epoch, ids, lcps, hits, std::max(1, out_stride));
  LCP_CK_LAUNCH();
  return LCP_OK;
}

// ---- persistent single-query server (serve_kernels.cuh) ----------------------
}  // extern "C"

struct lcp_server {
  const lcp_index* ix = nullptr;
  unsigned* box = nullptr;      // page-locked mailboxes: request (8 sectors), response (8 sectors)
  unsigned* d_box = nullptr;    // device alias
  cudaStream_t stream = nullptr;
  const uint16_t* row = nullptr;  // the caller's query row (host)
  char* out = nullptr;            // the caller's packed block (host)
  lcp_packed_layout lay{};
  int k = 0, mode = 0, stride = 0, nq = 0, nr = 0;
  unsigned seq = 0;
  size_t smem = 0;
  int (*launch)(lcp_server*, unsigned) = nullptr;
};

template <typename C, int T, int MODE>
static int serve_launch(lcp_server* s, unsigned last) {
  static const bool attr = [] {
    cudaFuncSetAttribute(k_serve_w1<C, T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaGetLastError();
    return true;
  }();
  (void)attr;
  k_serve_w1<C, T, MODE><<<1, 32, s->smem, s->stream>>>(s->ix->dv, s->d_box, s->d_box + SERVE_SECTORS * 8,
                                                        last, s->k, s->stride);
  LCP_CK_LAUNCH();
  return LCP_OK;
}

extern "C" {

int lcp_server_start(const lcp_index* ix, int32_t k, int32_t mode, int32_t out_stride, const uint16_t* query_row,
                     void* out_block, lcp_server** out) {
  if (!ix || !out || !query_row || !out_block) return fail(LCP_ERR_INVALID_INPUT, "null argument");
  *out = nullptr;
  const DevIndex& dv = ix->dv;
  if (mode < 0 || mode > 2) return fail(LCP_ERR_INVALID_INPUT, "unknown mode");
  if (mode == LCP_MODE_TAL && ix->tal_depth < 0)
    return fail(LCP_ERR_STATE, "index was built without a TAL bucket structure");
  if (dv.W != 1 || dv.n < 1 || k < 1 || k > FAST_KMAX)
    return fail(LCP_ERR_STATE, "the single-query server needs W == 1, n >= 1 and k <= 32");
  const long long need = mode == LCP_MODE_COMPLETE ? std::min<long long>(k, dv.n) : k;
  if (need > 32 || out_stride > 32) return fail(LCP_ERR_STATE, "the single-query server handles k <= 32");
  const long long ns = std::max<long long>(1, std::min<long long>(k, dv.n));
  if (out_stride < ns) return fail(LCP_ERR_INVALID_INPUT, "out_stride must be >= min(k, n)");
  const int nq = (dv.L + SERVE_SYMS_PER_SECTOR - 1) / SERVE_SYMS_PER_SECTOR;
  const int nr = (SERVE_P_IDS + 6 * out_stride + SERVE_PAYLOAD_PER_SECTOR - 1) / SERVE_PAYLOAD_PER_SECTOR;
  if (nq > SERVE_SECTORS || nr > SERVE_SECTORS) return fail(LCP_ERR_STATE, "query row too long for the server");
  auto* s = new lcp_server();
  s->ix = ix;
  s->k = k;
  s->mode = mode;
  s->stride = out_stride;
  s->nq = nq;
  s->nr = nr;
  s->lay = packed_layout(1, out_stride);
  s->row = query_row;
  s->out = static_cast<char*>(out_block);
  s->smem = 16 + (size_t)dv.smem_entries * 8 + 2 * SERVE_SECTORS * 8 * 4;
  void* c = nullptr;
  const size_t bytes = 2 * SERVE_SECTORS * 32;
  if (cudaHostAlloc(&c, bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
      cudaHostGetDevicePointer(reinterpret_cast<void**>(&s->d_box), c, 0) != cudaSuccess ||
      cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    if (c) cudaFreeHost(c);
    delete s;
    return fail(LCP_ERR_CUDA, "server allocation failed");
  }
  s->box = static_cast<unsigned*>(c);
  memset(s->box, 0, bytes);
  // the batch kernel's per-query body: 64-key leaf region for need <= 16,
  // 96 keys up to 32 (the batch path runs the list kernel there)
  static int (*const table[2][2][3])(lcp_server*, unsigned) = {
      {{serve_launch<u32, 2, 0>, serve_launch<u32, 2, 1>, serve_launch<u32, 2, 2>},
       {serve_launch<u32, 3, 0>, serve_launch<u32, 3, 1>, serve_launch<u32, 3, 2>}},
      {{serve_launch<u64, 2, 0>, serve_launch<u64, 2, 1>, serve_launch<u64, 2, 2>},
       {serve_launch<u64, 3, 0>, serve_launch<u64, 3, 1>, serve_launch<u64, 3, 2>}}};
  s->launch = table[dv.idbits < 32 ? 0 : 1][need <= 16 ? 0 : 1][mode];
  const int r = s->launch(s, 0);
  if (r != LCP_OK) {
    cudaStreamDestroy(s->stream);
    cudaFreeHost(s->box);
    delete s;
    return r;
  }
  *out = s;
  return LCP_OK;
}

// write tag `t` into every request sector, each after its symbols (the
// caller's row; none for a stop request, whose row may already be gone)
static void serve_post(lcp_server* s, unsigned t, bool with_row) {
  const int L = s->ix->dv.L;
  for (int j = 0; j < s->nq; ++j) {
    unsigned* sec = s->box + j * 8;
    const int first = j * SERVE_SYMS_PER_SECTOR;
    const int cnt = std::min(SERVE_SYMS_PER_SECTOR, L - first);
    if (with_row) memcpy(sec, s->row + first, (size_t)cnt * 2);
    __atomic_store_n(sec + 7, t, __ATOMIC_RELEASE);
  }
}

int lcp_server_query_row(lcp_server* s, const uint16_t* row) {
  if (!s || !row) return fail(LCP_ERR_INVALID_INPUT, "null server or row");
  const uint16_t* keep = s->row;
  s->row = row;
  const int r = lcp_server_query(s);
  s->row = keep;
  return r;
}

int lcp_server_query(lcp_server* s) {
  if (!s) return fail(LCP_ERR_INVALID_INPUT, "null server");
  const unsigned want = ++s->seq;
  if (want & SERVE_STOP) return fail(LCP_ERR_STATE, "single-query server sequence exhausted");
  serve_post(s, want, true);
  unsigned* resp = s->box + SERVE_SECTORS * 8;
  const auto t_start = std::chrono::steady_clock::now();
  for (unsigned spins = 1;; ++spins) {
    bool ready = true;
    for (int j = 0; j < s->nr && ready; ++j) ready = __atomic_load_n(resp + j * 8 + 7, __ATOMIC_ACQUIRE) == want;
    if (ready) break;
    if ((spins & 4095) == 0) {  // the warp idles out after SERVE_IDLE_NS: relaunch it
      if (std::chrono::steady_clock::now() - t_start > std::chrono::seconds(2)) {
        std::string tags;
        for (int j = 0; j < s->nr; ++j) tags += " " + std::to_string(__atomic_load_n(resp + j * 8 + 7, __ATOMIC_ACQUIRE));
        std::string rq;
        for (int j = 0; j < s->nq; ++j) rq += " " + std::to_string(__atomic_load_n(s->box + j * 8 + 7, __ATOMIC_ACQUIRE));
        return fail(LCP_ERR_INTERNAL, "single-query server: no answer after 2 s (request " + std::to_string(want) +
                                          ", request tags" + rq + ", response tags" + tags + ", stream " +
                                          cudaGetErrorString(cudaStreamQuery(s->stream)) + ")");
      }
      const cudaError_t e = cudaStreamQuery(s->stream);
      if (e == cudaSuccess) {
        bool again = true;
        for (int j = 0; j < s->nr && again; ++j) again = __atomic_load_n(resp + j * 8 + 7, __ATOMIC_ACQUIRE) == want;
        if (again) break;
        LCP_TRY(s->launch(s, want - 1));
      } else if (e != cudaErrorNotReady) {
        return fail(LCP_ERR_CUDA, std::string("single-query server: ") + cudaGetErrorString(e));
      }
    }
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
  // unpack the payload (28 bytes per sector) into the caller's packed block
  unsigned char pay[SERVE_SECTORS * SERVE_PAYLOAD_PER_SECTOR];
  for (int j = 0; j < s->nr; ++j) memcpy(pay + j * SERVE_PAYLOAD_PER_SECTOR, resp + j * 8, SERVE_PAYLOAD_PER_SECTOR);
  const int st = s->stride;
  memcpy(s->out + s->lay.ids, pay + SERVE_P_IDS, (size_t)st * 4);
  memcpy(s->out + s->lay.lcps, pay + SERVE_P_IDS + 4 * st, (size_t)st * 2);
  memcpy(s->out + s->lay.hits, pay + SERVE_P_HITS, 4);
  memcpy(s->out + s->lay.matched_depth, pay + SERVE_P_MD, 2);
  memcpy(s->out + s->lay.aux, pay + SERVE_P_AUX, 16);
  int err = 0;
  memcpy(&err, pay + SERVE_P_ERR, 4);
  memcpy(s->out + s->lay.err, &err, 4);
  if (err)
    return fail(LCP_ERR_INVALID_INPUT,
                "query symbol out of range for alphabet of size " + std::to_string(s->ix->dv.sigma));
  return LCP_OK;
}

int lcp_server_stop(lcp_server* s) {
  if (!s) return LCP_OK;
  serve_post(s, (s->seq + 1) | SERVE_STOP, false);
  const cudaError_t e = cudaStreamSynchronize(s->stream);
  cudaStreamDestroy(s->stream);
  cudaFreeHost(s->box);
  delete s;
  if (e != cudaSuccess) return fail(LCP_ERR_CUDA, std::string("single-query server: ") + cudaGetErrorString(e));
  return LCP_OK;
}

int lcp_pinned_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) return fail(LCP_ERR_INVALID_INPUT, "bad pinned allocation request");
  *out = nullptr;
  const size_t size = (size_t)std::max<int64_t>(bytes, 1);
  LCP_CK(cudaHostAlloc(out, size, cudaHostAllocMapped | cudaHostAllocPortable));
  void* dev = nullptr;
  if (cudaHostGetDevicePointer(&dev, *out, 0) != cudaSuccess) {
    cudaGetLastError();
    dev = nullptr;  // not device-addressable here: submissions copy instead
  }
  std::lock_guard<std::mutex> g(g_pinned_mu);
  g_pinned[reinterpret_cast<uintptr_t>(*out)] = {size, dev};
  return LCP_OK;
}

int lcp_pinned_free(void* p) {
  if (!p) return LCP_OK;
  {
    std::lock_guard<std::mutex> g(g_pinned_mu);
    g_pinned.erase(reinterpret_cast<uintptr_t>(p));
  }
  LCP_CK(cudaFreeHost(p));
  return LCP_OK;
}

int lcp_stream_sync(void* stream) {
  LCP_CK(cudaStreamSynchronize((cudaStream_t)stream));
  return LCP_OK;
}

#ifdef LCP_TRACE
int lcp_debug_trace(uint64_t* host, int64_t entries) {
  LCP_CK(cudaDeviceSynchronize());
  LCP_CK(cudaMemcpyFromSymbol(host, lcp_trace_buf, (size_t)entries * 8));
  return LCP_OK;
}
#endif

}  // extern "C"
