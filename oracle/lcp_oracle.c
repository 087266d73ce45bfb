/*
 * lcp_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference algorithm of arXiv 2602.04936's
 * `lcpsearch` package (/root/reference/pkg/src/lcpsearch/), used as the
 * parity checker by tests/, by __graft_entry__.smoke() and as the timed CPU
 * baseline (`cpu_baseline`, `bench.py --impl reference`).  The product path
 * (paper_2602_04936_b200/) never links, loads or calls this file.
 *
 * Parity is pinned: tests/test_oracle_golden.py checks every function here
 * against golden vectors produced by the Python reference itself
 * (tests/golden/make_golden.py).
 *
 * Each function follows one reference function, cited file:line:
 *   orc_lexicographic_order  core.py:162-174   stable lexicographic argsort
 *   orc_adjacent_lcp         core.py:177-184
 *   orc_trie_build           trie.py:397-431   per-depth arena
 *   orc_trie_query           trie.py:229-256 (descent) + trie.py:290-342 (collect)
 *   orc_tal_build            tal.py:29-82
 *   orc_tal_query            tal.py:116-194
 *   orc_oracle_top_k         oracle.py:38-59
 * The batch drivers run queries on `nthreads` pthreads (the reference fans
 * queries over a thread pool, bench.py:245-270).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ util */

static int row_cmp(const uint16_t* a, const uint16_t* b, int32_t L) {
  for (int32_t j = 0; j < L; ++j)
    if (a[j] != b[j]) return a[j] < b[j] ? -1 : 1;
  return 0;
}

static int64_t row_lcp(const uint16_t* a, const uint16_t* b, int32_t L) {
  for (int32_t j = 0; j < L; ++j)
    if (a[j] != b[j]) return j;
  return L;
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y);
}

/* k smallest of vals[0..m) ascending into out (k <= m); uses a bounded
 * max-heap when k is small relative to m (== np.partition + sort, trie.py:90-94). */
static void heap_sift_down(uint64_t* h, int64_t sz, int64_t i) {
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < sz && h[l] > h[m]) m = l;
    if (r < sz && h[r] > h[m]) m = r;
    if (m == i) return;
    uint64_t t = h[i];
    h[i] = h[m];
    h[m] = t;
    i = m;
  }
}

static void smallest_u64(const uint64_t* vals, int64_t m, int64_t k, uint64_t* out) {
  if (k <= 0) return;
  if (k >= m) {
    memcpy(out, vals, (size_t)m * 8);
    qsort(out, (size_t)m, 8, cmp_u64);
    return;
  }
  /* max-heap of the k smallest seen so far */
  memcpy(out, vals, (size_t)k * 8);
  for (int64_t i = k / 2 - 1; i >= 0; --i) heap_sift_down(out, k, i);
  for (int64_t i = k; i < m; ++i) {
    if (vals[i] < out[0]) {
      out[0] = vals[i];
      heap_sift_down(out, k, 0);
    }
  }
  qsort(out, (size_t)k, 8, cmp_u64);
}

/* ------------------------------------------ core.lexicographic_order */

static void merge_sort(int64_t* a, int64_t* tmp, int64_t lo, int64_t hi, const uint16_t* rows,
                       int32_t L) {
  if (hi - lo < 2) return;
  if (hi - lo <= 16) { /* stable insertion sort */
    for (int64_t i = lo + 1; i < hi; ++i) {
      int64_t v = a[i], j = i - 1;
      while (j >= lo && row_cmp(rows + a[j] * L, rows + v * L, L) > 0) {
        a[j + 1] = a[j];
        --j;
      }
      a[j + 1] = v;
    }
    return;
  }
  int64_t mid = lo + (hi - lo) / 2;
  merge_sort(a, tmp, lo, mid, rows, L);
  merge_sort(a, tmp, mid, hi, rows, L);
  int64_t i = lo, j = mid, o = lo;
  while (i < mid && j < hi) {
    /* take from the left run on ties: stability */
    if (row_cmp(rows + a[j] * L, rows + a[i] * L, L) < 0) tmp[o++] = a[j++];
    else tmp[o++] = a[i++];
  }
  while (i < mid) tmp[o++] = a[i++];
  while (j < hi) tmp[o++] = a[j++];
  memcpy(a + lo, tmp + lo, (size_t)(hi - lo) * 8);
}

void orc_lexicographic_order(const uint16_t* rows, int64_t n, int32_t L, int64_t* order) {
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  if (n < 2) return;
  int64_t* tmp = (int64_t*)malloc((size_t)n * 8);
  merge_sort(order, tmp, 0, n, rows, L);
  free(tmp);
}

/* --------------------------------------------------- core.adjacent_lcp */
void orc_adjacent_lcp(const uint16_t* sorted_rows, int64_t n, int32_t L, int64_t* adj) {
  for (int64_t i = 1; i < n; ++i)
    adj[i - 1] = row_lcp(sorted_rows + (i - 1) * L, sorted_rows + i * L, L);
}

/* ------------------------------------------------------------ trie.build */
typedef struct orc_trie {
  int64_t n;
  int32_t L, sigma;
  int32_t* order;
  int32_t* row_lo;
  uint16_t* edge;
  int64_t* level_offset; /* L + 2 */
  int64_t node_count;
} orc_trie;

orc_trie* orc_trie_build(const uint16_t* items, int64_t n, int32_t L, int32_t sigma) {
  orc_trie* t = (orc_trie*)calloc(1, sizeof(orc_trie));
  t->n = n;
  t->L = L;
  t->sigma = sigma;
  t->level_offset = (int64_t*)calloc((size_t)L + 2, 8);
  int64_t* order = (int64_t*)malloc((size_t)(n ? n : 1) * 8);
  orc_lexicographic_order(items, n, L, order);
  t->order = (int32_t*)malloc((size_t)(n ? n : 1) * 4);
  for (int64_t i = 0; i < n; ++i) t->order[i] = (int32_t)order[i];
  if (n == 0) {
    for (int32_t d = 1; d < L + 2; ++d) t->level_offset[d] = 1; /* trie.py:421 */
    t->node_count = 1;
    t->row_lo = (int32_t*)calloc(1, 4);
    t->edge = (uint16_t*)calloc(1, 2);
    free(order);
    return t;
  }
  uint16_t* rows = (uint16_t*)malloc((size_t)n * L * 2);
  for (int64_t i = 0; i < n; ++i) memcpy(rows + i * L, items + order[i] * L, (size_t)L * 2);
  int64_t* adj = (int64_t*)malloc((size_t)(n > 1 ? n - 1 : 1) * 8);
  orc_adjacent_lcp(rows, n, L, adj);
  /* count: level d has 1 + #{adj < d} nodes */
  int64_t total = 1;
  t->level_offset[0] = 0;
  t->level_offset[1] = 1;
  for (int32_t d = 1; d <= L; ++d) {
    int64_t c = 1;
    for (int64_t i = 0; i + 1 < n; ++i) c += adj[i] < d;
    total += c;
    t->level_offset[d + 1] = total;
  }
  t->node_count = total;
  t->row_lo = (int32_t*)malloc((size_t)total * 4);
  t->edge = (uint16_t*)malloc((size_t)total * 2);
  t->row_lo[0] = 0;
  t->edge[0] = 0;
  for (int32_t d = 1; d <= L; ++d) {
    int64_t p = t->level_offset[d];
    t->row_lo[p] = 0;
    t->edge[p] = rows[d - 1];
    ++p;
    for (int64_t i = 1; i < n; ++i) {
      if (adj[i - 1] < d) {
        t->row_lo[p] = (int32_t)i;
        t->edge[p] = rows[i * L + d - 1];
        ++p;
      }
    }
  }
  free(adj);
  free(rows);
  free(order);
  return t;
}

void orc_trie_free(orc_trie* t) {
  if (!t) return;
  free(t->order);
  free(t->row_lo);
  free(t->edge);
  free(t->level_offset);
  free(t);
}

int64_t orc_trie_node_count(const orc_trie* t) { return t->node_count; }

void orc_trie_export(const orc_trie* t, int32_t* order, int32_t* row_lo, uint16_t* edge,
                     int64_t* level_offset) {
  if (order) memcpy(order, t->order, (size_t)t->n * 4);
  if (row_lo) memcpy(row_lo, t->row_lo, (size_t)t->node_count * 4);
  if (edge) memcpy(edge, t->edge, (size_t)t->node_count * 2);
  if (level_offset) memcpy(level_offset, t->level_offset, (size_t)(t->L + 2) * 8);
}

/* searchsorted(arr[0..m), v, side="left") */
static int64_t lower_i32(const int32_t* arr, int64_t m, int32_t v) {
  int64_t a = 0, b = m;
  while (a < b) {
    int64_t mid = (a + b) >> 1;
    if (arr[mid] < v) a = mid + 1;
    else b = mid;
  }
  return a;
}

static int64_t lower_u16(const uint16_t* arr, int64_t m, uint16_t v) {
  int64_t a = 0, b = m;
  while (a < b) {
    int64_t mid = (a + b) >> 1;
    if (arr[mid] < v) a = mid + 1;
    else b = mid;
  }
  return a;
}

/* ids of order[lo..hi) excluding [xlo, xhi): the m smallest (ascending) */
static int64_t collect_smallest(const int32_t* order, int64_t lo, int64_t xlo, int64_t xhi,
                                int64_t hi, int64_t m, int32_t* out) {
  int64_t size = (xlo - lo) + (hi - xhi);
  if (m > size) m = size;
  if (m <= 0) return 0;
  uint64_t* vals = (uint64_t*)malloc((size_t)size * 8);
  uint64_t* sel = (uint64_t*)malloc((size_t)m * 8);
  int64_t p = 0;
  for (int64_t i = lo; i < xlo; ++i) vals[p++] = (uint64_t)(uint32_t)order[i];
  for (int64_t i = xhi; i < hi; ++i) vals[p++] = (uint64_t)(uint32_t)order[i];
  smallest_u64(vals, size, m, sel);
  for (int64_t i = 0; i < m; ++i) out[i] = (int32_t)sel[i];
  free(vals);
  free(sel);
  return m;
}

/* TrieIndex.query (trie.py:290-342) with _descend (trie.py:229-256).
 * mode 0 strict, 1 complete.  ids/lcps have room for min(k, n).
 * Returns the hit count; writes matched_depth and the WorkReport deltas. */
int64_t orc_trie_query(const orc_trie* t, const uint16_t* q, int64_t k, int32_t mode,
                       int32_t* ids, int64_t* lcps, int32_t* matched_depth, int64_t* symbols,
                       int64_t* nodes_visited) {
  const int64_t n = t->n;
  const int32_t L = t->L;
  int64_t pbuf[2 * 257];
  int64_t* plo = L <= 256 ? pbuf : (int64_t*)malloc((size_t)(L + 1) * 16);
  int64_t* phi = plo + (L + 1);
  int32_t pdepth = 0; /* path length - 1 */
  int64_t comparisons = 0;
  plo[0] = 0;
  phi[0] = n;
  if (n > 0) {
    int64_t lo = 0, hi = n;
    for (int32_t d = 0; d < L; ++d) {
      int64_t base = t->level_offset[d + 1], end = t->level_offset[d + 2];
      const int32_t* lvl = t->row_lo + base;
      int64_t c0 = base + lower_i32(lvl, end - base, (int32_t)lo);
      int64_t c1 = base + lower_i32(lvl, end - base, (int32_t)hi);
      comparisons += 1;
      const uint16_t* syms = t->edge + c0;
      int64_t j = lower_u16(syms, c1 - c0, q[d]);
      if (j == c1 - c0 || syms[j] != q[d]) break;
      int64_t node = c0 + j;
      lo = t->row_lo[node];
      hi = node + 1 < end ? t->row_lo[node + 1] : n;
      ++pdepth;
      plo[pdepth] = lo;
      phi[pdepth] = hi;
    }
  }
  *symbols = comparisons;
  int64_t nv = pdepth + 1;
  *matched_depth = pdepth;
  int64_t need = mode == 1 ? (k < n ? k : n) : k;
  int64_t got = collect_smallest(t->order, plo[pdepth], plo[pdepth], plo[pdepth], phi[pdepth],
                                 need, ids);
  for (int64_t i = 0; i < got; ++i) lcps[i] = pdepth;
  if (mode == 1 && got < need) {
    int64_t prev_lo = plo[pdepth], prev_hi = phi[pdepth];
    for (int32_t a = pdepth - 1; a >= 0; --a) {
      if (got >= need) break;
      nv += 1;
      int64_t m = collect_smallest(t->order, plo[a], prev_lo, prev_hi, phi[a], need - got,
                                   ids + got);
      for (int64_t i = 0; i < m; ++i) lcps[got + i] = a;
      got += m;
      prev_lo = plo[a];
      prev_hi = phi[a];
    }
  }
  *nodes_visited = nv;
  if (plo != pbuf) free(plo);
  return got;
}

/* ------------------------------------------------------------------ TAL */
typedef struct orc_tal {
  int64_t n;
  int32_t L, sigma, depth;
  int64_t buckets;  /* sigma**depth, -1 if > 2^62 */
  uint16_t* rows;   /* sorted */
  int64_t* item_index;
  int64_t* directory; /* buckets + 1 or NULL */
} orc_tal;

orc_tal* orc_tal_build(const uint16_t* items, int64_t n, int32_t L, int32_t sigma, int32_t depth) {
  orc_tal* e = (orc_tal*)calloc(1, sizeof(orc_tal));
  e->n = n;
  e->L = L;
  e->sigma = sigma;
  e->depth = depth;
  int64_t b = 1;
  for (int32_t j = 0; j < depth; ++j) {
    if (b > ((int64_t)1 << 62) / sigma) {
      b = -1;
      break;
    }
    b *= sigma;
  }
  e->buckets = b;
  e->item_index = (int64_t*)malloc((size_t)(n ? n : 1) * 8);
  orc_lexicographic_order(items, n, L, e->item_index);
  e->rows = (uint16_t*)malloc((size_t)(n ? n : 1) * L * 2);
  for (int64_t i = 0; i < n; ++i)
    memcpy(e->rows + i * L, items + e->item_index[i] * L, (size_t)L * 2);
  if (depth > 0 && b > 0 && b <= ((int64_t)1 << 24)) {
    /* directory[c] = searchsorted(codes, c), tal.py:76-82 */
    e->directory = (int64_t*)malloc((size_t)(b + 1) * 8);
    int64_t i = 0;
    for (int64_t c = 0; c <= b; ++c) {
      while (i < n) {
        int64_t code = 0;
        for (int32_t j = 0; j < depth; ++j) code = code * sigma + e->rows[i * L + j];
        if (code < c) ++i;
        else break;
      }
      e->directory[c] = i;
    }
  }
  return e;
}

void orc_tal_free(orc_tal* e) {
  if (!e) return;
  free(e->rows);
  free(e->item_index);
  free(e->directory);
  free(e);
}

int orc_tal_has_directory(const orc_tal* e) { return e->directory != NULL; }

void orc_tal_export(const orc_tal* e, int64_t* item_index, int64_t* directory) {
  if (item_index) memcpy(item_index, e->item_index, (size_t)e->n * 8);
  if (directory && e->directory) memcpy(directory, e->directory, (size_t)(e->buckets + 1) * 8);
}

/* bucket_range (tal.py:138-143): directory, else bucket_range_search (124-136) */
void orc_tal_bucket_range(const orc_tal* e, const uint16_t* q, int64_t* lo, int64_t* hi) {
  const int32_t d = e->depth, L = e->L;
  if (d == 0) {
    *lo = 0;
    *hi = e->n;
    return;
  }
  if (e->directory) {
    int64_t code = 0;
    for (int32_t j = 0; j < d; ++j) code = code * e->sigma + q[j];
    *lo = e->directory[code];
    *hi = e->directory[code + 1];
    return;
  }
  int64_t a = 0, b = e->n;
  while (a < b) {
    int64_t m = (a + b) >> 1;
    if (row_cmp(e->rows + m * L, q, d) < 0) a = m + 1;
    else b = m;
  }
  *lo = a;
  b = e->n;
  while (a < b) {
    int64_t m = (a + b) >> 1;
    if (row_cmp(e->rows + m * L, q, d) <= 0) a = m + 1;
    else b = m;
  }
  *hi = a;
}

/* TalEngine.query (tal.py:155-194); returns hits, writes counters */
int64_t orc_tal_query(const orc_tal* e, const uint16_t* q, int64_t k, int64_t* ids, int64_t* lcps,
                      int64_t* items_scanned, int64_t* symbols_compared) {
  int64_t lo, hi;
  orc_tal_bucket_range(e, q, &lo, &hi);
  const int32_t L = e->L;
  int64_t size = hi - lo;
  *items_scanned = 0;
  *symbols_compared = 0;
  if (size == 0) return 0;
  uint64_t* comp = (uint64_t*)malloc((size_t)size * 8);
  int64_t sym = 0;
  for (int64_t i = 0; i < size; ++i) {
    int64_t l = row_lcp(e->rows + (lo + i) * L, q, L);
    sym += (l + 1 < L ? l + 1 : L);
    comp[i] = ((uint64_t)(L - l) << 32) | (uint64_t)e->item_index[lo + i];
  }
  *items_scanned = size;
  *symbols_compared = sym;
  int64_t take = k < size ? k : size;
  uint64_t* sel = (uint64_t*)malloc((size_t)take * 8);
  smallest_u64(comp, size, take, sel);
  for (int64_t i = 0; i < take; ++i) {
    ids[i] = (int64_t)(sel[i] & 0xffffffffu);
    lcps[i] = L - (int64_t)(sel[i] >> 32);
  }
  free(sel);
  free(comp);
  return take;
}

/* ------------------------------------------------ oracle.oracle_top_k */
int64_t orc_oracle_top_k(const uint16_t* items, int64_t n, int32_t L, const uint16_t* q,
                         int64_t k, int64_t* ids, int64_t* lcps) {
  int64_t take = k < n ? k : n;
  if (take <= 0) return 0;
  /* bounded max-heap over the composite (L - lcp) << 32 | idx */
  uint64_t* heap = (uint64_t*)malloc((size_t)take * 8);
  int64_t sz = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t l = row_lcp(items + i * L, q, L);
    uint64_t c = ((uint64_t)(L - l) << 32) | (uint64_t)i;
    if (sz < take) {
      heap[sz++] = c;
      if (sz == take)
        for (int64_t h = take / 2 - 1; h >= 0; --h) heap_sift_down(heap, take, h);
    } else if (c < heap[0]) {
      heap[0] = c;
      heap_sift_down(heap, take, 0);
    }
  }
  qsort(heap, (size_t)take, 8, cmp_u64);
  for (int64_t i = 0; i < take; ++i) {
    ids[i] = (int64_t)(heap[i] & 0xffffffffu);
    lcps[i] = L - (int64_t)(heap[i] >> 32);
  }
  free(heap);
  return take;
}

/* --------------------------------------------------------- batch drivers
 * out rows have stride `stride` (>= min(k, n)).  Queries are handed out to
 * `nthreads` pthreads in blocks of 16 through an atomic cursor. */
typedef struct {
  int kind; /* 0 trie, 1 tal, 2 oracle */
  const void* eng;
  const uint16_t* items;
  int64_t n;
  int32_t L;
  const uint16_t* qs;
  int64_t count, k, stride;
  int32_t mode;
  void* ids;
  int64_t* lcps;
  int64_t* hits;
  int32_t* matched_depth;
  int64_t* c0;
  int64_t* c1;
  int64_t cursor;
} batch_job;

static void run_one(batch_job* j, int64_t i) {
  if (j->kind == 0) {
    const orc_trie* t = (const orc_trie*)j->eng;
    j->hits[i] = orc_trie_query(t, j->qs + i * t->L, j->k, j->mode,
                                (int32_t*)j->ids + i * j->stride, j->lcps + i * j->stride,
                                j->matched_depth + i, j->c0 + i, j->c1 + i);
  } else if (j->kind == 1) {
    const orc_tal* e = (const orc_tal*)j->eng;
    j->hits[i] = orc_tal_query(e, j->qs + i * e->L, j->k, (int64_t*)j->ids + i * j->stride,
                               j->lcps + i * j->stride, j->c0 + i, j->c1 + i);
  } else {
    j->hits[i] = orc_oracle_top_k(j->items, j->n, j->L, j->qs + i * j->L, j->k,
                                  (int64_t*)j->ids + i * j->stride, j->lcps + i * j->stride);
  }
}

static void* worker(void* arg) {
  batch_job* j = (batch_job*)arg;
  for (;;) {
    int64_t a = __atomic_fetch_add(&j->cursor, 16, __ATOMIC_RELAXED);
    if (a >= j->count) break;
    int64_t b = a + 16 < j->count ? a + 16 : j->count;
    for (int64_t i = a; i < b; ++i) run_one(j, i);
  }
  return NULL;
}

static void run_batch(batch_job* j, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  j->cursor = 0;
  if (nthreads == 1) {
    worker(j);
    return;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, worker, j);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th);
}

void orc_trie_query_batch(const orc_trie* t, const uint16_t* qs, int64_t count, int64_t k,
                          int32_t mode, int64_t stride, int32_t* ids, int64_t* lcps,
                          int64_t* hits, int32_t* matched_depth, int64_t* symbols,
                          int64_t* nodes, int32_t nthreads) {
  batch_job j = {0};
  j.kind = 0; j.eng = t; j.qs = qs; j.count = count; j.k = k; j.stride = stride; j.mode = mode;
  j.ids = ids; j.lcps = lcps; j.hits = hits; j.matched_depth = matched_depth;
  j.c0 = symbols; j.c1 = nodes;
  run_batch(&j, nthreads);
}

void orc_tal_query_batch(const orc_tal* e, const uint16_t* qs, int64_t count, int64_t k,
                         int64_t stride, int64_t* ids, int64_t* lcps, int64_t* hits,
                         int64_t* items_scanned, int64_t* symbols, int32_t nthreads) {
  batch_job j = {0};
  j.kind = 1; j.eng = e; j.qs = qs; j.count = count; j.k = k; j.stride = stride;
  j.ids = ids; j.lcps = lcps; j.hits = hits; j.c0 = items_scanned; j.c1 = symbols;
  run_batch(&j, nthreads);
}

void orc_oracle_top_k_batch(const uint16_t* items, int64_t n, int32_t L, const uint16_t* qs,
                            int64_t count, int64_t k, int64_t stride, int64_t* ids, int64_t* lcps,
                            int64_t* hits, int32_t nthreads) {
  batch_job j = {0};
  j.kind = 2; j.items = items; j.n = n; j.L = L; j.qs = qs; j.count = count; j.k = k;
  j.stride = stride; j.ids = ids; j.lcps = lcps; j.hits = hits;
  run_batch(&j, nthreads);
}
