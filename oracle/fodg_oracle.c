/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see fodg_oracle.h).
 *
 * Plain-C restatement of the reference CPU algorithms of the CAGRA hot path.
 * Compiled with -ffp-contract=off so every distance is the reference's
 * sequential fp32 chain without FMA contraction (dataset.hpp:33-43).
 * Parallelism (OpenMP) is only over independent rows / queries, so results do
 * not depend on the thread count (common.hpp:47-49 contract).
 */
#include "fodg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ID_MASK 0x7fffffffu
#define PARENT 0x80000000u
#define INVALID 0xffffffffu

enum { OK = 0, USAGE = 2, LOGIC = 6 };

/* ---------------------------------------------------------------- basics -- */

/* common.hpp:34-39 */
uint64_t orc_mix_seed(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* tests/test_util.hpp:11-18: std::mt19937_64 + uniform_real_distribution<float>
 * (libstdc++: generate_canonical<float,24> takes one 64-bit draw and scales it
 * by 2^-64 in float, clamping 1.0 to the float below it). */
void orc_uniform_dataset(uint64_t seed, uint64_t count, float* out) {
  enum { NN = 312, MM = 156 };
  uint64_t mt[NN];
  int idx;
  mt[0] = seed;
  for (idx = 1; idx < NN; ++idx)
    mt[idx] = 6364136223846793005ull * (mt[idx - 1] ^ (mt[idx - 1] >> 62)) + (uint64_t)idx;
  idx = NN;
  const float two64 = 18446744073709551616.0f;
  for (uint64_t i = 0; i < count; ++i) {
    if (idx >= NN) {
      for (int j = 0; j < NN; ++j) {
        uint64_t y = (mt[j] & 0xffffffff80000000ull) | (mt[(j + 1) % NN] & 0x7fffffffull);
        uint64_t v = mt[(j + MM) % NN] ^ (y >> 1);
        if (y & 1ull) v ^= 0xb5026f5aa96619e9ull;
        mt[j] = v;
      }
      idx = 0;
    }
    uint64_t x = mt[idx++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71d67fffeda60000ull;
    x ^= (x << 37) & 0xfff7eee000000000ull;
    x ^= (x >> 43);
    float r = (float)x / two64;
    if (r >= 1.0f) r = nextafterf(1.0f, 0.0f);
    out[i] = r * 1.0f + 0.0f;
  }
}

/* dataset.hpp:33-43 — strictly sequential, separate mul and add. */
float orc_squared_l2(const float* a, const float* b, uint32_t dim) {
  float acc = 0.0f;
  for (uint32_t i = 0; i < dim; ++i) {
    float diff = a[i] - b[i];
    acc += diff * diff;
  }
  return acc;
}

/* (dist, id) strict order, topk.cpp:15-19 / search.hpp:35-38 */
static int pair_less(float da, uint32_t ia, float db, uint32_t ib) {
  if (da != db) return da < db;
  return ia < ib;
}

/* ------------------------------------------------------------ exact top-k -- */

/* topk.cpp:10-43 restated: keep the k best by (dist, id) in an ascending
 * array; a new point enters only if it beats the current worst. */
int orc_exact_topk(const float* data, uint32_t n, uint32_t dim, const float* q, uint32_t k,
                   uint32_t* ids, float* dists) {
  if (k == 0 || k > n) return USAGE;
  uint32_t filled = 0;
  for (uint32_t i = 0; i < n; ++i) {
    float d = orc_squared_l2(data + (size_t)i * dim, q, dim);
    if (filled == k && !pair_less(d, i, dists[k - 1], ids[k - 1])) continue;
    uint32_t pos = filled < k ? filled : k - 1;
    while (pos > 0 && pair_less(d, i, dists[pos - 1], ids[pos - 1])) {
      dists[pos] = dists[pos - 1];
      ids[pos] = ids[pos - 1];
      --pos;
    }
    dists[pos] = d;
    ids[pos] = i;
    if (filled < k) ++filled;
  }
  return OK;
}

int orc_exact_topk_batch(const float* data, uint32_t n, uint32_t dim, const float* qs,
                         uint32_t nq, uint32_t k, uint32_t* ids, float* dists, int threads) {
  if (k == 0 || k > n) return USAGE;
  (void)threads;
#pragma omp parallel for schedule(dynamic, 4) num_threads(threads > 0 ? threads : omp_get_max_threads())
  for (int64_t qi = 0; qi < (int64_t)nq; ++qi)
    orc_exact_topk(data, n, dim, qs + (size_t)qi * dim, k, ids + (size_t)qi * k,
                   dists + (size_t)qi * k);
  return OK;
}

/* knn_build.cpp:40-63: top-(k+1) of the node's own row, self dropped. */
int orc_exact_knn_graph(const float* data, uint32_t n, uint32_t dim, uint32_t k,
                        uint32_t* ids, float* dists, int threads) {
  if (k == 0 || k >= n) return USAGE;
  (void)threads;
#pragma omp parallel num_threads(threads > 0 ? threads : omp_get_max_threads())
  {
    uint32_t* tid = (uint32_t*)malloc(sizeof(uint32_t) * (k + 1));
    float* tdist = (float*)malloc(sizeof(float) * (k + 1));
#pragma omp for schedule(dynamic, 16)
    for (int64_t vi = 0; vi < (int64_t)n; ++vi) {
      uint32_t v = (uint32_t)vi;
      orc_exact_topk(data, n, dim, data + (size_t)v * dim, k + 1, tid, tdist);
      uint32_t w = 0;
      for (uint32_t j = 0; j <= k && w < k; ++j) {
        if (tid[j] == v) continue;
        ids[(size_t)v * k + w] = tid[j];
        dists[(size_t)v * k + w] = tdist[j];
        ++w;
      }
    }
    free(tid);
    free(tdist);
  }
  return OK;
}

/* ------------------------------------------------------- graph optimize -- */

/* graph_opt.cpp:19-31 */
static int rows_sorted(const uint32_t* ids, const float* dists, uint32_t n, uint32_t deg) {
  for (uint64_t v = 0; v < n; ++v) {
    const uint32_t* r = ids + v * deg;
    const float* dd = dists + v * deg;
    for (uint32_t j = 1; j < deg; ++j)
      if (!(dd[j - 1] < dd[j] || (dd[j - 1] == dd[j] && r[j - 1] < r[j]))) return 0;
  }
  return 1;
}

typedef struct {
  uint32_t id, rank;
} idrank;

static int idrank_cmp(const void* a, const void* b) {
  uint32_t x = ((const idrank*)a)->id, y = ((const idrank*)b)->id;
  return x < y ? -1 : x > y;
}

/* graph_opt.cpp:45-96, rank mode: for each X, each Z = row[rz], each
 * Y = Z.row[rzy] with Y != X that is X's rank-ry neighbour (ry != rz), count
 * the route when max(rz, rzy) < ry. */
int orc_count_detourable_routes(const uint32_t* ids, const float* dists, uint32_t n,
                                uint32_t deg, uint32_t* counts) {
  if (!rows_sorted(ids, dists, n, deg)) return USAGE;
#pragma omp parallel
  {
    idrank* tab = (idrank*)malloc(sizeof(idrank) * deg);
#pragma omp for schedule(dynamic, 64)
    for (int64_t xi = 0; xi < (int64_t)n; ++xi) {
      uint32_t x = (uint32_t)xi;
      const uint32_t* xrow = ids + (size_t)x * deg;
      uint32_t* cnt = counts + (size_t)x * deg;
      for (uint32_t r = 0; r < deg; ++r) {
        tab[r].id = xrow[r];
        tab[r].rank = r;
        cnt[r] = 0;
      }
      qsort(tab, deg, sizeof(idrank), idrank_cmp);
      for (uint32_t rz = 0; rz < deg; ++rz) {
        const uint32_t* zrow = ids + (size_t)xrow[rz] * deg;
        for (uint32_t rzy = 0; rzy < deg; ++rzy) {
          uint32_t y = zrow[rzy];
          if (y == x) continue;
          uint32_t lo = 0, hi = deg;
          while (lo < hi) {
            uint32_t mid = (lo + hi) / 2;
            if (tab[mid].id < y) lo = mid + 1; else hi = mid;
          }
          if (lo == deg || tab[lo].id != y) continue;
          uint32_t ry = tab[lo].rank;
          if (ry == rz) continue;
          uint32_t mx = rz > rzy ? rz : rzy;
          if (mx < ry) ++cnt[ry];
        }
      }
    }
    free(tab);
  }
  return OK;
}

static int u64_cmp(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

/* graph_opt.cpp:98-124: stable sort of each row by count (ties keep the
 * initial rank), first d kept.  Stability comes from the (count, rank) key. */
int orc_reorder_and_prune(const uint32_t* ids, const uint32_t* counts, uint32_t n,
                          uint32_t deg, uint32_t d, uint32_t* pruned) {
  if (d == 0 || d > deg) return USAGE;
#pragma omp parallel
  {
    uint64_t* key = (uint64_t*)malloc(sizeof(uint64_t) * deg);
#pragma omp for schedule(static)
    for (int64_t v = 0; v < (int64_t)n; ++v) {
      for (uint32_t r = 0; r < deg; ++r)
        key[r] = ((uint64_t)counts[(size_t)v * deg + r] << 32) | r;
      qsort(key, deg, sizeof(uint64_t), u64_cmp);
      for (uint32_t j = 0; j < d; ++j)
        pruned[(size_t)v * d + j] = ids[(size_t)v * deg + (uint32_t)(key[j] & 0xffffffffu)];
    }
    free(key);
  }
  return OK;
}

/* graph_opt.cpp:141-160: row y = sources x of edges x->y ordered by
 * (rank of x->y, x), at most cap.  Restated with a counting pass + per-row
 * sort of (rank, source) keys. */
int orc_build_reverse_graph(const uint32_t* pruned, uint32_t n, uint32_t d, uint32_t cap,
                            uint32_t* rev_counts, uint32_t* rev_ids) {
  uint64_t* start = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  uint64_t edges = (uint64_t)n * d;
  for (uint64_t e = 0; e < edges; ++e) start[pruned[e] + 1]++;
  for (uint32_t y = 0; y < n; ++y) start[y + 1] += start[y];
  uint64_t* fill = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)n + 1));
  memcpy(fill, start, sizeof(uint64_t) * ((size_t)n + 1));
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (edges ? edges : 1));
  for (uint64_t x = 0; x < n; ++x)
    for (uint32_t r = 0; r < d; ++r) {
      uint32_t y = pruned[x * d + r];
      keys[fill[y]++] = ((uint64_t)r << 32) | x;
    }
  for (uint32_t y = 0; y < n; ++y) {
    uint64_t len = start[y + 1] - start[y];
    qsort(keys + start[y], len, sizeof(uint64_t), u64_cmp);
    uint32_t keep = len < cap ? (uint32_t)len : cap;
    rev_counts[y] = keep;
    for (uint32_t j = 0; j < keep; ++j)
      rev_ids[(size_t)y * cap + j] = (uint32_t)(keys[start[y] + j] & 0xffffffffu);
  }
  free(start);
  free(fill);
  free(keys);
  return OK;
}

/* graph_opt.cpp:162-209: slots alternate pruned (even) / reverse (odd); an
 * exhausted side is compensated by the other; ids already emitted are skipped
 * (and consumed). */
int orc_merge_graphs(const uint32_t* pruned, const uint32_t* rev_counts,
                     const uint32_t* rev_ids, uint32_t n, uint32_t d, uint32_t rev_cap,
                     uint32_t* out) {
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t v = 0; v < (int64_t)n; ++v) {
    const uint32_t* p = pruned + (size_t)v * d;
    const uint32_t* r = rev_ids + (size_t)v * rev_cap;
    uint32_t plen = d, rlen = rev_counts[v];
    uint32_t* o = out + (size_t)v * d;
    uint32_t pi = 0, ri = 0, emitted = 0;
    for (uint32_t slot = 0; slot < d; ++slot) {
      int got = 0;
      uint32_t id = 0;
      for (int attempt = 0; attempt < 2 && !got; ++attempt) {
        int from_p = ((slot % 2 == 0) ^ (attempt == 1));
        const uint32_t* src = from_p ? p : r;
        uint32_t* pos = from_p ? &pi : &ri;
        uint32_t len = from_p ? plen : rlen;
        while (*pos < len && !got) {
          uint32_t cand = src[(*pos)++];
          int dup = 0;
          for (uint32_t j = 0; j < emitted; ++j)
            if (o[j] == cand) { dup = 1; break; }
          if (!dup) { id = cand; got = 1; }
        }
      }
      if (!got) { bad = 1; break; }
      o[emitted++] = id;
    }
  }
  return bad ? USAGE : OK;
}

/* graph_opt.cpp:211-246, rank mode, reorder + add_reverse. */
int orc_optimize(const uint32_t* ids, const float* dists, uint32_t n, uint32_t deg,
                 uint32_t d, uint32_t* out) {
  if (d == 0 || d > deg) return USAGE;
  uint32_t* counts = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n * deg);
  uint32_t* pr = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n * d);
  uint32_t* rc = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
  uint32_t* ri = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n * d);
  int rc0 = orc_count_detourable_routes(ids, dists, n, deg, counts);
  if (!rc0) rc0 = orc_reorder_and_prune(ids, counts, n, deg, d, pr);
  if (!rc0) rc0 = orc_build_reverse_graph(pr, n, d, d, rc, ri);
  if (!rc0) rc0 = orc_merge_graphs(pr, rc, ri, n, d, d, out);
  free(counts);
  free(pr);
  free(rc);
  free(ri);
  return rc0;
}

/* ------------------------------------------------------------------ search -- */

typedef struct {
  uint32_t id;
  float dist;
} entry;

/* search.cpp:33-37 */
uint32_t orc_resolved_max_iterations(const orc_params* p) {
  if (p->max_iterations) return p->max_iterations;
  uint32_t it = (2 * p->topm + p->width - 1) / p->width;
  return it < 16 ? 16 : it > 256 ? 256 : it;
}

/* search.cpp:39-50 */
int orc_validate(const orc_params* p) {
  if (p->k == 0 || p->k > p->topm || p->width == 0) return USAGE;
  if (p->min_iterations > orc_resolved_max_iterations(p)) return USAGE;
  if (p->hash_policy == 1) {
    if (p->hash_bits < 4 || p->hash_bits > 24 || p->reset_interval == 0) return USAGE;
  }
  return OK;
}

/* VisitedTable (search.cpp:100-136): multiplicative hash + linear probing;
 * "full" is checked before probing. */
typedef struct {
  uint32_t* slot;
  uint32_t mask, count, forget;
} vtab;

enum { INS_NEW, INS_PRESENT, INS_FULL };

static int vt_init(vtab* t, uint32_t cap, uint32_t forget) {
  t->slot = (uint32_t*)malloc(sizeof(uint32_t) * cap);
  if (!t->slot) return LOGIC;
  memset(t->slot, 0xff, sizeof(uint32_t) * cap);
  t->mask = cap - 1;
  t->count = 0;
  t->forget = forget;
  return OK;
}

static int vt_insert(vtab* t, uint32_t id) {
  if (t->count == t->mask + 1) return INS_FULL;
  uint32_t h = (id * 2654435761u) & t->mask;
  for (;;) {
    uint32_t s = t->slot[h];
    if (s == INVALID) break;
    if (s == id) return INS_PRESENT;
    h = (h + 1) & t->mask;
  }
  t->slot[h] = id;
  t->count++;
  return INS_NEW;
}

static void vt_clear(vtab* t) {
  memset(t->slot, 0xff, sizeof(uint32_t) * (t->mask + 1));
  t->count = 0;
}

/* next_pow2 of 2*max(1,expected), search.cpp:14-19 + 104-108 */
static int standard_capacity(uint64_t expected, uint32_t* cap) {
  uint64_t want = 2 * (expected ? expected : 1), c = 1;
  while (c < want) c <<= 1;
  if (c > (1ull << 31)) return USAGE;
  *cap = (uint32_t)c;
  return OK;
}

typedef struct {
  const uint32_t* graph;
  uint32_t n, deg;
  const float* data;
  uint32_t dim;
  const float* q;
  orc_params p;
  uint32_t max_iter;
  entry* buf; /* m + c */
  uint32_t m, c;
  vtab own;
  vtab* tab;
  orc_stats st;
  uint64_t rng;
  int pending, done, err;
} trav;

static int entry_cmp(const void* a, const void* b) {
  const entry* x = (const entry*)a;
  const entry* y = (const entry*)b;
  if (x->dist != y->dist) return x->dist < y->dist ? -1 : 1;
  uint32_t ix = x->id & ID_MASK, iy = y->id & ID_MASK;
  return ix < iy ? -1 : ix > iy;
}

/* update_topm (search.cpp:55-85), restated as the reference test suite's own
 * equivalent definition (test_search.cpp:22-36): drop dummies, collapse equal
 * ids OR-ing the parent flag, full sort, keep M, pad dummies. */
static void update_topm(trav* t, entry* scratch) {
  uint32_t total = t->m + t->c, live = 0;
  for (uint32_t i = 0; i < total; ++i)
    if (t->buf[i].id != INVALID) scratch[live++] = t->buf[i];
  qsort(scratch, live, sizeof(entry), entry_cmp);
  uint32_t out = 0;
  for (uint32_t i = 0; i < live; ++i) {
    if (out && (scratch[out - 1].id & ID_MASK) == (scratch[i].id & ID_MASK)) {
      scratch[out - 1].id |= scratch[i].id & PARENT;
      continue;
    }
    scratch[out++] = scratch[i];
  }
  for (uint32_t i = 0; i < t->m; ++i) {
    if (i < out) t->buf[i] = scratch[i];
    else { t->buf[i].id = INVALID; t->buf[i].dist = INFINITY; }
  }
}

static void reset_with_topm(trav* t) {
  vt_clear(t->tab);
  for (uint32_t i = 0; i < t->m; ++i)
    if (t->buf[i].id != INVALID) vt_insert(t->tab, t->buf[i].id & ID_MASK);
}

/* eval_or_skip, search.cpp:168-190 */
static float eval_or_skip(trav* t, uint32_t id, int* evaluated) {
  int r = vt_insert(t->tab, id);
  if (r == INS_FULL) {
    if (t->tab->forget) {
      reset_with_topm(t);
      t->st.hash_resets++;
      r = vt_insert(t->tab, id);
    } else {
      t->err = LOGIC;
      r = INS_PRESENT;
    }
  }
  if (r == INS_NEW) {
    *evaluated = 1;
    t->st.distance_evals++;
    return orc_squared_l2(t->data + (size_t)id * t->dim, t->q, t->dim);
  }
  *evaluated = 0;
  return INFINITY;
}

/* Traversal ctor, search.cpp:147-166 (validation order kept) */
static int trav_init(trav* t, const uint32_t* graph, uint32_t n, uint32_t deg,
                     const float* data, uint32_t dim, const float* q, const orc_params* p,
                     vtab* shared) {
  memset(t, 0, sizeof(*t));
  if (orc_validate(p)) return USAGE;
  t->graph = graph;
  t->n = n;
  t->deg = deg;
  t->data = data;
  t->dim = dim;
  t->q = q;
  t->p = *p;
  t->max_iter = orc_resolved_max_iterations(p);
  t->m = p->topm;
  t->c = p->width * deg;
  t->buf = (entry*)malloc(sizeof(entry) * (t->m + t->c));
  for (uint32_t i = 0; i < t->m + t->c; ++i) {
    t->buf[i].id = INVALID;
    t->buf[i].dist = INFINITY;
  }
  if (shared) {
    t->tab = shared;
  } else {
    uint32_t cap;
    if (p->hash_policy == 1) {
      cap = 1u << p->hash_bits;
    } else if (standard_capacity((uint64_t)(t->max_iter + 1) * p->width * deg, &cap)) {
      free(t->buf);
      t->buf = NULL;
      return USAGE;
    }
    vt_init(&t->own, cap, p->hash_policy == 1);
    t->tab = &t->own;
  }
  t->rng = orc_mix_seed(p->seed ^ 0x5eedull);
  return OK;
}

static void trav_free(trav* t) {
  free(t->buf);
  if (t->tab == &t->own) free(t->own.slot);
}

/* init, search.cpp:192-201 */
static void trav_start(trav* t) {
  entry* cand = t->buf + t->m;
  for (uint32_t j = 0; j < t->c; ++j) {
    t->rng = orc_mix_seed(t->rng);
    uint32_t id = (uint32_t)(t->rng % t->n);
    int ev = 0;
    float d = eval_or_skip(t, id, &ev);
    cand[j].id = ev ? id : INVALID;
    cand[j].dist = ev ? d : INFINITY;
  }
  t->pending = 1;
}

/* step, search.cpp:218-245 (select_parents :87-98, expand :203-216) */
static int trav_step(trav* t, entry* scratch, uint32_t* parents) {
  if (t->done) return 0;
  update_topm(t, scratch);
  t->pending = 0;
  t->st.iterations++;
  uint32_t np = 0;
  for (uint32_t i = 0; i < t->m && np < t->p.width; ++i) {
    entry* e = &t->buf[i];
    if (e->id == INVALID || (e->id & PARENT)) continue;
    parents[np++] = e->id & ID_MASK;
    e->id |= PARENT;
  }
  if (np == 0) {
    t->st.converged = t->st.iterations >= t->p.min_iterations;
    t->done = 1;
    return 0;
  }
  entry* cand = t->buf + t->m;
  uint32_t slot = 0;
  for (uint32_t pi = 0; pi < np; ++pi) {
    const uint32_t* row = t->graph + (size_t)parents[pi] * t->deg;
    for (uint32_t j = 0; j < t->deg; ++j) {
      int ev = 0;
      float d = eval_or_skip(t, row[j], &ev);
      cand[slot].id = ev ? row[j] : INVALID;
      cand[slot].dist = ev ? d : INFINITY;
      ++slot;
    }
  }
  for (; slot < t->c; ++slot) {
    cand[slot].id = INVALID;
    cand[slot].dist = INFINITY;
  }
  t->pending = 1;
  if (t->tab->forget && t->st.iterations % t->p.reset_interval == 0) {
    reset_with_topm(t);
    t->st.hash_resets++;
  }
  if (t->st.iterations >= t->max_iter) t->done = 1;
  return !t->done;
}

/* finish, search.cpp:247-259 */
static uint32_t trav_finish(trav* t, entry* scratch, uint32_t k, uint32_t* ids, float* dists) {
  if (t->pending) update_topm(t, scratch);
  uint32_t w = 0;
  for (uint32_t i = 0; i < t->m && w < k; ++i) {
    if (t->buf[i].id == INVALID) break;
    ids[w] = t->buf[i].id & ID_MASK;
    dists[w] = t->buf[i].dist;
    ++w;
  }
  return w;
}

int orc_search_one(const uint32_t* graph, uint32_t n, uint32_t degree, const float* data,
                   uint32_t dim, const float* query, const orc_params* p, uint32_t* ids,
                   float* dists, uint32_t* count, orc_stats* st) {
  trav t;
  int rc = trav_init(&t, graph, n, degree, data, dim, query, p, NULL);
  if (rc) return rc;
  entry* scratch = (entry*)malloc(sizeof(entry) * (t.m + t.c));
  uint32_t* parents = (uint32_t*)malloc(sizeof(uint32_t) * p->width);
  trav_start(&t);
  while (trav_step(&t, scratch, parents)) {
  }
  *count = trav_finish(&t, scratch, p->k, ids, dists);
  for (uint32_t i = *count; i < p->k; ++i) {
    ids[i] = INVALID;
    dists[i] = INFINITY;
  }
  if (st) *st = t.st;
  rc = t.err;
  free(scratch);
  free(parents);
  trav_free(&t);
  return rc;
}

typedef struct {
  float d;
  uint32_t id;
} pool_ent;

static int pool_cmp(const void* a, const void* b) {
  const pool_ent* x = (const pool_ent*)a;
  const pool_ent* y = (const pool_ent*)b;
  if (x->d != y->d) return x->d < y->d ? -1 : 1;
  return x->id < y->id ? -1 : x->id > y->id;
}

/* shared_query_search + merge_team_results, engine.cpp:12-78 */
static int shared_search(const uint32_t* graph, uint32_t n, uint32_t degree,
                         const float* data, uint32_t dim, const float* q,
                         const orc_params* p, uint32_t teams, uint64_t qseed, uint32_t* ids,
                         float* dists, uint32_t* count, orc_stats* st) {
  orc_params tp = *p;
  tp.width = 1;
  tp.k = p->topm;
  tp.hash_policy = 0;
  uint32_t tmax = orc_resolved_max_iterations(&tp);
  if (tp.min_iterations > tmax) tp.min_iterations = tmax;
  uint32_t cap;
  if (standard_capacity((uint64_t)(tmax + 1) * teams * degree, &cap)) return USAGE;
  vtab shared;
  vt_init(&shared, cap, 0);
  trav* tv = (trav*)calloc(teams, sizeof(trav));
  int rc = OK;
  for (uint32_t t = 0; t < teams && !rc; ++t) {
    orc_params pp = tp;
    pp.seed = orc_mix_seed(qseed + 0x7ea4ull * (t + 1));
    rc = trav_init(&tv[t], graph, n, degree, data, dim, q, &pp, &shared);
  }
  entry* scratch = (entry*)malloc(sizeof(entry) * (p->topm + degree));
  uint32_t parent;
  if (!rc) {
    for (uint32_t t = 0; t < teams; ++t) trav_start(&tv[t]);
    int progressed = 1;
    while (progressed) { /* lockstep rounds, engine.cpp:63-72 */
      progressed = 0;
      for (uint32_t t = 0; t < teams; ++t)
        if (!tv[t].done) {
          trav_step(&tv[t], scratch, &parent);
          progressed = 1;
        }
    }
    pool_ent* pool = (pool_ent*)malloc(sizeof(pool_ent) * (size_t)teams * p->topm);
    uint32_t* tid = (uint32_t*)malloc(sizeof(uint32_t) * p->topm);
    float* tdist = (float*)malloc(sizeof(float) * p->topm);
    uint32_t np = 0;
    orc_stats agg;
    memset(&agg, 0, sizeof(agg));
    agg.converged = 1;
    for (uint32_t t = 0; t < teams; ++t) {
      uint32_t c = trav_finish(&tv[t], scratch, p->topm, tid, tdist);
      for (uint32_t i = 0; i < c; ++i) {
        pool[np].d = tdist[i];
        pool[np].id = tid[i];
        ++np;
      }
      agg.distance_evals += tv[t].st.distance_evals;
      agg.hash_resets += tv[t].st.hash_resets;
      if (tv[t].st.iterations > agg.iterations) agg.iterations = tv[t].st.iterations;
      agg.converged = agg.converged && tv[t].st.converged;
      if (tv[t].err) rc = tv[t].err;
    }
    qsort(pool, np, sizeof(pool_ent), pool_cmp);
    uint32_t w = 0, prev = INVALID;
    for (uint32_t i = 0; i < np && w < p->k; ++i) {
      if (pool[i].id == prev) continue;
      prev = pool[i].id;
      ids[w] = pool[i].id;
      dists[w] = pool[i].d;
      ++w;
    }
    *count = w;
    for (uint32_t i = w; i < p->k; ++i) {
      ids[i] = INVALID;
      dists[i] = INFINITY;
    }
    if (st) *st = agg;
    free(pool);
    free(tid);
    free(tdist);
  }
  for (uint32_t t = 0; t < teams; ++t)
    if (tv[t].buf) trav_free(&tv[t]);
  free(tv);
  free(scratch);
  free(shared.slot);
  return rc;
}

/* batch_search, engine.cpp:95-120 */
int orc_batch_search(const uint32_t* graph, uint32_t n, uint32_t degree, const float* data,
                     uint32_t dim, const float* queries, uint32_t nq, const orc_params* p,
                     uint32_t mode, uint32_t team_count, uint64_t query_offset,
                     uint32_t* ids, float* dists, uint32_t* counts, orc_stats* stats,
                     int threads) {
  if (nq == 0) return OK;
  if (orc_validate(p)) return USAGE;
  if (mode == 1 && team_count < 2) return USAGE;
  int rc = OK;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads > 0 ? threads : omp_get_max_threads()) reduction(max : rc)
  for (int64_t qi = 0; qi < (int64_t)nq; ++qi) {
    uint64_t qseed = orc_mix_seed(p->seed ^ (0x0badull + query_offset + (uint64_t)qi));
    const float* q = queries + (size_t)qi * dim;
    int r;
    if (mode == 0) {
      orc_params pp = *p;
      pp.seed = qseed;
      r = orc_search_one(graph, n, degree, data, dim, q, &pp, ids + (size_t)qi * p->k,
                         dists + (size_t)qi * p->k, counts + qi, stats ? stats + qi : NULL);
    } else {
      r = shared_search(graph, n, degree, data, dim, q, p, team_count, qseed,
                        ids + (size_t)qi * p->k, dists + (size_t)qi * p->k, counts + qi,
                        stats ? stats + qi : NULL);
    }
    if (r > rc) rc = r;
  }
  return rc;
}
