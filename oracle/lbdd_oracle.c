/*
 * lbdd_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference ASRAL solver, used by tests/ as the
 * parity checker and by bench.py as the "port" CPU baseline. It is never
 * linked into, loaded by, or called from the product package. Each function
 * cites the reference lines it restates
 * (/root/reference/proj/include/lbdd/...). Pinned against the unmodified
 * reference (oracle/_ref) and the reference tests' known answers by
 * tests/test_oracle_pinning.py.
 */
#define _GNU_SOURCE
#include "lbdd_oracle.h"

#include <math.h>
#include <setjmp.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ */
/* errors: reference exceptions become longjmp to the entry point      */
/* ------------------------------------------------------------------ */

static __thread char g_err[256];
static __thread jmp_buf* g_jmp;
static __thread int g_code;

const char* lbdd_oracle_last_error(void) { return g_err; }

static void raise_err(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  g_code = code;
  longjmp(*g_jmp, 1);
}

/* allocation arena, released on both normal and error exits */
typedef struct {
  void** ptrs;
  size_t len, cap;
  void** heaps; /* Heap arrays whose per-heap buffers are released at exit */
  int64_t* heap_counts;
  size_t nheaps;
} Arena;
static __thread Arena* g_arena;

static void* xalloc(size_t bytes) {
  void* p = calloc(1, bytes ? bytes : 1);
  if (!p) raise_err(LBDD_ERR_RUNTIME, "oracle: out of memory");
  if (g_arena->len == g_arena->cap) {
    g_arena->cap = g_arena->cap ? 2 * g_arena->cap : 64;
    g_arena->ptrs = realloc(g_arena->ptrs, g_arena->cap * sizeof(void*));
  }
  g_arena->ptrs[g_arena->len++] = p;
  return p;
}

static void register_heaps(void* heaps, int64_t count) {
  g_arena->heaps = realloc(g_arena->heaps, sizeof(void*) * (g_arena->nheaps + 1));
  g_arena->heap_counts =
      realloc(g_arena->heap_counts, sizeof(int64_t) * (g_arena->nheaps + 1));
  g_arena->heaps[g_arena->nheaps] = heaps;
  g_arena->heap_counts[g_arena->nheaps] = count;
  g_arena->nheaps++;
}
static void release_heaps(Arena* a);

#define ENTRY_BEGIN                      \
  jmp_buf jb__;                          \
  Arena arena__ = {0};                   \
  jmp_buf* prev_jmp__ = g_jmp;           \
  Arena* prev_arena__ = g_arena;         \
  g_jmp = &jb__;                         \
  g_arena = &arena__;                    \
  volatile int rc__ = LBDD_OK;           \
  if (setjmp(jb__)) {                    \
    rc__ = g_code;                       \
  } else {
#define ENTRY_END                                            \
  }                                                          \
  release_heaps(&arena__);                                   \
  for (size_t i__ = 0; i__ < arena__.len; ++i__) free(arena__.ptrs[i__]); \
  free(arena__.ptrs);                                        \
  g_jmp = prev_jmp__;                                        \
  g_arena = prev_arena__;                                    \
  return rc__;

/* core.hpp:25-39 checked 64-bit arithmetic */
static int64_t checked_add(int64_t a, int64_t b) {
  int64_t r;
  if (__builtin_add_overflow(a, b, &r))
    raise_err(LBDD_ERR_OVERFLOW, "lbdd: cost accumulator overflow");
  return r;
}
static int64_t checked_mul(int64_t a, int64_t b) {
  int64_t r;
  if (__builtin_mul_overflow(a, b, &r))
    raise_err(LBDD_ERR_OVERFLOW, "lbdd: cost accumulator overflow");
  return r;
}

static int64_t now_ns(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (int64_t)ts.tv_sec * 1000000000LL + ts.tv_nsec;
}

/* ------------------------------------------------------------------ */
/* instance                                                            */
/* ------------------------------------------------------------------ */

typedef struct {
  int64_t n, k;
  const int32_t* cm; /* n*k */
  const int64_t* cap;
  const int32_t* fam;
  const int64_t* off;
  const int64_t* par;
} Inst;

static Inst inst_from(const lbdd_instance_desc* d) {
  Inst I = {d->n, d->k, d->costs, d->capacity, d->penalty_family,
            d->penalty_offset, d->penalty_params};
  return I;
}

static inline int64_t CM(const Inst* I, int64_t d, int64_t s) {
  return I->cm[d * I->k + s];
}

/* PenaltySpec::at, core.hpp:60-74 */
static int64_t pen_at(const Inst* I, int64_t s, int64_t j) {
  if (j < 1) raise_err(LBDD_ERR_LOGIC, "lbdd: penalty index must be >= 1");
  const int64_t* p = I->par + I->off[s];
  switch (I->fam[s]) {
    case LBDD_PENALTY_CONSTANT: return p[0];
    case LBDD_PENALTY_LINEAR: return checked_add(p[0], checked_mul(p[1], j - 1));
    case LBDD_PENALTY_TABLE: {
      const int64_t len = I->off[s + 1] - I->off[s];
      const int64_t idx = j < len ? j : len;
      return p[idx - 1];
    }
  }
  raise_err(LBDD_ERR_LOGIC, "lbdd: bad penalty family");
  return 0;
}

/* PenaltySpec::total, core.hpp:77-95 */
static int64_t pen_total(const Inst* I, int64_t s, int64_t m) {
  if (m <= 0) return 0;
  const int64_t* p = I->par + I->off[s];
  switch (I->fam[s]) {
    case LBDD_PENALTY_CONSTANT: return checked_mul(p[0], m);
    case LBDD_PENALTY_LINEAR: {
      const int64_t tri = checked_mul(m, m - 1) / 2;
      return checked_add(checked_mul(p[0], m), checked_mul(p[1], tri));
    }
    case LBDD_PENALTY_TABLE: {
      int64_t sum = 0;
      for (int64_t j = 1; j <= m; ++j) sum = checked_add(sum, pen_at(I, s, j));
      return sum;
    }
  }
  raise_err(LBDD_ERR_LOGIC, "lbdd: bad penalty family");
  return 0;
}

/* marginal_penalty / refund_penalty, core.hpp:196-208 */
static int64_t marginal_penalty(const Inst* I, int64_t s, int64_t load) {
  if (load < 0) raise_err(LBDD_ERR_LOGIC, "lbdd: negative load");
  if (load < I->cap[s]) return 0;
  return pen_at(I, s, load - I->cap[s] + 1);
}
static int64_t refund_penalty(const Inst* I, int64_t s, int64_t load) {
  if (load < 0) raise_err(LBDD_ERR_LOGIC, "lbdd: negative load");
  if (load <= I->cap[s]) return 0;
  return pen_at(I, s, load - I->cap[s]);
}

/* validate_instance + require_valid_instance, core.hpp:250-313 */
static void require_valid(const Inst* I) {
  char msg[200];
#define FAIL(...)                                                       \
  do {                                                                  \
    char m2[160];                                                       \
    snprintf(m2, sizeof m2, __VA_ARGS__);                               \
    snprintf(msg, sizeof msg, "lbdd: invalid instance: %s", m2);        \
    raise_err(LBDD_ERR_INVALID_ARGUMENT, msg);                          \
  } while (0)
  if (I->k < 1) FAIL("instance has no service centers (k < 1)");
  if (I->n < 1) FAIL("instance has no demand units (n < 1)");
  for (int64_t s = 0; s < I->k; ++s) {
    const int64_t np = I->off[s + 1] - I->off[s];
    const int64_t* p = I->par + I->off[s];
    if (I->cap[s] < 0) FAIL("center %ld: negative capacity", (long)s);
    switch (I->fam[s]) {
      case LBDD_PENALTY_CONSTANT:
        if (np != 1) FAIL("center %ld: constant penalty takes one parameter", (long)s);
        if (p[0] <= 0) FAIL("center %ld: penalty not positive", (long)s);
        break;
      case LBDD_PENALTY_LINEAR:
        if (np != 2) FAIL("center %ld: linear penalty takes two parameters", (long)s);
        if (p[0] <= 0 || p[1] < 0) FAIL("center %ld: penalty not positive", (long)s);
        break;
      case LBDD_PENALTY_TABLE:
        if (np == 0) FAIL("center %ld: empty penalty table", (long)s);
        if (p[0] <= 0) FAIL("center %ld: penalty not positive", (long)s);
        for (int64_t i = 1; i < np; ++i)
          if (p[i] < p[i - 1]) FAIL("center %ld: penalty not monotone", (long)s);
        break;
      default: FAIL("center %ld: bad penalty family", (long)s);
    }
  }
  for (int64_t i = 0; i < I->n * I->k; ++i)
    if (I->cm[i] <= 0) FAIL("non-positive cost in cost matrix");
#undef FAIL
}

/* ------------------------------------------------------------------ */
/* SubspaceIndex: k*k addressable min-heaps, subspace.hpp:26-231       */
/* ------------------------------------------------------------------ */

typedef struct {
  int64_t key;
  int32_t demand;
} Entry;
typedef struct {
  Entry* data;
  int32_t size, cap;
} Heap;
typedef struct {
  const Inst* I;
  int64_t k, n;
  Heap* heaps;  /* from*k + to */
  int32_t* pos; /* d*k + to */
  int32_t* home;
} Index;

static void release_heaps(Arena* a) {
  for (size_t i = 0; i < a->nheaps; ++i) {
    Heap* h = (Heap*)a->heaps[i];
    for (int64_t j = 0; j < a->heap_counts[i]; ++j) free(h[j].data);
  }
  free(a->heaps);
  free(a->heap_counts);
}

static inline int entry_less(Entry a, Entry b) { /* subspace.hpp:145 */
  return a.key < b.key || (a.key == b.key && a.demand < b.demand);
}

static void index_init(Index* x, const Inst* I) {
  x->I = I;
  x->k = I->k;
  x->n = I->n;
  x->heaps = xalloc(sizeof(Heap) * (size_t)(I->k * I->k));
  register_heaps(x->heaps, I->k * I->k);
  x->pos = xalloc(sizeof(int32_t) * (size_t)(I->n * I->k));
  x->home = xalloc(sizeof(int32_t) * (size_t)I->n);
  for (int64_t i = 0; i < I->n * I->k; ++i) x->pos[i] = -1;
  for (int64_t d = 0; d < I->n; ++d) x->home[d] = -1;
}

static void swap_entries(Index* x, Heap* h, int64_t to, int32_t a, int32_t b) {
  Entry t = h->data[a];
  h->data[a] = h->data[b];
  h->data[b] = t;
  x->pos[(int64_t)h->data[a].demand * x->k + to] = a;
  x->pos[(int64_t)h->data[b].demand * x->k + to] = b;
}
static void sift_up(Index* x, Heap* h, int64_t to, int32_t i) {
  while (i > 0) {
    int32_t p = (i - 1) / 2;
    if (!entry_less(h->data[i], h->data[p])) break;
    swap_entries(x, h, to, i, p);
    i = p;
  }
}
static void sift_down(Index* x, Heap* h, int64_t to, int32_t i) {
  for (;;) {
    int32_t s = i, l = 2 * i + 1, r = 2 * i + 2;
    if (l < h->size && entry_less(h->data[l], h->data[s])) s = l;
    if (r < h->size && entry_less(h->data[r], h->data[s])) s = r;
    if (s == i) break;
    swap_entries(x, h, to, i, s);
    i = s;
  }
}
static void heap_push(Index* x, int64_t from, int64_t to, Entry e) {
  Heap* h = &x->heaps[from * x->k + to];
  if (h->size == h->cap) {
    int32_t nc = h->cap ? 2 * h->cap : 4;
    Entry* nd = realloc(h->data, sizeof(Entry) * (size_t)nc);
    if (!nd) raise_err(LBDD_ERR_RUNTIME, "oracle: out of memory");
    h->data = nd;
    h->cap = nc;
  }
  h->data[h->size] = e;
  x->pos[(int64_t)e.demand * x->k + to] = h->size;
  h->size++;
  sift_up(x, h, to, h->size - 1);
}
static void heap_erase(Index* x, int64_t from, int64_t to, int32_t d) {
  Heap* h = &x->heaps[from * x->k + to];
  int32_t idx = x->pos[(int64_t)d * x->k + to];
  if (idx < 0 || idx >= h->size || h->data[idx].demand != d)
    raise_err(LBDD_ERR_LOGIC, "lbdd: heap handle out of sync");
  int32_t last = h->size - 1;
  x->pos[(int64_t)d * x->k + to] = -1;
  if (idx != last) {
    h->data[idx] = h->data[last];
    x->pos[(int64_t)h->data[idx].demand * x->k + to] = idx;
    h->size--;
    sift_down(x, h, to, idx);
    sift_up(x, h, to, idx);
  } else {
    h->size--;
  }
}

/* SubspaceIndex::insert, subspace.hpp:46-56 */
static void index_insert(Index* x, int32_t d, int32_t c) {
  if (x->home[d] != -1) raise_err(LBDD_ERR_LOGIC, "lbdd: demand already indexed");
  for (int64_t j = 0; j < x->k; ++j) {
    if (j == c) continue;
    Entry e = {CM(x->I, d, j) - CM(x->I, d, c), d};
    heap_push(x, c, j, e);
  }
  x->home[d] = c;
}

/* min_transfer, subspace.hpp:73-80 */
static int min_transfer(const Index* x, int64_t from, int64_t to, Entry* out) {
  const Heap* h = &x->heaps[from * x->k + to];
  if (h->size == 0) return 0;
  *out = h->data[0];
  return 1;
}

/* Allotment, core.hpp:147-192 */
typedef struct {
  int32_t* assignment;
  int64_t* load;
} Allot;

static void allot_assign(Allot* a, int32_t d, int32_t s) {
  if (a->assignment[d] != -1) raise_err(LBDD_ERR_LOGIC, "lbdd: demand already assigned");
  a->assignment[d] = s;
  a->load[s]++;
}
static void allot_move(Allot* a, int32_t d, int32_t to) {
  if (a->assignment[d] == -1) raise_err(LBDD_ERR_LOGIC, "lbdd: cannot move an unassigned demand");
  a->load[a->assignment[d]]--;
  a->assignment[d] = to;
  a->load[to]++;
}

/* apply_transfer, subspace.hpp:83-118 (== parallel_index_update result) */
static void apply_transfer(Index* x, Allot* a, int32_t from, int32_t to, int32_t d) {
  if (from == to) raise_err(LBDD_ERR_LOGIC, "lbdd: transfer with identical endpoints");
  if (x->home[d] != from || a->assignment[d] != from)
    raise_err(LBDD_ERR_LOGIC, "lbdd: stale transfer edge");
  for (int64_t j = 0; j < x->k; ++j) {
    if (j != from) heap_erase(x, from, j, d);
    if (j != to) {
      Entry e = {CM(x->I, d, j) - CM(x->I, d, to), d};
      heap_push(x, to, j, e);
    }
  }
  x->home[d] = to;
  allot_move(a, d, to);
}

/* ------------------------------------------------------------------ */
/* anchored graphs (dense), subspace.hpp:243-371                        */
/* ------------------------------------------------------------------ */

enum { KIND_NONE = 0, KIND_TRANSFER = 1, KIND_DUMMY = 2, KIND_PENALTY = 3 };
#define UNREACH (INT64_MAX / 4) /* detail::kUnreachable, parallel.hpp:140 */

typedef struct {
  int32_t nodes; /* k + 1 */
  int32_t anchor;
  int64_t* w;     /* (nodes-1)*nodes, INT64_MAX = no edge */
  int8_t* kind;   /* same shape */
  int32_t* dem;   /* same shape */
} Graph;

static void graph_alloc(Graph* g, int32_t nodes, int32_t anchor) {
  g->nodes = nodes;
  g->anchor = anchor;
  size_t m = (size_t)(nodes - 1) * (size_t)nodes;
  g->w = xalloc(sizeof(int64_t) * m);
  g->kind = xalloc(m);
  g->dem = xalloc(sizeof(int32_t) * m);
  for (size_t i = 0; i < m; ++i) g->w[i] = INT64_MAX;
}

/* cheapest_pair_edge, subspace.hpp:294-307 */
static int cheapest_pair_edge(const Index* x, int64_t u, int64_t v,
                              const int64_t* dummies, int8_t* kind,
                              int32_t* dem, int64_t* cost) {
  Entry e;
  const int real = min_transfer(x, u, v, &e);
  const int dummy_ok = dummies != NULL && dummies[u] > 0;
  if (dummy_ok && (!real || e.key >= 0)) {
    *kind = KIND_DUMMY; *dem = -1; *cost = 0;
    return 1;
  }
  if (real) {
    *kind = KIND_TRANSFER; *dem = e.demand; *cost = e.key;
    return 1;
  }
  return 0;
}

static void set_edge(Graph* g, int32_t u, int32_t v, int8_t kind, int32_t dem, int64_t c) {
  size_t i = (size_t)u * (size_t)g->nodes + (size_t)v;
  g->w[i] = c;
  g->kind[i] = kind;
  g->dem[i] = dem;
}

/* build_negcycle_graph, subspace.hpp:313-331 */
static void build_negcycle_graph(Graph* g, const Index* x, int32_t anchor,
                                 const int64_t* dummies) {
  const int32_t k = (int32_t)x->k;
  graph_alloc(g, k + 1, anchor);
  for (int32_t u = 0; u < k; ++u)
    for (int32_t v = 0; v < k; ++v) {
      if (u == v) continue;
      int8_t kind; int32_t dem; int64_t c;
      if (!cheapest_pair_edge(x, u, v, dummies, &kind, &dem, &c)) continue;
      set_edge(g, u, v == anchor ? k : v, kind, dem, c);
    }
}

/* build_negpath_graph, subspace.hpp:337-371 */
static void build_negpath_graph(Graph* g, const Index* x, const Allot* a,
                                const Inst* I, int32_t anchor) {
  const int32_t k = (int32_t)x->k;
  const int64_t aload = a->load[anchor];
  if (aload <= I->cap[anchor])
    raise_err(LBDD_ERR_LOGIC, "lbdd: path graph requires an overloaded anchor");
  const int64_t refund = refund_penalty(I, anchor, aload);
  graph_alloc(g, k + 1, anchor);
  for (int32_t u = 0; u < k; ++u) {
    for (int32_t v = 0; v < k; ++v) {
      if (u == v || v == anchor) continue;
      int8_t kind; int32_t dem; int64_t c;
      if (!cheapest_pair_edge(x, u, v, NULL, &kind, &dem, &c)) continue;
      set_edge(g, u, v, kind, dem, c);
    }
    if (u != anchor) {
      const int64_t gain = marginal_penalty(I, u, a->load[u]) - refund;
      set_edge(g, u, k, KIND_PENALTY, -1, gain);
    }
  }
}

/* relax_nodes, parallel.hpp:145-169: parents are source nodes; dense
 * in-edge scan in ascending source order == in_edges sorted by source. */
static int relax_round_dense(int32_t nodes, const int64_t* w,
                             const int64_t* din, const int32_t* pin,
                             int64_t* dout, int32_t* pout) {
  int changed = 0;
  for (int32_t v = 0; v < nodes; ++v) {
    int64_t best = din[v];
    int32_t bp = pin[v];
    for (int32_t u = 0; u + 1 < nodes; ++u) {
      const int64_t c = w[(size_t)u * nodes + v];
      if (c == INT64_MAX) continue;
      const int64_t du = din[u];
      if (du >= UNREACH) continue;
      const int64_t cand = du + c;
      if (cand < best) { best = cand; bp = u; }
    }
    dout[v] = best;
    pout[v] = bp;
    if (best != din[v]) changed = 1;
  }
  return changed;
}

typedef struct {
  int found;
  int64_t cost;
  int32_t len;      /* edges */
  int32_t* nodes;   /* len + 1 nodes anchor-out .. anchor-in */
  int64_t* dist;
  int32_t* parent;
} PathRes;

/* lowest_cost_path, refine.hpp:28-81 */
static void lowest_cost_path(const Graph* g, PathRes* r, int64_t* rounds) {
  const int32_t N = g->nodes;
  int64_t* da = xalloc(sizeof(int64_t) * N);
  int64_t* db = xalloc(sizeof(int64_t) * N);
  int32_t* pa = xalloc(sizeof(int32_t) * N);
  int32_t* pb = xalloc(sizeof(int32_t) * N);
  for (int32_t i = 0; i < N; ++i) { da[i] = db[i] = UNREACH; pa[i] = pb[i] = -1; }
  da[g->anchor] = 0;
  int64_t *din = da, *dout = db;
  int32_t *pin = pa, *pout = pb;
  for (int32_t round = 1; round <= N; ++round) {
    const int changed = relax_round_dense(N, g->w, din, pin, dout, pout);
    if (rounds) ++*rounds;
    int64_t* td = din; din = dout; dout = td;
    int32_t* tp = pin; pin = pout; pout = tp;
    if (!changed) break;
    if (round == N) raise_err(LBDD_ERR_LOGIC, "lbdd: negative cycle witnessed in anchored graph");
  }
  r->dist = din;
  r->parent = pin;
  const int32_t sink = N - 1;
  r->found = 0;
  r->len = 0;
  if (din[sink] >= UNREACH) return;
  r->found = 1;
  r->cost = din[sink];
  int8_t* seen = xalloc((size_t)N);
  int32_t* rev = xalloc(sizeof(int32_t) * (size_t)(N + 1));
  int32_t node = sink, len = 0;
  rev[0] = sink;
  while (node != g->anchor) {
    if (seen[node]) raise_err(LBDD_ERR_LOGIC, "lbdd: lowest-cost path is not simple");
    seen[node] = 1;
    const int32_t u = pin[node];
    if (u < 0) raise_err(LBDD_ERR_LOGIC, "lbdd: broken parent chain");
    rev[++len] = u;
    node = u;
  }
  r->len = len;
  r->nodes = xalloc(sizeof(int32_t) * (size_t)(len + 1));
  for (int32_t i = 0; i <= len; ++i) r->nodes[i] = rev[len - i];
  int64_t sum = 0;
  for (int32_t i = 0; i < len; ++i)
    sum = checked_add(sum, g->w[(size_t)r->nodes[i] * N + r->nodes[i + 1]]);
  if (sum != r->cost) raise_err(LBDD_ERR_LOGIC, "lbdd: path cost does not match edge sum");
}

/* gamma_has_negative_cycle, refine.hpp:86-116 (Gauss-Seidel, edge order
 * u-major as the reference's edge vector) */
static int gamma_has_negative_cycle(const Index* x, const int64_t* dummies) {
  const int64_t k = x->k;
  int64_t* ef = xalloc(sizeof(int64_t) * (size_t)(k * k));
  int64_t* et = xalloc(sizeof(int64_t) * (size_t)(k * k));
  int64_t* ec = xalloc(sizeof(int64_t) * (size_t)(k * k));
  int64_t m = 0;
  for (int64_t u = 0; u < k; ++u)
    for (int64_t v = 0; v < k; ++v) {
      if (u == v) continue;
      int8_t kind; int32_t dem; int64_t c;
      if (cheapest_pair_edge(x, u, v, dummies, &kind, &dem, &c)) {
        ef[m] = u; et[m] = v; ec[m] = c; ++m;
      }
    }
  int64_t* dist = xalloc(sizeof(int64_t) * (size_t)k);
  for (int64_t pass = 0; pass <= k; ++pass) {
    int changed = 0;
    for (int64_t e = 0; e < m; ++e) {
      const int64_t cand = dist[ef[e]] + ec[e];
      if (cand < dist[et[e]]) { dist[et[e]] = cand; changed = 1; }
    }
    if (!changed) return 0;
  }
  return 1;
}

/* ------------------------------------------------------------------ */
/* SolverState + refinements, solver.hpp:34-69, refine.hpp:118-222      */
/* ------------------------------------------------------------------ */

typedef struct {
  const Inst* I;
  Allot a;
  Index x;
  int64_t* dummies; /* strict only */
  int strict;
  int64_t delta;
  lbdd_solve_report rep; /* stats + timings */
  int check_invariants;
} State;

static void state_init(State* st, const Inst* I) {
  memset(st, 0, sizeof *st);
  st->I = I;
  st->a.assignment = xalloc(sizeof(int32_t) * (size_t)I->n);
  st->a.load = xalloc(sizeof(int64_t) * (size_t)(I->k + 1));
  for (int64_t d = 0; d < I->n; ++d) st->a.assignment[d] = -1;
  index_init(&st->x, I);
}

static const int64_t* dummy_counts(const State* st) {
  return st->strict ? st->dummies : NULL;
}

/* detail::assert_no_negative_cycle, refine.hpp:125-132 */
static void assert_no_negative_cycle(State* st) {
  if (!st->check_invariants) return;
  st->rep.invariant_checks++;
  if (gamma_has_negative_cycle(&st->x, dummy_counts(st)))
    raise_err(LBDD_ERR_LOGIC, "lbdd: negative cycle survived refinement");
}

/* detail::apply_path_edges, refine.hpp:134-164 */
static void apply_path_edges(State* st, const Graph* g, const PathRes* p) {
  const int32_t k = g->nodes - 1;
  for (int32_t i = 0; i < p->len; ++i) {
    const int32_t u = p->nodes[i], v = p->nodes[i + 1];
    const size_t ei = (size_t)u * g->nodes + v;
    const int32_t cu = u == k ? g->anchor : u; /* node_center */
    const int32_t cv = v == k ? g->anchor : v;
    switch (g->kind[ei]) {
      case KIND_TRANSFER: {
        const int64_t t0 = now_ns();
        apply_transfer(&st->x, &st->a, cu, cv, g->dem[ei]);
        st->rep.index_update_ns += now_ns() - t0;
        st->rep.transfers_applied++;
        break;
      }
      case KIND_DUMMY:
        if (st->dummies == NULL || !st->strict || st->dummies[cu] <= 0)
          raise_err(LBDD_ERR_LOGIC, "lbdd: placeholder transfer without surplus");
        st->dummies[cu]--;
        st->dummies[cv]++;
        break;
      case KIND_PENALTY:
        if (i != p->len - 1) raise_err(LBDD_ERR_LOGIC, "lbdd: penalty edge inside a path");
        break;
    }
  }
}

typedef struct { int applied; int64_t gain; } Outcome;

/* negative_cycle_refine, refine.hpp:172-192 */
static Outcome negative_cycle_refine(State* st, int32_t anchor) {
  st->rep.cycle_refine_calls++;
  Graph g;
  build_negcycle_graph(&g, &st->x, anchor, dummy_counts(st));
  PathRes p;
  const int64_t t0 = now_ns();
  lowest_cost_path(&g, &p, &st->rep.relax_rounds);
  st->rep.bellman_ford_ns += now_ns() - t0;
  Outcome o = {0, 0};
  if (p.found && p.cost < 0) {
    apply_path_edges(st, &g, &p);
    st->delta = checked_add(st->delta, p.cost);
    st->rep.negative_cycles_removed++;
    st->rep.refinement_gain = checked_add(st->rep.refinement_gain, -p.cost);
    o.applied = 1;
    o.gain = p.cost;
  }
  assert_no_negative_cycle(st);
  return o;
}

/* negative_path_refine, refine.hpp:198-222 */
static Outcome negative_path_refine(State* st, int32_t anchor) {
  st->rep.path_refine_calls++;
  Graph g;
  build_negpath_graph(&g, &st->x, &st->a, st->I, anchor);
  PathRes p;
  const int64_t t0 = now_ns();
  lowest_cost_path(&g, &p, &st->rep.relax_rounds);
  st->rep.bellman_ford_ns += now_ns() - t0;
  Outcome o = {0, 0};
  if (p.found && p.cost < 0) {
    if (p.len == 0 ||
        g.kind[(size_t)p.nodes[p.len - 1] * g.nodes + p.nodes[p.len]] != KIND_PENALTY)
      raise_err(LBDD_ERR_LOGIC, "lbdd: path must close with a penalty edge");
    apply_path_edges(st, &g, &p);
    st->delta = checked_add(st->delta, p.cost);
    st->rep.negative_paths_removed++;
    st->rep.refinement_gain = checked_add(st->rep.refinement_gain, -p.cost);
    o.applied = 1;
    o.gain = p.cost;
  }
  assert_no_negative_cycle(st);
  return o;
}

/* evaluate_partial_objective over an assignment, core.hpp:216-233 */
static int64_t objective_of(const Inst* I, const int32_t* assignment, int partial) {
  int64_t* load = xalloc(sizeof(int64_t) * (size_t)I->k);
  int64_t total = 0;
  for (int64_t d = 0; d < I->n; ++d) {
    const int32_t s = assignment[d];
    if (s == -1) {
      if (!partial) raise_err(LBDD_ERR_INVALID_ARGUMENT, "lbdd: objective of incomplete allotment");
      continue;
    }
    if (s < 0 || s >= I->k) raise_err(LBDD_ERR_INVALID_ARGUMENT, "lbdd: allotment shape mismatch");
    total = checked_add(total, CM(I, d, s));
    load[s]++;
  }
  for (int64_t s = 0; s < I->k; ++s) total = checked_add(total, pen_total(I, s, load[s] - I->cap[s]));
  return total;
}

/* ------------------------------------------------------------------ */
/* solvers, solver.hpp                                                  */
/* ------------------------------------------------------------------ */

/* detail::row_min_center, solver.hpp:74-80 */
static int32_t row_min_center(const Inst* I, int64_t d) {
  int32_t best = 0;
  for (int32_t s = 1; s < I->k; ++s)
    if (CM(I, d, s) < CM(I, d, best)) best = s;
  return best;
}

typedef struct { int64_t cost; int32_t d; int32_t s; } Arrival;
static int arrival_cmp(const void* a, const void* b) {
  const Arrival* x = a;
  const Arrival* y = b;
  if (x->cost != y->cost) return x->cost < y->cost ? -1 : 1;
  if (x->d != y->d) return x->d < y->d ? -1 : 1;
  return (x->s > y->s) - (x->s < y->s);
}
/* build_arrival_queue, solver.hpp:84-96: a min-heap on (cost, d, s) pops in
 * ascending tuple order; d is unique, so a sort gives the same sequence. */
static Arrival* build_arrivals(const Inst* I) {
  Arrival* q = xalloc(sizeof(Arrival) * (size_t)I->n);
  for (int64_t d = 0; d < I->n; ++d) {
    const int32_t s = row_min_center(I, d);
    q[d].cost = CM(I, d, s);
    q[d].d = (int32_t)d;
    q[d].s = s;
  }
  qsort(q, (size_t)I->n, sizeof(Arrival), arrival_cmp);
  return q;
}

/* detail::finish_report, solver.hpp:110-129 */
static void finish_report(State* st, int32_t solver, int64_t start,
                          lbdd_solve_report* out, int32_t* assignment, int64_t* load) {
  st->rep.total_ns = now_ns() - start;
  for (int64_t d = 0; d < st->I->n; ++d)
    if (st->a.assignment[d] == -1)
      raise_err(LBDD_ERR_LOGIC, "lbdd: solver produced an incomplete allotment");
  const int64_t recount = objective_of(st->I, st->a.assignment, 0);
  if (recount != st->delta) raise_err(LBDD_ERR_LOGIC, "lbdd: tracked objective diverged from recount");
  st->rep.objective = st->delta;
  st->rep.solver = solver;
  *out = st->rep;
  if (assignment) memcpy(assignment, st->a.assignment, sizeof(int32_t) * (size_t)st->I->n);
  if (load) memcpy(load, st->a.load, sizeof(int64_t) * (size_t)st->I->k);
}

/* asral_solve main loop body, solver.hpp:143-167 (shared by the sample) */
static void asral_arrival(State* st, const Arrival* ar, int fixpoint) {
  const Inst* I = st->I;
  const int64_t t0 = now_ns();
  index_insert(&st->x, ar->d, ar->s);
  st->rep.index_update_ns += now_ns() - t0;
  allot_assign(&st->a, ar->d, ar->s);
  negative_cycle_refine(st, ar->s);
  const int64_t load = st->a.load[ar->s];
  if (load <= I->cap[ar->s]) {
    st->delta = checked_add(st->delta, ar->cost);
  } else {
    st->delta = checked_add(st->delta, checked_add(ar->cost, refund_penalty(I, ar->s, load)));
    Outcome o = negative_path_refine(st, ar->s);
    while (fixpoint && o.applied && st->a.load[ar->s] > I->cap[ar->s])
      o = negative_path_refine(st, ar->s);
  }
}

static void asral_solve(const Inst* I, const lbdd_solver_options* o, int32_t solver,
                        lbdd_solve_report* out, int32_t* assignment, int64_t* load) {
  require_valid(I);
  const int64_t start = now_ns();
  State st;
  state_init(&st, I);
  st.check_invariants = o && o->check_invariants;
  const int fixpoint = o && o->refine_to_fixpoint;
  Arrival* q = build_arrivals(I);
  for (int64_t i = 0; i < I->n; ++i) asral_arrival(&st, &q[i], fixpoint);
  finish_report(&st, solver, start, out, assignment, load);
}

/* greedy_solve, solver.hpp:172-189 */
static void greedy_solve(const Inst* I, lbdd_solve_report* out, int32_t* assignment,
                         int64_t* load) {
  require_valid(I);
  const int64_t start = now_ns();
  State st;
  memset(&st, 0, sizeof st);
  st.I = I;
  st.a.assignment = xalloc(sizeof(int32_t) * (size_t)I->n);
  st.a.load = xalloc(sizeof(int64_t) * (size_t)(I->k + 1));
  for (int64_t d = 0; d < I->n; ++d) st.a.assignment[d] = -1;
  Arrival* q = build_arrivals(I);
  for (int64_t i = 0; i < I->n; ++i) {
    allot_assign(&st.a, q[i].d, q[i].s);
    const int64_t l = st.a.load[q[i].s];
    st.delta = checked_add(st.delta, checked_add(q[i].cost, refund_penalty(I, q[i].s, l)));
  }
  finish_report(&st, LBDD_SOLVER_GREEDY, start, out, assignment, load);
}

/* augment_with_dummy_center + strict_solve, solver.hpp:194-301 */
static void strict_solve(const Inst* I0, const lbdd_solver_options* o,
                         lbdd_solve_report* out, int32_t* assignment, int64_t* load) {
  require_valid(I0);
  const int64_t start = now_ns();
  int64_t total_cap = 0;
  for (int64_t s = 0; s < I0->k; ++s) total_cap += I0->cap[s];
  const int excess = total_cap < I0->n;
  int64_t max_cost = 0;
  for (int64_t i = 0; i < I0->n * I0->k; ++i) if (I0->cm[i] > max_cost) max_cost = I0->cm[i];
  Inst A;
  const Inst* W = I0;
  if (excess) {
    const int64_t deficit = I0->n - total_cap;
    const int64_t k1 = I0->k + 1;
    int32_t* cm = xalloc(sizeof(int32_t) * (size_t)(I0->n * k1));
    for (int64_t d = 0; d < I0->n; ++d) {
      memcpy(cm + d * k1, I0->cm + d * I0->k, sizeof(int32_t) * (size_t)I0->k);
      if (max_cost + 1 > INT32_MAX) raise_err(LBDD_ERR_OVERFLOW, "oracle: overflow column exceeds int32");
      cm[d * k1 + I0->k] = (int32_t)(max_cost + 1);
    }
    int64_t* cap = xalloc(sizeof(int64_t) * (size_t)k1);
    int32_t* fam = xalloc(sizeof(int32_t) * (size_t)k1);
    int64_t* off = xalloc(sizeof(int64_t) * (size_t)(k1 + 1));
    int64_t* par = xalloc(sizeof(int64_t) * (size_t)(I0->off[I0->k] + 1));
    memcpy(cap, I0->cap, sizeof(int64_t) * (size_t)I0->k);
    memcpy(fam, I0->fam, sizeof(int32_t) * (size_t)I0->k);
    memcpy(off, I0->off, sizeof(int64_t) * (size_t)(I0->k + 1));
    memcpy(par, I0->par, sizeof(int64_t) * (size_t)I0->off[I0->k]);
    cap[I0->k] = deficit;
    fam[I0->k] = LBDD_PENALTY_CONSTANT;
    par[I0->off[I0->k]] = 1;
    off[k1] = I0->off[I0->k] + 1;
    A.n = I0->n; A.k = k1; A.cm = cm; A.cap = cap; A.fam = fam; A.off = off; A.par = par;
    W = &A;
  }
  const int64_t k = W->k;
  State st;
  state_init(&st, W);
  st.check_invariants = o && o->check_invariants;
  st.strict = 1;
  st.dummies = xalloc(sizeof(int64_t) * (size_t)k);
  for (int64_t s = 0; s < k; ++s) st.dummies[s] = W->cap[s];

  int32_t* order = xalloc(sizeof(int32_t) * (size_t)W->n);
  if (o && o->strict_order && o->strict_order_len > 0) {
    if (o->strict_order_len != W->n)
      raise_err(LBDD_ERR_INVALID_ARGUMENT, "lbdd: strict order must cover every demand");
    memcpy(order, o->strict_order, sizeof(int32_t) * (size_t)W->n);
  } else {
    for (int64_t d = 0; d < W->n; ++d) order[d] = (int32_t)d;
  }
  for (int64_t i = 0; i < W->n; ++i) {
    const int32_t d = order[i];
    int32_t target = -1;
    for (int32_t s = 0; s < k; ++s) {
      if (st.dummies[s] <= 0) continue;
      if (target == -1 || CM(W, d, s) < CM(W, d, target)) target = s;
    }
    if (target == -1) raise_err(LBDD_ERR_LOGIC, "lbdd: no residual capacity left");
    st.dummies[target]--;
    const int64_t t0 = now_ns();
    index_insert(&st.x, d, target);
    st.rep.index_update_ns += now_ns() - t0;
    allot_assign(&st.a, d, target);
    st.delta = checked_add(st.delta, CM(W, d, target));
    negative_cycle_refine(&st, target);
  }
  for (int64_t s = 0; s < k; ++s) {
    if (st.a.load[s] > W->cap[s]) raise_err(LBDD_ERR_LOGIC, "lbdd: strict solve exceeded a capacity");
    if (st.a.load[s] + st.dummies[s] != W->cap[s])
      raise_err(LBDD_ERR_LOGIC, "lbdd: placeholder accounting out of balance");
  }
  finish_report(&st, LBDD_SOLVER_STRICT, start, out, assignment, load);
  if (excess) {
    const int64_t deficit = I0->n - total_cap;
    out->strict_surcharge = checked_mul(deficit, max_cost + 1);
    out->has_dummy_center = 1;
    out->objective -= out->strict_surcharge;
  }
  if (load) memcpy(load, st.a.load, sizeof(int64_t) * (size_t)k);
}

/* ------------------------------------------------------------------ */
/* entry points                                                         */
/* ------------------------------------------------------------------ */

int lbdd_oracle_solve(const lbdd_instance_desc* desc, int32_t solver,
                      const lbdd_solver_options* opts, lbdd_solve_report* report,
                      int32_t* assignment, int64_t* load) {
  ENTRY_BEGIN
  const Inst I = inst_from(desc);
  memset(report, 0, sizeof *report);
  switch (solver) {
    case LBDD_SOLVER_ASRAL:
    case LBDD_SOLVER_PARA_ASRAL: asral_solve(&I, opts, solver, report, assignment, load); break;
    case LBDD_SOLVER_STRICT: strict_solve(&I, opts, report, assignment, load); break;
    case LBDD_SOLVER_GREEDY: greedy_solve(&I, report, assignment, load); break;
    default: raise_err(LBDD_ERR_INVALID_ARGUMENT, "unknown solver");
  }
  ENTRY_END
}

/* from_allotment: state over a preexisting allotment, solver.hpp:61-68 */
static void state_from_allotment(State* st, const Inst* I, const int32_t* assignment) {
  state_init(st, I);
  for (int64_t d = 0; d < I->n; ++d) {
    if (assignment[d] < 0) continue;
    allot_assign(&st->a, (int32_t)d, assignment[d]);
    index_insert(&st->x, (int32_t)d, assignment[d]);
  }
  st->delta = objective_of(I, st->a.assignment, 1);
}

int lbdd_oracle_build_index(const lbdd_instance_desc* desc, const int32_t* assignment,
                            int64_t* out) {
  ENTRY_BEGIN
  const Inst I = inst_from(desc);
  Index x;
  index_init(&x, &I);
  for (int64_t d = 0; d < I.n; ++d)
    if (assignment[d] >= 0) index_insert(&x, (int32_t)d, assignment[d]);
  for (int64_t u = 0; u < I.k; ++u)
    for (int64_t v = 0; v < I.k; ++v) {
      Entry e;
      int64_t packed = INT64_MAX;
      if (u != v && min_transfer(&x, u, v, &e))
        packed = (int64_t)(((uint64_t)e.key << 32) | (uint32_t)e.demand);
      out[u * I.k + v] = packed;
    }
  ENTRY_END
}

int lbdd_oracle_refine(const lbdd_instance_desc* desc, int32_t kind, int32_t anchor,
                       int32_t* assignment, int64_t* dummies, int32_t* applied,
                       int64_t* gain) {
  ENTRY_BEGIN
  const Inst I = inst_from(desc);
  State st;
  state_from_allotment(&st, &I, assignment);
  if (dummies) { st.strict = 1; st.dummies = dummies; }
  Outcome o = kind == 0 ? negative_cycle_refine(&st, anchor) : negative_path_refine(&st, anchor);
  *applied = o.applied;
  *gain = o.gain;
  memcpy(assignment, st.a.assignment, sizeof(int32_t) * (size_t)I.n);
  ENTRY_END
}

int lbdd_oracle_gamma_has_negative_cycle(const lbdd_instance_desc* desc,
                                         const int32_t* assignment, const int64_t* dummies,
                                         int32_t* has_cycle) {
  ENTRY_BEGIN
  const Inst I = inst_from(desc);
  Index x;
  index_init(&x, &I);
  for (int64_t d = 0; d < I.n; ++d)
    if (assignment[d] >= 0) index_insert(&x, (int32_t)d, assignment[d]);
  *has_cycle = gamma_has_negative_cycle(&x, dummies);
  ENTRY_END
}

int lbdd_oracle_lowest_cost_path(int32_t node_count, int32_t anchor, const int64_t* weights,
                                 int32_t* found, int64_t* cost, int64_t* dist,
                                 int32_t* parent_node, int32_t* path, int32_t* path_len) {
  ENTRY_BEGIN
  Graph g;
  g.nodes = node_count;
  g.anchor = anchor;
  g.w = (int64_t*)weights;
  PathRes r;
  lowest_cost_path(&g, &r, NULL);
  *found = r.found;
  *path_len = 0;
  if (r.found) {
    *cost = r.cost;
    memcpy(dist, r.dist, sizeof(int64_t) * (size_t)node_count);
    memcpy(parent_node, r.parent, sizeof(int32_t) * (size_t)node_count);
    memcpy(path, r.nodes, sizeof(int32_t) * (size_t)(r.len + 1));
    *path_len = r.len;
  }
  ENTRY_END
}

int lbdd_oracle_relax_round(int32_t node_count, const int64_t* weights, const int64_t* dist_in,
                            const int32_t* parent_in, int64_t* dist_out, int32_t* parent_out,
                            int32_t* changed) {
  ENTRY_BEGIN
  *changed = relax_round_dense(node_count, weights, dist_in, parent_in, dist_out, parent_out);
  ENTRY_END
}

int lbdd_oracle_evaluate_objective(const lbdd_instance_desc* desc, const int32_t* assignment,
                                   int32_t partial, int64_t* objective) {
  ENTRY_BEGIN
  const Inst I = inst_from(desc);
  *objective = objective_of(&I, assignment, partial);
  ENTRY_END
}

int lbdd_oracle_arrival_queue(const lbdd_instance_desc* desc, int32_t* best_center,
                              int64_t* best_cost, int32_t* order) {
  ENTRY_BEGIN
  const Inst I = inst_from(desc);
  Arrival* q = build_arrivals(&I);
  for (int64_t i = 0; i < I.n; ++i) {
    if (best_center) best_center[q[i].d] = q[i].s;
    if (best_cost) best_cost[q[i].d] = q[i].cost;
    if (order) order[i] = q[i].d;
  }
  ENTRY_END
}

int lbdd_oracle_asral_sample(const lbdd_instance_desc* desc, int64_t max_arrivals,
                             int32_t workers, int64_t* elapsed_ns, int64_t* arrivals_done,
                             int64_t* setup_ns) {
  (void)workers; /* the port is single-threaded */
  ENTRY_BEGIN
  const Inst I = inst_from(desc);
  require_valid(&I);
  const int64_t t0 = now_ns();
  State st;
  state_init(&st, &I);
  Arrival* q = build_arrivals(&I);
  *setup_ns = now_ns() - t0;
  int64_t m = max_arrivals < I.n ? max_arrivals : I.n;
  for (int64_t i = 0; i < m; ++i) asral_arrival(&st, &q[i], 0);
  *elapsed_ns = now_ns() - t0;
  *arrivals_done = m;
  ENTRY_END
}

/* ------------------------------------------------------------------ */
/* instgen.hpp: mt19937_64 and the euclidean generator                 */
/* ------------------------------------------------------------------ */

typedef struct { uint64_t mt[312]; int idx; } Mt64;
static void mt_seed(Mt64* m, uint64_t seed) {
  m->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    m->mt[i] = 6364136223846793005ULL * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
  m->idx = 312;
}
static uint64_t mt_next(Mt64* m) {
  if (m->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (m->mt[i] & 0xFFFFFFFF80000000ULL) | (m->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      m->mt[i] = m->mt[(i + 156) % 312] ^ xa;
    }
    m->idx = 0;
  }
  uint64_t y = m->mt[m->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}
/* gen_detail::uniform_below, instgen.hpp:57-66 */
static uint64_t uniform_below(Mt64* m, uint64_t bound) {
  const uint64_t threshold = (0 - bound) % bound;
  for (;;) {
    const unsigned __int128 p = (unsigned __int128)mt_next(m) * bound;
    if ((uint64_t)p >= threshold) return (uint64_t)(p >> 64);
  }
}
static double uniform01(Mt64* m) { return (double)(mt_next(m) >> 11) * 0x1.0p-53; }

int64_t lbdd_oracle_derive_center_count(int64_t n, double ratio) { /* instgen.hpp:45 */
  int64_t k = (int64_t)floor((double)n / ratio);
  return k < 1 ? 1 : k;
}

/* generate, instgen.hpp:245-294 (euclidean branch) */
int lbdd_oracle_generate(uint64_t seed, int64_t n, double ratio, double theta, int64_t pen_lo,
                         int64_t pen_hi, int64_t* k_out, int64_t* capacity, int64_t* penalty,
                         int32_t* costs) {
  ENTRY_BEGIN
  if (n < 1) raise_err(LBDD_ERR_INVALID_ARGUMENT, "lbdd: n must be >= 1");
  if (theta <= 0.0 || theta > 1.0) raise_err(LBDD_ERR_INVALID_ARGUMENT, "lbdd: theta must be in (0, 1]");
  if (pen_lo < 1 || pen_hi < pen_lo) raise_err(LBDD_ERR_INVALID_ARGUMENT, "lbdd: bad penalty range");
  if (ratio <= 0) raise_err(LBDD_ERR_INVALID_ARGUMENT, "lbdd: ratio must be positive");
  const int64_t k = lbdd_oracle_derive_center_count(n, ratio);
  *k_out = k;
  if (capacity != NULL) {
    const int64_t total = (int64_t)llround(theta * (double)n);
    Mt64* m = xalloc(sizeof(Mt64));
    mt_seed(m, seed);
    for (int64_t s = 0; s < k; ++s) capacity[s] = 0;
    for (int64_t u = 0; u < total; ++u) capacity[uniform_below(m, (uint64_t)k)]++;
    for (int64_t s = 0; s < k; ++s)
      penalty[s] = pen_lo + (int64_t)uniform_below(m, (uint64_t)(pen_hi - pen_lo + 1));
    double* cx = xalloc(sizeof(double) * (size_t)k);
    double* cy = xalloc(sizeof(double) * (size_t)k);
    for (int64_t s = 0; s < k; ++s) { cx[s] = uniform01(m); cy[s] = uniform01(m); }
    for (int64_t d = 0; d < n; ++d) {
      const double dx = uniform01(m), dy = uniform01(m);
      for (int64_t s = 0; s < k; ++s) {
        int64_t c = (int64_t)llround(hypot(dx - cx[s], dy - cy[s]) * 1000.0);
        costs[d * k + s] = (int32_t)(c < 1 ? 1 : c);
      }
    }
  }
  ENTRY_END
}
