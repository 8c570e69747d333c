/* oracle/e2_oracle.c — TEST INFRASTRUCTURE ONLY: a plain-C restatement of
 * the reference's E2 global-scheduler path, written for clarity, not speed
 * (linear scans, per-node timestamp deques, no incremental LRU index).
 *
 * It implements include/e2sched.h so the tests can swap it in for the
 * product or the reference shim.  Each function cites the reference code it
 * restates (paths relative to /root/reference/proj).  Parity is PINNED: it
 * reproduces the golden vectors recorded from the unmodified reference
 * (tests/golden) and is cross-checked against oracle/_ref/libe2ref.so by
 * tests/test_oracle.py.  Never linked into the product.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "e2sched.h"

/* ------------------------------------------------------------------ types */
typedef struct {
  double* t;
  int64_t head, n, cap; /* live stamps: t[head .. n) */
} Stamps;

typedef struct {
  uint64_t id;
  int64_t parent; /* node index, -1 for the root */
  int32_t* edge;
  int64_t len;
  int64_t* kids; /* node indices, sorted by first edge token */
  int64_t nkids, capkids;
  uint64_t caching, la_mask;
  double* la;     /* [G] */
  int32_t* ccc;   /* [G] cached_child_count */
  Stamps* hits;   /* [G] */
  int alive;
} Node;

typedef struct {
  double t;
  int64_t v, est;
} Ent;

typedef struct {
  Ent* e;
  int64_t head, n, cap;
} Deque;

typedef struct {
  int64_t key;
  int32_t gpu;
  int64_t cached, prompt;
  double arrival;
  uint64_t root;
  int used;
} Inflight;

typedef struct {
  uint64_t root;
  int64_t bucket;
  double sum;
  int64_t count;
  int alive;
} QCell;

struct e2_handle {
  int G;
  e2_sched_cfg cfg;
  e2_time_model m;
  e2_policy pol;
  Node* nodes;
  int64_t nn, capn;
  uint64_t next_id;
  int64_t node_count;
  int64_t cached_tokens[E2_MAX_GPUS];
  Deque sched[E2_MAX_GPUS], comp[E2_MAX_GPUS];
  int64_t missed_sum[E2_MAX_GPUS], missed_nz[E2_MAX_GPUS], output_sum[E2_MAX_GPUS];
  int64_t inflight_cached[E2_MAX_GPUS], inflight_prompt[E2_MAX_GPUS];
  int32_t redirect[E2_MAX_GPUS];
  Inflight* inf;
  int64_t ninf, capinf;
  QCell* q;
  int64_t nq, capq;
  int64_t rr_next;
  e2_stats st;
  char err[256];
};

static char g_err[256];

#define GROW(ptr, n, cap, T)                                           \
  do {                                                                 \
    if ((n) >= (cap)) {                                                \
      (cap) = (cap) ? 2 * (cap) : 16;                                  \
      (ptr) = (T*)realloc((ptr), (size_t)(cap) * sizeof(T));           \
    }                                                                  \
  } while (0)

static int fail(e2_handle* h, int code, const char* msg) {
  snprintf(h->err, sizeof h->err, "%s", msg);
  return code;
}

/* ------------------------------------------------------------ node basics */
static int64_t new_node(e2_handle* h, int64_t parent, const int32_t* edge, int64_t len) {
  GROW(h->nodes, h->nn, h->capn, Node);
  Node* n = &h->nodes[h->nn];
  memset(n, 0, sizeof *n);
  n->id = h->next_id++;
  n->parent = parent;
  n->len = len;
  n->edge = (int32_t*)malloc((size_t)(len ? len : 1) * 4);
  if (len) memcpy(n->edge, edge, (size_t)len * 4);
  n->la = (double*)calloc((size_t)h->G, sizeof(double));
  n->ccc = (int32_t*)calloc((size_t)h->G, sizeof(int32_t));
  n->hits = (Stamps*)calloc((size_t)h->G, sizeof(Stamps));
  n->alive = 1;
  return h->nn++;
}

static int cached_on(const Node* n, int g) { return (int)((n->caching >> g) & 1u); }

static void add_kid(e2_handle* h, int64_t p, int64_t c) {
  Node* np = &h->nodes[p];
  GROW(np->kids, np->nkids, np->capkids, int64_t);
  int64_t i = np->nkids;
  int32_t t = h->nodes[c].edge[0];
  while (i > 0 && h->nodes[np->kids[i - 1]].edge[0] > t) {
    np->kids[i] = np->kids[i - 1];
    --i;
  }
  np->kids[i] = c;
  np->nkids++;
}

static void del_kid(e2_handle* h, int64_t p, int64_t c) {
  Node* np = &h->nodes[p];
  for (int64_t i = 0; i < np->nkids; ++i)
    if (np->kids[i] == c) {
      memmove(&np->kids[i], &np->kids[i + 1], (size_t)(np->nkids - i - 1) * sizeof(int64_t));
      np->nkids--;
      return;
    }
}

static int64_t find_kid(const e2_handle* h, int64_t p, int32_t tok) {
  const Node* np = &h->nodes[p];
  for (int64_t i = 0; i < np->nkids; ++i)
    if (h->nodes[np->kids[i]].edge[0] == tok) return np->kids[i];
  return -1;
}

static void stamp_push(Stamps* s, double t) {
  if (s->n >= s->cap) {
    s->cap = s->cap ? 2 * s->cap : 8;
    s->t = (double*)realloc(s->t, (size_t)s->cap * sizeof(double));
  }
  s->t[s->n++] = t;
}

/* prune_hits (prefix_tree.cpp:37-43) */
static void prune_hits(e2_handle* h, Node* n, double now) {
  const double cut = now - h->cfg.history_window_ms;
  for (int g = 0; g < h->G; ++g) {
    Stamps* s = &n->hits[g];
    while (s->head < s->n && s->t[s->head] < cut) s->head++;
  }
}

/* recent_hits (prefix_tree.cpp:380-385) */
static int64_t recent_hits(e2_handle* h, Node* n, int g, double now) {
  prune_hits(h, n, now);
  return n->hits[g].n - n->hits[g].head;
}

/* ------------------------------------------------------------- tree walks */
typedef struct {
  int64_t matched_len, cached_len;
  int64_t per_gpu[E2_MAX_GPUS];
  uint64_t present;
  int64_t *span_node, *span_m;
  int64_t nspan;
} Match;

static void match_free(Match* m) {
  free(m->span_node);
  free(m->span_m);
}

/* walk (prefix_tree.cpp:79-114) */
static Match walk(const e2_handle* h, const int32_t* p, int64_t len) {
  Match m;
  memset(&m, 0, sizeof m);
  m.span_node = (int64_t*)malloc(8 * (size_t)(len + 1));
  m.span_m = (int64_t*)malloc(8 * (size_t)(len + 1));
  int64_t cur = 0, pos = 0;
  uint64_t alive = 0;
  int first = 1;
  while (pos < len) {
    int64_t c = find_kid(h, cur, p[pos]);
    if (c < 0) break;
    const Node* ch = &h->nodes[c];
    int64_t lim = ch->len < len - pos ? ch->len : len - pos, k = 0;
    while (k < lim && ch->edge[k] == p[pos + k]) ++k;
    if (k == 0) break;
    m.span_node[m.nspan] = c;
    m.span_m[m.nspan++] = k;
    if (first) {
      alive = ch->caching;
      m.present = alive;
      first = 0;
    } else {
      alive &= ch->caching;
    }
    for (int g = 0; g < h->G; ++g)
      if ((alive >> g) & 1u) m.per_gpu[g] += k;
    if (ch->caching) m.cached_len += k;
    pos += k;
    cur = c;
    if (k < ch->len) break;
  }
  m.matched_len = pos;
  return m;
}

static int64_t matched_on(const Match* m, int g) { return ((m->present >> g) & 1u) ? m->per_gpu[g] : 0; }

/* split_node (prefix_tree.cpp:122-154): node keeps [0,k) and its id; the
 * suffix gets a new id, the children and copies of the metadata. */
static int64_t split_node(e2_handle* h, int64_t x, int64_t k) {
  int64_t y = new_node(h, x, h->nodes[x].edge + k, h->nodes[x].len - k);
  Node* nx = &h->nodes[x];
  Node* ny = &h->nodes[y];
  nx->len = k;
  ny->kids = nx->kids;
  ny->nkids = nx->nkids;
  ny->capkids = nx->capkids;
  nx->kids = NULL;
  nx->nkids = nx->capkids = 0;
  for (int64_t i = 0; i < ny->nkids; ++i) h->nodes[ny->kids[i]].parent = y;
  ny->caching = nx->caching;
  ny->la_mask = nx->la_mask;
  for (int g = 0; g < h->G; ++g) {
    ny->la[g] = nx->la[g];
    Stamps* a = &nx->hits[g];
    for (int64_t i = a->head; i < a->n; ++i) stamp_push(&ny->hits[g], a->t[i]);
    ny->ccc[g] = nx->ccc[g];
    nx->ccc[g] = cached_on(nx, g) ? 1 : 0;
  }
  add_kid(h, x, y);
  h->node_count++;
  return y;
}

/* ensure_path (prefix_tree.cpp:156-185) */
static int64_t ensure_path(e2_handle* h, const int32_t* p, int64_t len) {
  int64_t cur = 0, pos = 0;
  while (pos < len) {
    int64_t c = find_kid(h, cur, p[pos]);
    if (c < 0) {
      int64_t l = new_node(h, cur, p + pos, len - pos);
      add_kid(h, cur, l);
      h->node_count++;
      return l;
    }
    Node* ch = &h->nodes[c];
    int64_t lim = ch->len < len - pos ? ch->len : len - pos, k = 0;
    while (k < lim && ch->edge[k] == p[pos + k]) ++k;
    pos += k;
    if (k == ch->len) {
      cur = c;
      continue;
    }
    split_node(h, c, k);
    if (pos == len) return c;
    cur = c;
  }
  return cur;
}

/* record_hit (prefix_tree.cpp:45-51) */
static void record_hit(e2_handle* h, int64_t x, int g, double now) {
  Node* n = &h->nodes[x];
  stamp_push(&n->hits[g], now);
  n->la_mask |= 1ull << g;
  if (now > n->la[g]) n->la[g] = now;
}

/* set_cached (prefix_tree.cpp:53-63) */
static void set_cached(e2_handle* h, int64_t x, int g) {
  Node* n = &h->nodes[x];
  if (x == 0 || cached_on(n, g)) return;
  n->caching |= 1ull << g;
  h->cached_tokens[g] += n->len;
  if (n->parent >= 0) h->nodes[n->parent].ccc[g] += 1;
}

/* clear_cached (prefix_tree.cpp:65-77) */
static int clear_cached(e2_handle* h, int64_t x, int g) {
  Node* n = &h->nodes[x];
  if (!cached_on(n, g)) return 0;
  n->caching &= ~(1ull << g);
  h->cached_tokens[g] -= n->len;
  if (n->parent >= 0) {
    if (--h->nodes[n->parent].ccc[g] < 0) return E2_ERR_SIM;
  }
  return 0;
}

/* mark_cached_path (prefix_tree.cpp:200-213) */
static void mark_cached_path(e2_handle* h, const int32_t* p, int64_t len, int g, double now) {
  if (len == 0) return;
  for (int64_t x = ensure_path(h, p, len); x > 0; x = h->nodes[x].parent) {
    set_cached(h, x, g);
    Node* n = &h->nodes[x];
    n->la_mask |= 1ull << g;
    if (now > n->la[g]) n->la[g] = now;
  }
}

/* mark_cached_node (prefix_tree.cpp:215-222) */
static void mark_cached_node(e2_handle* h, int64_t x, int g, double now) {
  if (x <= 0) return;
  set_cached(h, x, g);
  Node* n = &h->nodes[x];
  n->la_mask |= 1ull << g;
  if (now > n->la[g]) n->la[g] = now;
}

static void mark_cached_subtree(e2_handle* h, int64_t x, int g, double now) {
  mark_cached_node(h, x, g, now);
  for (int64_t i = 0; i < h->nodes[x].nkids; ++i) mark_cached_subtree(h, h->nodes[x].kids[i], g, now);
}

static int uncache_subtree(e2_handle* h, int64_t x, int g) {
  for (int64_t i = 0; i < h->nodes[x].nkids; ++i) {
    int rc = uncache_subtree(h, h->nodes[x].kids[i], g);
    if (rc) return rc;
  }
  return x ? clear_cached(h, x, g) : 0;
}

/* uncache_suffix (prefix_tree.cpp:237-271) */
static int uncache_suffix(e2_handle* h, const int32_t* seq, int64_t len, int64_t tail, int g) {
  if (len == 0 || tail <= 0) return 0;
  Match m = walk(h, seq, len);
  int64_t end = len < m.matched_len ? len : m.matched_len;
  int64_t start = len - tail;
  if (start < 0) start = 0;
  if (start >= end) {
    match_free(&m);
    return 0;
  }
  int64_t* targets = (int64_t*)malloc(8 * (size_t)(m.nspan + 1));
  int64_t nt = 0, off = 0;
  for (int64_t i = 0; i < m.nspan; ++i) {
    if (off >= end) break;
    int64_t x = m.span_node[i];
    int64_t node_end = off + m.span_m[i];
    if (m.span_m[i] < h->nodes[x].len) split_node(h, x, m.span_m[i]);
    if (node_end > start) {
      if (off < start) {
        x = split_node(h, x, start - off);
        off = start;
      }
      targets[nt++] = x;
    }
    off = node_end;
  }
  int rc = 0;
  for (int64_t i = nt - 1; i >= 0 && !rc; --i) rc = clear_cached(h, targets[i], g);
  free(targets);
  match_free(&m);
  return rc ? fail(h, E2_ERR_SIM, "prefix_tree: cached_child_count underflow") : 0;
}

/* plan_eviction (prefix_tree.cpp:273-308), restated as the naive scan of
 * tests/oracle/reference_match.cpp:150-202: repeatedly take the least
 * (last_access, id) cached node whose cached children are all planned. */
static int64_t plan_eviction(e2_handle* h, int g, int64_t need, int partial, int64_t* vnode, int64_t* vtok,
                             int64_t* nv) {
  *nv = 0;
  if (need <= 0) return 0;
  char* planned = (char*)calloc((size_t)h->nn, 1);
  int64_t freed = 0;
  while (freed < need) {
    int64_t best = -1;
    for (int64_t x = 1; x < h->nn; ++x) {
      Node* n = &h->nodes[x];
      if (!n->alive || planned[x] || !cached_on(n, g)) continue;
      int blocked = 0;
      for (int64_t i = 0; i < n->nkids && !blocked; ++i) {
        int64_t c = n->kids[i];
        if (cached_on(&h->nodes[c], g) && !planned[c]) blocked = 1;
      }
      if (blocked) continue;
      if (best < 0) {
        best = x;
        continue;
      }
      Node* b = &h->nodes[best];
      double la = ((n->la_mask >> g) & 1u) ? n->la[g] : 0.0, lb = ((b->la_mask >> g) & 1u) ? b->la[g] : 0.0;
      if (la < lb || (la == lb && n->id < b->id)) best = x;
    }
    if (best < 0) break;
    int64_t sz = h->nodes[best].len, rem = need - freed;
    if (partial && sz > rem) {
      vnode[*nv] = best;
      vtok[(*nv)++] = rem;
      freed += rem;
      break;
    }
    vnode[*nv] = best;
    vtok[(*nv)++] = sz;
    freed += sz;
    planned[best] = 1;
  }
  free(planned);
  return freed;
}

/* ----------------------------------------------------------- load windows */
static void dq_push(Deque* q, double t, int64_t v, int64_t est) {
  if (q->n >= q->cap) {
    q->cap = q->cap ? 2 * q->cap : 64;
    q->e = (Ent*)realloc(q->e, (size_t)q->cap * sizeof(Ent));
  }
  q->e[q->n].t = t;
  q->e[q->n].v = v;
  q->e[q->n].est = est;
  q->n++;
}

/* LoadWindow::prune (cost_model.cpp:31-42) */
static void win_prune(e2_handle* h, int g, double now) {
  const double cut = now - h->cfg.history_window_ms;
  Deque* s = &h->sched[g];
  while (s->head < s->n && s->e[s->head].t < cut) {
    h->missed_sum[g] -= s->e[s->head].v;
    if (s->e[s->head].v > 0) h->missed_nz[g]--;
    s->head++;
  }
  Deque* c = &h->comp[g];
  while (c->head < c->n && c->e[c->head].t < cut) {
    h->output_sum[g] -= c->e[c->head].v;
    c->head++;
  }
}

static double prefill_time(const e2_time_model* m, int64_t missed) {
  if (missed <= 0) return 0.0;
  return m->prefill_base_ms + m->prefill_per_token_ms * (double)missed;
}

/* LoadWindow::load_ms (cost_model.cpp:65-73) */
static double win_load(e2_handle* h, int g, double now) {
  win_prune(h, g, now);
  int64_t ns = h->sched[g].n - h->sched[g].head, nc = h->comp[g].n - h->comp[g].head;
  double avg = nc == 0 ? (double)h->cfg.default_output_len : (double)h->output_sum[g] / (double)nc;
  double prefill = h->m.prefill_base_ms * (double)h->missed_nz[g] + h->m.prefill_per_token_ms * (double)h->missed_sum[g];
  double decode = (double)ns * (h->m.decode_per_token_ms * avg);
  return prefill + decode;
}

/* load_cost (cost_model.cpp:75-100) */
static e2_cost load_cost(e2_handle* h, int g, int64_t missed, double now) {
  e2_cost c;
  memset(&c, 0, sizeof c);
  c.gpu = g;
  c.current_load_ms = win_load(h, g, now);
  c.prefill_ms = prefill_time(&h->m, missed);
  int64_t need = missed - (h->cfg.kv_capacity_tokens - h->cached_tokens[g]);
  if (need > 0) {
    int64_t* vn = (int64_t*)malloc(8 * (size_t)(h->nn + 1));
    int64_t* vt = (int64_t*)malloc(8 * (size_t)(h->nn + 1));
    int64_t nv;
    int64_t freed = plan_eviction(h, g, need, 0, vn, vt, &nv);
    c.eviction_infeasible = freed < need;
    win_prune(h, g, now);
    int64_t total = h->sched[g].n - h->sched[g].head;
    if (total > 0)
      for (int64_t i = 0; i < nv; ++i) {
        double nj = (double)recent_hits(h, &h->nodes[vn[i]], g, now) / (double)total;
        c.eviction_ms += prefill_time(&h->m, vt[i]) * nj;
      }
    free(vn);
    free(vt);
  }
  return c;
}

static double total_ms(const e2_cost* c) { return (c->current_load_ms + c->eviction_ms) + c->prefill_ms; }

/* pick_min_cost (global_scheduler.cpp:54-74) */
static int pick_min(const e2_cost* c, int n) {
  int best = -1;
  double bt = 0;
  for (int i = 0; i < n; ++i) {
    if (c[i].eviction_infeasible) continue;
    if (best < 0 || total_ms(&c[i]) < bt) {
      best = c[i].gpu;
      bt = total_ms(&c[i]);
    }
  }
  if (best >= 0) return best;
  for (int i = 0; i < n; ++i)
    if (best < 0 || total_ms(&c[i]) < bt) {
      best = c[i].gpu;
      bt = total_ms(&c[i]);
    }
  return best;
}

/* ---------------------------------------------------------- the scheduler */
/* update_redirects (global_scheduler.cpp:194-219) */
static void update_redirects(e2_handle* h, double now) {
  double loads[E2_MAX_GPUS];
  for (int g = 0; g < h->G; ++g) loads[g] = win_load(h, g, now);
  for (int s = 0; s < h->G; ++s)
    if (h->redirect[s] >= 0 && loads[s] <= h->cfg.th_bal * loads[h->redirect[s]]) h->redirect[s] = -1;
  int hi = 0, lo = 0;
  for (int g = 1; g < h->G; ++g) {
    if (loads[g] > loads[hi]) hi = g;
    if (loads[g] < loads[lo]) lo = g;
  }
  if (hi == lo || !(loads[hi] > h->cfg.th_bal * loads[lo])) return;
  if (h->redirect[hi] != lo) {
    h->redirect[hi] = lo;
    h->st.rebalance_installs++;
  }
}

/* decide (global_scheduler.cpp:76-158) */
static int decide(e2_handle* h, const int32_t* p, int64_t len, int64_t id, double now, e2_decision* d, e2_cost* costs,
                  double* ratios, Match* out_m) {
  memset(d, 0, sizeof *d);
  d->request = id;
  d->gpu = -1;
  d->pre_redirect_gpu = -1;
  d->branch = E2_BRANCH_EXPLORE;
  if (len > h->cfg.kv_capacity_tokens) return fail(h, E2_ERR_NO_ADMISSIBLE, "prompt exceeds every GPU's KV capacity");
  if (h->pol.mode == E2_MODE_ROUND_ROBIN) {
    d->branch = E2_BRANCH_ROUND_ROBIN;
    d->gpu = (int32_t)(h->rr_next % h->G);
    d->missed_len = d->missed_on_chosen = len;
    return 0;
  }
  h->st.tree_reads++;
  Match m = walk(h, p, len);
  d->matched_len = m.matched_len;
  d->cached_len = m.cached_len;
  d->missed_len = len - m.cached_len;
  int nc = 0;
  if (d->missed_len < d->cached_len) {
    d->branch = E2_BRANCH_EXPLOIT;
    int64_t best = 0;
    for (int g = 0; g < h->G; ++g)
      if (((m.present >> g) & 1u) && m.per_gpu[g] > best) best = m.per_gpu[g];
    for (int g = 0; g < h->G; ++g)
      if (((m.present >> g) & 1u) && m.per_gpu[g] == best) costs[nc++] = load_cost(h, g, len - m.per_gpu[g], now);
    d->gpu = pick_min(costs, nc);
    if (d->gpu >= 0 && h->redirect[d->gpu] >= 0 && h->redirect[d->gpu] != d->gpu) {
      int t = h->redirect[d->gpu], ti = -1;
      for (int i = 0; i < nc; ++i)
        if (costs[i].gpu == t) ti = i;
      if (ti < 0) {
        costs[nc] = load_cost(h, t, len - matched_on(&m, t), now);
        ti = nc++;
      }
      if (!costs[ti].eviction_infeasible) {
        d->redirected = 1;
        d->pre_redirect_gpu = d->gpu;
        d->gpu = t;
      }
    }
  } else {
    d->has_ratios = 1;
    int max_g = -1;
    double max_r = -1.0;
    for (int g = 0; g < h->G; ++g) {
      ratios[g] = h->inflight_prompt[g] <= 0 ? 0.0 : (double)h->inflight_cached[g] / (double)h->inflight_prompt[g];
      if (ratios[g] > max_r) {
        max_r = ratios[g];
        max_g = g;
      }
    }
    if (h->pol.pd_balance && max_r > h->cfg.imbal_ratio) {
      d->branch = E2_BRANCH_DECODE_PRESSURE;
      d->gpu = max_g;
    } else {
      for (int g = 0; g < h->G; ++g) costs[nc++] = load_cost(h, g, len - matched_on(&m, g), now);
      d->gpu = pick_min(costs, nc);
    }
  }
  d->n_costs = nc;
  if (d->gpu < 0 || d->gpu >= h->G) {
    match_free(&m);
    return fail(h, E2_ERR_SIM, "global_scheduler: cached spans are not root-contiguous on any GPU");
  }
  d->missed_on_chosen = len - matched_on(&m, d->gpu);
  if (out_m)
    *out_m = m;
  else
    match_free(&m);
  return 0;
}

static Inflight* inf_find(e2_handle* h, int64_t id) {
  for (int64_t i = 0; i < h->ninf; ++i)
    if (h->inf[i].used && h->inf[i].key == id) return &h->inf[i];
  return NULL;
}

/* commit (global_scheduler.cpp:160-175) */
static int commit(e2_handle* h, const int32_t* p, int64_t len, int64_t id, double arrival, const e2_decision* d,
                  double now) {
  if (h->pol.mode == E2_MODE_ROUND_ROBIN) {
    h->rr_next++;
    return 0;
  }
  if (len == 0) return fail(h, E2_ERR_SIM, "prefix_tree: insert of empty sequence");
  int64_t tail = ensure_path(h, p, len), first = tail;
  for (int64_t x = tail; x > 0; x = h->nodes[x].parent) {
    record_hit(h, x, d->gpu, now);
    first = x;
  }
  int g = d->gpu;
  dq_push(&h->sched[g], now, d->missed_on_chosen, h->cfg.default_output_len);
  h->missed_sum[g] += d->missed_on_chosen;
  if (d->missed_on_chosen > 0) h->missed_nz[g]++;
  h->inflight_cached[g] += d->cached_len;
  h->inflight_prompt[g] += len;
  Inflight* f = inf_find(h, id);
  if (!f) {
    GROW(h->inf, h->ninf, h->capinf, Inflight);
    f = &h->inf[h->ninf++];
  }
  f->used = 1;
  f->key = id;
  f->gpu = g;
  f->cached = d->cached_len;
  f->prompt = len;
  f->arrival = arrival;
  f->root = h->nodes[first].id;
  return 0;
}

static int64_t subtree_tokens(e2_handle* h, int64_t x) {
  int64_t t = h->nodes[x].len;
  for (int64_t i = 0; i < h->nodes[x].nkids; ++i) t += subtree_tokens(h, h->nodes[x].kids[i]);
  return t;
}

static uint64_t subtree_gpus(e2_handle* h, int64_t x) {
  uint64_t m = h->nodes[x].caching;
  for (int64_t i = 0; i < h->nodes[x].nkids; ++i) m |= subtree_gpus(h, h->nodes[x].kids[i]);
  return m;
}

typedef struct {
  int64_t node;
  double load;
} Kid;

static int kid_cmp_ctx_ids(const e2_handle* h, const Kid* a, const Kid* b) {
  if (a->load != b->load) return a->load > b->load ? -1 : 1;
  return h->nodes[a->node].id < h->nodes[b->node].id ? -1 : 1;
}

/* replicate_prefix (global_scheduler.cpp:299-338) */
static int replicate_prefix(e2_handle* h, int64_t rc, int target, double now) {
  mark_cached_node(h, rc, target, now);
  int64_t nk = h->nodes[rc].nkids;
  Kid* kids = (Kid*)malloc(sizeof(Kid) * (size_t)(nk + 1));
  for (int64_t i = 0; i < nk; ++i) {
    int64_t c = h->nodes[rc].kids[i];
    prune_hits(h, &h->nodes[c], now);
    int64_t hits = 0;
    for (int g = 0; g < h->G; ++g) hits += h->nodes[c].hits[g].n - h->nodes[c].hits[g].head;
    kids[i].node = c;
    kids[i].load = (double)hits * prefill_time(&h->m, subtree_tokens(h, c));
  }
  for (int64_t i = 1; i < nk; ++i) /* insertion sort: load desc, id asc */
    for (int64_t j = i; j > 0 && kid_cmp_ctx_ids(h, &kids[j], &kids[j - 1]) < 0; --j) {
      Kid t = kids[j];
      kids[j] = kids[j - 1];
      kids[j - 1] = t;
    }
  double stay = 0, move = 0;
  int rc2 = 0;
  for (int64_t i = 0; i < nk && !rc2; ++i) {
    if (move < stay) {
      move += kids[i].load;
      uint64_t owners = subtree_gpus(h, kids[i].node);
      mark_cached_subtree(h, kids[i].node, target, now);
      for (int g = 0; g < h->G && !rc2; ++g)
        if (((owners >> g) & 1u) && g != target) rc2 = uncache_subtree(h, kids[i].node, g);
    } else {
      stay += kids[i].load;
    }
  }
  free(kids);
  return rc2;
}

/* check_autoscale (global_scheduler.cpp:236-297) */
static int check_autoscale(e2_handle* h, double now) {
  const int64_t cur = (int64_t)floor(now / h->cfg.history_window_ms);
  /* process roots in ascending id order */
  uint64_t prev_root = 0;
  int have_prev = 0;
  for (;;) {
    uint64_t root = 0;
    int found = 0;
    for (int64_t i = 0; i < h->nq; ++i)
      if (h->q[i].alive && (!have_prev || h->q[i].root > prev_root) && (!found || h->q[i].root < root)) {
        root = h->q[i].root;
        found = 1;
      }
    if (!found) break;
    prev_root = root;
    have_prev = 1;
    int any = 0;
    QCell *pc = NULL, *cc = NULL;
    for (int64_t i = 0; i < h->nq; ++i) {
      QCell* q = &h->q[i];
      if (!q->alive || q->root != root) continue;
      if (q->bucket < cur - 1) {
        q->alive = 0;
        continue;
      }
      any = 1;
      if (q->bucket == cur - 1) pc = q;
      if (q->bucket == cur) cc = q;
    }
    if (!any) continue;
    int fired = 0;
    if (pc && cc && pc->count > 0 && cc->count > 0) {
      double pm = pc->sum / (double)pc->count, cm = cc->sum / (double)cc->count;
      if (pm > 0 && cm >= 2.0 * pm) {
        int64_t rcn = -1;
        for (int64_t i = 0; i < h->nodes[0].nkids; ++i)
          if (h->nodes[h->nodes[0].kids[i]].id == root) rcn = h->nodes[0].kids[i];
        int src = -1;
        if (rcn >= 0)
          for (int s = 0; s < h->G; ++s)
            if (h->redirect[s] >= 0 && cached_on(&h->nodes[rcn], s)) {
              src = s;
              break;
            }
        if (src >= 0) {
          int target = -1;
          double tl = 0;
          for (int g = 0; g < h->G; ++g) {
            if (cached_on(&h->nodes[rcn], g)) continue;
            double l = win_load(h, g, now);
            if (target < 0 || l < tl) {
              target = g;
              tl = l;
            }
          }
          if (target >= 0) {
            int rc = replicate_prefix(h, rcn, target, now);
            if (rc) return fail(h, E2_ERR_SIM, "prefix_tree: cached_child_count underflow");
            h->st.autoscale_events++;
            fired = 1;
          }
        }
      }
    }
    if (fired)
      for (int64_t i = 0; i < h->nq; ++i)
        if (h->q[i].root == root) h->q[i].alive = 0;
  }
  return 0;
}

/* -------------------------------------------------------------- C ABI */
const char* e2_backend(void) { return "oracle"; }

int e2_create(int32_t n, const e2_sched_cfg* cfg, const e2_time_model* m, const e2_policy* p, e2_handle** out) {
  *out = NULL;
  const char* why = NULL;
  if (n < 1) why = "cluster needs at least one GPU";
  else if (!(cfg->history_window_ms > 0)) why = "history_window_ms must be > 0";
  else if (!(cfg->th_bal > 1.0)) why = "th_bal must be > 1";
  else if (!(cfg->imbal_ratio > 0.0 && cfg->imbal_ratio <= 1.0)) why = "imbal_ratio must be in (0,1]";
  else if (cfg->priority_groups < 1) why = "priority_groups must be >= 1";
  else if (cfg->kv_capacity_tokens <= 0) why = "kv_capacity_tokens must be > 0";
  else if (cfg->default_output_len < 0) why = "default_output_len must be >= 0";
  if (why) {
    snprintf(g_err, sizeof g_err, "%s", why);
    return E2_ERR_CONFIG;
  }
  if (n > E2_MAX_GPUS) {
    snprintf(g_err, sizeof g_err, "at most 64 instances");
    return E2_ERR_ARG;
  }
  e2_handle* h = (e2_handle*)calloc(1, sizeof *h);
  h->G = n;
  h->cfg = *cfg;
  h->m = *m;
  h->pol = *p;
  for (int g = 0; g < E2_MAX_GPUS; ++g) h->redirect[g] = -1;
  new_node(h, -1, NULL, 0); /* root, id 0 (prefix_tree.cpp:9-12) */
  *out = h;
  return E2_OK;
}

static void free_state(e2_handle* h) {
  for (int64_t i = 0; i < h->nn; ++i) {
    Node* n = &h->nodes[i];
    free(n->edge);
    free(n->kids);
    free(n->la);
    free(n->ccc);
    for (int g = 0; g < h->G; ++g) free(n->hits[g].t);
    free(n->hits);
  }
  free(h->nodes);
  for (int g = 0; g < E2_MAX_GPUS; ++g) {
    free(h->sched[g].e);
    free(h->comp[g].e);
  }
  free(h->inf);
  free(h->q);
}

void e2_destroy(e2_handle* h) {
  if (!h) return;
  free_state(h);
  free(h);
}

int e2_reset(e2_handle* h) {
  int G = h->G;
  e2_sched_cfg c = h->cfg;
  e2_time_model m = h->m;
  e2_policy p = h->pol;
  free_state(h);
  memset(h, 0, sizeof *h);
  h->G = G;
  h->cfg = c;
  h->m = m;
  h->pol = p;
  for (int g = 0; g < E2_MAX_GPUS; ++g) h->redirect[g] = -1;
  new_node(h, -1, NULL, 0);
  return E2_OK;
}

int e2_set_stream(e2_handle* h, void* s) {
  (void)h;
  (void)s;
  return E2_OK;
}

const char* e2_last_error(const e2_handle* h) { return h ? h->err : g_err; }

static int bad_gpu(e2_handle* h, int g) { return (g < 0 || g >= h->G) ? fail(h, E2_ERR_ARG, "gpu id out of range") : 0; }

/* schedule_request (global_scheduler.cpp:177-192) */
int e2_schedule(e2_handle* h, const int32_t* p, int64_t len, int64_t id, double arrival, double now, e2_decision* out,
                e2_cost* costs, double* ratios) {
  if (h->pol.mode == E2_MODE_PREFIX_AWARE && h->pol.rebalance && h->G > 1) update_redirects(h, now);
  e2_decision d;
  e2_cost cs[E2_MAX_GPUS + 1];
  double rs[E2_MAX_GPUS];
  int rc = decide(h, p, len, id, now, &d, cs, rs, NULL);
  if (rc) return rc;
  rc = commit(h, p, len, id, arrival, &d, now);
  if (rc) return rc;
  switch (d.branch) {
    case E2_BRANCH_EXPLOIT: h->st.exploit++; break;
    case E2_BRANCH_EXPLORE: h->st.explore++; break;
    case E2_BRANCH_DECODE_PRESSURE: h->st.decode_pressure++; break;
    default: h->st.round_robin++; break;
  }
  if (d.redirected) h->st.redirected++;
  if (h->pol.mode == E2_MODE_PREFIX_AWARE && h->pol.autoscale) {
    rc = check_autoscale(h, now);
    if (rc) return rc;
  }
  if (out) *out = d;
  if (costs) memcpy(costs, cs, sizeof(e2_cost) * (size_t)d.n_costs);
  if (ratios && d.has_ratios) memcpy(ratios, rs, sizeof(double) * (size_t)h->G);
  return 0;
}

int e2_decide(e2_handle* h, const int32_t* p, int64_t len, int64_t id, double now, e2_decision* out, e2_cost* costs,
              double* ratios) {
  e2_decision d;
  e2_cost cs[E2_MAX_GPUS + 1];
  double rs[E2_MAX_GPUS];
  int rc = decide(h, p, len, id, now, &d, cs, rs, NULL);
  if (rc) return rc;
  if (out) *out = d;
  if (costs) memcpy(costs, cs, sizeof(e2_cost) * (size_t)d.n_costs);
  if (ratios && d.has_ratios) memcpy(ratios, rs, sizeof(double) * (size_t)h->G);
  return 0;
}

/* note_admitted (global_scheduler.cpp:340-348) */
int e2_note_admitted(e2_handle* h, int64_t id, double now) {
  if (h->pol.mode != E2_MODE_PREFIX_AWARE) return 0;
  Inflight* f = inf_find(h, id);
  if (!f) return 0;
  int64_t b = (int64_t)floor(now / h->cfg.history_window_ms);
  for (int64_t i = 0; i < h->nq; ++i)
    if (h->q[i].alive && h->q[i].root == f->root && h->q[i].bucket == b) {
      h->q[i].sum += now - f->arrival;
      h->q[i].count++;
      return 0;
    }
  GROW(h->q, h->nq, h->capq, QCell);
  QCell* q = &h->q[h->nq++];
  q->root = f->root;
  q->bucket = b;
  q->sum = now - f->arrival;
  q->count = 1;
  q->alive = 1;
  return 0;
}

int e2_note_prefill_cached(e2_handle* h, const int32_t* p, int64_t len, int32_t gpu, double now) {
  if (bad_gpu(h, gpu)) return E2_ERR_ARG;
  if (h->pol.mode != E2_MODE_PREFIX_AWARE) return 0;
  mark_cached_path(h, p, len, gpu, now);
  return 0;
}

int e2_note_eviction(e2_handle* h, const int32_t* seq, int64_t len, int64_t tail, int32_t gpu, double now) {
  (void)now;
  if (bad_gpu(h, gpu)) return E2_ERR_ARG;
  if (h->pol.mode != E2_MODE_PREFIX_AWARE) return 0;
  return uncache_suffix(h, seq, len, tail, gpu);
}

/* note_finished (global_scheduler.cpp:361-369) */
int e2_note_finished(e2_handle* h, int64_t id, double now, int64_t out) {
  Inflight* f = inf_find(h, id);
  if (!f) return 0;
  int g = f->gpu;
  dq_push(&h->comp[g], now, out, 0);
  h->output_sum[g] += out;
  h->inflight_cached[g] -= f->cached;
  h->inflight_prompt[g] -= f->prompt;
  f->used = 0;
  return 0;
}

int e2_decode_ratio(e2_handle* h, int32_t g, double* out) {
  if (bad_gpu(h, g)) return E2_ERR_ARG;
  *out = h->inflight_prompt[g] <= 0 ? 0.0 : (double)h->inflight_cached[g] / (double)h->inflight_prompt[g];
  return 0;
}

int e2_gpu_load_ms(e2_handle* h, int32_t g, double now, double* out) {
  if (bad_gpu(h, g)) return E2_ERR_ARG;
  *out = win_load(h, g, now);
  return 0;
}

/* remove_dead_nodes (prefix_tree.cpp:357-378) */
static int64_t remove_dead(e2_handle* h, int64_t x, double now) {
  int64_t removed = 0;
  for (int64_t i = 0; i < h->nodes[x].nkids;) {
    int64_t c = h->nodes[x].kids[i];
    removed += remove_dead(h, c, now);
    Node* n = &h->nodes[c];
    prune_hits(h, n, now);
    int empty = 1;
    for (int g = 0; g < h->G; ++g)
      if (n->hits[g].n > n->hits[g].head) empty = 0;
    if (!n->caching && n->nkids == 0 && empty) {
      n->alive = 0;
      del_kid(h, x, c);
      h->node_count--;
      removed++;
    } else {
      ++i;
    }
  }
  return removed;
}

int e2_prune_dead_nodes(e2_handle* h, double now, int64_t* removed) {
  *removed = remove_dead(h, 0, now);
  return 0;
}

int e2_cached_tokens(e2_handle* h, int32_t g, int64_t* out) {
  if (bad_gpu(h, g)) return E2_ERR_ARG;
  *out = h->cached_tokens[g];
  return 0;
}

int e2_node_count(e2_handle* h, int64_t* out) {
  *out = h->node_count;
  return 0;
}

int e2_redirects(e2_handle* h, int32_t* out) {
  for (int g = 0; g < h->G; ++g) out[g] = h->redirect[g];
  return 0;
}

int e2_get_stats(e2_handle* h, e2_stats* out) {
  *out = h->st;
  return 0;
}

int e2_load_cost(e2_handle* h, int32_t g, int64_t missed, double now, e2_cost* out) {
  if (bad_gpu(h, g)) return E2_ERR_ARG;
  *out = load_cost(h, g, missed, now);
  return 0;
}

int e2_match(e2_handle* h, const int32_t* seq, int64_t len, int64_t* ml, int64_t* cl, int64_t* per) {
  Match m = walk(h, seq, len);
  if (ml) *ml = m.matched_len;
  if (cl) *cl = m.cached_len;
  if (per)
    for (int g = 0; g < h->G; ++g) per[g] = matched_on(&m, g);
  match_free(&m);
  return 0;
}

/* export_nodes (prefix_tree.cpp:436-461): DFS, child-token order */
static void dfs(e2_handle* h, int64_t x, int64_t* order, int64_t* depth, int64_t* n, int64_t d) {
  order[*n] = x;
  depth[(*n)++] = d;
  for (int64_t i = 0; i < h->nodes[x].nkids; ++i) dfs(h, h->nodes[x].kids[i], order, depth, n, d + 1);
}

int e2_export_size(e2_handle* h, int64_t* nn, int64_t* nt) {
  int64_t* o = (int64_t*)malloc(8 * (size_t)h->nn);
  int64_t* d = (int64_t*)malloc(8 * (size_t)h->nn);
  int64_t n = 0, t = 0;
  dfs(h, 0, o, d, &n, 0);
  for (int64_t i = 0; i < n; ++i) t += h->nodes[o[i]].len;
  *nn = n;
  *nt = t;
  free(o);
  free(d);
  return 0;
}

static int64_t windowed(e2_handle* h, Node* n, int g, double now) {
  int64_t c = 0;
  for (int64_t i = n->hits[g].head; i < n->hits[g].n; ++i) c += n->hits[g].t[i] >= now - h->cfg.history_window_ms;
  return c;
}

int e2_export(e2_handle* h, double now, e2_node* nodes, int32_t* tokens, double* la, int64_t* hits) {
  int64_t* o = (int64_t*)malloc(8 * (size_t)h->nn);
  int64_t* d = (int64_t*)malloc(8 * (size_t)h->nn);
  int64_t n = 0, off = 0;
  dfs(h, 0, o, d, &n, 0);
  for (int64_t i = 0; i < n; ++i) {
    Node* x = &h->nodes[o[i]];
    if (nodes) {
      nodes[i].id = x->id;
      nodes[i].parent_id = x->parent >= 0 ? h->nodes[x->parent].id : x->id;
      nodes[i].edge_off = off;
      nodes[i].edge_len = x->len;
      nodes[i].caching_mask = x->caching;
      nodes[i].last_access_mask = x->la_mask;
      nodes[i].pin_count = 0;
    }
    if (tokens && x->len) memcpy(tokens + off, x->edge, (size_t)x->len * 4);
    off += x->len;
    for (int g = 0; g < h->G; ++g) {
      if (la) la[i * h->G + g] = ((x->la_mask >> g) & 1u) ? x->la[g] : 0.0;
      if (hits) hits[i * h->G + g] = windowed(h, x, g, now);
    }
  }
  free(o);
  free(d);
  return 0;
}

/* debug_dump (prefix_tree.cpp:411-455), with windowed counts */
int e2_debug_dump(e2_handle* h, double now, char* buf, size_t cap, size_t* needed) {
  int64_t* o = (int64_t*)malloc(8 * (size_t)h->nn);
  int64_t* d = (int64_t*)malloc(8 * (size_t)h->nn);
  int64_t n = 0;
  dfs(h, 0, o, d, &n, 0);
  size_t sz = 0, scap = 4096;
  char* s = (char*)malloc(scap);
  for (int64_t i = 0; i < n; ++i) {
    Node* x = &h->nodes[o[i]];
    char line[8192];
    int k = 0;
    for (int64_t j = 0; j < d[i]; ++j) k += snprintf(line + k, sizeof line - (size_t)k, "  ");
    k += snprintf(line + k, sizeof line - (size_t)k, "d%lld len=%lld gpus=[", (long long)d[i], (long long)x->len);
    int first = 1;
    for (int g = 0; g < h->G; ++g)
      if (cached_on(x, g)) {
        k += snprintf(line + k, sizeof line - (size_t)k, first ? "%d" : ",%d", g);
        first = 0;
      }
    k += snprintf(line + k, sizeof line - (size_t)k, "] hits=[");
    first = 1;
    for (int g = 0; g < h->G; ++g) {
      int64_t c = windowed(h, x, g, now);
      if (!c) continue;
      k += snprintf(line + k, sizeof line - (size_t)k, first ? "%d:%lld" : ",%d:%lld", g, (long long)c);
      first = 0;
    }
    k += snprintf(line + k, sizeof line - (size_t)k, "]\n");
    while (sz + (size_t)k + 1 > scap) {
      scap *= 2;
      s = (char*)realloc(s, scap);
    }
    memcpy(s + sz, line, (size_t)k);
    sz += (size_t)k;
  }
  if (needed) *needed = sz;
  if (buf && cap) {
    size_t k = sz < cap - 1 ? sz : cap - 1;
    memcpy(buf, s, k);
    buf[k] = 0;
  }
  free(s);
  free(o);
  free(d);
  return 0;
}

int e2_window_sizes(e2_handle* h, int32_t g, double now, int64_t* ns, int64_t* nc, int64_t* ic, int64_t* ip) {
  if (bad_gpu(h, g)) return E2_ERR_ARG;
  win_prune(h, g, now);
  if (ns) *ns = h->sched[g].n - h->sched[g].head;
  if (nc) *nc = h->comp[g].n - h->comp[g].head;
  if (ic) *ic = h->inflight_cached[g];
  if (ip) *ip = h->inflight_prompt[g];
  return 0;
}

/* path_tokens (prefix_tree.cpp:400-408) length: depth of the node's end */
static int64_t path_end(e2_handle* h, int64_t x, int32_t** out) {
  int64_t len = 0;
  for (int64_t y = x; y > 0; y = h->nodes[y].parent) len += h->nodes[y].len;
  *out = (int32_t*)malloc(4 * (size_t)(len + 1));
  int64_t pos = len;
  for (int64_t y = x; y > 0; y = h->nodes[y].parent) {
    pos -= h->nodes[y].len;
    memcpy(*out + pos, h->nodes[y].edge, (size_t)h->nodes[y].len * 4);
  }
  return len;
}

/* the generalised criterion-7 loop (acceptance_main.cpp:367-416; e2sched.h) */
int e2_replay(e2_handle* h, const int32_t* tokens, const int64_t* offsets, const int64_t* ids, const double* arrivals,
              const int64_t* outl, int64_t n, const e2_driver_cfg* drv, e2_decision* out, e2_cost* costs,
              double* ratios, int64_t* n_done) {
  int G = h->G;
  int64_t* fk = (int64_t*)malloc(8 * (size_t)(n + 1) * (size_t)G);
  int64_t* ft = (int64_t*)malloc(8 * (size_t)(n + 1) * (size_t)G);
  int64_t fh[E2_MAX_GPUS] = {0}, fn[E2_MAX_GPUS] = {0};
  double now = 0;
  double tick = drv->prune_interval_ms > 0 ? drv->prune_interval_ms : 0;
  int rc = 0;
  int64_t i;
  for (i = 0; i < n; ++i) {
    if (arrivals[i] > now) now = arrivals[i];
    while (tick > 0 && tick <= now) { /* prune ticks (simulator.cpp:217-229) */
      int64_t removed = 0;
      e2_prune_dead_nodes(h, tick, &removed);
      tick += drv->prune_interval_ms;
    }
    const int32_t* p = tokens + offsets[i];
    int64_t len = offsets[i + 1] - offsets[i];
    Match mm = walk(h, p, len);
    int64_t matched = mm.matched_len;
    match_free(&mm);
    e2_decision d;
    rc = e2_schedule(h, p, len, ids[i], arrivals[i], now, &d, costs ? costs + i * (G + 1) : NULL,
                     ratios ? ratios + i * G : NULL);
    if (rc) break;
    d.matched_len = h->pol.mode == E2_MODE_ROUND_ROBIN ? 0 : matched;
    if (out) out[i] = d;
    int g = d.gpu;
    if (drv->prefill_cached) e2_note_prefill_cached(h, p, len, g, now);
    if (drv->eviction == E2_EVICT_FIFO_TAIL) {
      fk[(size_t)g * (n + 1) + fn[g]] = i;
      ft[(size_t)g * (n + 1) + fn[g]] = len - drv->trunk_len;
      fn[g]++;
      while (h->cached_tokens[g] > drv->high_water && fh[g] < fn[g]) {
        int64_t k = fk[(size_t)g * (n + 1) + fh[g]], t = ft[(size_t)g * (n + 1) + fh[g]];
        fh[g]++;
        rc = e2_note_eviction(h, tokens + offsets[k], offsets[k + 1] - offsets[k], t, g, now);
        if (rc) break;
      }
    } else if (drv->eviction == E2_EVICT_MIRROR_LRU && h->cached_tokens[g] > drv->high_water &&
               h->pol.mode == E2_MODE_PREFIX_AWARE) {
      int64_t* vn = (int64_t*)malloc(8 * (size_t)h->nn);
      int64_t* vt = (int64_t*)malloc(8 * (size_t)h->nn);
      int64_t nv;
      plan_eviction(h, g, h->cached_tokens[g] - drv->high_water, 1, vn, vt, &nv);
      int32_t** seqs = (int32_t**)malloc(sizeof(int32_t*) * (size_t)(nv + 1));
      int64_t* lens = (int64_t*)malloc(8 * (size_t)(nv + 1));
      for (int64_t v = 0; v < nv; ++v) lens[v] = path_end(h, vn[v], &seqs[v]);
      for (int64_t v = 0; v < nv && !rc; ++v) rc = e2_note_eviction(h, seqs[v], lens[v], vt[v], g, now);
      for (int64_t v = 0; v < nv; ++v) free(seqs[v]);
      free(seqs);
      free(lens);
      free(vn);
      free(vt);
    }
    if (rc) break;
    if (i >= drv->finish_lag) e2_note_finished(h, ids[i - drv->finish_lag], now, outl[i - drv->finish_lag]);
  }
  free(fk);
  free(ft);
  if (n_done) *n_done = i;
  return rc;
}

int e2_replay_device(e2_handle* h, const int32_t* a, const int64_t* b, const int64_t* c, const double* d,
                     const int64_t* e, int64_t n, const e2_driver_cfg* drv, e2_decision* o, e2_cost* co, double* r,
                     void* s, int64_t* nd) {
  (void)a, (void)b, (void)c, (void)d, (void)e, (void)n, (void)drv, (void)o, (void)co, (void)r, (void)s, (void)nd;
  return fail(h, E2_ERR_ARG, "the C oracle has no device path");
}

int e2_profile_get(e2_handle* h, e2_profile* out) {
  (void)h;
  memset(out, 0, sizeof *out);
  return 0;
}

int e2_profile_reset(e2_handle* h, int32_t enable) {
  (void)h;
  (void)enable;
  return 0;
}

void e2_workload_default(int32_t archetype, e2_workload_spec* out) {
  memset(out, 0, sizeof *out);
  out->archetype = archetype;
}

int e2_generate(const e2_workload_spec* spec, uint64_t seed, double rps, uint64_t aseed, int64_t* nr, int64_t* nt,
                int32_t* tokens, int64_t* offsets, int64_t* ids, double* arrivals, int64_t* outl) {
  (void)spec, (void)seed, (void)rps, (void)aseed, (void)nr, (void)nt, (void)tokens, (void)offsets, (void)ids,
      (void)arrivals, (void)outl;
  snprintf(g_err, sizeof g_err, "the C oracle does not generate traces");
  return E2_ERR_ARG;
}
