/*
 * ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product library.
 *
 * Plain-C99 restatement of the reference flow-level simulator's hot path
 * (/root/reference/proj/src/core), written from its semantics in a different
 * structure: one event heap with stale entries (engine.cpp:110-112, 601-609),
 * full re-computation of classes and rates after every dirty event
 * (engine.cpp:278-293), the five policies (baselines.cpp, rmlq.cpp), the
 * strict-priority progressive filling (allocator.cpp:28-126), RMLQ promotion
 * (rmlq.cpp:101-193), Algorithm 1 (rmlq.cpp:268-382, inter_request.cpp), the
 * stage DAG (engine.cpp:295-593) and the report reduction (engine.cpp:659-707).
 * Inputs come from the same config text: fabric (topology.cpp), workload
 * synthesis with the same splitmix64 stream and libm calls (workload.cpp) and
 * derive_slos by isolated runs (workload.cpp:177-217).
 *
 * Pinned by tests/test_oracle_restatement.py against the golden fixtures that
 * the reference itself produced (tests/golden/). Exposes the same C ABI as
 * oracle/ref_harness.cpp (ref_result), so oracle/ref.py drives either.
 */
#define _GNU_SOURCE
#include <ctype.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define NOT (-1.0)
#define INF (__builtin_inf())
#define MAXK 64

/* ------------------------------------------------------------------ util */

typedef struct {
  void* p;
  long n, cap;
  size_t es;
} vec;

static void* vpush(vec* v, const void* x) {
  if (v->n == v->cap) {
    v->cap = v->cap ? v->cap * 2 : 16;
    v->p = realloc(v->p, v->cap * v->es);
  }
  void* dst = (char*)v->p + v->n * v->es;
  memcpy(dst, x, v->es);
  v->n++;
  return dst;
}
#define VEC(T) {NULL, 0, 0, sizeof(T)}
#define AT(v, T, i) (((T*)(v).p)[i])

static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */
static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */

typedef struct {
  int err;
  char msg[512];
} errstate;
static __thread errstate E;
static void fail(int code, const char* m) {
  if (!E.err) {
    E.err = code;
    snprintf(E.msg, sizeof E.msg, "%s", m);
  }
}

/* ------------------------------------------------------- config (config.cpp) */

typedef struct {
  char** k;
  char** v;
  int n;
} kvcfg;

static char* trimdup(const char* b, const char* e) {
  while (b < e && isspace((unsigned char)*b)) ++b;
  while (e > b && isspace((unsigned char)e[-1])) --e;
  char* s = malloc(e - b + 1);
  memcpy(s, b, e - b);
  s[e - b] = 0;
  return s;
}
static void cfg_set(kvcfg* c, const char* k, const char* v) {
  for (int i = 0; i < c->n; ++i)
    if (!strcmp(c->k[i], k)) {
      free(c->v[i]);
      c->v[i] = strdup(v);
      return;
    }
  c->k = realloc(c->k, sizeof(char*) * (c->n + 1));
  c->v = realloc(c->v, sizeof(char*) * (c->n + 1));
  c->k[c->n] = strdup(k);
  c->v[c->n] = strdup(v);
  c->n++;
}
static void cfg_parse(kvcfg* c, const char* text) { /* config.cpp:28-48 */
  const char* p = text;
  while (*p) {
    const char* nl = strchr(p, '\n');
    const char* end = nl ? nl : p + strlen(p);
    const char* hash = memchr(p, '#', end - p);
    const char* le = hash ? hash : end;
    const char* eq = memchr(p, '=', le - p);
    char* line = trimdup(p, le);
    if (*line) {
      if (!eq) {
        fail(2, "config: expected key = value");
      } else {
        char* k = trimdup(p, eq);
        char* v = trimdup(eq + 1, le);
        if (!*k) fail(2, "config: empty key");
        cfg_set(c, k, v);
        free(k);
        free(v);
      }
    }
    free(line);
    p = nl ? nl + 1 : end;
  }
}
static const char* cfg_raw(const kvcfg* c, const char* k) {
  for (int i = 0; i < c->n; ++i)
    if (!strcmp(c->k[i], k)) return c->v[i];
  return NULL;
}
static double cfg_num(const kvcfg* c, const char* k, double d) {
  const char* v = cfg_raw(c, k);
  if (!v) return d;
  char* e;
  double x = strtod(v, &e);
  if (e == v || *e) fail(2, "config: not a number");
  return x;
}
static long cfg_long(const kvcfg* c, const char* k, long d) {
  const char* v = cfg_raw(c, k);
  if (!v) return d;
  double x = cfg_num(c, k, 0);
  long l = (long)x;
  if ((double)l != x) fail(2, "config: expected integer");
  return l;
}
static int cfg_bool(const kvcfg* c, const char* k, int d) {
  const char* v = cfg_raw(c, k);
  if (!v) return d;
  char s[16];
  int i = 0;
  for (; v[i] && i < 15; ++i) s[i] = (char)tolower((unsigned char)v[i]);
  s[i] = 0;
  if (!strcmp(s, "true") || !strcmp(s, "1") || !strcmp(s, "yes") || !strcmp(s, "on")) return 1;
  if (!strcmp(s, "false") || !strcmp(s, "0") || !strcmp(s, "no") || !strcmp(s, "off")) return 0;
  fail(2, "config: expected boolean");
  return d;
}
static void cfg_free(kvcfg* c) {
  for (int i = 0; i < c->n; ++i) {
    free(c->k[i]);
    free(c->v[i]);
  }
  free(c->k);
  free(c->v);
}

/* ---------------------------------------------------- fabric (topology.cpp) */

typedef struct {
  int nn, nl;
  int* from;
  int* to;
  double* cap;
  int hosts;
  /* adjacency: out (ascending ids) and in, CSR */
  int *oo, *ol, *io, *il;
  /* routes per (src,dst) on demand: cache dist arrays per dst */
  int** dist;
} fabric;

static void fab_add_node(fabric* f) { f->nn++; }
static void fab_add_link(fabric* f, int a, int b, double c) {
  if (c <= 0) fail(2, "link capacity must be positive");
  f->from = realloc(f->from, sizeof(int) * (f->nl + 1));
  f->to = realloc(f->to, sizeof(int) * (f->nl + 1));
  f->cap = realloc(f->cap, sizeof(double) * (f->nl + 1));
  f->from[f->nl] = a;
  f->to[f->nl] = b;
  f->cap[f->nl] = c;
  f->nl++;
}
static void fab_finish(fabric* f) { /* build_routes prep (topology.cpp:32-40) */
  f->oo = calloc(f->nn + 1, sizeof(int));
  f->io = calloc(f->nn + 1, sizeof(int));
  for (int l = 0; l < f->nl; ++l) {
    f->oo[f->from[l] + 1]++;
    f->io[f->to[l] + 1]++;
  }
  for (int u = 0; u < f->nn; ++u) {
    f->oo[u + 1] += f->oo[u];
    f->io[u + 1] += f->io[u];
  }
  f->ol = malloc(sizeof(int) * (f->nl + 1));
  f->il = malloc(sizeof(int) * (f->nl + 1));
  int* co = calloc(f->nn, sizeof(int));
  int* ci = calloc(f->nn, sizeof(int));
  for (int l = 0; l < f->nl; ++l) { /* ids ascending per node */
    f->ol[f->oo[f->from[l]] + co[f->from[l]]++] = l;
    f->il[f->io[f->to[l]] + ci[f->to[l]]++] = l;
  }
  free(co);
  free(ci);
  f->dist = calloc(f->nn, sizeof(int*));
}
static const int* fab_dist(fabric* f, int dst) { /* reverse BFS (topology.cpp:44-58) */
  if (f->dist[dst]) return f->dist[dst];
  int* d = malloc(sizeof(int) * f->nn);
  for (int i = 0; i < f->nn; ++i) d[i] = -1;
  int* q = malloc(sizeof(int) * f->nn);
  int qh = 0, qt = 0;
  d[dst] = 0;
  q[qt++] = dst;
  while (qh < qt) {
    int u = q[qh++];
    for (int e = f->io[u]; e < f->io[u + 1]; ++e) {
      int v = f->from[f->il[e]];
      if (d[v] < 0) {
        d[v] = d[u] + 1;
        q[qt++] = v;
      }
    }
  }
  free(q);
  f->dist[dst] = d;
  return d;
}
/* route src->dst into out (returns length; -1 unreachable) (topology.cpp:59-79) */
static int fab_route(fabric* f, int src, int dst, int* out) {
  if (src == dst) return 0;
  const int* d = fab_dist(f, dst);
  if (d[src] < 0) return -1;
  int n = 0;
  for (int u = src; u != dst;) {
    int pick = -1;
    for (int e = f->oo[u]; e < f->oo[u + 1]; ++e)
      if (d[f->to[f->ol[e]]] == d[u] - 1) {
        pick = f->ol[e];
        break;
      }
    out[n++] = pick;
    u = f->to[pick];
  }
  return n;
}
static void fab_free(fabric* f) {
  free(f->from);
  free(f->to);
  free(f->cap);
  free(f->oo);
  free(f->ol);
  free(f->io);
  free(f->il);
  if (f->dist)
    for (int i = 0; i < f->nn; ++i) free(f->dist[i]);
  free(f->dist);
}
static void fab_duplex(fabric* f, int a, int b, double c) {
  fab_add_link(f, a, b, c);
  fab_add_link(f, b, a, c);
}
static void fab_star(fabric* f, int hosts, double c) { /* topology.cpp:98-106 */
  for (int h = 0; h <= hosts; ++h) fab_add_node(f);
  for (int h = 0; h < hosts; ++h) fab_duplex(f, h, hosts, c);
  f->hosts = hosts;
}
static void fab_fattree(fabric* f, int hosts, double c, double os) { /* topology.cpp:108-145 */
  /* extension: switch-to-switch links carry c / os (os = topology.oversubscription) */
  double u = os == 1.0 ? c : c / os;
  int k = 2;
  while (k * k * k / 4 < hosts) k += 2;
  int half = k / 2;
  for (int h = 0; h < hosts; ++h) fab_add_node(f);
  int base = hosts;
  /* per pod: half edges then half aggs; then cores */
  int npod = k * 2 * half;
  for (int i = 0; i < npod + half * half; ++i) fab_add_node(f);
#define EDGE(p, j) (base + (p)*2 * half + (j))
#define AGG(p, j) (base + (p)*2 * half + half + (j))
#define CORE(c) (base + npod + (c))
  for (int h = 0; h < hosts; ++h) {
    int slot = h / half;
    fab_duplex(f, h, EDGE(slot / half, slot % half), c);
  }
  for (int p = 0; p < k; ++p)
    for (int e = 0; e < half; ++e)
      for (int a = 0; a < half; ++a) fab_duplex(f, EDGE(p, e), AGG(p, a), u);
  for (int p = 0; p < k; ++p)
    for (int a = 0; a < half; ++a)
      for (int cc = a * half; cc < (a + 1) * half; ++cc) fab_duplex(f, AGG(p, a), CORE(cc), u);
  f->hosts = hosts;
}

/* ---------------------------------------------------- workload (workload.cpp) */

typedef struct {
  uint64_t s;
} sm64;
static uint64_t sm_next(sm64* r) { /* workload.hpp:18-23 */
  uint64_t z = (r->s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static double sm_u(sm64* r) { return (double)(sm_next(r) >> 11) * (1.0 / 9007199254740992.0); }

typedef struct {
  double arrival, reuse, deadline;
  long tokens;
  int unit, src, layers;
} req_in;

typedef struct {
  int layers;
  double alpha, beta, kv, coll;
  int units, hpu, dhosts;
  double tick, horizon_slack;
  int has_horizon;
  double horizon;
  long maxtok, livelock;
  int policy; /* 0 fs 1 sjf 2 edf 3 karuna 4 mfs 5 aalo 6 varys (extensions) */
  int K;
  double thr[MAXK];
  int prune;
  double dfrac;
} params;

static int draft_cmp(const void* a, const void* b) {
  const req_in* x = a;
  const req_in* y = b;
  if (x->arrival != y->arrival) return x->arrival < y->arrival ? -1 : 1;
  return x->unit - y->unit;
}

/* generate_workload (workload.cpp:76-130) */
static req_in* synth(const kvcfg* c, const params* P, long* nout) {
  double rate = cfg_num(c, "workload.rate_rps", 1.0);
  long count = cfg_long(c, "workload.request_count", 100);
  double pmean = cfg_num(c, "workload.prompt_mean_tokens", 2000.0);
  double psig = cfg_num(c, "workload.prompt_sigma", 0.0);
  double rmean = cfg_num(c, "workload.reuse_fraction_mean", 0.5);
  double skew = cfg_num(c, "workload.reuse_skew", 1.0);
  uint64_t seed = (uint64_t)cfg_long(c, "sim.seed", 1);
  if (!(rate > 0) || count < 0 || rmean < 0 || rmean > 1) fail(2, "config: workload");
  long total = count * P->units;
  req_in* d = calloc(total ? total : 1, sizeof(req_in));
  long n = 0;
  for (int u = 0; u < P->units; ++u) {
    sm64 mix = {seed ^ (0x5851f42d4c957f2dULL * ((uint64_t)u + 1))};
    sm64 r = {sm_next(&mix)};
    double t = 0.0;
    for (long i = 0; i < count; ++i) {
      double uu = sm_u(&r);
      t += -log1p(-uu) / rate;
      double tok;
      if (psig <= 0.0) {
        tok = pmean;
      } else {
        double u1 = 1.0 - sm_u(&r);
        double u2 = sm_u(&r);
        double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
        double mu = log(pmean) - 0.5 * psig * psig;
        tok = exp(mu + psig * z);
      }
      long lt = llround(tok);
      if (lt < 1) lt = 1;
      if (lt > P->maxtok) lt = P->maxtok;
      double w = 0.15;
      if (rmean < w) w = rmean;
      if (1.0 - rmean < w) w = 1.0 - rmean;
      double rf = rmean + w * (2.0 * sm_u(&r) - 1.0);
      int src = -1;
      if (rf > 0.0 && P->units > 1) { /* Zipf (workload.cpp:52-68) */
        double tot = 0.0;
        for (int v = 0; v < P->units; ++v)
          if (v != u) tot += 1.0 / pow((double)(v + 1), skew);
        double x = sm_u(&r) * tot;
        for (int v = 0; v < P->units && src < 0; ++v) {
          if (v == u) continue;
          x -= 1.0 / pow((double)(v + 1), skew);
          if (x <= 0.0) src = v;
        }
        for (int v = P->units - 1; v >= 0 && src < 0; --v)
          if (v != u) src = v;
      }
      if (P->units <= 1) rf = 0.0;
      req_in q = {t, rf, INF, lt, u, src, P->layers};
      d[n++] = q;
    }
  }
  qsort(d, n, sizeof(req_in), draft_cmp);
  if (n > count) n = count;
  *nout = n;
  return d;
}

/* load_trace (workload.cpp:132-175) */
static req_in* trace(const char* path, const params* P, long* nout) {
  FILE* fp = fopen(path, "r");
  if (!fp) {
    fail(4, "cannot open trace file");
    *nout = 0;
    return NULL;
  }
  vec v = VEC(req_in);
  char line[1024];
  int no = 0;
  while (fgets(line, sizeof line, fp)) {
    ++no;
    size_t L = strlen(line);
    while (L && (line[L - 1] == '\n' || line[L - 1] == '\r')) line[--L] = 0;
    if (!L) continue;
    if (no == 1 && !strncmp(line, "arrival_s", 9)) continue;
    char* cells[8];
    int nc = 0;
    char* p = line;
    cells[nc++] = p;
    for (; *p; ++p)
      if (*p == ',') {
        *p = 0;
        if (nc < 8) cells[nc++] = p + 1;
      }
    if (nc != 4) {
      fail(3, "trace: expected 4 columns");
      break;
    }
    req_in q;
    q.arrival = strtod(cells[0], NULL);
    q.tokens = strtol(cells[1], NULL, 10);
    q.reuse = strtod(cells[2], NULL);
    q.src = *cells[3] ? atoi(cells[3]) : -1;
    q.unit = (int)(v.n % P->units);
    if (q.src == q.unit) q.src = (q.src + 1) % P->units;
    if (P->units <= 1) {
      q.reuse = 0.0;
      q.src = -1;
    }
    q.layers = P->layers;
    q.deadline = INF;
    vpush(&v, &q);
  }
  fclose(fp);
  *nout = v.n;
  return (req_in*)v.p;
}

/* ------------------------------------------------------ engine (engine.cpp) */

enum { SREUSE = 0, SCOLL = 1, SP2D = 2 };
enum { PEND = 0, ACT = 1, DONE = 2, PRUN = 3 };
enum { URG = 0, EARLY = 1, DEFR = 2, SCAV = 3 };
enum { KFLOW = 0, KCOMP, KDEP, KARR, KADM, KREL, KTICK };

typedef struct {
  int req, batch, cof, stage, tl, state;
  int route; /* index into route table, -1 empty, -2 unreachable */
  double size, rem, rel, dl; /* dl NaN = none */
  int has_dl, scripted;
  double relat;
  int band, level, rank;
  /* engine bookkeeping */
  double rate, fin;
  int gen, apos;
  double arate; /* rate in the last allocation, -1 = absent */
  int aidx;     /* insertion index in the last allocation */
} flow;

typedef struct {
  int nmem, moff; /* members in the member pool */
  double admit;
  int layers, lbase, unit;
  int departed, admitted;
  double done; /* pipeline done_t */
  int open, rank; /* rank -1 = absent */
  vec fl;           /* flows_by_batch, registration order */
} batch;

typedef struct {
  double cost;
  int started, done;
  double start, end;
  int coll;
  vec reuse, p2d; /* flow ids */
} layer;

typedef struct {
  int batch, layer, open;
  double rel, done;
  vec mem;
} coflow;

typedef struct {
  double t;
  int klass;
  uint64_t seq;
  int kind, a, b;
} event;

typedef struct {
  params P;
  fabric* F;
  /* routes */
  vec roff, rlinks; /* CSR */
  /* state */
  vec flows, batches, layers, cofs, mpool, fpool;
  req_in* rq;
  long nreq;
  int *r_batch, *r_pruned, *r_open, *r_rank;
  double *r_ttft, *r_last;
  /* units */
  int *q_head, *q_tail, *busy;
  int* qlist; /* per-unit FIFO lists */
  int* qoff;
  /* events */
  event* heap;
  long hn, hcap;
  uint64_t seq;
  double now;
  long events, steps, streak;
  int dirty;
  int workload;
  /* active */
  vec active;
  /* last allocation insertion order (flow ids) */
  vec aorder;
  /* aalo (extension): bytes of finished flows per (batch layer, stage) */
  vec att;
  double* asum; /* per-decide sums, valid where astamp == adecide */
  long* astamp;
  long acap, adecide;
  double horizon;
  long pruned_count;
} engine;

#define FL(e, i) (AT((e)->flows, flow, i))
#define BA(e, i) (AT((e)->batches, batch, i))
#define LY(e, b, l) (AT((e)->layers, layer, BA(e, b).lbase + (l)))
/* extension: Aalo coflow of a flow = (batch, target layer, stage); dense index */
static long aalo_idx(engine* e, const flow* f) { /* -1: no (batch, layer) coflow */
  if (f->batch < 0 || f->tl < 1 || f->tl > BA(e, f->batch).layers) return -1;
  return ((long)BA(e, f->batch).lbase + f->tl - 1) * 3 + f->stage;
}
#define CF(e, i) (AT((e)->cofs, coflow, i))

static int klass_of(int k) { return k <= KDEP ? 0 : (k == KTICK ? 2 : 1); }
static int ev_later(const event* x, const event* y) { /* EventLater (engine.hpp:182-188) */
  if (x->t != y->t) return x->t > y->t;
  if (x->klass != y->klass) return x->klass > y->klass;
  return x->seq > y->seq;
}
static void push(engine* e, double t, int kind, int a, int b) { /* engine.cpp:110-112 */
  if (e->hn == e->hcap) {
    e->hcap = e->hcap ? e->hcap * 2 : 64;
    e->heap = realloc(e->heap, sizeof(event) * e->hcap);
  }
  event v = {t, klass_of(kind), e->seq++, kind, a, b};
  long i = e->hn++;
  while (i > 0) {
    long p = (i - 1) / 2;
    if (!ev_later(&e->heap[p], &v)) break;
    e->heap[i] = e->heap[p];
    i = p;
  }
  e->heap[i] = v;
}
static event pop(engine* e) {
  event top = e->heap[0];
  event last = e->heap[--e->hn];
  long i = 0;
  for (;;) {
    long c = 2 * i + 1;
    if (c >= e->hn) break;
    if (c + 1 < e->hn && ev_later(&e->heap[c], &e->heap[c + 1])) ++c;
    if (!ev_later(&last, &e->heap[c])) break;
    e->heap[i] = e->heap[c];
    i = c;
  }
  if (e->hn) e->heap[i] = last;
  return top;
}

static int rlen(engine* e, int r) { return r < 0 ? 0 : AT(e->roff, int, r + 1) - AT(e->roff, int, r); }
static const int* rlinks(engine* e, int r) { return &AT(e->rlinks, int, AT(e->roff, int, r)); }
static int add_route(engine* e, int src, int dst) {
  int buf[256];
  int n = fab_route(e->F, src, dst, buf);
  if (n < 0) return -2;
  if (e->roff.n == 0) {
    int z = 0;
    vpush(&e->roff, &z);
  }
  for (int i = 0; i < n; ++i) vpush(&e->rlinks, &buf[i]);
  int end = (int)e->rlinks.n;
  vpush(&e->roff, &end);
  return (int)e->roff.n - 2;
}

static int reg_flow(engine* e, flow* f) { /* register_flow (engine.cpp:122-137) */
  f->fin = NOT;
  f->gen = 0;
  f->apos = -1;
  f->rate = 0.0;
  f->arate = -1.0;
  f->state = PEND;
  f->band = EARLY;
  f->level = 1;
  f->rank = 0;
  f->rel = NOT;
  f->rem = f->size;
  int id = (int)e->flows.n;
  vpush(&e->flows, f);
  if (f->req >= 0) e->r_open[f->req]++;
  if (f->batch >= 0) {
    vpush(&BA(e, f->batch).fl, &id);
    BA(e, f->batch).open++;
  }
  return id;
}

/* --------------------------------------------------------------- pipeline */

static int l_curr(engine* e, int b) { /* engine.cpp:712-720 */
  int L = BA(e, b).layers;
  for (int l = 1; l <= L; ++l) {
    layer* y = &LY(e, b, l - 1);
    if (!y->done) return l;
    if (y->coll >= 0 && CF(e, y->coll).open > 0) return l;
  }
  return L > 1 ? L : 1;
}
static double rem_compute(engine* e, int b) {
  double t = 0.0;
  for (int i = 0; i < BA(e, b).layers; ++i)
    if (!LY(e, b, i).done) t += LY(e, b, i).cost;
  return t;
}
static int drained(engine* e, int b) { return BA(e, b).done != NOT && BA(e, b).open == 0; }
static int deps_met(engine* e, int b, int layer_) { /* engine.cpp:356-369 */
  int idx = layer_ - 1;
  if (layer_ > 1) {
    layer* p = &LY(e, b, idx - 1);
    if (!p->done) return 0;
    if (p->coll >= 0 && CF(e, p->coll).open > 0) return 0;
  }
  layer* y = &LY(e, b, idx);
  for (long k = 0; k < y->reuse.n; ++k) {
    flow* f = &FL(e, AT(y->reuse, int, k));
    if (f->req >= 0 && e->r_pruned[f->req]) continue;
    if (f->state != DONE) return 0;
  }
  return 1;
}
static void start_layers(engine* e, int b) { /* engine.cpp:371-382 */
  for (int l = 1; l <= BA(e, b).layers; ++l) {
    layer* y = &LY(e, b, l - 1);
    if (y->started) continue;
    if (!deps_met(e, b, l)) return;
    y->started = 1;
    y->start = e->now;
    push(e, e->now + y->cost, KCOMP, b, l);
    return;
  }
}
static void pipe_done(engine* e, int b) { /* engine.cpp:384-393 */
  if (BA(e, b).done != NOT) return;
  for (int i = 0; i < BA(e, b).layers; ++i) {
    layer* y = &LY(e, b, i);
    if (!y->done) return;
    if (y->coll >= 0 && CF(e, y->coll).open > 0) return;
  }
  BA(e, b).done = e->now;
  push(e, e->now, KDEP, b, -1);
}
static void complete_req(engine* e, int r) { /* engine.cpp:585-593 */
  if (e->r_ttft[r] != NOT) return;
  int b = e->r_batch[r];
  if (b < 0 || BA(e, b).done == NOT) return;
  if (e->r_open[r] > 0) return;
  double t = BA(e, b).done;
  if (e->r_last[r] != NOT) t = dmax(t, e->r_last[r]);
  e->r_ttft[r] = t;
}

/* ---------------------------------------------------- allocator.cpp:28-126 */

typedef struct {
  int* ids;  /* flow ids, classes contiguous */
  int* start; /* class starts, ncls+1 */
  int n, ncls;
  double* caps; /* by flow id, NAN = none; NULL = no caps */
} classes;

static void allocate(engine* e, const classes* C) {
  double* res = malloc(sizeof(double) * (e->F->nl + 1));
  int* cnt = calloc(e->F->nl + 1, sizeof(int));
  for (int l = 0; l < e->F->nl; ++l) res[l] = e->F->cap[l];
  e->aorder.n = 0;
  for (int c = 0; c < C->ncls; ++c) {
    int o0 = C->start[c], n = C->start[c + 1] - o0;
    if (n == 1) {
      flow* f = &FL(e, C->ids[o0]);
      const int* rl = rlinks(e, f->route);
      int rn = rlen(e, f->route);
      double r = INF;
      if (C->caps && !isnan(C->caps[C->ids[o0]])) r = dmax(0.0, C->caps[C->ids[o0]]);
      for (int k = 0; k < rn; ++k) r = dmin(r, dmax(0.0, res[rl[k]]));
      for (int k = 0; k < rn; ++k) res[rl[k]] -= r;
      f->arate = r;
      f->aidx = (int)e->aorder.n;
      vpush(&e->aorder, &C->ids[o0]);
      continue;
    }
    double* rate = calloc(n, sizeof(double));
    char* frozen = calloc(n, 1);
    double* cap = malloc(sizeof(double) * n);
    for (int i = 0; i < n; ++i) {
      cap[i] = INF;
      if (C->caps && !isnan(C->caps[C->ids[o0 + i]])) cap[i] = dmax(0.0, C->caps[C->ids[o0 + i]]);
    }
    int* touched = malloc(sizeof(int) * (e->F->nl + 1));
    long guard = (long)n + e->F->nl + 2;
    while (guard-- > 0) {
      int nt = 0, any = 0;
      for (int i = 0; i < n; ++i) {
        if (frozen[i]) continue;
        any = 1;
        flow* f = &FL(e, C->ids[o0 + i]);
        const int* rl = rlinks(e, f->route);
        for (int k = 0; k < rlen(e, f->route); ++k) {
          if (cnt[rl[k]] == 0) touched[nt++] = rl[k];
          cnt[rl[k]]++;
        }
      }
      if (!any) break;
      double inc = INF;
      for (int j = 0; j < nt; ++j) inc = dmin(inc, dmax(0.0, res[touched[j]]) / cnt[touched[j]]);
      for (int i = 0; i < n; ++i)
        if (!frozen[i] && cap[i] < INF) inc = dmin(inc, cap[i] - rate[i]);
      inc = dmax(inc, 0.0);
      for (int i = 0; i < n; ++i)
        if (!frozen[i]) rate[i] += inc;
      for (int j = 0; j < nt; ++j) res[touched[j]] -= inc * cnt[touched[j]];
      int froze = 0;
      for (int i = 0; i < n; ++i) {
        if (frozen[i]) continue;
        double eps = 1e-12 * dmax(1.0, cap[i] == INF ? 0.0 : cap[i]);
        int stop = rate[i] >= cap[i] - eps;
        flow* f = &FL(e, C->ids[o0 + i]);
        const int* rl = rlinks(e, f->route);
        for (int k = 0; !stop && k < rlen(e, f->route); ++k)
          if (res[rl[k]] <= 1e-12 * e->F->cap[rl[k]]) stop = 1;
        if (stop) {
          frozen[i] = 1;
          froze = 1;
        }
      }
      for (int j = 0; j < nt; ++j) cnt[touched[j]] = 0;
      if (!froze) {
        fail(6, "allocate_rates: filling made no progress");
        break;
      }
    }
    for (int i = 0; i < n; ++i) {
      flow* f = &FL(e, C->ids[o0 + i]);
      f->arate = rate[i];
      f->aidx = (int)e->aorder.n;
      vpush(&e->aorder, &C->ids[o0 + i]);
    }
    free(rate);
    free(frozen);
    free(cap);
    free(touched);
  }
  free(res);
  free(cnt);
}

/* ------------------------------------------------ policies (baselines.cpp) */

static engine* g_sort_engine;
static int sjf_cmp(const void* a, const void* b) { /* baselines.cpp:25-30 */
  flow* x = &FL(g_sort_engine, *(const int*)a);
  flow* y = &FL(g_sort_engine, *(const int*)b);
  if (x->rem != y->rem) return x->rem < y->rem ? -1 : 1;
  if (x->rel != y->rel) return x->rel < y->rel ? -1 : 1;
  return *(const int*)a - *(const int*)b;
}
static int edf_cmp(const void* a, const void* b) { /* baselines.cpp:68-74 */
  flow* x = &FL(g_sort_engine, *(const int*)a);
  flow* y = &FL(g_sort_engine, *(const int*)b);
  if (x->dl != y->dl) return x->dl < y->dl ? -1 : 1;
  if (x->rel != y->rel) return x->rel < y->rel ? -1 : 1;
  return *(const int*)a - *(const int*)b;
}

typedef struct {
  int id, band;
  double k1, k2, k3;
} mkey;
static int mfs_cmp(const void* a, const void* b) { /* rmlq.cpp:241-247 */
  const mkey* x = a;
  const mkey* y = b;
  if (x->band != y->band) return x->band < y->band ? -1 : 1;
  if (x->k1 != y->k1) return x->k1 < y->k1 ? -1 : 1;
  if (x->k2 != y->k2) return x->k2 < y->k2 ? -1 : 1;
  if (x->k3 != y->k3) return x->k3 < y->k3 ? -1 : 1;
  return x->id - y->id;
}

static void add_class(classes* C) { C->start[C->ncls++] = C->n; }

static void decide(engine* e, classes* C) {
  int A = (int)e->active.n;
  C->ids = malloc(sizeof(int) * (A + 1));
  C->start = malloc(sizeof(int) * (A + 2));
  C->n = 0;
  C->ncls = 0;
  C->caps = NULL;
  int* act = (int*)e->active.p;
  g_sort_engine = e;
  if (e->P.policy == 0) { /* fs */
    if (A) add_class(C);
    for (int i = 0; i < A; ++i) C->ids[C->n++] = act[i];
  } else if (e->P.policy == 1 || e->P.policy == 3) { /* sjf / karuna */
    int* rest = malloc(sizeof(int) * (A + 1));
    int nr = 0;
    if (e->P.policy == 3) {
      int nd = 0;
      int* dl = malloc(sizeof(int) * (A + 1));
      for (int i = 0; i < A; ++i)
        if (FL(e, act[i]).has_dl) dl[nd++] = act[i];
        else rest[nr++] = act[i];
      if (nd) { /* karuna caps (baselines.cpp:102-133) */
        C->caps = malloc(sizeof(double) * e->flows.n);
        for (long i = 0; i < e->flows.n; ++i) C->caps[i] = NAN;
        double* want = malloc(sizeof(double) * e->flows.n);
        char* has = calloc(e->flows.n, 1);
        double* dem = calloc(e->F->nl + 1, sizeof(double));
        for (int i = 0; i < nd; ++i) {
          flow* f = &FL(e, dl[i]);
          double slack = f->dl - e->now;
          if (slack > 0.0) {
            want[dl[i]] = f->rem / slack;
            has[dl[i]] = 1;
          }
        }
        for (int i = 0; i < nd; ++i) {
          if (!has[dl[i]]) continue;
          flow* f = &FL(e, dl[i]);
          const int* rl = rlinks(e, f->route);
          for (int k = 0; k < rlen(e, f->route); ++k) dem[rl[k]] += want[dl[i]];
        }
        for (int i = 0; i < nd; ++i) {
          if (!has[dl[i]]) continue;
          flow* f = &FL(e, dl[i]);
          double scale = 1.0;
          const int* rl = rlinks(e, f->route);
          for (int k = 0; k < rlen(e, f->route); ++k) {
            double c = e->F->cap[rl[k]];
            if (dem[rl[k]] > c) scale = dmin(scale, c / dem[rl[k]]);
          }
          C->caps[dl[i]] = want[dl[i]] * scale;
        }
        free(want);
        free(has);
        free(dem);
        add_class(C);
        for (int i = 0; i < nd; ++i) C->ids[C->n++] = dl[i];
      }
      free(dl);
    } else {
      for (int i = 0; i < A; ++i) rest[nr++] = act[i];
    }
    qsort(rest, nr, sizeof(int), sjf_cmp); /* sjf_classes (baselines.cpp:23-44) */
    for (int i = 0; i < nr; ++i) {
      if (i == 0 || FL(e, rest[i]).rem != FL(e, rest[i - 1]).rem ||
          FL(e, rest[i]).rel != FL(e, rest[i - 1]).rel)
        add_class(C);
      C->ids[C->n++] = rest[i];
    }
    free(rest);
  } else if (e->P.policy == 2) { /* edf */
    int* ex = malloc(sizeof(int) * (A + 1));
    int* im = malloc(sizeof(int) * (A + 1));
    int ne = 0, ni = 0;
    for (int i = 0; i < A; ++i)
      if (FL(e, act[i]).has_dl) ex[ne++] = act[i];
      else im[ni++] = act[i];
    qsort(ex, ne, sizeof(int), edf_cmp);
    for (int i = 0; i < ne; ++i) {
      if (i == 0 || FL(e, ex[i]).dl != FL(e, ex[i - 1]).dl ||
          FL(e, ex[i]).rel != FL(e, ex[i - 1]).rel)
        add_class(C);
      C->ids[C->n++] = ex[i];
    }
    if (ni) {
      add_class(C);
      for (int i = 0; i < ni; ++i) C->ids[C->n++] = im[i];
    }
    free(ex);
    free(im);
  } else if (e->P.policy == 5) {
    /* extension -- Aalo-style D-CLAS coflow scheduling (no reference oracle):
     * coflow c = (batch, target layer, stage); attained service
     * a_c = D_c + sum over c's transferable flows, in active order, of
     * (size - remaining), D_c = sizes of c's finished flows added in completion
     * order; queue q_c = #{i : a_c >= Q0 * E^i, i < K-1}; one class per coflow,
     * ordered by (q_c, coflow index = batch-major FIFO); a flow without a
     * (batch, layer) -- no batch, or a target layer outside the batch's layers
     * (manual scenarios) -- is its own coflow after every batch coflow of its
     * queue, by flow id. */
    if (e->acap < (long)e->att.n) {
      e->acap = (long)e->att.n * 2 + 64;
      e->asum = realloc(e->asum, sizeof(double) * e->acap);
      e->astamp = realloc(e->astamp, sizeof(long) * e->acap);
      memset(e->astamp, 0, sizeof(long) * e->acap);
      e->adecide = 0;
    }
    long st = ++e->adecide;
    mkey* k = malloc(sizeof(mkey) * (A + 1));
    double* own = malloc(sizeof(double) * (A + 1));
    for (int i = 0; i < A; ++i) {
      flow* f = &FL(e, act[i]);
      double v = f->size - f->rem;
      long c = aalo_idx(e, f);
      if (c >= 0) {
        if (e->astamp[c] != st) {
          e->astamp[c] = st;
          e->asum[c] = AT(e->att, double, c);
        }
        e->asum[c] += v;
      } else {
        own[i] = v;
      }
    }
    for (int i = 0; i < A; ++i) {
      flow* f = &FL(e, act[i]);
      long c = aalo_idx(e, f);
      double a = c >= 0 ? e->asum[c] : own[i];
      int q = 0;
      while (q < e->P.K - 1 && a >= e->P.thr[q]) ++q;
      mkey m = {act[i], q, c >= 0 ? (double)c : 0x1p40 + act[i], 0.0, 0.0};
      k[i] = m;
    }
    free(own);
    qsort(k, A, sizeof(mkey), mfs_cmp);
    for (int i = 0; i < A; ++i) {
      if (i == 0 || k[i].band != k[i - 1].band || k[i].k1 != k[i - 1].k1) add_class(C);
      C->ids[C->n++] = k[i].id;
    }
    free(k);
  } else if (e->P.policy == 6) {
    /* extension -- Varys-style SEBF + MADD coflow scheduling (no reference
     * oracle; clairvoyant: it reads the remaining bytes). Coflow c as in Aalo
     * (batch, target layer, stage; a flow without one is its own coflow).
     * Effective bottleneck Gamma_c = max over links l of L_cl / capacity_l,
     * L_cl = remaining bytes of c's active flows routed over l, summed in
     * active order. One class per coflow, ordered by (Gamma_c, coflow key);
     * MADD caps every member at remaining / Gamma_c (uncapped when Gamma_c is
     * 0) so that, bandwidth permitting, a coflow's flows finish together;
     * no backfilling beyond what the filling gives the lower classes. */
    mkey* k = malloc(sizeof(mkey) * (A + 1));
    for (int i = 0; i < A; ++i) {
      flow* f = &FL(e, act[i]);
      long c = aalo_idx(e, f);
      mkey m = {i, 0, c >= 0 ? (double)c : 0x1p40 + act[i], (double)i, 0.0};
      k[i] = m;
    }
    qsort(k, A, sizeof(mkey), mfs_cmp); /* members of a coflow, in active order */
    double* L = calloc(e->F->nl + 1, sizeof(double));
    double* gam = malloc(sizeof(double) * (A + 1));
    for (int g0 = 0; g0 < A;) {
      int g1 = g0 + 1;
      while (g1 < A && k[g1].k1 == k[g0].k1) ++g1;
      for (int i = g0; i < g1; ++i) {
        flow* f = &FL(e, act[k[i].id]);
        const int* rl = rlinks(e, f->route);
        for (int q = 0; q < rlen(e, f->route); ++q) L[rl[q]] += f->rem;
      }
      double gmax = 0.0;
      for (int i = g0; i < g1; ++i) {
        flow* f = &FL(e, act[k[i].id]);
        const int* rl = rlinks(e, f->route);
        for (int q = 0; q < rlen(e, f->route); ++q) gmax = dmax(gmax, L[rl[q]] / e->F->cap[rl[q]]);
      }
      for (int i = g0; i < g1; ++i) {
        flow* f = &FL(e, act[k[i].id]);
        const int* rl = rlinks(e, f->route);
        for (int q = 0; q < rlen(e, f->route); ++q) L[rl[q]] = 0.0;
        gam[k[i].id] = gmax;
      }
      g0 = g1;
    }
    free(L);
    C->caps = malloc(sizeof(double) * e->flows.n);
    for (long i = 0; i < e->flows.n; ++i) C->caps[i] = NAN;
    for (int i = 0; i < A; ++i) {
      flow* f = &FL(e, act[i]);
      long c = aalo_idx(e, f);
      mkey m = {act[i], 0, gam[i], c >= 0 ? (double)c : 0x1p40 + act[i], 0.0};
      k[i] = m;
      if (gam[i] > 0.0) C->caps[act[i]] = f->rem / gam[i];
    }
    free(gam);
    qsort(k, A, sizeof(mkey), mfs_cmp);
    for (int i = 0; i < A; ++i) {
      if (i == 0 || k[i].k1 != k[i - 1].k1 || k[i].k2 != k[i - 1].k2) add_class(C);
      C->ids[C->n++] = k[i].id;
    }
    free(k);
  } else { /* mfs arbitrate (rmlq.cpp:201-260) */
    mkey* k = malloc(sizeof(mkey) * (A + 1));
    for (int i = 0; i < A; ++i) {
      flow* f = &FL(e, act[i]);
      double d = f->has_dl ? f->dl : (f->req >= 0 ? e->rq[f->req].deadline : INF);
      mkey m = {act[i], f->band, 0.0, 0.0, 0.0};
      if (f->band == URG || f->band == DEFR) {
        m.k1 = f->level;
        m.k2 = d;
      } else if (f->band == EARLY) {
        m.k1 = f->level;
        m.k2 = f->rank;
        m.k3 = f->rel;
      } else {
        m.k1 = d;
      }
      k[i] = m;
    }
    qsort(k, A, sizeof(mkey), mfs_cmp);
    for (int i = 0; i < A; ++i) {
      if (i == 0 || k[i].band != k[i - 1].band || k[i].k1 != k[i - 1].k1 || k[i].k2 != k[i - 1].k2 ||
          k[i].k3 != k[i - 1].k3)
        add_class(C);
      C->ids[C->n++] = k[i].id;
    }
    free(k);
  }
  C->start[C->ncls] = C->n;
}

/* ------------------------------------------------------------ RMLQ (rmlq.cpp) */

static int outranks(int b1, int l1, int b2, int l2) { /* types.cpp:41-44 */
  if (b1 != b2) return b1 < b2;
  return l1 < l2;
}

/* iteration order of the last allocation's std::unordered_map<FlowId,double>
 * (libstdc++: nodes prepended per bucket, new buckets at the list head,
 * prime rehash schedule measured for single insertions from empty) */
static const int RH_AT[] = {0,     13,     29,     59,     127,    257,    541,
                            1109,  2357,   5087,   10273,  20753,  42043,  85229,
                            172933, 351061, 712697, 1447153, 2938679};
static const int RH_BK[] = {13,    29,     59,     127,    257,    541,     1109,
                            2357,  5087,   10273,  20753,  42043,  85229,   172933,
                            351061, 712697, 1447153, 2938679, 5967347};
static int* hash_rank(engine* e) {
  int n = (int)e->aorder.n;
  int* keys = (int*)e->aorder.p;
  int* next = malloc(sizeof(int) * (n + 1));
  int* rank = malloc(sizeof(int) * (n + 1));
  int* anchor = NULL;
  int head = -1, bc = 1, st = 0;
  for (int i = 0; i < n; ++i) {
    if (st < 19 && i == RH_AT[st]) {
      int nbc = RH_BK[st++];
      int* na = malloc(sizeof(int) * nbc);
      for (int b = 0; b < nbc; ++b) na[b] = -2;
      int p = head, bb = -1;
      head = -1;
      while (p != -1) {
        int nx = next[p], b = keys[p] % nbc;
        if (na[b] == -2) {
          next[p] = head;
          head = p;
          na[b] = -1;
          if (next[p] != -1) na[bb] = p;
          bb = b;
        } else if (na[b] == -1) {
          next[p] = head;
          head = p;
        } else {
          next[p] = next[na[b]];
          next[na[b]] = p;
        }
        p = nx;
      }
      free(anchor);
      anchor = na;
      bc = nbc;
    }
    int b = keys[i] % bc;
    if (anchor[b] != -2) {
      if (anchor[b] == -1) {
        next[i] = head;
        head = i;
      } else {
        next[i] = next[anchor[b]];
        next[anchor[b]] = i;
      }
    } else {
      next[i] = head;
      head = i;
      if (next[i] != -1) anchor[keys[next[i]] % bc] = i;
      anchor[b] = -1;
    }
  }
  int r = 0;
  for (int p = head; p != -1; p = next[p]) rank[p] = r++;
  free(next);
  free(anchor);
  return rank;
}

static int route_has(engine* e, int route, int l) {
  const int* rl = rlinks(e, route);
  for (int k = 0; k < rlen(e, route); ++k)
    if (rl[k] == l) return 1;
  return 0;
}

typedef struct {
  int r;
  double v;
} rv;
static int rv_cmp(const void* a, const void* b) { return ((const rv*)a)->r - ((const rv*)b)->r; }

/* load_fraction (allocator.cpp:128-141), summed in hash-map iteration order */
static double load_fraction(engine* e, int l, int band, int level) {
  int n = (int)e->aorder.n;
  rv* c = malloc(sizeof(rv) * (n + 1));
  int nc = 0;
  int* rank = NULL;
  for (int i = 0; i < n; ++i) {
    int fid = AT(e->aorder, int, i);
    flow* f = &FL(e, fid);
    double r = f->arate;
    if (r <= 0.0) continue;
    if (!(f->state == ACT || f->state == PRUN)) continue;
    if (!outranks(f->band, f->level, band, level)) continue;
    if (!route_has(e, f->route, l)) continue;
    c[nc].r = i;
    c[nc].v = r;
    nc++;
  }
  if (nc > 2) {
    rank = hash_rank(e);
    for (int i = 0; i < nc; ++i) c[i].r = rank[c[i].r];
    qsort(c, nc, sizeof(rv), rv_cmp);
    free(rank);
  }
  double used = 0.0;
  for (int i = 0; i < nc; ++i) used += c[i].v;
  free(c);
  double v = used / e->F->cap[l];
  return v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
}

/* LinkLoadIndex snapshot (allocator.cpp:143-171) */
typedef struct {
  int key, route;
  double rate;
} ixe;
typedef struct {
  ixe* v;
  int n;
} lindex;
static lindex idx_build(engine* e) {
  lindex X;
  X.v = malloc(sizeof(ixe) * (e->aorder.n + 1));
  X.n = 0;
  for (long i = 0; i < e->aorder.n; ++i) {
    flow* f = &FL(e, AT(e->aorder, int, i));
    if (f->arate <= 0.0 || !(f->state == ACT || f->state == PRUN)) continue;
    ixe x = {(f->band << 16) | f->level, f->route, f->arate};
    X.v[X.n++] = x;
  }
  return X;
}
typedef struct {
  int k;
  double r;
} kr;
static int kr_cmp(const void* a, const void* b) {
  const kr* x = a;
  const kr* y = b;
  if (x->k != y->k) return x->k < y->k ? -1 : 1;
  if (x->r != y->r) return x->r < y->r ? -1 : 1;
  return 0;
}
static double idx_query(engine* e, const lindex* X, int l, int band, int level) {
  int q = (band << 16) | level;
  kr* c = malloc(sizeof(kr) * (X->n + 1));
  int nc = 0;
  for (int i = 0; i < X->n; ++i)
    if (route_has(e, X->v[i].route, l)) {
      c[nc].k = X->v[i].key;
      c[nc].r = X->v[i].rate;
      nc++;
    }
  qsort(c, nc, sizeof(kr), kr_cmp);
  double run = 0.0;
  int any = 0;
  for (int i = 0; i < nc && c[i].k < q; ++i) {
    run += c[i].r;
    any = 1;
  }
  free(c);
  if (!any) return 0.0;
  double v = run / e->F->cap[l];
  return v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
}

/* natural_key (rmlq.cpp:101-127); X = NULL: load_fraction */
static void natural(engine* e, int fid, const lindex* X, int* ob, int* ol) {
  flow* f = &FL(e, fid);
  int lc = f->batch >= 0 ? l_curr(e, f->batch) : 1;
  if (f->stage != SP2D) {
    int v = f->tl - lc;
    if (v < 0) v = 0;
    if (v > e->P.K - 1) v = e->P.K - 1;
    *ob = EARLY;
    *ol = v + 1;
    return;
  }
  int pb = f->band, pl = f->level;
  if (pb == EARLY) {
    pb = DEFR;
    pl = e->P.K;
  }
  double size_rem = f->rem, time_rem = f->dl - e->now, value;
  int rn = rlen(e, f->route);
  if (f->route == -2) fail(5, "no route");
  if (rn == 0) {
    value = 0.0;
  } else {
    double best = INF;
    const int* rl = rlinks(e, f->route);
    for (int k = 0; k < rn; ++k) {
      double rho = X ? idx_query(e, X, rl[k], pb, pl) : load_fraction(e, rl[k], pb, pl);
      double eff = e->F->cap[rl[k]] * (1.0 - rho);
      if (eff < best) best = eff;
    }
    if (size_rem <= 0.0) value = 0.0;
    else if (time_rem <= 0.0) value = INF;
    else if (best <= 0.0) value = INF;
    else value = size_rem / (time_rem * best);
  }
  if (!(value >= 0.0)) fail(6, "mlu_to_level: negative urgency");
  int lv = e->P.K;
  for (int i = 1; i <= e->P.K - 1; ++i)
    if (value >= e->P.thr[i - 1]) {
      lv = i;
      break;
    }
  *ol = lv;
  *ob = lv == 1 ? URG : DEFR;
}
static int rank_of(engine* e, int fid) { /* rmlq.cpp:89-99 */
  flow* f = &FL(e, fid);
  if (f->req >= 0 && e->r_rank[f->req] >= 0) return e->r_rank[f->req];
  if (f->batch >= 0 && BA(e, f->batch).rank >= 0) return BA(e, f->batch).rank;
  return 0;
}
static void on_released(engine* e, int fid) { /* rmlq.cpp:137-148 */
  if (e->P.policy != 4) return;
  flow* f = &FL(e, fid);
  if (f->req >= 0 && e->r_pruned[f->req]) {
    f->band = SCAV;
    f->level = e->P.K;
    return;
  }
  int b, l;
  natural(e, fid, NULL, &b, &l);
  f = &FL(e, fid);
  f->band = b;
  f->level = l;
  f->rank = rank_of(e, fid);
  if (b == URG && f->stage != SP2D) fail(6, "urgent band is reserved for last-stage flows");
}
static int promote_batch(engine* e, int b, int p2d_only) { /* rmlq.cpp:150-193 */
  lindex X = idx_build(e);
  int changed = 0;
  batch* B = &BA(e, b);
  for (long i = 0; i < B->fl.n; ++i) {
    int fid = AT(B->fl, int, i);
    flow* f = &FL(e, fid);
    if (f->state == DONE || f->state == PRUN) continue;
    if (p2d_only && f->stage != SP2D) continue;
    if (f->band == SCAV) continue;
    int nb, nl;
    natural(e, fid, &X, &nb, &nl);
    f = &FL(e, fid);
    if (!outranks(nb, nl, f->band, f->level)) continue;
    f->band = nb;
    f->level = nl;
    changed = 1;
  }
  free(X.v);
  return changed;
}
static void layer_boundary(engine* e, int b) {
  if (e->P.policy == 4) promote_batch(e, b, 0);
}

/* ------------------------------------------ Algorithm 1 (inter_request.cpp) */

typedef struct {
  int id;
  double dl;
  double* load; /* dense per link */
} ireq;
typedef struct {
  int id;
  double admit, comp, red, dlo;
  ireq* r;
  int nr;
} ibatch;

static int dbl_cmp(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}
static void red_score(ibatch* B) { /* inter_request.cpp:7-43 */
  double* d = malloc(sizeof(double) * B->nr);
  for (int i = 0; i < B->nr; ++i) d[i] = B->r[i].dl;
  qsort(d, B->nr, sizeof(double), dbl_cmp);
  int n = B->nr;
  if (n == 1 || d[0] == d[n - 1]) {
    B->red = d[0];
    B->dlo = d[0];
  } else {
    int ks = 1;
    double best = d[1] - d[0];
    for (int k = 2; k < n; ++k)
      if (d[k] - d[k - 1] > best) {
        best = d[k] - d[k - 1];
        ks = k;
      }
    double f = (double)ks / (double)n;
    B->dlo = d[ks];
    B->red = f * d[0] + (1.0 - f) * d[ks];
  }
  free(d);
}
static int ib_cmp(const void* a, const void* b) { /* inter_request.cpp:113-117 */
  const ibatch* x = a;
  const ibatch* y = b;
  if (x->red != y->red) return x->red < y->red ? -1 : 1;
  if (x->admit != y->admit) return x->admit < y->admit ? -1 : 1;
  return x->id - y->id;
}
static double est_finish(engine* e, double comp, const double* S, const double* L, int* ustar) {
  double worst = 0.0;
  int inf = 0;
  *ustar = 0;
  for (int u = 0; u < e->F->nl; ++u) { /* inter_request.cpp:53-78 */
    double tot = S[u] + L[u], ratio = tot / e->F->cap[u];
    if (ratio > worst) {
      worst = ratio;
      *ustar = u;
      inf = (ratio == INF);
    }
  }
  return inf ? INF : e->now + comp + worst;
}
static int int_cmp(const void* a, const void* b) { return *(const int*)a - *(const int*)b; }

/* on_batch_event (rmlq.cpp:268-382); returns newly pruned ids (ascending) */
static int batch_event(engine* e, int* out) {
  int NL = e->F->nl, nb = 0;
  long NB = e->batches.n;
  ibatch* in = calloc(NB + 1, sizeof(ibatch));
  double* toks = calloc(NB + 1, sizeof(double));
  char* active = calloc(NB + 1, 1);
  for (long b = 0; b < NB; ++b) active[b] = !drained(e, (int)b);
  for (long b = 0; b < NB; ++b) {
    if (!active[b]) continue;
    batch* B = &BA(e, b);
    for (int k = 0; k < B->nmem; ++k) {
      int r = AT(e->mpool, int, B->moff + k);
      if (!e->r_pruned[r]) toks[b] += (double)e->rq[r].tokens;
    }
  }
  /* per-request dense loads, fold order: batches by id, flows by id */
  double** load = calloc(e->nreq + 1, sizeof(double*));
  for (long b = 0; b < NB; ++b) {
    if (!active[b]) continue;
    batch* B = &BA(e, b);
    for (long i = 0; i < B->fl.n; ++i) {
      flow* f = &FL(e, AT(B->fl, int, i));
      if (f->state == DONE || f->rem <= 0.0) continue;
      if (f->route < 0 || rlen(e, f->route) == 0) continue;
      const int* rl = rlinks(e, f->route);
      if (f->stage == SCOLL) {
        if (toks[b] <= 0.0) continue;
        for (int k = 0; k < B->nmem; ++k) {
          int r = AT(e->mpool, int, B->moff + k);
          if (e->r_pruned[r]) continue;
          double share = f->rem * (double)e->rq[r].tokens / toks[b];
          if (!load[r]) load[r] = calloc(NL, sizeof(double));
          for (int j = 0; j < rlen(e, f->route); ++j) load[r][rl[j]] += share;
        }
      } else if (f->req >= 0 && !e->r_pruned[f->req]) {
        if (!load[f->req]) load[f->req] = calloc(NL, sizeof(double));
        for (int j = 0; j < rlen(e, f->route); ++j) load[f->req][rl[j]] += f->rem;
      }
    }
  }
  long inflight = 0;
  for (long b = 0; b < NB; ++b) {
    if (!active[b]) continue;
    batch* B = &BA(e, b);
    ibatch ib = {(int)b, B->admit, rem_compute(e, (int)b), 0, 0, NULL, 0};
    ib.r = calloc(B->nmem + 1, sizeof(ireq));
    for (int k = 0; k < B->nmem; ++k) {
      int r = AT(e->mpool, int, B->moff + k);
      if (e->r_pruned[r]) continue;
      if (!load[r]) load[r] = calloc(NL, sizeof(double));
      ireq q = {r, e->rq[r].deadline, load[r]};
      ib.r[ib.nr++] = q;
      inflight++;
    }
    if (ib.nr) in[nb++] = ib;
    else free(ib.r);
  }
  int np = 0;
  if (nb) {
    long budget = e->P.prune ? (long)ceil(e->P.dfrac * (double)inflight) : 0;
    if (budget < 0) budget = 0;
    for (int i = 0; i < nb; ++i) red_score(&in[i]);
    qsort(in, nb, sizeof(ibatch), ib_cmp); /* ids unique: a total order */
    double* S = calloc(NL, sizeof(double));
    double* L = calloc(NL, sizeof(double));
    typedef struct {
      int id, pos;
      double* load;
    } pe;
    pe* pool = malloc(sizeof(pe) * (inflight + 1));
    int npool = 0;
    for (int k = 0; k < nb; ++k) {
      memset(L, 0, sizeof(double) * NL);
      for (int i = 0; i < in[k].nr; ++i) {
        pe x = {in[k].r[i].id, k, in[k].r[i].load};
        pool[npool++] = x;
        for (int u = 0; u < NL; ++u) L[u] += in[k].r[i].load[u];
      }
      int us;
      double fh = est_finish(e, in[k].comp, S, L, &us);
      while (fh > in[k].dlo && np < budget && npool > 0) {
        int v = npool;
        double vl = 0.0;
        for (int i = 0; i < npool; ++i) {
          double l = pool[i].load[us];
          if (l <= 0.0) continue;
          if (v == npool || l > vl || (l == vl && pool[i].id < pool[v].id)) {
            v = i;
            vl = l;
          }
        }
        if (v == npool) break;
        pe vic = pool[v];
        memmove(pool + v, pool + v + 1, sizeof(pe) * (npool - v - 1));
        npool--;
        out[np++] = vic.id;
        double* t = vic.pos == k ? L : S;
        for (int u = 0; u < NL; ++u) t[u] = dmax(0.0, t[u] - vic.load[u]);
        fh = est_finish(e, in[k].comp, S, L, &us);
      }
      for (int u = 0; u < NL; ++u) S[u] += L[u];
    }
    qsort(out, np, sizeof(int), int_cmp);
    for (int k = 0; k < nb; ++k) { /* ranks from sigma */
      batch* B = &BA(e, in[k].id);
      B->rank = k + 1;
      for (int m = 0; m < B->nmem; ++m) e->r_rank[AT(e->mpool, int, B->moff + m)] = k + 1;
    }
    for (long b = 0; b < NB; ++b) { /* rerank */
      if (!active[b]) continue;
      batch* B = &BA(e, b);
      for (long i = 0; i < B->fl.n; ++i) {
        int fid = AT(B->fl, int, i);
        if (FL(e, fid).state != DONE) FL(e, fid).rank = rank_of(e, fid);
      }
    }
    free(S);
    free(L);
    free(pool);
  }
  for (int i = 0; i < nb; ++i) free(in[i].r);
  for (long r = 0; r < e->nreq; ++r) free(load[r]);
  free(load);
  free(in);
  free(toks);
  free(active);
  return np;
}

/* --------------------------------------------------- handlers (engine.cpp) */

static void remove_active(engine* e, int fid) { /* engine.cpp:251-259 */
  int pos = FL(e, fid).apos;
  if (pos < 0) return;
  int last = AT(e->active, int, e->active.n - 1);
  AT(e->active, int, pos) = last;
  FL(e, last).apos = pos;
  e->active.n--;
  FL(e, fid).apos = -1;
}
static void finish_flow(engine* e, int fid);
static void release_flow(engine* e, int fid) { /* engine.cpp:295-316 */
  flow* f = &FL(e, fid);
  if (f->state != PEND) {
    fail(6, "flow released twice");
    return;
  }
  f->rel = e->now;
  int pr = f->req >= 0 && e->r_pruned[f->req];
  f->state = pr ? PRUN : ACT;
  on_released(e, fid);
  f = &FL(e, fid);
  if (f->cof >= 0 && CF(e, f->cof).rel == NOT) CF(e, f->cof).rel = e->now;
  if (f->size > 0.0 && f->route == -2) {
    fail(5, "no route");
    return;
  }
  if (f->size <= 0.0 || rlen(e, f->route) == 0) {
    finish_flow(e, fid);
    return;
  }
  f->apos = (int)e->active.n;
  vpush(&e->active, &fid);
  f->rate = 0.0;
  e->dirty = 1;
}
static void finish_flow(engine* e, int fid) { /* engine.cpp:318-354 */
  flow* f = &FL(e, fid);
  if (f->state == DONE) {
    fail(6, "flow finished twice");
    return;
  }
  if (f->apos >= 0 && !(f->rem <= 1e-6 * dmax(f->size, 1.0) + 1e-9)) {
    fail(6, "flow completed before its bytes were transferred");
    return;
  }
  f->rem = 0.0;
  f->state = DONE;
  f->fin = e->now;
  if (e->P.policy == 5 && aalo_idx(e, f) >= 0) AT(e->att, double, aalo_idx(e, f)) += f->size;
  remove_active(e, fid);
  f = &FL(e, fid);
  f->rate = 0.0;
  f->gen++;
  e->dirty = 1;
  if (f->batch >= 0) BA(e, f->batch).open--;
  if (f->cof >= 0) {
    coflow* c = &CF(e, f->cof);
    if (!(c->open > 0)) {
      fail(6, "coflow member finished after barrier");
      return;
    }
    if (--c->open == 0) {
      c->done = e->now;
      int cb = c->batch;
      layer_boundary(e, cb);
      start_layers(e, cb);
      pipe_done(e, cb);
    }
  }
  f = &FL(e, fid);
  if (f->req >= 0) {
    e->r_open[f->req]--;
    e->r_last[f->req] = dmax(e->r_last[f->req], e->now);
    if (f->stage == SREUSE && f->batch >= 0) {
      start_layers(e, f->batch);
      pipe_done(e, f->batch);
    }
    complete_req(e, f->req);
  }
}
static void apply_prunes(engine* e, int* ids, int n) { /* engine.cpp:565-583 */
  for (int i = 0; i < n; ++i) {
    int r = ids[i];
    e->r_pruned[r] = 1;
    int b = e->r_batch[r];
    if (b < 0) continue;
    batch* B = &BA(e, b);
    for (long j = 0; j < B->fl.n; ++j) {
      flow* f = &FL(e, AT(B->fl, int, j));
      if (f->req != r || f->state == DONE) continue;
      f->band = SCAV;
      if (f->state == ACT) f->state = PRUN;
    }
    start_layers(e, b);
    pipe_done(e, b);
  }
  if (n) e->dirty = 1;
  e->pruned_count += n;
}
static void batch_hook(engine* e) { /* engine.cpp:560-563 */
  if (e->P.policy != 4) return;
  int* ids = malloc(sizeof(int) * (e->nreq + 1));
  int n = batch_event(e, ids);
  apply_prunes(e, ids, n);
  free(ids);
}
static int new_batch(engine* e, int nmem, int moff, double admit, int nl) {
  batch B;
  memset(&B, 0, sizeof B);
  B.nmem = nmem;
  B.moff = moff;
  B.admit = admit;
  B.layers = nl;
  B.lbase = (int)e->layers.n;
  B.done = NOT;
  B.rank = -1;
  B.fl.es = sizeof(int);
  int b = (int)e->batches.n;
  vpush(&e->batches, &B);
  for (int l = 0; l < nl; ++l) {
    layer y;
    memset(&y, 0, sizeof y);
    y.start = y.end = NOT;
    y.coll = -1;
    y.reuse.es = y.p2d.es = sizeof(int);
    vpush(&e->layers, &y);
    double z = 0.0;
    for (int k = 0; k < 3; ++k) vpush(&e->att, &z);
  }
  return b;
}
static void admit_batch(engine* e, int unit, int moff, int nmem) { /* engine.cpp:455-533 */
  int b = new_batch(e, nmem, moff, e->now, e->P.layers);
  double bt = 0.0;
  for (int k = 0; k < nmem; ++k) {
    int r = AT(e->mpool, int, moff + k);
    e->r_batch[r] = b;
    bt += (double)e->rq[r].tokens;
  }
  BA(e, b).unit = unit;
  for (int l = 0; l < e->P.layers; ++l) LY(e, b, l).cost = e->P.alpha + e->P.beta * bt;
  vec rel = VEC(int);
  for (int k = 0; k < nmem; ++k) { /* build_msflows (engine.cpp:49-89) */
    int r = AT(e->mpool, int, moff + k);
    req_in* q = &e->rq[r];
    double tokens = (double)q->tokens;
    int lead = unit * e->P.hpu;
    int dec = e->P.units * e->P.hpu + (unit % e->P.dhosts);
    for (int l = 1; l <= q->layers; ++l) {
      double rb = q->reuse * tokens * e->P.kv;
      if (rb > 0.0) {
        if (q->src < 0) {
          fail(3, "reuse_fraction > 0 needs a reuse_source");
          return;
        }
        flow f;
        memset(&f, 0, sizeof f);
        f.req = r;
        f.batch = b;
        f.cof = -1;
        f.stage = SREUSE;
        f.route = add_route(e, q->src * e->P.hpu, lead);
        f.size = rb;
        f.tl = l;
        f.dl = NAN;
        int id = reg_flow(e, &f);
        vpush(&LY(e, b, l - 1).reuse, &id);
        vpush(&rel, &id);
      }
      double pb = tokens * e->P.kv;
      if (pb > 0.0) {
        flow f;
        memset(&f, 0, sizeof f);
        f.req = r;
        f.batch = b;
        f.cof = -1;
        f.stage = SP2D;
        f.route = add_route(e, lead, dec);
        f.size = pb;
        f.tl = l;
        f.dl = q->deadline;
        f.has_dl = 1;
        int id = reg_flow(e, &f);
        vpush(&LY(e, b, l - 1).p2d, &id);
      }
    }
  }
  double cb = bt * e->P.coll;
  if (cb > 0.0 && e->P.hpu > 1) {
    for (int l = 1; l <= e->P.layers; ++l) {
      coflow c;
      memset(&c, 0, sizeof c);
      c.batch = b;
      c.layer = l;
      c.rel = c.done = NOT;
      c.mem.es = sizeof(int);
      int ci = (int)e->cofs.n;
      vpush(&e->cofs, &c);
      for (int i = 0; i < e->P.hpu; ++i)
        for (int j = 0; j < e->P.hpu; ++j) {
          if (i == j) continue;
          flow f;
          memset(&f, 0, sizeof f);
          f.req = -1;
          f.batch = b;
          f.cof = ci;
          f.stage = SCOLL;
          f.route = add_route(e, unit * e->P.hpu + i, unit * e->P.hpu + j);
          f.size = cb;
          f.tl = l;
          f.dl = NAN;
          int id = reg_flow(e, &f);
          vpush(&CF(e, ci).mem, &id);
          CF(e, ci).open++;
        }
      LY(e, b, l - 1).coll = ci;
    }
  }
  for (long i = 0; i < rel.n; ++i) release_flow(e, AT(rel, int, i));
  free(rel.p);
  e->busy[unit] = 1;
  start_layers(e, b);
  pipe_done(e, b);
  batch_hook(e);
  e->dirty = 1;
}
static void admit_try(engine* e, int unit) { /* engine.cpp:440-453 */
  if (e->busy[unit] || e->q_head[unit] == e->q_tail[unit]) return;
  int h = e->q_head[unit], cnt = 0;
  long tok = 0;
  while (h + cnt < e->q_tail[unit]) {
    int r = e->qlist[e->qoff[unit] + h + cnt];
    long t = e->rq[r].tokens;
    if (cnt > 0 && tok + t > e->P.maxtok) break;
    cnt++;
    tok += t;
  }
  e->q_head[unit] = h + cnt;
  admit_batch(e, unit, e->qoff[unit] + h, cnt);
}
static void compute_complete(engine* e, int b, int layer_) { /* engine.cpp:395-418 */
  layer* y = &LY(e, b, layer_ - 1);
  if (!(y->started && !y->done) || !deps_met(e, b, layer_)) {
    fail(6, "compute completion out of order");
    return;
  }
  y->done = 1;
  y->end = e->now;
  layer_boundary(e, b);
  y = &LY(e, b, layer_ - 1);
  if (y->coll >= 0) {
    coflow* c = &CF(e, y->coll);
    for (long i = 0; i < c->mem.n; ++i) {
      int fid = AT(CF(e, y->coll).mem, int, i);
      if (!FL(e, fid).scripted && FL(e, fid).state == PEND) release_flow(e, fid);
    }
  }
  y = &LY(e, b, layer_ - 1);
  for (long i = 0; i < y->p2d.n; ++i) {
    int fid = AT(LY(e, b, layer_ - 1).p2d, int, i);
    if (!FL(e, fid).scripted && FL(e, fid).state == PEND) release_flow(e, fid);
  }
  start_layers(e, b);
  pipe_done(e, b);
  e->dirty = 1;
}
static int p2d_left(engine* e, int b) {
  batch* B = &BA(e, b);
  for (long i = 0; i < B->fl.n; ++i) {
    flow* f = &FL(e, AT(B->fl, int, i));
    if (f->stage == SP2D && f->state != DONE) return 1;
  }
  return 0;
}
static void depart(engine* e, int b) { /* engine.cpp:420-438 */
  if (BA(e, b).departed) return;
  BA(e, b).departed = 1;
  if (e->workload) {
    e->busy[BA(e, b).unit] = 0;
    push(e, e->now, KADM, BA(e, b).unit, -1);
  }
  if (p2d_left(e, b) && e->P.policy == 4) push(e, e->now + e->P.tick, KTICK, b, -1);
  batch_hook(e);
  for (int k = 0; k < BA(e, b).nmem; ++k) complete_req(e, AT(e->mpool, int, BA(e, b).moff + k));
  e->dirty = 1;
}
static void activate_manual(engine* e, int b) { /* engine.cpp:541-558 */
  if (BA(e, b).admitted) return;
  BA(e, b).admitted = 1;
  for (long i = 0; i < BA(e, b).fl.n; ++i) {
    int fid = AT(BA(e, b).fl, int, i);
    flow* f = &FL(e, fid);
    if (f->scripted) push(e, dmax(e->now, f->relat), KREL, fid, -1);
    else if (f->stage == SREUSE) release_flow(e, fid);
  }
  start_layers(e, b);
  pipe_done(e, b);
  batch_hook(e);
  e->dirty = 1;
}
static void recompute(engine* e) { /* engine.cpp:278-293 */
  classes C;
  decide(e, &C);
  e->steps++;
  for (long i = 0; i < e->aorder.n; ++i) FL(e, AT(e->aorder, int, i)).arate = -1.0;
  allocate(e, &C);
  for (long i = 0; i < e->active.n; ++i) {
    int fid = AT(e->active, int, i);
    flow* f = &FL(e, fid);
    double r = f->arate < 0 ? 0.0 : f->arate;
    if (r == f->rate) continue;
    f->rate = r;
    f->gen++;
    if (r > 0.0) push(e, e->now + f->rem / r, KFLOW, fid, f->gen);
  }
  free(C.ids);
  free(C.start);
  free(C.caps);
}
static void run(engine* e) { /* engine.cpp:595-657 */
  recompute(e);
  e->dirty = 0;
  double prev = -1.0;
  while (e->hn && !E.err) {
    if (e->heap[0].t > e->horizon) break;
    event v = pop(e);
    if (v.kind == KFLOW) {
      flow* f = &FL(e, v.a);
      if (f->state == DONE || v.b != f->gen) continue;
    }
    double dt = v.t - e->now;
    if (!(dt > -1e-9)) {
      fail(6, "event time went backwards");
      break;
    }
    if (dt > 0.0)
      for (long i = 0; i < e->active.n; ++i) {
        flow* f = &FL(e, AT(e->active, int, i));
        f->rem -= f->rate * dt;
        if (f->rem < 0.0) {
          if (!(f->rem > -1e-6 * dmax(f->size, 1.0) - 1e-9)) fail(6, "overshoot");
          f->rem = 0.0;
        }
      }
    e->now = v.t;
    e->events++;
    if (v.t == prev) {
      if (++e->streak > e->P.livelock) {
        fail(5, "livelock");
        break;
      }
    } else {
      e->streak = 0;
      prev = v.t;
    }
    switch (v.kind) {
      case KFLOW: finish_flow(e, v.a); break;
      case KCOMP: compute_complete(e, v.a, v.b); break;
      case KDEP: depart(e, v.a); break;
      case KARR: {
        int u = e->rq[v.a].unit;
        e->qlist[e->qoff[u] + e->q_tail[u]++] = v.a;
        push(e, e->now, KADM, u, -1);
        break;
      }
      case KADM:
        if (e->workload) admit_try(e, v.a);
        else activate_manual(e, v.a);
        break;
      case KREL:
        if (FL(e, v.a).state == PEND) release_flow(e, v.a);
        break;
      case KTICK:
        if (p2d_left(e, v.a)) {
          if (e->P.policy == 4 && promote_batch(e, v.a, 1)) e->dirty = 1;
          push(e, e->now + e->P.tick, KTICK, v.a, -1);
        }
        break;
    }
    if (e->dirty && !E.err) {
      recompute(e);
      e->dirty = 0;
    }
  }
}

/* ------------------------------------------------------- instances + ABI */

struct ref_result {
  long events, steps, pruned_count;
  int n_req, n_flows, n_coflows, n_batches;
  double t_run_s, t_setup_s;
  double *req_arrival, *req_deadline, *req_done;
  unsigned char* req_pruned;
  double* req_stall;
  int* req_batch;
  double* flow_finish;
  int *flow_band, *flow_level;
  double *cof_release, *cof_done, *cof_stall, *pipe_done;
  char *summary_json, *requests_csv;
  int err;
  char errmsg[512];
};

static void engine_init(engine* e, fabric* F, const params* P, req_in* rq, long nreq) {
  memset(e, 0, sizeof *e);
  e->P = *P;
  e->F = F;
  e->roff.es = e->rlinks.es = sizeof(int);
  e->flows.es = sizeof(flow);
  e->att.es = sizeof(double);
  e->batches.es = sizeof(batch);
  e->layers.es = sizeof(layer);
  e->cofs.es = sizeof(coflow);
  e->mpool.es = e->fpool.es = e->active.es = e->aorder.es = sizeof(int);
  e->rq = rq;
  e->nreq = nreq;
  long n = nreq ? nreq : 1;
  e->r_batch = malloc(sizeof(int) * n);
  e->r_pruned = calloc(n, sizeof(int));
  e->r_open = calloc(n, sizeof(int));
  e->r_rank = malloc(sizeof(int) * n);
  e->r_ttft = malloc(sizeof(double) * n);
  e->r_last = malloc(sizeof(double) * n);
  for (long i = 0; i < nreq; ++i) {
    e->r_batch[i] = -1;
    e->r_rank[i] = -1;
    e->r_ttft[i] = NOT;
    e->r_last[i] = NOT;
  }
}

static void engine_free(engine* e) {
  for (long b = 0; b < e->batches.n; ++b) free(BA(e, b).fl.p);
  for (long l = 0; l < e->layers.n; ++l) {
    free(AT(e->layers, layer, l).reuse.p);
    free(AT(e->layers, layer, l).p2d.p);
  }
  for (long c = 0; c < e->cofs.n; ++c) free(CF(e, c).mem.p);
  free(e->roff.p);
  free(e->rlinks.p);
  free(e->flows.p);
  free(e->batches.p);
  free(e->layers.p);
  free(e->att.p);
  free(e->asum);
  free(e->astamp);
  free(e->cofs.p);
  if (!e->workload) free(e->mpool.p);
  free(e->fpool.p);
  free(e->active.p);
  free(e->aorder.p);
  free(e->r_batch);
  free(e->r_pruned);
  free(e->r_open);
  free(e->r_rank);
  free(e->r_ttft);
  free(e->r_last);
  free(e->q_head);
  free(e->q_tail);
  free(e->busy);
  free(e->qlist);
  free(e->qoff);
  free(e->heap);
}

/* load_workload (engine.cpp:222-246) + run */
static void run_workload(engine* e, fabric* F, const params* P, req_in* rq, long n) {
  engine_init(e, F, P, rq, n);
  e->workload = 1;
  e->q_head = calloc(P->units, sizeof(int));
  e->q_tail = calloc(P->units, sizeof(int));
  e->busy = calloc(P->units, sizeof(int));
  e->qoff = calloc(P->units + 1, sizeof(int));
  for (long i = 0; i < n; ++i) e->qoff[rq[i].unit + 1]++;
  for (int u = 0; u < P->units; ++u) e->qoff[u + 1] += e->qoff[u];
  e->qlist = malloc(sizeof(int) * (n ? n : 1));
  e->mpool.p = e->qlist;
  double last = 0.0;
  for (long i = 0; i < n; ++i) {
    last = dmax(last, rq[i].arrival);
    push(e, rq[i].arrival, KARR, (int)i, -1);
  }
  e->horizon = P->has_horizon ? P->horizon : last + P->horizon_slack;
  run(e);
}

static int read_params(const kvcfg* c, params* P) {
  P->layers = (int)cfg_long(c, "model.layers", 4);
  P->alpha = cfg_num(c, "model.alpha_ms", 1.0) * 1e-3;
  P->beta = cfg_num(c, "model.beta_us_per_token", 1.0) * 1e-6;
  P->kv = cfg_num(c, "model.kv_bytes_per_token_layer", 1000.0);
  P->coll = cfg_num(c, "model.coll_bytes_per_token_layer", 250.0);
  P->units = (int)cfg_long(c, "cluster.prefill_units", 1);
  P->hpu = (int)cfg_long(c, "cluster.hosts_per_unit", 2);
  P->dhosts = (int)cfg_long(c, "cluster.decode_hosts", P->units);
  P->has_horizon = cfg_raw(c, "sim.horizon_s") != NULL;
  P->horizon = cfg_num(c, "sim.horizon_s", 0.0);
  P->horizon_slack = 300.0;
  P->tick = cfg_num(c, "sim.promotion_tick_ms", 1.0) * 1e-3;
  P->maxtok = cfg_long(c, "workload.max_batch_tokens", 8192);
  P->livelock = cfg_long(c, "sim.livelock_events", 1000000);
  const char* pol = cfg_raw(c, "policy");
  if (!pol) pol = "fs";
  P->policy = !strcmp(pol, "fs") ? 0 : !strcmp(pol, "sjf") ? 1 : !strcmp(pol, "edf") ? 2
            : !strcmp(pol, "karuna") ? 3 : !strcmp(pol, "mfs") ? 4
            : !strcmp(pol, "aalo") ? 5 : !strcmp(pol, "varys") ? 6 : -1;
  if (P->policy < 0) fail(2, "unknown policy");
  P->K = 8;
  if (P->policy == 5) { /* extension: Aalo D-CLAS queues, thresholds Q0 * E^i */
    P->K = (int)cfg_long(c, "aalo.K", 8);
    double E_ = cfg_num(c, "aalo.E", 10.0), q = cfg_num(c, "aalo.Q0", 1e-3);
    if (P->K < 2 || P->K > MAXK || !(E_ > 1.0) || !(q > 0.0) || q == INF) fail(2, "config: aalo");
    for (int i = 0; i + 1 < P->K && i < MAXK; ++i) {
      P->thr[i] = q;
      q *= E_;
    }
  }
  if (P->policy == 4) { /* rmlq.cpp:8-27, policy_factory.cpp:34-40 */
    P->K = (int)cfg_long(c, "mfs.K", 8);
    double E_ = cfg_num(c, "mfs.E", 4.0), U = cfg_num(c, "mfs.U", 0.5);
    if (P->K < 2 || P->K > MAXK || !(E_ > 1.0) || !(U > 0.0 && U <= 1.0)) fail(2, "config: mfs");
    double q = U;
    for (int i = 1; i < P->K && i <= MAXK; ++i) {
      q /= E_;
      P->thr[i - 1] = q;
    }
    P->prune = cfg_bool(c, "inter.enable_pruning", 1);
    P->dfrac = cfg_num(c, "inter.drop_budget_frac", 0.05);
  }
  if (P->layers < 1 || P->units < 1 || P->hpu < 1 || P->dhosts < 1 || !(P->tick > 0))
    fail(2, "config: invalid");
  return E.err;
}

static void build_fabric(const kvcfg* c, fabric* F) {
  const char* kind = cfg_raw(c, "topology.kind");
  if (!kind) kind = "star";
  long hosts = cfg_long(c, "topology.hosts", 2), nics = cfg_long(c, "topology.nics_per_host", 1);
  double cap = cfg_raw(c, "topology.link_bytes_per_s")
                   ? cfg_num(c, "topology.link_bytes_per_s", 0) * (double)nics
                   : cfg_num(c, "topology.link_gbps", 1.0) * 1e9 / 8.0 * (double)nics;
  double os = cfg_num(c, "topology.oversubscription", 1.0);
  if (!(os >= 1.0) || os == INF) fail(2, "config: topology.oversubscription must be >= 1");
  if (!strcmp(kind, "star")) {
    if (os != 1.0) fail(2, "config: oversubscription needs a fat-tree");
    fab_star(F, (int)hosts, cap);
  } else if (!strcmp(kind, "fattree")) fab_fattree(F, (int)hosts, cap, os);
  else fail(2, "config: unknown topology");
  fab_finish(F);
}

/* finalize (engine.cpp:659-707) and export */
static struct ref_result* export(engine* e) {
  struct ref_result* o = calloc(1, sizeof *o);
  o->events = e->events;
  o->steps = e->steps;
  o->pruned_count = e->pruned_count;
  o->n_req = (int)e->nreq;
  o->n_flows = (int)e->flows.n;
  o->n_coflows = (int)e->cofs.n;
  o->n_batches = (int)e->batches.n;
  long nr = e->nreq ? e->nreq : 1;
  o->req_arrival = malloc(sizeof(double) * nr);
  o->req_deadline = malloc(sizeof(double) * nr);
  o->req_done = malloc(sizeof(double) * nr);
  o->req_pruned = malloc(nr);
  o->req_stall = calloc(nr, sizeof(double));
  o->req_batch = malloc(sizeof(int) * nr);
  long nf = e->flows.n ? e->flows.n : 1, nc = e->cofs.n ? e->cofs.n : 1;
  o->flow_finish = malloc(sizeof(double) * nf);
  o->flow_band = malloc(sizeof(int) * nf);
  o->flow_level = malloc(sizeof(int) * nf);
  o->cof_release = malloc(sizeof(double) * nc);
  o->cof_done = malloc(sizeof(double) * nc);
  o->cof_stall = calloc(nc, sizeof(double));
  o->pipe_done = malloc(sizeof(double) * (e->batches.n ? e->batches.n : 1));
  double* bst = calloc(e->batches.n + 1, sizeof(double));
  for (long c = 0; c < e->cofs.n; ++c) {
    coflow* C = &CF(e, c);
    o->cof_release[c] = C->rel;
    o->cof_done[c] = C->done;
    if (C->done != NOT) {
      batch* B = &BA(e, C->batch);
      double other = LY(e, C->batch, C->layer - 1).end;
      if (C->layer < B->layers) {
        layer* nx = &LY(e, C->batch, C->layer);
        for (long k = 0; k < nx->reuse.n; ++k) {
          flow* f = &FL(e, AT(nx->reuse, int, k));
          if (f->req >= 0 && e->r_pruned[f->req]) continue;
          if (f->fin != NOT) other = dmax(other, f->fin);
        }
      }
      o->cof_stall[c] = dmax(0.0, C->done - other);
      bst[C->batch] += o->cof_stall[c];
    }
  }
  for (long r = 0; r < e->nreq; ++r) {
    o->req_arrival[r] = e->rq[r].arrival;
    o->req_deadline[r] = e->rq[r].deadline;
    o->req_done[r] = e->r_ttft[r] == NOT ? NAN : e->r_ttft[r];
    o->req_pruned[r] = (unsigned char)e->r_pruned[r];
    o->req_batch[r] = e->r_batch[r];
    if (e->r_batch[r] >= 0) o->req_stall[r] = bst[e->r_batch[r]];
  }
  for (long f = 0; f < e->flows.n; ++f) {
    o->flow_finish[f] = FL(e, f).fin;
    o->flow_band[f] = FL(e, f).band;
    o->flow_level[f] = FL(e, f).level;
  }
  for (long b = 0; b < e->batches.n; ++b) o->pipe_done[b] = BA(e, b).done;
  free(bst);
  return o;
}

void ref_free(struct ref_result* r) {
  if (!r) return;
  free(r->req_arrival);
  free(r->req_deadline);
  free(r->req_done);
  free(r->req_pruned);
  free(r->req_stall);
  free(r->req_batch);
  free(r->flow_finish);
  free(r->flow_band);
  free(r->flow_level);
  free(r->cof_release);
  free(r->cof_done);
  free(r->cof_stall);
  free(r->pipe_done);
  free(r->summary_json);
  free(r->requests_csv);
  free(r);
}

static struct ref_result* errres(void) {
  struct ref_result* o = calloc(1, sizeof *o);
  o->err = E.err;
  snprintf(o->errmsg, sizeof o->errmsg, "%s", E.msg);
  return o;
}

/* derive_slos (workload.cpp:199-217): one isolated FS run per distinct key */
typedef struct {
  long tok, bits;
  int unit, src;
  double low;
} slokey;

int ref_run_config(const char* text, struct ref_result** out) {
  memset(&E, 0, sizeof E);
  kvcfg c = {0};
  cfg_parse(&c, text);
  params P;
  memset(&P, 0, sizeof P);
  read_params(&c, &P);
  fabric F;
  memset(&F, 0, sizeof F);
  if (!E.err) build_fabric(&c, &F);
  if (!E.err && P.units * P.hpu + P.dhosts > F.hosts) fail(2, "layout needs more hosts");
  long n = 0;
  req_in* rq = NULL;
  clock_t t0 = clock();
  if (!E.err) {
    const char* tr = cfg_raw(&c, "workload.trace");
    rq = (tr && *tr) ? trace(tr, &P, &n) : synth(&c, &P, &n);
  }
  double mult = cfg_num(&c, "workload.slo_multiplier", 3.0);
  if (!E.err) {
    vec keys = VEC(slokey);
    for (long i = 0; i < n && !E.err; ++i) {
      if (rq[i].tokens > P.maxtok) fail(3, "prompt exceeds the batch token cap");
      long bits = llround(rq[i].reuse * 1e9);
      double low = -1;
      for (long k = 0; k < keys.n; ++k) {
        slokey* s = &AT(keys, slokey, k);
        if (s->tok == rq[i].tokens && s->bits == bits && s->unit == rq[i].unit && s->src == rq[i].src) {
          low = s->low;
          break;
        }
      }
      if (low < 0) {
        req_in probe = rq[i];
        probe.arrival = 0.0;
        probe.deadline = INF;
        params Q = P;
        Q.policy = 0;
        Q.has_horizon = 0;
        Q.horizon_slack = 1e9;
        engine iso;
        run_workload(&iso, &F, &Q, &probe, 1);
        low = iso.r_ttft[0];
        engine_free(&iso);
        slokey s = {rq[i].tokens, bits, rq[i].unit, rq[i].src, low};
        vpush(&keys, &s);
      }
      rq[i].deadline = rq[i].arrival + mult * low;
    }
    free(keys.p);
  }
  struct ref_result* o;
  if (E.err) {
    o = errres();
  } else {
    engine e;
    clock_t t1 = clock();
    run_workload(&e, &F, &P, rq, n);
    clock_t t2 = clock();
    o = E.err ? errres() : export(&e);
    o->t_setup_s = (double)(t1 - t0) / CLOCKS_PER_SEC;
    o->t_run_s = (double)(t2 - t1) / CLOCKS_PER_SEC;
    engine_free(&e);
  }
  free(rq);
  fab_free(&F);
  cfg_free(&c);
  *out = o;
  return o->err;
}

/* manual instances (engine.cpp:114-220) from the shared text spec */
int ref_run_manual(const char* spec, struct ref_result** out) {
  memset(&E, 0, sizeof E);
  kvcfg c = {0};
  params P;
  memset(&P, 0, sizeof P);
  P.horizon_slack = 300.0;
  P.tick = 1e-3;
  P.maxtok = 8192;
  P.livelock = 1000000;
  fabric F;
  memset(&F, 0, sizeof F);
  char pol[32] = "fs";
  /* pass 1: header lines */
  char* text = strdup(spec);
  vec ops = VEC(char*);
  for (char* line = strtok(text, "\n"); line; line = strtok(NULL, "\n")) {
    char* h = strchr(line, '#');
    if (h) *h = 0;
    char* t[12];
    int nt = 0;
    for (char* w = strtok_r(line, " \t\r", &h); w && nt < 12; w = strtok_r(NULL, " \t\r", &h)) t[nt++] = w;
    if (!nt) continue;
    if (!strcmp(t[0], "policy")) snprintf(pol, sizeof pol, "%s", t[1]);
    else if (!strcmp(t[0], "set")) cfg_set(&c, t[1], t[2]);
    else if (!strcmp(t[0], "param")) {
      double v = strtod(t[2], NULL);
      if (!strcmp(t[1], "promotion_tick")) P.tick = v;
      else if (!strcmp(t[1], "horizon")) {
        P.has_horizon = 1;
        P.horizon = v;
      } else if (!strcmp(t[1], "horizon_slack")) P.horizon_slack = v;
      else if (!strcmp(t[1], "max_batch_tokens")) P.maxtok = (long)v;
      else if (!strcmp(t[1], "livelock_events")) P.livelock = (long)v;
    } else if (!strcmp(t[0], "node")) fab_add_node(&F);
    else if (!strcmp(t[0], "link")) fab_add_link(&F, atoi(t[1]), atoi(t[2]), strtod(t[3], NULL));
    else if (!strcmp(t[0], "duplex")) fab_duplex(&F, atoi(t[1]), atoi(t[2]), strtod(t[3], NULL));
    else {
      /* re-join the op for pass 2 */
      char buf[512] = "";
      for (int i = 0; i < nt; ++i) {
        strcat(buf, t[i]);
        strcat(buf, " ");
      }
      char* d = strdup(buf);
      vpush(&ops, &d);
    }
  }
  free(text);
  cfg_set(&c, "policy", pol);
  int K = (int)cfg_long(&c, "mfs.K", 8);
  (void)K;
  params Q;
  memset(&Q, 0, sizeof Q);
  read_params(&c, &Q);
  P.policy = Q.policy;
  P.K = Q.K;
  memcpy(P.thr, Q.thr, sizeof P.thr);
  P.prune = Q.prune;
  P.dfrac = Q.dfrac;
  fab_finish(&F);
  /* requests first pass: count */
  vec rqv = VEC(req_in);
  for (long i = 0; i < ops.n; ++i) {
    char* s = AT(ops, char*, i);
    if (!strncmp(s, "request ", 8)) {
      req_in q;
      memset(&q, 0, sizeof q);
      char a[64], d[64];
      long tok = 0;
      int got = sscanf(s + 8, "%63s %63s %ld", a, d, &tok);
      q.arrival = strcmp(a, "-") ? strtod(a, NULL) : -1.0;
      q.deadline = strtod(d, NULL);
      q.tokens = got >= 3 ? tok : 0;
      q.src = -1;
      vpush(&rqv, &q);
    }
  }
  engine e;
  engine_init(&e, &F, &P, (req_in*)rqv.p, rqv.n);
  e.workload = 0;
  double last = 0.0;
  long rseen = 0;
  for (long i = 0; i < ops.n && !E.err; ++i) {
    char* s = AT(ops, char*, i);
    char* t[12];
    int nt = 0;
    char* save;
    for (char* w = strtok_r(s, " ", &save); w && nt < 12; w = strtok_r(NULL, " ", &save)) t[nt++] = w;
    if (!strcmp(t[0], "request")) {
      rseen++;
    } else if (!strcmp(t[0], "batch")) {
      double at = strcmp(t[1], "-") ? strtod(t[1], NULL) : -1.0;
      int moff = (int)e.mpool.n, nm = 0;
      if (strcmp(t[2], "-"))
        for (char* m = strtok_r(t[2], ",", &save); m; m = strtok_r(NULL, ",", &save)) {
          int r = atoi(m);
          vpush(&e.mpool, &r);
          nm++;
        }
      vec costs = VEC(double);
      if (strcmp(t[3], "-"))
        for (char* m = strtok_r(t[3], ",", &save); m; m = strtok_r(NULL, ",", &save)) {
          double x = strtod(m, NULL);
          vpush(&costs, &x);
        }
      int b = new_batch(&e, nm, moff, at, (int)costs.n);
      for (long l = 0; l < costs.n; ++l) LY(&e, b, l).cost = AT(costs, double, l);
      free(costs.p);
      for (int k = 0; k < nm; ++k) e.r_batch[AT(e.mpool, int, moff + k)] = b;
      last = dmax(last, at);
      push(&e, at, KADM, b, -1);
    } else if (!strcmp(t[0], "flow")) {
      flow f;
      memset(&f, 0, sizeof f);
      f.batch = atoi(t[1]);
      f.req = atoi(t[2]);
      f.stage = !strcmp(t[3], "reuse") ? SREUSE : !strcmp(t[3], "collective") ? SCOLL : SP2D;
      f.route = add_route(&e, atoi(t[4]), atoi(t[5]));
      f.size = strtod(t[6], NULL);
      f.tl = atoi(t[7]);
      f.scripted = strcmp(t[8], "-") != 0;
      f.relat = f.scripted ? strtod(t[8], NULL) : 0.0;
      f.has_dl = strcmp(t[9], "-") != 0;
      f.dl = f.has_dl ? strtod(t[9], NULL) : NAN;
      f.cof = -1;
      int id = reg_flow(&e, &f);
      int b = f.batch, idx = f.tl - 1;
      if (idx >= 0 && idx < BA(&e, b).layers) {
        layer* y = &LY(&e, b, idx);
        if (f.stage == SREUSE) vpush(&y->reuse, &id);
        else if (f.stage == SP2D) vpush(&y->p2d, &id);
        else {
          if (y->coll < 0) {
            coflow cf;
            memset(&cf, 0, sizeof cf);
            cf.batch = b;
            cf.layer = f.tl;
            cf.rel = cf.done = NOT;
            cf.mem.es = sizeof(int);
            LY(&e, b, idx).coll = (int)e.cofs.n;
            vpush(&e.cofs, &cf);
          }
          int ci = LY(&e, b, idx).coll;
          vpush(&CF(&e, ci).mem, &id);
          CF(&e, ci).open++;
          FL(&e, id).cof = ci;
        }
      }
    }
  }
  (void)rseen;
  e.horizon = P.has_horizon ? P.horizon : last + P.horizon_slack;
  clock_t t1 = clock();
  if (!E.err) run(&e);
  struct ref_result* o = E.err ? errres() : export(&e);
  o->t_run_s = (double)(clock() - t1) / CLOCKS_PER_SEC;
  engine_free(&e);
  free(rqv.p);
  for (long i = 0; i < ops.n; ++i) free(AT(ops, char*, i));
  free(ops.p);
  fab_free(&F);
  cfg_free(&c);
  *out = o;
  return o->err;
}

int ref_derive_deadlines(const char* text, struct ref_result** out) {
  struct ref_result* o = NULL;
  int rc = ref_run_config(text, &o);
  *out = o;
  return rc;
}
