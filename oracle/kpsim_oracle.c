/* TEST INFRASTRUCTURE ONLY -- the CPU oracle for the B200 hot path.
 *
 * A plain-C restatement of the reference's per-batch training path
 * (Trainer::process_batch, /root/reference/proj/src/trainer.cpp:115-259) and
 * everything it calls: working-set dedup, insert-if-absent table with fresh
 * init, pooling + MLP forward/backward (proj/src/model.cpp:76-191), averaged
 * sparse AdaGrad push (proj/src/store.cpp:191-208, optimizer.cpp:86-95) and
 * the k-step Adam engine (proj/src/optimizer.cpp:39-153, common.hpp:27-45).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this. It is never on the product path.
 *
 * Compiled twice by oracle/Makefile:
 *   ORC_REAL=double, prefix orc64_  -- must be BIT-EXACT against the compiled
 *       reference (oracle/_ref/libkpsim_ref.so) at S=1 + AdaGrad; this pins
 *       the restatement (tests/test_oracle_pin.py).
 *   ORC_REAL=float,  prefix orc32_  -- the same expression trees in fp32; its
 *       drift against the f64 oracle sets the tolerance envelope for the GPU.
 * Extensions the reference lacks (documented in DESIGN.md):
 *   - S slots per instance: pooled[b][s*e:(s+1)*e] sums the occurrences with
 *     slot id s; the MLP input width is S*e. S=1 is the reference exactly.
 *   - sparse Adam rule: the reference KStepEngine at N=1,k=1 applied per row
 *     (m=b1 m+(1-b1)g; v=b2 v+(1-b2)(g g); w=w-a m/sqrt(v)), fresh m=0, v=eps.
 * Build flags: -O2 -ffp-contract=off (the reference's, CMakeLists.txt:9).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef ORC_REAL
#define ORC_REAL double
#endif
#ifndef ORC_PFX
#define ORC_PFX orc64_
#endif
#define ORC_CAT(a, b) a##b
#define ORC_XCAT(a, b) ORC_CAT(a, b)
#define FN(n) ORC_XCAT(ORC_PFX, n)

typedef ORC_REAL real;
#define IS_F32 (sizeof(real) == 4)
static real r_exp(real x) { return IS_F32 ? (real)expf((float)x) : (real)exp((double)x); }
static real r_sqrt(real x) { return IS_F32 ? (real)sqrtf((float)x) : (real)sqrt((double)x); }
static real r_log1p(real x) { return IS_F32 ? (real)log1pf((float)x) : (real)log1p((double)x); }
static real r_tanh(real x) { return IS_F32 ? (real)tanhf((float)x) : (real)tanh((double)x); }
static real r_abs(real x) { return x < 0 ? -x : x; }

/* ---------------------------------------------------------------- rng --- */
/* splitmix64: proj/include/kpsim/common.hpp:54-59 */
uint64_t FN(splitmix64)(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* std::mt19937_64 (the standard's parameters) */
typedef struct { uint64_t mt[312]; int idx; } mt64;
static void mt64_seed(mt64* g, uint64_t s) {
  g->mt[0] = s;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}
static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}
/* libstdc++ uniform_real_distribution<double>(a,b): generate_canonical with a
 * single 64-bit draw, then u*(b-a)+a (bits/random.h, GCC 13). */
static double mt64_uniform(mt64* g, double a, double b) {
  double u = (double)mt64_next(g) / 18446744073709551616.0;
  if (u >= 1.0) u = nextafter(1.0, 0.0);
  return u * (b - a) + a;
}

/* CtrModel::init_dense (proj/src/model.cpp:68-74): U(-0.05,0.05) in f64 */
void FN(init_dense)(uint64_t seed, uint64_t dim, double* out) {
  mt64 g;
  mt64_seed(&g, FN(splitmix64)(seed ^ 0xD15EA5E0ULL));
  for (uint64_t i = 0; i < dim; ++i) out[i] = mt64_uniform(&g, -0.05, 0.05);
}

/* -------------------------------------------------------------- dedup --- */
static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}
/* Working-set dedup (proj/src/trainer.cpp:121-124: std::set insert): sorted
 * unique keys; inverse[i] = index of keys[i] in unique. Returns U. */
uint64_t FN(dedup)(const uint64_t* keys, uint64_t n, uint64_t* unique, uint32_t* inverse) {
  if (n == 0) return 0;
  uint64_t* tmp = (uint64_t*)malloc(n * 8);
  memcpy(tmp, keys, n * 8);
  qsort(tmp, n, 8, cmp_u64);
  uint64_t u = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (i == 0 || tmp[i] != tmp[i - 1]) unique[u++] = tmp[i];
  free(tmp);
  if (inverse)
    for (uint64_t i = 0; i < n; ++i) {
      uint64_t lo = 0, hi = u;
      while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        if (unique[mid] < keys[i]) lo = mid + 1; else hi = mid;
      }
      inverse[i] = (uint32_t)lo;
    }
  return u;
}

/* owner shard = key % G (proj/src/trainer.cpp:83); stable bucket of the
 * (ascending) unique keys; counts[G]; perm[i] = source index of slot i. */
void FN(shard)(const uint64_t* unique, uint64_t n, uint32_t G, uint32_t* perm, uint64_t* counts) {
  for (uint32_t g = 0; g < G; ++g) counts[g] = 0;
  for (uint64_t i = 0; i < n; ++i) counts[unique[i] % G]++;
  uint64_t* start = (uint64_t*)calloc(G, 8);
  for (uint32_t g = 1; g < G; ++g) start[g] = start[g - 1] + counts[g - 1];
  for (uint64_t i = 0; i < n; ++i) perm[start[unique[i] % G]++] = (uint32_t)i;
  free(start);
}

/* ----------------------------------------------------- sparse rules --- */
/* AdaGrad (proj/src/optimizer.cpp:86-95) */
void FN(adagrad)(real* w, real* acc, const real* g, uint64_t n, real lr) {
  for (uint64_t j = 0; j < n; ++j) {
    acc[j] += g[j] * g[j];
    w[j] -= lr * g[j] / r_sqrt(acc[j]);
  }
}
/* sparse Adam = KStepEngine N=1,k=1 per row (optimizer.cpp:39-46,56-84) */
void FN(sparse_adam)(real* w, real* m, real* v, const real* g, uint64_t n, real alpha,
                     real b1, real b2) {
  for (uint64_t j = 0; j < n; ++j) {
    m[j] = b1 * m[j] + ((real)1 - b1) * g[j];
    v[j] = b2 * v[j] + ((real)1 - b2) * (g[j] * g[j]);
    w[j] = w[j] - alpha * m[j] / r_sqrt(v[j]);
  }
}

/* --------------------------------------------------------- k-step Adam --- */
typedef struct { real *x, *m, *v, *vbar; uint64_t t; } wstate;

/* centered mean, ascending worker order (common.hpp:27-45) */
static void cmean(uint64_t n, uint64_t d, real* const* vecs, real* out) {
  for (uint64_t j = 0; j < d; ++j) {
    const real base = vecs[0][j];
    real acc = 0;
    for (uint64_t i = 0; i < n; ++i) acc += vecs[i][j] - base;
    out[j] = base + acc / (real)n;
  }
}

typedef struct {
  real alpha, beta1, beta2, eps;
  uint64_t k;
  int reset_v;
} hyper;

static void accumulate_moments(wstate* s, const real* g, uint64_t d, const hyper* h) {
  for (uint64_t j = 0; j < d; ++j) {
    s->m[j] = h->beta1 * s->m[j] + ((real)1 - h->beta1) * g[j];
    s->v[j] = h->beta2 * s->v[j] + ((real)1 - h->beta2) * (g[j] * g[j]);
  }
}
static void local_adam_step(wstate* s, const real* g, uint64_t d, const hyper* h) {
  accumulate_moments(s, g, d, h);
  for (uint64_t j = 0; j < d; ++j) s->x[j] = s->x[j] - h->alpha * s->m[j] / r_sqrt(s->vbar[j]);
  s->t += 1;
}
static void global_merge(wstate* st, uint64_t n, uint64_t d, const hyper* h) {
  real** ptr = (real**)malloc(n * sizeof(real*));
  real* vbar = (real*)malloc(d * sizeof(real));
  real* terms = (real*)malloc(n * d * sizeof(real));
  real* merged = (real*)malloc(d * sizeof(real));
  for (uint64_t i = 0; i < n; ++i) ptr[i] = st[i].v;
  cmean(n, d, ptr, vbar);
  for (uint64_t i = 0; i < n; ++i) {
    for (uint64_t j = 0; j < d; ++j)
      terms[i * d + j] = st[i].x[j] - h->alpha * st[i].m[j] / r_sqrt(vbar[j]);
    ptr[i] = terms + i * d;
  }
  cmean(n, d, ptr, merged);
  for (uint64_t i = 0; i < n; ++i) {
    memcpy(st[i].x, merged, d * sizeof(real));
    memcpy(st[i].vbar, vbar, d * sizeof(real));
    if (h->reset_v) memcpy(st[i].v, vbar, d * sizeof(real));
    st[i].t += 1;
  }
  free(ptr); free(vbar); free(terms); free(merged);
}
/* KStepEngine::step (optimizer.cpp:113-144); returns merged flag */
static int kstep(wstate* st, uint64_t n, uint64_t d, const hyper* h, uint64_t* t_global,
                 real* const* grads) {
  const uint64_t t = *t_global + 1;
  const int merged = (t % h->k) == 0;
  if (!merged) {
    for (uint64_t i = 0; i < n; ++i) local_adam_step(&st[i], grads[i], d, h);
  } else {
    for (uint64_t i = 0; i < n; ++i) accumulate_moments(&st[i], grads[i], d, h);
    global_merge(st, n, d, h);
  }
  *t_global = t;
  return merged;
}

/* standalone engine driver (mirrors oracle/ref_driver.cpp ref_kstep) */
int FN(kstep_run)(double alpha, double beta1, double beta2, double eps, uint64_t k, int reset_v,
                  uint64_t workers, uint64_t dim, const double* x0, uint64_t steps,
                  const double* grads, double* xs, double* ms, double* vs, double* vbars,
                  int32_t* merged) {
  hyper h = {(real)alpha, (real)beta1, (real)beta2, (real)eps, k, reset_v};
  wstate* st = (wstate*)calloc(workers, sizeof(wstate));
  real* buf = (real*)malloc(workers * dim * 4 * sizeof(real));
  real* g = (real*)malloc(workers * dim * sizeof(real));
  real** gp = (real**)malloc(workers * sizeof(real*));
  for (uint64_t i = 0; i < workers; ++i) {
    st[i].x = buf + (i * 4 + 0) * dim; st[i].m = buf + (i * 4 + 1) * dim;
    st[i].v = buf + (i * 4 + 2) * dim; st[i].vbar = buf + (i * 4 + 3) * dim;
    for (uint64_t j = 0; j < dim; ++j) {
      st[i].x[j] = (real)x0[j]; st[i].m[j] = 0; st[i].v[j] = (real)eps; st[i].vbar[j] = (real)eps;
    }
    gp[i] = g + i * dim;
  }
  uint64_t tg = 0;
  for (uint64_t t = 0; t < steps; ++t) {
    for (uint64_t i = 0; i < workers * dim; ++i) g[i] = (real)grads[t * workers * dim + i];
    merged[t] = kstep(st, workers, dim, &h, &tg, gp);
    for (uint64_t i = 0; i < workers; ++i)
      for (uint64_t j = 0; j < dim; ++j) {
        const uint64_t o = (t * workers + i) * dim + j;
        xs[o] = st[i].x[j]; ms[o] = st[i].m[j]; vs[o] = st[i].v[j]; vbars[o] = st[i].vbar[j];
      }
  }
  free(st); free(buf); free(g); free(gp);
  return 0;
}

/* --------------------------------------------------------------- AUC --- */
typedef struct { double s; int32_t y; } scored;
static int cmp_scored(const void* a, const void* b) {
  double x = ((const scored*)a)->s, y = ((const scored*)b)->s;
  return x < y ? -1 : x > y;
}
/* rank-sum AUC with tie averaging (proj/src/eval.cpp:8-39); NaN if undefined */
double FN(auc)(const double* scores, const int32_t* labels, uint64_t n) {
  uint64_t pos = 0;
  for (uint64_t i = 0; i < n; ++i) pos += (uint64_t)labels[i];
  const uint64_t neg = n - pos;
  if (pos == 0 || neg == 0) return NAN;
  scored* o = (scored*)malloc(n * sizeof(scored));
  for (uint64_t i = 0; i < n; ++i) { o[i].s = scores[i]; o[i].y = labels[i]; }
  qsort(o, n, sizeof(scored), cmp_scored);
  double prs = 0.0;
  uint64_t i = 0;
  while (i < n) {
    uint64_t j = i;
    while (j < n && o[j].s == o[i].s) ++j;
    const double avg = 0.5 * (double)(i + 1 + j);
    for (uint64_t t = i; t < j; ++t) if (o[t].y == 1) prs += avg;
    i = j;
  }
  free(o);
  const double p = (double)pos, m = (double)neg;
  return (prs - p * (p + 1.0) / 2.0) / (p * m);
}

/* -------------------------------------------------------------- table --- */
/* insert-if-absent store with fresh {w=0, acc=1e-6} (proj/src/store.cpp:153-168,
 * kFreshAccumulator store.hpp:49); sparse Adam: {w=0, m=0, v=eps}. */
typedef struct {
  uint64_t* slot_key;
  uint32_t* slot_row;
  uint64_t nslots, nrows, cap_rows;
  uint64_t* row_key;
  real *w, *s1, *s2;
  uint64_t e;
  int rule; /* 0 adagrad, 1 adam */
  real fresh1, fresh2;
} table;

static uint64_t hmix(uint64_t k) { return FN(splitmix64)(k); }
static void table_init(table* t, uint64_t e, int rule, real fresh1, real fresh2) {
  memset(t, 0, sizeof(*t));
  t->e = e; t->rule = rule; t->fresh1 = fresh1; t->fresh2 = fresh2;
  t->nslots = 1024;
  t->slot_key = (uint64_t*)malloc(t->nslots * 8);
  t->slot_row = (uint32_t*)malloc(t->nslots * 4);
  for (uint64_t i = 0; i < t->nslots; ++i) t->slot_row[i] = UINT32_MAX;
}
static void table_free(table* t) {
  free(t->slot_key); free(t->slot_row); free(t->row_key); free(t->w); free(t->s1); free(t->s2);
}
static int64_t table_find(const table* t, uint64_t key) {
  uint64_t i = hmix(key) & (t->nslots - 1);
  for (;;) {
    if (t->slot_row[i] == UINT32_MAX) return -1;
    if (t->slot_key[i] == key) return t->slot_row[i];
    i = (i + 1) & (t->nslots - 1);
  }
}
static void table_rehash(table* t) {
  uint64_t n2 = t->nslots * 2;
  uint64_t* k2 = (uint64_t*)malloc(n2 * 8);
  uint32_t* r2 = (uint32_t*)malloc(n2 * 4);
  for (uint64_t i = 0; i < n2; ++i) r2[i] = UINT32_MAX;
  for (uint64_t i = 0; i < t->nslots; ++i) {
    if (t->slot_row[i] == UINT32_MAX) continue;
    uint64_t j = hmix(t->slot_key[i]) & (n2 - 1);
    while (r2[j] != UINT32_MAX) j = (j + 1) & (n2 - 1);
    k2[j] = t->slot_key[i]; r2[j] = t->slot_row[i];
  }
  free(t->slot_key); free(t->slot_row);
  t->slot_key = k2; t->slot_row = r2; t->nslots = n2;
}
static uint32_t table_get_or_insert(table* t, uint64_t key) {
  int64_t r = table_find(t, key);
  if (r >= 0) return (uint32_t)r;
  if ((t->nrows + 1) * 2 > t->nslots) table_rehash(t);
  if (t->nrows == t->cap_rows) {
    t->cap_rows = t->cap_rows ? t->cap_rows * 2 : 1024;
    t->row_key = (uint64_t*)realloc(t->row_key, t->cap_rows * 8);
    t->w = (real*)realloc(t->w, t->cap_rows * t->e * sizeof(real));
    t->s1 = (real*)realloc(t->s1, t->cap_rows * t->e * sizeof(real));
    t->s2 = (real*)realloc(t->s2, t->cap_rows * t->e * sizeof(real));
  }
  const uint32_t row = (uint32_t)t->nrows++;
  uint64_t i = hmix(key) & (t->nslots - 1);
  while (t->slot_row[i] != UINT32_MAX) i = (i + 1) & (t->nslots - 1);
  t->slot_key[i] = key; t->slot_row[i] = row;
  t->row_key[row] = key;
  for (uint64_t j = 0; j < t->e; ++j) {
    t->w[row * t->e + j] = 0;
    t->s1[row * t->e + j] = t->fresh1;
    t->s2[row * t->e + j] = t->fresh2;
  }
  return row;
}

/* ------------------------------------------------------------- trainer --- */
typedef struct {
  uint64_t seed, n_workers, minibatch;
  double sparse_lr, alpha, beta1, beta2, eps;
  uint64_t k;
  int32_t reset_v;
  uint64_t emb_dim, n_slots;
  uint64_t hidden[8];
  int32_t n_hidden, activation, pooling, sparse_rule;
  double sparse_beta1, sparse_beta2, sparse_eps;
} orc_config;

typedef struct {
  orc_config c;
  hyper h;
  table tab;
  uint64_t widths[10];
  uint64_t n_layers, in_w, D;
  uint64_t w_off[9], b_off[9];
  wstate* st;
  real* state_buf;
  uint64_t t_global, merges;
  /* cumulative AUC history */
  double* hist_s;
  int32_t* hist_y;
  uint64_t hist_n, hist_cap;
  /* per-row scratch */
  real *wscr, *sscr;
  uint64_t* wstamp;
  uint64_t* sstamp;
  uint64_t scr_rows, stamp;
} trainer;

void* FN(trainer_create)(const orc_config* c) {
  trainer* T = (trainer*)calloc(1, sizeof(trainer));
  T->c = *c;
  T->h.alpha = (real)c->alpha; T->h.beta1 = (real)c->beta1; T->h.beta2 = (real)c->beta2;
  T->h.eps = (real)c->eps; T->h.k = c->k; T->h.reset_v = c->reset_v;
  const uint64_t S = c->n_slots ? c->n_slots : 1;
  T->in_w = S * c->emb_dim;
  T->widths[0] = T->in_w;
  for (int i = 0; i < c->n_hidden; ++i) T->widths[i + 1] = c->hidden[i];
  T->widths[c->n_hidden + 1] = 1;
  T->n_layers = (uint64_t)c->n_hidden + 1;
  /* flat layout: per layer W(out x in, row-major) then bias (model.cpp:55-66) */
  for (uint64_t l = 0; l < T->n_layers; ++l) {
    T->w_off[l] = T->D;
    T->D += T->widths[l] * T->widths[l + 1];
    T->b_off[l] = T->D;
    T->D += T->widths[l + 1];
  }
  double* x0 = (double*)malloc(T->D * 8);
  FN(init_dense)(c->seed, T->D, x0);
  T->st = (wstate*)calloc(c->n_workers, sizeof(wstate));
  T->state_buf = (real*)malloc(c->n_workers * T->D * 4 * sizeof(real));
  for (uint64_t i = 0; i < c->n_workers; ++i) {
    real* b = T->state_buf + i * 4 * T->D;
    T->st[i].x = b; T->st[i].m = b + T->D; T->st[i].v = b + 2 * T->D; T->st[i].vbar = b + 3 * T->D;
    for (uint64_t j = 0; j < T->D; ++j) {
      T->st[i].x[j] = (real)x0[j]; T->st[i].m[j] = 0;
      T->st[i].v[j] = (real)c->eps; T->st[i].vbar[j] = (real)c->eps;
    }
  }
  free(x0);
  if (c->sparse_rule == 0)
    table_init(&T->tab, c->emb_dim, 0, (real)1e-6, 0);
  else
    table_init(&T->tab, c->emb_dim, 1, 0, (real)c->sparse_eps);
  return T;
}

void FN(trainer_destroy)(void* h) {
  trainer* T = (trainer*)h;
  table_free(&T->tab);
  free(T->st); free(T->state_buf); free(T->hist_s); free(T->hist_y);
  free(T->wscr); free(T->sscr); free(T->wstamp); free(T->sstamp);
  free(T);
}

uint64_t FN(trainer_dense_dim)(void* h) { return ((trainer*)h)->D; }
uint64_t FN(trainer_steps)(void* h) { return ((trainer*)h)->t_global; }
uint64_t FN(trainer_merges)(void* h) { return ((trainer*)h)->merges; }

static real sigmoid(real z) {
  if (z >= 0) return (real)1 / ((real)1 + r_exp(-z));
  const real e = r_exp(z);
  return e / ((real)1 + e);
}
static real softplus(real z) { return (z > 0 ? z : (real)0) + r_log1p(r_exp(-r_abs(z))); }

typedef struct {
  uint64_t n;
  real* pooled; /* [n][in_w] */
  real* pre[9];  /* [n][width] */
  real* act[9];
  real* logit;
  real* pred;
} fwd_cache;

static void fwd_free(fwd_cache* f, uint64_t L) {
  free(f->pooled); free(f->logit); free(f->pred);
  for (uint64_t l = 0; l < L; ++l) { free(f->pre[l]); free(f->act[l]); }
}

/* CtrModel::forward (proj/src/model.cpp:76-124) with S slots */
static void forward(trainer* T, const real* x, const uint64_t* offs, const uint64_t* keys,
                    const uint16_t* slots, uint64_t first, uint64_t n, fwd_cache* f) {
  const uint64_t e = T->c.emb_dim, S = T->in_w / e, L = T->n_layers;
  f->n = n;
  f->pooled = (real*)calloc(n * T->in_w, sizeof(real));
  f->logit = (real*)malloc(n * sizeof(real));
  f->pred = (real*)malloc(n * sizeof(real));
  for (uint64_t l = 0; l < L; ++l) {
    f->pre[l] = (real*)calloc(n * T->widths[l + 1], sizeof(real));
    f->act[l] = (real*)calloc(n * T->widths[l + 1], sizeof(real));
  }
  uint64_t cnt[4096];
  for (uint64_t b = 0; b < n; ++b) {
    const uint64_t inst = first + b;
    real* pooled = f->pooled + b * T->in_w;
    for (uint64_t s = 0; s < S; ++s) cnt[s] = 0;
    for (uint64_t o = offs[inst]; o < offs[inst + 1]; ++o) {
      const uint64_t s = slots ? slots[o] : 0;
      const int64_t row = table_find(&T->tab, keys[o]);
      const real* emb = T->tab.w + (uint64_t)row * e;
      for (uint64_t j = 0; j < e; ++j) pooled[s * e + j] += emb[j];
      cnt[s]++;
    }
    if (T->c.pooling == 1)
      for (uint64_t s = 0; s < S; ++s) {
        if (!cnt[s]) continue;
        const real inv = (real)1 / (real)cnt[s];
        for (uint64_t j = 0; j < e; ++j) pooled[s * e + j] *= inv;
      }
    const real* input = pooled;
    for (uint64_t l = 0; l < L; ++l) {
      const uint64_t in_w = T->widths[l], out_w = T->widths[l + 1];
      real* pre = f->pre[l] + b * out_w;
      real* act = f->act[l] + b * out_w;
      for (uint64_t o = 0; o < out_w; ++o) {
        real z = x[T->b_off[l] + o];
        const real* w = x + T->w_off[l] + o * in_w;
        for (uint64_t i = 0; i < in_w; ++i) z += w[i] * input[i];
        pre[o] = z;
        if (l + 1 == L) act[o] = z;
        else act[o] = T->c.activation == 0 ? (z > 0 ? z : (real)0) : r_tanh(z);
      }
      input = act;
    }
    f->logit[b] = f->act[L - 1][b];
    f->pred[b] = sigmoid(f->logit[b]);
  }
}

static void ensure_scratch(trainer* T) {
  if (T->scr_rows >= T->tab.nrows) return;
  uint64_t n = T->tab.cap_rows, e = T->c.emb_dim;
  T->wscr = (real*)realloc(T->wscr, n * e * sizeof(real));
  T->sscr = (real*)realloc(T->sscr, n * e * sizeof(real));
  T->wstamp = (uint64_t*)realloc(T->wstamp, n * 8);
  T->sstamp = (uint64_t*)realloc(T->sstamp, n * 8);
  for (uint64_t i = T->scr_rows; i < n; ++i) T->wstamp[i] = T->sstamp[i] = 0;
  T->scr_rows = n;
}

/* CtrModel::backward (proj/src/model.cpp:137-191). Sparse grads accumulate
 * into wscr rows (stamped `wst`), touched rows appended to `touched`. */
static double backward(trainer* T, const real* x, const uint64_t* offs, const uint64_t* keys,
                       const uint16_t* slots, const int32_t* labels, uint64_t first,
                       const fwd_cache* f, real* dgrad, uint64_t wst, uint32_t* touched,
                       uint64_t* n_touched) {
  const uint64_t n = f->n, L = T->n_layers, e = T->c.emb_dim, S = T->in_w / e;
  for (uint64_t j = 0; j < T->D; ++j) dgrad[j] = 0;
  /* mean_bce (model.cpp:126-135) */
  real loss = 0;
  for (uint64_t b = 0; b < n; ++b) {
    const real z = f->logit[b];
    const real y = (real)labels[first + b];
    loss += softplus(z) - y * z;
  }
  loss = loss / (real)n;
  uint64_t maxw = T->in_w;
  for (uint64_t l = 0; l <= L; ++l) if (T->widths[l] > maxw) maxw = T->widths[l];
  real* delta = (real*)malloc(maxw * sizeof(real));
  real* next = (real*)malloc(maxw * sizeof(real));
  uint64_t cnt[4096];
  for (uint64_t b = 0; b < n; ++b) {
    const uint64_t inst = first + b;
    delta[0] = (f->pred[b] - (real)labels[inst]) / (real)n;
    for (uint64_t l = L; l-- > 0;) {
      const uint64_t in_w = T->widths[l], out_w = T->widths[l + 1];
      const real* input = l == 0 ? f->pooled + b * T->in_w : f->act[l - 1] + b * in_w;
      for (uint64_t j = 0; j < in_w; ++j) next[j] = 0;
      for (uint64_t o = 0; o < out_w; ++o) {
        real dz = delta[o];
        if (l + 1 != L) {
          const real z = f->pre[l][b * out_w + o], y = f->act[l][b * out_w + o];
          dz *= T->c.activation == 0 ? (z > 0 ? (real)1 : (real)0) : (real)1 - y * y;
        }
        dgrad[T->b_off[l] + o] += dz;
        real* wg = dgrad + T->w_off[l] + o * in_w;
        const real* w = x + T->w_off[l] + o * in_w;
        for (uint64_t j = 0; j < in_w; ++j) {
          wg[j] += dz * input[j];
          next[j] += dz * w[j];
        }
      }
      memcpy(delta, next, in_w * sizeof(real));
    }
    /* delta = d loss / d pooled; per-slot coefficient (model.cpp:180-188) */
    for (uint64_t s = 0; s < S; ++s) cnt[s] = 0;
    for (uint64_t o = offs[inst]; o < offs[inst + 1]; ++o) cnt[slots ? slots[o] : 0]++;
    for (uint64_t o = offs[inst]; o < offs[inst + 1]; ++o) {
      const uint64_t s = slots ? slots[o] : 0;
      const real coeff = T->c.pooling == 1 ? (real)1 / (real)cnt[s] : (real)1;
      const uint32_t row = (uint32_t)table_find(&T->tab, keys[o]);
      real* g = T->wscr + (uint64_t)row * e;
      if (T->wstamp[row] != wst) {
        T->wstamp[row] = wst;
        for (uint64_t j = 0; j < e; ++j) g[j] = 0;
        touched[(*n_touched)++] = row;
      }
      for (uint64_t j = 0; j < e; ++j) g[j] += coeff * delta[s * e + j];
    }
  }
  free(delta); free(next);
  return (double)loss;
}

static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}

/* Trainer::process_batch (proj/src/trainer.cpp:115-259). preds (optional)
 * receives the predict-first sigmoid outputs. */
int FN(trainer_batch)(void* h, const uint64_t* offs, const uint64_t* keys, const uint16_t* slots,
                      const int32_t* labels, uint64_t n, int predict_first, double* loss_out,
                      double* auc_out, double* cum_auc_out, double* preds) {
  trainer* T = (trainer*)h;
  const uint64_t N = T->c.n_workers, e = T->c.emb_dim, D = T->D;
  if (n == 0) return 1;
  /* pull: every batch key resolved (inserted) before predict/train */
  for (uint64_t i = 0; i < offs[n]; ++i) table_get_or_insert(&T->tab, keys[i]);
  ensure_scratch(T);
  *auc_out = NAN; *cum_auc_out = NAN;
  if (predict_first) {
    real** xs = (real**)malloc(N * sizeof(real*));
    for (uint64_t i = 0; i < N; ++i) xs[i] = T->st[i].x;
    real* xbar = (real*)malloc(D * sizeof(real));
    cmean(N, D, xs, xbar);
    fwd_cache f;
    forward(T, xbar, offs, keys, slots, 0, n, &f);
    double* sc = (double*)malloc(n * 8);
    for (uint64_t b = 0; b < n; ++b) sc[b] = (double)f.pred[b];
    if (preds) memcpy(preds, sc, n * 8);
    *auc_out = FN(auc)(sc, labels, n);
    if (T->hist_n + n > T->hist_cap) {
      T->hist_cap = (T->hist_n + n) * 2;
      T->hist_s = (double*)realloc(T->hist_s, T->hist_cap * 8);
      T->hist_y = (int32_t*)realloc(T->hist_y, T->hist_cap * 4);
    }
    memcpy(T->hist_s + T->hist_n, sc, n * 8);
    memcpy(T->hist_y + T->hist_n, labels, n * 4);
    T->hist_n += n;
    *cum_auc_out = FN(auc)(T->hist_s, T->hist_y, T->hist_n);
    free(sc); fwd_free(&f, T->n_layers); free(xs); free(xbar);
  }
  /* shard_batch (trainer.cpp:32-53,153-156) */
  const uint64_t per = N * T->c.minibatch;
  uint64_t n_mb = (n + per - 1) / per;
  if (n_mb < 1) n_mb = 1;
  const uint64_t cells = N * n_mb, base = n / cells, extra = n % cells;
  uint64_t* cstart = (uint64_t*)malloc((cells + 1) * 8);
  cstart[0] = 0;
  for (uint64_t c = 0; c < cells; ++c) cstart[c + 1] = cstart[c] + base + (c < extra ? 1 : 0);

  real* dg = (real*)malloc(N * D * sizeof(real));
  real** dgp = (real**)malloc(N * sizeof(real*));
  for (uint64_t i = 0; i < N; ++i) dgp[i] = dg + i * D;
  uint32_t* wtouched = (uint32_t*)malloc((offs[n] + 1) * 4);
  uint32_t* stouched = (uint32_t*)malloc((offs[n] + 1) * 4);
  double batch_total = 0;
  uint64_t batch_count = 0;
  for (uint64_t j = 0; j < n_mb; ++j) {
    double loss_sum = 0;
    uint64_t loss_count = 0, ns = 0;
    const uint64_t sst = ++T->stamp;
    for (uint64_t i = 0; i < N; ++i) {
      const uint64_t c = i * n_mb + j, first = cstart[c], len = cstart[c + 1] - cstart[c];
      if (len == 0) { for (uint64_t q = 0; q < D; ++q) dgp[i][q] = 0; continue; }
      fwd_cache f;
      forward(T, T->st[i].x, offs, keys, slots, first, len, &f);
      uint64_t nw = 0;
      const uint64_t wst = ++T->stamp;
      const double l = backward(T, T->st[i].x, offs, keys, slots, labels, first, &f, dgp[i], wst,
                                wtouched, &nw);
      fwd_free(&f, T->n_layers);
      loss_sum += l * (double)len;
      loss_count += len;
      /* sparse_sum: ascending worker (trainer.cpp:180-186) */
      for (uint64_t q = 0; q < nw; ++q) {
        const uint32_t row = wtouched[q];
        real* s = T->sscr + (uint64_t)row * e;
        const real* g = T->wscr + (uint64_t)row * e;
        if (T->sstamp[row] != sst) {
          T->sstamp[row] = sst;
          for (uint64_t z = 0; z < e; ++z) s[z] = 0;
          stouched[ns++] = row;
        }
        for (uint64_t z = 0; z < e; ++z) s[z] += g[z];
      }
    }
    /* x 1/N then push (trainer.cpp:202-208); per-key independent */
    if (ns) {
      const real inv_n = (real)1 / (real)N;
      qsort(stouched, ns, 4, cmp_u32);
      for (uint64_t q = 0; q < ns; ++q) {
        const uint64_t row = stouched[q];
        real* g = T->sscr + row * e;
        for (uint64_t z = 0; z < e; ++z) g[z] *= inv_n;
        if (T->tab.rule == 0)
          FN(adagrad)(T->tab.w + row * e, T->tab.s1 + row * e, g, e, (real)T->c.sparse_lr);
        else
          FN(sparse_adam)(T->tab.w + row * e, T->tab.s1 + row * e, T->tab.s2 + row * e, g, e,
                          (real)T->c.sparse_lr, (real)T->c.sparse_beta1, (real)T->c.sparse_beta2);
      }
    }
    T->merges += (uint64_t)kstep(T->st, N, D, &T->h, &T->t_global, dgp);
    if (loss_count > 0) {
      batch_total += loss_sum / (double)loss_count;
      batch_count++;
    }
  }
  *loss_out = batch_count ? batch_total / (double)batch_count : NAN;
  free(cstart); free(dg); free(dgp); free(wtouched); free(stouched);
  return 0;
}

int FN(trainer_worker_state)(void* h, uint64_t worker, double* x, double* m, double* v,
                             double* vbar) {
  trainer* T = (trainer*)h;
  if (worker >= T->c.n_workers) return 1;
  for (uint64_t j = 0; j < T->D; ++j) {
    x[j] = T->st[worker].x[j]; m[j] = T->st[worker].m[j];
    v[j] = T->st[worker].v[j]; vbar[j] = T->st[worker].vbar[j];
  }
  return 0;
}

uint64_t FN(trainer_table_size)(void* h) { return ((trainer*)h)->tab.nrows; }

typedef struct { uint64_t key; uint32_t row; } krow;
static int cmp_krow(const void* a, const void* b) {
  uint64_t x = ((const krow*)a)->key, y = ((const krow*)b)->key;
  return x < y ? -1 : x > y;
}
/* full table, ascending key: w and the rule's state (acc | m,v) */
int FN(trainer_table)(void* h, uint64_t* keys, double* w, double* s1, double* s2) {
  trainer* T = (trainer*)h;
  const uint64_t n = T->tab.nrows, e = T->c.emb_dim;
  krow* kr = (krow*)malloc((n + 1) * sizeof(krow));
  for (uint64_t i = 0; i < n; ++i) { kr[i].key = T->tab.row_key[i]; kr[i].row = (uint32_t)i; }
  qsort(kr, n, sizeof(krow), cmp_krow);
  for (uint64_t i = 0; i < n; ++i) {
    keys[i] = kr[i].key;
    for (uint64_t j = 0; j < e; ++j) {
      w[i * e + j] = T->tab.w[(uint64_t)kr[i].row * e + j];
      s1[i * e + j] = T->tab.s1[(uint64_t)kr[i].row * e + j];
      if (s2) s2[i * e + j] = T->tab.s2[(uint64_t)kr[i].row * e + j];
    }
  }
  free(kr);
  return 0;
}
