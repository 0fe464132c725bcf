/*
 * oracle/spardl_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C restatement of the SparDL sparse All-Reduce exactly as the
 * reference implements it in /root/reference/proj/include/spardl/ (*.hpp)
 * (abbreviated `inc/` below).  Every function cites the reference file:line
 * it follows.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library; the product
 * path (paper_2304_00737_b200/) never does.
 *
 * The file is compiled twice (oracle/Makefile):
 *   liboracle_f64.so  ORC_REAL=double -- the reference's own precision; pinned
 *                     bit-exact against oracle/_ref (the unmodified reference
 *                     headers) and against the reference tests' golden values.
 *   liboracle_f32.so  ORC_REAL=float  -- the same algorithm in the GPU's value
 *                     type (fp32 values, IEEE round-to-nearest, no FMA
 *                     contraction: built with -ffp-contract=off), so the CUDA
 *                     path can be checked bit-exactly on ANY input, not only on
 *                     grid-snapped ones.
 * Indices are int64 here (inc/sparse.hpp:27); the device uses int32 (N < 2^31).
 * The alpha-beta audit sums (inc/pipeline.hpp:305-334) and the B-SAG
 * controller (inc/sag.hpp:37-90) stay in double in both builds, as in the
 * reference.
 *
 * Error model: every reference exception class maps to one status code
 * (see include/spardl_cuda.h SPARDL_E_*); the message text is identical.
 */
#include <math.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef ORC_REAL
#define ORC_REAL double
#endif
typedef ORC_REAL real;

#ifdef ORC_F32
#define RABS(x) fabsf(x)
#else
#define RABS(x) fabs(x)
#endif

#define EXPORT __attribute__((visibility("default")))

/* status codes, identical to SPARDL_E_* in include/spardl_cuda.h */
enum {
  E_OK = 0,
  E_ERROR = 1,           /* spardl::error                  inc/error.hpp:23 */
  E_PARTITION = 2,       /* partition_error                inc/error.hpp:29 */
  E_BLOCK_MISMATCH = 3,  /* block_mismatch_error           inc/error.hpp:35 */
  E_SCHEDULE = 4,        /* schedule_violation_error       inc/error.hpp:41 */
  E_THEOREM = 5,         /* theorem_violation_error        inc/error.hpp:47 */
  E_GROUP_SIZE = 6,      /* group_size_error               inc/error.hpp:53 */
  E_CONFIG = 7,          /* config_error                   inc/error.hpp:60 */
  E_STATE = 8,           /* state_error                    inc/error.hpp:66 */
  E_CONSISTENCY = 9      /* consistency_error              inc/error.hpp:72 */
};

/* ------------------------------------------------------------------ */
/* exceptions-by-longjmp and a per-call arena                          */
/* ------------------------------------------------------------------ */
static __thread char g_msg[512];
static __thread jmp_buf *g_jmp;

typedef struct arena_node { struct arena_node *next; } arena_node;
static __thread arena_node *g_arena;

static void *amalloc(size_t bytes) {
  arena_node *n = (arena_node *)malloc(sizeof(arena_node) + (bytes ? bytes : 1));
  if (!n) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
  n->next = g_arena;
  g_arena = n;
  return (void *)(n + 1);
}
static void arena_release(void) {
  while (g_arena) { arena_node *n = g_arena->next; free(g_arena); g_arena = n; }
}

__attribute__((noreturn, format(printf, 2, 3)))
static void throw_err(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_msg, sizeof g_msg, fmt, ap);
  va_end(ap);
  longjmp(*g_jmp, code);
}

/* Every exported entry point brackets its body with API_BEGIN / API_END. */
#define API_BEGIN                       \
  jmp_buf jb__;                         \
  jmp_buf *prev__ = g_jmp;              \
  arena_node *arena_prev__ = g_arena;   \
  g_arena = NULL;                       \
  int rc__ = setjmp(jb__);              \
  if (rc__ != 0) {                      \
    arena_release();                    \
    g_arena = arena_prev__;             \
    g_jmp = prev__;                     \
    return rc__;                        \
  }                                     \
  g_jmp = &jb__;                        \
  g_msg[0] = 0;
#define API_END          \
  arena_release();       \
  g_arena = arena_prev__; \
  g_jmp = prev__;        \
  return E_OK;

EXPORT const char *orc_last_error(void) { return g_msg; }

/* ------------------------------------------------------------------ */
/* inc/mathutil.hpp:21-44                                               */
/* ------------------------------------------------------------------ */
static int is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }
static int ceil_log2(int64_t x) {        /* inc/mathutil.hpp:26-34 */
  int t = 0;
  int64_t v = 1;
  while (v < x) { v <<= 1; ++t; }
  return t;
}
static int exact_log2(int64_t x) {       /* inc/mathutil.hpp:37-44 */
  int t = 0;
  while (x > 1) { x >>= 1; ++t; }
  return t;
}

/* ------------------------------------------------------------------ */
/* inc/sparse.hpp -- SparseBlock, partition, top-k, merge_add, scale    */
/* ------------------------------------------------------------------ */
typedef struct {
  int block_id;
  int64_t lo, hi;   /* IndexRange */
  int64_t n;        /* nnz */
  int64_t *idx;
  real *val;
} blk;

static blk blk_new(int id, int64_t lo, int64_t hi, int64_t cap) {
  blk b;
  b.block_id = id; b.lo = lo; b.hi = hi; b.n = 0;
  b.idx = (int64_t *)amalloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
  b.val = (real *)amalloc(sizeof(real) * (size_t)(cap > 0 ? cap : 1));
  return b;
}
static blk blk_copy(const blk *s) {
  blk b = blk_new(s->block_id, s->lo, s->hi, s->n);
  b.n = s->n;
  memcpy(b.idx, s->idx, sizeof(int64_t) * (size_t)s->n);
  memcpy(b.val, s->val, sizeof(real) * (size_t)s->n);
  return b;
}

typedef struct { int64_t n; int count; int64_t *lo, *hi; } partition_t;

/* inc/sparse.hpp:98-117 */
static partition_t make_partition(int64_t n, int count) {
  if (count <= 0 || (int64_t)count > n)
    throw_err(E_PARTITION, "partition requires 1 <= B <= N, got B=%d N=%lld", count,
              (long long)n);
  partition_t p;
  p.n = n; p.count = count;
  p.lo = (int64_t *)amalloc(sizeof(int64_t) * (size_t)count);
  p.hi = (int64_t *)amalloc(sizeof(int64_t) * (size_t)count);
  const int64_t base = n / count, rem = n % count;
  int64_t lo = 0;
  for (int b = 0; b < count; ++b) {
    const int64_t len = base + (b < rem ? 1 : 0);
    p.lo[b] = lo; p.hi[b] = lo + len; lo += len;
  }
  return p;
}

/* inc/sparse.hpp:88-95 */
static int block_of(const partition_t *p, int64_t i) {
  const int64_t base = p->n / p->count, rem = p->n % p->count;
  const int64_t split = rem * (base + 1);
  if (i < split) return (int)(i / (base + 1));
  return (int)(rem + (i - split) / base);
}

/* selection order: |v| desc, index asc -- inc/sparse.hpp:122-127 */
typedef struct { real a; int64_t i; } keyed;
static inline int before(const keyed *x, const keyed *y) {
  if (x->a != y->a) return x->a > y->a;
  return x->i < y->i;
}
static inline void kswap(keyed *a, keyed *b) { keyed t = *a; *a = *b; *b = t; }

/* Places the element of rank `k` (in selection order) at a[k].  The order is
 * total (indices are unique), so the result is deterministic; this plays the
 * role of std::nth_element at inc/sparse.hpp:151. */
static void nth_select(keyed *a, int64_t n, int64_t k) {
  int64_t lo = 0, hi = n - 1;
  while (hi > lo) {
    const int64_t mid = lo + (hi - lo) / 2;
    /* median of three -> a[mid] */
    if (before(&a[mid], &a[lo])) kswap(&a[mid], &a[lo]);
    if (before(&a[hi], &a[lo])) kswap(&a[hi], &a[lo]);
    if (before(&a[hi], &a[mid])) kswap(&a[hi], &a[mid]);
    const keyed p = a[mid];
    int64_t i = lo, j = hi;
    while (i <= j) {
      while (before(&a[i], &p)) ++i;
      while (before(&p, &a[j])) --j;
      if (i <= j) { kswap(&a[i], &a[j]); ++i; --j; }
    }
    if (k <= j) hi = j;
    else if (k >= i) lo = i;
    else return;
  }
}

/* inc/sparse.hpp:136-162.  Input entries are index-sorted (SparseBlock
 * invariant, inc/sparse.hpp:64-66), so classifying them in input order against
 * the rank-(budget-1) element yields the two index-sorted outputs that the
 * reference obtains with nth_element + two index sorts. */
static void top_k(const blk *in, int64_t budget, blk *sel, blk *disc) {
  if (budget < 0) throw_err(E_ERROR, "top_k_select: negative budget");
  *sel = blk_new(in->block_id, in->lo, in->hi, in->n);
  *disc = blk_new(in->block_id, in->lo, in->hi, in->n);
  if (budget >= in->n) {
    sel->n = in->n;
    memcpy(sel->idx, in->idx, sizeof(int64_t) * (size_t)in->n);
    memcpy(sel->val, in->val, sizeof(real) * (size_t)in->n);
    return;
  }
  keyed thr = {0, 0};
  if (budget > 0) {
    keyed *order = (keyed *)malloc(sizeof(keyed) * (size_t)in->n);
    if (!order) throw_err(E_ERROR, "oracle: out of memory");
    for (int64_t e = 0; e < in->n; ++e) { order[e].a = RABS(in->val[e]); order[e].i = in->idx[e]; }
    nth_select(order, in->n, budget - 1);
    thr = order[budget - 1];
    free(order);
  }
  for (int64_t e = 0; e < in->n; ++e) {
    keyed x = {RABS(in->val[e]), in->idx[e]};
    const int take = budget > 0 && !before(&thr, &x);
    blk *dst = take ? sel : disc;
    dst->idx[dst->n] = in->idx[e];
    dst->val[dst->n] = in->val[e];
    dst->n++;
  }
}

/* inc/sparse.hpp:167-177 -- every index of the slice is an entry (zeros too). */
static void top_k_slice(const real *g, int id, int64_t lo, int64_t hi, int64_t budget,
                        blk *sel, blk *disc) {
  blk dense = blk_new(id, lo, hi, hi - lo);
  for (int64_t i = lo; i < hi; ++i) { dense.idx[dense.n] = i; dense.val[dense.n] = g[i]; dense.n++; }
  top_k(&dense, budget, sel, disc);
}

/* inc/sparse.hpp:182-208 -- exact zero sums are retained. */
static blk merge_add(const blk *a, const blk *b) {
  if (a->block_id != b->block_id)
    throw_err(E_BLOCK_MISMATCH, "merge_add: block ids differ (%d vs %d)", a->block_id,
              b->block_id);
  blk out = blk_new(a->block_id, a->lo, a->hi, a->n + b->n);
  int64_t ia = 0, ib = 0;
  while (ia < a->n && ib < b->n) {
    if (a->idx[ia] < b->idx[ib]) {
      out.idx[out.n] = a->idx[ia]; out.val[out.n] = a->val[ia]; ++ia;
    } else if (b->idx[ib] < a->idx[ia]) {
      out.idx[out.n] = b->idx[ib]; out.val[out.n] = b->val[ib]; ++ib;
    } else {
      out.idx[out.n] = a->idx[ia]; out.val[out.n] = a->val[ia] + b->val[ib]; ++ia; ++ib;
    }
    out.n++;
  }
  for (; ia < a->n; ++ia, ++out.n) { out.idx[out.n] = a->idx[ia]; out.val[out.n] = a->val[ia]; }
  for (; ib < b->n; ++ib, ++out.n) { out.idx[out.n] = b->idx[ib]; out.val[out.n] = b->val[ib]; }
  return out;
}

/* inc/sparse.hpp:211-215 (factor is a dyadic share, exact in fp32 too). */
static blk scale_blk(const blk *in, double factor) {
  blk out = blk_copy(in);
  for (int64_t e = 0; e < out.n; ++e) out.val[e] = (real)(out.val[e] * (real)factor);
  return out;
}

/* ------------------------------------------------------------------ */
/* inc/fabric.hpp:54-134 -- lockstep rounds + alpha-beta ledger         */
/* ------------------------------------------------------------------ */
typedef struct { int64_t rounds, scalars; } wcost;
typedef struct {
  int has;
  int target;
  int nblk;
  blk *payload;
} send_t;
typedef struct { int nblk; blk *blocks; } inbox_t;

typedef struct { int p; wcost *cost; } fabric_t;

/* inc/fabric.hpp:74-108 */
static inbox_t *fabric_exchange(fabric_t *f, send_t *plan) {
  const int p = f->p;
  inbox_t *inbox = (inbox_t *)amalloc(sizeof(inbox_t) * (size_t)p);
  char *targeted = (char *)amalloc((size_t)p);
  char *part = (char *)amalloc((size_t)p);
  memset(inbox, 0, sizeof(inbox_t) * (size_t)p);
  memset(targeted, 0, (size_t)p);
  memset(part, 0, (size_t)p);
  for (int s = 0; s < p; ++s) {
    if (!plan[s].has) continue;
    const int t = plan[s].target;
    if (t < 0 || t >= p) throw_err(E_SCHEDULE, "message target out of range: %d", t);
    if (targeted[t]) throw_err(E_SCHEDULE, "two messages target worker %d in one round", t);
    targeted[t] = 1; part[s] = 1; part[t] = 1;
    int64_t volume = 0;
    for (int b = 0; b < plan[s].nblk; ++b) volume += 2 * plan[s].payload[b].n;
    f->cost[t].scalars += volume;
    inbox[t].nblk = plan[s].nblk;
    inbox[t].blocks = plan[s].payload;
  }
  for (int w = 0; w < p; ++w) if (part[w]) f->cost[w].rounds += 1;
  return inbox;
}

static wcost *ledger_snapshot(const fabric_t *f) {
  wcost *s = (wcost *)amalloc(sizeof(wcost) * (size_t)f->p);
  memcpy(s, f->cost, sizeof(wcost) * (size_t)f->p);
  return s;
}
/* inc/fabric.hpp:124-134 */
static wcost delta_since(const fabric_t *f, const wcost *snap) {
  wcost d = {0, 0};
  for (int w = 0; w < f->p; ++w) {
    const int64_t r = f->cost[w].rounds - snap[w].rounds;
    const int64_t s = f->cost[w].scalars - snap[w].scalars;
    if (r > d.rounds) d.rounds = r;
    if (s > d.scalars) d.scalars = s;
  }
  return d;
}

/* ------------------------------------------------------------------ */
/* inc/collectives.hpp:46-114 -- Bruck all-gather over several groups  */
/* ------------------------------------------------------------------ */
typedef struct { int m; const int *workers; const blk *blocks; } group_gather;

/* returns out[g][i*m + s] = block of source s as held by member i */
static blk **bruck_multi(fabric_t *f, const group_gather *groups, int ngroups) {
  blk ***buf = (blk ***)amalloc(sizeof(blk **) * (size_t)ngroups);
  int **cnt = (int **)amalloc(sizeof(int *) * (size_t)ngroups);
  int max_steps = 0;
  for (int g = 0; g < ngroups; ++g) {
    const int m = groups[g].m;
    if (m == 0) throw_err(E_GROUP_SIZE, "all-gather on empty group");
    buf[g] = (blk **)amalloc(sizeof(blk *) * (size_t)m);
    cnt[g] = (int *)amalloc(sizeof(int) * (size_t)m);
    for (int i = 0; i < m; ++i) {
      buf[g][i] = (blk *)amalloc(sizeof(blk) * (size_t)m);
      buf[g][i][0] = groups[g].blocks[i];
      cnt[g][i] = 1;
    }
    const int st = ceil_log2(m);
    if (st > max_steps) max_steps = st;
  }
  for (int t = 0; t < max_steps; ++t) {
    const int dist = 1 << t;
    send_t *plan = (send_t *)amalloc(sizeof(send_t) * (size_t)f->p);
    memset(plan, 0, sizeof(send_t) * (size_t)f->p);
    for (int g = 0; g < ngroups; ++g) {
      const int m = groups[g].m;
      if (dist >= m) continue;
      const int count = dist < m - dist ? dist : m - dist;
      for (int i = 0; i < m; ++i) {
        const int target = (i - dist + m) % m;
        send_t *s = &plan[groups[g].workers[i]];
        s->has = 1;
        s->target = groups[g].workers[target];
        s->nblk = count;
        s->payload = (blk *)amalloc(sizeof(blk) * (size_t)count);
        for (int c = 0; c < count; ++c) s->payload[c] = buf[g][i][c];
      }
    }
    inbox_t *inbox = fabric_exchange(f, plan);
    for (int g = 0; g < ngroups; ++g) {
      const int m = groups[g].m;
      if (dist >= m) continue;
      for (int i = 0; i < m; ++i) {
        inbox_t *in = &inbox[groups[g].workers[i]];
        for (int c = 0; c < in->nblk; ++c) buf[g][i][cnt[g][i]++] = in->blocks[c];
      }
    }
  }
  blk **out = (blk **)amalloc(sizeof(blk *) * (size_t)ngroups);
  for (int g = 0; g < ngroups; ++g) {
    const int m = groups[g].m;
    out[g] = (blk *)amalloc(sizeof(blk) * (size_t)m * (size_t)m);
    for (int i = 0; i < m; ++i)
      for (int t = 0; t < m; ++t) out[g][i * m + (i + t) % m] = buf[g][i][t];
  }
  return out;
}

/* ------------------------------------------------------------------ */
/* inc/reduce_scatter.hpp:40-74 -- bag schedule                         */
/* ------------------------------------------------------------------ */
typedef struct {
  int m, rank, l, preservation, remainder;
  int *bag_size;    /* [l] */
  int **bag;        /* bag[j-1][s] */
} bags_t;

static bags_t build_bags(int m, int rank) {
  if (m < 1 || rank < 0 || rank >= m) throw_err(E_CONFIG, "build_bags: rank out of range");
  bags_t s;
  s.m = m; s.rank = rank; s.preservation = rank; s.l = ceil_log2(m);
  s.remainder = 0; s.bag_size = NULL; s.bag = NULL;
  if (m == 1) return s;
  s.remainder = m - (1 << (s.l - 1));
  s.bag_size = (int *)amalloc(sizeof(int) * (size_t)s.l);
  s.bag = (int **)amalloc(sizeof(int *) * (size_t)s.l);
  int next = rank + 1;
  for (int j = 1; j <= s.l; ++j) {
    const int size = (j < s.l) ? (1 << (j - 1)) : s.remainder;
    s.bag_size[j - 1] = size;
    s.bag[j - 1] = (int *)amalloc(sizeof(int) * (size_t)size);
    for (int q = 0; q < size; ++q) { s.bag[j - 1][q] = next % m; ++next; }
  }
  return s;
}

/* ------------------------------------------------------------------ */
/* inc/residual.hpp:52-177 -- ResidualStore                              */
/* ------------------------------------------------------------------ */
enum { RES_GRES = 0, RES_PRES = 1, RES_LRES = 2 };
typedef struct {
  int mode;
  int64_t n;
  real *carry;          /* persistent across iterations */
  /* per-iteration (arena) state */
  real *g_copy;
  real *div_rem;
  blk *xi;
  partition_t part;
  int in_iter;
} rstore;

static void require_in_iteration(const rstore *s, const char *op) {
  if (!s->in_iter) throw_err(E_STATE, "%s outside an iteration", op);
}

/* inc/residual.hpp:63-71 */
static real *rs_apply(rstore *s, const real *g) {
  real *combined = (real *)amalloc(sizeof(real) * (size_t)s->n);
  for (int64_t i = 0; i < s->n; ++i) combined[i] = g[i] + s->carry[i];
  memset(s->carry, 0, sizeof(real) * (size_t)s->n);
  return combined;
}

/* inc/residual.hpp:75-92 */
static void rs_begin(rstore *s, const real *combined, const partition_t *part) {
  if (s->in_iter) throw_err(E_STATE, "begin_iteration called twice without finalize");
  if (part->n != s->n) throw_err(E_CONFIG, "begin_iteration: dimension mismatch");
  s->g_copy = (real *)amalloc(sizeof(real) * (size_t)s->n);
  memcpy(s->g_copy, combined, sizeof(real) * (size_t)s->n);
  s->part = *part;
  s->xi = (blk *)amalloc(sizeof(blk) * (size_t)part->count);
  for (int b = 0; b < part->count; ++b) s->xi[b] = blk_new(b, part->lo[b], part->hi[b], 0);
  s->div_rem = (real *)amalloc(sizeof(real) * (size_t)s->n);
  memset(s->div_rem, 0, sizeof(real) * (size_t)s->n);
  s->in_iter = 1;
}

/* inc/residual.hpp:96-99 */
static void rs_record_dividing_remainder(rstore *s, const blk *rem) {
  require_in_iteration(s, "record_dividing_remainder");
  for (int64_t e = 0; e < rem->n; ++e) s->div_rem[rem->idx[e]] = rem->val[e];
}

/* inc/residual.hpp:104-124 */
static void rs_record_inproc(rstore *s, int block_id, const blk *disc, double weight) {
  require_in_iteration(s, "record_inproc");
  if (block_id < 0 || block_id >= s->part.count)
    throw_err(E_CONFIG, "record_inproc: unknown block id");
  if (weight <= 0.0 || weight > 1.0)
    throw_err(E_CONFIG, "record_inproc: weight must be in (0, 1]");
  blk *acc = &s->xi[block_id];
  for (int64_t e = 0; e < disc->n; ++e)
    if (!(disc->idx[e] >= acc->lo && disc->idx[e] < acc->hi))
      throw_err(E_CONFIG, "record_inproc: index %lld outside block range",
                (long long)disc->idx[e]);
  blk scaled = scale_blk(disc, weight);
  scaled.block_id = block_id;
  scaled.lo = acc->lo; scaled.hi = acc->hi;
  *acc = merge_add(acc, &scaled);
}

/* inc/residual.hpp:153-160 */
static real rs_xi_value(const rstore *s, int64_t index) {
  const blk *acc = &s->xi[block_of(&s->part, index)];
  int64_t lo = 0, hi = acc->n;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (acc->idx[mid] < index) lo = mid + 1; else hi = mid;
  }
  if (lo < acc->n && acc->idx[lo] == index) return acc->val[lo];
  return (real)0.0;
}

/* inc/residual.hpp:128-150 */
static void rs_finalize(rstore *s, const int64_t *gidx, int64_t gnnz) {
  require_in_iteration(s, "finalize");
  switch (s->mode) {
    case RES_GRES: {
      memcpy(s->carry, s->g_copy, sizeof(real) * (size_t)s->n);
      for (int64_t e = 0; e < gnnz; ++e) s->carry[gidx[e]] = rs_xi_value(s, gidx[e]);
      break;
    }
    case RES_PRES: {
      memcpy(s->carry, s->g_copy, sizeof(real) * (size_t)s->n);
      for (int64_t e = 0; e < gnnz; ++e) s->carry[gidx[e]] = (real)0.0;
      break;
    }
    case RES_LRES: {
      memcpy(s->carry, s->div_rem, sizeof(real) * (size_t)s->n);
      break;
    }
  }
  s->in_iter = 0;
}

/* ------------------------------------------------------------------ */
/* inc/sag.hpp:37-90 -- HController (Algorithm 2), double precision    */
/* ------------------------------------------------------------------ */
typedef struct {
  double lower, upper;
  int64_t target;
  double h, step;
  int32_t flag;
  int32_t pad_;
} orc_hctrl;

static void hctrl_init(orc_hctrl *c, int64_t workers, int64_t k, int64_t teams) {
  /* member initialisers run before the validity check, exactly as the
   * reference constructor does (inc/sag.hpp:40-52) */
  if (workers < 1 || teams < 1 || k < 1 || k % workers != 0 || (teams * k) % workers != 0)
    throw_err(E_CONFIG, "HController: invalid (P, k, d)");
  c->lower = (double)k / (double)workers;
  c->upper = (double)(teams * k) / (double)workers;
  c->target = teams * k / workers;
  c->h = c->lower;
  c->step = 0.01 * (double)k * (double)(teams - 1) / (double)workers;
  c->flag = 0;
  c->pad_ = 0;
}
/* inc/sag.hpp:61-63 */
static int64_t hctrl_budget(const orc_hctrl *c) {
  const int64_t r = (int64_t)llround(c->h);
  return r > 1 ? r : 1;
}
/* inc/sag.hpp:66-81 */
static void hctrl_observe(orc_hctrl *c, int64_t n_t) {
  const int over = n_t > c->target;
  const int rising = c->step > 0.0;
  if (over != rising) {
    if (c->flag) { c->step *= 2.0; c->flag = 0; }
    else c->flag = 1;
  } else {
    c->step = -c->step / 2.0;
    c->flag = 0;
  }
  double v = c->h + c->step;
  if (v < c->lower) v = c->lower;
  else if (c->upper < v) v = c->upper;
  c->h = v;
}

/* inc/sag.hpp:108-118 */
static int cmp_desc(const void *a, const void *b) {
  const double x = *(const double *)a, y = *(const double *)b;
  return (x < y) - (x > y);
}
static double *dyadic_shares(int count) {
  double *s = (double *)amalloc(sizeof(double) * (size_t)(count > 1 ? count : 1));
  int n = 1;
  s[0] = 1.0;
  while (n < count) {
    const double half = s[0] / 2.0;
    memmove(s, s + 1, sizeof(double) * (size_t)(n - 1));
    n -= 1;
    s[n++] = half;
    s[n++] = half;
    qsort(s, (size_t)n, sizeof(double), cmp_desc);
  }
  return s;
}

/* ------------------------------------------------------------------ */
/* discard sink -> ResidualStore::record_inproc, inc/pipeline.hpp:155-160 */
/* ------------------------------------------------------------------ */
typedef struct { rstore *stores; } sink_t;
static void on_discard(sink_t *sk, int worker, int block_id, const blk *d, double w) {
  if (sk && sk->stores) rs_record_inproc(&sk->stores[worker], block_id, d, w);
}

/* inc/reduce_scatter.hpp:102-110 */
static void sparsify_slot(blk *slot, int has, int64_t budget, int worker, sink_t *sk) {
  if (!has || slot->n <= budget) return;
  blk sel, disc;
  top_k(slot, budget, &sel, &disc);
  if (disc.n > 0) on_discard(sk, worker, disc.block_id, &disc, 1.0);
  *slot = sel;
}

/* ------------------------------------------------------------------ */
/* inc/reduce_scatter.hpp:120-236 -- Spar-Reduce-Scatter over teams     */
/* blocks[t][i*m + b] = member i of team t, position b.  Returns the    */
/* reserved (preservation) block per team member: out[t][i].             */
/* ------------------------------------------------------------------ */
enum { TIMING_OPT = 0, TIMING_NAIVE = 1 };

static blk **run_srs_teams(fabric_t *f, int nteams, int m, int **workers, blk **blocks,
                           int64_t budget, int timing, sink_t *sk) {
  if (nteams < 1) throw_err(E_GROUP_SIZE, "reduce-scatter with no teams");
  const int l = ceil_log2(m);
  bags_t **sched = (bags_t **)amalloc(sizeof(bags_t *) * (size_t)nteams);
  blk **held = (blk **)amalloc(sizeof(blk *) * (size_t)nteams);
  char **has = (char **)amalloc(sizeof(char *) * (size_t)nteams);
  for (int t = 0; t < nteams; ++t) {
    sched[t] = (bags_t *)amalloc(sizeof(bags_t) * (size_t)m);
    held[t] = (blk *)amalloc(sizeof(blk) * (size_t)m * (size_t)m);
    has[t] = (char *)amalloc((size_t)m * (size_t)m);
    for (int i = 0; i < m; ++i) {
      sched[t][i] = build_bags(m, i);
      for (int b = 0; b < m; ++b) {
        const blk *bl = &blocks[t][i * m + b];
        if (bl->n > budget)
          throw_err(E_CONFIG,
                    "reduce-scatter: initial block exceeds budget; sparsify during dividing "
                    "first");
        held[t][i * m + b] = *bl;
        has[t][i * m + b] = 1;
      }
    }
  }
  for (int step = 1; step <= l; ++step) {
    const int dist = 1 << (l - step);
    const int bag_index = l - step + 1;
    send_t *plan = (send_t *)amalloc(sizeof(send_t) * (size_t)f->p);
    memset(plan, 0, sizeof(send_t) * (size_t)f->p);
    for (int t = 0; t < nteams; ++t) {
      for (int i = 0; i < m; ++i) {
        const bags_t *s = &sched[t][i];
        const int bs = s->bag_size[bag_index - 1];
        send_t *snd = &plan[workers[t][i]];
        snd->has = 1;
        snd->target = workers[t][(i + dist) % m];
        snd->nblk = bs;
        snd->payload = (blk *)amalloc(sizeof(blk) * (size_t)bs);
        for (int q = 0; q < bs; ++q) {
          const int pos = s->bag[bag_index - 1][q];
          if (!has[t][i * m + pos]) throw_err(E_THEOREM, "sending a block already given up");
          if (held[t][i * m + pos].n > budget)
            throw_err(E_ERROR, "budget discipline violated before send");
          snd->payload[q] = held[t][i * m + pos];
          has[t][i * m + pos] = 0;
        }
      }
    }
    inbox_t *inbox = fabric_exchange(f, plan);
    for (int t = 0; t < nteams; ++t) {
      for (int i = 0; i < m; ++i) {
        const int self = workers[t][i];
        inbox_t *in = &inbox[self];
        for (int q = 0; q < in->nblk; ++q) {
          const blk *rcv = &in->blocks[q];
          if (rcv->block_id < 0 || rcv->block_id >= m)
            throw_err(E_THEOREM, "received block id out of range");
          if (!has[t][i * m + rcv->block_id])
            throw_err(E_THEOREM, "received block %d not held by worker %d", rcv->block_id,
                      self);
          held[t][i * m + rcv->block_id] = merge_add(&held[t][i * m + rcv->block_id], rcv);
        }
        if (timing == TIMING_NAIVE) {
          for (int b = 0; b < m; ++b)
            sparsify_slot(&held[t][i * m + b], has[t][i * m + b], budget, self, sk);
        } else if (step < l) {
          const bags_t *s = &sched[t][i];
          for (int q = 0; q < s->bag_size[bag_index - 2]; ++q) {
            const int pos = s->bag[bag_index - 2][q];
            sparsify_slot(&held[t][i * m + pos], has[t][i * m + pos], budget, self, sk);
          }
        }
      }
    }
  }
  blk **out = (blk **)amalloc(sizeof(blk *) * (size_t)nteams);
  for (int t = 0; t < nteams; ++t) {
    out[t] = (blk *)amalloc(sizeof(blk) * (size_t)m);
    for (int i = 0; i < m; ++i) {
      const int self = workers[t][i];
      const int p = sched[t][i].preservation;
      if (!has[t][i * m + p]) throw_err(E_ERROR, "preservation block missing after reduce-scatter");
      sparsify_slot(&held[t][i * m + p], 1, budget, self, sk);
      out[t][i] = held[t][i * m + p];
    }
  }
  return out;
}

/* ------------------------------------------------------------------ */
/* inc/sag.hpp:125-173 -- R-SAG over position groups                    */
/* gblocks[g][i]: block of member i (team i) of position group g        */
/* ------------------------------------------------------------------ */
static void rsag_groups(fabric_t *f, int ngroups, int d, int **gworkers, blk **gblocks,
                        int64_t budget, sink_t *sk) {
  if (ngroups < 1) throw_err(E_GROUP_SIZE, "rsag with no groups");
  if (d < 2 || !is_pow2(d)) throw_err(E_GROUP_SIZE, "rsag requires a power-of-two team count >= 2");
  const int steps = exact_log2(d);
  for (int t = 0; t < steps; ++t) {
    const int dist = 1 << t;
    send_t *plan = (send_t *)amalloc(sizeof(send_t) * (size_t)f->p);
    memset(plan, 0, sizeof(send_t) * (size_t)f->p);
    for (int g = 0; g < ngroups; ++g)
      for (int i = 0; i < d; ++i) {
        send_t *s = &plan[gworkers[g][i]];
        s->has = 1;
        s->target = gworkers[g][i ^ dist];
        s->nblk = 1;
        s->payload = (blk *)amalloc(sizeof(blk));
        s->payload[0] = gblocks[g][i];
      }
    inbox_t *inbox = fabric_exchange(f, plan);
    const double share = 1.0 / (double)(2 * dist);
    for (int g = 0; g < ngroups; ++g)
      for (int i = 0; i < d; ++i) {
        const int self = gworkers[g][i];
        inbox_t *in = &inbox[self];
        if (in->nblk < 1) throw_err(E_ERROR, "rsag: missing partner block");
        blk merged = merge_add(&gblocks[g][i], &in->blocks[0]);
        if (merged.n > budget) {
          blk sel, disc;
          top_k(&merged, budget, &sel, &disc);
          on_discard(sk, self, disc.block_id, &disc, share);
          merged = sel;
        }
        gblocks[g][i] = merged;
      }
  }
}

/* ------------------------------------------------------------------ */
/* inc/sag.hpp:189-249 -- B-SAG over position groups                    */
/* ------------------------------------------------------------------ */
static void bsag_groups(fabric_t *f, int ngroups, int d, int **gworkers, blk **gblocks,
                        const int64_t *pre_budgets, int64_t budget, sink_t *sk,
                        int64_t *union_sizes) {
  if (ngroups < 1) throw_err(E_GROUP_SIZE, "bsag with no groups");
  if (d < 2) throw_err(E_GROUP_SIZE, "bsag requires >= 2 teams");
  group_gather *gg = (group_gather *)amalloc(sizeof(group_gather) * (size_t)ngroups);
  for (int g = 0; g < ngroups; ++g) {
    blk *pre = (blk *)amalloc(sizeof(blk) * (size_t)d);
    for (int i = 0; i < d; ++i) {
      blk b = gblocks[g][i];
      if (b.n > pre_budgets[g]) {
        blk sel, disc;
        top_k(&b, pre_budgets[g], &sel, &disc);
        on_discard(sk, gworkers[g][i], disc.block_id, &disc, 1.0);
        b = sel;
      }
      pre[i] = b;
    }
    gg[g].m = d; gg[g].workers = gworkers[g]; gg[g].blocks = pre;
  }
  blk **gathered = bruck_multi(f, gg, ngroups);
  double *shares = dyadic_shares(d);
  for (int g = 0; g < ngroups; ++g) {
    for (int i = 0; i < d; ++i) {
      blk acc = gathered[g][i * d + 0];
      for (int s = 1; s < d; ++s) acc = merge_add(&acc, &gathered[g][i * d + s]);
      union_sizes[g] = acc.n;
      if (acc.n > budget) {
        blk sel, disc;
        top_k(&acc, budget, &sel, &disc);
        on_discard(sk, gworkers[g][i], disc.block_id, &disc, shares[i]);
        acc = sel;
      }
      gblocks[g][i] = acc;
    }
  }
}

/* ------------------------------------------------------------------ */
/* inc/sag.hpp:295-346, inc/reduce_scatter.hpp:257-262 -- closed forms  */
/* ------------------------------------------------------------------ */
enum { SAG_NONE = 0, SAG_RSAG = 1, SAG_BSAG = 2 };

static void expected_cost_sag(int64_t workers, int64_t k, int64_t teams, int mode,
                              int64_t *rounds, int64_t *low, int64_t *high) {
  if (workers < 1 || k < 1 || k % workers != 0)
    throw_err(E_CONFIG, "expected_cost_sag: k must be divisible by P");
  if (teams < 1 || workers % teams != 0) throw_err(E_CONFIG, "expected_cost_sag: d must divide P");
  const int64_t c = k / workers, p = workers, d = teams;
  switch (mode) {
    case SAG_NONE: {
      if (d != 1) throw_err(E_CONFIG, "expected_cost_sag: none requires d=1");
      const int64_t sc = 4 * c * (p - 1);
      *rounds = 2 * ceil_log2(p); *low = sc; *high = sc;
      return;
    }
    case SAG_RSAG: {
      if (d < 2 || !is_pow2(d)) throw_err(E_CONFIG, "rsag requires power-of-two d");
      const int64_t lg = exact_log2(d);
      const int64_t sc = 2 * c * (2 * p - 2 * d) + 2 * c * d * lg;
      *rounds = 2 * ceil_log2(p / d) + lg; *low = sc; *high = sc;
      return;
    }
    case SAG_BSAG: {
      if (d < 2) throw_err(E_CONFIG, "bsag requires d >= 2");
      const int64_t m = p / d;
      *rounds = 2 * ceil_log2(m) + ceil_log2(d);
      *low = 2 * c * (d + m - 2);
      *high = 2 * c * (d * d + 2 * p - 3 * d);
      return;
    }
  }
  throw_err(E_CONFIG, "expected_cost_sag: unknown mode");
}

/* ------------------------------------------------------------------ */
/* inc/pipeline.hpp:39-99 -- ClusterConfig, validate                    */
/* ------------------------------------------------------------------ */
typedef struct {
  int64_t workers, dimension, k, teams;
  int32_t sag, residual, timing, pad_;
  uint64_t seed;
} orc_config;

static void validate(const orc_config *c) {
  if (c->workers < 1) throw_err(E_CONFIG, "P must be >= 1");
  if (c->dimension < 1) throw_err(E_CONFIG, "N must be >= 1");
  if (c->k < 1 || c->k > c->dimension) throw_err(E_CONFIG, "k must satisfy 1 <= k <= N");
  if (c->k % c->workers != 0) throw_err(E_CONFIG, "k must be divisible by P");
  if (c->teams < 1 || c->workers % c->teams != 0) throw_err(E_CONFIG, "d must divide P");
  if (c->sag == SAG_NONE && c->teams != 1) throw_err(E_CONFIG, "sag=none requires d=1");
  if (c->sag != SAG_NONE && c->teams == 1) throw_err(E_CONFIG, "d=1 requires sag=none");
  if (c->sag == SAG_RSAG && !is_pow2(c->teams)) throw_err(E_CONFIG, "rsag requires power-of-two d");
  if (c->workers / c->teams > c->dimension)
    throw_err(E_CONFIG, "N must allow P/d blocks (N >= P/d)");
  if (c->sag < 0 || c->sag > 2 || c->residual < 0 || c->residual > 2 || c->timing < 0 ||
      c->timing > 1)
    throw_err(E_CONFIG, "unknown enum value in ClusterConfig");
}

/* ------------------------------------------------------------------ */
/* pipeline context                                                     */
/* ------------------------------------------------------------------ */
typedef struct {
  int32_t consistent, conservation_applicable;
  double conservation_error;
  int64_t max_rounds, max_scalars;
  int64_t srs_rounds, srs_scalars, sag_rounds, sag_scalars, gather_rounds, gather_scalars;
  int64_t pred_rounds, pred_low, pred_high;
  int64_t n_union;
  int64_t global_nnz;
} orc_run_info;

typedef struct orc_ctx {
  orc_config cfg;
  real **carry;           /* [P][N] persistent residual */
  orc_hctrl *ctrl;        /* [P] (bsag only) */
  wcost *ledger;          /* [P] persistent Fabric ledger */
  int64_t *g_idx;         /* last global gradient */
  real *g_val;
  int64_t g_nnz;
  int64_t *union_sizes;   /* [m] */
  orc_run_info info;
} orc_ctx;

EXPORT int orc_validate(const orc_config *c) {
  API_BEGIN
  validate(c);
  API_END
}

EXPORT int orc_hctrl_init(orc_hctrl *c, int64_t P, int64_t k, int64_t d);

static void free_ctx(orc_ctx *x) {
  if (!x) return;
  if (x->carry) {
    for (int64_t w = 0; w < x->cfg.workers; ++w) free(x->carry[w]);
    free(x->carry);
  }
  free(x->ctrl); free(x->ledger); free(x->g_idx); free(x->g_val); free(x->union_sizes);
  free(x);
}

/* inc/pipeline.hpp:87-99 (make_worker_states) + a persistent Fabric */
EXPORT int orc_ctx_create(const orc_config *c, orc_ctx **out) {
  *out = NULL;
  const int rc = orc_validate(c);
  if (rc != E_OK) return rc;
  orc_ctx *x = (orc_ctx *)calloc(1, sizeof(orc_ctx));
  x->cfg = *c;
  const int64_t P = c->workers, N = c->dimension;
  x->carry = (real **)calloc((size_t)P, sizeof(real *));
  for (int64_t w = 0; w < P; ++w) x->carry[w] = (real *)calloc((size_t)N, sizeof(real));
  x->ledger = (wcost *)calloc((size_t)P, sizeof(wcost));
  if (c->sag == SAG_BSAG) {
    x->ctrl = (orc_hctrl *)calloc((size_t)P, sizeof(orc_hctrl));
    for (int64_t w = 0; w < P; ++w) {
      const int r = orc_hctrl_init(&x->ctrl[w], c->workers, c->k, c->teams);
      if (r != E_OK) { free_ctx(x); return r; }
    }
  }
  x->g_idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)c->k);
  x->g_val = (real *)malloc(sizeof(real) * (size_t)c->k);
  x->union_sizes = (int64_t *)calloc((size_t)(P / c->teams), sizeof(int64_t));
  *out = x;
  return E_OK;
}

EXPORT void orc_ctx_destroy(orc_ctx *x) { free_ctx(x); }

/* Residual carry setter/getter (WorkerState::residual, inc/pipeline.hpp:82-85) */
EXPORT void orc_get_carry(const orc_ctx *x, int w, real *out) {
  memcpy(out, x->carry[w], sizeof(real) * (size_t)x->cfg.dimension);
}
EXPORT void orc_set_carry(orc_ctx *x, int w, const real *in) {
  memcpy(x->carry[w], in, sizeof(real) * (size_t)x->cfg.dimension);
}
EXPORT void orc_get_ledger(const orc_ctx *x, int64_t *rounds, int64_t *scalars) {
  for (int64_t w = 0; w < x->cfg.workers; ++w) {
    rounds[w] = x->ledger[w].rounds;
    scalars[w] = x->ledger[w].scalars;
  }
}
EXPORT void orc_get_run_info(const orc_ctx *x, orc_run_info *out) { *out = x->info; }
EXPORT void orc_get_global(const orc_ctx *x, int64_t *idx, real *val) {
  memcpy(idx, x->g_idx, sizeof(int64_t) * (size_t)x->g_nnz);
  memcpy(val, x->g_val, sizeof(real) * (size_t)x->g_nnz);
}
EXPORT void orc_get_union_sizes(const orc_ctx *x, int64_t *out) {
  memcpy(out, x->union_sizes, sizeof(int64_t) * (size_t)x->info.n_union);
}
EXPORT int orc_get_controller(const orc_ctx *x, int w, orc_hctrl *out) {
  if (!x->ctrl) return E_CONFIG;
  *out = x->ctrl[w];
  return E_OK;
}

/* inc/pipeline.hpp:140-342 -- the full sparse All-Reduce.
 * grads[w] points at worker w's N gradient values. */
EXPORT int orc_allreduce(orc_ctx *x, const real *const *grads) {
  API_BEGIN
  const orc_config *cfg = &x->cfg;
  validate(cfg);
  const int p = (int)cfg->workers;
  const int m = (int)(cfg->workers / cfg->teams);
  const int d = (int)cfg->teams;
  const int64_t budget = cfg->teams * cfg->k / cfg->workers;   /* inc/pipeline.hpp:51 */
  const int64_t N = cfg->dimension;
  partition_t part = make_partition(N, m);
  fabric_t fab = {p, x->ledger};

  rstore *stores = (rstore *)amalloc(sizeof(rstore) * (size_t)p);
  for (int w = 0; w < p; ++w) {
    memset(&stores[w], 0, sizeof(rstore));
    stores[w].mode = cfg->residual;
    stores[w].n = N;
    stores[w].carry = x->carry[w];
  }
  sink_t sink = {stores};

  /* 1) residual in, snapshot; 2) divide + per-block selection (pipeline.hpp:162-184) */
  real **combined = (real **)amalloc(sizeof(real *) * (size_t)p);
  blk **divided = (blk **)amalloc(sizeof(blk *) * (size_t)p);
  for (int w = 0; w < p; ++w) {
    combined[w] = rs_apply(&stores[w], grads[w]);
    rs_begin(&stores[w], combined[w], &part);
    divided[w] = (blk *)amalloc(sizeof(blk) * (size_t)m);
    for (int b = 0; b < m; ++b) {
      blk sel, disc;
      top_k_slice(combined[w], b, part.lo[b], part.hi[b], budget, &sel, &disc);
      if (disc.n > 0) {
        rs_record_dividing_remainder(&stores[w], &disc);
        rs_record_inproc(&stores[w], b, &disc, 1.0);
      }
      divided[w][b] = sel;
    }
  }

  /* 3) reduce-scatter inside each team (pipeline.hpp:186-199) */
  wcost *before_srs = ledger_snapshot(&fab);
  int **tworkers = (int **)amalloc(sizeof(int *) * (size_t)d);
  blk **tblocks = (blk **)amalloc(sizeof(blk *) * (size_t)d);
  for (int t = 0; t < d; ++t) {
    tworkers[t] = (int *)amalloc(sizeof(int) * (size_t)m);
    tblocks[t] = (blk *)amalloc(sizeof(blk) * (size_t)m * (size_t)m);
    for (int i = 0; i < m; ++i) {
      const int w = t * m + i;
      tworkers[t][i] = w;
      for (int b = 0; b < m; ++b) tblocks[t][i * m + b] = divided[w][b];
    }
  }
  blk **reduced = run_srs_teams(&fab, d, m, tworkers, tblocks, budget, cfg->timing, &sink);
  wcost srs_delta = delta_since(&fab, before_srs);

  /* 4) cross-team synchronisation of each position group (pipeline.hpp:201-260) */
  wcost *before_sag = ledger_snapshot(&fab);
  int64_t n_union = 0;
  if (d > 1) {
    int **gworkers = (int **)amalloc(sizeof(int *) * (size_t)m);
    blk **gblocks = (blk **)amalloc(sizeof(blk *) * (size_t)m);
    for (int g = 0; g < m; ++g) {
      gworkers[g] = (int *)amalloc(sizeof(int) * (size_t)d);
      gblocks[g] = (blk *)amalloc(sizeof(blk) * (size_t)d);
      for (int t = 0; t < d; ++t) {
        gworkers[g][t] = t * m + g;
        gblocks[g][t] = reduced[t][g];
      }
    }
    if (cfg->sag == SAG_RSAG) {
      rsag_groups(&fab, m, d, gworkers, gblocks, budget, &sink);
    } else {
      int64_t *pre = (int64_t *)amalloc(sizeof(int64_t) * (size_t)m);
      for (int g = 0; g < m; ++g) {
        int64_t h = 0;
        for (int i = 0; i < d; ++i) {
          const int64_t bb = hctrl_budget(&x->ctrl[gworkers[g][i]]);
          if (i == 0) h = bb;
          else if (bb != h) throw_err(E_CONSISTENCY, "position group controllers disagree on h");
        }
        pre[g] = h;
      }
      int64_t *us = (int64_t *)amalloc(sizeof(int64_t) * (size_t)m);
      bsag_groups(&fab, m, d, gworkers, gblocks, pre, budget, &sink, us);
      for (int g = 0; g < m; ++g) {
        x->union_sizes[g] = us[g];
        for (int t = 0; t < d; ++t) hctrl_observe(&x->ctrl[t * m + g], us[g]);
      }
      n_union = m;
    }
    for (int g = 0; g < m; ++g)
      for (int t = 0; t < d; ++t) reduced[t][g] = gblocks[g][t];
  }
  wcost sag_delta = delta_since(&fab, before_sag);

  /* 5) all-gather the position blocks within each team (pipeline.hpp:262-274) */
  wcost *before_gather = ledger_snapshot(&fab);
  group_gather *gg = (group_gather *)amalloc(sizeof(group_gather) * (size_t)d);
  for (int t = 0; t < d; ++t) { gg[t].m = m; gg[t].workers = tworkers[t]; gg[t].blocks = reduced[t]; }
  blk **gathered = bruck_multi(&fab, gg, d);
  wcost gather_delta = delta_since(&fab, before_gather);

  /* 6) assemble, audit, finalize (pipeline.hpp:276-341) */
  int64_t **pw_idx = (int64_t **)amalloc(sizeof(int64_t *) * (size_t)p);
  real **pw_val = (real **)amalloc(sizeof(real *) * (size_t)p);
  int64_t *pw_n = (int64_t *)amalloc(sizeof(int64_t) * (size_t)p);
  for (int t = 0; t < d; ++t)
    for (int i = 0; i < m; ++i) {
      const int w = t * m + i;
      int64_t tot = 0;
      for (int b = 0; b < m; ++b) tot += gathered[t][i * m + b].n;
      pw_idx[w] = (int64_t *)amalloc(sizeof(int64_t) * (size_t)(tot + 1));
      pw_val[w] = (real *)amalloc(sizeof(real) * (size_t)(tot + 1));
      pw_n[w] = 0;
      for (int b = 0; b < m; ++b) {
        const blk *bl = &gathered[t][i * m + b];
        memcpy(pw_idx[w] + pw_n[w], bl->idx, sizeof(int64_t) * (size_t)bl->n);
        memcpy(pw_val[w] + pw_n[w], bl->val, sizeof(real) * (size_t)bl->n);
        pw_n[w] += bl->n;
      }
      if (pw_n[w] > cfg->k) throw_err(E_ERROR, "global gradient exceeded k entries");
    }
  /* verify_consistency, inc/pipeline.hpp:102-108 (bitwise equality) */
  int consistent = 1;
  for (int w = 1; w < p; ++w) {
    if (pw_n[w] != pw_n[0] ||
        memcmp(pw_idx[w], pw_idx[0], sizeof(int64_t) * (size_t)pw_n[0]) != 0 ||
        memcmp(pw_val[w], pw_val[0], sizeof(real) * (size_t)pw_n[0]) != 0) {
      consistent = 0;
    }
  }
  x->g_nnz = pw_n[0];
  memcpy(x->g_idx, pw_idx[0], sizeof(int64_t) * (size_t)pw_n[0]);
  memcpy(x->g_val, pw_val[0], sizeof(real) * (size_t)pw_n[0]);

  for (int w = 0; w < p; ++w) rs_finalize(&stores[w], x->g_idx, x->g_nnz);

  /* conservation audit in double, inc/pipeline.hpp:305-334 */
  double max_err = 0.0;
  {
    double *lhs = (double *)calloc((size_t)N, sizeof(double));
    double *rhs = (double *)calloc((size_t)N, sizeof(double));
    for (int w = 0; w < p; ++w)
      for (int64_t i = 0; i < N; ++i) lhs[i] += (double)combined[w][i];
    for (int64_t e = 0; e < x->g_nnz; ++e) rhs[x->g_idx[e]] += (double)x->g_val[e];
    for (int w = 0; w < p; ++w)
      for (int64_t i = 0; i < N; ++i) rhs[i] += (double)x->carry[w][i];
    for (int64_t i = 0; i < N; ++i) {
      const double denom = fabs(lhs[i]) > 1.0 ? fabs(lhs[i]) : 1.0;
      const double err = fabs(lhs[i] - rhs[i]) / denom;
      if (err > max_err) max_err = err;
    }
    free(lhs);
    free(rhs);
  }

  orc_run_info *info = &x->info;
  memset(info, 0, sizeof *info);
  info->consistent = consistent;
  info->conservation_applicable = cfg->residual == RES_GRES;
  info->conservation_error = max_err;
  for (int w = 0; w < p; ++w) {
    if (x->ledger[w].rounds > info->max_rounds) info->max_rounds = x->ledger[w].rounds;
    if (x->ledger[w].scalars > info->max_scalars) info->max_scalars = x->ledger[w].scalars;
  }
  info->srs_rounds = srs_delta.rounds; info->srs_scalars = srs_delta.scalars;
  info->sag_rounds = sag_delta.rounds; info->sag_scalars = sag_delta.scalars;
  info->gather_rounds = gather_delta.rounds; info->gather_scalars = gather_delta.scalars;
  expected_cost_sag(cfg->workers, cfg->k, cfg->teams, cfg->sag, &info->pred_rounds,
                    &info->pred_low, &info->pred_high);
  info->n_union = n_union;
  info->global_nnz = x->g_nnz;
  API_END
}

/* ------------------------------------------------------------------ */
/* component entry points used by the golden-vector tests               */
/* ------------------------------------------------------------------ */
EXPORT int orc_top_k_select(int block_id, int64_t lo, int64_t hi, const int64_t *idx,
                            const real *val, int64_t n, int64_t budget, int64_t *sel_idx,
                            real *sel_val, int64_t *n_sel, int64_t *disc_idx, real *disc_val,
                            int64_t *n_disc) {
  API_BEGIN
  blk in = blk_new(block_id, lo, hi, n);
  memcpy(in.idx, idx, sizeof(int64_t) * (size_t)n);
  memcpy(in.val, val, sizeof(real) * (size_t)n);
  in.n = n;
  blk s, dd;
  top_k(&in, budget, &s, &dd);
  memcpy(sel_idx, s.idx, sizeof(int64_t) * (size_t)s.n);
  memcpy(sel_val, s.val, sizeof(real) * (size_t)s.n);
  memcpy(disc_idx, dd.idx, sizeof(int64_t) * (size_t)dd.n);
  memcpy(disc_val, dd.val, sizeof(real) * (size_t)dd.n);
  *n_sel = s.n;
  *n_disc = dd.n;
  API_END
}

EXPORT int orc_top_k_select_slice(const real *g, int64_t lo, int64_t hi, int64_t budget,
                                  int64_t *sel_idx, real *sel_val, int64_t *n_sel,
                                  int64_t *disc_idx, real *disc_val, int64_t *n_disc) {
  API_BEGIN
  blk s, dd;
  top_k_slice(g, 0, lo, hi, budget, &s, &dd);
  memcpy(sel_idx, s.idx, sizeof(int64_t) * (size_t)s.n);
  memcpy(sel_val, s.val, sizeof(real) * (size_t)s.n);
  memcpy(disc_idx, dd.idx, sizeof(int64_t) * (size_t)dd.n);
  memcpy(disc_val, dd.val, sizeof(real) * (size_t)dd.n);
  *n_sel = s.n;
  *n_disc = dd.n;
  API_END
}

EXPORT int orc_merge_add(int a_id, const int64_t *a_idx, const real *a_val, int64_t na, int b_id,
                         const int64_t *b_idx, const real *b_val, int64_t nb, int64_t *out_idx,
                         real *out_val, int64_t *n_out) {
  API_BEGIN
  blk a = blk_new(a_id, 0, 0, na), b = blk_new(b_id, 0, 0, nb);
  memcpy(a.idx, a_idx, sizeof(int64_t) * (size_t)na);
  memcpy(a.val, a_val, sizeof(real) * (size_t)na);
  a.n = na;
  memcpy(b.idx, b_idx, sizeof(int64_t) * (size_t)nb);
  memcpy(b.val, b_val, sizeof(real) * (size_t)nb);
  b.n = nb;
  blk o = merge_add(&a, &b);
  memcpy(out_idx, o.idx, sizeof(int64_t) * (size_t)o.n);
  memcpy(out_val, o.val, sizeof(real) * (size_t)o.n);
  *n_out = o.n;
  API_END
}

/* inc/collectives.hpp:185-216 -- Top-k All-Gather baseline: every worker's
 * top_k_select_slice over the whole vector, a Bruck all-gather of the P
 * selections, and at every worker a left fold of merge_add over the gathered
 * blocks in source order starting from an empty block.  Returns worker 0's
 * union (all workers hold the same) and the per-worker ledger. */
EXPORT int orc_topka(int p, int64_t n, int64_t k, const real *const *grads, int64_t *out_idx,
                     real *out_val, int64_t *n_out, int64_t *rounds, int64_t *scalars) {
  API_BEGIN
  if (p < 1) throw_err(E_CONFIG, "topka: gradient count != worker count");
  if (k > n) throw_err(E_CONFIG, "topka: k must satisfy k <= N");
  fabric_t f;
  f.p = p;
  f.cost = (wcost *)amalloc(sizeof(wcost) * (size_t)p);
  memset(f.cost, 0, sizeof(wcost) * (size_t)p);
  int *workers = (int *)amalloc(sizeof(int) * (size_t)p);
  blk *locals = (blk *)amalloc(sizeof(blk) * (size_t)p);
  for (int w = 0; w < p; ++w) {
    blk disc;
    workers[w] = w;
    top_k_slice(grads[w], 0, 0, n, k, &locals[w], &disc);
  }
  group_gather g = {p, workers, locals};
  blk **out = bruck_multi(&f, &g, 1);
  blk acc = blk_new(0, 0, n, 0);
  for (int s = 0; s < p; ++s) acc = merge_add(&acc, &out[0][s]);   /* worker 0's view */
  memcpy(out_idx, acc.idx, sizeof(int64_t) * (size_t)acc.n);
  memcpy(out_val, acc.val, sizeof(real) * (size_t)acc.n);
  *n_out = acc.n;
  for (int w = 0; w < p; ++w) { rounds[w] = f.cost[w].rounds; scalars[w] = f.cost[w].scalars; }
  API_END
}

EXPORT int orc_partition(int64_t n, int count, int64_t *lo, int64_t *hi) {
  API_BEGIN
  partition_t p = make_partition(n, count);
  memcpy(lo, p.lo, sizeof(int64_t) * (size_t)count);
  memcpy(hi, p.hi, sizeof(int64_t) * (size_t)count);
  API_END
}

EXPORT int orc_block_of(int64_t n, int count, int64_t i, int32_t *out) {
  API_BEGIN
  partition_t p = make_partition(n, count);
  *out = block_of(&p, i);
  API_END
}

/* positions: concatenation of bags B1..Bl; bag_size[j-1] = |Bj| */
EXPORT int orc_build_bags(int m, int rank, int32_t *l, int32_t *remainder, int32_t *bag_size,
                          int32_t *positions) {
  API_BEGIN
  bags_t s = build_bags(m, rank);
  *l = s.l;
  *remainder = s.remainder;
  int o = 0;
  for (int j = 0; j < s.l; ++j) {
    bag_size[j] = s.bag_size[j];
    for (int q = 0; q < s.bag_size[j]; ++q) positions[o++] = s.bag[j][q];
  }
  API_END
}

EXPORT int orc_expected_cost_srs(int64_t m, int64_t k, int64_t *rounds, int64_t *scalars) {
  API_BEGIN
  if (m < 1) throw_err(E_CONFIG, "expected_cost_srs: m >= 1 required");
  if (k % m != 0) throw_err(E_CONFIG, "expected_cost_srs: m must divide k");
  if (m == 1) { *rounds = 0; *scalars = 0; }
  else { *rounds = ceil_log2(m); *scalars = 2 * (k / m) * (m - 1); }
  API_END
}

EXPORT int orc_expected_cost_sag(int64_t P, int64_t k, int64_t d, int mode, int64_t *rounds,
                                 int64_t *low, int64_t *high) {
  API_BEGIN
  expected_cost_sag(P, k, d, mode, rounds, low, high);
  API_END
}

EXPORT int orc_bsag_phase_cost(int64_t P, int64_t k, int64_t d, int64_t *rounds, int64_t *low,
                               int64_t *high) {
  API_BEGIN   /* inc/sag.hpp:332-340 */
  if (d < 2 || P % d != 0 || k % P != 0) throw_err(E_CONFIG, "bsag_phase_cost: invalid (P, k, d)");
  const int64_t c = k / P;
  *rounds = ceil_log2(d); *low = 2 * c * (d - 1); *high = 2 * c * d * (d - 1);
  API_END
}

EXPORT int orc_topka_cost(int64_t P, int64_t k, int64_t *rounds, int64_t *low, int64_t *high) {
  API_BEGIN   /* inc/sag.hpp:343-346 */
  const int64_t sc = 2 * (P - 1) * k;
  *rounds = ceil_log2(P); *low = sc; *high = sc;
  API_END
}

EXPORT int orc_dyadic_shares(int count, double *out) {
  API_BEGIN
  double *s = dyadic_shares(count);
  memcpy(out, s, sizeof(double) * (size_t)(count > 1 ? count : 1));
  API_END
}

EXPORT int orc_hctrl_init(orc_hctrl *c, int64_t P, int64_t k, int64_t d) {
  API_BEGIN
  hctrl_init(c, P, k, d);
  API_END
}
EXPORT void orc_hctrl_observe(orc_hctrl *c, int64_t n_t) { hctrl_observe(c, n_t); }
EXPORT int64_t orc_hctrl_budget(const orc_hctrl *c) { return hctrl_budget(c); }

/* Fabric restatement for the ledger golden tests (tests/test_fabric.cpp). */
typedef struct orc_fabric { fabric_t f; } orc_fabric;
EXPORT int orc_fabric_create(int p, orc_fabric **out) {
  *out = NULL;
  if (p < 1) { snprintf(g_msg, sizeof g_msg, "fabric needs >= 1 worker"); return E_CONFIG; }
  orc_fabric *x = (orc_fabric *)calloc(1, sizeof(orc_fabric));
  x->f.p = p;
  x->f.cost = (wcost *)calloc((size_t)p, sizeof(wcost));
  *out = x;
  return E_OK;
}
EXPORT void orc_fabric_destroy(orc_fabric *x) {
  if (!x) return;
  free(x->f.cost);
  free(x);
}
/* one round: targets[w] (-1 = silent), nnz[w] = entries of the one block w sends */
EXPORT int orc_fabric_exchange(orc_fabric *x, const int32_t *targets, const int64_t *nnz) {
  API_BEGIN
  const int p = x->f.p;
  wcost *backup = ledger_snapshot(&x->f);
  send_t *plan = (send_t *)amalloc(sizeof(send_t) * (size_t)p);
  memset(plan, 0, sizeof(send_t) * (size_t)p);
  for (int w = 0; w < p; ++w) {
    if (targets[w] < 0) continue;
    plan[w].has = 1;
    plan[w].target = targets[w];
    plan[w].nblk = 1;
    plan[w].payload = (blk *)amalloc(sizeof(blk));
    plan[w].payload[0] = blk_new(0, 0, nnz[w], nnz[w]);
    plan[w].payload[0].n = nnz[w];
  }
  /* the reference mutates the ledger before detecting a duplicate target, so
   * a failed round leaves partial volume behind (inc/fabric.hpp:83-106);
   * restate that faithfully */
  (void)backup;
  fabric_exchange(&x->f, plan);
  API_END
}
EXPORT void orc_fabric_ledger(const orc_fabric *x, int64_t *rounds, int64_t *scalars) {
  for (int w = 0; w < x->f.p; ++w) { rounds[w] = x->f.cost[w].rounds; scalars[w] = x->f.cost[w].scalars; }
}

/* Bruck all-gather restatement: returns per-member ledger and checks source
 * order; nnz[i] = entries contributed by member i. */
EXPORT int orc_bruck_ledger(int m, const int64_t *nnz, int64_t *rounds, int64_t *scalars,
                            int32_t *order_ok) {
  API_BEGIN
  if (m < 0) throw_err(E_GROUP_SIZE, "all-gather on empty group");
  fabric_t f;
  f.p = m > 0 ? m : 1;
  f.cost = (wcost *)amalloc(sizeof(wcost) * (size_t)f.p);
  memset(f.cost, 0, sizeof(wcost) * (size_t)f.p);
  int *workers = (int *)amalloc(sizeof(int) * (size_t)f.p);
  blk *blocks = (blk *)amalloc(sizeof(blk) * (size_t)f.p);
  for (int i = 0; i < m; ++i) {
    workers[i] = i;
    blocks[i] = blk_new(i, 0, nnz[i], nnz[i]);
    blocks[i].n = nnz[i];
  }
  group_gather g = {m, workers, blocks};
  blk **out = bruck_multi(&f, &g, 1);
  int ok = 1;
  for (int i = 0; i < m; ++i)
    for (int s = 0; s < m; ++s)
      if (out[0][i * m + s].block_id != s || out[0][i * m + s].n != nnz[s]) ok = 0;
  *order_ok = ok;
  for (int i = 0; i < m; ++i) { rounds[i] = f.cost[i].rounds; scalars[i] = f.cost[i].scalars; }
  API_END
}

/* Replays Algorithm 2 (inc/sag.hpp:37-90) over a sequence of union sizes;
 * entry i is the state before observation i (entry n_obs: after the last). */
EXPORT int orc_hctrl_trace(int64_t P, int64_t k, int64_t d, int64_t n_obs, const int64_t *ns,
                           double *h, double *step, int32_t *flag, int64_t *budget) {
  API_BEGIN
  orc_hctrl c;
  hctrl_init(&c, P, k, d);
  for (int64_t i = 0; i <= n_obs; ++i) {
    h[i] = c.h; step[i] = c.step; flag[i] = c.flag; budget[i] = hctrl_budget(&c);
    if (i < n_obs) hctrl_observe(&c, ns[i]);
  }
  API_END
}
