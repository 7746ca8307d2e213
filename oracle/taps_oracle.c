/*
 * taps_oracle.c — TEST INFRASTRUCTURE ONLY (see taps_oracle.h).
 *
 * A from-scratch C99 restatement of the reference's hot path. Every function
 * cites the reference file:line it restates; all paths below are relative to
 * /root/reference/proj/include/topoplan/. Floating-point expressions keep the
 * reference's operation order so results are bit-identical.
 */
#include "taps_oracle.h"

#include <stdlib.h>
#include <string.h>

#define O_MAXD 64    /* device-matrix depth */
#define O_MAXR 64    /* unified tensor rank */
#define O_MAXP 64    /* parts per tensor dim */
#define O_MAXOPS 256 /* plan length */

/* ------------------------------------------------------------------------ */
/* small helpers                                                            */
/* ------------------------------------------------------------------------ */

/* graph.hpp:115 */
static int is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }

/* graph.hpp:117-121 */
static int log2_exact(int64_t n) {
  int e = 0;
  while (((int64_t)1 << e) < n) ++e;
  return e;
}

/* A device matrix stored the reference's way: dims[] outermost first,
 * extent(k) = dims[depth-1-k] (layout.hpp:35-56). */
typedef struct {
  int depth;
  int64_t dims[O_MAXD];
} o_matrix;

static int64_t m_extent(const o_matrix* m, int k) { return m->dims[m->depth - 1 - k]; }

static int64_t m_total(const o_matrix* m) {
  int64_t n = 1;
  for (int i = 0; i < m->depth; ++i) n *= m->dims[i];
  return n;
}

typedef struct {
  int rank;
  int e[O_MAXR];
} o_map;

/* layout.hpp:83-93 */
static int map_contains(const o_map* m, int k) {
  for (int i = 0; i < m->rank; ++i)
    if (m->e[i] == k) return 1;
  return 0;
}
static int map_axis_of(const o_map* m, int k) {
  for (int i = 0; i < m->rank; ++i)
    if (m->e[i] == k) return i;
  return -1;
}
static int map_eq(const o_map* a, const o_map* b) {
  if (a->rank != b->rank) return 0;
  for (int i = 0; i < a->rank; ++i)
    if (a->e[i] != b->e[i]) return 0;
  return 1;
}

/* ------------------------------------------------------------------------ */
/* strategies: layout.hpp:222-328                                           */
/* ------------------------------------------------------------------------ */

typedef struct {
  int p;
  int64_t degrees[TP_MAX_AXES];
  int dmap[TP_MAX_AXES];
  o_matrix matrix; /* canonical: one dim per sharded axis */
} o_strategy;

/* layout.hpp:222-244 — closed-form count. */
int64_t oracle_strategy_count(int32_t p, int64_t total_devices) {
  if (p < 1 || !is_pow2(total_devices)) return -1;
  const int n = log2_exact(total_devices);
  if (n == 0) return 1;
  int64_t count = 0, fact = 1;
  for (int i = 1; i <= (p < n ? p : n); ++i) {
    fact *= i;
    int64_t c1 = 1, c2 = 1;
    for (int j = 0; j < i; ++j) c1 = c1 * (p - j) / (j + 1);
    for (int j = 0; j < i - 1; ++j) c2 = c2 * (n - 1 - j) / (j + 1);
    count += fact * c1 * c2;
  }
  return count;
}

/* Lexicographically-previous permutation (std::prev_permutation). */
static int prev_perm(int* a, int n) {
  int i = n - 1;
  while (i > 0 && a[i - 1] <= a[i]) --i;
  if (i <= 0) {
    for (int l = 0, r = n - 1; l < r; ++l, --r) { int t = a[l]; a[l] = a[r]; a[r] = t; }
    return 0;
  }
  int j = n - 1;
  while (a[j] >= a[i - 1]) --j;
  int t = a[i - 1]; a[i - 1] = a[j]; a[j] = t;
  for (int l = i, r = n - 1; l < r; ++l, --r) { t = a[l]; a[l] = a[r]; a[r] = t; }
  return 1;
}

static int cmp_strategy(const void* pa, const void* pb) {
  const o_strategy* a = (const o_strategy*)pa;
  const o_strategy* b = (const o_strategy*)pb;
  /* layout.hpp:322-326: degrees ascending, then device_map descending. */
  for (int i = 0; i < a->p; ++i) {
    if (a->degrees[i] != b->degrees[i]) return a->degrees[i] < b->degrees[i] ? -1 : 1;
  }
  for (int i = 0; i < a->p; ++i) {
    if (a->dmap[i] != b->dmap[i]) return a->dmap[i] > b->dmap[i] ? -1 : 1;
  }
  return 0;
}

/* layout.hpp:249-263 (compositions, first part varying slowest) and
 * layout.hpp:270-328 (placements by prev_permutation, then sort). */
static int64_t enumerate_into(int p, int64_t N, o_strategy* out, int64_t cap) {
  if (!is_pow2(N) || p < 1 || p > TP_MAX_AXES) return -1;
  const int n = log2_exact(N);
  int64_t count = 0;
  int exps[TP_MAX_AXES];
  /* iterate compositions of n into p non-negative parts, lexicographically */
  for (int i = 0; i < p; ++i) exps[i] = 0;
  exps[p - 1] = n;
  for (;;) {
    int sharded[TP_MAX_AXES], ns = 0;
    for (int a = 0; a < p; ++a)
      if (exps[a] > 0) sharded[ns++] = a;
    o_strategy base;
    memset(&base, 0, sizeof(base));
    base.p = p;
    for (int a = 0; a < p; ++a) { base.degrees[a] = (int64_t)1 << exps[a]; base.dmap[a] = -1; }
    if (ns == 0) {
      if (count < cap) out[count] = base;
      ++count;
    } else {
      int pos[TP_MAX_AXES];
      for (int j = 0; j < ns; ++j) pos[j] = ns - 1 - j; /* descending */
      do {
        o_strategy s = base;
        s.matrix.depth = ns;
        for (int j = 0; j < ns; ++j) s.dmap[sharded[j]] = pos[j];
        for (int j = 0; j < ns; ++j) s.matrix.dims[ns - 1 - pos[j]] = s.degrees[sharded[j]];
        if (count < cap) out[count] = s;
        ++count;
      } while (prev_perm(pos, ns));
    }
    /* next composition in lexicographic order (layout.hpp:258-262) */
    int k = p - 2;
    while (k >= 0) {
      /* parts 0..k fixed-prefix; can we increase exps[k]? */
      int prefix = 0;
      for (int a = 0; a <= k; ++a) prefix += exps[a];
      if (prefix < n) break;
      --k;
    }
    if (k < 0) break;
    exps[k] += 1;
    int prefix = 0;
    for (int a = 0; a <= k; ++a) prefix += exps[a];
    for (int a = k + 1; a < p - 1; ++a) exps[a] = 0;
    exps[p - 1] = n - prefix;
  }
  if (count <= cap) qsort(out, (size_t)count, sizeof(o_strategy), cmp_strategy);
  return count;
}

int64_t oracle_enumerate(int32_t p, int64_t total_devices, int64_t* degrees,
                         int32_t* device_map, int64_t* matrix_dims,
                         int32_t* matrix_depth) {
  int64_t n = oracle_strategy_count(p, total_devices);
  if (n < 0) return -1;
  o_strategy* s = (o_strategy*)malloc(sizeof(o_strategy) * (size_t)(n ? n : 1));
  int64_t got = enumerate_into(p, total_devices, s, n);
  if (got != n) { free(s); return -1; }
  for (int64_t i = 0; i < n; ++i) {
    for (int a = 0; a < p; ++a) {
      if (degrees) degrees[i * p + a] = s[i].degrees[a];
      if (device_map) device_map[i * p + a] = s[i].dmap[a];
      if (matrix_dims) matrix_dims[i * p + a] = a < s[i].matrix.depth ? s[i].matrix.dims[a] : 0;
    }
    if (matrix_depth) matrix_depth[i] = s[i].matrix.depth;
  }
  free(s);
  return n;
}

/* ------------------------------------------------------------------------ */
/* cost model: cost_model.hpp:39-230                                        */
/* ------------------------------------------------------------------------ */

typedef struct {
  double intra, inter;
  int64_t local;
} o_env;

/* cost_model.hpp:39-43 */
static double allreduce_volume(int64_t group, double data) {
  if (group <= 1) return 0;
  const double n = (double)group;
  return 2.0 * (n - 1) / n * data;
}
/* cost_model.hpp:46-49 */
static double allgather_volume(int64_t group, double shard) {
  if (group <= 1) return 0;
  return (double)(group - 1) * shard;
}
/* cost_model.hpp:52-56 */
static double alltoall_volume(int64_t group, double shard) {
  if (group <= 1) return 0;
  const double n = (double)group;
  return (n - 1) / n * shard;
}

/* cost_model.hpp:75-97 (paper Alg. 2) */
static int64_t ct_allreduce(const o_matrix* m, const o_map* map, int64_t local) {
  int64_t pd = m_total(m);
  for (int i = 0; i < map->rank; ++i)
    if (map->e[i] >= 0) pd /= m_extent(m, map->e[i]);
  int64_t remain = local, dev_in = 1;
  for (int k = 0; k < m->depth; ++k) {
    if (!map_contains(map, k) && remain > 1) {
      dev_in *= remain > m_extent(m, k) ? m_extent(m, k) : remain;
    }
    remain /= m_extent(m, k);
  }
  if (dev_in >= pd) return 0;
  if (dev_in > 1) return local / dev_in;
  return local;
}

/* cost_model.hpp:108-135 (paper Alg. 3) */
static void ct_allgather_dim(const o_matrix* m, const o_map* map, int g,
                             int64_t local, int64_t* ct, int64_t* repeat,
                             int64_t* gin) {
  const int64_t pd = m_extent(m, g);
  int64_t temp = 1, rep = 1;
  for (int k = 0; k < g; ++k) {
    temp *= m_extent(m, k);
    if (!map_contains(map, k)) rep *= m_extent(m, k);
  }
  if (rep > local) rep = local;
  *repeat = rep;
  if (temp >= local) {
    *gin = 1;
    *ct = local / rep;
  } else {
    const int64_t remain = local / temp;
    *gin = pd < remain ? pd : remain;
    *ct = remain >= pd ? 0 : temp / rep;
  }
}

/* cost_model.hpp:148-151 */
static double eff_bw(int64_t ct, const o_env* env) {
  if (ct <= 0) return env->intra;
  return env->inter / (double)ct;
}

/* cost_model.hpp:176-225, AllGather and AllToAll branches */
static double gather_like_cost(int is_a2a, int64_t group, double shard,
                               const o_matrix* m, const o_map* working, int dim,
                               const o_env* env, int64_t* ct_out) {
  int64_t ct, rep, gin;
  if (!is_a2a) {
    const double vol = allgather_volume(group, shard);
    ct_allgather_dim(m, working, dim, env->local, &ct, &rep, &gin);
    if (ct_out) *ct_out = ct;
    return vol / eff_bw(ct, env);
  }
  const double vol = alltoall_volume(group, shard);
  ct_allgather_dim(m, working, dim, env->local, &ct, &rep, &gin);
  const int64_t p = group, k = gin;
  if (p <= 1) {
    if (ct_out) *ct_out = 0;
    return 0;
  }
  if (k >= p) {
    if (ct_out) *ct_out = 0;
    return vol / env->intra;
  }
  int64_t c = env->local / (k * rep);
  if (c < 1) c = 1;
  if (ct_out) *ct_out = c;
  const double bw = eff_bw(c, env);
  const double scale = (double)k * (double)(p - k) / (double)(p - 1);
  return scale * vol / bw;
}

/* ------------------------------------------------------------------------ */
/* unification: redistribution.hpp:82-346                                   */
/* ------------------------------------------------------------------------ */

typedef struct {
  int64_t extent;
  int map;
} o_part;

typedef struct {
  int n;
  o_part p[O_MAXP];
} o_dimparts;

typedef struct {
  int rank;
  int64_t shape[TP_MAX_RANK];
  int element_size;
  o_matrix m;
  o_map map;
} o_layout;

/* redistribution.hpp:92-115 */
static int expand_over_run(int64_t extent, const int* run, int nrun,
                           const int64_t* exts, o_dimparts* out) {
  out->n = 0;
  if (nrun == 0) {
    out->p[out->n++] = (o_part){extent, -1};
    return 0;
  }
  int64_t rem = extent;
  for (int j = 0; j + 1 < nrun; ++j) {
    const int64_t d = exts[run[j]];
    if (rem % d != 0) return TP_E_FACTORIZATION;
    out->p[out->n++] = (o_part){d, run[j]};
    rem /= d;
  }
  if (rem % exts[run[nrun - 1]] != 0) return TP_E_FACTORIZATION;
  out->p[out->n++] = (o_part){rem, run[nrun - 1]};
  return 0;
}

/* redistribution.hpp:120-156 */
static int reexpress(const o_layout* L, const int64_t* exts, int nexts,
                     o_dimparts* dims) {
  const int h = L->m.depth;
  int64_t ocum[O_MAXD + 1], ucum[O_MAXD + 1];
  ocum[0] = 1;
  for (int k = 0; k < h; ++k) ocum[k + 1] = ocum[k] * m_extent(&L->m, k);
  ucum[0] = 1;
  for (int k = 0; k < nexts; ++k) ucum[k + 1] = ucum[k] * exts[k];
  int run[O_MAXD][O_MAXD], nrun[O_MAXD];
  for (int k = 0; k < h; ++k) {
    nrun[k] = 0;
    for (int u = nexts - 1; u >= 0; --u) {
      if (ucum[u] >= ocum[k] && ucum[u + 1] <= ocum[k + 1] && exts[u] > 1)
        run[k][nrun[k]++] = u;
    }
    if (nrun[k] == 0 && m_extent(&L->m, k) > 1) return TP_E_NOT_UNIFIABLE;
  }
  for (int i = 0; i < L->rank; ++i) {
    const int64_t e = L->shape[i];
    const int m = L->map.e[i];
    if (m < 0 || m_extent(&L->m, m) == 1) {
      dims[i].n = 1;
      dims[i].p[0] = (o_part){e, -1};
    } else {
      int st = expand_over_run(e, run[m], nrun[m], exts, &dims[i]);
      if (st) return st;
    }
  }
  return 0;
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* redistribution.hpp:167-221. Returns 0 = refined, 1 = split requested
 * (*split_dim, *split_outer), or an error kind (> 1, negated to avoid
 * collisions: returned as -kind). */
static int refine_side(o_dimparts* parts, const int64_t* bnd, int nb,
                       const int64_t* exts, int* split_dim, int64_t* split_outer) {
  o_dimparts ref;
  ref.n = 0;
  int64_t pos = 1;
  for (int pi = 0; pi < parts->n; ++pi) {
    const o_part part = parts->p[pi];
    const int64_t lo = pos, hi = pos * part.extent;
    int64_t cuts[O_MAXP * 2];
    int nc = 0;
    for (int b = 0; b < nb; ++b) {
      if (bnd[b] > lo && bnd[b] < hi) {
        if (bnd[b] % lo != 0 || part.extent % (bnd[b] / lo) != 0) return -TP_E_REFINE;
        cuts[nc++] = bnd[b] / lo;
      }
    }
    qsort(cuts, (size_t)nc, sizeof(int64_t), cmp_i64);
    if (nc == 0) {
      ref.p[ref.n++] = part;
    } else if (part.map < 0) {
      int64_t prev = 1;
      for (int c = 0; c < nc; ++c) { ref.p[ref.n++] = (o_part){cuts[c] / prev, -1}; prev = cuts[c]; }
      ref.p[ref.n++] = (o_part){part.extent / prev, -1};
    } else {
      const int64_t d = exts[part.map];
      const int64_t f1 = cuts[0];
      if (f1 % d == 0) {
        int64_t prev = 1;
        for (int c = 0; c < nc; ++c) {
          ref.p[ref.n++] = (o_part){cuts[c] / prev, c == 0 ? part.map : -1};
          prev = cuts[c];
        }
        ref.p[ref.n++] = (o_part){part.extent / prev, -1};
      } else if (d % f1 == 0 && f1 > 1) {
        *split_dim = part.map;
        *split_outer = f1;
        return 1;
      } else {
        return -TP_E_REFINE;
      }
    }
    if (ref.n > O_MAXP - 2) return -TP_E_CAPACITY;
    pos = hi;
  }
  *parts = ref;
  return 0;
}

/* redistribution.hpp:226-252 */
static int split_device_dim(int64_t* exts, int* nexts, int k, int64_t f,
                            o_dimparts* a, o_dimparts* b, int rank) {
  const int64_t inner = exts[k] / f;
  exts[k] = inner;
  if (*nexts + 1 > O_MAXD) return TP_E_CAPACITY;
  for (int u = *nexts; u > k + 1; --u) exts[u] = exts[u - 1];
  exts[k + 1] = f;
  *nexts += 1;
  o_dimparts* sides[2] = {a, b};
  for (int s = 0; s < 2; ++s) {
    for (int i = 0; i < rank; ++i) {
      o_dimparts* dim = &sides[s][i];
      o_dimparts rw;
      rw.n = 0;
      for (int pi = 0; pi < dim->n; ++pi) {
        o_part part = dim->p[pi];
        if (part.map > k) {
          part.map += 1;
          rw.p[rw.n++] = part;
        } else if (part.map == k) {
          if (part.extent % f != 0 || (part.extent / f) % inner != 0) return TP_E_DEVICE_SPLIT;
          rw.p[rw.n++] = (o_part){f, k + 1};
          rw.p[rw.n++] = (o_part){part.extent / f, k};
        } else {
          rw.p[rw.n++] = part;
        }
        if (rw.n > O_MAXP - 2) return TP_E_CAPACITY;
      }
      *dim = rw;
    }
  }
  return 0;
}

typedef struct {
  o_matrix m;
  int urank;
  int64_t shape[O_MAXR];
  o_map from, to;
} o_unified;

static int sort_unique(int64_t* v, int n) {
  qsort(v, (size_t)n, sizeof(int64_t), cmp_i64);
  int w = 0;
  for (int i = 0; i < n; ++i)
    if (w == 0 || v[w - 1] != v[i]) v[w++] = v[i];
  return w;
}

/* redistribution.hpp:259-346 */
static int unify(const o_layout* from, const o_layout* to, o_unified* out) {
  if (from->rank != to->rank) return TP_E_SHAPE_MISMATCH;
  for (int i = 0; i < from->rank; ++i)
    if (from->shape[i] != to->shape[i]) return TP_E_SHAPE_MISMATCH;
  if (m_total(&from->m) != m_total(&to->m)) return TP_E_NOT_UNIFIABLE;

  /* step 1, :270-289 */
  int64_t cums[2 * O_MAXD];
  int nc = 0;
  const o_matrix* ms[2] = {&from->m, &to->m};
  for (int s = 0; s < 2; ++s) {
    int64_t c = 1;
    for (int k = 0; k < ms[s]->depth; ++k) {
      c *= m_extent(ms[s], k);
      if (c > 1) cums[nc++] = c;
    }
  }
  nc = sort_unique(cums, nc);
  int64_t exts[O_MAXD + 1];
  int nexts = 0;
  int64_t prev = 1;
  for (int i = 0; i < nc; ++i) {
    if (cums[i] % prev != 0) return TP_E_NOT_UNIFIABLE;
    exts[nexts++] = cums[i] / prev;
    prev = cums[i];
  }

  static __thread o_dimparts fd[TP_MAX_RANK], td[TP_MAX_RANK];
  int st = reexpress(from, exts, nexts, fd);
  if (st) return st;
  st = reexpress(to, exts, nexts, td);
  if (st) return st;

  /* step 2, :294-328 */
  const int rank = from->rank;
  int rounds = 0;
  for (;;) {
    if (++rounds > 64) return TP_E_NO_CONVERGE;
    int restarted = 0;
    for (int i = 0; i < rank && !restarted; ++i) {
      int64_t bnd[2 * O_MAXP];
      int nb = 0;
      o_dimparts* sides[2] = {&fd[i], &td[i]};
      for (int s = 0; s < 2; ++s) {
        int64_t c = 1;
        for (int pi = 0; pi < sides[s]->n; ++pi) {
          c *= sides[s]->p[pi].extent;
          bnd[nb++] = c;
        }
      }
      nb = sort_unique(bnd, nb);
      for (int s = 0; s < 2; ++s) {
        int sd = -1;
        int64_t so = 1;
        int r = refine_side(sides[s], bnd, nb, exts, &sd, &so);
        if (r < 0) return -r;
        if (r == 1) {
          st = split_device_dim(exts, &nexts, sd, so, fd, td, rank);
          if (st) return st;
          restarted = 1;
          break;
        }
      }
    }
    if (!restarted) break;
  }

  /* read-off, :330-345 */
  out->m.depth = nexts;
  for (int k = 0; k < nexts; ++k) out->m.dims[k] = exts[nexts - 1 - k];
  out->urank = 0;
  for (int i = 0; i < rank; ++i) {
    if (fd[i].n != td[i].n) return TP_E_REFINE_MISMATCH;
    for (int j = 0; j < fd[i].n; ++j) {
      if (fd[i].p[j].extent != td[i].p[j].extent) return TP_E_REFINE_MISMATCH;
      if (out->urank >= O_MAXR) return TP_E_CAPACITY;
      out->shape[out->urank] = fd[i].p[j].extent;
      out->from.e[out->urank] = fd[i].p[j].map;
      out->to.e[out->urank] = td[i].p[j].map;
      out->urank++;
    }
  }
  out->from.rank = out->to.rank = out->urank;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* sequence inference: redistribution.hpp:350-451 (paper Alg. 1)           */
/* ------------------------------------------------------------------------ */

enum { K_SLICE = 0, K_ALLGATHER = 1, K_ALLTOALL = 2 };

typedef struct {
  int kind, dim, axis, dest, fallback;
} o_op;

typedef struct {
  int n;
  o_op ops[O_MAXOPS];
} o_plan;

static int push_op(o_plan* p, int kind, int dim, int axis, int dest, int fb) {
  if (p->n >= O_MAXOPS) return TP_E_CAPACITY;
  p->ops[p->n++] = (o_op){kind, dim, axis, dest, fb};
  return 0;
}

/* :350-365 */
static int infer_slice(o_map* w, const o_map* to, o_plan* p, int* any) {
  *any = 0;
  for (int i = 0; i < w->rank; ++i) {
    const int k = to->e[i];
    if (w->e[i] == -1 && k >= 0 && !map_contains(w, k)) {
      if (push_op(p, K_SLICE, k, i, -1, 0)) return TP_E_CAPACITY;
      w->e[i] = k;
      *any = 1;
    }
  }
  return 0;
}

/* :367-385 */
static int infer_all2all(o_map* w, const o_map* to, o_plan* p, int* any) {
  *any = 0;
  for (int i = 0; i < w->rank; ++i) {
    const int k = w->e[i];
    if (k < 0 || to->e[i] == k) continue;
    const int j = map_axis_of(to, k);
    if (j >= 0 && j != i && w->e[j] == -1) {
      if (push_op(p, K_ALLTOALL, k, i, j, 0)) return TP_E_CAPACITY;
      w->e[i] = -1;
      w->e[j] = k;
      *any = 1;
    }
  }
  return 0;
}

/* :387-401 and :403-417 */
static int infer_gather(o_map* w, const o_map* to, o_plan* p) {
  for (int i = 0; i < w->rank; ++i) {
    const int k = w->e[i];
    if (k >= 0 && to->e[i] == -1) {
      if (push_op(p, K_ALLGATHER, k, i, -1, 0)) return TP_E_CAPACITY;
      w->e[i] = -1;
      return 0;
    }
  }
  for (int i = 0; i < w->rank; ++i) {
    if (w->e[i] != to->e[i] && w->e[i] >= 0) {
      if (push_op(p, K_ALLGATHER, w->e[i], i, -1, 1)) return TP_E_CAPACITY;
      w->e[i] = -1;
      return 0;
    }
  }
  return TP_E_DEADLOCK;
}

/* :419-451 with enable_all2all = true (RedistStage::kOptimized, :501-507) */
static int run_inference(int depth, const o_map* from, const o_map* to, o_plan* p) {
  o_map w = *from;
  p->n = 0;
  int guard = (depth + 1) * (from->rank + 1) * 4 + 16;
  while (!map_eq(&w, to)) {
    if (--guard < 0) return TP_E_NO_TERMINATE;
    int progress = 1;
    while (progress) {
      int any;
      if (infer_slice(&w, to, p, &any)) return TP_E_CAPACITY;
      progress = any;
      int a2a = 1;
      while (a2a) {
        if (infer_all2all(&w, to, p, &any)) return TP_E_CAPACITY;
        a2a = any;
        progress |= a2a;
      }
    }
    if (map_eq(&w, to)) break;
    int st = infer_gather(&w, to, p);
    if (st) return st;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* pricing: redistribution.hpp:510-553, cost_model.hpp:233-263              */
/* ------------------------------------------------------------------------ */

/* redistribution.hpp:510-517 */
static double shard_bytes_under(const o_matrix* m, const o_map* map, double bytes) {
  double div = 1;
  for (int i = 0; i < map->rank; ++i)
    if (map->e[i] >= 0) div *= (double)m_extent(m, map->e[i]);
  return bytes / div;
}

static void apply_op(o_map* w, const o_op* op) {
  switch (op->kind) {
    case K_SLICE: w->e[op->axis] = op->dim; break;
    case K_ALLGATHER: w->e[op->axis] = -1; break;
    case K_ALLTOALL: w->e[op->axis] = -1; w->e[op->dest] = op->dim; break;
  }
}

/* redistribution.hpp:521-553 */
static double plan_volume(const o_unified* u, const o_plan* p, double bytes) {
  double vol = 0;
  o_map w = u->from;
  for (int i = 0; i < p->n; ++i) {
    const o_op* op = &p->ops[i];
    const double shard = shard_bytes_under(&u->m, &w, bytes);
    const double d = (double)m_extent(&u->m, op->dim);
    double v = 0;
    if (op->kind == K_ALLGATHER) v = (d - 1) * shard;
    else if (op->kind == K_ALLTOALL) v = (d - 1) / d * shard;
    vol += v;
    apply_op(&w, op);
  }
  return vol;
}

/* cost_model.hpp:233-263 */
static double plan_seconds(const o_unified* u, const o_plan* p, double bytes,
                           const o_env* env, int64_t* cts, double* secs) {
  double seconds = 0;
  o_map w = u->from;
  for (int i = 0; i < p->n; ++i) {
    const o_op* op = &p->ops[i];
    const double shard = shard_bytes_under(&u->m, &w, bytes);
    double s = 0;
    int64_t ct = 0;
    if (op->kind != K_SLICE) {
      s = gather_like_cost(op->kind == K_ALLTOALL, m_extent(&u->m, op->dim), shard,
                           &u->m, &w, op->dim, env, &ct);
      seconds += s;
    }
    if (cts) cts[i] = ct;
    if (secs) secs[i] = s;
    apply_op(&w, op);
  }
  return seconds;
}

int oracle_redistribute(const tp_redist_query* q, tp_redist_result* r) {
  memset(r, 0, sizeof(*r));
  if (q->rank > TP_MAX_RANK || q->from_depth > O_MAXD || q->to_depth > O_MAXD) {
    r->status = TP_E_CAPACITY;
    return r->status;
  }
  o_layout f, t;
  memset(&f, 0, sizeof f);
  memset(&t, 0, sizeof t);
  f.rank = t.rank = q->rank;
  for (int i = 0; i < q->rank; ++i) {
    f.shape[i] = t.shape[i] = q->shape[i];
    f.map.e[i] = q->from_map[i];
    t.map.e[i] = q->to_map[i];
  }
  f.map.rank = t.map.rank = q->rank;
  f.m.depth = q->from_depth;
  for (int k = 0; k < q->from_depth; ++k) f.m.dims[k] = q->from_dims[k];
  t.m.depth = q->to_depth;
  for (int k = 0; k < q->to_depth; ++k) t.m.dims[k] = q->to_dims[k];
  o_unified u;
  int st = unify(&f, &t, &u);
  if (st) { r->status = st; return st; }
  static __thread o_plan p;
  st = run_inference(u.m.depth, &u.from, &u.to, &p);
  if (st) { r->status = st; return st; }
  if (u.m.depth > TP_MAX_UNIFIED_DEPTH || u.urank > TP_MAX_UNIFIED_RANK || p.n > TP_MAX_PLAN_OPS) {
    r->status = TP_E_CAPACITY;
    return r->status;
  }
  r->depth = u.m.depth;
  for (int k = 0; k < u.m.depth; ++k) r->dims[k] = u.m.dims[k];
  r->urank = u.urank;
  for (int i = 0; i < u.urank; ++i) {
    r->shape[i] = u.shape[i];
    r->from_map[i] = u.from.e[i];
    r->to_map[i] = u.to.e[i];
  }
  r->num_ops = p.n;
  for (int i = 0; i < p.n; ++i) {
    r->ops[i][0] = p.ops[i].kind;
    r->ops[i][1] = p.ops[i].dim;
    r->ops[i][2] = p.ops[i].axis;
    r->ops[i][3] = p.ops[i].dest;
    r->ops[i][4] = p.ops[i].fallback;
  }
  o_env env = {q->intra_bandwidth, q->inter_bandwidth, q->local_device_num};
  r->volume_bytes = plan_volume(&u, &p, q->tensor_bytes);
  r->seconds = plan_seconds(&u, &p, q->tensor_bytes, &env, r->op_ct, r->op_seconds);
  return 0;
}

int64_t oracle_ct_allreduce(int32_t depth, const int64_t* dims, int32_t rank,
                            const int32_t* map, int64_t local) {
  o_matrix m;
  o_map mp;
  m.depth = depth;
  for (int k = 0; k < depth; ++k) m.dims[k] = dims[k];
  mp.rank = rank;
  for (int i = 0; i < rank; ++i) mp.e[i] = map[i];
  return ct_allreduce(&m, &mp, local);
}

void oracle_ct_allgather_dim(int32_t depth, const int64_t* dims, int32_t rank,
                             const int32_t* map, int32_t g, int64_t local,
                             int64_t* ct, int64_t* repeat, int64_t* gin) {
  o_matrix m;
  o_map mp;
  m.depth = depth;
  for (int k = 0; k < depth; ++k) m.dims[k] = dims[k];
  mp.rank = rank;
  for (int i = 0; i < rank; ++i) mp.e[i] = map[i];
  ct_allgather_dim(&m, &mp, g, local, ct, repeat, gin);
}

/* ------------------------------------------------------------------------ */
/* graph helpers: graph.hpp:131-184                                         */
/* ------------------------------------------------------------------------ */

typedef struct {
  const tp_graph_desc* g;
  int num_ops, num_edges;
} o_graph;

/* graph.hpp:135-140 — first operator with the id */
static int find_op(const tp_graph_desc* g, int id) {
  for (int i = 0; i < g->num_ops; ++i)
    if (g->op_id[i] == id) return i;
  return -1;
}

/* graph.hpp:158-183 (Kahn). Returns 0 on success, fills order. */
static int topo_order(const tp_graph_desc* g, int* order) {
  const int n = g->num_ops;
  int* indeg = (int*)calloc((size_t)n + 1, sizeof(int));
  int* eu = (int*)malloc(sizeof(int) * ((size_t)g->num_edges + 1));
  int* ew = (int*)malloc(sizeof(int) * ((size_t)g->num_edges + 1));
  for (int e = 0; e < g->num_edges; ++e) {
    eu[e] = find_op(g, g->edge_from[e]);
    ew[e] = find_op(g, g->edge_to[e]);
    if (eu[e] < 0 || ew[e] < 0) continue;
    ++indeg[ew[e]];
  }
  /* successor lists in edge order: scan edges per popped node */
  int* ready = (int*)malloc(sizeof(int) * ((size_t)n + 1));
  int nr = 0;
  for (int i = 0; i < n; ++i)
    if (indeg[i] == 0) ready[nr++] = i;
  int no = 0;
  for (int head = 0; head < nr; ++head) {
    const int u = ready[head];
    order[no++] = u;
    for (int e = 0; e < g->num_edges; ++e) {
      if (eu[e] != u || ew[e] < 0) continue;
      if (--indeg[ew[e]] == 0) ready[nr++] = ew[e];
    }
  }
  free(indeg); free(eu); free(ew); free(ready);
  return no == n ? 0 : -1;
}

/* Per-op slot table: the reference keys an operator's layouts by tensor
 * name, the last occurrence's spec winning (layout.hpp:339-347). */
typedef struct {
  int nslots;
  int name[64];
  int spec[64]; /* tensor index of the winning spec */
} o_slots;

static int slot_of(const o_slots* s, int name) {
  for (int i = 0; i < s->nslots; ++i)
    if (s->name[i] == name) return i;
  return -1;
}

static int build_slots(const tp_graph_desc* g, int op, o_slots* s) {
  s->nslots = 0;
  for (int t = g->op_tensor_begin[op]; t < g->op_tensor_begin[op + 1]; ++t) {
    int k = slot_of(s, g->tensor_name[t]);
    if (k < 0) {
      if (s->nslots >= 64) return TP_E_CAPACITY;
      k = s->nslots++;
      s->name[k] = g->tensor_name[t];
    }
    s->spec[k] = t;
  }
  return 0;
}

static int t_rank(const tp_graph_desc* g, int t) {
  return g->tensor_shape_begin[t + 1] - g->tensor_shape_begin[t];
}
static const int64_t* t_shape(const tp_graph_desc* g, int t) {
  return g->shape + g->tensor_shape_begin[t];
}

/* layout.hpp:333-370 — layouts of every slot under strategy s. */
static int derive_layouts(const tp_graph_desc* g, int op, const o_slots* sl,
                          const o_strategy* s, o_layout* lay) {
  for (int k = 0; k < sl->nslots; ++k) {
    const int t = sl->spec[k];
    o_layout* L = &lay[k];
    L->rank = t_rank(g, t);
    if (L->rank > TP_MAX_RANK) return TP_E_CAPACITY;
    for (int i = 0; i < L->rank; ++i) L->shape[i] = t_shape(g, t)[i];
    L->element_size = g->tensor_element_size[t];
    L->m = s->matrix;
    L->map.rank = L->rank;
    for (int i = 0; i < L->rank; ++i) L->map.e[i] = -1;
  }
  const int a0 = g->op_axis_begin[op];
  for (int a = 0; a < s->p; ++a) {
    for (int sl_i = g->axis_slice_begin[a0 + a]; sl_i < g->axis_slice_begin[a0 + a + 1]; ++sl_i) {
      const int k = slot_of(sl, g->slice_tensor[sl_i]);
      if (k < 0) return TP_E_UNKNOWN_SLICE_TENSOR;
      o_layout* L = &lay[k];
      const int dim = g->slice_dim[sl_i];
      if (dim < 0 || dim >= L->rank) return TP_E_CAPACITY;
      if (L->shape[dim] % s->degrees[a] != 0) return TP_E_INDIVISIBLE_EXTENT;
      L->map.e[dim] = s->dmap[a];
    }
  }
  return 0;
}

/* layout.hpp:117-129 */
static double layout_shard_bytes(const o_layout* L) {
  int64_t div = 1;
  for (int i = 0; i < L->rank; ++i)
    if (L->map.e[i] >= 0) div *= m_extent(&L->m, L->map.e[i]);
  int64_t el = 1;
  for (int i = 0; i < L->rank; ++i) el *= L->shape[i];
  return (double)(el / div) * L->element_size;
}

/* graph.hpp:52-54 */
static double layout_bytes(const o_layout* L) {
  int64_t el = 1;
  for (int i = 0; i < L->rank; ++i) el *= L->shape[i];
  return (double)el * L->element_size;
}

/* aux_graph.hpp:120-147 */
static void intra_cost(const tp_graph_desc* g, int op, const o_slots* sl,
                       const o_strategy* s, const o_layout* lay,
                       const o_env* env, double* seconds, double* volume) {
  double sec = 0, vol = 0;
  const int a0 = g->op_axis_begin[op];
  for (int t = g->op_tensor_begin[op]; t < g->op_tensor_begin[op + 1]; ++t) {
    const int name = g->tensor_name[t];
    int64_t group = 1;
    for (int a = 0; a < s->p; ++a) {
      int slices_this = 0;
      for (int q = g->axis_slice_begin[a0 + a]; q < g->axis_slice_begin[a0 + a + 1]; ++q) {
        if (g->slice_tensor[q] == name) { slices_this = 1; break; }
      }
      if (!slices_this) group *= s->degrees[a];
    }
    if (group <= 1) continue;
    const o_layout* L = &lay[slot_of(sl, name)];
    const double sb = layout_shard_bytes(L);
    /* collective_cost_detail kAllReduce, cost_model.hpp:180-186 */
    const double v = allreduce_volume(group, sb);
    const int64_t ct = ct_allreduce(&L->m, &L->map, env->local);
    vol += allreduce_volume(group, sb);
    sec += v / eff_bw(ct, env);
  }
  *seconds = sec;
  *volume = vol;
}

/* aux_graph.hpp:151-167 */
static double node_memory(const tp_graph_desc* g, int op, const o_slots* sl,
                          const o_layout* lay) {
  double bytes = 0;
  const int t0 = g->op_tensor_begin[op];
  const int nin = g->op_num_inputs[op];
  for (int t = t0; t < t0 + nin; ++t) {
    int fed = 0;
    for (int e = 0; e < g->num_edges; ++e) {
      if (g->edge_to[e] == g->op_id[op] && g->edge_tensor[e] == g->tensor_name[t]) { fed = 1; break; }
    }
    if (!fed) bytes += layout_shard_bytes(&lay[slot_of(sl, g->tensor_name[t])]);
  }
  for (int t = t0 + nin; t < g->op_tensor_begin[op + 1]; ++t)
    bytes += layout_shard_bytes(&lay[slot_of(sl, g->tensor_name[t])]);
  return bytes;
}

/* ------------------------------------------------------------------------ */
/* the memo: aux_graph.hpp:257-271, keyed like TensorLayout::operator<      */
/* (layout.hpp:173-179): shape, matrix dims, map of both sides              */
/* ------------------------------------------------------------------------ */

typedef struct {
  uint64_t h;
  int used;
  o_layout f, t; /* only shape/matrix/map compared */
  double sec, vol;
} o_memo_entry;

typedef struct {
  o_memo_entry* slots;
  size_t cap, n;
} o_memo;

static uint64_t mix(uint64_t h, uint64_t v) {
  h ^= v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
  return h * 0xff51afd7ed558ccdULL;
}

static uint64_t layout_hash(uint64_t h, const o_layout* L) {
  h = mix(h, (uint64_t)L->rank);
  for (int i = 0; i < L->rank; ++i) h = mix(h, (uint64_t)L->shape[i]);
  h = mix(h, (uint64_t)L->m.depth);
  for (int k = 0; k < L->m.depth; ++k) h = mix(h, (uint64_t)L->m.dims[k]);
  for (int i = 0; i < L->rank; ++i) h = mix(h, (uint64_t)(int64_t)L->map.e[i]);
  return h;
}

static int layout_key_eq(const o_layout* a, const o_layout* b) {
  if (a->rank != b->rank || a->m.depth != b->m.depth) return 0;
  for (int i = 0; i < a->rank; ++i)
    if (a->shape[i] != b->shape[i] || a->map.e[i] != b->map.e[i]) return 0;
  for (int k = 0; k < a->m.depth; ++k)
    if (a->m.dims[k] != b->m.dims[k]) return 0;
  return 1;
}

/* TensorLayout::operator== (layout.hpp:169-171): spec (name equal here),
 * shape, element size, matrix, map. */
static int layout_full_eq(const o_layout* a, const o_layout* b) {
  return a->element_size == b->element_size && layout_key_eq(a, b);
}

static o_memo_entry* memo_find(o_memo* M, const o_layout* f, const o_layout* t, int* found) {
  if ((M->n + 1) * 2 > M->cap) {
    size_t nc = M->cap ? M->cap * 2 : 1024;
    o_memo_entry* ns = (o_memo_entry*)calloc(nc, sizeof(o_memo_entry));
    for (size_t i = 0; i < M->cap; ++i) {
      if (!M->slots[i].used) continue;
      size_t j = M->slots[i].h & (nc - 1);
      while (ns[j].used) j = (j + 1) & (nc - 1);
      ns[j] = M->slots[i];
    }
    free(M->slots);
    M->slots = ns;
    M->cap = nc;
  }
  const uint64_t h = layout_hash(layout_hash(0x230104285ULL, f), t);
  size_t j = h & (M->cap - 1);
  while (M->slots[j].used) {
    if (M->slots[j].h == h && layout_key_eq(&M->slots[j].f, f) && layout_key_eq(&M->slots[j].t, t)) {
      *found = 1;
      return &M->slots[j];
    }
    j = (j + 1) & (M->cap - 1);
  }
  *found = 0;
  M->slots[j].used = 1;
  M->slots[j].h = h;
  M->slots[j].f = *f;
  M->slots[j].t = *t;
  M->n++;
  return &M->slots[j];
}

/* redistribution.hpp:557-561 then aux_graph.hpp:264-268 */
static int price_pair(const o_layout* f, const o_layout* t, const o_env* env,
                      double* sec, double* vol) {
  o_unified u;
  int st = unify(f, t, &u);
  if (st) return st;
  static __thread o_plan p;
  st = run_inference(u.m.depth, &u.from, &u.to, &p);
  if (st) return st;
  const double bytes = layout_bytes(f);
  *vol = plan_volume(&u, &p, bytes);
  *sec = plan_seconds(&u, &p, bytes, env, NULL, NULL);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* build: aux_graph.hpp:211-315                                             */
/* ------------------------------------------------------------------------ */

static int status_of(int kind) {
  if (kind == 0) return TP_OK;
  if (kind == TP_E_EDGE_TENSOR_MISSING) return TP_ERR_OUT_OF_RANGE;
  if (kind == TP_E_CAPACITY) return TP_ERR_CAPACITY;
  return TP_ERR_TOPOPLAN;
}

int oracle_sizes(const tp_graph_desc* g, const tp_topology_desc* t,
                 int64_t* num_aux_nodes, int64_t* num_aux_edges, int64_t* num_rows) {
  const int64_t N = (int64_t)t->node_count * t->local_device_num;
  int64_t nodes = 0, edges = 0, rows = 0;
  int64_t* cnt = (int64_t*)calloc((size_t)g->num_ops + 1, sizeof(int64_t));
  for (int i = 0; i < g->num_ops; ++i) {
    const int p = g->op_axis_begin[i + 1] - g->op_axis_begin[i];
    cnt[i] = oracle_strategy_count(p, N);
    if (cnt[i] < 0) { free(cnt); return TP_ERR_TOPOPLAN; }
    nodes += cnt[i];
  }
  for (int e = 0; e < g->num_edges; ++e) {
    const int u = find_op(g, g->edge_from[e]), w = find_op(g, g->edge_to[e]);
    if (u < 0 || w < 0) { free(cnt); return TP_ERR_TOPOPLAN; }
    edges += cnt[u] * cnt[w];
    rows += cnt[u];
  }
  free(cnt);
  if (num_aux_nodes) *num_aux_nodes = nodes;
  if (num_aux_edges) *num_aux_edges = edges;
  if (num_rows) *num_rows = rows;
  return TP_OK;
}

static int build_impl(const tp_graph_desc* g, const tp_topology_desc* topo,
                      tp_aux_index* index, tp_cost_tensors* out, int memoize,
                      int32_t* error_kind) {
  int kind = 0;
  const int n_ops = g->num_ops;
  const int64_t N = (int64_t)topo->node_count * topo->local_device_num;
  const o_env env = {topo->intra_bandwidth, topo->inter_bandwidth, topo->local_device_num};

  int* order = (int*)malloc(sizeof(int) * ((size_t)n_ops + 1));
  int64_t* node_base = (int64_t*)calloc((size_t)n_ops + 1, sizeof(int64_t));
  int* strat_off = (int*)calloc((size_t)n_ops + 1, sizeof(int));
  o_slots* slots = (o_slots*)calloc((size_t)n_ops + 1, sizeof(o_slots));
  o_strategy** tables = (o_strategy**)calloc((size_t)n_ops + 1, sizeof(o_strategy*));
  o_layout** layouts = (o_layout**)calloc((size_t)n_ops + 1, sizeof(o_layout*));
  int* in_deg = (int*)calloc((size_t)n_ops + 1, sizeof(int));
  int* out_deg = (int*)calloc((size_t)n_ops + 1, sizeof(int));
  double *n_sec = NULL, *n_vol = NULL, *n_mem = NULL;
  o_memo memo = {NULL, 0, 0};

  /* :223-226 */
  if (n_ops > 0 && topo_order(g, order) != 0) { kind = TP_E_CYCLE; goto done; }
  /* :231-234, graph.hpp:142-154 (by id string) */
  for (int i = 0; i < n_ops; ++i) {
    for (int e = 0; e < g->num_edges; ++e) {
      in_deg[i] += g->edge_to[e] == g->op_id[i];
      out_deg[i] += g->edge_from[e] == g->op_id[i];
    }
  }
  /* node phase :236-253. The reference enumerates then derives op by op,
   * so an enumeration failure at op i only wins over derivation failures of
   * ops >= i: count first, remember the first enumeration failure, derive
   * the ops before it, then report it. */
  int64_t total_nodes = 0;
  int enum_err_op = n_ops, enum_err_kind = 0;
  for (int i = 0; i < n_ops; ++i) {
    const int p = g->op_axis_begin[i + 1] - g->op_axis_begin[i];
    int ek = 0;
    if (!is_pow2(N)) ek = TP_E_DEVICES_NOT_POW2;
    else if (p < 1) ek = TP_E_NO_AXES;
    else if (p > TP_MAX_AXES) ek = TP_E_CAPACITY;
    else ek = build_slots(g, i, &slots[i]);
    if (ek) { enum_err_op = i; enum_err_kind = ek; break; }
    const int64_t S = oracle_strategy_count(p, N);
    tables[i] = (o_strategy*)malloc(sizeof(o_strategy) * (size_t)S);
    enumerate_into(p, N, tables[i], S);
    node_base[i] = total_nodes;
    total_nodes += S;
  }
  for (int i = enum_err_op; i <= n_ops; ++i) node_base[i] = total_nodes;
  n_sec = (double*)malloc(sizeof(double) * (size_t)(total_nodes + 1));
  n_vol = (double*)malloc(sizeof(double) * (size_t)(total_nodes + 1));
  n_mem = (double*)malloc(sizeof(double) * (size_t)(total_nodes + 1));
  for (int i = 0; i < enum_err_op; ++i) {
    const int64_t S = node_base[i + 1] - node_base[i];
    const int ns = slots[i].nslots;
    layouts[i] = (o_layout*)malloc(sizeof(o_layout) * (size_t)(S * ns + 1));
    for (int64_t s = 0; s < S; ++s) {
      o_layout* lay = &layouts[i][s * ns];
      if ((kind = derive_layouts(g, i, &slots[i], &tables[i][s], lay))) goto done;
      const int64_t id = node_base[i] + s;
      intra_cost(g, i, &slots[i], &tables[i][s], lay, &env, &n_sec[id], &n_vol[id]);
      n_mem[id] = node_memory(g, i, &slots[i], lay);
    }
  }

  if (enum_err_kind) { kind = enum_err_kind; goto done; }

  /* edge phase :273-296 */
  int64_t ebase = 0, rbase = 0;
  for (int e = 0; e < g->num_edges; ++e) {
    const int u = find_op(g, g->edge_from[e]), w = find_op(g, g->edge_to[e]);
    if (u < 0 || w < 0) { kind = TP_E_DANGLING_EDGE; goto done; }
    if (index && index->edge_base) index->edge_base[e] = ebase;
    if (index && index->edge_from_op) index->edge_from_op[e] = u;
    if (index && index->edge_to_op) index->edge_to_op[e] = w;
    const int ku = slot_of(&slots[u], g->edge_tensor[e]);
    const int kw = slot_of(&slots[w], g->edge_tensor[e]);
    const int64_t Su = node_base[u + 1] - node_base[u];
    const int64_t Sw = node_base[w + 1] - node_base[w];
    if ((ku < 0 || kw < 0) && Su > 0) { kind = TP_E_EDGE_TENSOR_MISSING; goto done; }
    double pmin_c = 1.0 / 0.0, pmin_v = 1.0 / 0.0; /* pair_min, solver.hpp:254-255 */
    for (int64_t su = 0; su < Su; ++su) {
      const o_layout* from = &layouts[u][su * slots[u].nslots + ku];
      double rmin_c = 1.0 / 0.0, rmin_v = 1.0 / 0.0;
      for (int64_t sw = 0; sw < Sw; ++sw) {
        const o_layout* to = &layouts[w][sw * slots[w].nslots + kw];
        double rs = 0, rv = 0;
        if (!layout_full_eq(from, to)) {
          if (memoize) {
            int found;
            o_memo_entry* me = memo_find(&memo, from, to, &found);
            if (found) {
              rs = me->sec;
              rv = me->vol;
            } else {
              if ((kind = price_pair(from, to, &env, &rs, &rv))) goto done;
              me->sec = rs;
              me->vol = rv;
            }
          } else {
            if ((kind = price_pair(from, to, &env, &rs, &rv))) goto done;
          }
        }
        const int64_t wn = node_base[w] + sw;
        const int64_t idx = ebase + su * Sw + sw;
        const double c = n_sec[wn] + rs;
        const double v = n_vol[wn] + rv;
        const double m = n_mem[wn] / in_deg[w];
        if (out) {
          if (out->edge_cost_s) out->edge_cost_s[idx] = c;
          if (out->edge_volume_bytes) out->edge_volume_bytes[idx] = v;
          if (out->edge_memory_bytes) out->edge_memory_bytes[idx] = m;
          if (out->aux_edge_records) {
            unsigned char* rec = (unsigned char*)out->aux_edge_records + idx * 40;
            int32_t ints[4] = {e, (int32_t)(node_base[u] + su), (int32_t)wn, 0};
            memcpy(rec, ints, 16);
            memcpy(rec + 16, &c, 8);
            memcpy(rec + 24, &v, 8);
            memcpy(rec + 32, &m, 8);
          }
        }
        if (c < rmin_c) rmin_c = c;
        if (v < rmin_v) rmin_v = v;
      }
      if (out && out->row_min_cost_s) out->row_min_cost_s[rbase + su] = rmin_c;
      if (out && out->row_min_volume_bytes) out->row_min_volume_bytes[rbase + su] = rmin_v;
      if (rmin_c < pmin_c) pmin_c = rmin_c;
      if (rmin_v < pmin_v) pmin_v = rmin_v;
    }
    if (out && out->edge_pair_min_cost_s) out->edge_pair_min_cost_s[e] = pmin_c;
    if (out && out->edge_pair_min_volume_bytes) out->edge_pair_min_volume_bytes[e] = pmin_v;
    ebase += Su * Sw;
    rbase += Su;
  }
  if (index && index->edge_base) index->edge_base[g->num_edges] = ebase;

done:
  if (!kind) {
    if (index) {
      if (index->node_base)
        for (int i = 0; i <= n_ops; ++i) index->node_base[i] = node_base[i];
      if (index->in_degree)
        for (int i = 0; i < n_ops; ++i) index->in_degree[i] = in_deg[i];
      if (index->out_degree)
        for (int i = 0; i < n_ops; ++i) index->out_degree[i] = out_deg[i];
      if (index->topo_order)
        for (int i = 0; i < n_ops; ++i) index->topo_order[i] = order[i];
    }
    if (out) {
      const int64_t nn = node_base[n_ops];
      if (out->node_intra_cost_s) memcpy(out->node_intra_cost_s, n_sec, sizeof(double) * (size_t)nn);
      if (out->node_intra_volume_bytes) memcpy(out->node_intra_volume_bytes, n_vol, sizeof(double) * (size_t)nn);
      if (out->node_memory_bytes) memcpy(out->node_memory_bytes, n_mem, sizeof(double) * (size_t)nn);
    }
  }
  for (int i = 0; i < n_ops; ++i) { free(tables[i]); free(layouts[i]); }
  free(order); free(node_base); free(strat_off); free(slots); free(tables); free(layouts);
  free(in_deg); free(out_deg); free(n_sec); free(n_vol); free(n_mem); free(memo.slots);
  if (error_kind) *error_kind = kind;
  return status_of(kind);
}

int oracle_build(const tp_graph_desc* g, const tp_topology_desc* t,
                 tp_aux_index* index, tp_cost_tensors* out, int32_t* error_kind) {
  return build_impl(g, t, index, out, 1, error_kind);
}

int oracle_build_unmemoized(const tp_graph_desc* g, const tp_topology_desc* t,
                            tp_aux_index* index, tp_cost_tensors* out,
                            int32_t* error_kind) {
  return build_impl(g, t, index, out, 0, error_kind);
}
