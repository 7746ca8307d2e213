// tp_core.cuh — per-thread algorithms of the B200 cost-tensor engine.
//
// Everything here runs inside one CUDA thread (a strategy, an aux node or a
// (producer strategy, consumer strategy) pair) with fixed-size register /
// local arrays. The arithmetic is re-designed for the GPU rather than
// translated:
//
//  * Every device-matrix extent produced by the strategy enumeration is a
//    power of two (degrees are 2^e, layout.hpp:291-292), so device dims are
//    carried as uint8 log2 exponents and all "x % d" / "x / d" of the
//    reference become exponent compares / subtractions.
//  * A tensor extent E = o * 2^t (o odd) enters the layout unification
//    (redistribution.hpp:259-346) only through t and through whether o > 1:
//    every refinement boundary except the last is a power of two dividing E
//    (a part of a dim is a power of two unless it is the dim's last part,
//    which carries o). Boundaries of one tensor dim are therefore a bitmask
//    of exponents, cuts are bit scans, and the divisibility checks reduce to
//    exponent compares. The unified shape is never materialised (pricing
//    never reads it).
//  * The redistribution sequence (redistribution.hpp:350-451) is priced while
//    it is inferred: each op's cost depends only on the working map before
//    the op (cost_model.hpp:233-263), so no op list is stored; the shard size
//    is tracked as an exponent sum.
//
// Floating-point expressions keep the reference's operation order and are
// compiled with -fmad=false, so results are bit-identical to the CPU.
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define TP_HD __host__ __device__ __forceinline__
#else
#define TP_HD inline
#endif

namespace tpk {

constexpr int kMaxAxes = 8;   // partitionable axes per operator
constexpr int kMaxR = 8;      // tensor rank
constexpr int kMaxD = 16;     // device-matrix depth (log2 of total devices)
constexpr int kMaxPD = 24;    // parts per tensor dim per side
constexpr int kMaxU = 32;     // unified tensor rank
constexpr int kMaxOps = 64;   // plan length (trace export only)

// tp_error_kind of include/taps_b200.h
enum ErrKind : int {
  kOk = 0,
  kCycle = 1,
  kDangling = 2,
  kNotPow2 = 3,
  kNoAxes = 4,
  kUnknownSliceTensor = 5,
  kIndivisible = 6,
  kShapeMismatch = 7,
  kNotUnifiable = 8,
  kFactorization = 9,
  kRefine = 10,
  kDeviceSplit = 11,
  kNoConverge = 12,
  kRefineMismatch = 13,
  kDeadlock = 14,
  kNoTerminate = 15,
  kEdgeTensorMissing = 16,
  kAxisCount = 17,
  kCapacity = 18,
};

// One row of a strategy table (layout.hpp:188-217), exponent form.
struct alignas(32) Strat {
  uint8_t p;
  uint8_t depth;             // canonical matrix depth = number of sharded axes
  uint8_t deg[kMaxAxes];     // log2 degree per axis
  int8_t dmap[kMaxAxes];     // canonical device-dim index per axis, -1 if unsharded
  uint8_t mx[kMaxAxes];      // log2 extent per device dim, index 0 = innermost
  uint8_t pad[6];
};

// A tensor layout over a strategy's canonical matrix.
struct Lay {
  uint8_t depth;
  uint8_t mx[kMaxD];  // log2 extent(k), k = 0 innermost
  int8_t map[kMaxR];  // per tensor dim: device dim or -1
};

// Per tensor dim: E = o * 2^t; `odd` records o > 1.
struct DimT {
  uint8_t t;
  uint8_t odd;
};

struct Env {
  double intra;
  double inter;
  int64_t local;
};

TP_HD int64_t factorial_i(int i) {
  int64_t f = 1;
  for (int k = 2; k <= i; ++k) f *= k;
  return f;
}

// Closed-form strategy count (layout.hpp:222-244).
TP_HD int64_t strategy_count(int p, int n) {
  if (n == 0) return 1;
  int64_t count = 0, fact = 1;
  const int lim = p < n ? p : n;
  for (int i = 1; i <= lim; ++i) {
    fact *= i;
    int64_t c1 = 1, c2 = 1;
    for (int j = 0; j < i; ++j) c1 = c1 * (p - j) / (j + 1);
    for (int j = 0; j < i - 1; ++j) c2 = c2 * (n - 1 - j) / (j + 1);
    count += fact * c1 * c2;
  }
  return count;
}

// Strategy `s` of the sorted enumeration (layout.hpp:270-328) by unranking:
// degree tuples ascend lexicographically (= exponent compositions in lex
// order), and within one tuple the placements of the i sharded axes run in
// DESCENDING lexicographic order, i.e. ascending rank i!-1-r.
TP_HD void unrank_strategy(int p, int n, int64_t s, Strat& out) {
  int exps[kMaxAxes];
  for (int a = 0; a < p; ++a) exps[a] = 0;
  exps[p - 1] = n;
  int64_t acc = 0, r = 0;
  int nsh = 0;
  for (;;) {
    nsh = 0;
    for (int a = 0; a < p; ++a) nsh += exps[a] > 0;
    const int64_t cnt = factorial_i(nsh);
    if (s < acc + cnt) {
      r = s - acc;
      break;
    }
    acc += cnt;
    // next composition, first part varying slowest (layout.hpp:249-263)
    int k = p - 2, prefix = 0;
    for (; k >= 0; --k) {
      prefix = 0;
      for (int a = 0; a <= k; ++a) prefix += exps[a];
      if (prefix < n) break;
    }
    if (k < 0) break;  // s out of range: leaves the last composition
    exps[k] += 1;
    prefix += 1;
    for (int a = k + 1; a < p - 1; ++a) exps[a] = 0;
    exps[p - 1] = n - prefix;
  }
  out.p = (uint8_t)p;
  out.depth = (uint8_t)nsh;
  for (int a = 0; a < kMaxAxes; ++a) {
    out.deg[a] = a < p ? (uint8_t)exps[a] : 0;
    out.dmap[a] = -1;
    out.mx[a] = 0;
  }
  for (int q = 0; q < 6; ++q) out.pad[q] = 0;
  // Lehmer decode of ascending rank q over positions {0..nsh-1}
  int64_t q = factorial_i(nsh) - 1 - r;
  int avail[kMaxAxes];
  for (int j = 0; j < nsh; ++j) avail[j] = j;
  int navail = nsh, j = 0;
  for (int a = 0; a < p; ++a) {
    if (exps[a] == 0) continue;
    const int64_t f = factorial_i(nsh - 1 - j);
    const int idx = (int)(q / f);
    q %= f;
    const int pos = avail[idx];
    for (int t = idx; t + 1 < navail; ++t) avail[t] = avail[t + 1];
    --navail;
    out.dmap[a] = (int8_t)pos;
    out.mx[pos] = (uint8_t)exps[a];
    ++j;
  }
}

// Layout of a tensor whose dim d is sliced by axis sa[d] (or -1), under
// strategy s (layout.hpp:333-370 restricted to one tensor).
TP_HD void side_layout(const Strat& s, const int8_t* sa, int R, Lay& L) {
  L.depth = s.depth;
  for (int k = 0; k < kMaxD; ++k) L.mx[k] = k < s.depth ? s.mx[k] : 0;
  for (int d = 0; d < R; ++d) L.map[d] = sa[d] >= 0 ? s.dmap[sa[d]] : (int8_t)-1;
}

TP_HD bool same_layout(const Lay& a, const Lay& b, int R) {
  if (a.depth != b.depth) return false;
  for (int k = 0; k < a.depth; ++k)
    if (a.mx[k] != b.mx[k]) return false;
  for (int d = 0; d < R; ++d)
    if (a.map[d] != b.map[d]) return false;
  return true;
}

// 2^e as an exact double.
TP_HD double exp2d(int e) {
  union {
    uint64_t u;
    double d;
  } v;
  v.u = (uint64_t)(1023 + e) << 52;
  return v.d;
}

TP_HD double eff_bw(int64_t ct, const Env& env) {  // cost_model.hpp:148-151
  if (ct <= 0) return env.intra;
  return env.inter / (double)ct;
}

// Optional trace of one redistribution for the verification export.
struct Trace {
  int depth;
  uint8_t ext[kMaxD];       // unified exts, index 0 innermost (log2)
  int urank;
  uint8_t pe[kMaxU];        // log2 of each unified part (odd factor on a dim's last part)
  uint8_t plast[kMaxU];     // 1 if the part is its dim's last part
  uint8_t pdim[kMaxU];      // original tensor dim of each unified part
  int8_t from_map[kMaxU];
  int8_t to_map[kMaxU];
  int nops;
  int8_t ops[kMaxOps][5];
  int64_t ct[kMaxOps];
  double sec[kMaxOps];
};

// Unification state of one side: parts of each tensor dim, outer first.
template <int RM>
struct Parts {
  uint8_t n[RM];
  uint8_t e[RM][kMaxPD];
  int8_t m[RM][kMaxPD];
};

// redistribution.hpp:120-156 (re-expression over the step-1 unified matrix),
// including expand_over_run (:92-115).
template <int RM>
TP_HD int reexpress(const Lay& L, const DimT* dt, const uint8_t* ext, int next, Parts<RM>& P, int R) {
  uint8_t ocum[kMaxD + 1], ucum[kMaxD + 1];
  ocum[0] = 0;
  for (int k = 0; k < L.depth; ++k) ocum[k + 1] = (uint8_t)(ocum[k] + L.mx[k]);
  ucum[0] = 0;
  for (int u = 0; u < next; ++u) ucum[u + 1] = (uint8_t)(ucum[u] + ext[u]);
  // every original dim of extent > 1 must be covered by unified dims (:140)
  for (int k = 0; k < L.depth; ++k) {
    if (L.mx[k] == 0) continue;
    bool any = false;
    for (int u = next - 1; u >= 0; --u)
      any |= ucum[u] >= ocum[k] && ucum[u + 1] <= ocum[k + 1] && ext[u] > 0;
    if (!any) return kNotUnifiable;
  }
  for (int i = 0; i < R; ++i) {
    const int m = L.map[i];
    if (m < 0 || L.mx[m] == 0) {
      P.n[i] = 1;
      P.e[i][0] = dt[i].t;
      P.m[i][0] = -1;
      continue;
    }
    int rem = dt[i].t, np = 0, last = -1;
    for (int u = next - 1; u >= 0; --u) {  // run_of[m], outer to inner
      if (!(ucum[u] >= ocum[m] && ucum[u + 1] <= ocum[m + 1] && ext[u] > 0)) continue;
      if (last >= 0) {  // the previous run member was not the last one
        if (rem < ext[last]) return kFactorization;
        P.e[i][np] = ext[last];
        P.m[i][np] = (int8_t)last;
        ++np;
        rem -= ext[last];
      }
      last = u;
    }
    if (rem < ext[last]) return kFactorization;
    P.e[i][np] = (uint8_t)rem;
    P.m[i][np] = (int8_t)last;
    P.n[i] = (uint8_t)(np + 1);
  }
  return kOk;
}

// redistribution.hpp:167-221 on one dim. Returns kOk (refined), -1 (device
// split requested: *sk, *sy) or an error. Boundaries: bit c of `bmask` set
// for every power-of-two boundary 2^c.
template <int RM>
TP_HD int refine_dim(Parts<RM>& P, int i, uint64_t bmask, const DimT& dt, const uint8_t* ext,
                     int* sk, int* sy) {
  uint8_t ne[kMaxPD];
  int8_t nm[kMaxPD];
  int nn = 0, pos = 0;
  const int n = P.n[i];
  for (int j = 0; j < n; ++j) {
    const int e = P.e[i][j], m = P.m[i][j];
    const int end = pos + e;
    const int limit = (j == n - 1) ? end + (dt.odd ? 1 : 0) : end;  // cut c inside iff pos < c < limit
    uint64_t cuts = 0;
    if (limit > pos + 1) {
      const uint64_t hi = limit >= 64 ? ~0ull : ((1ull << limit) - 1ull);
      const uint64_t lo = (pos + 1) >= 64 ? ~0ull : ((1ull << (pos + 1)) - 1ull);
      cuts = bmask & hi & ~lo;
    }
    if (cuts == 0) {
      if (nn >= kMaxPD) return kCapacity;
      ne[nn] = (uint8_t)e;
      nm[nn] = (int8_t)m;
      ++nn;
    } else {
      int c1 = 0;
      while (!((cuts >> c1) & 1ull)) ++c1;
      if (m >= 0 && c1 - pos < ext[m]) {  // d % f1 == 0 && f1 > 1: split
        *sk = m;
        *sy = c1 - pos;
        return -1;
      }
      // replicated part, or mapped part whose outer piece keeps the map
      int prev = pos;
      bool first = true;
      for (int c = c1; c < 64; ++c) {
        if (!((cuts >> c) & 1ull)) continue;
        if (nn >= kMaxPD) return kCapacity;
        ne[nn] = (uint8_t)(c - prev);
        nm[nn] = (int8_t)((first && m >= 0) ? m : -1);
        ++nn;
        prev = c;
        first = false;
      }
      if (nn >= kMaxPD) return kCapacity;
      ne[nn] = (uint8_t)(end - prev);
      nm[nn] = -1;
      ++nn;
    }
    pos = end;
  }
  P.n[i] = (uint8_t)nn;
  for (int j = 0; j < nn; ++j) {
    P.e[i][j] = ne[j];
    P.m[i][j] = nm[j];
  }
  return kOk;
}

// redistribution.hpp:226-252
template <int RM>
TP_HD int split_device_dim(uint8_t* ext, int& next, int k, int y, Parts<RM>& A, Parts<RM>& B, int R) {
  if (next + 1 > kMaxD) return kCapacity;
  const int inner = ext[k] - y;
  ext[k] = (uint8_t)inner;
  for (int u = next; u > k + 1; --u) ext[u] = ext[u - 1];
  ext[k + 1] = (uint8_t)y;
  ++next;
  Parts<RM>* sides[2] = {&A, &B};
  for (int s = 0; s < 2; ++s) {
    Parts<RM>& P = *sides[s];
    for (int i = 0; i < R; ++i) {
      uint8_t ne[kMaxPD];
      int8_t nm[kMaxPD];
      int nn = 0;
      for (int j = 0; j < P.n[i]; ++j) {
        const int e = P.e[i][j], m = P.m[i][j];
        if (m == k) {
          if (e < y || e - y < inner) return kDeviceSplit;
          if (nn + 2 > kMaxPD) return kCapacity;
          ne[nn] = (uint8_t)y;
          nm[nn++] = (int8_t)(k + 1);
          ne[nn] = (uint8_t)(e - y);
          nm[nn++] = (int8_t)k;
        } else {
          if (nn >= kMaxPD) return kCapacity;
          ne[nn] = (uint8_t)e;
          nm[nn++] = (int8_t)(m > k ? m + 1 : m);
        }
      }
      P.n[i] = (uint8_t)nn;
      for (int j = 0; j < nn; ++j) {
        P.e[i][j] = ne[j];
        P.m[i][j] = nm[j];
      }
    }
  }
  return kOk;
}

template <int RM>
TP_HD uint64_t boundary_mask(const Parts<RM>& P, int i) {
  uint64_t b = 0;
  int c = 0;
  for (int j = 0; j + 1 < P.n[i]; ++j) {  // the last cumulative product is E
    c += P.e[i][j];
    b |= 1ull << c;
  }
  return b;
}

// Shard-size bookkeeping and the per-op price (cost_model.hpp:176-263) for
// the working map `w` (unified rank u) BEFORE the op.
struct PriceState {
  int s;  // sum of log2 extents of mapped entries of the working map
};

// infer_ct_allgather_dim (cost_model.hpp:108-135) with cnt[k] = number of
// working-map entries equal to k.
TP_HD void ct_gather(const uint8_t* ext, const uint8_t* cnt, int g, int64_t L, int64_t& ct,
                     int64_t& rep, int64_t& gin) {
  const int64_t pd = (int64_t)1 << ext[g];
  int te = 0, re = 0;
  for (int k = 0; k < g; ++k) {
    te += ext[k];
    if (cnt[k] == 0) re += ext[k];
  }
  const int64_t temp = (int64_t)1 << te;
  rep = (int64_t)1 << re;
  if (rep > L) rep = L;
  if (temp >= L) {
    gin = 1;
    ct = L / rep;
  } else {
    const int64_t remain = L / temp;
    gin = pd < remain ? pd : remain;
    ct = remain >= pd ? 0 : temp / rep;
  }
}

// One AllGather (a2a=false) or AllToAll on device dim g: returns seconds and
// adds the plan volume (redistribution.hpp:521-553) to *vol.
TP_HD double price_op(bool a2a, int g, const uint8_t* ext, const uint8_t* cnt, int s,
                      double bytes, const Env& env, double* vol, int64_t* ct_out) {
  const double shard = bytes / exp2d(s);
  const int64_t p = (int64_t)1 << ext[g];
  const double d = (double)p;
  int64_t ct, rep, gin;
  ct_gather(ext, cnt, g, env.local, ct, rep, gin);
  if (!a2a) {
    *vol += (d - 1) * shard;
    const double v = (double)(p - 1) * shard;
    if (ct_out) *ct_out = ct;
    return v / eff_bw(ct, env);
  }
  *vol += (d - 1) / d * shard;
  const double v = (d - 1) / d * shard;
  const int64_t k = gin;
  if (k >= p) {
    if (ct_out) *ct_out = 0;
    return v / env.intra;
  }
  int64_t c = env.local / (k * rep);
  if (c < 1) c = 1;
  if (ct_out) *ct_out = c;
  const double bw = eff_bw(c, env);
  const double scale = (double)k * (double)(p - k) / (double)(p - 1);
  return scale * v / bw;
}

// unify (redistribution.hpp:259-346) + inference (:419-451, all2all on) +
// pricing (:533-553, cost_model.hpp:233-263) of one (from, to) pair.
// Inputs are layouts over power-of-two matrices with equal totals.
template <int RM>
TP_HD int redist_cost(int R, const Lay& F, const Lay& T, const DimT* dt, double bytes, const Env& env,
                      double& sec_out, double& vol_out, Trace* tr) {
  // ---- step 1: unified matrix = union of inner cumulative exponents ----
  uint32_t cm = 0;
  {
    int c = 0;
    for (int k = 0; k < F.depth; ++k) {
      c += F.mx[k];
      if (c > 0) cm |= 1u << c;
    }
    c = 0;
    for (int k = 0; k < T.depth; ++k) {
      c += T.mx[k];
      if (c > 0) cm |= 1u << c;
    }
  }
  uint8_t ext[kMaxD + 1];
  int next = 0;
  {
    int prev = 0;
    for (int c = 1; c < 32; ++c) {
      if (!((cm >> c) & 1u)) continue;
      if (next >= kMaxD) return kCapacity;
      ext[next++] = (uint8_t)(c - prev);
      prev = c;
    }
  }
  Parts<RM> A, B;
  int st = reexpress<RM>(F, dt, ext, next, A, R);
  if (st) return st;
  st = reexpress<RM>(T, dt, ext, next, B, R);
  if (st) return st;

  // ---- step 2: refine the shape, splitting device dims on demand ----
  for (int rounds = 1;; ++rounds) {
    if (rounds > 64) return kNoConverge;
    bool restarted = false;
    for (int i = 0; i < R && !restarted; ++i) {
      const uint64_t bm = boundary_mask<RM>(A, i) | boundary_mask<RM>(B, i);
      int sk = -1, sy = 0;
      int r = refine_dim<RM>(A, i, bm, dt[i], ext, &sk, &sy);
      if (r == kOk) r = refine_dim<RM>(B, i, bm, dt[i], ext, &sk, &sy);
      if (r == -1) {
        st = split_device_dim<RM>(ext, next, sk, sy, A, B, R);
        if (st) return st;
        restarted = true;
      } else if (r != kOk) {
        return r;
      }
    }
    if (!restarted) break;
  }

  // ---- read-off (:330-345) ----
  int8_t w[kMaxU], to[kMaxU];
  int U = 0;
  for (int i = 0; i < R; ++i) {
    if (A.n[i] != B.n[i]) return kRefineMismatch;
    for (int j = 0; j < A.n[i]; ++j) {
      if (A.e[i][j] != B.e[i][j]) return kRefineMismatch;
      if (U >= kMaxU) return kCapacity;
      if (tr) {
        tr->pe[U] = A.e[i][j];
        tr->plast[U] = j == A.n[i] - 1;
        tr->pdim[U] = (uint8_t)i;
      }
      w[U] = A.m[i][j];
      to[U] = B.m[i][j];
      ++U;
    }
  }
  if (tr) {
    tr->depth = next;
    for (int k = 0; k < next; ++k) tr->ext[k] = ext[k];
    tr->urank = U;
    for (int u = 0; u < U; ++u) {
      tr->from_map[u] = w[u];
      tr->to_map[u] = to[u];
    }
    tr->nops = 0;
  }

  // ---- inference with on-the-fly pricing ----
  uint8_t cnt[kMaxD];
  int8_t first_to[kMaxD];
  for (int k = 0; k < kMaxD; ++k) {
    cnt[k] = 0;
    first_to[k] = -1;
  }
  int s = 0;
  for (int u = 0; u < U; ++u) {
    if (w[u] >= 0) {
      cnt[w[u]]++;
      s += ext[w[u]];
    }
  }
  for (int u = U - 1; u >= 0; --u)
    if (to[u] >= 0) first_to[to[u]] = (int8_t)u;
  int mism = 0;
  for (int u = 0; u < U; ++u) mism += w[u] != to[u];

  double sec = 0, vol = 0;
  int guard = (next + 1) * (U + 1) * 4 + 16;
  auto record = [&](int kind, int k, int i, int j, int fb, int64_t ct, double sc) {
    if (!tr) return;
    if (tr->nops >= kMaxOps) {
      tr->nops = kMaxOps + 1;
      return;
    }
    int8_t* o = tr->ops[tr->nops];
    o[0] = (int8_t)kind;
    o[1] = (int8_t)k;
    o[2] = (int8_t)i;
    o[3] = (int8_t)j;
    o[4] = (int8_t)fb;
    tr->ct[tr->nops] = ct;
    tr->sec[tr->nops] = sc;
    tr->nops++;
  };
  while (mism) {
    if (--guard < 0) return kNoTerminate;
    bool progress = true;
    while (progress) {
      // InferSlice (:350-365)
      progress = false;
      for (int i = 0; i < U; ++i) {
        const int k = to[i];
        if (w[i] == -1 && k >= 0 && cnt[k] == 0) {
          record(0, k, i, -1, 0, 0, 0.0);
          w[i] = (int8_t)k;
          cnt[k]++;
          s += ext[k];
          mism -= 1;  // w[i] now equals to[i]
          progress = true;
        }
      }
      // InferAll2All until none applies (:367-385)
      bool a2a = true;
      while (a2a) {
        a2a = false;
        for (int i = 0; i < U; ++i) {
          const int k = w[i];
          if (k < 0 || to[i] == k) continue;
          const int j = first_to[k];
          if (j >= 0 && j != i && w[j] == -1) {
            int64_t ct = 0;
            const double c = price_op(true, k, ext, cnt, s, bytes, env, &vol, tr ? &ct : nullptr);
            sec += c;
            record(2, k, i, j, 0, ct, c);
            // w[i]: k -> -1 ; w[j]: -1 -> k (to[j] == k)
            mism += (to[i] == -1) ? -1 : 0;
            mism -= 1;
            w[i] = -1;
            w[j] = (int8_t)k;
            a2a = true;
          }
        }
        progress |= a2a;
      }
    }
    if (!mism) break;
    // InferAllGather (:387-401), else the fallback (:403-417)
    int gi = -1, fb = 0;
    for (int i = 0; i < U; ++i) {
      if (w[i] >= 0 && to[i] == -1) {
        gi = i;
        break;
      }
    }
    if (gi < 0) {
      for (int i = 0; i < U; ++i) {
        if (w[i] != to[i] && w[i] >= 0) {
          gi = i;
          fb = 1;
          break;
        }
      }
      if (gi < 0) return kDeadlock;
    }
    const int k = w[gi];
    int64_t ct = 0;
    const double c = price_op(false, k, ext, cnt, s, bytes, env, &vol, tr ? &ct : nullptr);
    sec += c;
    record(1, k, gi, -1, fb, ct, c);
    w[gi] = -1;
    cnt[k]--;
    s -= ext[k];
    mism += (to[gi] == -1) ? -1 : 0;  // a regular gather fixes the entry
    if (fb) mism += 0;                // a fallback gather leaves it mismatched
  }
  sec_out = sec;
  vol_out = vol;
  return kOk;
}

// Dispatch on the tensor rank: rank <= 2 covers every model builder.
TP_HD int redist_cost_any(int R, const Lay& F, const Lay& T, const DimT* dt, double bytes,
                          const Env& env, double& sec, double& vol, Trace* tr) {
  if (R == 2) return redist_cost<2>(2, F, T, dt, bytes, env, sec, vol, tr);
  if (R >= 1 && R <= 4) return redist_cost<4>(R, F, T, dt, bytes, env, sec, vol, tr);
  if (R >= 5 && R <= kMaxR) return redist_cost<kMaxR>(R, F, T, dt, bytes, env, sec, vol, tr);
  // rank 0: both maps empty, equal layouts; nothing to move
  sec = 0;
  vol = 0;
  return R == 0 ? kOk : kCapacity;
}

// ---------------------------------------------------------------------------
// Verification export: one arbitrary redistribution query
// (redistribution.hpp:557-561 + plan_volume + redistribution_cost).
// ---------------------------------------------------------------------------
struct QueryPOD {
  int32_t rank;
  int32_t fdepth, tdepth;
  int32_t local;
  int64_t shape[kMaxR];
  int64_t fdims[kMaxD];  // outermost first, as DeviceMatrix::dims
  int64_t tdims[kMaxD];
  int32_t fmap[kMaxR];
  int32_t tmap[kMaxR];
  double bytes, intra, inter;
};

TP_HD int ilog2_exact(int64_t v) {  // -1 unless v is a power of two
  if (v <= 0 || (v & (v - 1))) return -1;
  int e = 0;
  while (((int64_t)1 << e) < v) ++e;
  return e;
}

TP_HD int ctz64(int64_t v) {
  int t = 0;
  while (t < 63 && !((v >> t) & 1)) ++t;
  return t;
}

// Fills a tp_redist_result-shaped record; returns the tp_error_kind.
template <typename Result>
TP_HD int run_query(const QueryPOD& q, Result& r) {
  r.status = 0;
  r.depth = 0;
  r.urank = 0;
  r.num_ops = 0;
  r.volume_bytes = 0;
  r.seconds = 0;
  if (q.rank < 0 || q.rank > kMaxR || q.fdepth > kMaxAxes || q.tdepth > kMaxAxes) return kCapacity;
  Lay F, T;
  F.depth = (uint8_t)q.fdepth;
  T.depth = (uint8_t)q.tdepth;
  int64_t ftot = 1, ttot = 1;
  for (int k = 0; k < kMaxD; ++k) F.mx[k] = T.mx[k] = 0;
  for (int k = 0; k < q.fdepth; ++k) {
    const int e = ilog2_exact(q.fdims[q.fdepth - 1 - k]);
    if (e < 0) return kCapacity;  // non-power-of-two device dims: not produced by enumeration
    F.mx[k] = (uint8_t)e;
    ftot *= q.fdims[k];
  }
  for (int k = 0; k < q.tdepth; ++k) {
    const int e = ilog2_exact(q.tdims[q.tdepth - 1 - k]);
    if (e < 0) return kCapacity;
    T.mx[k] = (uint8_t)e;
    ttot *= q.tdims[k];
  }
  DimT dt[kMaxR];
  for (int i = 0; i < q.rank; ++i) {
    if (q.shape[i] < 1) return kCapacity;
    if (q.fmap[i] < -1 || q.fmap[i] >= q.fdepth || q.tmap[i] < -1 || q.tmap[i] >= q.tdepth)
      return kCapacity;
    F.map[i] = (int8_t)q.fmap[i];
    T.map[i] = (int8_t)q.tmap[i];
    dt[i].t = (uint8_t)ctz64(q.shape[i]);
    dt[i].odd = (q.shape[i] >> dt[i].t) > 1;
  }
  if (ftot != ttot) return kNotUnifiable;
  Env env{q.intra, q.inter, (int64_t)q.local};
  Trace tr;
  double sec = 0, vol = 0;
  const int st = redist_cost_any(q.rank, F, T, dt, q.bytes, env, sec, vol, &tr);
  if (st) return st;
  if (tr.nops > kMaxOps) return kCapacity;
  r.depth = tr.depth;
  for (int k = 0; k < tr.depth; ++k) r.dims[k] = (int64_t)1 << tr.ext[tr.depth - 1 - k];
  r.urank = tr.urank;
  for (int u = 0; u < tr.urank; ++u) {
    const int i = tr.pdim[u];
    const int64_t odd = q.shape[i] >> dt[i].t;
    r.shape[u] = ((int64_t)1 << tr.pe[u]) * (tr.plast[u] ? odd : 1);
    r.from_map[u] = tr.from_map[u];
    r.to_map[u] = tr.to_map[u];
  }
  r.num_ops = tr.nops;
  for (int o = 0; o < tr.nops; ++o) {
    for (int f = 0; f < 5; ++f) r.ops[o][f] = tr.ops[o][f];
    r.op_ct[o] = tr.ct[o];
    r.op_seconds[o] = tr.sec[o];
  }
  r.volume_bytes = vol;
  r.seconds = sec;
  return kOk;
}

}  // namespace tpk
