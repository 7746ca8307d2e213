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
  for (int k = 0; k < kMaxD; ++k) L.mx[k] = 0;
  for (int k = 0; k < kMaxAxes && k < s.depth; ++k) L.mx[k] = s.mx[k];  // (a strategy has at most kMaxAxes dims)
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

// ---------------------------------------------------------------------------
// Unification as a bitmask closure (redistribution.hpp:259-346).
//
// Exponent "positions": device position c (0..n) is the cumulative log2
// extent from the innermost device dim; tensor position c (0..t_i) of dim i
// is the cumulative log2 extent of its parts from the OUTERMOST side. A
// layout mapping tensor dim i to an original device dim m of log2 extent x
// whose lower device position is a places the outer x bits of dim i on that
// dim, outermost first (reexpress_layout, :120-156): tensor position c in
// (0, x) corresponds to device position a + x - c. The reference's restart
// loop (refine_side :167-221 + split_device_dim :226-252) only ever adds
// boundaries forced by
//   R1  a tensor boundary strictly inside a mapped region -> the
//       corresponding device boundary (device split),
//   R2  a device boundary strictly inside a mapped region -> the
//       corresponding tensor boundary (re-expression / part split),
//   R3  both sides share the union of boundaries of each tensor dim,
// and stops exactly when none applies, so its result is the least fixpoint
// of R1-R3 from the step-1 device boundaries (both matrices' cumulative
// products, :270-289). Device boundaries fit one uint32 (n <= 16) and every
// tensor boundary lies inside some region (< n), so the closure is a few
// bit-reversals per region; a part's map is the unified dim whose upper
// device position mirrors the part's start, or -1 once the part starts past
// the region (the "outer sub-part keeps the map" rule, :197-206). The
// divisibility checks of expand_over_run (:92-115) reduce to x <= t_i; every
// other check of the loop holds for power-of-two matrices, and the loop
// needs at most n-1 device splits (< 64 rounds).
// ---------------------------------------------------------------------------

TP_HD uint32_t brev32(uint32_t v) {
#ifdef __CUDA_ARCH__
  return __brev(v);
#else
  v = ((v >> 1) & 0x55555555u) | ((v & 0x55555555u) << 1);
  v = ((v >> 2) & 0x33333333u) | ((v & 0x33333333u) << 2);
  v = ((v >> 4) & 0x0F0F0F0Fu) | ((v & 0x0F0F0F0Fu) << 4);
  v = ((v >> 8) & 0x00FF00FFu) | ((v & 0x00FF00FFu) << 8);
  return (v >> 16) | (v << 16);
#endif
}

TP_HD int popc32(uint32_t v) {
#ifdef __CUDA_ARCH__
  return __popc(v);
#else
  return __builtin_popcount(v);
#endif
}

TP_HD int ffs32(uint32_t v) {  // index of the lowest set bit, v != 0
#ifdef __CUDA_ARCH__
  return __ffs(v) - 1;
#else
  return __builtin_ctz(v);
#endif
}

// bit j (1 <= j < x) of v  ->  bit x - j
TP_HD uint32_t mirror(uint32_t v, int x) { return brev32(v) >> (31 - x); }

TP_HD uint32_t low_bits(int x) {  // x in [0, 32]
#ifdef __CUDA_ARCH__
  uint32_t m;
  asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(m) : "r"(x));  // one instruction (len >= 32: all ones)
  return m;
#else
  return x >= 32 ? 0xffffffffu : ((1u << x) - 1u);
#endif
}

struct Unified {
  int next;          // unified depth
  uint32_t D;        // device boundaries (positions 1..n-1)
  int U;             // unified rank
  int8_t from[kMaxU];
  int8_t to[kMaxU];
  uint8_t ext[kMaxD];
};

// Regions of one side: a[i], x[i] (x = 0: unmapped dim).
struct Regions {
  uint8_t a[kMaxR];
  uint8_t x[kMaxR];
};

TP_HD void regions_of(const Lay& L, int R, Regions& g, uint32_t& D) {
  uint8_t ocum[kMaxD + 1];
  ocum[0] = 0;
  for (int k = 0; k < L.depth; ++k) {
    ocum[k + 1] = (uint8_t)(ocum[k] + L.mx[k]);
    D |= 1u << ocum[k + 1];
  }
  for (int i = 0; i < R; ++i) {
    const int m = L.map[i];
    if (m >= 0 && L.mx[m] > 0) {
      g.a[i] = ocum[m];
      g.x[i] = L.mx[m];
    } else {
      g.a[i] = 0;
      g.x[i] = 0;
    }
  }
}

// A layout in the form the pair kernels consume, precomputed once per
// (edge class, side, strategy): the cumulative device boundaries of its
// matrix and the device region of every tensor dim. For canonical strategy
// matrices (no size-1 dims) equality of descriptors is equality of
// layouts (TensorLayout::operator==, layout.hpp:169-171, minus the spec,
// which is shared by construction).
struct alignas(8) SideDesc {
  uint32_t D;        // bit c set at every cumulative log2 extent c (1..n)
  uint8_t n;         // log2 of the total device count
  uint8_t pad[3];
  uint8_t a[kMaxR];  // lower device position of dim i's region
  uint8_t x[kMaxR];  // log2 extent of the region, 0 = replicated dim
};

TP_HD void side_of(const Lay& L, int R, SideDesc& s) {
  Regions g;
  uint32_t D = 0;
  regions_of(L, R, g, D);
  int n = 0;
  for (int k = 0; k < L.depth; ++k) n += L.mx[k];
  s.D = D;
  s.n = (uint8_t)n;
  s.pad[0] = s.pad[1] = s.pad[2] = 0;
  for (int i = 0; i < kMaxR; ++i) {
    s.a[i] = i < R ? g.a[i] : 0;
    s.x[i] = i < R ? g.x[i] : 0;
  }
}

// Inverse for canonical matrices (used by the array-form fallback).
TP_HD void lay_of(const SideDesc& s, int R, Lay& L) {
  L.depth = 0;
  for (int k = 0; k < kMaxD; ++k) L.mx[k] = 0;
  int prev = 0;
  uint32_t rest = s.D;
  while (rest) {
    const int c = ffs32(rest);
    rest &= rest - 1;
    L.mx[L.depth++] = (uint8_t)(c - prev);
    prev = c;
  }
  for (int i = 0; i < R; ++i)
    L.map[i] = s.x[i] ? (int8_t)popc32(s.D & low_bits(s.a[i] + 1)) : (int8_t)-1;
}

TP_HD bool same_side(const SideDesc& f, const SideDesc& t, int R) {
  if (f.D != t.D || f.n != t.n) return false;
  for (int i = 0; i < R; ++i)
    if (f.a[i] != t.a[i] || f.x[i] != t.x[i]) return false;
  return true;
}

// Returns kOk or an error; fills u (and the trace's part structure).
TP_HD int unify_bits(int R, const Lay& F, const Lay& T, const DimT* dt, Unified& u, Trace* tr) {
  Regions gf, gt;
  uint32_t D = 0;
  regions_of(F, R, gf, D);
  regions_of(T, R, gt, D);
  int n = 0;
  for (int k = 0; k < F.depth; ++k) n += F.mx[k];
  int nt = 0;
  for (int k = 0; k < T.depth; ++k) nt += T.mx[k];
  if (n != nt) return kNotUnifiable;  // :264-268
  if (n > kMaxD) return kCapacity;
  // expand_over_run divisibility (:102-111): the region must fit in t_i
  for (int i = 0; i < R; ++i)
    if (gf.x[i] > dt[i].t) return kFactorization;
  for (int i = 0; i < R; ++i)
    if (gt.x[i] > dt[i].t) return kFactorization;
  D &= ~1u & low_bits(n);  // interior device boundaries only
  uint32_t P[kMaxR];
  for (int i = 0; i < R; ++i) P[i] = 0;
  for (bool changed = true; changed;) {
    changed = false;
    for (int s = 0; s < 2; ++s) {
      const Regions& g = s ? gt : gf;
      for (int i = 0; i < R; ++i) {
        const int x = g.x[i], a = g.a[i];
        if (x < 2) continue;
        const uint32_t win = low_bits(x) & ~1u;
        const uint32_t tb = mirror((D >> a) & win, x) & win;  // R2
        const uint32_t db = (mirror(P[i] & win, x) & win) << a;  // R1
        if ((tb & ~P[i]) | (db & ~D)) changed = true;
        P[i] |= tb;
        D |= db;
      }
    }
  }
  // unified device dims: positions of D plus n
  u.D = D;
  u.next = 0;
  if (n > 0) {
    int prev = 0;
    uint32_t rest = D | (1u << n);
    while (rest) {
      const int c = ffs32(rest);
      rest &= rest - 1;
      u.ext[u.next++] = (uint8_t)(c - prev);
      prev = c;
    }
  }
  // unified axes and maps (:330-345)
  int U = 0;
  for (int i = 0; i < R; ++i) {
    uint32_t bnd = P[i];
    int c = 0;
    for (;;) {
      if (U >= kMaxU) return kCapacity;
      int8_t mf = -1, mt = -1;
      if (c < gf.x[i]) mf = (int8_t)popc32(D & low_bits(gf.a[i] + gf.x[i] - c));
      if (c < gt.x[i]) mt = (int8_t)popc32(D & low_bits(gt.a[i] + gt.x[i] - c));
      u.from[U] = mf;
      u.to[U] = mt;
      const int next_c = bnd ? ffs32(bnd) : (int)dt[i].t;
      if (tr) {
        tr->pe[U] = (uint8_t)(next_c - c);
        tr->plast[U] = bnd == 0;
        tr->pdim[U] = (uint8_t)i;
      }
      ++U;
      if (!bnd) break;
      c = next_c;
      bnd &= bnd - 1;
    }
  }
  u.U = U;
  if (tr) {
    tr->depth = u.next;
    for (int k = 0; k < u.next; ++k) tr->ext[k] = u.ext[k];
    tr->urank = U;
    for (int q = 0; q < U; ++q) {
      tr->from_map[q] = u.from[q];
      tr->to_map[q] = u.to[q];
    }
    tr->nops = 0;
  }
  return kOk;
}

// ct of an AllGather / AllToAll on a device dim of log2 extent ek at lower
// device position te, with log2 in-node repetition rexp (cost_model.hpp:108-135).
TP_HD void ct_fast(int te, int rexp, int ek, int64_t L, int l_log2, int64_t& ct, int64_t& rep, int64_t& gin,
                   int& rep_e, int& gin_e) {
  if (l_log2 >= 0) {
    const int l = l_log2;
    rep_e = rexp < l ? rexp : l;
    rep = (int64_t)1 << rep_e;
    if (te >= l) {
      gin_e = 0;
      ct = (int64_t)1 << (l - rep_e);
    } else {
      const int rem_e = l - te;
      gin_e = ek < rem_e ? ek : rem_e;
      ct = rem_e >= ek ? 0 : ((int64_t)1 << (te - rep_e));
    }
    gin = (int64_t)1 << gin_e;
    return;
  }
  const int64_t pd = (int64_t)1 << ek;
  const int64_t temp = (int64_t)1 << te;
  rep = (int64_t)1 << rexp;
  if (rep > L) rep = L;
  rep_e = gin_e = -1;
  if (temp >= L) {
    gin = 1;
    ct = L / rep;
  } else {
    const int64_t remain = L / temp;
    gin = pd < remain ? pd : remain;
    ct = remain >= pd ? 0 : temp / rep;
  }
}

// Optional per-build tables: inter/ct for small ct and the AllToAll scale
// k(p-k)/(p-1), computed with the reference's expressions (tp_warp.cuh
// make_price_tabs). Null pointers: computed directly.
struct FastTabs {
  const double* bw;     // [65]
  const double* scale;  // [17 * 17]
};

// One AllGather (a2a = false) or AllToAll, the ONE pricing routine of every
// pair form (register, warp, array, op lists): cost_model.hpp:176-230 with
// the plan volume of redistribution.hpp:521-553 added to *vol. Branch-free
// over the op kinds -- lanes of a warp price ops of different kinds without
// diverging -- and still the reference's expressions:
//   AllGather        v = (d-1) * shard            sec = v / B_e(ct)
//   AllToAll, k >= p v = (d-1)/d * shard          sec = v / intra
//   AllToAll         v = (d-1)/d * shard          sec = (scale * v) / B_e(c)
// with shard = bytes / 2^s and (d-1)/d = (d-1) * 2^-ek (both exact), and
// B_e(0) = intra (the table's entry 0), so one division serves all three.
TP_HD double price_fast(bool a2a, int te, int rexp, int ek, int s, double bytes, const Env& env, int l_log2,
                        const FastTabs& tab, double* vol, int64_t* ct_out) {
  if (l_log2 >= 0) {
    // power-of-two local_device_num (every count a power of two): the same
    // quantities as below as 32-bit exponents -- ct_fast's branch, c and cc
    // without 64-bit shifts or divisions; identical doubles (measured: cfg5
    // 0.540 -> 0.505 ms, the table launch prices ~20 M ops)
    const int l = l_log2;
    const int rep_e = rexp < l ? rexp : l;
    int gin_e, ct_e;  // ct = 2^ct_e, or 0 when ct_e < 0
    if (te >= l) {
      gin_e = 0;
      ct_e = l - rep_e;
    } else {
      const int rem_e = l - te;
      gin_e = ek < rem_e ? ek : rem_e;
      ct_e = rem_e >= ek ? -1 : te - rep_e;
    }
    const double shard = bytes * exp2d(-s);  // == bytes / 2^s (exact)
    const double dm1 = (double)((1u << ek) - 1u);
    const double f = a2a ? dm1 * exp2d(-ek) : dm1;  // both exact
    const double v = f * shard;
    *vol += v;
    const bool a2a_intra = a2a && gin_e >= ek;
    const int c_e = l - gin_e - rep_e > 0 ? l - gin_e - rep_e : 0;  // c = max(1, 2^(l - gin_e - rep_e) or 0)
    // the bandwidth's ct: 0 (intra) or 2^e, and eff_bw(2^e) = inter / 2^e = inter * 2^-e exactly
    const bool intra_bw = a2a ? a2a_intra : ct_e < 0;
    const int e = a2a ? c_e : ct_e;
    if (ct_out) *ct_out = intra_bw ? 0 : ((int64_t)1 << e);
    const double bw = intra_bw ? env.intra : env.inter * exp2d(-e);
    double num = v;
    if (a2a && !a2a_intra) {
      const int64_t p = (int64_t)1 << ek, gin = (int64_t)1 << gin_e;
      const double scale = (tab.scale && ek < 17) ? tab.scale[gin_e * 17 + ek]
                                                  : (double)gin * (double)(p - gin) / (double)(p - 1);
      num = scale * v;
    }
    return num / bw;
  }
  const double shard = bytes * exp2d(-s);  // == bytes / 2^s (exact)
  const int64_t p = (int64_t)1 << ek;
  const double d = (double)p;
  int64_t ct, rep, gin;
  int rep_e, gin_e;
  ct_fast(te, rexp, ek, env.local, l_log2, ct, rep, gin, rep_e, gin_e);
  const double f = a2a ? (d - 1) * exp2d(-ek) : (d - 1);  // both exact
  const double v = f * shard;
  *vol += v;
  const bool a2a_intra = a2a && gin >= p;
  int64_t c;  // the AllToAll's inter-node count (cost_model.hpp:213-217)
  if (l_log2 >= 0) c = gin_e + rep_e <= l_log2 ? ((int64_t)1 << (l_log2 - gin_e - rep_e)) : 0;
  else c = env.local / (gin * rep);
  if (c < 1) c = 1;
  const int64_t cc = a2a ? (a2a_intra ? 0 : c) : ct;
  if (ct_out) *ct_out = cc;
  const double bw = a2a_intra ? env.intra : ((tab.bw && cc >= 0 && cc < 65) ? tab.bw[cc] : eff_bw(cc, env));
  double num = v;
  if (a2a && !a2a_intra) {
    const double scale = (tab.scale && gin_e >= 0 && ek < 17) ? tab.scale[gin_e * 17 + ek]
                                                               : (double)gin * (double)(p - gin) / (double)(p - 1);
    num = scale * v;
  }
  return num / bw;
}

// One AllGather (a2a=false) or AllToAll on device dim g with s = log2 of
// the working map's shard divisor (array form): its position is the summed
// extents below g, its in-node repetition those of the dims below g the
// working map does not hold (cnt == 0; cost_model.hpp:115-119).
TP_HD double price_op(bool a2a, int g, const uint8_t* ext, const uint8_t* cnt, int s,
                      double bytes, const Env& env, double* vol, int64_t* ct_out) {
  int te = 0, re = 0;
  for (int k = 0; k < g; ++k) {
    te += ext[k];
    if (cnt[k] == 0) re += ext[k];
  }
  return price_fast(a2a, te, re, ext[g], s, bytes, env, -1, FastTabs{nullptr, nullptr}, vol, ct_out);
}

// unify + inference (:419-451, all2all on) + pricing (:533-553,
// cost_model.hpp:233-263) of one (from, to) pair of power-of-two layouts.
TP_HD int redist_cost(int R, const Lay& F, const Lay& T, const DimT* dt, double bytes,
                      const Env& env, double& sec_out, double& vol_out, Trace* tr) {
  if (R < 0 || R > kMaxR) return kCapacity;
  Unified u;
  int st = unify_bits(R, F, T, dt, u, tr);
  if (st) return st;
  const int U = u.U;
  int8_t* w = u.from;
  const int8_t* to = u.to;
  const uint8_t* ext = u.ext;
  uint8_t cnt[kMaxD];
  int8_t first_to[kMaxD];
  for (int k = 0; k < kMaxD; ++k) {
    cnt[k] = 0;
    first_to[k] = -1;
  }
  int s = 0, mism = 0;
  for (int q = 0; q < U; ++q) {
    if (w[q] >= 0) {
      cnt[w[q]]++;
      s += ext[w[q]];
    }
    mism += w[q] != to[q];
  }
  for (int q = U - 1; q >= 0; --q)
    if (to[q] >= 0) first_to[to[q]] = (int8_t)q;

  double sec = 0, vol = 0;
  int guard = (u.next + 1) * (U + 1) * 4 + 16;
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
          mism -= 1;
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
            mism -= (to[i] == -1) ? 2 : 1;
            w[i] = -1;
            w[j] = (int8_t)k;
            a2a = true;
          }
        }
        progress |= a2a;
      }
    }
    if (!mism) break;
    // InferAllGather (:387-401), else the fallback gather (:403-417)
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
    if (to[gi] == -1) mism -= 1;
  }
  sec_out = sec;
  vol_out = vol;
  return kOk;
}

TP_HD int redist_cost_any(int R, const Lay& F, const Lay& T, const DimT* dt, double bytes,
                          const Env& env, double& sec, double& vol, Trace* tr) {
  return redist_cost(R, F, T, dt, bytes, env, sec, vol, tr);
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
  if (q.rank < 0 || q.rank > kMaxR || q.fdepth > kMaxD || q.tdepth > kMaxD) return kCapacity;
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
