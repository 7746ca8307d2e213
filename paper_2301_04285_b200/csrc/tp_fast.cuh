// tp_fast.cuh — register-resident pricing of one (from, to) pair per thread.
//
// The kernels' pair path. Same algorithm as tp_core.cuh's redist_cost (the
// bitmask-closure unification, then the reference's greedy inference priced
// on the fly), with every per-axis array packed into registers:
//   * unified maps: 8-bit fields (device dim + 1, 0 = replicated) in four
//     uint64 words per map (<= 32 unified axes);
//   * the position sets the inference scans — occupied (w >= 0), targeted
//     (to >= 0), matched (w == to) — are uint32 masks, so InferSlice /
//     InferAll2All / InferAllGather (redistribution.hpp:350-417) visit only
//     candidate positions via find-first-set;
//   * to.axis_of(k) is precomputed per device dim; "k in the working map" is
//     a device-dim mask and the ct repetition (cost_model.hpp:115-119) is a
//     popcount over the mask of device BITS the working map holds;
//   * with a power-of-two local_device_num the ct divisions are shifts.
// A working map that holds one device dim twice (an axis slicing two dims
// of one tensor) needs multiplicity counts; such pairs take the array form
// (tp_core.cuh redist_cost) instead.
#pragma once

#include "tp_core.cuh"

namespace tpk {

struct Pack4 {  // 32 x 8-bit fields
  uint64_t w[4];
};

TP_HD int pget(const Pack4& p, int i) {
  const int q = i >> 3;
  const uint64_t word = q == 0 ? p.w[0] : (q == 1 ? p.w[1] : (q == 2 ? p.w[2] : p.w[3]));
  return (int)((word >> ((i & 7) * 8)) & 0xffu);
}

TP_HD void pset(Pack4& p, int i, int v) {
  const int q = i >> 3, sh = (i & 7) * 8;
  const uint64_t clr = ~(0xffull << sh), val = (uint64_t)(v & 0xff) << sh;
  if (q == 0) p.w[0] = (p.w[0] & clr) | val;
  else if (q == 1) p.w[1] = (p.w[1] & clr) | val;
  else if (q == 2) p.w[2] = (p.w[2] & clr) | val;
  else p.w[3] = (p.w[3] & clr) | val;
}

struct Pack2 {  // 16 x 8-bit fields
  uint64_t lo, hi;
};

TP_HD int p2get(const Pack2& p, int i) {
  return (int)(((i < 8 ? p.lo : p.hi) >> ((i & 7) * 8)) & 0xffu);
}

TP_HD void p2set(Pack2& p, int i, int v) {
  const int sh = (i & 7) * 8;
  const uint64_t clr = ~(0xffull << sh), val = (uint64_t)(v & 0xff) << sh;
  if (i < 8) p.lo = (p.lo & clr) | val;
  else p.hi = (p.hi & clr) | val;
}

// Scenarios that differ only in their bandwidths share a pair's unification,
// op sequence, volumes and ct: the op list is inferred once and priced for
// every member environment (members 1..g-1; member 0 is the caller's own env),
// each member's seconds summed in op order like the reference's.
#ifndef TP_GROUP_MAX
#define TP_GROUP_MAX 16  // measured on cfg5: 4 / 8 / 16 / 32 / 64 -> 3.05 / 2.55 / 2.26 / 2.62 / 3.53 ms
#endif
constexpr int kGroupMax = TP_GROUP_MAX;
// The members of a bandwidth group. Member q's Env and bandwidth table are
// read in place from its argument block (base + idx[q] * stride) and its
// seconds accumulate in sec[q * sec_stride] (shared memory on the device):
// no per-member copies or read-modify-writes in local memory.
constexpr int kBwEntries = 65;  // bw[] entries before the scale table (== kBwTab, tp_warp.cuh)

struct MultiSec {
  int g;
  const char* base;
  const int32_t* idx;
  int stride, env_off, bw_off;
  double* sec;
  int sec_stride;
  TP_HD const char* blk(int q) const { return base + (size_t)idx[q] * stride; }
  TP_HD const Env& env(int q) const { return *reinterpret_cast<const Env*>(blk(q) + env_off); }
  TP_HD FastTabs tab(int q) const {
    const double* bw = *reinterpret_cast<const double* const*>(blk(q) + bw_off);
    return FastTabs{bw, bw + kBwEntries};
  }
  TP_HD double& s(int q) { return sec[q * sec_stride]; }
};

#if defined(__CUDACC__)
#define TP_HD_NOINL __host__ __device__ __noinline__
#else
#define TP_HD_NOINL inline  // host builds (tests/devcheck)
#endif

// One op priced for members 1..g-1 (out of line: one copy of the code for
// both call sites keeps the kernels' instruction footprint small).
TP_HD_NOINL void price_members(MultiSec* ms, bool a2a, int pos, int rexp, int e, int s, double bytes,
                                  int l_log2) {
  for (int q = 1; q < ms->g; ++q) {
    double dv = 0;
    ms->s(q) += price_fast(a2a, pos, rexp, e, s, bytes, ms->env(q), l_log2, ms->tab(q), &dv, nullptr);
  }
}

// The op list of one pair, recorded instead of priced (kRecord): an op is
// priced by price_fast from (AllToAll?, lower position, in-node repetition
// exponent, log2 extent, shard exponent) alone, all of which the inference
// fixes independently of the tensor bytes and the bandwidths. A sweep infers
// each distinct (layouts, dims) pair once and prices it per scenario
// (price_ops): the same additions in the same order as pricing on the fly.
constexpr int kOpWords = 16;  // header + up to 15 ops (64 B)
constexpr uint32_t kOpsSame = 1u << 16;  // from == to: no redistribution (aux_graph.hpp:169-171, 260)
constexpr uint32_t kOpsFull = 1u << 17;  // not representable: price with pair_cost_sd
struct OpRec {
  uint32_t w[kOpWords];
  int n;
  TP_HD bool push(bool a2a, int pos, int rexp, int e, int s) {
    if (n >= kOpWords - 1) return false;
    w[1 + n++] = (uint32_t)a2a | ((uint32_t)pos << 1) | ((uint32_t)rexp << 6) | ((uint32_t)e << 11) |
                 ((uint32_t)s << 16);
    return true;
  }
};

TP_HD void price_ops(const uint32_t* ops, int n, double bytes, const Env& env, int l_log2, const FastTabs& tab,
                     double& sec_out, double& vol_out) {
  double sec = 0, vol = 0;
  for (int o = 0; o < n; ++o) {
    const uint32_t w = ops[o];
    sec += price_fast(w & 1u, (w >> 1) & 31, (w >> 6) & 31, (w >> 11) & 31, (w >> 16) & 31, bytes, env, l_log2,
                      tab, &vol, nullptr);
  }
  sec_out = sec;
  vol_out = vol;
}

// Returns the tp_error_kind, or -1 when the pair needs the array form
// (a device dim held twice by the working map; with kRecord also when the
// op list does not fit an OpRec).
template <bool kRecord = false>
TP_HD int redist_cost_fast(int R, const SideDesc& gf, const SideDesc& gt, const DimT* dt, double bytes,
                           const Env& env, int l_log2, const FastTabs& tab, double& sec_out, double& vol_out,
                           Trace* tr, MultiSec* ms = nullptr, OpRec* rec = nullptr) {
  if (R < 0 || R > kMaxR) return kCapacity;
  // ---- unify: bitmask closure (see tp_core.cuh) ----
  uint32_t D = gf.D | gt.D;
  const int n = gf.n, nt = gt.n;
  if (n != nt) return kNotUnifiable;  // redistribution.hpp:264-268
  if (n > kMaxD) return kCapacity;
  for (int i = 0; i < R; ++i)
    if (gf.x[i] > dt[i].t) return kFactorization;  // :102-111
  for (int i = 0; i < R; ++i)
    if (gt.x[i] > dt[i].t) return kFactorization;
  D &= ~1u & low_bits(n);
  uint32_t P[kMaxR];
  for (int i = 0; i < R; ++i) P[i] = 0;
  for (bool changed = true; changed;) {
    changed = false;
    for (int sd = 0; sd < 2; ++sd) {
      const SideDesc& g = sd ? gt : gf;
      for (int i = 0; i < R; ++i) {
        const int x = g.x[i], a = g.a[i];
        if (x < 2) continue;
        const uint32_t win = low_bits(x) & ~1u;
        const uint32_t tb = mirror((D >> a) & win, x) & win;
        const uint32_t db = (mirror(P[i] & win, x) & win) << a;
        if ((tb & ~P[i]) | (db & ~D)) changed = true;
        P[i] |= tb;
        D |= db;
      }
    }
  }
  // ---- unified device dims: log2 extent and lower position per dim ----
  Pack2 EXT{0, 0}, POS{0, 0};
  int next = 0;
  if (n > 0) {
    int prev = 0;
    uint32_t rest = D | (1u << n);
    while (rest) {
      const int c = ffs32(rest);
      rest &= rest - 1;
      p2set(EXT, next, c - prev);
      p2set(POS, next, prev);
      ++next;
      prev = c;
    }
  }
  // ---- unified axes (:330-345) into packed maps and position masks ----
  Pack4 W{{0, 0, 0, 0}}, TO{{0, 0, 0, 0}};
  Pack2 FIRST{0, 0};  // to.axis_of(k) + 1
  uint32_t OCC = 0, TGT = 0, MATCH = 0, PM = 0, PB = 0;
  int U = 0, s = 0;
  bool dup = false;
  for (int i = 0; i < R; ++i) {
    uint32_t bnd = P[i];
    int c = 0;
    for (;;) {
      if (U >= kMaxU) return kCapacity;
      int mf = -1, mt = -1;
      if (c < gf.x[i]) mf = popc32(D & low_bits(gf.a[i] + gf.x[i] - c));
      if (c < gt.x[i]) mt = popc32(D & low_bits(gt.a[i] + gt.x[i] - c));
      const uint32_t bit = 1u << U;
      pset(W, U, mf + 1);
      pset(TO, U, mt + 1);
      if (mf >= 0) {
        OCC |= bit;
        if ((PM >> mf) & 1u) dup = true;
        PM |= 1u << mf;
        const int e = p2get(EXT, mf), pos = p2get(POS, mf);
        PB |= low_bits(pos + e) & ~low_bits(pos);
        s += e;
      }
      if (mt >= 0) {
        TGT |= bit;
        if (p2get(FIRST, mt) == 0) p2set(FIRST, mt, U + 1);
      }
      if (mf == mt) MATCH |= bit;
      const int next_c = bnd ? ffs32(bnd) : (int)dt[i].t;
      if (tr) {
        tr->pe[U] = (uint8_t)(next_c - c);
        tr->plast[U] = bnd == 0;
        tr->pdim[U] = (uint8_t)i;
        tr->from_map[U] = (int8_t)mf;
        tr->to_map[U] = (int8_t)mt;
      }
      ++U;
      if (!bnd) break;
      c = next_c;
      bnd &= bnd - 1;
    }
  }
  if (dup) return -1;
  if (tr) {
    tr->depth = next;
    for (int k = 0; k < next; ++k) tr->ext[k] = (uint8_t)p2get(EXT, k);
    tr->urank = U;
    tr->nops = 0;
  }
  const uint32_t ALL = low_bits(U);
  // ---- inference with on-the-fly pricing (:419-451) ----
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
  while ((~MATCH) & ALL) {
    if (--guard < 0) return kNoTerminate;
    bool progress = true;
    while (progress) {
      // InferSlice (:350-365): free positions with a target, ascending
      progress = false;
      uint32_t cand = ~OCC & TGT & ALL;
      while (cand) {
        const int i = ffs32(cand);
        cand &= cand - 1;
        const int k = pget(TO, i) - 1;
        if ((PM >> k) & 1u) continue;
        record(0, k, i, -1, 0, 0, 0.0);
        pset(W, i, k + 1);
        const uint32_t bit = 1u << i;
        OCC |= bit;
        MATCH |= bit;
        PM |= 1u << k;
        const int e = p2get(EXT, k), pos = p2get(POS, k);
        PB |= low_bits(pos + e) & ~low_bits(pos);
        s += e;
        progress = true;
      }
      // InferAll2All until none applies (:367-385)
      bool a2a = true;
      while (a2a) {
        a2a = false;
        uint32_t ca = OCC & ~MATCH & ALL;
        while (ca) {
          const int i = ffs32(ca);
          ca &= ca - 1;
          const int k = pget(W, i) - 1;
          const int j = p2get(FIRST, k) - 1;
          if (j < 0 || j == i || ((OCC >> j) & 1u)) continue;
          const int e = p2get(EXT, k), pos = p2get(POS, k);
          const int rexp = pos - popc32(PB & low_bits(pos));
          if (kRecord) {
            if (!rec->push(true, pos, rexp, e, s)) return -1;
          } else {
            int64_t ct = 0;
            const double c = price_fast(true, pos, rexp, e, s, bytes, env, l_log2, tab, &vol, tr ? &ct : nullptr);
            sec += c;
            if (ms) price_members(ms, true, pos, rexp, e, s, bytes, l_log2);
            record(2, k, i, j, 0, ct, c);
          }
          const uint32_t bi = 1u << i, bj = 1u << j;
          pset(W, i, 0);
          pset(W, j, k + 1);
          OCC = (OCC & ~bi) | bj;
          MATCH = (MATCH & ~bi) | (TGT & bi ? 0u : bi) | bj;
          a2a = true;
        }
        progress |= a2a;
      }
    }
    if (!((~MATCH) & ALL)) break;
    // InferAllGather (:387-401), else the fallback gather (:403-417)
    uint32_t gm = OCC & ~TGT & ALL;
    int fb = 0;
    if (!gm) {
      gm = OCC & ~MATCH & ALL;
      fb = 1;
      if (!gm) return kDeadlock;
    }
    const int i = ffs32(gm);
    const int k = pget(W, i) - 1;
    const int e = p2get(EXT, k), pos = p2get(POS, k);
    const int rexp = pos - popc32(PB & low_bits(pos));
    if (kRecord) {
      if (!rec->push(false, pos, rexp, e, s)) return -1;
    } else {
      int64_t ct = 0;
      const double c = price_fast(false, pos, rexp, e, s, bytes, env, l_log2, tab, &vol, tr ? &ct : nullptr);
      sec += c;
      if (ms) price_members(ms, false, pos, rexp, e, s, bytes, l_log2);
      record(1, k, i, -1, fb, ct, c);
    }
    const uint32_t bi = 1u << i;
    pset(W, i, 0);
    OCC &= ~bi;
    MATCH = (MATCH & ~bi) | (TGT & bi ? 0u : bi);
    PM &= ~(1u << k);
    PB &= ~(low_bits(pos + e) & ~low_bits(pos));
    s -= e;
  }
  sec_out = sec;
  vol_out = vol;
  return kOk;
}

// The kernels' entry: the register form, or the array form for working maps
// that hold a device dim twice (Fl/Tl: the original layouts when known).
TP_HD int pair_cost_sd(int R, const SideDesc& F, const SideDesc& T, const Lay* Fl, const Lay* Tl, const DimT* dt,
                       double bytes, const Env& env, int l_log2, const FastTabs& tab, double& sec, double& vol,
                       Trace* tr, MultiSec* ms = nullptr) {
  if (ms)
    for (int q = 1; q < ms->g; ++q) ms->s(q) = 0;
  const int st = redist_cost_fast(R, F, T, dt, bytes, env, l_log2, tab, sec, vol, tr, ms);
  if (st != -1) return st;
  Lay a, b;
  if (Fl) a = *Fl; else lay_of(F, R, a);
  if (Tl) b = *Tl; else lay_of(T, R, b);
  // the array form (rare: a device dim held twice), once per member, one call site
  for (int q = ms ? ms->g - 1 : 0; q >= 0; --q) {
    double sc = 0, v = 0;
    const int e = redist_cost(R, a, b, dt, bytes, q ? ms->env(q) : env, sc, v, q ? nullptr : tr);
    if (e) return e;
    if (q) {
      ms->s(q) = sc;
    } else {
      sec = sc;
      vol = v;
    }
  }
  return kOk;
}

// The op list of one class-table entry (the sweep's inference pass): the
// header word holds the op count, the tp_error_kind << 8 and the flags.
TP_HD void infer_ops(int R, const SideDesc& F, const SideDesc& T, const DimT* dt, uint32_t* out) {
  OpRec r;
  r.n = 0;
  uint32_t flags = 0;
  int st = kOk;
  if (same_side(F, T, R)) {
    flags = kOpsSame;
  } else {
    double sec = 0, vol = 0;
    st = redist_cost_fast<true>(R, F, T, dt, 0.0, Env{0, 0, 0}, -1, FastTabs{nullptr, nullptr}, sec, vol, nullptr,
                                nullptr, &r);
    if (st == -1) {
      st = kOk;
      flags = kOpsFull;
      r.n = 0;
    } else if (st) {
      r.n = 0;
    }
  }
  r.w[0] = (uint32_t)r.n | ((uint32_t)st << 8) | flags;
  for (int o = 0; o < kOpWords; ++o) out[o] = o <= r.n ? r.w[o] : 0u;
}

TP_HD int pair_cost(int R, const Lay& F, const Lay& T, const DimT* dt, double bytes, const Env& env, int l_log2,
                    const FastTabs& tab, double& sec, double& vol, Trace* tr) {
  SideDesc f, t;
  side_of(F, R, f);
  side_of(T, R, t);
  return pair_cost_sd(R, f, t, &F, &T, dt, bytes, env, l_log2, tab, sec, vol, tr);
}

// Verification export: one query through pair_cost (the kernels' path).
template <typename Result>
TP_HD int run_query_fast(const QueryPOD& q, Result& r, const FastTabs& tab) {
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
    if (q.fmap[i] < -1 || q.fmap[i] >= q.fdepth || q.tmap[i] < -1 || q.tmap[i] >= q.tdepth) return kCapacity;
    F.map[i] = (int8_t)q.fmap[i];
    T.map[i] = (int8_t)q.tmap[i];
    dt[i].t = (uint8_t)ctz64(q.shape[i]);
    dt[i].odd = (q.shape[i] >> dt[i].t) > 1;
  }
  if (ftot != ttot) return kNotUnifiable;
  Env env{q.intra, q.inter, (int64_t)q.local};
  Trace tr;
  double sec = 0, vol = 0;
  const int st = pair_cost(q.rank, F, T, dt, q.bytes, env, ilog2_exact((int64_t)q.local), tab, sec, vol, &tr);
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
