// tp_warp.cuh — warp-cooperative pricing of one (from, to) layout pair.
//
// The form the kernels run for small class tables: one warp prices one
// pair. Everything that was a sequential loop in the scalar form is spread
// over lanes:
//   * the unification closure (tp_core.cuh): lane (side, dim) reflects its
//     own region, the boundary sets are combined with one shuffle and one
//     __reduce_or_sync per round;
//   * unified device dim k sits on lane k (log2 extent, lower position,
//     found with __fns), unified tensor axis q on lane q (its dim and part
//     start located by a prefix over the dims' part counts);
//   * the sequence search's scans (redistribution.hpp:350-417) are ballots +
//     find-first-set, "device dim k is held" is a __reduce_or_sync mask and
//     the ct repetition (cost_model.hpp:115-119) a __reduce_add_sync;
//   * with a power-of-two local_device_num every ct division is a shift, and
//     inter/ct and the AllToAll scale k(p-k)/(p-1) (cost_model.hpp:148-151,
//     218) come from per-build tables computed with the reference's own
//     expressions (so the values are the same IEEE results).
// Control flow is warp-uniform; the order of the inferred ops — and so the
// fp64 summation order — is exactly the reference's.
#pragma once

#include "tp_core.cuh"

namespace tpk {

constexpr int kBwTab = 65;      // inter/ct for ct in [0, 64] (ct = 0 -> intra)
constexpr int kScaleDim = 17;   // scale[log2 k][log2 p], k < p <= 2^16

// Per-build pricing tables (host-computed, same expressions as the reference).
struct PriceTabs {
  const double* bw;     // [kBwTab]
  const double* scale;  // [kScaleDim * kScaleDim]
};

struct WarpEnv {
  Env env;
  int l_log2;     // log2(local_device_num) when it is a power of two, else -1
  PriceTabs tab;  // may hold null pointers: then computed directly
};

// AllGather / AllToAll on a device dim with log2 extent ek at lower device
// position te; rexp = log2 of the in-node repetition; s = log2 of the
// working map's shard divisor: the one pricing routine (tp_core.cuh
// price_fast, branch-free, so the lanes pricing a batch of mixed ops do not
// diverge).
__device__ __forceinline__ double price_op_warp(bool a2a, int te, int rexp, int ek, int s, double bytes,
                                                const WarpEnv& we, double* vol, int64_t* ct_out) {
  return price_fast(a2a, te, rexp, ek, s, bytes, we.env, we.l_log2, FastTabs{we.tab.bw, we.tab.scale}, vol, ct_out);
}

// All 32 lanes call this with identical arguments. pf/pt point at the two
// layout descriptors (global or local memory: lanes index them by dim).
// Returns the tp_error_kind; sec/vol are valid on every lane. `tr`
// (verification export only) is written by lane 0.
__device__ int redist_cost_warp(int R, const SideDesc* pf, const SideDesc* pt, const DimT* dt, double bytes,
                                const WarpEnv& we, double& sec_out, double& vol_out, Trace* tr,
                                unsigned* prof = nullptr) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const long long c_start = prof ? clock64() : 0;
  int rounds = 0;
  if (R < 0 || R > kMaxR) return kCapacity;
  const int n = pf->n;
  if (n != pt->n) return kNotUnifiable;  // redistribution.hpp:264-268
  if (n > kMaxD) return kCapacity;
  // ---- unify: closure with lane (side, dim) owning one region ----
  const bool rl = lane < 2 * R;
  const int side = lane >= R ? 1 : 0;
  const int dim = rl ? lane - side * R : 0;
  const SideDesc* me = side ? pt : pf;
  const int x = rl ? me->x[dim] : 0;
  const int a = rl ? me->a[dim] : 0;
  const int tdim = dt[dim].t;
  if (__any_sync(FULL, rl && x > tdim)) return kFactorization;  // :102-111
  const long long c_loads = prof ? clock64() : 0;
  uint32_t D = (pf->D | pt->D) & ~1u & low_bits(n);
  uint32_t P = 0;  // boundaries of tensor dim `dim` (lanes of both sides agree)
  const int partner = rl ? (side ? lane - R : lane + R) : lane;
  const uint32_t win = low_bits(x) & ~1u;
  // Each round updates the tensor boundaries from the device ones, then the
  // device boundaries from the NEW tensor ones (the least fixed point is the
  // same in any order; this one needs about half the rounds), and folds
  // "some lane's P changed" into bit 31 of the same reduction (D uses bits
  // 0..16): a shuffle and a reduction per round, no vote.
  for (;;) {
    const uint32_t tb = x >= 2 ? (mirror((D >> a) & win, x) & win) : 0u;
    const uint32_t nP = P | tb | __shfl_sync(FULL, tb, partner);
    const uint32_t db = x >= 2 ? ((mirror(nP & win, x) & win) << a) : 0u;
    const uint32_t red = __reduce_or_sync(FULL, db | (nP != P ? 0x80000000u : 0u));
    const uint32_t nD = D | (red & 0x7fffffffu);
    const bool changed = (red >> 31) != 0 || nD != D;
    P = nP;
    D = nD;
    ++rounds;
    if (!changed) break;
  }
  const long long c_closure = prof ? clock64() : 0;
  // ---- unified device dims: lane k <- (log2 extent, lower position) ----
  int my_ext = 0, my_pos = n, next = 0;
  if (n > 0) {
    int prev = 0;
    uint32_t rest = D | (1u << n);
    while (rest) {  // warp-uniform
      const int c = ffs32(rest);
      rest &= rest - 1;
      if (lane == next) {
        my_ext = c - prev;
        my_pos = prev;
      }
      ++next;
      prev = c;
    }
  }
  // ---- unified tensor axes: lane q <- (from, to) of axis q (:330-345) ----
  int U = 0, qi = -1, qj = 0;
  uint32_t Pq = 0;
  int my_w = -1, my_to = -1, my_c = 0;
  {
    // lane q finds its axis directly: dim i has popc(P_i) + 1 parts, part j
    // starts at the j-th boundary of P_i (0 for j = 0)
    for (int i = 0; i < R; ++i) {
      const uint32_t Pi = __shfl_sync(FULL, P, i);
      const int np = popc32(Pi) + 1;
      if (lane >= U && lane < U + np) {
        qi = i;
        qj = lane - U;
        Pq = Pi;
      }
      U += np;
    }
    if (U > 32) return kCapacity;
    if (qi >= 0) {
      const int af = pf->a[qi], xf = pf->x[qi], at = pt->a[qi], xt = pt->x[qi];
      int c = 0;
      if (qj > 0) {
        uint32_t b = Pq;
        for (int t = 1; t < qj; ++t) b &= b - 1;
        c = ffs32(b);
      }
      my_c = c;
      if (c < xf) my_w = popc32(D & low_bits(af + xf - c));
      if (c < xt) my_to = popc32(D & low_bits(at + xt - c));
    }
  }
  if (tr) {
    for (int q = 0; q < U; ++q) {
      const int fw = __shfl_sync(FULL, my_w, q), ft = __shfl_sync(FULL, my_to, q);
      const int di = __shfl_sync(FULL, qi, q), dj = __shfl_sync(FULL, qj, q);
      const uint32_t Pd = __shfl_sync(FULL, Pq, q);
      const int c0 = __shfl_sync(FULL, my_c, q);
      if (lane == 0) {
        const int np = popc32(Pd);
        const uint32_t above = Pd & ~low_bits(c0 + 1);
        const int c1 = dj < np ? ffs32(above) : (int)dt[di].t;
        tr->pe[q] = (uint8_t)(c1 - c0);
        tr->plast[q] = dj == np;
        tr->pdim[q] = (uint8_t)di;
        tr->from_map[q] = (int8_t)fw;
        tr->to_map[q] = (int8_t)ft;
      }
    }
    for (int k = 0; k < next; ++k) {
      const int e = __shfl_sync(FULL, my_ext, k);
      if (lane == 0) tr->ext[k] = (uint8_t)e;
    }
    if (lane == 0) {
      tr->depth = next;
      tr->urank = U;
      tr->nops = 0;
    }
  }
  const long long c_axes = prof ? clock64() : 0;
  // ---- sequence inference with on-the-fly pricing (:419-451) ----
  uint32_t PM = __reduce_or_sync(FULL, my_w >= 0 ? (1u << my_w) : 0u);
  const int ext_w = __shfl_sync(FULL, my_ext, my_w >= 0 ? my_w : 0);
  int s = (int)__reduce_add_sync(FULL, (unsigned)(my_w >= 0 ? ext_w : 0));
  uint32_t mism = __ballot_sync(FULL, my_w != my_to);
  double sec = 0, vol = 0;
  int guard = (next + 1) * (U + 1) * 4 + 16;
  int nops = 0;
  auto record = [&](int kind, int k, int i, int j, int fb, int64_t ct, double sc) {
    if (tr && lane == 0) {
      if (nops < kMaxOps) {
        int8_t* o = tr->ops[nops];
        o[0] = (int8_t)kind;
        o[1] = (int8_t)k;
        o[2] = (int8_t)i;
        o[3] = (int8_t)j;
        o[4] = (int8_t)fb;
        tr->ct[nops] = ct;
        tr->sec[nops] = sc;
      }
      tr->nops = nops + 1 > kMaxOps ? kMaxOps + 1 : nops + 1;
    }
    ++nops;
  };
  // log2 of the in-node repetition below device dim k (cost_model.hpp:115-119):
  // extents of the dims inner to k that the working map does not hold
  auto rexp_below = [&](int k, int te) -> int {
    const int held = (int)__reduce_add_sync(FULL, (unsigned)((lane < k && ((PM >> lane) & 1u)) ? my_ext : 0));
    return te - held;
  };
  // Priced ops. With a trace they are priced on the spot. Otherwise op t is
  // parked on lane t and a batch is priced by all lanes at once -- the fp64
  // chains of up to 32 ops overlap -- then summed in op order, the same
  // additions as pricing each op in turn (the search never reads sec/vol).
  int nb = 0;
  int b_te = 0, b_rexp = 0, b_ek = 0, b_s = 0;
  bool b_a2a = false;
  auto flush = [&]() {
    double c = 0, v = 0;
    if (lane < nb) {
      int64_t ct = 0;
      c = price_op_warp(b_a2a, b_te, b_rexp, b_ek, b_s, bytes, we, &v, &ct);  // v = 0 + op volume
    }
    for (int t = 0; t < nb; ++t) {
      vol += __shfl_sync(FULL, v, t);
      sec += __shfl_sync(FULL, c, t);
    }
    nb = 0;
  };
  auto op = [&](bool a2a_op, int te, int rexp, int ek, int k, int i, int j, int fb) {
    if (tr) {
      int64_t ct = 0;
      const double c = price_op_warp(a2a_op, te, rexp, ek, s, bytes, we, &vol, &ct);
      sec += c;
      record(a2a_op ? 2 : 1, k, i, j, fb, ct, c);
      return;
    }
    if (lane == nb) {
      b_te = te;
      b_rexp = rexp;
      b_ek = ek;
      b_s = s;
      b_a2a = a2a_op;
    }
    ++nops;
    if (++nb == 32) flush();
  };
  while (mism) {
    if (--guard < 0) return kNoTerminate;
    bool progress = true;
    while (progress) {
      // InferSlice (:350-365). The to-map's device dims are distinct, so
      // the slices of one pass never conflict and commute (a slice prices
      // nothing): they are applied together; the trace lists them in
      // position order like the reference.
      progress = false;
      const uint32_t cand = __ballot_sync(FULL, my_w == -1 && my_to >= 0 && !((PM >> (my_to & 31)) & 1u));
      if (cand) {
        if (tr) {
          for (uint32_t c = cand; c; c &= c - 1) {
            const int i = ffs32(c);
            record(0, __shfl_sync(FULL, my_to, i), i, -1, 0, 0, 0.0);
          }
        } else {
          nops += __popc(cand);
        }
        const bool me = (cand >> lane) & 1u;
        const int ext_to = __shfl_sync(FULL, my_ext, my_to >= 0 ? my_to : 0);
        PM |= __reduce_or_sync(FULL, me ? (1u << my_to) : 0u);
        s += (int)__reduce_add_sync(FULL, me ? (unsigned)ext_to : 0u);
        if (me) my_w = my_to;
        progress = true;
      }
      // InferAll2All until none applies (:367-385): a pass takes positions
      // in ascending order, each checked against the state the earlier moves
      // of the pass left. Lane i qualifies when it holds a dim k it must not
      // keep and the position whose to-map is k holds nothing (free_to).
      bool a2a = true;
      while (a2a) {
        a2a = false;
        int cursor = -1;
        for (;;) {
          const uint32_t free_to = __reduce_or_sync(FULL, (my_to >= 0 && my_w == -1) ? (1u << my_to) : 0u);
          const uint32_t ok = __ballot_sync(FULL, lane > cursor && my_w >= 0 && my_w != my_to &&
                                                      ((free_to >> (my_w & 31)) & 1u));
          if (!ok) break;
          const int i = ffs32(ok);
          const int k = __shfl_sync(FULL, my_w, i);
          const int j = ffs32(__ballot_sync(FULL, my_to == k));  // to.axis_of(k)
          const int te = __shfl_sync(FULL, my_pos, k), ek = __shfl_sync(FULL, my_ext, k);
          op(true, te, rexp_below(k, te), ek, k, i, j, 0);
          if (lane == i) my_w = -1;
          if (lane == j) my_w = k;
          cursor = i;
          a2a = true;
        }
        progress |= a2a;
      }
    }
    mism = __ballot_sync(FULL, my_w != my_to);
    if (!mism) break;
    // InferAllGather (:387-401), else the fallback gather (:403-417)
    uint32_t gm = __ballot_sync(FULL, my_w >= 0 && my_to == -1);
    int fb = 0;
    if (!gm) {
      gm = __ballot_sync(FULL, my_w >= 0 && my_w != my_to);
      fb = 1;
      if (!gm) return kDeadlock;
    }
    const int i = ffs32(gm);
    const int k = __shfl_sync(FULL, my_w, i);
    const int te = __shfl_sync(FULL, my_pos, k), ek = __shfl_sync(FULL, my_ext, k);
    op(false, te, rexp_below(k, te), ek, k, i, -1, fb);
    if (lane == i) my_w = -1;
    PM = __reduce_or_sync(FULL, my_w >= 0 ? (1u << my_w) : 0u);
    s -= ek;
    mism = __ballot_sync(FULL, my_w != my_to);
  }
  flush();
  sec_out = sec;
  vol_out = vol;
  if (prof && lane == 0) {
    const long long c_end = clock64();
    prof[0] = (unsigned)(c_closure - c_start);
    prof[1] = (unsigned)(c_axes - c_closure);
    prof[2] = (unsigned)(c_end - c_axes);
    prof[3] = (unsigned)nops;
    prof[4] = (unsigned)U;
    prof[5] = (unsigned)next;
    prof[6] = (unsigned)rounds;
    prof[7] = (unsigned)(c_loads - c_start);  // of prof[0]: the descriptor reads before the closure
  }
  return kOk;
}

// Verification export on a warp: exactly the kernels' code path.
template <typename Result>
__device__ int run_query_warp(const QueryPOD& q, Result& r, Trace& tr, const PriceTabs& tabs) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    r.status = 0;
    r.depth = 0;
    r.urank = 0;
    r.num_ops = 0;
    r.volume_bytes = 0;
    r.seconds = 0;
  }
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
  for (int i = 0; i < kMaxR; ++i) {
    dt[i].t = 0;
    dt[i].odd = 0;
  }
  for (int i = 0; i < q.rank; ++i) {
    if (q.shape[i] < 1) return kCapacity;
    if (q.fmap[i] < -1 || q.fmap[i] >= q.fdepth || q.tmap[i] < -1 || q.tmap[i] >= q.tdepth) return kCapacity;
    F.map[i] = (int8_t)q.fmap[i];
    T.map[i] = (int8_t)q.tmap[i];
    dt[i].t = (uint8_t)ctz64(q.shape[i]);
    dt[i].odd = (q.shape[i] >> dt[i].t) > 1;
  }
  if (ftot != ttot) return kNotUnifiable;
  WarpEnv we;
  we.env = Env{q.intra, q.inter, (int64_t)q.local};
  we.l_log2 = ilog2_exact((int64_t)q.local);
  we.tab = tabs;
  double sec = 0, vol = 0;
  SideDesc fs, ts;
  side_of(F, q.rank, fs);
  side_of(T, q.rank, ts);
  const int st = redist_cost_warp(q.rank, &fs, &ts, dt, q.bytes, we, sec, vol, &tr);
  if (st) return st;
  __syncwarp();
  if (lane == 0) {
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
  }
  return kOk;
}

// Host-side construction of the pricing tables for one environment.
inline void make_price_tabs(const Env& env, double* bw, double* scale) {
  for (int ct = 0; ct < kBwTab; ++ct) bw[ct] = eff_bw(ct, env);  // cost_model.hpp:148-151
  for (int ke = 0; ke < kScaleDim; ++ke) {
    for (int pe = 0; pe < kScaleDim; ++pe) {
      const int64_t k = (int64_t)1 << ke, p = (int64_t)1 << pe;
      scale[ke * kScaleDim + pe] = ke < pe ? (double)k * (double)(p - k) / (double)(p - 1) : 0.0;  // :218
    }
  }
}

}  // namespace tpk
