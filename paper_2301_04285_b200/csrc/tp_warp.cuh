// tp_warp.cuh — warp-cooperative pricing of one (from, to) layout pair.
//
// The form the kernels run: one warp prices one pair. Lane q holds unified
// tensor axis q (working-map entry w, target entry to) and unified device
// dim q (log2 extent, lower device position). The sequence search's scans
// (redistribution.hpp:350-417) become ballots + find-first-set, "device dim
// k is in the working map" is a __reduce_or_sync mask, and with a
// power-of-two local_device_num every integer division of the ct formulas
// (cost_model.hpp:108-135, 197-222) is a shift. Control flow is
// warp-uniform; the order of the inferred ops — and so the fp64 summation
// order — is exactly the reference's. tp_core.cuh's scalar redist_cost is
// the same algorithm one thread at a time (used by the host-side check).
#pragma once

#include "tp_core.cuh"

namespace tpk {

struct WarpEnv {
  Env env;
  int l_log2;  // log2(local_device_num) when it is a power of two, else -1
};

__device__ __forceinline__ void ct_gather_warp(int te, int rexp, int ek, const WarpEnv& we, int64_t& ct,
                                               int& rep_e, int64_t& rep, int64_t& gin, int& gin_e) {
  if (we.l_log2 >= 0) {
    const int l = we.l_log2;
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
  const int64_t L = we.env.local;
  const int64_t pd = (int64_t)1 << ek;
  const int64_t temp = (int64_t)1 << te;
  rep = (int64_t)1 << rexp;
  if (rep > L) rep = L;
  rep_e = -1;
  gin_e = -1;
  if (temp >= L) {
    gin = 1;
    ct = L / rep;
  } else {
    const int64_t remain = L / temp;
    gin = pd < remain ? pd : remain;
    ct = remain >= pd ? 0 : temp / rep;
  }
}

// AllGather / AllToAll on a device dim with log2 extent ek at lower device
// position te; rexp = log2 of the in-node repetition; s = log2 of the
// working map's shard divisor (cost_model.hpp:176-225, redistribution.hpp:521-553).
__device__ __forceinline__ double price_op_warp(bool a2a, int te, int rexp, int ek, int s, double bytes,
                                                const WarpEnv& we, double* vol, int64_t* ct_out) {
  const double shard = bytes / exp2d(s);
  const int64_t p = (int64_t)1 << ek;
  const double d = (double)p;
  int64_t ct, rep, gin;
  int rep_e, gin_e;
  ct_gather_warp(te, rexp, ek, we, ct, rep_e, rep, gin, gin_e);
  if (!a2a) {
    *vol += (d - 1) * shard;
    const double v = (double)(p - 1) * shard;
    *ct_out = ct;
    return v / eff_bw(ct, we.env);
  }
  *vol += (d - 1) / d * shard;
  const double v = (d - 1) / d * shard;
  const int64_t k = gin;
  if (k >= p) {
    *ct_out = 0;
    return v / we.env.intra;
  }
  int64_t c;
  if (we.l_log2 >= 0) {
    c = gin_e + rep_e <= we.l_log2 ? ((int64_t)1 << (we.l_log2 - gin_e - rep_e)) : 0;
  } else {
    c = we.env.local / (k * rep);
  }
  if (c < 1) c = 1;
  *ct_out = c;
  const double bw = eff_bw(c, we.env);
  const double scale = (double)k * (double)(p - k) / (double)(p - 1);
  return scale * v / bw;
}

// All 32 lanes call this with identical arguments. Returns the
// tp_error_kind; sec/vol are valid on every lane. `tr` (verification
// export only) is written by lane 0.
__device__ int redist_cost_warp(int R, const SideDesc& gf, const SideDesc& gt, const DimT* dt, double bytes,
                                const WarpEnv& we, double& sec_out, double& vol_out, Trace* tr) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  if (R < 0 || R > kMaxR) return kCapacity;
  // ---- unify: the bitmask closure of tp_core.cuh (warp-uniform) ----
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
  // lane k <- (log2 extent, lower position) of unified device dim k
  int my_ext = 0, my_pos = n, next = 0;
  if (n > 0) {
    int prev = 0;
    uint32_t rest = D | (1u << n);
    while (rest) {
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
  // lane q <- (from, to) maps of unified tensor axis q (:330-345)
  int my_w = -1, my_to = -1, U = 0;
  for (int i = 0; i < R; ++i) {
    uint32_t bnd = P[i];
    int c = 0;
    for (;;) {
      if (U >= 32) return kCapacity;
      if (lane == U) {
        if (c < gf.x[i]) my_w = popc32(D & low_bits(gf.a[i] + gf.x[i] - c));
        if (c < gt.x[i]) my_to = popc32(D & low_bits(gt.a[i] + gt.x[i] - c));
      }
      const int next_c = bnd ? ffs32(bnd) : (int)dt[i].t;
      if (tr && lane == 0) {
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
  if (tr) {
    for (int q = 0; q < U; ++q) {
      const int fw = __shfl_sync(FULL, my_w, q), ft = __shfl_sync(FULL, my_to, q);
      if (lane == 0) {
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
  while (mism) {
    if (--guard < 0) return kNoTerminate;
    bool progress = true;
    while (progress) {
      // InferSlice (:350-365), positions ascending
      progress = false;
      uint32_t cand = __ballot_sync(FULL, my_w == -1 && my_to >= 0 && !((PM >> (my_to & 31)) & 1u));
      while (cand) {
        const int i = ffs32(cand);
        cand &= cand - 1;
        const int k = __shfl_sync(FULL, my_to, i);
        if ((PM >> k) & 1u) continue;  // an earlier slice of this pass took k
        record(0, k, i, -1, 0, 0, 0.0);
        if (lane == i) my_w = k;
        PM |= 1u << k;
        s += __shfl_sync(FULL, my_ext, k);
        progress = true;
      }
      // InferAll2All until none applies (:367-385); each candidate is
      // re-checked against the state the earlier moves of the pass left
      bool a2a = true;
      while (a2a) {
        a2a = false;
        uint32_t ca = __ballot_sync(FULL, my_w >= 0 && my_w != my_to);
        while (ca) {
          const int i = ffs32(ca);
          ca &= ca - 1;
          const int k = __shfl_sync(FULL, my_w, i);
          const int ti = __shfl_sync(FULL, my_to, i);
          if (k < 0 || ti == k) continue;
          const uint32_t tk = __ballot_sync(FULL, my_to == k);
          if (!tk) continue;
          const int j = ffs32(tk);  // to.axis_of(k)
          if (j == i || __shfl_sync(FULL, my_w, j) != -1) continue;
          const int te = __shfl_sync(FULL, my_pos, k), ek = __shfl_sync(FULL, my_ext, k);
          int64_t ct = 0;
          const double c = price_op_warp(true, te, rexp_below(k, te), ek, s, bytes, we, &vol, &ct);
          sec += c;
          record(2, k, i, j, 0, ct, c);
          if (lane == i) my_w = -1;
          if (lane == j) my_w = k;
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
    int64_t ct = 0;
    const double c = price_op_warp(false, te, rexp_below(k, te), ek, s, bytes, we, &vol, &ct);
    sec += c;
    record(1, k, i, -1, fb, ct, c);
    if (lane == i) my_w = -1;
    PM = __reduce_or_sync(FULL, my_w >= 0 ? (1u << my_w) : 0u);
    s -= ek;
    mism = __ballot_sync(FULL, my_w != my_to);
  }
  sec_out = sec;
  vol_out = vol;
  return kOk;
}

// Verification export on a warp: exactly the kernels' code path.
template <typename Result>
__device__ int run_query_warp(const QueryPOD& q, Result& r, Trace& tr) {
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
  double sec = 0, vol = 0;
  SideDesc fs, ts;
  side_of(F, q.rank, fs);
  side_of(T, q.rank, ts);
  const int st = redist_cost_warp(q.rank, fs, ts, dt, q.bytes, we, sec, vol, &tr);
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

}  // namespace tpk
