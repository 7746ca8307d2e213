// tp_kernels.cuh — the device code: set-up kernels, node rows, class pairs,
// fan-out, the fused and batched builds, price_assignment, row minima and the
// verification export.
// Part of the single translation unit tp_engine.cu (included from there, in order).
#pragma once

namespace {

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
// K0 (at upload): strategy tables by unranking (layout.hpp:270-328).
__global__ void table_kernel(const TableDesc* __restrict__ tabs, int ntabs, int64_t total,
                             Strat* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  int t = 0;
  while (t + 1 < ntabs && tabs[t + 1].offset <= i) ++t;
  Strat s;
  tpk::unrank_strategy(tabs[t].p, tabs[t].n, i - tabs[t].offset, s);
  out[i] = s;
}

// K0b (at upload): layout descriptors of every (edge class, side, strategy).
__device__ __forceinline__ void side_one(const SideJob* __restrict__ jobs, int njobs, int64_t i,
                                         const Strat* __restrict__ tables, tpk::SideDesc* __restrict__ out) {
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].out <= i) lo = mid; else hi = mid - 1;
  }
  const SideJob j = jobs[lo];
  Lay L;
  tpk::side_layout(tables[j.tab + (i - j.out)], j.sa, j.R, L);
  tpk::SideDesc d;
  tpk::side_of(L, j.R, d);
  out[i] = d;
}

__global__ void side_kernel(const SideJob* __restrict__ jobs, int njobs, int64_t total,
                            const Strat* __restrict__ tables, tpk::SideDesc* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  side_one(jobs, njobs, i, tables, out);
}

// Everything one class-table entry's pricing reads, gathered at upload so a
// pair warp starts from one dependent load (not pair -> class -> maps ->
// layouts).
struct alignas(16) PairRec {
  tpk::SideDesc F, T;  // producer / consumer layouts (first strategies with them)
  double bytes;        // tensor bytes (after the memo's first-writer rule)
  int32_t sig, local;  // edge class; su * Sw + sw of the first such strategy pair
  int32_t R, pad;
  DimT dt[tpk::kMaxR];
};

__device__ __forceinline__ void pair_rec_of(const SigDesc* __restrict__ sigs, const int32_t* __restrict__ pair_sig,
                                            const int32_t* __restrict__ maps, const tpk::SideDesc* __restrict__ sides,
                                            const double* __restrict__ overrides, int64_t idx, PairRec& r) {
  const int sig = pair_sig[idx];
  const SigDesc& sg = sigs[sig];
  const int32_t t = (int32_t)(idx - sg.pair_begin);
  const int32_t ui = t / sg.Wn, wi = t - ui * sg.Wn;
  const int32_t su = maps[sg.rep_u + ui], sw = maps[sg.rep_w + wi];
  r.F = sides[sg.side_u + su];
  r.T = sides[sg.side_w + sw];
  r.bytes = (sg.has_override && overrides) ? overrides[idx] : sg.bytes;
  r.sig = sig;
  r.local = su * sg.Sw + sw;
  r.R = sg.R;
  r.pad = 0;
  for (int d = 0; d < tpk::kMaxR; ++d) r.dt[d] = sg.dt[d];
}

__device__ __forceinline__ void pair_rec_one(const SigDesc* __restrict__ sigs, const int32_t* __restrict__ pair_sig,
                                             const int32_t* __restrict__ maps, const tpk::SideDesc* __restrict__ sides,
                                             const double* __restrict__ overrides, int64_t idx,
                                             PairRec* __restrict__ out) {
  PairRec r;
  pair_rec_of(sigs, pair_sig, maps, sides, overrides, idx, r);
  out[idx] = r;
}

__global__ void pair_rec_kernel(const SigDesc* __restrict__ sigs, const int32_t* __restrict__ pair_sig,
                                const int32_t* __restrict__ maps, const tpk::SideDesc* __restrict__ sides,
                                const double* __restrict__ overrides, int64_t total, PairRec* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  pair_rec_one(sigs, pair_sig, maps, sides, overrides, idx, out);
}

// The set-up kernels of many plans in one launch each (batched uploads):
// thread i finds its plan by bisection over the prefix sums.
struct UpJob {
  const SideJob* jobs;
  const Strat* tables;
  tpk::SideDesc* sides;
  const SigDesc* sigs;
  const int32_t* pair_sig;
  const int32_t* maps;
  const double* overrides;
  PairRec* recs;
  int32_t njobs, pad;
};

__device__ __forceinline__ int bisect_off(const int64_t* off, int n, int64_t x) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void batch_side_kernel(const UpJob* __restrict__ up, int n, const int64_t* __restrict__ off) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= off[n]) return;
  const int q = bisect_off(off, n, i);
  const UpJob& u = up[q];
  side_one(u.jobs, u.njobs, i - off[q], u.tables, u.sides);
}

__global__ void batch_pair_rec_kernel(const UpJob* __restrict__ up, int n, const int64_t* __restrict__ off) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= off[n]) return;
  const int q = bisect_off(off, n, i);
  const UpJob& u = up[q];
  pair_rec_one(u.sigs, u.pair_sig, u.maps, u.sides, u.overrides, i - off[q], u.recs);
}

// Scheduling state of a launch. Zeroed once (memset) when the arena is set
// up; afterwards the last CTA of every launch zeroes the counters it used, so
// a build is one kernel node with no memset in front. Errors alternate
// between two slots by launch parity: a launch writes err_c[parity] and
// clears the other slot for the next one.
// A counter alone on its 128-B line: the waiting CTAs poll these while the
// warps bump them, and lines shared with other counters would queue all of
// that traffic on one L2 slice.
struct alignas(128) Line {
  int v;
  int pad[31];
};

struct Sched {
  unsigned long long err_c[2];  // ~(smallest error key); 0 = no error
  int head;                  // unused
  int exit_count;            // CTAs done (the last one resets)
  int timeline;              // record the timestamps below
  int pad;
  // %globaltimer ns (min fields stored as complements): kernel start (min),
  // node rows done, first pair done (min), pairs done, first fan-out tile
  // past its wait (min), kernel end
  unsigned long long t[6];
  Line unit_head;            // next phase-1 unit: node row, then class pair (chunk)
  Line node_done;            // node-class rows finished
  Line pairs_done[1];        // per edge class (allocated to the class count)
};

__device__ __forceinline__ void flag_error(unsigned long long* err, uint64_t key) {
  atomicMax(err, ~(unsigned long long)key);  // max of ~key = min of key
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// timeline slot k: max of the timestamp, or min for the complemented slots
// (`on`: the execute's timeline flag, passed in the kernel arguments)
__device__ __forceinline__ void stamp(Sched* s, int on, int k, bool is_min) {
  if (!on) return;
  const unsigned long long t = gtimer();
  atomicMax(&s->t[k], is_min ? ~t : t);
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// counter bump that publishes this thread's earlier stores (pairs with ld_acquire)
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" : : "l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Spin (relaxed: an acquire load also invalidates the SM's L1, which the
// other CTAs there are reading through) until *p >= v, then acquire once.
__device__ __forceinline__ void wait_relaxed(const int* p, int v) {
  for (unsigned ns = 64; ld_relaxed(p) < v; ns = ns < 512 ? 2 * ns : ns) __nanosleep(ns);
}

__device__ __forceinline__ void wait_at_least(const int* p, int v) {
  wait_relaxed(p, v);
  (void)ld_acquire(p);
}

// Class-table entries are published without fences: a pair warp stores its
// entry and bumps the class counter with a relaxed add; a fan-out range
// waits for the counters of the classes it reads (node rows use a release). The counter may become visible before an entry's store, so entries
// start as kUnset (a signalling NaN no arithmetic produces) and a reader that
// finds kUnset retries until the store lands. (A CTA reaches phase 2 only
// after the unit queue is drained, so every entry it may wait for belongs to
// a running warp.) Two parity blocks of tables alternate between launches;
// a launch refills the other one.
constexpr unsigned long long kUnset = 0xfff4000000000badull;

__device__ __forceinline__ double ld_acquire_f64(const double* p) {
  double v;
  asm volatile("ld.acquire.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// The retry is an acquire load: it also drops the SM's L1 lines, so the
// stale copy that returned kUnset does not fail the next reads of its line.
__device__ __forceinline__ double table_load(const double* p);

// A (cost, volume) entry, written by one 16-B store.
__device__ __forceinline__ double2 table_load2(const double2* p) {
  double2 v = *p;
  if (__double_as_longlong(v.x) == (long long)kUnset || __double_as_longlong(v.y) == (long long)kUnset) {
    v.x = table_load(&p->x);
    v.y = table_load(&p->y);
  }
  return v;
}

__device__ __forceinline__ double table_load(const double* p) {
  double v = *p;
  if (__double_as_longlong(v) != (long long)kUnset) return v;
  v = ld_acquire_f64(p);
  for (unsigned ns = 64; __double_as_longlong(v) == (long long)kUnset; ns = ns < 512 ? 2 * ns : ns) {
    __nanosleep(ns);
    v = ld_acquire_f64(p);
  }
  return v;
}

__global__ void fill_kernel(double* __restrict__ p, int64_t n, unsigned long long bits) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = __longlong_as_double((long long)bits);
}

__device__ __forceinline__ void red_relaxed_add(int* p, int v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" : : "l"(p), "r"(v) : "memory");
}

struct FusedArgs {
  int timeline;  // phase timestamps on (the kernel parameter, not a device read at launch)
  // node classes
  const ClassDesc* classes;
  int ncls;
  int64_t total_rows;
  const SliceChk* chks;
  const SlotDesc* slots;
  const Occ* occs;
  double2* cls_sv;     // node-class rows: (intra cost, intra volume)
  double* cls_mem;
  double* cls_memdiv;
  // edge classes
  unsigned* pair_ns;  // timeline: per class pair / node-row item duration
  unsigned* item_ns;
  unsigned* fan_ns;
  const SigDesc* sigs;
  int nsigs;
  const int32_t* pair_sig;  // edge class of every table entry
  const PairRec* pairs;     // per table entry
  unsigned* pair_prof;      // timeline: per entry clocks of the pricing sections
  unsigned* warp_exit;      // timeline: globaltimer (low bits) when each warp leaves phase 1
  const int32_t* row_cls;   // node class of every class row
  const int32_t* maps;

  int64_t total_pairs;
  const double* overrides;
  const tpk::SideDesc* sides;
  double2* r_tab;      // this launch's class tables (cost, volume) (parity buffer), kUnset-filled
  double* next_tables; // the other parity's block (all tables), refilled during this launch
  int64_t tables_len;  // doubles per parity block
  // fan-out
  const EdgeDesc* edges;  // graph edges, by id
  const FanSeg* fsegs;    // per graph edge
  const int32_t* range_first;   // first edge of every edge range
  const int32_t* nrange_first;  // first operator of every node range
  int e0, e1;             // the execute's edge range
  int64_t A0, A1;         // its aux ids
  int64_t range_len;      // aux edges per fan-out item
  double* e_sec;
  double* e_vol;
  double* e_mem;
  char* records;
  int general_store;  // records requested or not all three SoA tensors given
  const int64_t* op_node;  // node_base per operator [num_ops + 1]
  const int64_t* op_row;   // class row of strategy 0 per operator
  int nops;
  int64_t num_nodes;
  int64_t node_range_len;  // aux nodes per node range
  double* n_sec;
  double* n_vol;
  double* n_mem;
  // phase-2 items: [0, i_exp) node ranges, [i_exp, i_end) edge ranges
  int i_exp, i_end;
  int warp_form;  // pairs: 1 = warp per pair, 0 = thread per pair
  // batches (thread form): plans equal but for their bandwidths share their
  // class pairs -- the leader infers every pair once and prices it for each
  // member (group: member indices into the batch's args, the leader first);
  // a member's pairs are not units of its own
  const int32_t* group;
  int group_n;
  int priced_by_leader;
  // batches (thread form): the op list of every class-table entry, inferred
  // once per distinct class key of the batch by infer_kernel; table entry r
  // of base class c is oplists + (cls_ops[c] + r - pair_begin(c)) * kOpWords
  const uint32_t* oplists;
  const int64_t* cls_ops;
  int direct;  // priced in the fan-out from the op lists: no pair units, no class tables
  int rows_thread;  // node-class rows one per thread, 32 per unit (batches without published counters)

  // shared
  const Strat* tables;
  Env env;
  int l_log2;
  int n_log2;
  const double* bw_tab;     // inter/ct, tpk::kBwTab entries
  const double* scale_tab;  // AllToAll scale, kScaleDim^2 entries
  Sched* sched;
  unsigned long long* err;  // this launch's error slot
  int parity;               // of the launch (error slot)
  int nsigs_reset;          // pairs_done counters the last CTA zeroes
};

constexpr int kFusedThreads = 256;
// bandwidth-group member seconds of the batch kernel's thread-form pricing
// (pair_thread), one column per thread: dynamic shared memory of fused_batch_kernel
static_assert(tpk::kBwEntries == tpk::kBwTab, "bandwidth table layout");
constexpr int kMsecBytes = (int)(tpk::kGroupMax * kFusedThreads * sizeof(double));
constexpr int kUC5 = 4;  // units per chunk of form 5's table launch

// The terms of one tensor occurrence of a node-class row (aux_graph.hpp:120-167):
// its shard bytes tm (added to the memory if has_m) and, for a tensor the
// operator's non-slicing axes replicate (group > 1), the AllReduce volume tv
// and seconds tc (infer_ct_allreduce, cost_model.hpp:75-97; has_v).
__device__ __forceinline__ void occ_terms(const FusedArgs& a, const ClassDesc& cd, const Strat& st, int q, double& tv,
                                          double& tc, double& tm, bool& has_v, bool& has_m) {
  const Occ oc = a.occs[q];
  const SlotDesc& sd = a.slots[cd.slot_begin + oc.slot];
  int sdiv = 0;
  for (int d = 0; d < sd.R; ++d)
    if (sd.sa[d] >= 0) sdiv += st.deg[sd.sa[d]];
  const int64_t shard_el = sdiv >= 63 ? 0 : (sd.elements >> sdiv);
  const double sb = (double)shard_el * sd.es;  // layout.hpp:125-129
  has_m = oc.in_memory;                        // aux_graph.hpp:151-167
  tm = sb;
  tv = tc = 0;
  has_v = false;
  int glog = 0;
  for (int ax = 0; ax < cd.p; ++ax)
    if ((oc.nonslicing >> ax) & 1) glog += st.deg[ax];
  if (glog > 0) {  // group > 1
    const int64_t pd = sdiv > a.n_log2 ? 0 : ((int64_t)1 << (a.n_log2 - sdiv));
    int64_t remain = a.env.local, dev_in = 1;
    for (int k = 0; k < st.depth; ++k) {
      bool contains = false;
      for (int d = 0; d < sd.R; ++d) contains |= sd.sa[d] >= 0 && st.dmap[sd.sa[d]] == k;
      const int64_t ek = (int64_t)1 << st.mx[k];
      if (!contains && remain > 1) dev_in *= remain > ek ? ek : remain;
      remain >>= st.mx[k];  // remain / ek, ek a power of two, remain >= 0
    }
    const int64_t ct = dev_in >= pd ? 0 : (dev_in > 1 ? a.env.local / dev_in : a.env.local);
    const double n = (double)((int64_t)1 << glog);
    tv = 2.0 * (n - 1) / n * sb;  // allreduce_volume, cost_model.hpp:39-43
    tc = tv / tpk::eff_bw(ct, a.env);
    has_v = true;
  }
}

// One aux-node row of a node class (aux_graph.hpp:120-167) on one warp:
// lanes take the slice checks and the tensor occurrences in parallel (their
// descriptor loads overlap), lane 0 then accumulates the terms in occurrence
// order, so the sums round exactly as the reference's sequential loop.
__device__ void node_row(const FusedArgs& a, int64_t row) {
  const int lane = threadIdx.x & 31;
  const ClassDesc cd = a.classes[a.row_cls[row]];
  const int64_t s = row - cd.row_base;
  const Strat& st = a.tables[cd.table + s];  // indexed by axis: read in place (L1), not copied to local memory
  // layout.hpp:349-367: every slice in axis order must divide its extent;
  // the first failing one (in order) names the error
  for (int c0 = cd.chk_begin; c0 < cd.chk_end; c0 += 32) {
    const int c = c0 + lane;
    int kind = 0;
    if (c < cd.chk_end) {
      const SliceChk k = a.chks[c];
      if (k.slot < 0) kind = tpk::kUnknownSliceTensor;
      else if (st.deg[k.axis] > k.v) kind = tpk::kIndivisible;
    }
    const unsigned bad = __ballot_sync(0xffffffffu, kind != 0);
    if (bad) {
      if (lane == __ffs(bad) - 1) {
        flag_error(a.err, ekey(1 + (uint64_t)(cd.first_node + s) * 2 + 1, kind));
        a.cls_sv[row] = make_double2(0.0, 0.0);
        a.cls_mem[row] = a.cls_memdiv[row] = 0;
      }
      return;
    }
  }
  double sec = 0, vol = 0, mem = 0;
  for (int q0 = cd.occ_begin; q0 < cd.occ_end; q0 += 32) {
    const int q = q0 + lane;
    double tv = 0, tc = 0, tm = 0;  // this occurrence's terms
    bool has_v = false, has_m = false;
    if (q < cd.occ_end) occ_terms(a, cd, st, q, tv, tc, tm, has_v, has_m);
    const int cnt = min(32, cd.occ_end - q0);
    for (int i = 0; i < cnt; ++i) {  // in occurrence order
      const double v = __shfl_sync(0xffffffffu, tv, i);
      const double c = __shfl_sync(0xffffffffu, tc, i);
      const double m = __shfl_sync(0xffffffffu, tm, i);
      const unsigned flags = __shfl_sync(0xffffffffu, (has_v ? 1u : 0u) | (has_m ? 2u : 0u), i);
      if (flags & 2u) mem += m;
      if (flags & 1u) {
        vol += v;
        sec += c;
      }
    }
  }
  if (lane == 0) {
    a.cls_sv[row] = make_double2(sec, vol);
    a.cls_mem[row] = mem;
    a.cls_memdiv[row] = mem / cd.indeg;  // aux_graph.hpp:292
  }
}

// The same row on one thread (batches: 32 consecutive rows per warp, mostly
// of one class, so the lanes run the same loops): checks, then occurrences,
// in order.
__device__ void node_row_thread(const FusedArgs& a, int64_t row) {
  const ClassDesc cd = a.classes[a.row_cls[row]];
  const int64_t s = row - cd.row_base;
  const Strat& st = a.tables[cd.table + s];
  for (int c = cd.chk_begin; c < cd.chk_end; ++c) {
    const SliceChk k = a.chks[c];
    const int kind = k.slot < 0 ? tpk::kUnknownSliceTensor : (st.deg[k.axis] > k.v ? tpk::kIndivisible : 0);
    if (kind) {
      flag_error(a.err, ekey(1 + (uint64_t)(cd.first_node + s) * 2 + 1, kind));
      a.cls_sv[row] = make_double2(0.0, 0.0);
      a.cls_mem[row] = a.cls_memdiv[row] = 0;
      return;
    }
  }
  double sec = 0, vol = 0, mem = 0;
  for (int q = cd.occ_begin; q < cd.occ_end; ++q) {
    double tv, tc, tm;
    bool has_v, has_m;
    occ_terms(a, cd, st, q, tv, tc, tm, has_v, has_m);
    if (has_m) mem += tm;
    if (has_v) {
      vol += tv;
      sec += tc;
    }
  }
  a.cls_sv[row] = make_double2(sec, vol);
  a.cls_mem[row] = mem;
  a.cls_memdiv[row] = mem / cd.indeg;  // aux_graph.hpp:292
}

__device__ __forceinline__ int sig_of_pair(const FusedArgs& a, int64_t idx) { return a.pair_sig[idx]; }

// One class-table entry on one thread (register form, tp_fast.cuh); with a
// bandwidth group (batches) the entry of every member, inferred once. One
// call site of the register form keeps the kernels' code (and the
// instruction-cache footprint) single.
__device__ void pair_thread(const FusedArgs& a, int64_t idx, const double* price,
                            const FusedArgs* __restrict__ all = nullptr) {
  const PairRec& pr = a.pairs[idx];
  const tpk::SideDesc F = pr.F, T = pr.T;
  const int R = pr.R;
  const int g = (all && a.group_n > 1) ? a.group_n : 1;
  // member seconds in the batch kernel's dynamic shared memory (kMsecBytes)
  extern __shared__ double s_msec[];
  tpk::MultiSec ms;
  ms.g = g;
  ms.base = reinterpret_cast<const char*>(all);
  ms.idx = a.group;
  ms.stride = (int)sizeof(FusedArgs);
  ms.env_off = (int)offsetof(FusedArgs, env);
  ms.bw_off = (int)offsetof(FusedArgs, bw_tab);
  ms.sec = s_msec + threadIdx.x;
  ms.sec_stride = kFusedThreads;
  for (int q = 1; q < g; ++q) ms.s(q) = 0;
  double sec = 0, vol = 0;
  if (!tpk::same_side(F, T, R)) {  // aux_graph.hpp:260
    const int st = tpk::pair_cost_sd(R, F, T, nullptr, nullptr, pr.dt, pr.bytes, a.env, a.l_log2,
                                     tpk::FastTabs{price, price + tpk::kBwTab}, sec, vol, nullptr,
                                     g > 1 ? &ms : nullptr);
    if (st) {
      const uint64_t key = ekey(kEdgePhase + (uint64_t)(a.sigs[pr.sig].first_aux + pr.local) * 2 + 1, st);
      flag_error(a.err, key);
      for (int q = 1; q < g; ++q) flag_error(all[a.group[q]].err, key);
      sec = vol = 0;
      for (int q = 1; q < g; ++q) ms.s(q) = 0;
    }
  }
  a.r_tab[idx] = make_double2(sec, vol);
  for (int q = 1; q < g; ++q) all[a.group[q]].r_tab[idx] = make_double2(ms.s(q), vol);
}

// The inference pass of a batch: one thread per distinct class-table entry
// (job q covers entries recs[0, count) of its first plan), writing the op
// lists the fan-out prices for every plan with that class key.
struct InferJob {
  // the first plan with the class key: its descriptors (pair_rec_of)
  const SigDesc* sigs;
  const int32_t* pair_sig;
  const int32_t* maps;
  const tpk::SideDesc* sides;
  int64_t first;  // the class's first table entry in that plan
  int64_t out;    // its first op list (in entries)
};

__global__ void infer_kernel(const InferJob* __restrict__ jobs, int njobs, const int64_t* __restrict__ off,
                             uint32_t* __restrict__ oplists) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= off[njobs]) return;
  const int q = bisect_off(off, njobs, i);
  const InferJob& jb = jobs[q];
  PairRec pr;
  pair_rec_of(jb.sigs, jb.pair_sig, jb.maps, jb.sides, nullptr, jb.first + (i - off[q]), pr);
  uint32_t w[tpk::kOpWords];
  tpk::infer_ops(pr.R, pr.F, pr.T, pr.dt, w);
  uint4* o = reinterpret_cast<uint4*>(oplists + (jobs[q].out + (i - off[q])) * tpk::kOpWords);
#pragma unroll
  for (int k = 0; k < tpk::kOpWords / 4; ++k) o[k] = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
}

// One class-table entry on one warp (warp form, tp_warp.cuh); lane 0 writes.
__device__ void pair_warp(const FusedArgs& a, int64_t idx, const double* price) {
  const int lane = threadIdx.x & 31;
  const PairRec* pr = a.pairs + idx;
  double sec = 0, vol = 0;
  const int R = pr->R;
  if (!tpk::same_side(pr->F, pr->T, R)) {  // aux_graph.hpp:260
    tpk::WarpEnv we;
    we.env = a.env;
    we.l_log2 = a.l_log2;
    we.tab = tpk::PriceTabs{price, price + tpk::kBwTab};
    const int st = tpk::redist_cost_warp(R, &pr->F, &pr->T, pr->dt, pr->bytes, we, sec, vol, nullptr,
                                         a.pair_prof ? a.pair_prof + 8 * idx : nullptr);
    if (st) {
      if (lane == 0)
        flag_error(a.err, ekey(kEdgePhase + (uint64_t)(a.sigs[pr->sig].first_aux + pr->local) * 2 + 1, st));
      sec = vol = 0;
    }
  }
  if (lane == 0) {
    a.r_tab[idx] = make_double2(sec, vol);  // one 16-B store
  }
}

// Fan-out range: the aux edges [start, end) of the execute's edge range,
// contiguous in the reference's id order (edge, su, sw) and so in every
// output array; all ranges have the same length, one wave of CTAs. Thread 0
// stages the range's edges (up to kSegs at a time) in shared memory and waits
// (acquire) for the node rows and the tables of their classes. Each thread
// then walks its ids: aux id -> edge segment -> (su, sw) -> consumer class
// row + table entry (aux_graph.hpp:286-295). Consecutive lanes write
// consecutive ids, so every warp store is one 256-B segment per array.
constexpr int kSegs = 32;  // one per lane of warp 0

// An aux edge's redistribution priced in the fan-out (batches with op
// lists): the entry's op list with the base class's bytes and this plan's
// bandwidths -- the same expressions and order as its table entry would
// have. An inference error is flagged at the aux edge's own id: the smallest
// such id is the entry's first use, where the reference throws.
__device__ __noinline__ void full_entry(const FusedArgs& a, int64_t r, int64_t o, double& sec, double& vol) {
  PairRec pr;  // from the descriptors (a batch priced in the fan-out uploads no pair records)
  pair_rec_of(a.sigs, a.pair_sig, a.maps, a.sides, a.overrides, r, pr);
  double s2 = 0, v2 = 0;
  const int st = tpk::pair_cost_sd(pr.R, pr.F, pr.T, nullptr, nullptr, pr.dt, pr.bytes, a.env, a.l_log2,
                                   tpk::FastTabs{a.bw_tab, a.bw_tab + tpk::kBwTab}, s2, v2, nullptr);
  if (st) flag_error(a.err, ekey(kEdgePhase + (uint64_t)o * 2 + 1, st));
  sec = st ? 0.0 : s2;
  vol = st ? 0.0 : v2;
}

__device__ __forceinline__ void direct_entry(const FusedArgs& a, const FanSeg& g, int64_t r, int64_t o, double& sec,
                                             double& vol) {
  const uint32_t* ol = a.oplists + (g.opb + (r - g.pb)) * tpk::kOpWords;
  const uint32_t h = ol[0];
  sec = vol = 0;
  if (h & tpk::kOpsFull) {
    full_entry(a, r, o, sec, vol);
    return;
  }
  const int st = (h >> 8) & 0xff;
  if (st) {
    flag_error(a.err, ekey(kEdgePhase + (uint64_t)o * 2 + 1, st));
    return;
  }
  if (h & 0xff)
    tpk::price_ops(ol + 1, h & 0xff, g.ovr ? a.overrides[r] : g.bytes, a.env, a.l_log2,
                   tpk::FastTabs{a.bw_tab, a.bw_tab + tpk::kBwTab}, sec, vol);
}

// One class-table entry of a batch plan from its inferred op list: the
// reference's expressions summed in op order (tp_fast.cuh price_ops) with
// this plan's bytes and bandwidths; entries the op list cannot represent take
// the full register form. Errors keep the entry's first aux id (its class's
// first edge, first strategy pair with these layouts).
__device__ __noinline__ void pair_entry_full(const FusedArgs& a, int64_t idx, const double* price) {
  PairRec pr;
  pair_rec_of(a.sigs, a.pair_sig, a.maps, a.sides, a.overrides, idx, pr);
  double sec = 0, vol = 0;
  const int st = tpk::pair_cost_sd(pr.R, pr.F, pr.T, nullptr, nullptr, pr.dt, pr.bytes, a.env, a.l_log2,
                                   tpk::FastTabs{price, price + tpk::kBwTab}, sec, vol, nullptr);
  if (st) flag_error(a.err, ekey(kEdgePhase + (uint64_t)(a.sigs[pr.sig].first_aux + pr.local) * 2 + 1, st));
  a.r_tab[idx] = st ? make_double2(0.0, 0.0) : make_double2(sec, vol);
}

__device__ __forceinline__ void pair_from_ops(const FusedArgs& a, int64_t idx, const double* price) {
  const int sig = a.pair_sig[idx];
  const SigDesc& sg = a.sigs[sig];
  const uint32_t* ol = a.oplists + (a.cls_ops[sig] + (idx - sg.pair_begin)) * tpk::kOpWords;
  const uint32_t h = ol[0];
  if (h & tpk::kOpsFull) {
    pair_entry_full(a, idx, price);
    return;
  }
  double sec = 0, vol = 0;
  const int st = (h >> 8) & 0xff;
  if (st) {
    PairRec pr;
    pair_rec_of(a.sigs, a.pair_sig, a.maps, a.sides, a.overrides, idx, pr);
    flag_error(a.err, ekey(kEdgePhase + (uint64_t)(sg.first_aux + pr.local) * 2 + 1, st));
  } else if (h & 0xff) {
    tpk::price_ops(ol + 1, h & 0xff, sg.has_override ? a.overrides[idx] : sg.bytes, a.env, a.l_log2,
                   tpk::FastTabs{price, price + tpk::kBwTab}, sec, vol);
  }
  a.r_tab[idx] = make_double2(sec, vol);
}

// kDirect: priced here from the op lists (no class tables); kWait = false:
// the tables and rows come from an earlier launch (no counters, no unset
// checks).
// The fan-out's common case in a batch's second launch (measured: cfg5
// 0.735 -> 0.697 ms; the single-plan build is not faster with it, 32.9 vs
// 33.2 us, and keeps one id per thread): the three SoA tensors from class
// tables, no AuxEdge records. A thread writes two consecutive ids (an even output
// position and the next), so each tensor gets one 16-B store per pair, and
// keeps its edge's fields in registers while it stays in the edge; the warp
// still writes 512 consecutive bytes per tensor and instruction. Pairs start
// at 16-B aligned output positions (`par`: the tensors' phase); ids of a pair
// outside [pos, span_end) are skipped (a span starting at an edge boundary may
// be misaligned: its first pair then starts one id early).
struct PairIds {  // (edge segment, su, sw) of an id, and the segment's fields
  int si;
  int32_t su, sw, Sw, Wn, uid_u, uid_w, ident;
  int64_t end, pb, wrow;
  double f;
};

__device__ __forceinline__ void enter_seg(const FanSeg* seg, int si, int64_t o, PairIds& c) {
  const FanSeg& g = seg[si];
  c.si = si;
  c.Sw = g.Sw;
  c.Wn = g.Wn;
  c.uid_u = g.uid_u;
  c.uid_w = g.uid_w;
  c.ident = g.ident;
  c.end = g.end;
  c.pb = g.pb;
  c.wrow = g.wrow;
  c.f = g.f;
  const int32_t j = (int32_t)(o - g.begin);
  c.su = j / c.Sw;
  c.sw = j - c.su * c.Sw;
}

template <bool kWait>
__device__ __forceinline__ void pair_vals(const FusedArgs& a, const PairIds& c, double& cs, double& vs, double& ms) {
  const int64_t r = c.ident ? c.pb + (int64_t)c.su * c.Sw + c.sw
                            : c.pb + (int64_t)a.maps[c.uid_u + c.su] * c.Wn + a.maps[c.uid_w + c.sw];
  const int64_t row = c.wrow + c.sw;
  const double2 cv = a.cls_sv[row];
  const double2 rv = kWait ? table_load2(a.r_tab + r) : a.r_tab[r];
  cs = cv.x + rv.x * c.f;  // aux_graph.hpp:290-291
  vs = cv.y + rv.y * c.f;
  ms = a.cls_memdiv[row];  // :292
}

template <bool kWait>
__device__ __forceinline__ void fanout_pairs(const FusedArgs& a, const FanSeg* seg, int64_t pos, int64_t span_end,
                                             int par) {
  constexpr int64_t kStep = 2 * kFusedThreads;
  const int64_t base = pos - ((pos - a.A0 + par) & 1);  // a 16-B aligned output position
  PairIds c;
  c.si = -1;
  int32_t st_q = 0, st_r = 0;  // (su, sw) stride of kStep ids in this edge
  for (int64_t o = base + 2 * threadIdx.x; o < span_end; o += kStep) {
    const int64_t o1 = o + 1;
    const bool in0 = o >= pos, in1 = o1 < span_end;
    // the pair's first id: (su, sw) advanced by the stride, or a new edge
    if (c.si >= 0 && o < c.end) {
      c.su += st_q;
      c.sw += st_r;
      if (c.sw >= c.Sw) {
        c.sw -= c.Sw;
        ++c.su;
      }
    } else {
      int si = c.si < 0 ? 0 : c.si;
      const int64_t oo = o < pos ? pos : o;  // an id before the span: locate from the span start
      while (oo >= seg[si].end) ++si;
      enter_seg(seg, si, o < seg[si].begin ? seg[si].begin : o, c);
      if (o < seg[si].begin) {  // o is the previous edge's last id (skipped): (su, sw) one before
        if (c.sw == 0) {
          c.sw = c.Sw - 1;
          --c.su;
        } else {
          --c.sw;
        }
      }
      st_q = (int32_t)(kStep / c.Sw);
      st_r = (int32_t)(kStep - (int64_t)st_q * c.Sw);
    }
    double cs0 = 0, vs0 = 0, ms0 = 0, cs1 = 0, vs1 = 0, ms1 = 0;
    if (in0) pair_vals<kWait>(a, c, cs0, vs0, ms0);
    if (in1) {  // the second id: the next (su, sw), or the next edge's (0, 0)
      if (o1 < c.end) {
        PairIds d = c;
        if (++d.sw == d.Sw) {  // (from a skipped first id of the previous edge, (-1, Sw-1) -> (0, 0))
          d.sw = 0;
          ++d.su;
        }
        pair_vals<kWait>(a, d, cs1, vs1, ms1);
      } else {
        PairIds d;
        enter_seg(seg, c.si + 1, o1, d);
        pair_vals<kWait>(a, d, cs1, vs1, ms1);
      }
    }
    const int64_t q = o - a.A0;
    if (in0 && in1) {  // one 16-B streaming store per tensor
      __stcs(reinterpret_cast<double2*>(a.e_sec + q), make_double2(cs0, cs1));
      __stcs(reinterpret_cast<double2*>(a.e_vol + q), make_double2(vs0, vs1));
      __stcs(reinterpret_cast<double2*>(a.e_mem + q), make_double2(ms0, ms1));
    } else if (in0) {
      __stcs(a.e_sec + q, cs0);
      __stcs(a.e_vol + q, vs0);
      __stcs(a.e_mem + q, ms0);
    } else if (in1) {
      __stcs(a.e_sec + q + 1, cs1);
      __stcs(a.e_vol + q + 1, vs1);
      __stcs(a.e_mem + q + 1, ms1);
    }
  }
}

// kPer: output positions a thread has in flight (the loads of kPer ids
// overlap). The single-plan build keeps kFanPer (measured best with its
// short ranges); a batch's second launch reads its tables from L2 / DRAM and
// needs more in flight.
template <bool kDirect, bool kWait = true, int kPer = kFanPer, bool kLean = false>
__device__ void fanout_range(const FusedArgs& a, int item, FanSeg* seg, int* s_n, int* s_edge) {
  const unsigned long long t0 = a.fan_ns ? gtimer() : 0;
  const int64_t start = a.A0 + (int64_t)item * a.range_len;
  const int64_t end = min(start + a.range_len, a.A1);
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) *s_edge = a.range_first[item];  // host-computed
  int64_t pos = start;
  bool first = true;
  // the common case (the three SoA tensors, no records, tables): pairs of ids
  // per thread, when the three tensors share their 16-B alignment phase
  const int par = (int)((reinterpret_cast<uintptr_t>(a.e_sec) >> 3) & 1);
  const bool lean = kLean && !kDirect && !a.general_store &&
                    par == (int)((reinterpret_cast<uintptr_t>(a.e_vol) >> 3) & 1) &&
                    par == (int)((reinterpret_cast<uintptr_t>(a.e_mem) >> 3) & 1);
  while (pos < end) {
    __syncthreads();
    if (threadIdx.x < 32) {  // warp 0 stages the next kSegs edges, lane per edge
      const int e = *s_edge + lane;
      FanSeg g;
      bool in = false;
      if (e < a.e1) {
        g = a.fsegs[e];
        in = g.begin < end;
      }
      if (in) {
        // relaxed: the entries are unset-checked; an acquire here would also
        // drop the L1 lines the SM's other CTAs are reading
        if (kDirect) g.opb = a.cls_ops[g.base];
        else if (kWait) wait_relaxed(&a.sched->pairs_done[g.base].v, g.need);
        seg[lane] = g;
      }
      const int n = __popc(__ballot_sync(0xffffffffu, in));  // a prefix of the lanes
      if (kWait && first) {
        if (lane == 0) wait_at_least(&a.sched->node_done.v, (int)a.total_rows);
        __syncwarp();
      }
      if (lane == 0) {
        *s_n = n;
        *s_edge += n;
        if (first) {
          stamp(a.sched, a.timeline, 4, true);
          if (a.fan_ns) {
            a.fan_ns[3 * item] = (unsigned)t0;
            a.fan_ns[3 * item + 1] = (unsigned)(gtimer() - t0);
          }
        }
      }
    }
    first = false;
    __syncthreads();
    const int n = *s_n;
    const int64_t span_end = min(end, seg[n - 1].end);
    if (lean) {
      fanout_pairs<kWait>(a, seg, pos, span_end, par);
      pos = span_end;
      continue;
    }
    if (!kDirect && kPer == 1 && !a.general_store) {
      // The three SoA tensors (the single build's common case): edge by edge,
      // the edge's fields in registers, 32-bit (su, sw) coordinates and table
      // offsets, one division per edge per thread. Same ids per thread as the
      // general loop below: id o belongs to thread (o - pos) mod kFusedThreads.
      for (int i = 0; i < n; ++i) {
        const FanSeg& gs = seg[i];
        const int64_t lo = max(pos, gs.begin), hi = min(span_end, gs.end);
        int64_t d = (pos + (int64_t)threadIdx.x - lo) % kFusedThreads;
        if (d < 0) d += kFusedThreads;
        int64_t o = lo + d;
        if (o >= hi) continue;
        const int32_t Sw = gs.Sw, Wn = gs.Wn, st_q = gs.st_q, st_r = gs.st_r;
        const bool ident = gs.ident != 0;
        const double f = gs.f;
        const int32_t* mu = a.maps + gs.uid_u;
        const int32_t* mw = a.maps + gs.uid_w;
        const double2* tab = a.r_tab + gs.pb;
        const double2* sv = a.cls_sv + gs.wrow;
        const double* md = a.cls_memdiv + gs.wrow;
        const int32_t j = (int32_t)(o - gs.begin);
        int32_t su = j / Sw, sw = j - su * Sw;
        double* es = a.e_sec - a.A0;
        double* ev = a.e_vol - a.A0;
        double* em = a.e_mem - a.A0;
        for (; o < hi; o += kFusedThreads) {
          const int32_t t = ident ? su * Sw + sw : mu[su] * Wn + mw[sw];
          const double2 cv = sv[sw];
          const double2 rv = kWait ? table_load2(tab + t) : tab[t];
          const double m = md[sw];
          __stcs(es + o, cv.x + rv.x * f);  // aux_graph.hpp:290-291
          __stcs(ev + o, cv.y + rv.y * f);
          __stcs(em + o, m);  // :292
          su += st_q;
          sw += st_r;
          if (sw >= Sw) {
            sw -= Sw;
            ++su;
          }
        }
      }
      pos = span_end;
      continue;
    }
    // (su, sw) of a thread's ids advance by a fixed stride within an edge;
    // a division only where the thread enters an edge
    int si = -1;
    int32_t su = 0, sw = 0;
    for (int64_t o0 = pos + threadIdx.x; o0 < span_end; o0 += kFusedThreads * kPer) {
      double cs[kPer], vs[kPer], ms[kPer];
      int64_t q[kPer];
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int64_t o = o0 + (int64_t)k * kFusedThreads;
        q[k] = -1;
        if (o >= span_end) continue;
        if (si >= 0 && o < seg[si].end) {
          su += seg[si].st_q;
          sw += seg[si].st_r;
          if (sw >= seg[si].Sw) {
            sw -= seg[si].Sw;
            ++su;
          }
        } else {
          if (si < 0) si = 0;
          while (o >= seg[si].end) ++si;
          const int32_t j = (int32_t)(o - seg[si].begin);
          su = j / seg[si].Sw;
          sw = j - su * seg[si].Sw;
        }
        const FanSeg& g = seg[si];
        const int32_t j = su * g.Sw + sw;
        const int64_t r = g.ident ? g.pb + j : g.pb + (int64_t)a.maps[g.uid_u + su] * g.Wn + a.maps[g.uid_w + sw];
        // class rows and tables: written before the acquire above, reused
        // across the range's ids (L1)
        // class rows (released, acquired above) and tables: reused across
        // the range's ids, through L1
        const int64_t row = g.wrow + sw;
        const double2 cv = a.cls_sv[row];
        double2 rv;
        if (kDirect) direct_entry(a, g, r, o, rv.x, rv.y);
        else if (kWait) rv = table_load2(a.r_tab + r);
        else rv = a.r_tab[r];
        cs[k] = cv.x + rv.x * g.f;  // aux_graph.hpp:290-291
        vs[k] = cv.y + rv.y * g.f;
        ms[k] = a.cls_memdiv[row];                               // :292
        q[k] = o - a.A0;
        if (a.records) {  // topoplan::AuxEdge, 40 bytes (aux_graph.hpp:52-59)
          char* rec = a.records + q[k] * 40;
          *reinterpret_cast<int2*>(rec) = make_int2(g.e, (int)(g.nb_u + su));
          *reinterpret_cast<int2*>(rec + 8) = make_int2((int)(g.nb_w + sw), 0);
        }
      }
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        if (q[k] < 0) continue;
        if (!a.general_store) {
          __stcs(a.e_sec + q[k], cs[k]);  // streaming: written once, read by the host
          __stcs(a.e_vol + q[k], vs[k]);
          __stcs(a.e_mem + q[k], ms[k]);
        } else {
          if (a.e_sec) __stcs(a.e_sec + q[k], cs[k]);
          if (a.e_vol) __stcs(a.e_vol + q[k], vs[k]);
          if (a.e_mem) __stcs(a.e_mem + q[k], ms[k]);
          if (a.records) {
            char* rec = a.records + q[k] * 40;
            *reinterpret_cast<double*>(rec + 16) = cs[k];
            *reinterpret_cast<double*>(rec + 24) = vs[k];
            *reinterpret_cast<double*>(rec + 32) = ms[k];
          }
        }
      }
    }
    pos = span_end;
  }
  if (a.fan_ns) {
    __syncthreads();
    if (threadIdx.x == 0) a.fan_ns[3 * item + 2] = (unsigned)(gtimer() - t0);
  }
}

// Node tensors: every member operator of a node class gets the class rows.
// Node range: the aux nodes [start, end) get their node class's rows
// (aux_graph.hpp:120-167 values, one copy per member operator). Same walk as
// the fan-out: warp 0 finds and stages the operators (lane per operator),
// each thread copies its ids with kFanPer loads in flight.
struct NodeSeg {
  int64_t begin, end, row;
};

template <bool kWait = true>
__device__ void node_range(const FusedArgs& a, int item, NodeSeg* seg, int* s_n, int* s_op) {
  const int64_t start = (int64_t)item * a.node_range_len;
  const int64_t end = min(start + a.node_range_len, a.num_nodes);
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    *s_op = a.nrange_first[item];  // host-computed
    if (kWait) wait_at_least(&a.sched->node_done.v, (int)a.total_rows);
  }
  int64_t pos = start;
  while (pos < end) {
    __syncthreads();
    if (threadIdx.x < 32) {
      const int op = *s_op + lane;
      const bool in = op < a.nops && a.op_node[op] < end;
      if (in) seg[lane] = NodeSeg{a.op_node[op], a.op_node[op + 1], a.op_row[op]};
      const int n = __popc(__ballot_sync(0xffffffffu, in));
      if (lane == 0) {
        *s_n = n;
        *s_op += n;
      }
    }
    __syncthreads();
    const int64_t span_end = min(end, seg[*s_n - 1].end);
    int si = 0;
    for (int64_t o0 = pos + threadIdx.x; o0 < span_end; o0 += kFusedThreads * kFanPer) {
      double cs[kFanPer], vs[kFanPer], ms[kFanPer];
      int64_t q[kFanPer];
#pragma unroll
      for (int k = 0; k < kFanPer; ++k) {
        const int64_t o = o0 + (int64_t)k * kFusedThreads;
        q[k] = -1;
        if (o >= span_end) continue;
        while (o >= seg[si].end) ++si;
        const int64_t row = seg[si].row + (o - seg[si].begin);
        const double2 cv = a.cls_sv[row];
        cs[k] = cv.x;
        vs[k] = cv.y;
        ms[k] = a.cls_mem[row];
        q[k] = o;
      }
#pragma unroll
      for (int k = 0; k < kFanPer; ++k) {
        if (q[k] < 0) continue;
        if (a.n_sec) __stcs(a.n_sec + q[k], cs[k]);
        if (a.n_vol) __stcs(a.n_vol + q[k], vs[k]);
        if (a.n_mem) __stcs(a.n_mem + q[k], ms[k]);
      }
    }
    pos = span_end;
  }
}

// One phase-1 unit u of a plan: a node-class row, or a class pair (warp
// form) / 32 class pairs (thread form).
// kSync = false: the fan-out runs in a later launch (the kernel boundary
// orders everything), so no counters are published; kOps: thread-form pairs
// priced from the batch's op lists (pair_from_ops).
template <bool kWarpForm, bool kSync = true, bool kOps = false>
__device__ __forceinline__ void run_unit(const FusedArgs& a, int64_t u, const double* price,
                                         const FusedArgs* all = nullptr) {
  const int lane = threadIdx.x & 31;
  const unsigned long long t0 = (a.pair_ns || a.item_ns) ? gtimer() : 0;
  const int64_t row_units = a.rows_thread ? (a.total_rows + 31) / 32 : a.total_rows;
  if (!kSync && a.rows_thread && u < row_units) {
    const int64_t row = u * 32 + lane;
    if (row < a.total_rows) node_row_thread(a, row);
    return;
  }
  if (!a.rows_thread && u < a.total_rows) {
    node_row(a, u);
    if (kSync && lane == 0) {
      red_release_add(&a.sched->node_done.v, 1);  // rows: off the critical path, released
      if (a.item_ns) {
        a.item_ns[2 * u] = (unsigned)t0;
        a.item_ns[2 * u + 1] = (unsigned)(gtimer() - t0);
      }
    }
  } else if (kWarpForm) {
    const int64_t idx = u - row_units;
    pair_warp(a, idx, price);
    const int sig = a.pairs[idx].sig;
    if (lane == 0) {
      if (a.pair_ns) {
        a.pair_ns[2 * idx] = (unsigned)t0;
        a.pair_ns[2 * idx + 1] = (unsigned)(gtimer() - t0);
      }
      red_relaxed_add(&a.sched->pairs_done[sig].v, 1);  // no fence: see table_load
    }
  } else {
    const int64_t idx = (u - row_units) * 32 + lane;
    const bool valid = idx < a.total_pairs;
    const int sig = valid ? sig_of_pair(a, idx) : -1;
    const bool grouped = all && a.group_n > 1;
    if (valid) {
      if constexpr (kOps) pair_from_ops(a, idx, price);
      else pair_thread(a, idx, price, all);
    }
    if (!kSync) return;
    if (a.pair_ns && valid) {
      a.pair_ns[2 * idx] = (unsigned)t0;
      a.pair_ns[2 * idx + 1] = (unsigned)(gtimer() - t0);
    }
    // one counter update per (warp, edge class); no fence: see table_load
    const unsigned grp = __match_any_sync(0xffffffffu, sig);
    if (valid && lane == __ffs(grp) - 1) {
      if (grouped)
        for (int q = 0; q < a.group_n; ++q) red_relaxed_add(&all[a.group[q]].sched->pairs_done[sig].v, __popc(grp));
      else
        red_relaxed_add(&a.sched->pairs_done[sig].v, __popc(grp));
    }
  }
}

__device__ __forceinline__ int64_t plan_units(const FusedArgs& a) {
  const int64_t rows = a.rows_thread ? (a.total_rows + 31) / 32 : a.total_rows;
  if (a.priced_by_leader || a.direct) return rows;
  return rows + (a.warp_form ? a.total_pairs : (a.total_pairs + 31) / 32);
}

// The plan's per-launch reset, done by the last CTA to leave (one thread).
__device__ __forceinline__ void reset_plan(const FusedArgs& a) {
  Sched* sc = a.sched;
  sc->head = 0;
  sc->unit_head.v = 0;
  sc->node_done.v = 0;
  for (int i = 0; i < a.nsigs_reset; ++i) sc->pairs_done[i].v = 0;
  sc->err_c[a.parity ^ 1] = 0;
  sc->exit_count = 0;
}

// The whole build in one persistent launch. Phase 1: warps take units --
// node-class rows first (every fan-out needs them), then class pairs (one per
// warp, or 32 per warp in the thread form). CTA b starts with units 8b..8b+7
// (no atomic), then a warp claims further units alone from a counter behind
// all the static ones, skipping the atomic once the queue is drained, so no
// start-up burst serialises on the counter and a slow pair never idles the
// other warps of its CTA. Each
// finished unit bumps its counter with a release add. Phase 2: block work
// items for the fan-out tiles and the node fan-out; a tile waits (acquire)
// only for its own edge class's table and the node rows. A CTA reaches phase
// 2 only after its warps drained the unit queue, and every claimed unit runs
// to completion, so the waits always end. The latency-bound pricing and the
// write-bound fan-out overlap, with no launch gap or wave tail between them.
template <bool kWarpForm>
__global__ void __launch_bounds__(kFusedThreads, 4) fused_kernel(FusedArgs a) {
  __shared__ int s_unit, s_edge, s_nseg;
  __shared__ union {
    FanSeg f[kSegs];
    NodeSeg n[kSegs];
  } s_seg;
  const int lane = threadIdx.x & 31;
  const int64_t units = plan_units(a);
  if (threadIdx.x == 0) {
    stamp(a.sched, a.timeline, 0, true);
    // first units by CTA index: no start-up burst of atomics on one counter
    // (measured: units start ~0.6 us earlier, the build ~2 us shorter)
    s_unit = blockIdx.x * (kFusedThreads / 32);
  }
  // The pricing tables are read where they are (L1): staging them in shared
  // memory first held every warp behind their load from DRAM after the L2
  // flush (measured: pairs end ~1 us later, the build 30.8 vs 28.9 us).
  __syncthreads();
  // phase 1: node-class rows, then class pairs
  int64_t u = (int64_t)s_unit + (threadIdx.x >> 5);
  while (u < units) {
    run_unit<kWarpForm>(a, u, a.bw_tab);
    int next = 0;
    if (lane == 0)
    {  // the dynamic queue starts after every CTA's static first units
      const int base = (int)gridDim.x * (kFusedThreads / 32);
      next = base + ld_relaxed(&a.sched->unit_head.v) >= units ? INT_MAX : base + atomicAdd(&a.sched->unit_head.v, 1);
    }
    u = __shfl_sync(0xffffffffu, next, 0);
  }
  if (a.warp_exit && lane == 0) a.warp_exit[blockIdx.x * (kFusedThreads / 32) + (threadIdx.x >> 5)] = (unsigned)gtimer();
  // the next launch's tables start unset: every CTA refills a slice
  {
    const int64_t per = (a.tables_len + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = (int64_t)blockIdx.x * per, b1 = min(b0 + per, a.tables_len);
    for (int64_t i = b0 + threadIdx.x; i < b1; i += kFusedThreads)
      a.next_tables[i] = __longlong_as_double((long long)kUnset);
  }
  // phase 2: node ranges, then edge ranges; CTA b takes items b, b + grid, ...
  for (int item = blockIdx.x;; item += gridDim.x) {
    __syncthreads();  // s_seg reuse
    if (item >= a.i_end) {
      if (threadIdx.x == 0) {
        stamp(a.sched, a.timeline, 5, false);
        __threadfence();
        if (atomicAdd(&a.sched->exit_count, 1) == (int)gridDim.x - 1) {
          // every other CTA has finished: reset for the next launch
          reset_plan(a);
          __threadfence();
        }
      }
      return;
    }
    if (item < a.i_exp) node_range(a, item, s_seg.n, &s_nseg, &s_edge);
    else fanout_range<false>(a, item - a.i_exp, s_seg.f, &s_nseg, &s_edge);
  }
}

// Batches of plans (a sweep of independent scenarios) in ONE persistent
// launch: the units of all plans form one queue, then the phase-2 items of
// all plans; every unit and item runs exactly the single-plan code on its
// own plan's arguments, counters and tables. Offsets are prefix sums over the
// plans; a warp's (a CTA's) claims only increase, so it finds the plan of its
// next unit (item) by walking forward from the previous one.
struct BatchHdr {
  Line unit_head;
  Line exit_count;
};

__device__ __forceinline__ int find_plan(const int64_t* off, int n, int64_t x, int p) {
  // the plan q with off[q] <= x < off[q + 1]: gallop forward from the previous
  // plan (claims only increase), then bisect
  if (p >= 0 && off[p] <= x && (p + 1 >= n || off[p + 1] > x)) return p;
  int lo = (p < 0 || off[p] > x) ? 0 : p, hi;
  int step = 1;
  for (;;) {
    hi = lo + step;
    if (hi >= n || off[hi] > x) break;
    lo = hi;
    step <<= 1;
  }
  if (hi > n - 1) hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// pair forms in the batch: 1 = warp only, 2 = thread only, 0 = mixed;
// 3 = thread only with 2 CTAs per SM (128 registers: the register form's
// state without spills); 4 = thread form priced from the batch's op lists
// in the fan-out from the batch's op lists (infer_kernel ran first; the
// units are node rows only)
// kPhase (form 5, two launches): 1 = the units only (node rows and table
// entries, nothing published), 2 = the ranges only (reading what launch 1
// wrote; the kernel boundary orders them); 3 = both in one launch.
template <int kForm, int kPhase = 3>
__global__ void __launch_bounds__(kFusedThreads, kForm == 3 ? 2 : 4)
    fused_batch_kernel(const FusedArgs* __restrict__ args, int n, const int64_t* __restrict__ unit_off,
                       const int64_t* __restrict__ item_off, const int64_t* __restrict__ tab_off, BatchHdr* hdr,
                       unsigned long long* __restrict__ err_out, const int32_t* __restrict__ chunk_plan) {
  __shared__ int s_unit, s_edge, s_nseg, s_last;
  __shared__ union {
    FanSeg f[kSegs];
    NodeSeg n[kSegs];
  } s_seg;
  const int lane = threadIdx.x & 31;
  const int64_t units = unit_off[n];
  // a warp claims kUC consecutive units at a time: one atomic per chunk and a
  // plan lookup that mostly stays in the previous plan (measured: with one
  // unit per claim the counter and the lookups were the top stalls of a
  // 1,000-plan batch). Node rows (form 4's only units) are short; priced
  // pairs keep one unit per claim for balance.
  // Form 5's first launch has nothing else to wait for: its warps stride over
  // the chunks statically (chunk c, c + warps, ...), no counter at all.
  // (measured on cfg5: static chunks of 2 or 4 units are equal; the
  // counter-claimed chunks of the other forms are far slower here)
  constexpr int kUC = kForm == 4 ? 8 : (kForm == 5 ? kUC5 : 1);
  const int64_t chunks = (units + kUC - 1) / kUC;
  if (threadIdx.x == 0) s_unit = blockIdx.x * (kFusedThreads / 32);  // static first chunks, as fused_kernel
  __syncthreads();
  int64_t c = (int64_t)s_unit + (threadIdx.x >> 5);
  int p = -1;
  if constexpr (kForm == 5 && (kPhase & 1) != 0) {
    for (; c < chunks; c += (int64_t)gridDim.x * (kFusedThreads / 32)) {
      const int64_t u1 = min(units, (c + 1) * kUC);
      // the plan of the chunk's first unit from the host's table (a warp's
      // chunks are a grid of warps apart: a search per chunk otherwise)
      if (chunk_plan) p = chunk_plan[c];
      for (int64_t u = c * kUC; u < u1; ++u) {
        if (chunk_plan) {
          while (unit_off[p + 1] <= u) ++p;  // (a chunk may end in a later plan)
        } else {
          p = find_plan(unit_off, n, u, p);
        }
        run_unit<false, false, true>(args[p], u - unit_off[p], args[p].bw_tab);
      }
    }
  } else if constexpr ((kPhase & 1) != 0) while (c < chunks) {
    const int64_t u1 = min(units, (c + 1) * kUC);
    for (int64_t u = c * kUC; u < u1; ++u) {
      p = find_plan(unit_off, n, u, p);
      const FusedArgs& a = args[p];
      if (kForm == 1 || (kForm == 0 && a.warp_form)) run_unit<true>(a, u - unit_off[p], a.bw_tab);
      else if (kForm == 4) run_unit<true>(a, u - unit_off[p], a.bw_tab);  // node rows only (a.direct)
      else run_unit<false>(a, u - unit_off[p], a.bw_tab, args);
    }
    int next = 0;
    if (lane == 0) {
      const int64_t base = (int64_t)gridDim.x * (kFusedThreads / 32);
      next = base + ld_relaxed(&hdr->unit_head.v) >= chunks ? INT_MAX : (int)(base + atomicAdd(&hdr->unit_head.v, 1));
    }
    c = __shfl_sync(0xffffffffu, next, 0);
  }
  if (kForm != 4 && kForm != 5) {  // every plan's other-parity tables start unset: one slice of the concatenation per CTA
    const int64_t total = tab_off[n];
    const int64_t per = (total + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = (int64_t)blockIdx.x * per, b1 = min(b0 + per, total);
    int q = -1;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += kFusedThreads) {
      q = find_plan(tab_off, n, i, q);
      args[q].next_tables[i - tab_off[q]] = __longlong_as_double((long long)kUnset);
    }
  }
  const int64_t items = item_off[n];
  int ip = -1;
  if constexpr ((kPhase & 2) != 0) for (int64_t item = blockIdx.x;; item += gridDim.x) {
    __syncthreads();  // s_seg reuse
    if (item >= items) break;
    ip = find_plan(item_off, n, item, ip);
    const FusedArgs& a = args[ip];
    const int li = (int)(item - item_off[ip]);
    if (li < a.i_exp) node_range<kPhase == 3>(a, li, s_seg.n, &s_nseg, &s_edge);
    else if (kForm == 4) fanout_range<true>(a, li - a.i_exp, s_seg.f, &s_nseg, &s_edge);
    else if (kForm == 5) fanout_range<false, false, TP_BATCH_FAN_PER, true>(a, li - a.i_exp, s_seg.f, &s_nseg, &s_edge);
    else fanout_range<false>(a, li - a.i_exp, s_seg.f, &s_nseg, &s_edge);
  }
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&hdr->exit_count.v, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {  // every other CTA has finished: reset every plan and the batch queue
    __threadfence();
    for (int q = threadIdx.x; (kPhase & 2) && q < n; q += kFusedThreads) {
      if (err_out) err_out[q] = *args[q].err;  // this launch's error slot of every plan
      reset_plan(args[q]);
    }
    if (threadIdx.x == 0) {
      hdr->unit_head.v = 0;
      hdr->exit_count.v = 0;
    }
    __threadfence();
  }
}

// price_assignment (aux_graph.hpp:326-348) of K strategy assignments, one
// warp per assignment: lanes gather a chunk of 32 summation terms (node or
// edge payloads at the assignment's aux ids) into shared memory, lane 0 adds
// them in the reference's order (topological order; a source's virtual edge,
// then its in-edges ascending), so both cost modes and the memory sum are the
// reference's own roundings.
constexpr int kPriceWarps = 4;
__global__ void __launch_bounds__(32 * kPriceWarps) price_kernel(
    const int4* __restrict__ terms, int nterms, const int64_t* __restrict__ node_base,
    const int64_t* __restrict__ edge_base, const int32_t* __restrict__ edge_to_op, const int32_t* __restrict__ asg,
    int nops, int k, const double* __restrict__ n_sec, const double* __restrict__ n_vol,
    const double* __restrict__ n_mem, const double* __restrict__ e_sec, const double* __restrict__ e_vol,
    const double* __restrict__ e_mem, double* __restrict__ o_sec, double* __restrict__ o_vol,
    double* __restrict__ o_mem) {
  __shared__ double sv[kPriceWarps][3][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a = blockIdx.x * kPriceWarps + w;
  if (a >= k) return;
  const int32_t* as = asg + (int64_t)a * nops;
  double c = 0, v = 0, m = 0;
  for (int t0 = 0; t0 < nterms; t0 += 32) {
    const int t = t0 + lane;
    if (t < nterms) {
      const int4 tm = terms[t];
      double x, y, z;
      if (tm.x == 0) {
        const int64_t id = node_base[tm.w] + as[tm.w];
        x = n_sec[id];
        y = n_vol[id];
        z = n_mem[id];
      } else {
        const int wo = edge_to_op[tm.y];
        const int64_t id =
            edge_base[tm.y] + (int64_t)as[tm.z] * (node_base[wo + 1] - node_base[wo]) + as[tm.w];
        x = e_sec[id];
        y = e_vol[id];
        z = e_mem[id];
      }
      sv[w][0][lane] = x;
      sv[w][1][lane] = y;
      sv[w][2][lane] = z;
    }
    __syncwarp();
    if (lane == 0) {
      const int cnt = min(32, nterms - t0);
      for (int i = 0; i < cnt; ++i) {
        c += sv[w][0][i];
        v += sv[w][1][i];
        m += sv[w][2][i];
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    if (o_sec) o_sec[a] = c;
    if (o_vol) o_vol[a] = v;
    if (o_mem) o_mem[a] = m;
  }
}

// K3 (optional): cond_min (solver.hpp:239-253), warp per (edge, su) row.
__global__ void rowmin_kernel(const EdgeDesc* __restrict__ edges, const int64_t* __restrict__ row_base,
                              int e0, int nedges, int64_t nrows, const SigDesc* __restrict__ sigs,
                              const int32_t* __restrict__ maps,
                              const double2* __restrict__ r_tab, const double2* __restrict__ cls_sv,
                              double* __restrict__ out_c, double* __restrict__ out_v) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= nrows) return;
  int lo = 0, hi = nedges - 1;  // row_base is relative to edge e0
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (row_base[mid] <= row) lo = mid; else hi = mid - 1;
  }
  const EdgeDesc ed = edges[e0 + lo];
  const SigDesc& sg = sigs[ed.sig];
  const int64_t su = row - row_base[lo];
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  double mc = inf, mv = inf;
  const int64_t rbase = sg.pair_begin + (int64_t)maps[sg.uid_u + su] * sg.Wn;
  for (int64_t sw = lane; sw < sg.Sw; sw += 32) {
    const int64_t j = rbase + maps[sg.uid_w + sw];
    const double2 cv = cls_sv[ed.wrow + sw], rv = r_tab[j];
    const double c = cv.x + rv.x * sg.scale;
    const double v = cv.y + rv.y * sg.scale;
    mc = c < mc ? c : mc;
    mv = v < mv ? v : mv;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double oc = __shfl_xor_sync(0xffffffffu, mc, off);
    const double ov = __shfl_xor_sync(0xffffffffu, mv, off);
    mc = oc < mc ? oc : mc;
    mv = ov < mv ? ov : mv;
  }
  if (lane == 0) {
    out_c[row] = mc;
    out_v[row] = mv;
  }
}

// K4 (optional): pair_min (solver.hpp:254-255), warp per edge over the row
// minima written by K3. min is exact, so the lane order cannot change a bit;
// the select keeps std::min's "first wins on ties / NaN" form.
__global__ void pairmin_kernel(const int64_t* __restrict__ row_base, int64_t nedges,
                               const double* __restrict__ row_c, const double* __restrict__ row_v,
                               double* __restrict__ out_c, double* __restrict__ out_v) {
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (e >= nedges) return;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  double mc = inf, mv = inf;
  for (int64_t r = row_base[e] + lane; r < row_base[e + 1]; r += 32) {
    const double c = row_c[r], v = row_v[r];
    mc = c < mc ? c : mc;
    mv = v < mv ? v : mv;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double oc = __shfl_xor_sync(0xffffffffu, mc, off);
    const double ov = __shfl_xor_sync(0xffffffffu, mv, off);
    mc = oc < mc ? oc : mc;
    mv = ov < mv ? ov : mv;
  }
  if (lane == 0) {
    out_c[e] = mc;
    out_v[e] = mv;
  }
}

// Verification export through the kernels' pair paths: thread form...
__global__ void query_kernel(const tpk::QueryPOD* __restrict__ q, int n, tp_redist_result* __restrict__ r,
                             const double* __restrict__ tabs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* t = tabs + (int64_t)i * (tpk::kBwTab + tpk::kScaleDim * tpk::kScaleDim);
  tp_redist_result res;
  res.status = tpk::run_query_fast(q[i], res, tpk::FastTabs{t, t + tpk::kBwTab});
  r[i] = res;
}

// ... and warp form (one warp per query).
__global__ void query_kernel_warp(const tpk::QueryPOD* __restrict__ q, int n, tp_redist_result* __restrict__ r,
                                  tpk::Trace* __restrict__ traces, const double* __restrict__ tabs) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  const double* t = tabs + (int64_t)i * (tpk::kBwTab + tpk::kScaleDim * tpk::kScaleDim);
  const int st = tpk::run_query_warp(q[i], r[i], traces[i], tpk::PriceTabs{t, t + tpk::kBwTab});
  if ((threadIdx.x & 31) == 0) r[i].status = st;
}

}  // namespace
