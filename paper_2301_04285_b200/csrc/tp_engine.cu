// tp_engine.cu — B200 (sm_100a) cost-tensor engine behind include/taps_b200.h.
//
// Replaces topoplan::build_auxiliary_graph (aux_graph.hpp:211-315).
//
// Host analysis (tp_plan_create) groups the work into classes:
//   * node classes — operators whose slicing, tensor shapes, element sizes,
//     fed inputs and in-degree agree have identical per-strategy costs
//     (aux_graph.hpp:120-167); each class is priced once per strategy;
//   * edge classes — graph edges whose (shape, tensor bytes, producer and
//     consumer slicing, axis counts) agree have identical |Su| x |Sw|
//     redistribution tables; each class is priced once per pair (the
//     reference's memo, aux_graph.hpp:257-271, made static).
// Device pipeline of one build: ONE persistent launch (fused_kernel) whose
// CTAs pull work items from an atomic queue:
//   node rows      one thread per (node class, strategy): intra-operator
//                  AllReduce cost/volume and memory (aux_graph.hpp:120-167)
//   class pairs    one warp (or thread) per (edge class, su, sw): unify +
//                  sequence inference + topology-aware pricing (tp_warp.cuh /
//                  tp_fast.cuh)
//   fan-out tiles  the write-bound part: every aux edge gets
//                  cost = intra(w) + redist, volume likewise, memory =
//                  mem(w) / in_degree(w), lane-contiguous fp64 stores; a tile
//                  waits only for its own edge class's pairs
//   node fan-out   class rows to every member operator's aux nodes
// rowmin_kernel (optional, second launch): warp per (edge, su) row, lanes
// over sw, shuffle min — the solver's cond_min (solver.hpp:239-253).
// The strategy tables (layout.hpp:270-328) are built once per plan by
// table_kernel at upload and cached per device.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <climits>
#include <cmath>
#include <array>
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>
#include <atomic>
#include <mutex>
#include <thread>

#include "../../include/taps_b200.h"
#include "tp_core.cuh"
#include "tp_fast.cuh"
#include "tp_warp.cuh"

using tpk::DimT;
using tpk::Env;
using tpk::Lay;
using tpk::Strat;

namespace {

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
// POD thread-locals only (a non-trivial thread_local in a dlopen'ed library
// is fragile when other runtimes were loaded first).
thread_local char g_err[512];
thread_local int g_err_kind = 0;

tp_status set_err(tp_status st, int kind, const std::string& msg) {
  std::strncpy(g_err, msg.c_str(), sizeof(g_err) - 1);
  g_err[sizeof(g_err) - 1] = 0;
  g_err_kind = kind;
  return st;
}

tp_status status_of_kind(int kind) {
  if (kind == tpk::kOk) return TP_OK;
  if (kind == tpk::kEdgeTensorMissing) return TP_ERR_OUT_OF_RANGE;
  if (kind == tpk::kCapacity) return TP_ERR_CAPACITY;
  return TP_ERR_TOPOPLAN;
}

const char* kind_text(int kind) {
  switch (kind) {
    case tpk::kCycle: return "build_auxiliary_graph: graph has a cycle";
    case tpk::kDangling: return "auxiliary graph: dangling edge";
    case tpk::kNotPow2: return "enumerate_strategies: device count must be a power of two";
    case tpk::kNoAxes: return "enumerate_strategies: operator has no axes";
    case tpk::kUnknownSliceTensor: return "axis references unknown tensor";
    case tpk::kIndivisible: return "extent is not divisible by the axis degree";
    case tpk::kShapeMismatch: return "unify_layouts: layouts describe different tensor shapes";
    case tpk::kNotUnifiable: return "device matrices are not unifiable";
    case tpk::kFactorization: return "extent not divisible during device-matrix factorization";
    case tpk::kRefine: return "tensor extent not divisible during shape unification";
    case tpk::kDeviceSplit: return "tensor extent not divisible during device split";
    case tpk::kNoConverge: return "unify_layouts failed to converge";
    case tpk::kRefineMismatch: return "unify_layouts: internal refinement mismatch";
    case tpk::kDeadlock: return "redistribution deadlock: no gatherable axis";
    case tpk::kNoTerminate: return "redistribution failed to terminate";
    case tpk::kEdgeTensorMissing: return "map::at (edge tensor absent from an endpoint)";
    case tpk::kCapacity: return "input exceeds a fixed engine bound";
    default: return "error";
  }
}

#define CUDA_TRY(expr)                                                                       \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess)                                                                   \
      return set_err(TP_ERR_CUDA, 0, std::string(#expr ": ") + cudaGetErrorString(_e));      \
  } while (0)

// Error keys: (order << 6) | kind; the smallest key is the error the
// reference would throw first (its iteration order). Node phase orders are
// 1 + 2*node (+1 for derivation errors), edge phase orders start at 2^46.
constexpr uint64_t kEdgePhase = 1ull << 46;
__host__ __device__ inline uint64_t ekey(uint64_t order, int kind) { return (order << 6) | (uint64_t)kind; }

// ---------------------------------------------------------------------------
// device descriptors
// ---------------------------------------------------------------------------
struct SliceChk {
  int16_t slot;  // -1: the slice names a tensor the op does not carry
  int8_t axis;
  int8_t v;      // 2-adic valuation of the sliced extent (capped at 63)
};

struct SlotDesc {
  int64_t elements;
  int32_t es;
  int8_t R;
  int8_t sa[tpk::kMaxR];
  int8_t pad[3];
};

struct Occ {
  int16_t slot;
  uint8_t nonslicing;  // axes with no slice naming this tensor
  uint8_t in_memory;   // output, or input not fed by an edge
};

struct ClassDesc {     // a node class
  int64_t row_base;    // first row of the class in the class row tables
  int64_t first_node;  // aux node id of strategy 0 of the class's first member
  double indeg;        // in-degree shared by the members (memory / in_degree)
  int32_t p, table;
  int32_t chk_begin, chk_end, occ_begin, occ_end, slot_begin, mem_begin, mem_end, S;
};

struct SigDesc {       // an edge class
  int64_t pair_begin;  // its table (a derived class: the base class's table)
  int64_t first_aux;   // aux id of (su=0, sw=0) of the class's first edge
  double bytes;
  double scale;        // derived class: exact power-of-two factor on the base table
  int32_t R, Su, Sw, tab_u, tab_w, has_override;
  int32_t side_u, side_w;  // first producer / consumer SideDesc of the class
  int32_t base;        // class whose pairs are computed (itself unless derived)
  // distinct producer / consumer layouts: the class table is Un x Wn; maps
  // (offsets into FusedArgs::maps) take a strategy to its distinct layout
  // (uid_*, [S*]) and a distinct layout to its first strategy (rep_*, [*n])
  int32_t Un, Wn, uid_u, uid_w, rep_u, rep_w;
  int32_t ident;       // the maps are identities (every strategy a distinct layout)
  int32_t pad2;
  int8_t sa_u[tpk::kMaxR];
  int8_t sa_w[tpk::kMaxR];
  DimT dt[tpk::kMaxR];
};

// Everything the fan-out reads about one graph edge (host-built at plan
// creation, one load per lane when a range stages its edges).
struct FanSeg {
  int64_t begin, end;  // aux ids of the edge
  int64_t pb, wrow;    // its class table, consumer class row of sw = 0
  int64_t nb_u, nb_w;  // records only
  double f;            // exact factor of a derived class
  int32_t e, Sw, Wn, uid_u, uid_w, ident;
  int32_t st_q, st_r;  // a thread's stride (kFusedThreads ids) in (su, sw)
  int32_t base, need;  // table owner and its entry count (pairs_done target)
};

struct EdgeDesc {
  int64_t aux_base;    // aux id of the edge's (0, 0)
  int64_t nb_u, nb_w;  // first aux node of the producer / consumer
  int64_t wrow;        // class row of the consumer's strategy 0
  int32_t sig, e;
};



struct TableDesc {
  int64_t offset, count;
  int32_t p, n;
};

struct SideJob {       // the SideDescs of one (edge class, side)
  int64_t out;         // first SideDesc
  int32_t tab, count;  // strategy table offset, strategies
  int8_t sa[tpk::kMaxR];
  int32_t R, pad;
};

// Below this many class pairs the GPU cannot be filled with one thread per
// pair (latency-bound), so a warp cooperates on each pair; above it the
// register-resident thread form has ~6x fewer instructions per pair.
constexpr int64_t kWarpPairLimit = 16384;
#ifndef TP_FAN_PER
#define TP_FAN_PER 1
#endif
constexpr int kFanPer = TP_FAN_PER;  // output positions a fan-out thread has in flight

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

__device__ __forceinline__ void pair_rec_one(const SigDesc* __restrict__ sigs, const int32_t* __restrict__ pair_sig,
                                             const int32_t* __restrict__ maps, const tpk::SideDesc* __restrict__ sides,
                                             const double* __restrict__ overrides, int64_t idx,
                                             PairRec* __restrict__ out) {
  const int sig = pair_sig[idx];
  const SigDesc& sg = sigs[sig];
  const int32_t t = (int32_t)(idx - sg.pair_begin);
  const int32_t ui = t / sg.Wn, wi = t - ui * sg.Wn;
  const int32_t su = maps[sg.rep_u + ui], sw = maps[sg.rep_w + wi];
  PairRec r;
  r.F = sides[sg.side_u + su];
  r.T = sides[sg.side_w + sw];
  r.bytes = sg.has_override ? overrides[idx] : sg.bytes;
  r.sig = sig;
  r.local = su * sg.Sw + sw;
  r.R = sg.R;
  r.pad = 0;
  for (int d = 0; d < tpk::kMaxR; ++d) r.dt[d] = sg.dt[d];
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
__device__ __forceinline__ void stamp(Sched* s, int k, bool is_min) {
  if (!s->timeline) return;
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
    if (q < cd.occ_end) {
      const Occ oc = a.occs[q];
      const SlotDesc& sd = a.slots[cd.slot_begin + oc.slot];
      int sdiv = 0;
      for (int d = 0; d < sd.R; ++d)
        if (sd.sa[d] >= 0) sdiv += st.deg[sd.sa[d]];
      const int64_t shard_el = sdiv >= 63 ? 0 : (sd.elements >> sdiv);
      const double sb = (double)shard_el * sd.es;  // layout.hpp:125-129
      has_m = oc.in_memory;                        // aux_graph.hpp:151-167
      tm = sb;
      int glog = 0;
      for (int ax = 0; ax < cd.p; ++ax)
        if ((oc.nonslicing >> ax) & 1) glog += st.deg[ax];
      if (glog > 0) {  // group > 1
        // infer_ct_allreduce (cost_model.hpp:75-97)
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
  tpk::MultiSec ms;
  ms.g = g;
  for (int q = 1; q < g; ++q) {
    const FusedArgs& b = all[a.group[q]];
    ms.env[q] = b.env;
    ms.tab[q] = tpk::FastTabs{b.bw_tab, b.bw_tab + tpk::kBwTab};
    ms.sec[q] = 0;
  }
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
      for (int q = 1; q < g; ++q) ms.sec[q] = 0;
    }
  }
  a.r_tab[idx] = make_double2(sec, vol);
  for (int q = 1; q < g; ++q) all[a.group[q]].r_tab[idx] = make_double2(ms.sec[q], vol);
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

__device__ void fanout_range(const FusedArgs& a, int item, FanSeg* seg, int* s_n, int* s_edge) {
  const unsigned long long t0 = a.fan_ns ? gtimer() : 0;
  const int64_t start = a.A0 + (int64_t)item * a.range_len;
  const int64_t end = min(start + a.range_len, a.A1);
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) *s_edge = a.range_first[item];  // host-computed
  int64_t pos = start;
  bool first = true;
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
        wait_relaxed(&a.sched->pairs_done[g.base].v, g.need);
        seg[lane] = g;
      }
      const int n = __popc(__ballot_sync(0xffffffffu, in));  // a prefix of the lanes
      if (first) {
        if (lane == 0) wait_at_least(&a.sched->node_done.v, (int)a.total_rows);
        __syncwarp();
      }
      if (lane == 0) {
        *s_n = n;
        *s_edge += n;
        if (first) {
          stamp(a.sched, 4, true);
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
    // (su, sw) of a thread's ids advance by a fixed stride within an edge;
    // a division only where the thread enters an edge
    int si = -1;
    int32_t su = 0, sw = 0;
    for (int64_t o0 = pos + threadIdx.x; o0 < span_end; o0 += kFusedThreads * kFanPer) {
      double cs[kFanPer], vs[kFanPer], ms[kFanPer];
      int64_t q[kFanPer];
#pragma unroll
      for (int k = 0; k < kFanPer; ++k) {
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
        const double2 rv = table_load2(a.r_tab + r);
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
      for (int k = 0; k < kFanPer; ++k) {
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

__device__ void node_range(const FusedArgs& a, int item, NodeSeg* seg, int* s_n, int* s_op) {
  const int64_t start = (int64_t)item * a.node_range_len;
  const int64_t end = min(start + a.node_range_len, a.num_nodes);
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    *s_op = a.nrange_first[item];  // host-computed
    wait_at_least(&a.sched->node_done.v, (int)a.total_rows);
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
template <bool kWarpForm>
__device__ __forceinline__ void run_unit(const FusedArgs& a, int64_t u, const double* price,
                                         const FusedArgs* all = nullptr) {
  const int lane = threadIdx.x & 31;
  const unsigned long long t0 = (a.pair_ns || a.item_ns) ? gtimer() : 0;
  if (u < a.total_rows) {
    node_row(a, u);
    if (lane == 0) {
      red_release_add(&a.sched->node_done.v, 1);  // rows: off the critical path, released
      if (a.item_ns) {
        a.item_ns[2 * u] = (unsigned)t0;
        a.item_ns[2 * u + 1] = (unsigned)(gtimer() - t0);
      }
    }
  } else if (kWarpForm) {
    const int64_t idx = u - a.total_rows;
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
    const int64_t idx = (u - a.total_rows) * 32 + lane;
    const bool valid = idx < a.total_pairs;
    const int sig = valid ? sig_of_pair(a, idx) : -1;
    const bool grouped = all && a.group_n > 1;
    if (valid) pair_thread(a, idx, price, all);
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
  if (a.priced_by_leader) return a.total_rows;
  return a.total_rows + (a.warp_form ? a.total_pairs : (a.total_pairs + 31) / 32);
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
  __shared__ double s_price[tpk::kBwTab + tpk::kScaleDim * tpk::kScaleDim];  // the pricing tables
  const int lane = threadIdx.x & 31;
  const int64_t units = plan_units(a);
  if (threadIdx.x == 0) {
    stamp(a.sched, 0, true);
    // first units by CTA index: no start-up burst of atomics on one counter
    // (measured: units start ~0.6 us earlier, the build ~2 us shorter)
    s_unit = blockIdx.x * (kFusedThreads / 32);
  }
  if (a.total_pairs > 0)
    for (int i = threadIdx.x; i < tpk::kBwTab + tpk::kScaleDim * tpk::kScaleDim; i += kFusedThreads)
      s_price[i] = a.bw_tab[i];  // bw_tab and scale_tab are one array
  __syncthreads();
  // phase 1: node-class rows, then class pairs
  int64_t u = (int64_t)s_unit + (threadIdx.x >> 5);
  while (u < units) {
    run_unit<kWarpForm>(a, u, s_price);
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
        stamp(a.sched, 5, false);
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
    else fanout_range(a, item - a.i_exp, s_seg.f, &s_nseg, &s_edge);
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
// state without spills)
template <int kForm>
__global__ void __launch_bounds__(kFusedThreads, kForm == 3 ? 2 : 4)
    fused_batch_kernel(const FusedArgs* __restrict__ args, int n, const int64_t* __restrict__ unit_off,
                       const int64_t* __restrict__ item_off, const int64_t* __restrict__ tab_off, BatchHdr* hdr,
                       unsigned long long* __restrict__ err_out) {
  __shared__ int s_unit, s_edge, s_nseg, s_last;
  __shared__ union {
    FanSeg f[kSegs];
    NodeSeg n[kSegs];
  } s_seg;
  const int lane = threadIdx.x & 31;
  const int64_t units = unit_off[n];
  if (threadIdx.x == 0) s_unit = blockIdx.x * (kFusedThreads / 32);  // static first units, as fused_kernel
  __syncthreads();
  int64_t u = (int64_t)s_unit + (threadIdx.x >> 5);
  int p = -1;
  while (u < units) {
    p = find_plan(unit_off, n, u, p);
    const FusedArgs& a = args[p];
    if (kForm == 1 || (kForm == 0 && a.warp_form)) run_unit<true>(a, u - unit_off[p], a.bw_tab);
    else run_unit<false>(a, u - unit_off[p], a.bw_tab, args);
    int next = 0;
    if (lane == 0) {
      const int64_t base = (int64_t)gridDim.x * (kFusedThreads / 32);
      next = base + ld_relaxed(&hdr->unit_head.v) >= units ? INT_MAX : (int)(base + atomicAdd(&hdr->unit_head.v, 1));
    }
    u = __shfl_sync(0xffffffffu, next, 0);
  }
  {  // every plan's other-parity tables start unset: one slice of the concatenation per CTA
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
  for (int64_t item = blockIdx.x;; item += gridDim.x) {
    __syncthreads();  // s_seg reuse
    if (item >= items) break;
    ip = find_plan(item_off, n, item, ip);
    const FusedArgs& a = args[ip];
    const int li = (int)(item - item_off[ip]);
    if (li < a.i_exp) node_range(a, li, s_seg.n, &s_nseg, &s_edge);
    else fanout_range(a, li - a.i_exp, s_seg.f, &s_nseg, &s_edge);
  }
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&hdr->exit_count.v, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {  // every other CTA has finished: reset every plan and the batch queue
    __threadfence();
    for (int q = threadIdx.x; q < n; q += kFusedThreads) {
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

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  bool view = false;  // points into another buffer (the descriptor pack)
  void set_view(void* at, size_t bytes) {
    release();
    p = at;
    cap = bytes;
    view = true;
  }
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p && !view) cudaFree(p);
    p = nullptr;
    cap = 0;
    view = false;
    size_t want = bytes < 256 ? 256 : bytes;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p && !view) cudaFree(p);
    p = nullptr;
    cap = 0;
    view = false;
  }
};

// The plan's descriptor arrays go up in ONE copy: packed (256-B aligned) into
// pinned staging memory, copied into one device buffer, each DevBuf a view.
struct DescPack {
  struct Piece {
    DevBuf* buf;
    const void* src;
    size_t bytes;
  };
  std::vector<Piece> pieces;
  template <typename T>
  void add(DevBuf& b, const std::vector<T>& v) { pieces.push_back({&b, v.data(), v.size() * sizeof(T)}); }
  static size_t pad(size_t n) { return (n + 16 + 255) & ~(size_t)255; }
  size_t total() const {
    size_t t = 0;
    for (auto& x : pieces) t += pad(x.bytes);
    return t;
  }
};

template <typename T>
cudaError_t upload(DevBuf& b, const std::vector<T>& v, cudaStream_t s) {
  cudaError_t e = b.ensure(v.size() * sizeof(T) + 16);
  if (e != cudaSuccess || v.empty()) return e;
  return cudaMemcpyAsync(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s);
}

int log2_floor(int64_t v) {
  int e = 0;
  while (((int64_t)1 << (e + 1)) <= v) ++e;
  return e;
}

int v2_capped(int64_t v) {
  return v == 0 ? 63 : std::min(63, __builtin_ctzll((unsigned long long)v));
}

}  // namespace

// ---------------------------------------------------------------------------
// the plan
// ---------------------------------------------------------------------------
// Device memory and stream of a plan. User-created plans own one; the
// one-shot tp_build_cost_tensors reuses a per-thread, per-device arena so
// repeated builds pay neither cudaMalloc nor the strategy-table kernel.
struct Arena {
  int device = 0;
  cudaStream_t stream = nullptr;
  DevBuf d_tabs, d_tables, d_classes, d_chks, d_slots, d_occs, d_members, d_sigs, d_edges,
      d_over, d_tables2, d_opnode, d_oprow, d_rowbase, d_sched, d_sidejobs,
      d_sides, d_price, d_pairsigs, d_trace, d_maps, d_rowcls, d_pairrec, d_prof, d_fsegs, d_rfirst;
  DevBuf out[9];  // one-shot staging of the requested outputs
  DevBuf d_desc;  // the descriptor pack
  void* h_stage = nullptr;  // pinned staging of the pack
  size_t h_stage_cap = 0;
  cudaEvent_t stage_done = nullptr;  // the last pack copy out of h_stage
  bool sched_clean = false;  // Sched zero (set up, or left so by the last launch)
  int64_t tables_L = -1;     // table layout (doubles per parity) the clean state is for
  size_t sched_bytes = 0;
  bool timeline_set = false;
  int parity = 0;
  std::vector<std::array<int64_t, 4>> table_key;  // (offset, count, p, n) of the resident tables
  void release() {
    for (DevBuf* b : {&d_tabs, &d_tables, &d_classes, &d_chks, &d_slots, &d_occs, &d_members, &d_sigs,
                      &d_edges, &d_over, &d_tables2, &d_opnode, &d_oprow, &d_rowbase, &d_sched, &d_sidejobs, &d_sides, &d_price, &d_pairsigs, &d_trace, &d_maps, &d_rowcls, &d_pairrec, &d_prof, &d_fsegs, &d_rfirst})
      b->release();
    for (auto& b : out) b.release();
    d_desc.release();
    if (h_stage) cudaFreeHost(h_stage);
    h_stage = nullptr;
    h_stage_cap = 0;
    if (stage_done) cudaEventDestroy(stage_done);
    stage_done = nullptr;
    table_key.clear();
    if (stream) cudaStreamDestroy(stream);
    stream = nullptr;
  }
};

struct tp_plan {
  int device = 0;
  Arena* arena = nullptr;
  bool owns_arena = true;
  int32_t num_ops = 0, num_edges = 0;
  int64_t N = 1;
  int n_log2 = 0;
  Env env{};
  std::vector<int64_t> node_base;  // [num_ops + 1]
  std::vector<int64_t> edge_base;  // [num_edges + 1]
  std::vector<int64_t> row_base;   // [num_edges + 1]
  std::vector<int32_t> edge_from_op, edge_to_op, in_deg, out_deg, topo;
  // price_assignment's summation terms (aux_graph.hpp:326-348), host-built on
  // first use: per op in topological order a source's virtual edge, then the
  // edges whose `to` id equals the op's id, ascending
  std::vector<int32_t> op_dense_id, edge_to_dense;
  std::vector<int4> price_terms;  // (kind 0 node / 1 edge, e, u, op)
  DevBuf* d_terms = nullptr;      // their device copy (owned)
  int64_t terms_bytes = 0;
  int64_t num_aux_nodes = 0, num_aux_edges = 0, num_rows = 0, num_virtual = 0;
  int valid_ops = 0;    // ops whose nodes are built (before a host node-phase error)
  int valid_edges = 0;  // edges processed before a host edge-phase error
  uint64_t host_err = ~0ull;
  // device descriptors (host copies)
  std::vector<TableDesc> tabs;
  int64_t table_total = 0;
  std::vector<ClassDesc> classes;
  std::vector<int64_t> members;  // member node bases, CSR by class
  int64_t total_rows = 0;
  std::vector<SliceChk> chks;
  std::vector<SlotDesc> slots;
  std::vector<Occ> occs;
  std::vector<SigDesc> sigs;
  std::vector<EdgeDesc> edges;
  std::vector<int32_t> sig_edges;  // edges grouped by class, edge order within
  std::vector<int32_t> sig_edge_begin;
  std::vector<double> overrides;   // per pair; empty if no class needs one
  std::vector<int32_t> pair_sig;   // edge class of every table entry
  std::vector<int32_t> row_cls;    // node class of every class row
  std::vector<int32_t> maps;       // SigDesc uid_* / rep_* arrays
  std::vector<FanSeg> fsegs;       // per valid graph edge
  std::vector<int32_t> range_first;   // per execute: first edge of every edge range,
  std::array<int64_t, 4> range_key{{-1, -1, -1, -1}};  // then first op of every node range
  int64_t total_pairs = 0;
  int64_t h2d_bytes = 0;
  bool uploaded = false;
  std::vector<int64_t> op_row;  // class row of strategy 0 per operator
  std::vector<SideJob> side_jobs;
  int64_t side_total = 0;
  int64_t last_launches = 0;
  cudaStream_t last_stream = nullptr;
  cudaEvent_t prof_start = nullptr, prof_stop = nullptr;  // recorded around K2
  bool timeline = false;
  int last_parity = -1;  // error slot of the last launch (-1: none)
  int64_t last_grid = 0;
  int64_t trace_n[3] = {0, 0, 0};  // pairs, node-row items, fan-out items traced
  int pair_form = 0;  // 0 = by size, 1 = warp per pair, 2 = thread per pair
  bool in_big_batch = false;  // by size: judged by the whole batch's pairs (thread form)
  uint64_t shash = 0;         // struct_hash, cached (a plan's structure never changes)
  bool shash_ok = false;
  int resident_blocks = 0;  // persistent grid size (SMs x resident CTAs)
};

namespace {

// hash of a POD byte range, 8 bytes at a time (host class dedup)
inline uint64_t hash_words(uint64_t h, const void* data, size_t bytes) {
  const unsigned char* b = (const unsigned char*)data;
  size_t i = 0;
  for (; i + 8 <= bytes; i += 8) {
    uint64_t w;
    std::memcpy(&w, b + i, 8);
    h = (h ^ w) * 0x100000001b3ull;
    h ^= h >> 29;
  }
  if (i < bytes) {
    uint64_t w = 0;
    std::memcpy(&w, b + i, bytes - i);
    h = (h ^ w) * 0x100000001b3ull;
    h ^= h >> 29;
  }
  return h ^ (bytes << 7);
}

#ifdef TP_HOST_PROF
double g_hprof[8];
std::chrono::steady_clock::time_point g_hlast;
#define HPROF(k)                                                                                  \
  do {                                                                                            \
    auto now_ = std::chrono::steady_clock::now();                                                 \
    if (k) g_hprof[k] += std::chrono::duration<double, std::micro>(now_ - g_hlast).count();       \
    g_hlast = now_;                                                                               \
  } while (0)
#else
#define HPROF(k) \
  do {           \
  } while (0)
#endif

struct Builder {
  const tp_graph_desc* g;
  const tp_topology_desc* t;
  tp_plan* P;

  int num_tensors() const { return g->op_tensor_begin[g->num_ops]; }
  int rank_of(int tensor) const { return g->tensor_shape_begin[tensor + 1] - g->tensor_shape_begin[tensor]; }
  const int64_t* shape_of(int tensor) const { return g->shape + g->tensor_shape_begin[tensor]; }

  tp_status check_desc() {
    if (!g || !t) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null descriptor");
    if (g->num_ops < 0 || g->num_edges < 0) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "negative counts");
    if (g->num_ops > 0 && (!g->op_id || !g->op_tensor_begin || !g->op_num_inputs || !g->op_axis_begin))
      return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null operator arrays");
    if (g->num_edges > 0 && (!g->edge_from || !g->edge_to || !g->edge_tensor))
      return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null edge arrays");
    if (g->num_ops == 0) return TP_OK;
    if (g->op_tensor_begin[0] != 0 || g->op_axis_begin[0] != 0)
      return set_err(TP_ERR_INVALID_ARGUMENT, 0, "CSR offsets must start at 0");
    for (int i = 0; i < g->num_ops; ++i) {
      if (g->op_tensor_begin[i + 1] < g->op_tensor_begin[i] || g->op_axis_begin[i + 1] < g->op_axis_begin[i])
        return set_err(TP_ERR_INVALID_ARGUMENT, 0, "CSR offsets must be non-decreasing");
      const int nt = g->op_tensor_begin[i + 1] - g->op_tensor_begin[i];
      if (g->op_num_inputs[i] < 0 || g->op_num_inputs[i] > nt)
        return set_err(TP_ERR_INVALID_ARGUMENT, 0, "op_num_inputs out of range");
    }
    const int nt = num_tensors();
    const int na = g->op_axis_begin[g->num_ops];
    if (nt > 0 && (!g->tensor_name || !g->tensor_shape_begin || !g->tensor_element_size))
      return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null tensor arrays");
    if (na > 0 && !g->axis_slice_begin) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null axis arrays");
    if (nt > 0) {
      if (g->tensor_shape_begin[0] != 0) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "shape CSR must start at 0");
      for (int k = 0; k < nt; ++k)
        if (g->tensor_shape_begin[k + 1] < g->tensor_shape_begin[k])
          return set_err(TP_ERR_INVALID_ARGUMENT, 0, "shape CSR must be non-decreasing");
      if (g->tensor_shape_begin[nt] > 0 && !g->shape) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null shape");
    }
    if (na > 0) {
      if (g->axis_slice_begin[0] != 0) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "slice CSR must start at 0");
      for (int a = 0; a < na; ++a)
        if (g->axis_slice_begin[a + 1] < g->axis_slice_begin[a])
          return set_err(TP_ERR_INVALID_ARGUMENT, 0, "slice CSR must be non-decreasing");
      if (g->axis_slice_begin[na] > 0 && (!g->slice_tensor || !g->slice_dim))
        return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null slice arrays");
    }
    return TP_OK;
  }

  // Per-op slots: the reference keys an operator's layouts by tensor name,
  // the last occurrence's spec winning (layout.hpp:339-347).
  // Flat over all operators: op i owns slots [slot_begin[i], slot_begin[i + 1]).
  std::vector<int32_t> slot_begin, slot_name, slot_spec;
  std::vector<std::array<int8_t, tpk::kMaxR>> slot_sa;  // tensor dim -> slicing axis, per slot
  int find_slot(int op, int nm) const {  // local slot index of tensor name nm, or -1
    const int b = slot_begin[op], e = slot_begin[op + 1];
    for (int i = b; i < e; ++i)
      if (slot_name[i] == nm) return i - b;
    return -1;
  }
  int spec_of(int op, int k) const { return slot_spec[slot_begin[op] + k]; }
  const std::array<int8_t, tpk::kMaxR>& sa_of(int op, int k) const { return slot_sa[slot_begin[op] + k]; }
  std::map<int, int64_t> table_of_p;
  // node classes by key hash: first class with a hash, then a chain per class
  std::unordered_map<uint64_t, int32_t> class_head;
  std::vector<int32_t> class_next;
  std::vector<int32_t> class_nslot;
  // per-operator scratch, reused
  std::vector<SliceChk> chk;
  std::vector<SlotDesc> slots;
  std::vector<Occ> occ;
  std::vector<int64_t> key;
  std::vector<std::vector<int64_t>> class_members;
  // tensors fed by edges, CSR by dense op id (op_key[i] = dense id of op i)
  std::vector<int32_t> fed_begin, fed_list, op_key;
  std::vector<int64_t> wrow_of_op;

  tp_status run() {
    static const bool prof = getenv("TP_PROFILE_HOST") != nullptr;
    auto clk = [] { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
    double tc0 = prof ? clk() : 0;
    tp_status st = check_desc();
    double tc1 = prof ? clk() : 0;
    if (st) return st;
    tp_plan& p = *P;
    p.num_ops = g->num_ops;
    p.num_edges = g->num_edges;
    p.N = (int64_t)t->node_count * (int64_t)t->local_device_num;
    p.env = Env{t->intra_bandwidth, t->inter_bandwidth, (int64_t)t->local_device_num};

    // graph.hpp:135-154 find_op (first operator with the id), degrees by id.
    // Ids are made dense first: a direct table when they span a small range
    // (the usual case), a hash map otherwise.
    {
      int32_t lo = INT32_MAX, hi = INT32_MIN;
      auto span = [&](int32_t v) { lo = std::min(lo, v); hi = std::max(hi, v); };
      for (int i = 0; i < g->num_ops; ++i) span(g->op_id[i]);
      for (int e = 0; e < g->num_edges; ++e) span(g->edge_from[e]), span(g->edge_to[e]);
      const int64_t range = g->num_ops + g->num_edges == 0 ? 0 : (int64_t)hi - lo + 1;
      std::vector<int32_t> direct;
      std::unordered_map<int32_t, int32_t> hashed;
      const bool use_direct = range <= 4 * (int64_t)(g->num_ops + g->num_edges) + 1024;
      if (use_direct) direct.assign(range, -1);
      int32_t ndense = 0;
      auto dense = [&](int32_t id) -> int32_t {  // id -> dense index, allocated on first use
        if (use_direct) {
          int32_t& d = direct[id - lo];
          if (d < 0) d = ndense++;
          return d;
        }
        auto ins = hashed.emplace(id, ndense);
        if (ins.second) ++ndense;
        return ins.first->second;
      };
      std::vector<int32_t> op_dense(g->num_ops), from_dense(g->num_edges), to_dense(g->num_edges);
      for (int i = 0; i < g->num_ops; ++i) op_dense[i] = dense(g->op_id[i]);
      for (int e = 0; e < g->num_edges; ++e) from_dense[e] = dense(g->edge_from[e]), to_dense[e] = dense(g->edge_to[e]);
      std::vector<int32_t> first_op(ndense, -1), to_count(ndense, 0), from_count(ndense, 0);
      for (int i = g->num_ops - 1; i >= 0; --i) first_op[op_dense[i]] = i;
      fed_begin.assign(ndense + 1, 0);
      for (int e = 0; e < g->num_edges; ++e) {
        to_count[to_dense[e]]++;
        from_count[from_dense[e]]++;
      }
      for (int d = 0; d < ndense; ++d) fed_begin[d + 1] = fed_begin[d] + to_count[d];
      fed_list.assign(g->num_edges, 0);
      std::vector<int32_t> fill(fed_begin.begin(), fed_begin.end() - 1);
      for (int e = 0; e < g->num_edges; ++e) fed_list[fill[to_dense[e]]++] = g->edge_tensor[e];
      op_key.assign(op_dense.begin(), op_dense.end());
      p.op_dense_id = op_dense;
      p.edge_to_dense = to_dense;
      p.in_deg.resize(g->num_ops);
      p.out_deg.resize(g->num_ops);
      for (int i = 0; i < g->num_ops; ++i) {
        p.in_deg[i] = to_count[op_dense[i]];
        p.out_deg[i] = from_count[op_dense[i]];
      }
      p.edge_from_op.resize(g->num_edges);
      p.edge_to_op.resize(g->num_edges);
      for (int e = 0; e < g->num_edges; ++e) {
        p.edge_from_op[e] = first_op[from_dense[e]];
        p.edge_to_op[e] = first_op[to_dense[e]];
      }
    }
    p.node_base.assign(g->num_ops + 1, 0);
    p.edge_base.assign(g->num_edges + 1, 0);
    p.row_base.assign(g->num_edges + 1, 0);
    // Kahn's algorithm (graph.hpp:158-183)
    {
      std::vector<int32_t> indeg(g->num_ops, 0), sb(g->num_ops + 1, 0), succ(g->num_edges);
      for (int e = 0; e < g->num_edges; ++e) {  // successors, CSR in edge order
        const int u = p.edge_from_op[e], w = p.edge_to_op[e];
        if (u < 0 || w < 0) continue;
        ++sb[u + 1];
        ++indeg[w];
      }
      for (int i = 0; i < g->num_ops; ++i) sb[i + 1] += sb[i];
      {
        std::vector<int32_t> fill(sb.begin(), sb.end() - 1);
        for (int e = 0; e < g->num_edges; ++e) {
          const int u = p.edge_from_op[e], w = p.edge_to_op[e];
          if (u >= 0 && w >= 0) succ[fill[u]++] = w;
        }
      }
      p.topo.reserve(g->num_ops);
      for (int i = 0; i < g->num_ops; ++i)
        if (indeg[i] == 0) p.topo.push_back(i);
      for (size_t h = 0; h < p.topo.size(); ++h) {
        const int u = p.topo[h];
        for (int k = sb[u]; k < sb[u + 1]; ++k)
          if (--indeg[succ[k]] == 0) p.topo.push_back(succ[k]);
      }
      if ((int)p.topo.size() != g->num_ops) {  // aux_graph.hpp:224-226
        p.topo.assign(g->num_ops, 0);
        p.host_err = ekey(0, tpk::kCycle);
        p.valid_ops = 0;
        return TP_OK;
      }
    }

    double tc2 = prof ? clk() : 0;
    // ---------------- node phase (aux_graph.hpp:236-253) -----------------
    const bool pow2 = p.N > 0 && (p.N & (p.N - 1)) == 0;
    p.n_log2 = pow2 ? log2_floor(p.N) : 0;
    if (pow2 && p.n_log2 > tpk::kMaxD) return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "more than 2^16 devices");
    slot_begin.assign(g->num_ops + 1, 0);
    slot_name.clear();
    slot_spec.clear();
    slot_sa.clear();
    wrow_of_op.assign(g->num_ops, 0);
    p.op_row.assign(g->num_ops, 0);
    int64_t nodes = 0;
    p.valid_ops = g->num_ops;
    for (int i = 0; i < g->num_ops; ++i) {
      p.node_base[i] = nodes;
      const int np = g->op_axis_begin[i + 1] - g->op_axis_begin[i];
      int ek = 0;
      if (!pow2) ek = tpk::kNotPow2;
      else if (np < 1) ek = tpk::kNoAxes;
      if (ek) {
        p.host_err = ekey(1 + (uint64_t)nodes * 2, ek);
        p.valid_ops = i;
        break;
      }
      if (np > tpk::kMaxAxes) return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "operator with more than 8 axes");
      const int64_t S = tpk::strategy_count(np, p.n_log2);
      if (S > (1 << 20)) return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "more than 2^20 strategies per operator");
      if (!table_of_p.count(np)) {
        table_of_p[np] = p.table_total;
        p.tabs.push_back(TableDesc{p.table_total, S, np, p.n_log2});
        p.table_total += S;
      }
      st = build_op(i, np, S, nodes);
      if (st) return st;
      nodes += S;
    }
    for (int i = p.valid_ops; i <= g->num_ops; ++i) p.node_base[i] = nodes;
    for (int i = p.valid_ops; i <= g->num_ops; ++i) slot_begin[i] = (int32_t)slot_name.size();  // unbuilt: no slots
    p.num_aux_nodes = nodes;
    for (size_t c = 0; c < p.classes.size(); ++c) {  // class member CSR + fan-out work
      p.classes[c].mem_begin = (int32_t)p.members.size();
      for (int64_t nb : class_members[c]) p.members.push_back(nb);
      p.classes[c].mem_end = (int32_t)p.members.size();
    }

    double tc3 = prof ? clk() : 0;
    // ---------------- edge phase (aux_graph.hpp:273-296) -----------------
    int64_t aux = 0, rows = 0;
    p.valid_edges = 0;
    std::unordered_map<uint64_t, int32_t> sig_head;  // key hash -> first class; chains below
    std::vector<int32_t> sig_next, sig_pu, sig_pw;
    std::vector<int64_t> sig_shape;  // kMaxR extents per class
    std::vector<std::vector<int32_t>> edges_of_sig;
    if (p.host_err == ~0ull) {
      p.valid_edges = g->num_edges;
      for (int e = 0; e < g->num_edges; ++e) {
        p.edge_base[e] = aux;
        p.row_base[e] = rows;
        const int u = p.edge_from_op[e], w = p.edge_to_op[e];
        if (u < 0 || w < 0) {
          p.host_err = ekey(kEdgePhase + (uint64_t)aux * 2, tpk::kDangling);
          p.valid_edges = e;
          break;
        }
        const int ku = find_slot(u, g->edge_tensor[e]);
        const int kw = find_slot(w, g->edge_tensor[e]);
        if (ku < 0 || kw < 0) {
          p.host_err = ekey(kEdgePhase + (uint64_t)aux * 2, tpk::kEdgeTensorMissing);
          p.valid_edges = e;
          break;
        }
        const int tu = spec_of(u, ku), tw = spec_of(w, kw);
        const int R = rank_of(tu);
        bool same_shape = R == rank_of(tw);
        for (int d = 0; same_shape && d < R; ++d) same_shape = shape_of(tu)[d] == shape_of(tw)[d];
        if (!same_shape) {
          p.host_err = ekey(kEdgePhase + (uint64_t)aux * 2 + 1, tpk::kShapeMismatch);
          p.valid_edges = e;
          break;
        }
        const int pu = g->op_axis_begin[u + 1] - g->op_axis_begin[u];
        const int pw = g->op_axis_begin[w + 1] - g->op_axis_begin[w];
        const int64_t Su = p.node_base[u + 1] - p.node_base[u];
        const int64_t Sw = p.node_base[w + 1] - p.node_base[w];
        if (Su * Sw >= ((int64_t)1 << 31) - 4096)
          return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "more than 2^31 pairs on one edge");
        int64_t elements = 1;
        for (int d = 0; d < R; ++d) elements *= shape_of(tu)[d];
        const double bytes = (double)elements * g->tensor_element_size[tu];  // graph.hpp:52-54
        // edge class key (the reference's memo key, aux_graph.hpp:257-271, plus
        // the bytes and axis counts): hashed, compared field by field on a hit
        int64_t bbits;
        std::memcpy(&bbits, &bytes, 8);
        const auto& sau = sa_of(u, ku);
        const auto& saw = sa_of(w, kw);
        uint64_t h = hash_words(0x51ed27f3c6a8b9d1ull ^ ((uint64_t)pu << 40) ^ ((uint64_t)pw << 20) ^ (uint64_t)R,
                                &bbits, 8);
        h = hash_words(h, shape_of(tu), sizeof(int64_t) * R);
        h = hash_words(h, sau.data(), R);
        h = hash_words(h, saw.data(), R);
        int32_t sig = -1;
        auto it = sig_head.find(h);
        for (int32_t c = it == sig_head.end() ? -1 : it->second; c >= 0; c = sig_next[c]) {
          const SigDesc& o = p.sigs[c];
          if (o.R == R && o.tab_u == (int32_t)table_of_p[pu] && o.tab_w == (int32_t)table_of_p[pw] &&
              sig_pu[c] == pu && sig_pw[c] == pw && !std::memcmp(&o.bytes, &bytes, 8) &&
              !std::memcmp(sig_shape.data() + (size_t)c * tpk::kMaxR, shape_of(tu), sizeof(int64_t) * R) &&
              !std::memcmp(o.sa_u, sau.data(), R) && !std::memcmp(o.sa_w, saw.data(), R)) {
            sig = c;
            break;
          }
        }
        if (sig < 0) {
          sig = (int32_t)p.sigs.size();
          sig_next.push_back(it == sig_head.end() ? -1 : it->second);
          sig_head[h] = sig;
          sig_pu.push_back(pu);
          sig_pw.push_back(pw);
          sig_shape.resize(sig_shape.size() + tpk::kMaxR, 0);
          std::memcpy(sig_shape.data() + (size_t)sig * tpk::kMaxR, shape_of(tu), sizeof(int64_t) * R);
          SigDesc sd{};
          sd.pair_begin = p.total_pairs;
          sd.first_aux = aux;
          sd.bytes = bytes;
          sd.R = R;
          sd.Su = (int32_t)Su;
          sd.Sw = (int32_t)Sw;
          sd.tab_u = (int32_t)table_of_p[pu];
          sd.tab_w = (int32_t)table_of_p[pw];
          for (int side = 0; side < 2; ++side) {
            SideJob j{};
            j.out = p.side_total;
            j.tab = side ? sd.tab_w : sd.tab_u;
            j.count = (int32_t)(side ? Sw : Su);
            j.R = R;
            for (int d = 0; d < tpk::kMaxR; ++d) j.sa[d] = d < R ? (side ? sa_of(w, kw)[d] : sa_of(u, ku)[d]) : -1;
            (side ? sd.side_w : sd.side_u) = (int32_t)p.side_total;
            p.side_jobs.push_back(j);
            p.side_total += j.count;
          }
          for (int d = 0; d < tpk::kMaxR; ++d) {
            sd.sa_u[d] = d < R ? sa_of(u, ku)[d] : -1;
            sd.sa_w[d] = d < R ? sa_of(w, kw)[d] : -1;
            const int64_t E = d < R ? shape_of(tu)[d] : 1;
            const int v = v2_capped(E);
            sd.dt[d].t = (uint8_t)v;
            sd.dt[d].odd = (E >> v) > 1;
          }
          p.sigs.push_back(sd);
          edges_of_sig.emplace_back();
          p.total_pairs += Su * Sw;
        }
        edges_of_sig[sig].push_back(e);
        EdgeDesc ed{};
        ed.aux_base = aux;
        ed.nb_u = p.node_base[u];
        ed.nb_w = p.node_base[w];
        ed.wrow = wrow_of_op[w];
        ed.sig = sig;
        ed.e = e;
        p.edges.push_back(ed);
        aux += Su * Sw;
        rows += Su;
      }
      for (int e = p.valid_edges; e <= g->num_edges; ++e) {
        p.edge_base[e] = aux;
        p.row_base[e] = rows;
      }
    }
    p.num_aux_edges = aux;
    p.num_rows = rows;
    p.sig_edge_begin.push_back(0);
    for (auto& v : edges_of_sig) {
      for (int e : v) p.sig_edges.push_back(e);
      p.sig_edge_begin.push_back((int32_t)p.sig_edges.size());
    }
    for (int i = 0; i < p.valid_ops; ++i)
      if (p.in_deg[i] == 0) p.num_virtual += p.node_base[i + 1] - p.node_base[i];
    for (auto& sd : p.sigs) {
      sd.base = (int32_t)(&sd - p.sigs.data());
      sd.scale = 1.0;
    }
    double tc4 = prof ? clk() : 0;
    st = memo_aliasing();
    double tc5 = prof ? clk() : 0;
    if (st) return st;
    layout_tables(p.overrides.empty());
    double tc6 = prof ? clk() : 0;
    p.fsegs.clear();
    p.fsegs.reserve(p.edges.size());
    for (size_t e = 0; e < p.edges.size(); ++e) {
      const EdgeDesc& ed = p.edges[e];
      const SigDesc& sg = p.sigs[ed.sig];
      const SigDesc& bs = p.sigs[sg.base];
      FanSeg f{};
      f.begin = ed.aux_base;
      f.end = p.edge_base[e + 1];
      f.pb = sg.pair_begin;
      f.wrow = ed.wrow;
      f.nb_u = ed.nb_u;
      f.nb_w = ed.nb_w;
      f.f = sg.scale;
      f.e = ed.e;
      f.Sw = sg.Sw;
      f.Wn = sg.Wn;
      f.uid_u = sg.uid_u;
      f.uid_w = sg.uid_w;
      f.ident = sg.ident;
      f.st_q = kFusedThreads / sg.Sw;
      f.st_r = kFusedThreads % sg.Sw;
      f.base = sg.base;
      f.need = bs.Un * bs.Wn;
      p.fsegs.push_back(f);
    }
    p.pair_sig.assign(p.total_pairs, 0);
    for (size_t c = 0; c < p.sigs.size(); ++c)
      if (p.sigs[c].base == (int32_t)c)
        std::fill(p.pair_sig.begin() + p.sigs[c].pair_begin,
                  p.pair_sig.begin() + p.sigs[c].pair_begin + (int64_t)p.sigs[c].Un * p.sigs[c].Wn, (int32_t)c);
    p.row_cls.assign(p.total_rows, 0);
    for (size_t c = 0; c < p.classes.size(); ++c)
      std::fill(p.row_cls.begin() + p.classes[c].row_base, p.row_cls.begin() + p.classes[c].row_base + p.classes[c].S,
                (int32_t)c);
    if (prof)
      fprintf(stderr, "[tp host] check %.0f us, graph %.0f, node phase %.0f, edge phase %.0f, memo %.0f, tables %.0f, rest %.0f\n",
              tc1 - tc0, tc2 - tc1, tc3 - tc2, tc4 - tc3, tc5 - tc4, tc6 - tc5, clk() - tc6);
    p.h2d_bytes = (int64_t)(p.tabs.size() * sizeof(TableDesc) + p.classes.size() * sizeof(ClassDesc) +
                            p.members.size() * sizeof(int64_t) + p.chks.size() * sizeof(SliceChk) +
                            p.slots.size() * sizeof(SlotDesc) + p.occs.size() * sizeof(Occ) +
                            p.sigs.size() * sizeof(SigDesc) + p.edges.size() * sizeof(EdgeDesc) +
                            p.side_jobs.size() * sizeof(SideJob) +
                            p.overrides.size() * sizeof(double) + p.maps.size() * sizeof(int32_t) +
                            (p.pair_sig.size() + p.row_cls.size()) * sizeof(int32_t));
    return st;
  }

  // Slots, slice checks, occurrences of one op; then its node class.
  tp_status build_op(int i, int np, int64_t S, int64_t nb) {
    tp_plan& p = *P;
    HPROF(0);
    const int t0 = g->op_tensor_begin[i], t1 = g->op_tensor_begin[i + 1];
    const int sb = (int)slot_name.size();
    slot_begin[i] = sb;
    for (int t = t0; t < t1; ++t) {
      int k = -1;
      for (int x = sb; x < (int)slot_name.size(); ++x)
        if (slot_name[x] == g->tensor_name[t]) k = x - sb;
      if (k < 0) {
        k = (int)slot_name.size() - sb;
        slot_name.push_back(g->tensor_name[t]);
        slot_spec.push_back(t);
      }
      slot_spec[sb + k] = t;
      if (rank_of(t) > tpk::kMaxR) return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "tensor rank above 8");
      for (int d = 0; d < rank_of(t); ++d)
        if (shape_of(t)[d] < 1) return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "tensor extent < 1 is unsupported");
    }
    HPROF(1);
    const int nslot = (int)slot_name.size() - sb;
    slot_begin[i + 1] = sb + nslot;
    if (nslot > 32000) return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "too many tensors per op");
    std::array<int8_t, tpk::kMaxR> none;
    none.fill(-1);
    slot_sa.resize(sb + nslot, none);
    std::array<int8_t, tpk::kMaxR>* sa = slot_sa.data() + sb;
    chk.clear();
    const int a0 = g->op_axis_begin[i];
    for (int a = 0; a < np; ++a) {
      for (int s = g->axis_slice_begin[a0 + a]; s < g->axis_slice_begin[a0 + a + 1]; ++s) {
        const int k = find_slot(i, g->slice_tensor[s]);
        SliceChk c{};
        c.axis = (int8_t)a;
        c.slot = (int16_t)k;
        c.v = 0;
        if (k >= 0) {
          const int dim = g->slice_dim[s];
          const int tk = spec_of(i, k);
          if (dim < 0 || dim >= rank_of(tk))
            return set_err(TP_ERR_INVALID_ARGUMENT, 0, "slice dimension out of range");
          c.v = (int8_t)v2_capped(shape_of(tk)[dim]);
          sa[k][dim] = (int8_t)a;  // later slices overwrite (layout.hpp:366)
        }
        chk.push_back(c);
      }
    }
    HPROF(2);
    slots.clear();
    for (int k = 0; k < nslot; ++k) {
      SlotDesc sd{};
      const int tk = spec_of(i, k);
      int64_t el = 1;
      for (int d = 0; d < rank_of(tk); ++d) el *= shape_of(tk)[d];
      sd.elements = el;
      sd.es = g->tensor_element_size[tk];
      sd.R = (int8_t)rank_of(tk);
      for (int d = 0; d < tpk::kMaxR; ++d) sd.sa[d] = sa[k][d];
      slots.push_back(sd);
    }
    HPROF(3);
    occ.clear();
    const int nin = g->op_num_inputs[i];
    const int32_t* fed0 = fed_list.data() + fed_begin[op_key[i]];
    const int32_t* fed1 = fed_list.data() + fed_begin[op_key[i] + 1];
    for (int t = t0; t < t1; ++t) {
      Occ oc{};
      const int nm = g->tensor_name[t];
      oc.slot = (int16_t)find_slot(i, nm);
      uint8_t mask = 0;
      for (int a = 0; a < np; ++a) {
        bool slices = false;
        for (int s = g->axis_slice_begin[a0 + a]; s < g->axis_slice_begin[a0 + a + 1]; ++s)
          slices |= g->slice_tensor[s] == nm;
        if (!slices) mask |= (uint8_t)(1u << a);
      }
      oc.nonslicing = mask;
      if (t - t0 < nin) {
        bool fed = false;  // aux_graph.hpp:155-162
        for (const int32_t* x = fed0; x < fed1; ++x) fed |= *x == nm;
        oc.in_memory = !fed;
      } else {
        oc.in_memory = 1;
      }
      occ.push_back(oc);
    }
    HPROF(4);
    // node class key: everything the per-node costs depend on -- the axis
    // count, the in-degree and the slice checks, slots and occurrences (POD,
    // padding zeroed), hashed as words and compared bytewise on a hit
    uint64_t h = hash_words(0x9e3779b97f4a7c15ull ^ ((uint64_t)np << 32) ^ (uint64_t)(uint32_t)p.in_deg[i], chk.data(),
                            chk.size() * sizeof(SliceChk));
    h = hash_words(h ^ chk.size(), slots.data(), slots.size() * sizeof(SlotDesc));
    h = hash_words(h ^ slots.size(), occ.data(), occ.size() * sizeof(Occ));
    HPROF(5);
    int32_t cls = -1;
    auto it = class_head.find(h);
    for (int32_t c = it == class_head.end() ? -1 : it->second; c >= 0; c = class_next[c]) {
      const ClassDesc& cd = p.classes[c];
      if (cd.p == np && cd.indeg == (double)p.in_deg[i] && cd.chk_end - cd.chk_begin == (int)chk.size() &&
          class_nslot[c] == (int)slots.size() && cd.occ_end - cd.occ_begin == (int)occ.size() &&
          !std::memcmp(p.chks.data() + cd.chk_begin, chk.data(), chk.size() * sizeof(SliceChk)) &&
          !std::memcmp(p.slots.data() + cd.slot_begin, slots.data(), slots.size() * sizeof(SlotDesc)) &&
          !std::memcmp(p.occs.data() + cd.occ_begin, occ.data(), occ.size() * sizeof(Occ))) {
        cls = c;
        break;
      }
    }
    if (cls < 0) {
      cls = (int32_t)p.classes.size();
      class_next.push_back(it == class_head.end() ? -1 : it->second);
      class_head[h] = cls;
      class_nslot.push_back((int32_t)slots.size());
      ClassDesc cd{};
      cd.row_base = p.total_rows;
      cd.first_node = nb;
      cd.indeg = (double)p.in_deg[i];
      cd.S = (int32_t)S;
      cd.p = np;
      cd.table = (int32_t)table_of_p[np];
      cd.chk_begin = (int32_t)p.chks.size();
      p.chks.insert(p.chks.end(), chk.begin(), chk.end());
      cd.chk_end = (int32_t)p.chks.size();
      cd.slot_begin = (int32_t)p.slots.size();
      p.slots.insert(p.slots.end(), slots.begin(), slots.end());
      cd.occ_begin = (int32_t)p.occs.size();
      p.occs.insert(p.occs.end(), occ.begin(), occ.end());
      cd.occ_end = (int32_t)p.occs.size();
      p.classes.push_back(cd);
      class_members.emplace_back();
      p.total_rows += S;
    }
    HPROF(6);
    class_members[cls].push_back(nb);
    wrow_of_op[i] = p.classes[cls].row_base;
    p.op_row[i] = p.classes[cls].row_base;
    return TP_OK;
  }

  // Class tables over distinct layouts. A pair's price is a function of the
  // two layout descriptors (and the class's dims and bytes) only, so a class
  // computes one entry per (distinct producer layout, distinct consumer
  // layout) -- the reference's own memo key (aux_graph.hpp:257-271) -- and the
  // fan-out reads it through the strategy -> layout maps. An entry's error
  // is attributed to its first (su, sw), which is the smallest aux id any
  // strategy pair with those layouts has.
  //
  // Two edge classes with the same axis counts and slicings see the same
  // layouts. When every tensor dim of both has 2-adic valuation >= log2 N, no
  // layout can fail a divisibility check (a region spans at most log2 N
  // bits), so their plans are identical and every priced quantity is linear
  // in the tensor bytes; with a power-of-two byte ratio the later class's
  // table is the earlier one's times that ratio, exactly (scaling by 2^k
  // commutes with IEEE rounding). Such a class reuses the base table.
  //
  // With per-pair byte overrides (memo_aliasing) the tables stay per
  // strategy pair (identity maps).
  void layout_tables(bool dedup) {
    tp_plan& p = *P;
    p.maps.clear();
    std::map<std::vector<int64_t>, std::array<int32_t, 3>> side_cache;  // -> uid, rep, count
    auto side_maps = [&](int32_t tab, const int8_t* sa, int R, int32_t S) {
      std::vector<int64_t> key{tab, R};
      for (int d = 0; d < R; ++d) key.push_back(sa[d]);
      auto it = side_cache.find(key);
      if (it != side_cache.end()) return it->second;
      std::array<int32_t, 3> r{(int32_t)p.maps.size(), 0, 0};
      std::vector<int32_t> uid(S), reps;
      if (dedup) {
        const TableDesc* td = nullptr;
        for (const auto& t : p.tabs)
          if (t.offset == tab) td = &t;
        // distinct layout descriptors (POD, zeroed), by hash with a chain per id
        std::unordered_map<uint64_t, int32_t> head;
        std::vector<int32_t> next;
        std::vector<tpk::SideDesc> seen;
        for (int32_t s = 0; s < S; ++s) {
          Strat st;
          tpk::unrank_strategy((int)td->p, (int)td->n, s, st);
          Lay L;
          tpk::side_layout(st, sa, R, L);
          tpk::SideDesc d;
          std::memset(&d, 0, sizeof(d));
          tpk::side_of(L, R, d);
          const uint64_t h = hash_words(0x2545f4914f6cdd1dull, &d, sizeof(d));
          auto it = head.find(h);
          int32_t id = -1;
          for (int32_t c = it == head.end() ? -1 : it->second; c >= 0; c = next[c])
            if (!std::memcmp(&seen[c], &d, sizeof(d))) {
              id = c;
              break;
            }
          if (id < 0) {
            id = (int32_t)reps.size();
            next.push_back(it == head.end() ? -1 : it->second);
            head[h] = id;
            seen.push_back(d);
            reps.push_back(s);
          }
          uid[s] = id;
        }
      } else {
        for (int32_t s = 0; s < S; ++s) uid[s] = s, reps.push_back(s);
      }
      p.maps.insert(p.maps.end(), uid.begin(), uid.end());
      r[1] = (int32_t)p.maps.size();
      r[2] = (int32_t)reps.size();
      p.maps.insert(p.maps.end(), reps.begin(), reps.end());
      side_cache.emplace(key, r);
      return r;
    };
    const bool derive = dedup && p.N > 0 && (p.N & (p.N - 1)) == 0;
    std::map<std::vector<int64_t>, int32_t> base_of;
    int64_t pairs = 0;
    for (size_t c = 0; c < p.sigs.size(); ++c) {
      SigDesc& sd = p.sigs[c];
      const auto mu = side_maps(sd.tab_u, sd.sa_u, sd.R, sd.Su);
      const auto mw = side_maps(sd.tab_w, sd.sa_w, sd.R, sd.Sw);
      sd.uid_u = mu[0], sd.rep_u = mu[1], sd.Un = mu[2];
      sd.uid_w = mw[0], sd.rep_w = mw[1], sd.Wn = mw[2];
      sd.ident = sd.Un == sd.Su && sd.Wn == sd.Sw;  // ids are assigned in first-seen order
      bool safe = derive;
      for (int d = 0; d < sd.R; ++d) safe &= sd.dt[d].t >= p.n_log2;
      std::vector<int64_t> key{sd.tab_u, sd.tab_w, sd.R};
      for (int d = 0; d < sd.R; ++d) key.insert(key.end(), {(int64_t)sd.sa_u[d], (int64_t)sd.sa_w[d]});
      if (safe) {
        auto it = base_of.find(key);
        if (it != base_of.end()) {
          const SigDesc& b = p.sigs[it->second];
          int ex = 0;
          const double m = std::frexp(sd.bytes / b.bytes, &ex);
          if (m == 0.5 && sd.bytes == std::ldexp(b.bytes, ex - 1) && ex > -900 && ex < 900) {
            sd.base = it->second;
            sd.scale = std::ldexp(1.0, ex - 1);
            sd.pair_begin = b.pair_begin;
            continue;
          }
        } else {
          base_of.emplace(key, (int32_t)c);
        }
      }
      sd.pair_begin = pairs;  // compact the computed tables
      pairs += (int64_t)sd.Un * sd.Wn;
    }
    p.total_pairs = pairs;
  }

  // The reference memo (aux_graph.hpp:257-271) keys on (shape, matrix, map)
  // of both layouts but prices with the FIRST edge's tensor bytes. Only when
  // same-shape edge classes carry different bytes can that be observed; then
  // the first writer's bytes are resolved per pair here (host, rare path).
  tp_status memo_aliasing() {
    tp_plan& p = *P;
    std::map<std::vector<int64_t>, std::vector<int32_t>> by_shape;
    std::vector<std::vector<int64_t>> shape_of_sig(p.sigs.size());
    for (size_t s = 0; s < p.sigs.size(); ++s) {
      const EdgeDesc& ed = p.edges[p.sig_edges[p.sig_edge_begin[s]]];
      const int u = p.edge_from_op[ed.e];
      const int tu = spec_of(u, find_slot(u, g->edge_tensor[ed.e]));
      shape_of_sig[s].assign(shape_of(tu), shape_of(tu) + rank_of(tu));
      by_shape[shape_of_sig[s]].push_back((int32_t)s);
    }
    bool hazard = false;
    for (auto& kv : by_shape)
      for (int32_t s : kv.second)
        if (p.sigs[s].bytes != p.sigs[kv.second[0]].bytes) hazard = true;
    if (!hazard) return TP_OK;
    if (p.total_pairs > (int64_t)1 << 26) return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "aliasing graph too large");
    std::map<int64_t, std::vector<Strat>> host_tab;  // by table offset
    for (auto& td : p.tabs) {
      auto& v = host_tab[td.offset];
      v.resize(td.count);
      for (int64_t s = 0; s < td.count; ++s) tpk::unrank_strategy(td.p, td.n, s, v[s]);
    }
    p.overrides.assign(p.total_pairs, 0.0);
    std::vector<int32_t> order(p.sigs.size());
    for (size_t s = 0; s < order.size(); ++s) order[s] = (int32_t)s;
    std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
      return p.sigs[a].first_aux < p.sigs[b].first_aux;
    });
    std::unordered_map<std::string, double> first;
    for (int32_t s : order) {
      SigDesc& sd = p.sigs[s];
      sd.has_override = 1;
      const std::string shape_key(reinterpret_cast<const char*>(shape_of_sig[s].data()),
                                  shape_of_sig[s].size() * sizeof(int64_t));
      for (int64_t su = 0; su < sd.Su; ++su) {
        Lay F;
        tpk::side_layout(host_tab[sd.tab_u][su], sd.sa_u, sd.R, F);
        for (int64_t sw = 0; sw < sd.Sw; ++sw) {
          Lay T;
          tpk::side_layout(host_tab[sd.tab_w][sw], sd.sa_w, sd.R, T);
          const int64_t idx = sd.pair_begin + su * sd.Sw + sw;
          p.overrides[idx] = sd.bytes;
          if (tpk::same_layout(F, T, sd.R)) continue;
          std::string key = shape_key;
          key.push_back((char)F.depth);
          key.append(reinterpret_cast<const char*>(F.mx), F.depth);
          key.append(reinterpret_cast<const char*>(F.map), sd.R);
          key.push_back((char)T.depth);
          key.append(reinterpret_cast<const char*>(T.mx), T.depth);
          key.append(reinterpret_cast<const char*>(T.map), sd.R);
          auto it = first.find(key);
          if (it == first.end()) first.emplace(key, sd.bytes);
          else p.overrides[idx] = it->second;
        }
      }
    }
    return TP_OK;
  }
};

tp_status ensure_stream(tp_plan* p) {
  CUDA_TRY(cudaSetDevice(p->device));
  if (!p->arena) {
    p->arena = new Arena();
    p->arena->device = p->device;
    p->owns_arena = true;
  }
  if (!p->arena->stream) CUDA_TRY(cudaStreamCreateWithFlags(&p->arena->stream, cudaStreamNonBlocking));
  return TP_OK;
}

Arena* thread_arena(int device) {
  static thread_local Arena* arenas[64];  // one per device ordinal; POD
  if (device < 0 || device >= 64) return nullptr;
  Arena*& a = arenas[device];
  if (!a) {
    a = new Arena();
    a->device = device;
  }
  return a;
}

// --- batches: a host worker pool and pooled per-device arenas ---------------
// Arenas outlive a batch call so later batches pay neither cudaMalloc nor the
// strategy-table kernel; a worker holds one for the whole call.
std::mutex g_pool_mu;
std::vector<Arena*> g_pool[64];

Arena* arena_pool_get(int device) {
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto& v = g_pool[device & 63];
    if (!v.empty()) {
      Arena* a = v.back();
      v.pop_back();
      return a;
    }
  }
  Arena* a = new Arena();
  a->device = device;
  return a;
}

void arena_pool_put(Arena* a) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  g_pool[a->device & 63].push_back(a);
}

int pool_size(int n, int host_threads) {
  int t = host_threads > 0 ? host_threads : (int)std::min(32u, std::max(1u, std::thread::hardware_concurrency()));
  return std::max(1, std::min(t, n));
}

// fn(item, worker) over items [0, n), items claimed one at a time. The
// workers make `device` current first (a new host thread starts on device 0:
// anything they allocate must land on the plans' device).
template <typename F>
void run_pool(int n, int workers, F&& fn, int device = -1) {
  workers = pool_size(n, workers);
  std::atomic<int> next{0};
  auto body = [&](int w) {
    if (device >= 0 && w > 0) cudaSetDevice(device);
    for (int i = next.fetch_add(1); i < n; i = next.fetch_add(1)) fn(i, w);
  };
  std::vector<std::thread> th;
  for (int w = 1; w < workers; ++w) th.emplace_back(body, w);
  body(0);
  for (auto& x : th) x.join();
}

// a worker's status and message (tp_last_error is per thread)
struct BatchErr {
  tp_status st = TP_OK;
  int kind = 0;
  std::string msg;
  void take(tp_status s) {
    st = s;
    if (s) {
      kind = g_err_kind;
      msg = g_err;
    }
  }
};

tp_status batch_status(const std::vector<BatchErr>& errs, int32_t* status_out) {
  const BatchErr* first = nullptr;
  for (size_t i = 0; i < errs.size(); ++i) {
    if (status_out) status_out[i] = errs[i].st;
    if (errs[i].st && !first) first = &errs[i];
  }
  if (!first) {
    g_err[0] = 0;
    g_err_kind = 0;
    return TP_OK;
  }
  return set_err(first->st, first->kind, first->msg);
}
}  // namespace

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

int32_t tp_abi_version(void) { return TP_ABI_VERSION; }
const char* tp_last_error(void) { return g_err; }
int32_t tp_last_error_kind(void) { return g_err_kind; }

tp_status tp_plan_create(const tp_graph_desc* graph, const tp_topology_desc* topo, int32_t device,
                         tp_plan** plan_out) {
  if (!plan_out) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null plan_out");
  *plan_out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_err(TP_ERR_CUDA, 0, "no CUDA device: the engine has no CPU path");
  tp_plan* p = new tp_plan();
  if (device < 0) cudaGetDevice(&p->device);
  else p->device = device;
  Builder b{graph, topo, p};
  tp_status st = b.run();
  if (st) {
    delete p;
    return st;
  }
  *plan_out = p;
  g_err[0] = 0;
  g_err_kind = 0;
  return TP_OK;
}

void tp_plan_destroy(tp_plan* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  if (p->d_terms) {
    p->d_terms->release();
    delete p->d_terms;
  }
  if (p->arena) {
    if (p->arena->stream) cudaStreamSynchronize(p->arena->stream);
    if (p->owns_arena) {
      p->arena->release();
      delete p->arena;
    }
  }
  delete p;
}

tp_status tp_plan_sizes(const tp_plan* p, tp_plan_sizes_t* s) {
  if (!p || !s) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null argument");
  s->num_ops = p->num_ops;
  s->num_edges = p->num_edges;
  s->num_aux_nodes = p->num_aux_nodes;
  s->num_aux_edges = p->num_aux_edges;
  s->num_virtual_edges = p->num_virtual;
  s->num_rows = p->num_rows;
  s->num_signatures = (int64_t)p->sigs.size();
  s->num_pair_evals = p->total_pairs;
  s->h2d_bytes = p->h2d_bytes;
  s->num_class_rows = p->total_rows;
  s->num_pair_slots = 0;
  for (const auto& sd : p->sigs) s->num_pair_slots += (int64_t)sd.Su * sd.Sw;
  return TP_OK;
}

tp_status tp_plan_index(const tp_plan* p, tp_aux_index* x) {
  if (!p || !x) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null argument");
  if (x->node_base) std::memcpy(x->node_base, p->node_base.data(), sizeof(int64_t) * (p->num_ops + 1));
  if (x->edge_base) std::memcpy(x->edge_base, p->edge_base.data(), sizeof(int64_t) * (p->num_edges + 1));
  if (x->edge_from_op && p->num_edges)
    std::memcpy(x->edge_from_op, p->edge_from_op.data(), sizeof(int32_t) * p->num_edges);
  if (x->edge_to_op && p->num_edges) std::memcpy(x->edge_to_op, p->edge_to_op.data(), sizeof(int32_t) * p->num_edges);
  if (x->in_degree && p->num_ops) std::memcpy(x->in_degree, p->in_deg.data(), sizeof(int32_t) * p->num_ops);
  if (x->out_degree && p->num_ops) std::memcpy(x->out_degree, p->out_deg.data(), sizeof(int32_t) * p->num_ops);
  if (x->topo_order && p->num_ops) std::memcpy(x->topo_order, p->topo.data(), sizeof(int32_t) * p->num_ops);
  return TP_OK;
}

namespace {
// Persistent grid of the fused kernel on the plan's device (cached per device).
int g_resident[64];
tp_status resident_of(tp_plan* p) {
  int& r = g_resident[p->device & 63];
  if (r == 0) {
    int sms = 0, per_sm = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device));
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_kernel<true>, kFusedThreads, 0));
    r = std::max(1, sms * std::max(1, per_sm));
  }
  p->resident_blocks = r;
  return TP_OK;
}

// Phase 2: the aux nodes and the edge range's aux edges cut into equal
// ranges, one per resident CTA.
void range_layout(const tp_plan* p, int64_t total_out, int64_t total_nodes, int64_t& range_len, int64_t& exp_items,
                  int64_t& nfan_items) {
  const int64_t nranges = std::max(1, p->resident_blocks - 2);  // the two ceilings below add at most 2
  range_len = std::max<int64_t>(kFusedThreads * kFanPer, (total_out + total_nodes + nranges - 1) / nranges);
  exp_items = (total_out + range_len - 1) / range_len;
  nfan_items = (total_nodes + range_len - 1) / range_len;
}

// First edge / operator of every range.
void fill_range_first(tp_plan* p, int32_t e0, int32_t e1, int64_t range_len, int64_t exp_items, int64_t nfan_items) {
  const int64_t out_offset = p->edge_base[e0];
  p->range_first.assign(exp_items + nfan_items, 0);
  for (int64_t r = 0; r < exp_items; ++r) {
    const int64_t start = out_offset + r * range_len;
    auto it = std::upper_bound(p->edge_base.begin() + e0, p->edge_base.begin() + e1, start);
    p->range_first[r] = (int32_t)(it - p->edge_base.begin()) - 1;
  }
  for (int64_t r = 0; r < nfan_items; ++r) {
    const int64_t start = r * range_len;
    auto it = std::upper_bound(p->node_base.begin(), p->node_base.begin() + p->num_ops, start);
    p->range_first[exp_items + r] = (int32_t)(it - p->node_base.begin()) - 1;
  }
}
}  // namespace

// doubles per parity block of the published tables
static int64_t tables_len(const tp_plan* p) { return 2 * (p->total_pairs + 1) + 4 * (p->total_rows + 1); }

}  // extern "C"

namespace {
// An upload in pieces (tp_plan_upload runs them back to back; the host batch
// packs every plan's descriptors into one copy and runs the set-up kernels
// of all plans as two launches).
struct UploadPrep {
  DescPack pk;
  bool new_tables = false;
  std::vector<std::array<int64_t, 4>> key;
  std::vector<double> price;
  bool packed_ranges = false;
  std::array<int64_t, 4> def_key{{-1, -1, -1, -1}};
};

// Host only: the descriptor pieces of the plan (and its default range table).
tp_status upload_prepare(tp_plan* p, UploadPrep& U) {
  Arena& A = *p->arena;
  // strategy tables: a pure function of (p, N), cached on the arena
  for (auto& td : p->tabs) U.key.push_back({td.offset, td.count, td.p, td.n});
  U.new_tables = U.key != A.table_key && p->table_total > 0;
  U.price.resize(tpk::kBwTab + tpk::kScaleDim * tpk::kScaleDim);
  tpk::make_price_tabs(p->env, U.price.data(), U.price.data() + tpk::kBwTab);
  DescPack& pk = U.pk;
  if (U.new_tables) pk.add(A.d_tabs, p->tabs);
  pk.add(A.d_sidejobs, p->side_jobs);
  pk.add(A.d_price, U.price);
  pk.add(A.d_classes, p->classes);
  pk.add(A.d_opnode, p->node_base);
  pk.add(A.d_oprow, p->op_row);
  pk.add(A.d_members, p->members);
  pk.add(A.d_chks, p->chks);
  pk.add(A.d_slots, p->slots);
  pk.add(A.d_occs, p->occs);
  pk.add(A.d_sigs, p->sigs);
  pk.add(A.d_pairsigs, p->pair_sig);
  pk.add(A.d_rowcls, p->row_cls);
  pk.add(A.d_maps, p->maps);
  pk.add(A.d_edges, p->edges);
  pk.add(A.d_fsegs, p->fsegs);
  pk.add(A.d_over, p->overrides);
  // the range table of the default execute (whole graph, every tensor) goes
  // up with the pack; another edge range or output set re-uploads its own
  if (!(p->host_err != ~0ull && (p->host_err >> 6) == 0)) {
    tp_status rs = resident_of(p);
    if (rs) return rs;
    const bool edge_phase = p->host_err >= ekey(kEdgePhase, 0);
    const int32_t e1 = p->valid_edges;
    const int64_t total_out =
        (edge_phase && p->edge_base[e1] > p->edge_base[0]) ? p->edge_base[e1] - p->edge_base[0] : 0;
    int64_t rl, ei, ni;
    range_layout(p, total_out, p->num_aux_nodes, rl, ei, ni);
    fill_range_first(p, 0, e1, rl, ei, ni);
    U.def_key = {{0, e1, rl, ni}};
    pk.add(A.d_rfirst, p->range_first);
    U.packed_ranges = true;
  }
  return TP_OK;
}

// Copy the pieces into pinned staging at `host` and point the plan's views
// at `dev` (same offsets); the caller copies host -> dev.
void upload_stage(UploadPrep& U, char* host, char* dev) {
  for (auto& x : U.pk.pieces) x.buf->release();
  size_t off = 0;
  for (auto& x : U.pk.pieces) {
    if (x.bytes) std::memcpy(host + off, x.src, x.bytes);
    x.buf->set_view(dev + off, DescPack::pad(x.bytes));
    off += DescPack::pad(x.bytes);
  }
}

// Device buffers the set-up kernels and the launches write (cudaMalloc only
// when an arena grows), the clean state, the plan's flags.
tp_status upload_finish(tp_plan* p, UploadPrep& U) {
  CUDA_TRY(cudaSetDevice(p->device));  // the buffers below belong on the plan's device
  Arena& A = *p->arena;
  CUDA_TRY(A.d_sides.ensure(sizeof(tpk::SideDesc) * (p->side_total + 1)));
  CUDA_TRY(A.d_pairrec.ensure(sizeof(PairRec) * (p->total_pairs + 1)));
  if (U.new_tables) CUDA_TRY(A.d_tables.ensure(sizeof(Strat) * (p->table_total + 1)));
  // per parity: (cost, volume) [total_pairs + 1]; (cost, volume), mem, mem / indeg [total_rows + 1]
  // A finished launch leaves the counters zero and the next parity's tables
  // unset, so an arena whose table layout and counter block are unchanged
  // stays clean for the next plan; anything else is reset before its launch.
  const int64_t L = tables_len(p);
  const size_t sched_bytes = sizeof(Sched) + sizeof(Line) * (p->sigs.size() + 1);
  const bool same_layout = A.d_tables2.p && A.d_tables2.cap >= sizeof(double) * 2 * L && A.d_sched.p &&
                           A.d_sched.cap >= sched_bytes && A.tables_L == L && A.sched_bytes == sched_bytes;
  CUDA_TRY(A.d_tables2.ensure(sizeof(double) * 2 * L));
  CUDA_TRY(A.d_sched.ensure(sched_bytes));
  if (!same_layout) A.sched_clean = false;
  A.tables_L = L;
  A.sched_bytes = sched_bytes;
  p->range_key = U.packed_ranges ? U.def_key : std::array<int64_t, 4>{{-1, -1, -1, -1}};
  p->uploaded = true;
  return TP_OK;
}

tp_status upload_tables(tp_plan* p, UploadPrep& U, cudaStream_t s) {
  Arena& A = *p->arena;
  if (!U.new_tables) return TP_OK;
  table_kernel<<<(unsigned)((p->table_total + 127) / 128), 128, 0, s>>>(
      (const TableDesc*)A.d_tabs.p, (int)p->tabs.size(), p->table_total, (Strat*)A.d_tables.p);
  CUDA_TRY(cudaGetLastError());
  A.table_key = U.key;
  return TP_OK;
}
}  // namespace

extern "C" {

tp_status tp_plan_upload(tp_plan* p, void* stream) {
  if (!p) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null plan");
  tp_status st = ensure_stream(p);
  if (st) return st;
  Arena& A = *p->arena;
  cudaStream_t s = stream ? (cudaStream_t)stream : A.stream;
  UploadPrep U;
  st = upload_prepare(p, U);
  if (st) return st;
  const size_t total = U.pk.total();
  if (A.stage_done) CUDA_TRY(cudaEventSynchronize(A.stage_done));  // h_stage free again
  if (A.h_stage_cap < total) {
    if (A.h_stage) cudaFreeHost(A.h_stage);
    A.h_stage = nullptr;
    A.h_stage_cap = 0;
    CUDA_TRY(cudaMallocHost(&A.h_stage, total));
    A.h_stage_cap = total;
  }
  // views first (d_desc may be reallocated, which frees nothing the views own)
  for (auto& x : U.pk.pieces) x.buf->release();
  CUDA_TRY(A.d_desc.ensure(total));
  upload_stage(U, (char*)A.h_stage, (char*)A.d_desc.p);
  CUDA_TRY(cudaMemcpyAsync(A.d_desc.p, A.h_stage, total, cudaMemcpyHostToDevice, s));
  if (!A.stage_done) CUDA_TRY(cudaEventCreateWithFlags(&A.stage_done, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(A.stage_done, s));
  st = upload_finish(p, U);
  if (st) return st;
  st = upload_tables(p, U, s);
  if (st) return st;
  // layout descriptors of every (edge class, side, strategy)
  if (p->side_total > 0) {
    side_kernel<<<(unsigned)((p->side_total + 127) / 128), 128, 0, s>>>(
        (const SideJob*)A.d_sidejobs.p, (int)p->side_jobs.size(), p->side_total, (const Strat*)A.d_tables.p,
        (tpk::SideDesc*)A.d_sides.p);
    CUDA_TRY(cudaGetLastError());
  }
  if (p->total_pairs > 0) {
    pair_rec_kernel<<<(unsigned)((p->total_pairs + 127) / 128), 128, 0, s>>>(
        (const SigDesc*)A.d_sigs.p, (const int32_t*)A.d_pairsigs.p, (const int32_t*)A.d_maps.p,
        (const tpk::SideDesc*)A.d_sides.p, (const double*)A.d_over.p, p->total_pairs, (PairRec*)A.d_pairrec.p);
    CUDA_TRY(cudaGetLastError());
  }
  return TP_OK;
}

}  // extern "C"

namespace {
// The host half of an execute, up to the fused launch: per-arena set-up on
// stream s, the range tables, the kernel arguments. X.launch says whether a
// fused launch is needed (X.a, X.grid); tp_plan_execute launches it alone,
// tp_plan_execute_batch together with other plans'.
struct ExecPrep {
  FusedArgs a{};
  int64_t grid = 0;
  bool launch = false;
  bool done = false;  // nothing at all to run (host-detected cycle)
  int32_t e0 = 0, e1 = 0;
  int64_t out_offset = 0;
  bool edge_phase = false;
  int64_t units = 0, items = 0;
};

tp_status prepare_execute(tp_plan* p, const tp_build_opts* opts, tp_cost_tensors* out, cudaStream_t s, ExecPrep& X) {
  Arena& A = *p->arena;
  p->last_stream = s;
  int32_t e0 = opts ? opts->edge_begin : 0;
  int32_t e1 = opts ? opts->edge_end : -1;
  if (e1 < 0 || e1 > p->valid_edges) e1 = p->valid_edges;
  if (e0 < 0) e0 = 0;
  if (e0 > e1) e0 = e1;
  const bool skip_nodes = opts && opts->skip_nodes;
  static const tp_cost_tensors none{};
  if (!out) out = const_cast<tp_cost_tensors*>(&none);
  Sched* sched = (Sched*)A.d_sched.p;
  if (!A.sched_clean) {
    CUDA_TRY(cudaMemsetAsync(sched, 0, sizeof(Sched) + sizeof(Line) * (p->sigs.size() + 1), s));
    fill_kernel<<<64, 256, 0, s>>>((double*)A.d_tables2.p, 2 * tables_len(p), kUnset);  // both parities
    CUDA_TRY(cudaGetLastError());
    A.sched_clean = true;
    A.parity = 0;
  }
  p->last_parity = -1;
  if (p->timeline || A.timeline_set) {
    CUDA_TRY(cudaMemsetAsync(&sched->timeline, 0, sizeof(int) * 2 + sizeof(sched->t), s));
    if (p->timeline) CUDA_TRY(cudaMemsetAsync(&sched->timeline, 0x01, 1, s));
    A.timeline_set = p->timeline;
  }
  if (p->host_err != ~0ull && (p->host_err >> 6) == 0) {  // cycle: nothing to build
    X.done = true;
    return TP_OK;
  }
  const bool edge_phase = p->host_err >= ekey(kEdgePhase, 0);
  const bool nodes_out = !skip_nodes && (out->node_intra_cost_s || out->node_intra_volume_bytes ||
                                         out->node_memory_bytes);
  const int64_t out_offset = p->edge_base[e0];
  const bool edges_out = p->edge_base[e1] > out_offset && edge_phase &&
                         (out->edge_cost_s || out->edge_volume_bytes || out->edge_memory_bytes ||
                          out->aux_edge_records);
  if (p->resident_blocks == 0) {
    tp_status rs = resident_of(p);
    if (rs) return rs;
  }
  const int64_t total_out = edges_out ? p->edge_base[e1] - out_offset : 0;
  const int64_t total_nodes = nodes_out ? p->num_aux_nodes : 0;
  int64_t range_len, exp_items, nfan_items;
  range_layout(p, total_out, total_nodes, range_len, exp_items, nfan_items);
  const std::array<int64_t, 4> rkey{{e0, e1, range_len, nfan_items}};
  if (p->range_key != rkey) {  // first edge / operator of every range (cached)
    fill_range_first(p, e0, e1, range_len, exp_items, nfan_items);
    CUDA_TRY(upload(A.d_rfirst, p->range_first, s));
    p->range_key = rkey;
  }
  FusedArgs& a = X.a;
  a.classes = (const ClassDesc*)A.d_classes.p;
  a.ncls = (int)p->classes.size();
  a.total_rows = p->total_rows;
  a.chks = (const SliceChk*)A.d_chks.p;
  a.slots = (const SlotDesc*)A.d_slots.p;
  a.occs = (const Occ*)A.d_occs.p;
  {
    const int64_t L = tables_len(p), P = p->total_pairs + 1, R = p->total_rows + 1;
    double* t = (double*)A.d_tables2.p + A.parity * L;
    a.r_tab = reinterpret_cast<double2*>(t);  // 16-B aligned: L and P, R offsets are even
    a.cls_sv = reinterpret_cast<double2*>(t + 2 * P);
    a.cls_mem = t + 2 * P + 2 * R;
    a.cls_memdiv = t + 2 * P + 3 * R;
    a.next_tables = (double*)A.d_tables2.p + (A.parity ^ 1) * L;
    a.tables_len = L;
  }
  a.sigs = (const SigDesc*)A.d_sigs.p;
  a.nsigs = (int)p->sigs.size();
  a.pair_sig = (const int32_t*)A.d_pairsigs.p;
  a.pairs = (const PairRec*)A.d_pairrec.p;
  a.row_cls = (const int32_t*)A.d_rowcls.p;
  a.maps = (const int32_t*)A.d_maps.p;

  a.total_pairs = edge_phase ? p->total_pairs : 0;
  a.overrides = (const double*)A.d_over.p;
  a.sides = (const tpk::SideDesc*)A.d_sides.p;

  a.edges = (const EdgeDesc*)A.d_edges.p;
  a.fsegs = (const FanSeg*)A.d_fsegs.p;
  a.range_first = (const int32_t*)A.d_rfirst.p;
  a.nrange_first = a.range_first + exp_items;
  a.e0 = e0;
  a.e1 = e1;
  a.A0 = out_offset;
  a.A1 = p->edge_base[e1];
  a.range_len = range_len;
  a.e_sec = out->edge_cost_s;
  a.e_vol = out->edge_volume_bytes;
  a.e_mem = out->edge_memory_bytes;
  a.records = (char*)out->aux_edge_records;
  a.general_store = a.records || !(a.e_sec && a.e_vol && a.e_mem);
  a.op_node = (const int64_t*)A.d_opnode.p;
  a.op_row = (const int64_t*)A.d_oprow.p;
  a.nops = p->num_ops;
  a.num_nodes = p->num_aux_nodes;
  a.node_range_len = range_len;
  a.n_sec = nodes_out ? out->node_intra_cost_s : nullptr;
  a.n_vol = nodes_out ? out->node_intra_volume_bytes : nullptr;
  a.n_mem = nodes_out ? out->node_memory_bytes : nullptr;
  a.tables = (const Strat*)A.d_tables.p;
  a.env = p->env;
  a.l_log2 = (p->env.local > 0 && (p->env.local & (p->env.local - 1)) == 0) ? log2_floor(p->env.local) : -1;
  a.n_log2 = p->n_log2;
  a.bw_tab = (const double*)A.d_price.p;
  a.scale_tab = (const double*)A.d_price.p + tpk::kBwTab;
  a.sched = sched;
  a.parity = A.parity;
  a.err = &sched->err_c[A.parity];
  a.nsigs_reset = (int)p->sigs.size();
  if (p->timeline) {
    p->trace_n[0] = p->total_pairs;
    p->trace_n[1] = p->total_rows;
    p->trace_n[2] = exp_items;
    const int64_t n = 2 * p->trace_n[0] + 2 * p->trace_n[1] + 3 * p->trace_n[2] + 1;
    CUDA_TRY(A.d_trace.ensure(sizeof(unsigned) * n));
    CUDA_TRY(cudaMemsetAsync(A.d_trace.p, 0, sizeof(unsigned) * n, s));
    a.pair_ns = (unsigned*)A.d_trace.p;
    a.item_ns = a.pair_ns + 2 * p->trace_n[0];
    a.fan_ns = a.item_ns + 2 * p->trace_n[1];
    const size_t nprof = 8 * (p->total_pairs + 1) + 8 * 4096;
    CUDA_TRY(A.d_prof.ensure(sizeof(unsigned) * nprof));
    CUDA_TRY(cudaMemsetAsync(A.d_prof.p, 0, sizeof(unsigned) * nprof, s));
    a.pair_prof = (unsigned*)A.d_prof.p;
    a.warp_exit = a.pair_prof + 8 * (p->total_pairs + 1);
  }
  // by size: a warp per pair while the launch has too few pairs to fill the
  // GPU with one thread per pair; a big batch of plans is judged as a whole
  a.warp_form = p->pair_form == 1 || (p->pair_form == 0 && !p->in_big_batch && a.total_pairs <= kWarpPairLimit);

  // phase-1 units: node rows, then class pairs (warp form) or 32-pair chunks;
  // phase-2 items: node ranges, then edge ranges
  const int64_t units = p->total_rows + (a.warp_form ? a.total_pairs : (a.total_pairs + 31) / 32);
  const int64_t total_items = exp_items + nfan_items;
  if (total_items >= (1ll << 30) || units >= (1ll << 30))
    return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "too many work items");
  a.i_exp = (int)nfan_items;
  a.i_end = (int)total_items;
  X.e0 = e0;
  X.e1 = e1;
  X.out_offset = out_offset;
  X.edge_phase = edge_phase;
  X.units = units;
  X.items = total_items;
  X.launch = total_items > 0 || units > 0;
  if (X.launch) {
    const int64_t blocks_needed = std::max<int64_t>(total_items, (units + 7) / 8);
    X.grid = std::max<int64_t>(1, std::min<int64_t>(blocks_needed, p->resident_blocks));
  }
  return TP_OK;
}

// After the fused launch of a prepared plan (alone or in a batch).
void after_launch(tp_plan* p) {
  Arena& A = *p->arena;
  p->last_parity = A.parity;
  A.parity ^= 1;
}

// K3 (optional row minima) and the launch count of a prepared execute.
tp_status finish_execute(tp_plan* p, tp_cost_tensors* out, cudaStream_t s, const ExecPrep& X, int64_t launches) {
  Arena& A = *p->arena;
  const int32_t e0 = X.e0, e1 = X.e1;
  const int64_t out_offset = X.out_offset;
  const bool edge_phase = X.edge_phase;
  const FusedArgs& a = X.a;
  if (p->edge_base[e1] > out_offset && edge_phase) {
    // K3: row minima
    if (out->row_min_cost_s && out->row_min_volume_bytes) {
      const int64_t r0 = p->row_base[e0], r1 = p->row_base[e1];
      std::vector<int64_t> rb(p->row_base.begin() + e0, p->row_base.begin() + e1 + 1);
      for (auto& v : rb) v -= r0;
      CUDA_TRY(upload(A.d_rowbase, rb, s));
      const int64_t rows = r1 - r0;
      const int th = 256;
      rowmin_kernel<<<(unsigned)((rows * 32 + th - 1) / th), th, 0, s>>>(
          (const EdgeDesc*)A.d_edges.p, (const int64_t*)A.d_rowbase.p, e0, e1 - e0, rows,
          (const SigDesc*)A.d_sigs.p, (const int32_t*)A.d_maps.p, a.r_tab, a.cls_sv,
          out->row_min_cost_s, out->row_min_volume_bytes);
      ++launches;
    }
  }
  CUDA_TRY(cudaGetLastError());
  p->last_launches = launches;
  return TP_OK;
}

}  // namespace

extern "C" {

tp_status tp_plan_execute(tp_plan* p, const tp_build_opts* opts, tp_cost_tensors* out) {
  if (!p) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null plan");
  tp_status st = ensure_stream(p);
  if (st) return st;
  if (!p->uploaded) {
    st = tp_plan_upload(p, opts ? opts->stream : nullptr);
    if (st) return st;
  }
  cudaStream_t s = (opts && opts->stream) ? (cudaStream_t)opts->stream : p->arena->stream;
  ExecPrep X;
  st = prepare_execute(p, opts, out, s, X);
  if (st) return st;
  if (X.done) {
    p->last_launches = 0;
    return TP_OK;
  }
  Arena& A = *p->arena;
  int64_t launches = 0;
  if (X.launch) {
    if (p->prof_start) CUDA_TRY(cudaEventRecord(p->prof_start, s));
    if (X.a.warp_form) fused_kernel<true><<<(unsigned)X.grid, kFusedThreads, 0, s>>>(X.a);
    else fused_kernel<false><<<(unsigned)X.grid, kFusedThreads, 0, s>>>(X.a);
    if (cudaPeekAtLastError() != cudaSuccess) A.sched_clean = false;
    after_launch(p);
    p->last_grid = X.grid;
    ++launches;
    if (p->prof_stop) CUDA_TRY(cudaEventRecord(p->prof_stop, s));
  }
  static tp_cost_tensors none{};
  return finish_execute(p, out ? out : &none, s, X, launches);
}

}  // extern "C"

namespace {
// Per-device staging of batched launches: the plans' kernel arguments and the
// unit / item / table prefix sums go up in one pinned copy per launch.
struct BatchCtx {
  std::mutex mu;
  std::mutex host_mu;  // the one-shot host batch: output staging below
  DevBuf d_args, d_hdr, d_err;
  DevBuf out[6];
  unsigned long long* h_err = nullptr;
  size_t h_err_cap = 0;
  void* h_stage = nullptr;
  size_t h_cap = 0;
  cudaEvent_t copied = nullptr;  // the last staging copy
  bool hdr_clean = false;
  int resident = 0, resident_wide = 0;
  // arenas of the one-shot host batch, by position: scenario i of a batch
  // always gets arena i, so a repeated sweep finds its buffers sized (no
  // cudaMalloc / cudaFree, which would synchronise the device)
  std::vector<Arena*> host_arenas;
  // batched uploads: every plan's descriptor pack + the set-up jobs, one copy
  void* h_pack = nullptr;
  size_t h_pack_cap = 0;
  DevBuf d_pack;
};
BatchCtx g_batch[64];

// Everything a plan's class pairs are priced from, except the bandwidths:
// equal for two plans of one graph and mesh under different intra/inter
// bandwidths (a sweep's ratio axis).
uint64_t struct_hash_raw(const tp_plan* p) {
  uint64_t h = hash_words(0x7f4a7c159e3779b9ull ^ (uint64_t)p->env.local, &p->total_pairs, sizeof(p->total_pairs));
  h = hash_words(h, p->sigs.data(), p->sigs.size() * sizeof(SigDesc));
  h = hash_words(h, p->side_jobs.data(), p->side_jobs.size() * sizeof(SideJob));
  h = hash_words(h, p->maps.data(), p->maps.size() * sizeof(int32_t));
  h = hash_words(h, p->tabs.data(), p->tabs.size() * sizeof(TableDesc));
  h = hash_words(h, p->overrides.data(), p->overrides.size() * sizeof(double));
  return h;
}

uint64_t struct_hash(tp_plan* p) {
  if (!p->shash_ok) {
    p->shash = struct_hash_raw(p);
    p->shash_ok = true;
  }
  return p->shash;
}

template <typename T>
bool same_vec(const std::vector<T>& a, const std::vector<T>& b) {
  return a.size() == b.size() && (a.empty() || !std::memcmp(a.data(), b.data(), sizeof(T) * a.size()));
}

bool same_structure(const tp_plan* a, const tp_plan* b) {
  return a->env.local == b->env.local && a->n_log2 == b->n_log2 && a->total_pairs == b->total_pairs &&
         a->pair_form == b->pair_form && same_vec(a->sigs, b->sigs) && same_vec(a->side_jobs, b->side_jobs) &&
         same_vec(a->maps, b->maps) && same_vec(a->tabs, b->tabs) && same_vec(a->pair_sig, b->pair_sig) &&
         same_vec(a->overrides, b->overrides);
}

// err_dev: optional device array [n] that receives every launched plan's
// error slot (in `live` order via live_out) -- the host batch checks all
// plans with one copy instead of one synchronising read per plan.
tp_status execute_batch_impl(tp_plan* const* plans, int32_t n, tp_cost_tensors* device_outs, void* stream,
                             unsigned long long* err_dev, std::vector<int>* live_out) {
  if (n < 0 || (n > 0 && (!plans || !device_outs))) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null batch arrays");
  if (n == 0) return TP_OK;
  for (int i = 0; i < n; ++i)
    if (!plans[i]) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null plan in batch");
  const int device = plans[0]->device;
  for (int i = 1; i < n; ++i)
    if (plans[i]->device != device) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "batch plans on different devices");
  if (device < 0 || device >= 64) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "device ordinal out of range");
  CUDA_TRY(cudaSetDevice(device));
  tp_status st = ensure_stream(plans[0]);
  if (st) return st;
  cudaStream_t s = stream ? (cudaStream_t)stream : plans[0]->arena->stream;
  BatchCtx& B = g_batch[device];
  std::lock_guard<std::mutex> lk(B.mu);
  std::vector<ExecPrep> X(n);
  std::vector<int> live;
  int64_t batch_pairs = 0;
  for (int i = 0; i < n; ++i) batch_pairs += plans[i]->total_pairs;
  for (int i = 0; i < n; ++i) plans[i]->in_big_batch = batch_pairs > kWarpPairLimit;
  for (int i = 0; i < n; ++i) {
    tp_plan* p = plans[i];
    st = ensure_stream(p);
    if (st) return st;
    if (!p->uploaded) {
      st = tp_plan_upload(p, s);
      if (st) return st;
    }
    st = prepare_execute(p, nullptr, &device_outs[i], s, X[i]);
    p->in_big_batch = false;
    if (st) return st;
    if (!X[i].done && X[i].launch) live.push_back(i);
  }
  const int m = (int)live.size();
  if (m > 0) {
    if (B.resident == 0) {
      int sms = 0, per_sm = 0;
      CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_batch_kernel<0>, kFusedThreads, 0));
      B.resident = std::max(1, sms * std::max(1, per_sm));
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_batch_kernel<3>, kFusedThreads, 0));
      B.resident_wide = std::max(1, sms * std::max(1, per_sm));
    }
    int nwarp = 0;
    for (int k : live) nwarp += X[k].a.warp_form != 0;
    // bandwidth groups (thread form only): plans whose pricing inputs are
    // identical but for intra/inter bandwidth share their class pairs
    std::vector<int32_t> glist;                       // member lists, leader first (live order)
    std::vector<std::pair<int, int>> gspan(m, {-1, 0});  // per leader: (offset in glist, size)
    static const bool no_groups = getenv("TP_BATCH_NO_GROUPS") != nullptr;
    if (nwarp == 0 && !no_groups) {
      std::vector<std::vector<int32_t>> groups;             // live indices, the leader first
      std::unordered_map<uint64_t, std::vector<int>> open;  // structure hash -> group ids
      for (int k = 0; k < m; ++k) {
        tp_plan* p = plans[live[k]];
        if (p->total_pairs == 0 || !X[live[k]].edge_phase) continue;
        const uint64_t h = struct_hash(p);
        auto& og = open[h];
        if (og.empty() || groups[og.back()].size() >= (size_t)tpk::kGroupMax) {
          og.push_back((int)groups.size());
          groups.emplace_back();
        }
        groups[og.back()].push_back(k);
      }
      // verify the members against their leader in parallel; a hash
      // collision just leaves the plan pricing its own pairs
      std::vector<std::pair<int, int>> chk;  // (group, position)
      for (int gi = 0; gi < (int)groups.size(); ++gi)
        for (int q = 1; q < (int)groups[gi].size(); ++q) chk.push_back({gi, q});
      std::vector<char> ok(chk.size(), 1);
      run_pool((int)chk.size(), 0, [&](int c, int) {
        const auto& gr = groups[chk[c].first];
        ok[c] = same_structure(plans[live[gr[0]]], plans[live[gr[chk[c].second]]]);
      });
      for (size_t c = chk.size(); c-- > 0;)
        if (!ok[c]) groups[chk[c].first][chk[c].second] = -1;
      for (auto& gr : groups) gr.erase(std::remove(gr.begin(), gr.end(), -1), gr.end());
      for (const auto& g : groups) {
        if (g.size() < 2) continue;
        gspan[g[0]] = {(int)glist.size(), (int)g.size()};
        glist.insert(glist.end(), g.begin(), g.end());
        for (size_t q = 1; q < g.size(); ++q) {
          ExecPrep& x = X[live[g[q]]];
          x.a.priced_by_leader = 1;
          x.units = plans[live[g[q]]]->total_rows;
        }
      }
    }
    // staging: args[m] | unit_off[m+1] | item_off[m+1] | tab_off[m+1] | group lists
    const size_t args_b = sizeof(FusedArgs) * m, off_b = sizeof(int64_t) * (m + 1);
    const size_t total = args_b + 3 * off_b + sizeof(int32_t) * (glist.size() + 1);
    if (B.copied) CUDA_TRY(cudaEventSynchronize(B.copied));
    if (B.h_cap < total) {
      if (B.h_stage) cudaFreeHost(B.h_stage);
      B.h_stage = nullptr;
      B.h_cap = 0;
      CUDA_TRY(cudaMallocHost(&B.h_stage, total));
      B.h_cap = total;
    }
    CUDA_TRY(B.d_args.ensure(total));
    FusedArgs* ha = (FusedArgs*)B.h_stage;
    int64_t* uo = (int64_t*)((char*)B.h_stage + args_b);
    int64_t* io = uo + (m + 1);
    int64_t* to = io + (m + 1);
    int32_t* hg = (int32_t*)(to + (m + 1));
    const int32_t* dg = (const int32_t*)((const char*)B.d_args.p + args_b + 3 * off_b);
    // the heaviest plans first (their units are claimed first, so the long
    // pricing chains do not form the batch's tail): args in `ord` order, the
    // group lists translated to it
    std::vector<int> ord(m), pos(m);
    {
      std::vector<double> w(m);
      for (int k = 0; k < m; ++k) {
        const ExecPrep& x = X[live[k]];
        w[k] = (double)x.units * (gspan[k].second >= 2 ? 1.0 + 0.5 * (gspan[k].second - 1) : 1.0);
        ord[k] = k;
      }
      std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return w[a] > w[b]; });
      for (int j = 0; j < m; ++j) pos[ord[j]] = j;
    }
    for (size_t q = 0; q < glist.size(); ++q) hg[q] = pos[glist[q]];
    uo[0] = io[0] = to[0] = 0;
    for (int j = 0; j < m; ++j) {
      const int k = ord[j];
      const ExecPrep& x = X[live[k]];
      ha[j] = x.a;
      if (gspan[k].second >= 2) {
        ha[j].group = dg + gspan[k].first;
        ha[j].group_n = gspan[k].second;
      }
      uo[j + 1] = uo[j] + x.units;
      io[j + 1] = io[j] + x.items;
      to[j + 1] = to[j] + x.a.tables_len;
    }
    {  // callers map the kernel's per-plan outputs (error slots) in args order
      std::vector<int> l2(m);
      for (int j = 0; j < m; ++j) l2[j] = live[ord[j]];
      live.swap(l2);
    }
    if (uo[m] >= (1ll << 30) || io[m] >= (1ll << 30))
      return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "too many work items in one batch");
    CUDA_TRY(cudaMemcpyAsync(B.d_args.p, B.h_stage, total, cudaMemcpyHostToDevice, s));
    if (!B.copied) CUDA_TRY(cudaEventCreateWithFlags(&B.copied, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(B.copied, s));
    CUDA_TRY(B.d_hdr.ensure(sizeof(BatchHdr)));
    if (!B.hdr_clean) {
      CUDA_TRY(cudaMemsetAsync(B.d_hdr.p, 0, sizeof(BatchHdr), s));
      B.hdr_clean = true;
    }
    const int64_t blocks_needed = std::max<int64_t>(io[m], (uo[m] + 7) / 8);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(blocks_needed, B.resident));
    const FusedArgs* da = (const FusedArgs*)B.d_args.p;
    const int64_t* duo = (const int64_t*)((const char*)B.d_args.p + args_b);
    static const int wide = getenv("TP_BATCH_WIDE") ? atoi(getenv("TP_BATCH_WIDE")) : 0;  // measured: 4 CTAs/SM with spills beats 2 without
    const int form = nwarp == m ? 1 : (nwarp == 0 ? (wide ? 3 : 2) : 0);
    const dim3 gd((unsigned)std::min<int64_t>(grid, form == 3 ? B.resident_wide : B.resident)), bd(kFusedThreads);
    const int64_t* dio = duo + (m + 1);
    const int64_t* dto = duo + 2 * (m + 1);
    BatchHdr* hd = (BatchHdr*)B.d_hdr.p;
    if (form == 1) fused_batch_kernel<1><<<gd, bd, 0, s>>>(da, m, duo, dio, dto, hd, err_dev);
    else if (form == 2) fused_batch_kernel<2><<<gd, bd, 0, s>>>(da, m, duo, dio, dto, hd, err_dev);
    else if (form == 3) fused_batch_kernel<3><<<gd, bd, 0, s>>>(da, m, duo, dio, dto, hd, err_dev);
    else fused_batch_kernel<0><<<gd, bd, 0, s>>>(da, m, duo, dio, dto, hd, err_dev);
    if (cudaPeekAtLastError() != cudaSuccess) {
      B.hdr_clean = false;
      for (int k : live) plans[k]->arena->sched_clean = false;
    }
    for (int k : live) {
      after_launch(plans[k]);
      plans[k]->last_grid = grid;
    }
  }
  for (int i = 0; i < n; ++i) {
    if (X[i].done) {
      plans[i]->last_launches = 0;
      continue;
    }
    st = finish_execute(plans[i], &device_outs[i], s, X[i], X[i].launch ? 1 : 0);
    if (st) return st;
  }
  if (live_out) *live_out = live;
  return TP_OK;
}
}  // namespace

extern "C" {

tp_status tp_plan_execute_batch(tp_plan* const* plans, int32_t n, tp_cost_tensors* device_outs, void* stream) {
  return execute_batch_impl(plans, n, device_outs, stream, nullptr, nullptr);
}

tp_status tp_plan_set_bandwidth(tp_plan* p, double intra_bandwidth, double inter_bandwidth) {
  if (!p) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null plan");
  // nothing of the host analysis depends on the bandwidths (classes, layouts,
  // op sequences, volumes, ct): only the pricing tables and the kernels' Env
  p->env.intra = intra_bandwidth;
  p->env.inter = inter_bandwidth;
  p->uploaded = false;  // the next execute uploads the new pricing tables
  return TP_OK;
}

int64_t tp_plan_last_launches(const tp_plan* p) { return p ? p->last_launches : 0; }

tp_status tp_plan_set_pair_form(tp_plan* p, int32_t form) {
  if (!p || form < 0 || form > 2) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "pair form must be 0, 1 or 2");
  p->pair_form = form;
  return TP_OK;
}

tp_status tp_plan_set_profile_events(tp_plan* p, void* start_event, void* stop_event) {
  if (!p) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null plan");
  p->prof_start = (cudaEvent_t)start_event;
  p->prof_stop = (cudaEvent_t)stop_event;
  return TP_OK;
}

tp_status tp_plan_set_timeline(tp_plan* p, int32_t on) {
  if (!p) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null plan");
  p->timeline = on != 0;
  return TP_OK;
}

tp_status tp_plan_timeline(tp_plan* p, int64_t* ns_out) {
  if (!p || !ns_out) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null plan or output");
  if (!p->arena || !p->arena->d_sched.p) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "plan not executed");
  CUDA_TRY(cudaSetDevice(p->device));
  CUDA_TRY(cudaStreamSynchronize(p->last_stream));
  unsigned long long t[6];
  CUDA_TRY(cudaMemcpy(t, ((Sched*)p->arena->d_sched.p)->t, sizeof(t), cudaMemcpyDeviceToHost));
  const unsigned long long t0 = ~t[0];
  for (int k = 1; k < 6; ++k) {
    const bool is_min = k == 2 || k == 4;
    const unsigned long long v = is_min ? ~t[k] : t[k];
    ns_out[k - 1] = (t[k] == 0 || v < t0) ? -1 : (int64_t)(v - t0);
  }
  return TP_OK;
}

tp_status tp_plan_timeline_detail(tp_plan* p, int32_t section, uint32_t* out, int64_t* count) {
  if (!p || !count || section < 0 || section > 4) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "bad argument");
  if (section == 4) {  // phase-1 exit of every warp of the last launch (ns after kernel start)
    if (!p->timeline || !p->arena || !p->arena->d_prof.p)
      return set_err(TP_ERR_INVALID_ARGUMENT, 0, "timeline not recorded");
    if (!out) {
      *count = p->last_grid * (kFusedThreads / 32);
      return TP_OK;
    }
    CUDA_TRY(cudaSetDevice(p->device));
    CUDA_TRY(cudaStreamSynchronize(p->last_stream));
    unsigned long long t0 = 0;
    CUDA_TRY(cudaMemcpy(&t0, &((Sched*)p->arena->d_sched.p)->t[0], sizeof(t0), cudaMemcpyDeviceToHost));
    t0 = ~t0;
    CUDA_TRY(cudaMemcpy(out, (const unsigned*)p->arena->d_prof.p + 8 * (p->total_pairs + 1),
                        sizeof(unsigned) * *count, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < *count; ++i) out[i] -= (unsigned)t0;
    return TP_OK;
  }
  if (section == 3) {  // pricing-section clocks per class pair (warp form), 8 values each
    if (!p->timeline || !p->arena || !p->arena->d_prof.p)
      return set_err(TP_ERR_INVALID_ARGUMENT, 0, "timeline not recorded");
    if (!out) {
      *count = p->total_pairs;
      return TP_OK;
    }
    CUDA_TRY(cudaSetDevice(p->device));
    CUDA_TRY(cudaStreamSynchronize(p->last_stream));
    if (*count) CUDA_TRY(cudaMemcpy(out, p->arena->d_prof.p, sizeof(unsigned) * 8 * *count, cudaMemcpyDeviceToHost));
    return TP_OK;
  }
  if (!p->timeline || !p->arena || !p->arena->d_trace.p)
    return set_err(TP_ERR_INVALID_ARGUMENT, 0, "timeline not recorded");
  const int64_t n[3] = {p->trace_n[0], p->trace_n[1], p->trace_n[2]};
  const int width[3] = {2, 2, 3};
  const int out_width[3] = {3, 2, 3};  // pairs also get their edge class
  if (!out) {
    *count = n[section];
    return TP_OK;
  }
  if (*count != n[section]) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "timeline count differs from the plan's");
  CUDA_TRY(cudaSetDevice(p->device));
  CUDA_TRY(cudaStreamSynchronize(p->last_stream));
  unsigned long long t0 = 0;
  CUDA_TRY(cudaMemcpy(&t0, &((Sched*)p->arena->d_sched.p)->t[0], sizeof(t0), cudaMemcpyDeviceToHost));
  t0 = ~t0;
  int64_t off = 0;
  for (int k = 0; k < section; ++k) off += width[k] * n[k];
  const int w = width[section];
  std::vector<unsigned> h(w * n[section]);
  if (!h.empty())
    CUDA_TRY(cudaMemcpy(h.data(), (const unsigned*)p->arena->d_trace.p + off, sizeof(unsigned) * h.size(),
                        cudaMemcpyDeviceToHost));
  const int ow = out_width[section];
  for (int64_t i = 0; i < n[section]; ++i) {  // start after kernel start, then durations
    out[ow * i] = (uint32_t)(h[w * i] - (unsigned)t0);
    for (int k = 1; k < w; ++k) out[ow * i + k] = h[w * i + k];
    if (section == 0) out[ow * i + 2] = (uint32_t)p->pair_sig[i];
  }
  return TP_OK;
}

tp_status tp_plan_check_errors(tp_plan* p) {
  if (!p) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null plan");
  CUDA_TRY(cudaSetDevice(p->device));
  unsigned long long dev = ~0ull;
  if (p->arena && p->arena->d_sched.p && p->last_stream) {
    unsigned long long c = 0;
    if (p->last_parity >= 0) {
      CUDA_TRY(cudaMemcpyAsync(&c, &((Sched*)p->arena->d_sched.p)->err_c[p->last_parity], sizeof(c),
                               cudaMemcpyDeviceToHost, p->last_stream));
    }
    CUDA_TRY(cudaStreamSynchronize(p->last_stream));
    dev = ~c;  // Sched::err_c holds the complement of the smallest key
  }
  const uint64_t key = std::min<uint64_t>(dev, p->host_err);
  if (key == ~0ull) return TP_OK;
  const int kind = (int)(key & 63);
  return set_err(status_of_kind(kind), kind, kind_text(kind));
}

tp_status tp_plan_execute_host(tp_plan* p, const tp_build_opts* opts, tp_aux_index* index_out,
                               tp_cost_tensors* host_out) {
  if (!p) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null plan");
  tp_status st = ensure_stream(p);
  if (st) return st;
  if (!p->uploaded) {
    st = tp_plan_upload(p, nullptr);
    if (st) return st;
  }
  int32_t e0 = opts ? opts->edge_begin : 0;
  int32_t e1 = opts ? opts->edge_end : -1;
  if (e1 < 0 || e1 > p->valid_edges) e1 = p->valid_edges;
  if (e0 < 0) e0 = 0;
  if (e0 > e1) e0 = e1;
  const int64_t ne = p->edge_base[e1] - p->edge_base[e0];
  const int64_t nr = p->row_base[e1] - p->row_base[e0];
  const int64_t nn = p->num_aux_nodes;
  tp_cost_tensors h = host_out ? *host_out : tp_cost_tensors{};
  DevBuf* b = p->arena->out;
  tp_cost_tensors d{};
  bool oom = false;
  auto dev = [&](DevBuf& buf, void* host, int64_t n, size_t el) -> void* {
    if (!host || n <= 0) return nullptr;
    if (buf.ensure((size_t)n * el) != cudaSuccess) {
      oom = true;
      return nullptr;
    }
    return buf.p;
  };
  d.node_intra_cost_s = (double*)dev(b[0], h.node_intra_cost_s, nn, 8);
  d.node_intra_volume_bytes = (double*)dev(b[1], h.node_intra_volume_bytes, nn, 8);
  d.node_memory_bytes = (double*)dev(b[2], h.node_memory_bytes, nn, 8);
  d.edge_cost_s = (double*)dev(b[3], h.edge_cost_s, ne, 8);
  d.edge_volume_bytes = (double*)dev(b[4], h.edge_volume_bytes, ne, 8);
  d.edge_memory_bytes = (double*)dev(b[5], h.edge_memory_bytes, ne, 8);
  d.aux_edge_records = dev(b[6], h.aux_edge_records, ne, 40);
  d.row_min_cost_s = (double*)dev(b[7], h.row_min_cost_s, nr, 8);
  d.row_min_volume_bytes = (double*)dev(b[8], h.row_min_volume_bytes, nr, 8);
  if (oom) return set_err(TP_ERR_CUDA, 0, "device allocation for the outputs failed");
  tp_build_opts o = opts ? *opts : tp_build_opts{0, -1, 0, -1, nullptr};
  o.stream = nullptr;
  st = tp_plan_execute(p, &o, &d);
  if (st) return st;
  cudaStream_t s = p->arena->stream;
  auto back = [&](void* hst, void* dv, int64_t n, size_t el) -> cudaError_t {
    if (!hst || !dv || n <= 0) return cudaSuccess;
    return cudaMemcpyAsync(hst, dv, (size_t)n * el, cudaMemcpyDeviceToHost, s);
  };
  cudaError_t ce = cudaSuccess;
  if (!o.skip_nodes) {
    ce = ce ? ce : back(h.node_intra_cost_s, d.node_intra_cost_s, nn, 8);
    ce = ce ? ce : back(h.node_intra_volume_bytes, d.node_intra_volume_bytes, nn, 8);
    ce = ce ? ce : back(h.node_memory_bytes, d.node_memory_bytes, nn, 8);
  }
  ce = ce ? ce : back(h.edge_cost_s, d.edge_cost_s, ne, 8);
  ce = ce ? ce : back(h.edge_volume_bytes, d.edge_volume_bytes, ne, 8);
  ce = ce ? ce : back(h.edge_memory_bytes, d.edge_memory_bytes, ne, 8);
  ce = ce ? ce : back(h.aux_edge_records, d.aux_edge_records, ne, 40);
  ce = ce ? ce : back(h.row_min_cost_s, d.row_min_cost_s, nr, 8);
  ce = ce ? ce : back(h.row_min_volume_bytes, d.row_min_volume_bytes, nr, 8);
  st = tp_plan_check_errors(p);  // synchronises the stream
  if (ce != cudaSuccess) return set_err(TP_ERR_CUDA, 0, cudaGetErrorString(ce));
  if (st) return st;
  if (index_out) tp_plan_index(p, index_out);
  return TP_OK;
}

tp_status tp_build_cost_tensors(const tp_graph_desc* graph, const tp_topology_desc* topo,
                                const tp_build_opts* opts, tp_aux_index* index_out,
                                tp_cost_tensors* host_out) {
  tp_plan* p = nullptr;
  tp_status st = tp_plan_create(graph, topo, opts ? opts->device : -1, &p);
  if (st) return st;
  p->arena = thread_arena(p->device);  // reused across one-shot calls
  p->owns_arena = p->arena == nullptr;
  st = tp_plan_execute_host(p, opts, index_out, host_out);
  tp_plan_destroy(p);
  return st;
}

tp_status tp_plan_create_batch(const tp_graph_desc* const* graphs, const tp_topology_desc* const* topos, int32_t n,
                               int32_t device, int32_t host_threads, tp_plan** plans_out, int32_t* status_out) {
  if (n < 0 || (n > 0 && (!graphs || !topos || !plans_out)))
    return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null batch arrays");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_err(TP_ERR_CUDA, 0, "no CUDA device: the engine has no CPU path");
  if (device < 0) CUDA_TRY(cudaGetDevice(&device));
  std::vector<BatchErr> errs(n);
  static const bool prof = getenv("TP_PROFILE_HOST") != nullptr;
  const auto c0 = std::chrono::steady_clock::now();
  run_pool(
      n, host_threads,
      [&](int i, int) {
    tp_plan* p = nullptr;
    const tp_status st = tp_plan_create(graphs[i], topos[i], device, &p);
    if (p) struct_hash(p);  // cached for the batch's bandwidth groups
    plans_out[i] = p;
    errs[i].take(st);
      },
      device);
  if (prof)
    fprintf(stderr, "[tp batch] %d plans created in %.0f us on %d threads\n", n,
            std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - c0).count(),
            pool_size(n, host_threads));
  return batch_status(errs, status_out);
}

}  // extern "C"

namespace {
// One execute_host per plan on the worker threads (plans on several devices).
tp_status execute_host_each(tp_plan* const* plans, int32_t n, tp_aux_index* index_outs, tp_cost_tensors* host_outs,
                            int32_t host_threads, int32_t* status_out) {
  if (n < 0 || (n > 0 && (!plans || !host_outs))) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null batch arrays");
  std::vector<BatchErr> errs(n);
  const int workers = pool_size(n, host_threads);
  int64_t batch_pairs = 0;
  for (int i = 0; i < n; ++i) batch_pairs += plans[i] ? plans[i]->total_pairs : 0;
  std::vector<Arena*> borrowed(workers, nullptr);
  std::vector<int> borrowed_dev(workers, -1);
  run_pool(n, workers, [&](int i, int w) {
    tp_plan* p = plans[i];
    if (!p) {
      errs[i].take(set_err(TP_ERR_INVALID_ARGUMENT, 0, "null plan"));
      return;
    }
    const bool borrow = p->arena == nullptr;
    if (borrow) {
      if (borrowed[w] && borrowed_dev[w] != p->device) {
        arena_pool_put(borrowed[w]);
        borrowed[w] = nullptr;
      }
      if (!borrowed[w]) {
        borrowed[w] = arena_pool_get(p->device);
        borrowed_dev[w] = p->device;
      }
      p->arena = borrowed[w];
      p->owns_arena = false;
      p->uploaded = false;
    }
    p->in_big_batch = batch_pairs > kWarpPairLimit;  // the workers' plans share the GPU
    errs[i].take(tp_plan_execute_host(p, nullptr, index_outs ? &index_outs[i] : nullptr, &host_outs[i]));
    p->in_big_batch = false;
    if (borrow) {  // the arena's descriptors belong to the next plan now
      p->arena = nullptr;
      p->owns_arena = true;
      p->uploaded = false;
      p->range_key = {{-1, -1, -1, -1}};
    }
  });
  for (Arena* a : borrowed)
    if (a) arena_pool_put(a);
  return batch_status(errs, status_out);
}


// Error status of plan p from its device error slot value (complemented key).
tp_status status_from_slot(tp_plan* p, unsigned long long c) {
  const uint64_t key = std::min<uint64_t>(~c, p->host_err);
  if (key == ~0ull) return TP_OK;
  const int kind = (int)(key & 63);
  return set_err(status_of_kind(kind), kind, kind_text(kind));
}
}  // namespace

extern "C" {

// One device: every plan's descriptors uploaded (worker threads, pooled
// arenas), ONE batched launch into staging buffers, the tensors copied back
// with one copy per tensor kind when the caller's host slices are contiguous
// (as engine.Sweep allocates them), and every plan's error read by one copy.
tp_status tp_plan_execute_host_batch(tp_plan* const* plans, int32_t n, tp_aux_index* index_outs,
                                     tp_cost_tensors* host_outs, int32_t host_threads, int32_t* status_out) {
  if (n < 0 || (n > 0 && (!plans || !host_outs))) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null batch arrays");
  if (n == 0) return TP_OK;
  bool one_device = plans[0] != nullptr;
  for (int i = 0; one_device && i < n; ++i) one_device = plans[i] && plans[i]->device == plans[0]->device;
  if (!one_device || plans[0]->device < 0 || plans[0]->device >= 64)
    return execute_host_each(plans, n, index_outs, host_outs, host_threads, status_out);
  const int device = plans[0]->device;
  CUDA_TRY(cudaSetDevice(device));
  BatchCtx& B = g_batch[device];
  std::lock_guard<std::mutex> hl(B.host_mu);
  static const bool prof = getenv("TP_PROFILE_HOST") != nullptr;
  auto clk = [] { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double hb0 = prof ? clk() : 0;
  // arenas: plans without one borrow the batch's arena of their position
  std::vector<char> borrowed(n, 0);
  while ((int)B.host_arenas.size() < n) {
    Arena* a = new Arena();
    a->device = device;
    B.host_arenas.push_back(a);
  }
  for (int i = 0; i < n; ++i) {
    tp_plan* p = plans[i];
    if (p->arena) continue;
    p->arena = B.host_arenas[i];
    p->owns_arena = false;
    p->uploaded = false;
    borrowed[i] = 1;
  }
  auto give_back = [&]() {
    for (int i = 0; i < n; ++i) {
      if (!borrowed[i]) continue;
      tp_plan* p = plans[i];
      p->arena = nullptr;
      p->owns_arena = true;
      p->uploaded = false;
      p->range_key = {{-1, -1, -1, -1}};
    }
  };
  tp_status st = ensure_stream(plans[0]);
  if (st) {
    give_back();
    return st;
  }
  cudaStream_t s = plans[0]->arena->stream;
  // uploads: plans on their own arenas the usual way; the borrowed ones in
  // ONE packed copy (descriptors packed by the workers) and two set-up launches
  std::vector<BatchErr> errs(n);
  for (int i = 0; i < n; ++i)
    if (!borrowed[i] && !plans[i]->uploaded) errs[i].take(tp_plan_upload(plans[i], s));
  std::vector<int> todo;
  for (int i = 0; i < n; ++i)
    if (borrowed[i]) todo.push_back(i);
  std::vector<UploadPrep> U(todo.size());
  run_pool((int)todo.size(), host_threads, [&](int j, int) { errs[todo[j]].take(upload_prepare(plans[todo[j]], U[j])); },
           device);
  for (int i = 0; i < n; ++i)
    if (errs[i].st) {
      give_back();
      return batch_status(errs, status_out);
    }
  if (!todo.empty()) {
    const int m = (int)todo.size();
    std::vector<size_t> off(m + 1, 0);
    for (int j = 0; j < m; ++j) off[j + 1] = off[j] + U[j].pk.total();
    const size_t jobs_at = (off[m] + 255) & ~(size_t)255;
    const size_t total = jobs_at + sizeof(UpJob) * m + 2 * sizeof(int64_t) * (m + 1);
    if (B.h_pack_cap < total) {
      if (B.h_pack) cudaFreeHost(B.h_pack);
      B.h_pack = nullptr;
      B.h_pack_cap = 0;
      CUDA_TRY(cudaMallocHost(&B.h_pack, total));
      B.h_pack_cap = total;
    }
    CUDA_TRY(B.d_pack.ensure(total));
    char* hp = (char*)B.h_pack;
    char* dp = (char*)B.d_pack.p;
    run_pool(
        m, host_threads,
        [&](int j, int) {
          tp_plan* p = plans[todo[j]];
          upload_stage(U[j], hp + off[j], dp + off[j]);
          errs[todo[j]].take(upload_finish(p, U[j]));
        },
        device);
    for (int i = 0; i < n; ++i)
      if (errs[i].st) {
        give_back();
        return batch_status(errs, status_out);
      }
    UpJob* jobs = (UpJob*)(hp + jobs_at);
    int64_t* so = (int64_t*)(hp + jobs_at + sizeof(UpJob) * m);
    int64_t* po = so + (m + 1);
    so[0] = po[0] = 0;
    for (int j = 0; j < m; ++j) {
      tp_plan* p = plans[todo[j]];
      Arena& A = *p->arena;
      jobs[j] = UpJob{(const SideJob*)A.d_sidejobs.p, (const Strat*)A.d_tables.p, (tpk::SideDesc*)A.d_sides.p,
                      (const SigDesc*)A.d_sigs.p, (const int32_t*)A.d_pairsigs.p, (const int32_t*)A.d_maps.p,
                      (const double*)A.d_over.p, (PairRec*)A.d_pairrec.p, (int32_t)p->side_jobs.size(), 0};
      so[j + 1] = so[j] + p->side_total;
      po[j + 1] = po[j] + p->total_pairs;
    }
    CUDA_TRY(cudaMemcpyAsync(dp, hp, total, cudaMemcpyHostToDevice, s));
    for (int j = 0; j < m; ++j) {
      st = upload_tables(plans[todo[j]], U[j], s);
      if (st) {
        give_back();
        return st;
      }
    }
    const UpJob* dj = (const UpJob*)(dp + jobs_at);
    const int64_t* dso = (const int64_t*)(dp + jobs_at + sizeof(UpJob) * m);
    if (so[m] > 0) batch_side_kernel<<<(unsigned)((so[m] + 127) / 128), 128, 0, s>>>(dj, m, dso);
    if (po[m] > 0) batch_pair_rec_kernel<<<(unsigned)((po[m] + 127) / 128), 128, 0, s>>>(dj, m, dso + (m + 1));
    CUDA_TRY(cudaGetLastError());
  }
  const double hb1 = prof ? clk() : 0;
  // device staging of the outputs, one buffer per tensor kind
  std::vector<int64_t> nn(n), ne(n);
  int64_t tn = 0, te = 0;
  for (int i = 0; i < n; ++i) {
    nn[i] = plans[i]->num_aux_nodes;
    ne[i] = plans[i]->edge_base[plans[i]->valid_edges] - plans[i]->edge_base[0];
    tn += nn[i];
    te += ne[i];
  }
  double* h_of[6];
  auto host_ptr = [&](int i, int k) -> double* {
    const tp_cost_tensors& h = host_outs[i];
    double* const v[6] = {h.node_intra_cost_s, h.node_intra_volume_bytes, h.node_memory_bytes,
                          h.edge_cost_s,       h.edge_volume_bytes,       h.edge_memory_bytes};
    return v[k];
  };
  std::vector<tp_cost_tensors> dev(n);
  bool want[6];
  for (int k = 0; k < 6; ++k) {
    want[k] = false;
    for (int i = 0; i < n; ++i) want[k] |= host_ptr(i, k) != nullptr;
    const int64_t tot = k < 3 ? tn : te;
    if (want[k]) CUDA_TRY(B.out[k].ensure(sizeof(double) * (size_t)std::max<int64_t>(tot, 1)));
    h_of[k] = (double*)B.out[k].p;
  }
  {
    int64_t on = 0, oe = 0;
    for (int i = 0; i < n; ++i) {
      double* d[6];
      for (int k = 0; k < 6; ++k) d[k] = want[k] && host_ptr(i, k) ? h_of[k] + (k < 3 ? on : oe) : nullptr;
      dev[i] = tp_cost_tensors{d[0], d[1], d[2], d[3], d[4], d[5], nullptr, nullptr, nullptr};
      on += nn[i];
      oe += ne[i];
    }
  }
  CUDA_TRY(B.d_err.ensure(sizeof(unsigned long long) * n));
  std::vector<int> live;
  st = execute_batch_impl(plans, n, dev.data(), s, (unsigned long long*)B.d_err.p, &live);
  if (st) {
    give_back();
    return st;
  }
  const double hb2 = prof ? clk() : 0;
  // back to the host: one copy per tensor kind where the caller's slices are contiguous
  for (int k = 0; k < 6; ++k) {
    if (!want[k]) continue;
    bool contiguous = true;
    for (int i = 0; contiguous && i < n; ++i) {
      contiguous = host_ptr(i, k) != nullptr;
      if (contiguous && i + 1 < n) contiguous = host_ptr(i + 1, k) == host_ptr(i, k) + (k < 3 ? nn[i] : ne[i]);
    }
    const int64_t tot = k < 3 ? tn : te;
    if (contiguous) {
      if (tot > 0) CUDA_TRY(cudaMemcpyAsync(host_ptr(0, k), h_of[k], sizeof(double) * tot, cudaMemcpyDeviceToHost, s));
      continue;
    }
    int64_t off = 0;
    for (int i = 0; i < n; ++i) {
      const int64_t c = k < 3 ? nn[i] : ne[i];
      if (host_ptr(i, k) && c > 0)
        CUDA_TRY(cudaMemcpyAsync(host_ptr(i, k), h_of[k] + off, sizeof(double) * c, cudaMemcpyDeviceToHost, s));
      off += c;
    }
  }
  if (B.h_err_cap < (size_t)n) {
    if (B.h_err) cudaFreeHost(B.h_err);
    B.h_err = nullptr;
    B.h_err_cap = 0;
    CUDA_TRY(cudaMallocHost(&B.h_err, sizeof(unsigned long long) * n));
    B.h_err_cap = n;
  }
  if (!live.empty())
    CUDA_TRY(cudaMemcpyAsync(B.h_err, B.d_err.p, sizeof(unsigned long long) * live.size(), cudaMemcpyDeviceToHost, s));
  const double hb3 = prof ? clk() : 0;
  CUDA_TRY(cudaStreamSynchronize(s));
  if (prof)
    fprintf(stderr, "[tp batch] %d plans: uploads %.0f us, launch prep %.0f, copies enqueued %.0f, wait %.0f\n", n,
            hb1 - hb0, hb2 - hb1, hb3 - hb2, clk() - hb3);
  std::vector<unsigned long long> slot(n, 0);
  for (size_t k = 0; k < live.size(); ++k) slot[live[k]] = B.h_err[k];
  for (int i = 0; i < n; ++i) {
    errs[i].take(status_from_slot(plans[i], slot[i]));
    if (index_outs) tp_plan_index(plans[i], &index_outs[i]);
  }
  give_back();
  return batch_status(errs, status_out);
}

tp_status tp_plan_price_assignments(tp_plan* p, const tp_cost_tensors* t, const int32_t* assignments, int32_t k,
                                    double* cost_s, double* volume_bytes, double* memory_bytes, void* stream) {
  if (!p || !t || (k > 0 && !assignments)) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null argument");
  if (k < 0) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "negative assignment count");
  if (p->host_err != ~0ull) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "the plan's build has an error");
  if (!t->node_intra_cost_s || !t->node_intra_volume_bytes || !t->node_memory_bytes || !t->edge_cost_s ||
      !t->edge_volume_bytes || !t->edge_memory_bytes)
    return set_err(TP_ERR_INVALID_ARGUMENT, 0, "all six cost tensors are needed");
  if (k == 0 || p->num_ops == 0) return TP_OK;
  tp_status st = ensure_stream(p);
  if (st) return st;
  cudaStream_t s = stream ? (cudaStream_t)stream : p->arena->stream;
  if (!p->d_terms) {  // the summation terms and the index arrays they read, once per plan
    p->price_terms.clear();
    // edges by the dense id of their `to`, ascending edge order
    int32_t nd = 0;
    for (int v : p->op_dense_id) nd = std::max(nd, v + 1);
    for (int v : p->edge_to_dense) nd = std::max(nd, v + 1);
    std::vector<int32_t> db(nd + 1, 0), de(p->num_edges);
    for (int e = 0; e < p->num_edges; ++e) ++db[p->edge_to_dense[e] + 1];
    for (int d = 0; d < nd; ++d) db[d + 1] += db[d];
    {
      std::vector<int32_t> f(db.begin(), db.end() - 1);
      for (int e = 0; e < p->num_edges; ++e) de[f[p->edge_to_dense[e]]++] = e;
    }
    for (int op : p->topo) {
      if (p->in_deg[op] == 0) p->price_terms.push_back(make_int4(0, -1, -1, op));
      const int d = p->op_dense_id[op];
      for (int q = db[d]; q < db[d + 1]; ++q) {
        const int e = de[q];
        p->price_terms.push_back(make_int4(1, e, p->edge_from_op[e], op));
      }
    }
    std::vector<int64_t> idx64;
    idx64.insert(idx64.end(), p->node_base.begin(), p->node_base.end());
    idx64.insert(idx64.end(), p->edge_base.begin(), p->edge_base.end());
    const size_t b_terms = sizeof(int4) * std::max<size_t>(p->price_terms.size(), 1);
    const size_t b_idx = sizeof(int64_t) * idx64.size();
    const size_t b_to = sizeof(int32_t) * std::max<int>(p->num_edges, 1);
    p->d_terms = new DevBuf();
    CUDA_TRY(p->d_terms->ensure(b_terms + b_idx + b_to));
    char* base = (char*)p->d_terms->p;
    CUDA_TRY(cudaMemcpyAsync(base, p->price_terms.data(), sizeof(int4) * p->price_terms.size(),
                             cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(base + b_terms, idx64.data(), b_idx, cudaMemcpyHostToDevice, s));
    if (p->num_edges)
      CUDA_TRY(cudaMemcpyAsync(base + b_terms + b_idx, p->edge_to_op.data(), sizeof(int32_t) * p->num_edges,
                               cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaStreamSynchronize(s));  // the host vectors above are pageable and temporary
    p->terms_bytes = (int64_t)b_terms;
  }
  const char* base = (const char*)p->d_terms->p;
  const int4* terms = (const int4*)base;
  const int64_t* nb = (const int64_t*)(base + p->terms_bytes);
  const int64_t* eb = nb + (p->num_ops + 1);
  const int32_t* to = (const int32_t*)(eb + (p->num_edges + 1));
  const int blocks = (k + kPriceWarps - 1) / kPriceWarps;
  price_kernel<<<blocks, 32 * kPriceWarps, 0, s>>>(terms, (int)p->price_terms.size(), nb, eb, to, assignments,
                                                   p->num_ops, k, t->node_intra_cost_s, t->node_intra_volume_bytes,
                                                   t->node_memory_bytes, t->edge_cost_s, t->edge_volume_bytes,
                                                   t->edge_memory_bytes, cost_s, volume_bytes, memory_bytes);
  CUDA_TRY(cudaGetLastError());
  return TP_OK;
}

tp_status tp_enumerate_strategies(int32_t p, int64_t total_devices, int64_t* count, int64_t* degrees,
                                  int32_t* device_map, int64_t* matrix_dims, int32_t* matrix_depth) {
  if (p < 1) return set_err(TP_ERR_TOPOPLAN, tpk::kNoAxes, "strategy_count: axis count must be >= 1");
  if (total_devices <= 0 || (total_devices & (total_devices - 1)))
    return set_err(TP_ERR_TOPOPLAN, tpk::kNotPow2, "device count is not a power of two");
  if (p > tpk::kMaxAxes) return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "more than 8 axes");
  const int n = log2_floor(total_devices);
  if (n > tpk::kMaxD) return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "more than 2^16 devices");
  const int64_t S = tpk::strategy_count(p, n);
  if (count) *count = S;
  if (!degrees && !device_map && !matrix_dims && !matrix_depth) return TP_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_err(TP_ERR_CUDA, 0, "no CUDA device: the engine has no CPU path");
  TableDesc td{0, S, p, n};
  DevBuf dt, dout;
  CUDA_TRY(dt.ensure(sizeof(td)));
  CUDA_TRY(dout.ensure(sizeof(Strat) * S));
  CUDA_TRY(cudaMemcpy(dt.p, &td, sizeof(td), cudaMemcpyHostToDevice));
  table_kernel<<<(unsigned)((S + 127) / 128), 128>>>((const TableDesc*)dt.p, 1, S, (Strat*)dout.p);
  std::vector<Strat> h(S);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpy(h.data(), dout.p, sizeof(Strat) * S, cudaMemcpyDeviceToHost));
  dt.release();
  dout.release();
  for (int64_t i = 0; i < S; ++i) {
    for (int a = 0; a < p; ++a) {
      if (degrees) degrees[i * p + a] = (int64_t)1 << h[i].deg[a];
      if (device_map) device_map[i * p + a] = h[i].dmap[a];
      // DeviceMatrix::dims, outermost first: dims[j] = extent(depth-1-j)
      if (matrix_dims)
        matrix_dims[i * p + a] = a < h[i].depth ? ((int64_t)1 << h[i].mx[h[i].depth - 1 - a]) : 0;
    }
    if (matrix_depth) matrix_depth[i] = h[i].depth;
  }
  return TP_OK;
}

tp_status tp_redistribute_batch(const tp_redist_query* q, int32_t n, tp_redist_result* r) {
  return tp_redistribute_batch_form(q, n, r, 2);
}

tp_status tp_redistribute_batch_form(const tp_redist_query* q, int32_t n, tp_redist_result* r, int32_t form) {
  if (n <= 0) return TP_OK;
  if (!q || !r) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null argument");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_err(TP_ERR_CUDA, 0, "no CUDA device: the engine has no CPU path");
  std::vector<tpk::QueryPOD> pod(n);
  for (int i = 0; i < n; ++i) {
    tpk::QueryPOD& x = pod[i];
    std::memset(&x, 0, sizeof(x));
    x.rank = q[i].rank;
    x.fdepth = q[i].from_depth;
    x.tdepth = q[i].to_depth;
    x.local = q[i].local_device_num;
    x.bytes = q[i].tensor_bytes;
    x.intra = q[i].intra_bandwidth;
    x.inter = q[i].inter_bandwidth;
    if (x.rank > tpk::kMaxR || x.fdepth > tpk::kMaxD || x.tdepth > tpk::kMaxD || x.rank < 0) {
      x.rank = tpk::kMaxR + 1;  // flagged as capacity by the kernel
      continue;
    }
    for (int d = 0; d < x.rank; ++d) {
      x.shape[d] = q[i].shape[d];
      x.fmap[d] = q[i].from_map[d];
      x.tmap[d] = q[i].to_map[d];
    }
    for (int k = 0; k < x.fdepth; ++k) x.fdims[k] = q[i].from_dims[k];
    for (int k = 0; k < x.tdepth; ++k) x.tdims[k] = q[i].to_dims[k];
  }
  // per-query pricing tables, exactly as a plan builds them
  constexpr int kTab = tpk::kBwTab + tpk::kScaleDim * tpk::kScaleDim;
  std::vector<double> tabs((size_t)n * kTab);
  for (int i = 0; i < n; ++i)
    tpk::make_price_tabs(Env{pod[i].intra, pod[i].inter, (int64_t)pod[i].local}, &tabs[(size_t)i * kTab],
                         &tabs[(size_t)i * kTab + tpk::kBwTab]);
  DevBuf dq, dr, dtr, dtab;
  CUDA_TRY(dq.ensure(sizeof(tpk::QueryPOD) * n));
  CUDA_TRY(dr.ensure(sizeof(tp_redist_result) * n));
  CUDA_TRY(dtab.ensure(sizeof(double) * tabs.size()));
  CUDA_TRY(cudaMemcpy(dq.p, pod.data(), sizeof(tpk::QueryPOD) * n, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dtab.p, tabs.data(), sizeof(double) * tabs.size(), cudaMemcpyHostToDevice));
  if (form == 1) {
    CUDA_TRY(dtr.ensure(sizeof(tpk::Trace) * n));
    query_kernel_warp<<<(n + 3) / 4, 128>>>((const tpk::QueryPOD*)dq.p, n, (tp_redist_result*)dr.p,
                                             (tpk::Trace*)dtr.p, (const double*)dtab.p);
  } else {
    query_kernel<<<(n + 63) / 64, 64>>>((const tpk::QueryPOD*)dq.p, n, (tp_redist_result*)dr.p,
                                        (const double*)dtab.p);
  }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpy(r, dr.p, sizeof(tp_redist_result) * n, cudaMemcpyDeviceToHost));
  dq.release();
  dr.release();
  dtr.release();
  dtab.release();
  return TP_OK;
}

}  // extern "C"
