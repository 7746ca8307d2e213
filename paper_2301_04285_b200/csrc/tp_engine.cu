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
#include <cmath>
#include <array>
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

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
  int32_t pad;
  int8_t sa_u[tpk::kMaxR];
  int8_t sa_w[tpk::kMaxR];
  DimT dt[tpk::kMaxR];
};

struct EdgeDesc {
  int64_t aux_base;    // aux id of the edge's (0, 0)
  int64_t nb_u, nb_w;  // first aux node of the producer / consumer
  int64_t wrow;        // class row of the consumer's strategy 0
  int32_t sig, e;
};

struct Work {
  int32_t sig;
  int32_t ebeg, eend;  // into the per-execute FanEdge list
  int32_t j0;          // first pair of the tile within the class block
};

struct FanEdge {       // one graph edge of an execute's range
  int64_t out_base;    // output index of its pair (0, 0)
  int64_t wrow;        // class row of the consumer's strategy 0
  int64_t nb_u, nb_w;  // first aux node of producer / consumer (records)
  int32_t e, pad;
};

struct NodeWork {      // fan-out of one node class's rows to a chunk of its members
  int32_t cls;
  int32_t mbeg, mend;
  int32_t pad;
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
constexpr int kExpPer = 4;
constexpr int kExpTile = 256 * kExpPer;  // class pairs per fan-out tile
constexpr int kMaxChunk = 64;            // edges per fan-out tile

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
__global__ void side_kernel(const SideJob* __restrict__ jobs, int njobs, int64_t total,
                            const Strat* __restrict__ tables, tpk::SideDesc* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
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

// Per-execute scheduling state, zeroed by one memset before the launch.
struct Sched {
  unsigned long long err_c;  // ~(smallest error key); 0 = no error
  int head;                  // next block work item (node rows, then fan-out)
  int pair_head;             // next class pair (warp form) / pair chunk (thread form)
  int node_done;             // node-class rows finished
  int pad;
  int pairs_done[2];         // per edge class (allocated to the class count)
};

__device__ __forceinline__ void flag_error(Sched* s, uint64_t key) {
  atomicMax(&s->err_c, ~(unsigned long long)key);  // max of ~key = min of key
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct FusedArgs {
  // node classes
  const ClassDesc* classes;
  int ncls;
  int64_t total_rows;
  const SliceChk* chks;
  const SlotDesc* slots;
  const Occ* occs;
  double* cls_sec;
  double* cls_vol;
  double* cls_mem;
  double* cls_memdiv;
  // edge classes
  const SigDesc* sigs;
  int nsigs;
  const int32_t* pair_sigs;
  int npair_sigs;
  int64_t total_pairs;
  const double* overrides;
  const tpk::SideDesc* sides;
  double* r_sec;
  double* r_vol;
  // fan-out
  const Work* work;
  const FanEdge* fan;
  double* e_sec;
  double* e_vol;
  double* e_mem;
  char* records;
  int general_store;  // records requested or not all three SoA tensors given
  const NodeWork* nwork;
  const int64_t* member_nb;
  double* n_sec;
  double* n_vol;
  double* n_mem;
  // work-item ranges: [0, i_pair) node rows, [i_pair, i_exp) pairs,
  // [i_exp, i_nfan) fan-out tiles, [i_nfan, i_end) node fan-out
  int i_pair, i_exp, i_nfan, i_end;
  int warp_form;  // pairs: 1 = warp per pair, 0 = thread per pair
  // shared
  const Strat* tables;
  Env env;
  int l_log2;
  int n_log2;
  const double* bw_tab;     // inter/ct, tpk::kBwTab entries
  const double* scale_tab;  // AllToAll scale, kScaleDim^2 entries
  Sched* sched;
};

constexpr int kFusedThreads = 256;
constexpr int kWarpPairsPerItem = kFusedThreads / 32;

// One aux-node row of a node class (aux_graph.hpp:120-167).
__device__ void node_row(const FusedArgs& a, int64_t row) {
  int lo = 0, hi = a.ncls - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.classes[mid].row_base <= row) lo = mid; else hi = mid - 1;
  }
  const ClassDesc cd = a.classes[lo];
  const int64_t s = row - cd.row_base;
  const Strat st = a.tables[cd.table + s];
  // layout.hpp:349-367: every slice in axis order must divide its extent
  for (int c = cd.chk_begin; c < cd.chk_end; ++c) {
    const SliceChk k = a.chks[c];
    int kind = 0;
    if (k.slot < 0) kind = tpk::kUnknownSliceTensor;
    else if (st.deg[k.axis] > k.v) kind = tpk::kIndivisible;
    if (kind) {
      flag_error(a.sched, ekey(1 + (uint64_t)(cd.first_node + s) * 2 + 1, kind));
      a.cls_sec[row] = a.cls_vol[row] = a.cls_mem[row] = a.cls_memdiv[row] = 0;
      return;
    }
  }
  double sec = 0, vol = 0, mem = 0;
  for (int q = cd.occ_begin; q < cd.occ_end; ++q) {
    const Occ oc = a.occs[q];
    const SlotDesc sd = a.slots[cd.slot_begin + oc.slot];
    int sdiv = 0;
    for (int d = 0; d < sd.R; ++d)
      if (sd.sa[d] >= 0) sdiv += st.deg[sd.sa[d]];
    const int64_t shard_el = sdiv >= 63 ? 0 : (sd.elements >> sdiv);
    const double sb = (double)shard_el * sd.es;  // layout.hpp:125-129
    if (oc.in_memory) mem += sb;                 // aux_graph.hpp:151-167
    int glog = 0;
    for (int ax = 0; ax < cd.p; ++ax)
      if ((oc.nonslicing >> ax) & 1) glog += st.deg[ax];
    if (glog == 0) continue;  // group <= 1
    // infer_ct_allreduce (cost_model.hpp:75-97)
    const int64_t pd = sdiv > a.n_log2 ? 0 : ((int64_t)1 << (a.n_log2 - sdiv));
    int64_t remain = a.env.local, dev_in = 1;
    for (int k = 0; k < st.depth; ++k) {
      bool contains = false;
      for (int d = 0; d < sd.R; ++d) contains |= sd.sa[d] >= 0 && st.dmap[sd.sa[d]] == k;
      const int64_t ek = (int64_t)1 << st.mx[k];
      if (!contains && remain > 1) dev_in *= remain > ek ? ek : remain;
      remain /= ek;
    }
    const int64_t ct = dev_in >= pd ? 0 : (dev_in > 1 ? a.env.local / dev_in : a.env.local);
    const double n = (double)((int64_t)1 << glog);
    const double v = 2.0 * (n - 1) / n * sb;  // allreduce_volume, cost_model.hpp:39-43
    vol += v;
    sec += v / tpk::eff_bw(ct, a.env);
  }
  a.cls_sec[row] = sec;
  a.cls_vol[row] = vol;
  a.cls_mem[row] = mem;
  a.cls_memdiv[row] = mem / cd.indeg;  // aux_graph.hpp:292
}

__device__ __forceinline__ int sig_of_pair(const FusedArgs& a, int64_t idx) {
  int lo = 0, hi = a.npair_sigs - 1;  // classes that own a table, by pair_begin
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.sigs[a.pair_sigs[mid]].pair_begin <= idx) lo = mid; else hi = mid - 1;
  }
  return a.pair_sigs[lo];
}

// One (edge class, su, sw) pair on one thread (register form, tp_fast.cuh).
__device__ void pair_thread(const FusedArgs& a, int64_t idx, int sig) {
  const SigDesc& sg = a.sigs[sig];
  const int32_t local = (int32_t)(idx - sg.pair_begin);
  const int32_t su = local / sg.Sw, sw = local - su * sg.Sw;
  const tpk::SideDesc F = a.sides[sg.side_u + su];
  const tpk::SideDesc T = a.sides[sg.side_w + sw];
  double sec = 0, vol = 0;
  if (!tpk::same_side(F, T, sg.R)) {  // aux_graph.hpp:260
    const double bytes = sg.has_override ? a.overrides[idx] : sg.bytes;
    const int st = tpk::pair_cost_sd(sg.R, F, T, nullptr, nullptr, sg.dt, bytes, a.env, a.l_log2,
                                     tpk::FastTabs{a.bw_tab, a.scale_tab}, sec, vol, nullptr);
    if (st) {
      flag_error(a.sched, ekey(kEdgePhase + (uint64_t)(sg.first_aux + local) * 2 + 1, st));
      sec = vol = 0;
    }
  }
  a.r_sec[idx] = sec;
  a.r_vol[idx] = vol;
}

// One pair on one warp (warp form, tp_warp.cuh); lane 0 writes.
__device__ void pair_warp(const FusedArgs& a, int64_t idx, int sig) {
  const SigDesc& sg = a.sigs[sig];
  const int32_t local = (int32_t)(idx - sg.pair_begin);
  const int32_t su = local / sg.Sw, sw = local - su * sg.Sw;
  const tpk::SideDesc* F = a.sides + sg.side_u + su;
  const tpk::SideDesc* T = a.sides + sg.side_w + sw;
  double sec = 0, vol = 0;
  if (!tpk::same_side(*F, *T, sg.R)) {  // aux_graph.hpp:260
    const double bytes = sg.has_override ? a.overrides[idx] : sg.bytes;
    tpk::WarpEnv we;
    we.env = a.env;
    we.l_log2 = a.l_log2;
    we.tab = tpk::PriceTabs{a.bw_tab, a.scale_tab};
    const int st = tpk::redist_cost_warp(sg.R, F, T, sg.dt, bytes, we, sec, vol, nullptr);
    if (st) {
      if ((threadIdx.x & 31) == 0) flag_error(a.sched, ekey(kEdgePhase + (uint64_t)(sg.first_aux + local) * 2 + 1, st));
      sec = vol = 0;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    a.r_sec[idx] = sec;
    a.r_vol[idx] = vol;
  }
}

// Fan-out tile: every edge of a chunk of one edge class gets the class
// tile's values at out_base(edge) + pair, lane-contiguous (256-B warp
// stores); class rows are reloaded only when the consumer class changes
// (edges are sorted by it).
__device__ void fanout_tile(const FusedArgs& a, const Work& wk, FanEdge* sedge) {
  const int nE = wk.eend - wk.ebeg;
  for (int t = threadIdx.x; t < nE; t += kFusedThreads) sedge[t] = a.fan[wk.ebeg + t];
  const SigDesc& sg = a.sigs[wk.sig];
  const int32_t Sw = sg.Sw;
  const int32_t P = sg.Su * Sw;
  const int64_t pb = sg.pair_begin;
  const double f = sg.scale;  // 1, or the exact factor of a derived class
  if (threadIdx.x == 0) {  // wait for the class table and the node rows
    while (ld_acquire(&a.sched->pairs_done[sg.base]) < P) __nanosleep(64);
    while (ld_acquire(&a.sched->node_done) < a.total_rows) __nanosleep(64);
  }
  __syncthreads();
  const int32_t step = kFusedThreads % Sw;
  int32_t jj[kExpPer], sw[kExpPer];
  double rs[kExpPer], rv[kExpPer];
  int32_t cur = (wk.j0 + (int32_t)threadIdx.x) % Sw;
#pragma unroll
  for (int k = 0; k < kExpPer; ++k) {
    const int32_t j = wk.j0 + (int32_t)threadIdx.x + k * kFusedThreads;
    jj[k] = j < P ? j : -1;
    sw[k] = cur;
    cur += step;
    if (cur >= Sw) cur -= Sw;
    const int64_t jc = j < P ? j : 0;
    rs[k] = __ldcg(a.r_sec + pb + jc) * f;  // L2: written by other SMs in this launch
    rv[k] = __ldcg(a.r_vol + pb + jc) * f;
  }
  double c[kExpPer], v[kExpPer], m[kExpPer];
  int64_t cur_row = -1;
  for (int ei = 0; ei < nE; ++ei) {
    const int64_t base = sedge[ei].out_base;
    const int64_t wrow = sedge[ei].wrow;
    if (wrow != cur_row) {  // block-uniform
      cur_row = wrow;
#pragma unroll
      for (int k = 0; k < kExpPer; ++k) {
        c[k] = __ldcg(a.cls_sec + wrow + sw[k]) + rs[k];  // aux_graph.hpp:290-291
        v[k] = __ldcg(a.cls_vol + wrow + sw[k]) + rv[k];
        m[k] = __ldcg(a.cls_memdiv + wrow + sw[k]);       // :292
      }
    }
    if (!a.general_store) {
#pragma unroll
      for (int k = 0; k < kExpPer; ++k) {
        if (jj[k] < 0) continue;
        const int64_t o = base + jj[k];
        __stcs(a.e_sec + o, c[k]);  // streaming: written once, read by the host
        __stcs(a.e_vol + o, v[k]);
        __stcs(a.e_mem + o, m[k]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < kExpPer; ++k) {
        if (jj[k] < 0) continue;
        const int64_t o = base + jj[k];
        if (a.e_sec) __stcs(a.e_sec + o, c[k]);
        if (a.e_vol) __stcs(a.e_vol + o, v[k]);
        if (a.e_mem) __stcs(a.e_mem + o, m[k]);
        if (!a.records) continue;
        // topoplan::AuxEdge, 40 bytes (aux_graph.hpp:52-59)
        const int32_t su = jj[k] / Sw;
        char* rec = a.records + o * 40;
        *reinterpret_cast<int2*>(rec) = make_int2(sedge[ei].e, (int)(sedge[ei].nb_u + su));
        *reinterpret_cast<int2*>(rec + 8) = make_int2((int)(sedge[ei].nb_w + sw[k]), 0);
        *reinterpret_cast<double*>(rec + 16) = c[k];
        *reinterpret_cast<double*>(rec + 24) = v[k];
        *reinterpret_cast<double*>(rec + 32) = m[k];
      }
    }
  }
}

// Node tensors: every member operator of a node class gets the class rows.
__device__ void node_fanout(const FusedArgs& a, const NodeWork& nw) {
  if (threadIdx.x == 0)
    while (ld_acquire(&a.sched->node_done) < a.total_rows) __nanosleep(64);
  __syncthreads();
  const ClassDesc cd = a.classes[nw.cls];
  const int64_t total = (int64_t)(nw.mend - nw.mbeg) * cd.S;
  for (int64_t t = threadIdx.x; t < total; t += kFusedThreads) {
    const int64_t mm = t / cd.S, sidx = t - mm * cd.S;
    const int64_t node = a.member_nb[nw.mbeg + mm] + sidx;
    const int64_t row = cd.row_base + sidx;
    if (a.n_sec) __stcs(a.n_sec + node, __ldcg(a.cls_sec + row));
    if (a.n_vol) __stcs(a.n_vol + node, __ldcg(a.cls_vol + row));
    if (a.n_mem) __stcs(a.n_mem + node, __ldcg(a.cls_mem + row));
  }
}

// The whole build in one persistent launch. Phase 1: block work items for
// the node-class rows (few). Phase 2: every warp pulls class pairs from an
// atomic counter on its own — no block barrier, so a slow pair never idles
// the other warps of its CTA. Phase 3: block work items for the fan-out tiles
// and the node fan-out; a tile waits (acquire) only for its own edge class's
// pair counter. Every pair is dequeued before any fan-out item and each
// dequeued item runs to completion, so the waits always end. The
// latency-bound pair work and the HBM-bound fan-out overlap, with no launch
// gap or wave tail between them.
template <bool kWarpForm>
__global__ void __launch_bounds__(kFusedThreads, 4) fused_kernel(FusedArgs a) {
  __shared__ int s_item;
  __shared__ FanEdge sedge[kMaxChunk];
  const int lane = threadIdx.x & 31;
  // phase 1: node-class rows; the first item past them is kept for phase 3
  int carried;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(&a.sched->head, 1);
    __syncthreads();
    const int item = s_item;
    __syncthreads();
    if (item >= a.i_pair) {
      carried = item;
      break;
    }
    const int64_t row = (int64_t)item * kFusedThreads + threadIdx.x;
    if (row < a.total_rows) node_row(a, row);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t rem = a.total_rows - (int64_t)item * kFusedThreads;
      atomicAdd(&a.sched->node_done, (int)(rem < kFusedThreads ? rem : kFusedThreads));
    }
  }
  // phase 2: class pairs, dequeued per warp
  // the next index is fetched while the current one is priced
  if (kWarpForm) {
    int next_idx = 0;
    if (lane == 0) next_idx = atomicAdd(&a.sched->pair_head, 1);
    for (;;) {
      const int64_t idx = __shfl_sync(0xffffffffu, next_idx, 0);
      if (idx >= a.total_pairs) break;
      if (lane == 0) next_idx = atomicAdd(&a.sched->pair_head, 1);
      const int sig = sig_of_pair(a, idx);
      pair_warp(a, idx, sig);
      if (lane == 0) {
        __threadfence();
        atomicAdd(&a.sched->pairs_done[sig], 1);
      }
    }
  } else {
    int next_chunk = 0;
    if (lane == 0) next_chunk = atomicAdd(&a.sched->pair_head, 1);
    for (;;) {
      const int64_t chunk = __shfl_sync(0xffffffffu, next_chunk, 0);
      const int64_t idx = chunk * 32 + lane;
      if (chunk * 32 >= a.total_pairs) break;
      if (lane == 0) next_chunk = atomicAdd(&a.sched->pair_head, 1);
      const bool valid = idx < a.total_pairs;
      const int sig = valid ? sig_of_pair(a, idx) : -1;
      if (valid) pair_thread(a, idx, sig);
      __threadfence();
      // one counter update per (warp, edge class)
      const unsigned grp = __match_any_sync(0xffffffffu, sig);
      if (valid && lane == __ffs(grp) - 1) atomicAdd(&a.sched->pairs_done[sig], __popc(grp));
    }
  }
  // phase 3: fan-out tiles and node fan-out (every pair is dequeued by now)
  for (bool first = true;; first = false) {
    int item = carried;
    if (!first) {
      if (threadIdx.x == 0) s_item = atomicAdd(&a.sched->head, 1);
      __syncthreads();
      item = s_item;
      __syncthreads();
    }
    if (item >= a.i_end) return;
    if (item < a.i_nfan) fanout_tile(a, a.work[item - a.i_exp], sedge);
    else node_fanout(a, a.nwork[item - a.i_nfan]);
  }
}

// K3 (optional): cond_min (solver.hpp:239-253), warp per (edge, su) row.
__global__ void rowmin_kernel(const EdgeDesc* __restrict__ edges, const int64_t* __restrict__ row_base,
                              int e0, int nedges, int64_t nrows, const SigDesc* __restrict__ sigs,
                              const double* __restrict__ r_sec, const double* __restrict__ r_vol,
                              const double* __restrict__ cls_sec, const double* __restrict__ cls_vol,
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
  for (int64_t sw = lane; sw < sg.Sw; sw += 32) {
    const int64_t j = sg.pair_begin + su * sg.Sw + sw;
    const double c = cls_sec[ed.wrow + sw] + r_sec[j] * sg.scale;
    const double v = cls_vol[ed.wrow + sw] + r_vol[j] * sg.scale;
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
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = bytes < 256 ? 256 : bytes;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
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
  int t = 0;
  while (t < 63 && !((v >> t) & 1)) ++t;
  return t;
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
  DevBuf d_tabs, d_tables, d_classes, d_chks, d_slots, d_occs, d_members, d_sigs, d_edges, d_list,
      d_work, d_over, d_rsec, d_rvol, d_csec, d_cvol, d_cmem, d_cmem0, d_nwork, d_rowbase, d_sched, d_sidejobs,
      d_sides, d_price, d_pairsigs;
  DevBuf out[9];  // one-shot staging of the requested outputs
  std::vector<std::array<int64_t, 4>> table_key;  // (offset, count, p, n) of the resident tables
  void release() {
    for (DevBuf* b : {&d_tabs, &d_tables, &d_classes, &d_chks, &d_slots, &d_occs, &d_members, &d_sigs,
                      &d_edges, &d_list, &d_work, &d_over, &d_rsec, &d_rvol, &d_csec, &d_cvol, &d_cmem,
                      &d_cmem0, &d_nwork, &d_rowbase, &d_sched, &d_sidejobs, &d_sides, &d_price, &d_pairsigs})
      b->release();
    for (auto& b : out) b.release();
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
  std::vector<int32_t> pair_sigs;  // classes whose tables are computed, by pair_begin
  int64_t total_pairs = 0;
  int64_t h2d_bytes = 0;
  bool uploaded = false;
  std::vector<Work> work;
  std::vector<NodeWork> nwork;
  std::vector<SideJob> side_jobs;
  int64_t side_total = 0;
  int64_t last_launches = 0;
  int32_t last_e0 = -1, last_e1 = -1;
  cudaStream_t last_stream = nullptr;
  cudaEvent_t prof_start = nullptr, prof_stop = nullptr;  // recorded around K2
  int pair_form = 0;  // 0 = by size, 1 = warp per pair, 2 = thread per pair
  int resident_blocks = 0;  // persistent grid size (SMs x resident CTAs)
};

namespace {

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
  struct OpSlots {
    std::vector<int32_t> name, spec;
    int find(int nm) const {
      for (size_t i = 0; i < name.size(); ++i)
        if (name[i] == nm) return (int)i;
      return -1;
    }
  };
  std::vector<OpSlots> op_slots;
  std::vector<std::vector<std::array<int8_t, tpk::kMaxR>>> slot_sa;  // per op, per slot
  std::map<int, int64_t> table_of_p;
  std::map<std::vector<int64_t>, int32_t> class_of_key;
  std::vector<std::vector<int64_t>> class_members;
  std::unordered_map<int32_t, std::vector<int32_t>> fed_names;  // op id -> tensors fed by edges
  std::vector<int64_t> wrow_of_op;

  tp_status run() {
    tp_status st = check_desc();
    if (st) return st;
    tp_plan& p = *P;
    p.num_ops = g->num_ops;
    p.num_edges = g->num_edges;
    p.N = (int64_t)t->node_count * (int64_t)t->local_device_num;
    p.env = Env{t->intra_bandwidth, t->inter_bandwidth, (int64_t)t->local_device_num};

    // graph.hpp:135-154 find_op (first operator with the id), degrees by id
    std::unordered_map<int32_t, int32_t> first_op, to_count, from_count;
    for (int i = 0; i < g->num_ops; ++i) first_op.emplace(g->op_id[i], i);
    for (int e = 0; e < g->num_edges; ++e) {
      to_count[g->edge_to[e]]++;
      from_count[g->edge_from[e]]++;
      fed_names[g->edge_to[e]].push_back(g->edge_tensor[e]);
    }
    p.in_deg.resize(g->num_ops);
    p.out_deg.resize(g->num_ops);
    for (int i = 0; i < g->num_ops; ++i) {
      auto a = to_count.find(g->op_id[i]);
      auto b = from_count.find(g->op_id[i]);
      p.in_deg[i] = a == to_count.end() ? 0 : a->second;
      p.out_deg[i] = b == from_count.end() ? 0 : b->second;
    }
    p.edge_from_op.resize(g->num_edges);
    p.edge_to_op.resize(g->num_edges);
    for (int e = 0; e < g->num_edges; ++e) {
      auto a = first_op.find(g->edge_from[e]);
      auto b = first_op.find(g->edge_to[e]);
      p.edge_from_op[e] = a == first_op.end() ? -1 : a->second;
      p.edge_to_op[e] = b == first_op.end() ? -1 : b->second;
    }
    p.node_base.assign(g->num_ops + 1, 0);
    p.edge_base.assign(g->num_edges + 1, 0);
    p.row_base.assign(g->num_edges + 1, 0);
    // Kahn's algorithm (graph.hpp:158-183)
    {
      std::vector<int32_t> indeg(g->num_ops, 0);
      std::vector<std::vector<int32_t>> succ(g->num_ops);
      for (int e = 0; e < g->num_edges; ++e) {
        const int u = p.edge_from_op[e], w = p.edge_to_op[e];
        if (u < 0 || w < 0) continue;
        succ[u].push_back(w);
        ++indeg[w];
      }
      std::vector<int32_t> ready;
      for (int i = 0; i < g->num_ops; ++i)
        if (indeg[i] == 0) ready.push_back(i);
      for (size_t h = 0; h < ready.size(); ++h) {
        p.topo.push_back(ready[h]);
        for (int w : succ[ready[h]])
          if (--indeg[w] == 0) ready.push_back(w);
      }
      if ((int)p.topo.size() != g->num_ops) {  // aux_graph.hpp:224-226
        p.topo.assign(g->num_ops, 0);
        p.host_err = ekey(0, tpk::kCycle);
        p.valid_ops = 0;
        return TP_OK;
      }
    }

    // ---------------- node phase (aux_graph.hpp:236-253) -----------------
    const bool pow2 = p.N > 0 && (p.N & (p.N - 1)) == 0;
    p.n_log2 = pow2 ? log2_floor(p.N) : 0;
    if (pow2 && p.n_log2 > tpk::kMaxD) return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "more than 2^16 devices");
    op_slots.resize(g->num_ops);
    slot_sa.resize(g->num_ops);
    wrow_of_op.assign(g->num_ops, 0);
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
    p.num_aux_nodes = nodes;
    for (size_t c = 0; c < p.classes.size(); ++c) {  // class member CSR + fan-out work
      p.classes[c].mem_begin = (int32_t)p.members.size();
      for (int64_t nb : class_members[c]) p.members.push_back(nb);
      p.classes[c].mem_end = (int32_t)p.members.size();
      const int per = std::max(1, 2048 / std::max(1, p.classes[c].S));
      for (int m = p.classes[c].mem_begin; m < p.classes[c].mem_end; m += per)
        p.nwork.push_back(NodeWork{(int32_t)c, m, std::min(p.classes[c].mem_end, m + per), 0});
    }

    // ---------------- edge phase (aux_graph.hpp:273-296) -----------------
    int64_t aux = 0, rows = 0;
    p.valid_edges = 0;
    std::map<std::vector<int64_t>, int32_t> sig_of_key;
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
        const int ku = op_slots[u].find(g->edge_tensor[e]);
        const int kw = op_slots[w].find(g->edge_tensor[e]);
        if (ku < 0 || kw < 0) {
          p.host_err = ekey(kEdgePhase + (uint64_t)aux * 2, tpk::kEdgeTensorMissing);
          p.valid_edges = e;
          break;
        }
        const int tu = op_slots[u].spec[ku], tw = op_slots[w].spec[kw];
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
        if (Su * Sw >= ((int64_t)1 << 31) - kExpTile)
          return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "more than 2^31 pairs on one edge");
        int64_t elements = 1;
        for (int d = 0; d < R; ++d) elements *= shape_of(tu)[d];
        const double bytes = (double)elements * g->tensor_element_size[tu];  // graph.hpp:52-54
        std::vector<int64_t> key;
        key.reserve(8 + 3 * R);
        int64_t bbits;
        std::memcpy(&bbits, &bytes, 8);
        key.insert(key.end(), {(int64_t)pu, (int64_t)pw, (int64_t)R, bbits});
        for (int d = 0; d < R; ++d) key.push_back(shape_of(tu)[d]);
        for (int d = 0; d < R; ++d) key.push_back(slot_sa[u][ku][d]);
        for (int d = 0; d < R; ++d) key.push_back(slot_sa[w][kw][d]);
        auto it = sig_of_key.find(key);
        int32_t sig;
        if (it == sig_of_key.end()) {
          sig = (int32_t)p.sigs.size();
          sig_of_key.emplace(key, sig);
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
            for (int d = 0; d < tpk::kMaxR; ++d) j.sa[d] = d < R ? (side ? slot_sa[w][kw][d] : slot_sa[u][ku][d]) : -1;
            (side ? sd.side_w : sd.side_u) = (int32_t)p.side_total;
            p.side_jobs.push_back(j);
            p.side_total += j.count;
          }
          for (int d = 0; d < tpk::kMaxR; ++d) {
            sd.sa_u[d] = d < R ? slot_sa[u][ku][d] : -1;
            sd.sa_w[d] = d < R ? slot_sa[w][kw][d] : -1;
            const int64_t E = d < R ? shape_of(tu)[d] : 1;
            const int v = v2_capped(E);
            sd.dt[d].t = (uint8_t)v;
            sd.dt[d].odd = (E >> v) > 1;
          }
          p.sigs.push_back(sd);
          edges_of_sig.emplace_back();
          p.total_pairs += Su * Sw;
        } else {
          sig = it->second;
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
    st = memo_aliasing();
    if (st) return st;
    if (p.overrides.empty() && p.N > 0 && (p.N & (p.N - 1)) == 0) derive_classes();
    p.pair_sigs.clear();
    for (size_t c = 0; c < p.sigs.size(); ++c)
      if (p.sigs[c].base == (int32_t)c) p.pair_sigs.push_back((int32_t)c);
    p.h2d_bytes = (int64_t)(p.tabs.size() * sizeof(TableDesc) + p.classes.size() * sizeof(ClassDesc) +
                            p.members.size() * sizeof(int64_t) + p.chks.size() * sizeof(SliceChk) +
                            p.slots.size() * sizeof(SlotDesc) + p.occs.size() * sizeof(Occ) +
                            p.sigs.size() * sizeof(SigDesc) + p.edges.size() * sizeof(EdgeDesc) +
                            p.side_jobs.size() * sizeof(SideJob) +
                            p.overrides.size() * sizeof(double));
    return st;
  }

  // Slots, slice checks, occurrences of one op; then its node class.
  tp_status build_op(int i, int np, int64_t S, int64_t nb) {
    tp_plan& p = *P;
    OpSlots& os = op_slots[i];
    const int t0 = g->op_tensor_begin[i], t1 = g->op_tensor_begin[i + 1];
    for (int t = t0; t < t1; ++t) {
      int k = os.find(g->tensor_name[t]);
      if (k < 0) {
        k = (int)os.name.size();
        os.name.push_back(g->tensor_name[t]);
        os.spec.push_back(t);
      }
      os.spec[k] = t;
      if (rank_of(t) > tpk::kMaxR) return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "tensor rank above 8");
      for (int d = 0; d < rank_of(t); ++d)
        if (shape_of(t)[d] < 1) return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "tensor extent < 1 is unsupported");
    }
    if (os.name.size() > 32000) return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "too many tensors per op");
    auto& sa = slot_sa[i];
    sa.assign(os.name.size(), std::array<int8_t, tpk::kMaxR>{});
    for (auto& a : sa) a.fill(-1);
    std::vector<SliceChk> chk;
    const int a0 = g->op_axis_begin[i];
    for (int a = 0; a < np; ++a) {
      for (int s = g->axis_slice_begin[a0 + a]; s < g->axis_slice_begin[a0 + a + 1]; ++s) {
        const int k = os.find(g->slice_tensor[s]);
        SliceChk c{};
        c.axis = (int8_t)a;
        c.slot = (int16_t)k;
        c.v = 0;
        if (k >= 0) {
          const int dim = g->slice_dim[s];
          const int tk = os.spec[k];
          if (dim < 0 || dim >= rank_of(tk))
            return set_err(TP_ERR_INVALID_ARGUMENT, 0, "slice dimension out of range");
          c.v = (int8_t)v2_capped(shape_of(tk)[dim]);
          sa[k][dim] = (int8_t)a;  // later slices overwrite (layout.hpp:366)
        }
        chk.push_back(c);
      }
    }
    std::vector<SlotDesc> slots;
    for (size_t k = 0; k < os.name.size(); ++k) {
      SlotDesc sd{};
      const int tk = os.spec[k];
      int64_t el = 1;
      for (int d = 0; d < rank_of(tk); ++d) el *= shape_of(tk)[d];
      sd.elements = el;
      sd.es = g->tensor_element_size[tk];
      sd.R = (int8_t)rank_of(tk);
      for (int d = 0; d < tpk::kMaxR; ++d) sd.sa[d] = sa[k][d];
      slots.push_back(sd);
    }
    std::vector<Occ> occ;
    const int nin = g->op_num_inputs[i];
    auto fit = fed_names.find(g->op_id[i]);
    for (int t = t0; t < t1; ++t) {
      Occ oc{};
      const int nm = g->tensor_name[t];
      oc.slot = (int16_t)os.find(nm);
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
        if (fit != fed_names.end())
          for (int32_t x : fit->second) fed |= x == nm;
        oc.in_memory = !fed;
      } else {
        oc.in_memory = 1;
      }
      occ.push_back(oc);
    }
    // node class key: everything the per-node costs depend on
    std::vector<int64_t> key{(int64_t)np, (int64_t)p.in_deg[i], (int64_t)chk.size(), (int64_t)slots.size(),
                             (int64_t)occ.size()};
    for (auto& c : chk) key.insert(key.end(), {(int64_t)c.slot, (int64_t)c.axis, (int64_t)c.v});
    for (auto& s : slots) {
      key.insert(key.end(), {s.elements, (int64_t)s.es, (int64_t)s.R});
      for (int d = 0; d < tpk::kMaxR; ++d) key.push_back(s.sa[d]);
    }
    for (auto& o : occ) key.insert(key.end(), {(int64_t)o.slot, (int64_t)o.nonslicing, (int64_t)o.in_memory});
    auto it = class_of_key.find(key);
    int32_t cls;
    if (it == class_of_key.end()) {
      cls = (int32_t)p.classes.size();
      class_of_key.emplace(key, cls);
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
    } else {
      cls = it->second;
    }
    class_members[cls].push_back(nb);
    wrow_of_op[i] = p.classes[cls].row_base;
    return TP_OK;
  }

  // Two edge classes with the same axis counts and slicings see the same
  // layout pairs. When every tensor dim of both has 2-adic valuation >= log2
  // N, no strategy can fail a divisibility check (a region spans at most
  // log2 N bits), so their plans are identical and every priced quantity is
  // linear in the tensor bytes; with a power-of-two byte ratio the later
  // class's table is the earlier one's times that ratio, exactly (scaling by
  // 2^k commutes with IEEE rounding). Such a class reuses the base table.
  void derive_classes() {
    tp_plan& p = *P;
    std::map<std::vector<int64_t>, int32_t> base_of;
    int64_t pairs = 0;
    for (size_t c = 0; c < p.sigs.size(); ++c) {
      SigDesc& sd = p.sigs[c];
      bool safe = true;
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
      pairs += (int64_t)sd.Su * sd.Sw;
    }
    for (auto& sd : p.sigs)
      if (sd.base != (int32_t)(&sd - p.sigs.data())) sd.pair_begin = p.sigs[sd.base].pair_begin;
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
      const int tu = op_slots[u].spec[op_slots[u].find(g->edge_tensor[ed.e])];
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

// CTA work items for edges [e0, e1): class tiles x edge chunks.
void make_work(tp_plan* p, int32_t e0, int32_t e1, std::vector<Work>& out, std::vector<FanEdge>& list) {
  out.clear();
  list.clear();
  std::vector<int32_t> begin(1, 0);
  int64_t total = 0;
  const int64_t out_offset = p->edge_base[e0];
  for (size_t s = 0; s < p->sigs.size(); ++s) {
    for (int i = p->sig_edge_begin[s]; i < p->sig_edge_begin[s + 1]; ++i) {
      const int e = p->sig_edges[i];
      if (e >= e0 && e < e1) {
        const EdgeDesc& ed = p->edges[e];
        list.push_back(FanEdge{ed.aux_base - out_offset, ed.wrow, ed.nb_u, ed.nb_w, ed.e, 0});
        total += (int64_t)p->sigs[s].Su * p->sigs[s].Sw;
      }
    }
    begin.push_back((int32_t)list.size());
  }
  // ~4 CTAs per SM; each CTA reuses its class tile across a chunk of edges
  const int64_t target = std::max<int64_t>(kExpTile, total / (148 * 4) + 1);
  for (size_t s = 0; s < p->sigs.size(); ++s) {
    const int b = begin[s], en = begin[s + 1];
    if (b == en) continue;
    const int64_t P = (int64_t)p->sigs[s].Su * p->sigs[s].Sw;
    const int64_t tile = std::min<int64_t>(P, kExpTile);
    const int chunk = (int)std::min<int64_t>(kMaxChunk, std::max<int64_t>(1, target / std::max<int64_t>(tile, 1)));
    for (int64_t j0 = 0; j0 < P; j0 += kExpTile) {
      for (int c = b; c < en; c += chunk) {
        Work w{};
        w.sig = (int32_t)s;
        w.ebeg = c;
        w.eend = std::min(en, c + chunk);
        w.j0 = (int32_t)j0;
        out.push_back(w);
      }
    }
  }
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

tp_status tp_plan_upload(tp_plan* p, void* stream) {
  if (!p) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null plan");
  tp_status st = ensure_stream(p);
  if (st) return st;
  Arena& A = *p->arena;
  cudaStream_t s = stream ? (cudaStream_t)stream : A.stream;
  // strategy tables: a pure function of (p, N), cached on the arena
  std::vector<std::array<int64_t, 4>> key;
  for (auto& td : p->tabs) key.push_back({td.offset, td.count, td.p, td.n});
  if (key != A.table_key && p->table_total > 0) {
    CUDA_TRY(upload(A.d_tabs, p->tabs, s));
    CUDA_TRY(A.d_tables.ensure(sizeof(Strat) * (p->table_total + 1)));
    table_kernel<<<(unsigned)((p->table_total + 127) / 128), 128, 0, s>>>(
        (const TableDesc*)A.d_tabs.p, (int)p->tabs.size(), p->table_total, (Strat*)A.d_tables.p);
    CUDA_TRY(cudaGetLastError());
    A.table_key = key;
  }
  // layout descriptors of every (edge class, side, strategy)
  CUDA_TRY(upload(A.d_sidejobs, p->side_jobs, s));
  CUDA_TRY(A.d_sides.ensure(sizeof(tpk::SideDesc) * (p->side_total + 1)));
  if (p->side_total > 0) {
    side_kernel<<<(unsigned)((p->side_total + 127) / 128), 128, 0, s>>>(
        (const SideJob*)A.d_sidejobs.p, (int)p->side_jobs.size(), p->side_total, (const Strat*)A.d_tables.p,
        (tpk::SideDesc*)A.d_sides.p);
    CUDA_TRY(cudaGetLastError());
  }
  {
    std::vector<double> tabs(tpk::kBwTab + tpk::kScaleDim * tpk::kScaleDim);
    tpk::make_price_tabs(p->env, tabs.data(), tabs.data() + tpk::kBwTab);
    CUDA_TRY(upload(A.d_price, tabs, s));
  }
  CUDA_TRY(upload(A.d_classes, p->classes, s));
  CUDA_TRY(upload(A.d_nwork, p->nwork, s));
  CUDA_TRY(upload(A.d_members, p->members, s));
  CUDA_TRY(upload(A.d_chks, p->chks, s));
  CUDA_TRY(upload(A.d_slots, p->slots, s));
  CUDA_TRY(upload(A.d_occs, p->occs, s));
  CUDA_TRY(upload(A.d_sigs, p->sigs, s));
  CUDA_TRY(upload(A.d_pairsigs, p->pair_sigs, s));
  CUDA_TRY(upload(A.d_edges, p->edges, s));
  CUDA_TRY(upload(A.d_over, p->overrides, s));
  CUDA_TRY(A.d_rsec.ensure(sizeof(double) * (p->total_pairs + 1)));
  CUDA_TRY(A.d_rvol.ensure(sizeof(double) * (p->total_pairs + 1)));
  CUDA_TRY(A.d_csec.ensure(sizeof(double) * (p->total_rows + 1)));
  CUDA_TRY(A.d_cvol.ensure(sizeof(double) * (p->total_rows + 1)));
  CUDA_TRY(A.d_cmem.ensure(sizeof(double) * (p->total_rows + 1)));
  CUDA_TRY(A.d_cmem0.ensure(sizeof(double) * (p->total_rows + 1)));
  CUDA_TRY(A.d_sched.ensure(sizeof(Sched) + sizeof(int) * (p->sigs.size() + 2)));
  p->uploaded = true;
  p->last_e0 = p->last_e1 = -1;
  return TP_OK;
}

tp_status tp_plan_execute(tp_plan* p, const tp_build_opts* opts, tp_cost_tensors* out) {
  if (!p) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null plan");
  tp_status st = ensure_stream(p);
  if (st) return st;
  if (!p->uploaded) {
    st = tp_plan_upload(p, opts ? opts->stream : nullptr);
    if (st) return st;
  }
  Arena& A = *p->arena;
  cudaStream_t s = (opts && opts->stream) ? (cudaStream_t)opts->stream : A.stream;
  p->last_stream = s;
  int32_t e0 = opts ? opts->edge_begin : 0;
  int32_t e1 = opts ? opts->edge_end : -1;
  if (e1 < 0 || e1 > p->valid_edges) e1 = p->valid_edges;
  if (e0 < 0) e0 = 0;
  if (e0 > e1) e0 = e1;
  const bool skip_nodes = opts && opts->skip_nodes;
  tp_cost_tensors none{};
  if (!out) out = &none;
  int64_t launches = 0;
  Sched* sched = (Sched*)A.d_sched.p;
  const size_t sched_bytes = sizeof(Sched) + sizeof(int) * (p->sigs.size() + 2);
  CUDA_TRY(cudaMemsetAsync(sched, 0, sched_bytes, s));
  if (p->host_err != ~0ull && (p->host_err >> 6) == 0) {  // cycle: nothing to build
    p->last_launches = 0;
    return TP_OK;
  }
  const bool edge_phase = p->host_err >= ekey(kEdgePhase, 0);
  const bool nodes_out = !skip_nodes && (out->node_intra_cost_s || out->node_intra_volume_bytes ||
                                         out->node_memory_bytes);
  const int64_t out_offset = p->edge_base[e0];
  const bool edges_out = p->edge_base[e1] > out_offset && edge_phase &&
                         (out->edge_cost_s || out->edge_volume_bytes || out->edge_memory_bytes ||
                          out->aux_edge_records);
  if (edges_out && (p->last_e0 != e0 || p->last_e1 != e1)) {
    std::vector<FanEdge> list;
    make_work(p, e0, e1, p->work, list);
    CUDA_TRY(upload(A.d_work, p->work, s));
    CUDA_TRY(upload(A.d_list, list, s));
    p->last_e0 = e0;
    p->last_e1 = e1;
  }
  FusedArgs a{};
  a.classes = (const ClassDesc*)A.d_classes.p;
  a.ncls = (int)p->classes.size();
  a.total_rows = p->total_rows;
  a.chks = (const SliceChk*)A.d_chks.p;
  a.slots = (const SlotDesc*)A.d_slots.p;
  a.occs = (const Occ*)A.d_occs.p;
  a.cls_sec = (double*)A.d_csec.p;
  a.cls_vol = (double*)A.d_cvol.p;
  a.cls_mem = (double*)A.d_cmem0.p;
  a.cls_memdiv = (double*)A.d_cmem.p;
  a.sigs = (const SigDesc*)A.d_sigs.p;
  a.nsigs = (int)p->sigs.size();
  a.pair_sigs = (const int32_t*)A.d_pairsigs.p;
  a.npair_sigs = (int)p->pair_sigs.size();
  a.total_pairs = edge_phase ? p->total_pairs : 0;
  a.overrides = (const double*)A.d_over.p;
  a.sides = (const tpk::SideDesc*)A.d_sides.p;
  a.r_sec = (double*)A.d_rsec.p;
  a.r_vol = (double*)A.d_rvol.p;
  a.work = (const Work*)A.d_work.p;
  a.fan = (const FanEdge*)A.d_list.p;
  a.e_sec = out->edge_cost_s;
  a.e_vol = out->edge_volume_bytes;
  a.e_mem = out->edge_memory_bytes;
  a.records = (char*)out->aux_edge_records;
  a.general_store = a.records || !(a.e_sec && a.e_vol && a.e_mem);
  a.nwork = (const NodeWork*)A.d_nwork.p;
  a.member_nb = (const int64_t*)A.d_members.p;
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
  a.warp_form = p->pair_form == 1 || (p->pair_form == 0 && a.total_pairs <= kWarpPairLimit);
  // block queue: [0, i_pair) node-row items, then [i_exp, i_nfan) fan-out
  // tiles, [i_nfan, i_end) node fan-out; the pairs have their own warp queue
  const int64_t node_items = (p->total_rows + kFusedThreads - 1) / kFusedThreads;
  const int64_t exp_items = edges_out ? (int64_t)p->work.size() : 0;
  const int64_t nfan_items = nodes_out ? (int64_t)p->nwork.size() : 0;
  const int64_t total_items = node_items + exp_items + nfan_items;
  if (total_items >= (1ll << 31) || a.total_pairs >= (1ll << 36))
    return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "too many work items");
  a.i_pair = (int)node_items;
  a.i_exp = (int)node_items;
  a.i_nfan = (int)(node_items + exp_items);
  a.i_end = (int)total_items;
  if (total_items > 0 || a.total_pairs > 0) {
    if (p->resident_blocks == 0) {
      int sms = 0, per_sm = 0;
      CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device));
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_kernel<true>, kFusedThreads, 0));
      p->resident_blocks = std::max(1, sms * std::max(1, per_sm));
    }
    const int64_t warps_needed = a.warp_form ? a.total_pairs : (a.total_pairs + 31) / 32;
    const int64_t blocks_needed = std::max<int64_t>(total_items, (warps_needed + 7) / 8);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(blocks_needed, p->resident_blocks));
    if (p->prof_start) CUDA_TRY(cudaEventRecord(p->prof_start, s));
    if (a.warp_form) fused_kernel<true><<<(unsigned)grid, kFusedThreads, 0, s>>>(a);
    else fused_kernel<false><<<(unsigned)grid, kFusedThreads, 0, s>>>(a);
    ++launches;
    if (p->prof_stop) CUDA_TRY(cudaEventRecord(p->prof_stop, s));
  }
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
          (const SigDesc*)A.d_sigs.p, (const double*)A.d_rsec.p, (const double*)A.d_rvol.p,
          (const double*)A.d_csec.p, (const double*)A.d_cvol.p, out->row_min_cost_s, out->row_min_volume_bytes);
      ++launches;
    }
  }
  CUDA_TRY(cudaGetLastError());
  p->last_launches = launches;
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

tp_status tp_plan_check_errors(tp_plan* p) {
  if (!p) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null plan");
  CUDA_TRY(cudaSetDevice(p->device));
  unsigned long long dev = ~0ull;
  if (p->arena && p->arena->d_sched.p && p->last_stream) {
    unsigned long long c = 0;
    CUDA_TRY(cudaMemcpyAsync(&c, p->arena->d_sched.p, sizeof(c), cudaMemcpyDeviceToHost, p->last_stream));
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
