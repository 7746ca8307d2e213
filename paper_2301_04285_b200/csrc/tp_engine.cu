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
// pairmin_kernel (optional, third launch): warp per edge over its row minima —
// the solver's pair_min (solver.hpp:254-255).
// The strategy tables (layout.hpp:270-328) are built once per plan by
// table_kernel at upload and cached per device. Sweeps of many scenarios run
// as one batched launch (fused_batch_kernel, tp_plan_execute_batch).
//
// One translation unit, in order: tp_desc.cuh (descriptors), tp_kernels.cuh
// (device code), tp_plan.cuh (arenas, tp_plan, host analysis), then the
// C-ABI below (plans, uploads, executes, batches, verification export).
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
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <malloc.h>

#include "../../include/taps_b200.h"
#include "../../include/taps_b200/lp_export.hpp"
#include "tp_core.cuh"
#include "tp_fast.cuh"
#include "tp_warp.cuh"

using tpk::DimT;
using tpk::Env;
using tpk::Lay;
using tpk::Strat;

#include "tp_desc.cuh"
#include "tp_kernels.cuh"
#include "tp_plan.cuh"

namespace {
// TP_MALLOPT=1: keep freed host memory in the heap instead of mapping and
// unmapping large blocks (an A/B switch for the host analysis of sweeps).
struct MalloptInit {
  MalloptInit() {
    const char* v = getenv("TP_MALLOPT");
    if (v && atoi(v) > 0) {
      mallopt(M_MMAP_THRESHOLD, 32 << 20);
      mallopt(M_TRIM_THRESHOLD, 1 << 30);
    }
  }
} g_mallopt_init;
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
  if (device >= ndev || device >= 64) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "device ordinal out of range");
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
  DeviceGuard dg;
  if (!p) return;
  for (tp_plan* q : p->shards) tp_plan_destroy(q);
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
// A batch sets min_len (batch_range_len): its ranges are cut for the batch
// as a whole, not per plan -- a small plan is one range, not dozens of
// 256-id ones whose staging and barriers would cost more than their stores.
void range_layout(const tp_plan* p, int64_t total_out, int64_t total_nodes, int64_t& range_len, int64_t& exp_items,
                  int64_t& nfan_items, int64_t min_len = kFusedThreads * kFanPer) {
  const int64_t nranges = std::max(1, p->resident_blocks - 2);  // the two ceilings below add at most 2
  range_len = std::max<int64_t>(min_len, (total_out + total_nodes + nranges - 1) / nranges);
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

// Host only: the descriptor pieces of the plan (and its default range table;
// min_len: a batch's range length, batch_range_len).
tp_status upload_prepare(tp_plan* p, UploadPrep& U, int64_t min_len = kFusedThreads * kFanPer) {
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
    range_layout(p, total_out, p->num_aux_nodes, rl, ei, ni, min_len);
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
  DeviceGuard dg;
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

// batch_mode: 0 = a plan on its own (or in a batch with class tables
// published inside one launch); 4 = priced in the fan-out from op lists
// (units = node rows); 5 = tables priced from op lists in a launch of their
// own. Modes 4 and 5 never rely on unset-filled tables.
tp_status prepare_execute(tp_plan* p, const tp_build_opts* opts, tp_cost_tensors* out, cudaStream_t s, ExecPrep& X,
                          int batch_mode = 0, int64_t min_len = kFusedThreads * kFanPer) {
  const bool direct = batch_mode == 4;
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
  if ((out->edge_pair_min_cost_s || out->edge_pair_min_volume_bytes) &&
      !(out->row_min_cost_s && out->row_min_volume_bytes && out->edge_pair_min_cost_s &&
        out->edge_pair_min_volume_bytes))
    return set_err(TP_ERR_INVALID_ARGUMENT, 0, "pair minima need both row minima and both pair outputs");
  Sched* sched = (Sched*)A.d_sched.p;
  if (!A.sched_clean) {
    CUDA_TRY(cudaMemsetAsync(sched, 0, sizeof(Sched) + sizeof(Line) * (p->sigs.size() + 1), s));
    fill_kernel<<<64, 256, 0, s>>>((double*)A.d_tables2.p, 2 * tables_len(p), kUnset);  // both parities
    CUDA_TRY(cudaGetLastError());
    A.sched_clean = true;
    A.tables_dirty = false;
    A.parity = 0;
  } else if (A.tables_dirty && batch_mode == 0) {  // the last launch left the tables un-reset
    fill_kernel<<<64, 256, 0, s>>>((double*)A.d_tables2.p, 2 * tables_len(p), kUnset);
    CUDA_TRY(cudaGetLastError());
    A.tables_dirty = false;
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
  range_layout(p, total_out, total_nodes, range_len, exp_items, nfan_items, min_len);
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
  a.direct = direct;
  // a two-launch batch (mode 5) publishes nothing: its rows run one per thread
  a.rows_thread = batch_mode == 5 && !a.warp_form;
  a.timeline = p->timeline ? 1 : 0;
  const int64_t row_units = a.rows_thread ? (p->total_rows + 31) / 32 : p->total_rows;
  const int64_t units =
      row_units + (direct ? 0 : (a.warp_form ? a.total_pairs : (a.total_pairs + 31) / 32));
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
      // K4: pair_min (solver.hpp:254-255), a warp per graph edge over its row minima
      if (out->edge_pair_min_cost_s) {
        const int64_t edges = e1 - e0;
        pairmin_kernel<<<(unsigned)((edges * 32 + th - 1) / th), th, 0, s>>>(
            (const int64_t*)A.d_rowbase.p, edges, out->row_min_cost_s, out->row_min_volume_bytes,
            out->edge_pair_min_cost_s, out->edge_pair_min_volume_bytes);
        ++launches;
      }
    }
  }
  CUDA_TRY(cudaGetLastError());
  p->last_launches = launches;
  return TP_OK;
}

}  // namespace

extern "C" {

tp_status tp_plan_execute(tp_plan* p, const tp_build_opts* opts, tp_cost_tensors* out) {
  DeviceGuard dg;
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
  DevBuf d_hdr, d_err, d_ops;
  int64_t last_launches = 0;  // kernel launches of the last batched execute
  // output staging, double-buffered by slot: chunk k builds into out[k & 1]
  // while the copy stream drains chunk k - 1 from the other half
  DevBuf out[2][6];
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t prof_start = nullptr, prof_stop = nullptr;  // tp_batch_set_profile_events
  cudaEvent_t built[2] = {nullptr, nullptr}, drained[2] = {nullptr, nullptr};
  unsigned long long* h_err = nullptr;
  size_t h_err_cap = 0;
  // Host staging is double-buffered by slot: a pipelined sweep packs chunk
  // k + 1 while chunk k's copies still wait on the stream behind chunk k - 1.
  // Kernel arguments (per launch) and descriptor packs (per host batch):
  void* h_stage[2] = {nullptr, nullptr};
  size_t h_cap[2] = {0, 0};
  DevBuf d_args[2];
  cudaEvent_t copied[2] = {nullptr, nullptr};  // the last argument copy out of h_stage[slot]
  void* h_pack[2] = {nullptr, nullptr};
  size_t h_pack_cap[2] = {0, 0};
  DevBuf d_pack[2];
  cudaEvent_t packed[2] = {nullptr, nullptr};  // the last pack copy out of h_pack[slot]
  bool hdr_clean = false;
  int resident = 0, resident_wide = 0;
  cudaStream_t stream = nullptr;  // the host batch's stream (every chunk, in order)
  // arenas of the one-shot host batch, by position: scenario i of a batch
  // always gets arena i, so a repeated sweep finds its buffers sized (no
  // cudaMalloc / cudaFree, which would synchronise the device)
  std::vector<Arena*> host_arenas;
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

// Per edge class of a plan (base classes only): everything its class-table
// entries' op lists depend on -- both sides' strategy tables (p, log2 N) and
// slicings, the dims (2-adic valuation, odd part), the table shape and the
// layout dedup mode -- but not the bytes or bandwidths. Equal keys (any plans)
// have identical op lists entry by entry. Cached on the plan.
const std::vector<std::pair<uint64_t, std::vector<int64_t>>>& class_keys(tp_plan* p) {
  if (p->class_keys.size() == p->sigs.size()) return p->class_keys;
  p->class_keys.assign(p->sigs.size(), {});
  auto pn = [&](int32_t tab) -> int64_t {
    for (const auto& t : p->tabs)
      if (t.offset == tab) return ((int64_t)t.p << 8) | t.n;
    return -1;
  };
  for (size_t c = 0; c < p->sigs.size(); ++c) {
    const SigDesc& sd = p->sigs[c];
    if (sd.base != (int32_t)c) continue;
    std::vector<int64_t> k{sd.R, pn(sd.tab_u), pn(sd.tab_w), sd.Un, sd.Wn, (int64_t)p->overrides.empty()};
    for (int d = 0; d < sd.R; ++d) k.insert(k.end(), {sd.sa_u[d], sd.sa_w[d], sd.dt[d].t, sd.dt[d].odd});
    p->class_keys[c] = {hash_words(0x6a09e667f3bcc909ull, k.data(), k.size() * sizeof(int64_t)), std::move(k)};
  }
  return p->class_keys;
}

// A big batch (thread form) is priced in the fan-out from op lists: every
// class key of the batch inferred once (infer_kernel), each aux edge priced
// from its entry's op list with its own plan's bytes and bandwidths -- no
// class tables and no pair records. Needs every plan's edge tensors written
// (errors are found where they are written) and no row minima (they read the
// tables); TP_BATCH_OPLISTS=0 keeps the class tables (and bandwidth groups).
// Range length of a batch's fan-out: about four ranges per resident CTA over
// the whole batch (aux edges and nodes of every plan), at least the
// single-plan minimum.
int64_t batch_range_len(tp_plan* const* plans, int32_t n) {
  int64_t total = 0;
  for (int i = 0; i < n; ++i)
    if (plans[i]) total += plans[i]->num_aux_edges + plans[i]->num_aux_nodes;
  int resident = 0;
  if (n > 0 && plans[0]) {
    if (plans[0]->resident_blocks == 0) resident_of(plans[0]);
    resident = plans[0]->resident_blocks;
  }
  const int64_t want = total / std::max<int64_t>(1, 4 * (int64_t)std::max(resident, 1));
  const int64_t unit = kFusedThreads * kFanPer;
  return std::max<int64_t>(unit, std::min<int64_t>(32768, (want + unit - 1) / unit * unit));
}

// Returns the batch mode (prepare_execute): 0 = class tables published in
// one launch; 4 = priced in the fan-out; 5 = tables from op lists, two launches.
// TP_BATCH_MODE = 0 / 4 / 5 forces one (A/B); the default is 5.
int batch_mode_of(tp_plan* const* plans, int32_t n, const tp_cost_tensors* outs) {
  static const int forced = getenv("TP_BATCH_MODE") ? atoi(getenv("TP_BATCH_MODE")) : -1;
  const int want = forced >= 0 ? forced : 5;
  int64_t batch_pairs = 0;
  for (int i = 0; i < n; ++i) batch_pairs += plans[i]->total_pairs;
  if (want == 0 || batch_pairs <= kWarpPairLimit) return 0;
  for (int i = 0; i < n; ++i) {
    const tp_cost_tensors& o = outs[i];
    if (plans[i]->pair_form == 1) return 0;
    if (want == 4) {
      if (o.row_min_cost_s || o.row_min_volume_bytes || o.edge_pair_min_cost_s || o.edge_pair_min_volume_bytes)
        return 0;
      if (plans[i]->total_pairs > 0 &&
          !(o.edge_cost_s || o.edge_volume_bytes || o.edge_memory_bytes || o.aux_edge_records))
        return 0;
    }
  }
  return want;
}

// err_dev: optional device array [n] that receives every launched plan's
// error slot (in `live` order via live_out) -- the host batch checks all
// plans with one copy instead of one synchronising read per plan.
tp_status execute_batch_impl(tp_plan* const* plans, int32_t n, tp_cost_tensors* device_outs, void* stream,
                             unsigned long long* err_dev, std::vector<int>* live_out, int slot = 0,
                             int64_t min_range = 0) {
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
  static const bool prof = getenv("TP_PROFILE_HOST") != nullptr;
  double tp0 = prof ? now_us() : 0, tp1 = 0, tp2 = 0;
  std::vector<ExecPrep> X(n);
  std::vector<int> live;
  int64_t batch_pairs = 0;
  for (int i = 0; i < n; ++i) batch_pairs += plans[i]->total_pairs;
  for (int i = 0; i < n; ++i) plans[i]->in_big_batch = batch_pairs > kWarpPairLimit;
  const int bmode = batch_mode_of(plans, n, device_outs);
  const bool use_ops = bmode != 0;
  const int64_t brange = min_range > 0 ? min_range : (bmode ? batch_range_len(plans, n) : kFusedThreads * kFanPer);
  for (int i = 0; i < n; ++i) {
    tp_plan* p = plans[i];
    st = ensure_stream(p);
    if (st) return st;
    if (!p->uploaded) {
      st = tp_plan_upload(p, s);
      if (st) return st;
    }
    st = prepare_execute(p, nullptr, &device_outs[i], s, X[i], bmode, brange);
    p->in_big_batch = false;
    if (st) return st;
    if (!X[i].done && X[i].launch) live.push_back(i);
  }
  const int m = (int)live.size();
  if (prof) tp1 = now_us();
  if (m > 0) {
    if (B.resident == 0) {
      int sms = 0, per_sm = 0;
      CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_batch_kernel<0>, kFusedThreads, kMsecBytes));
      B.resident = std::max(1, sms * std::max(1, per_sm));
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_batch_kernel<3>, kFusedThreads, kMsecBytes));
      B.resident_wide = std::max(1, sms * std::max(1, per_sm));
    }
    int nwarp = 0;
    for (int k : live) nwarp += X[k].a.warp_form != 0;
    // bandwidth groups (thread form only): plans whose pricing inputs are
    // identical but for intra/inter bandwidth share their class pairs
    std::vector<int32_t> glist;                       // member lists, leader first (live order)
    std::vector<std::pair<int, int>> gspan(m, {-1, 0});  // per leader: (offset in glist, size)
    static const bool no_groups = getenv("TP_BATCH_NO_GROUPS") != nullptr;
    if (use_ops && nwarp != 0) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "internal: op lists with warp-form plans");
    std::vector<InferJob> ijobs;
    std::vector<int64_t> ioff{0};
    std::vector<int64_t> clsops;
    std::vector<size_t> clsops_at(m, 0);
    if (use_ops) {
      std::unordered_map<uint64_t, std::vector<int>> by_hash;  // key hash -> jobs
      std::vector<const std::vector<int64_t>*> job_key;
      for (int k = 0; k < m; ++k) {
        tp_plan* p = plans[live[k]];
        clsops_at[k] = clsops.size();
        clsops.resize(clsops.size() + p->sigs.size() + 1, 0);
        if (p->total_pairs == 0 || !X[live[k]].edge_phase) continue;
        const auto& keys = class_keys(p);
        for (size_t c = 0; c < p->sigs.size(); ++c) {
          const SigDesc& sd = p->sigs[c];
          if (sd.base != (int32_t)c) continue;
          auto& cand = by_hash[keys[c].first];
          int job = -1;
          for (int j : cand)
            if (*job_key[j] == keys[c].second) {
              job = j;
              break;
            }
          if (job < 0) {
            job = (int)ijobs.size();
            cand.push_back(job);
            job_key.push_back(&keys[c].second);
            Arena& A = *p->arena;
            ijobs.push_back(InferJob{(const SigDesc*)A.d_sigs.p, (const int32_t*)A.d_pairsigs.p,
                                     (const int32_t*)A.d_maps.p, (const tpk::SideDesc*)A.d_sides.p, sd.pair_begin,
                                     ioff.back()});
            ioff.push_back(ioff.back() + (int64_t)sd.Un * sd.Wn);
          }
          clsops[clsops_at[k] + c] = ijobs[job].out;
        }
      }
    }
    if (prof) tp2 = now_us();
    if (nwarp == 0 && !no_groups && !use_ops) {
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
    // staging: args[m] | unit_off[m+1] | item_off[m+1] | tab_off[m+1] | class op-list offsets |
    // infer jobs | their prefix sums | group lists
    const size_t args_b = sizeof(FusedArgs) * m, off_b = sizeof(int64_t) * (m + 1);
    const size_t cls_b = sizeof(int64_t) * clsops.size(), jobs_b = sizeof(InferJob) * ijobs.size(),
                 ioff_b = sizeof(int64_t) * ioff.size();
    // form 5's table launch: the plan of every chunk of kUC5 units (its first unit)
    int64_t units_all = 0;
    for (int k = 0; k < m; ++k) units_all += X[live[k]].units;
    const int64_t nchunks5 = bmode == 5 ? (units_all + kUC5 - 1) / kUC5 : 0;
    const size_t cp_b = sizeof(int32_t) * (size_t)nchunks5;
    const size_t total = args_b + 3 * off_b + cls_b + jobs_b + ioff_b + sizeof(int32_t) * (glist.size() + 1) + cp_b;
    if (B.copied[slot]) CUDA_TRY(cudaEventSynchronize(B.copied[slot]));
    if (B.h_cap[slot] < total) {
      if (B.h_stage[slot]) cudaFreeHost(B.h_stage[slot]);
      B.h_stage[slot] = nullptr;
      B.h_cap[slot] = 0;
      CUDA_TRY(cudaMallocHost(&B.h_stage[slot], total));
      B.h_cap[slot] = total;
    }
    CUDA_TRY(B.d_args[slot].ensure(total));
    void* const h_stage = B.h_stage[slot];
    FusedArgs* ha = (FusedArgs*)h_stage;
    int64_t* uo = (int64_t*)((char*)h_stage + args_b);
    int64_t* io = uo + (m + 1);
    int64_t* to = io + (m + 1);
    int64_t* hcls = to + (m + 1);
    InferJob* hjobs = (InferJob*)((char*)hcls + cls_b);
    int64_t* hioff = (int64_t*)((char*)hjobs + jobs_b);
    int32_t* hg = (int32_t*)((char*)hioff + ioff_b);
    const char* dbase = (const char*)B.d_args[slot].p;
    const int64_t* dcls = (const int64_t*)(dbase + args_b + 3 * off_b);
    const InferJob* djobs = (const InferJob*)(dbase + args_b + 3 * off_b + cls_b);
    const int64_t* dioff = (const int64_t*)(dbase + args_b + 3 * off_b + cls_b + jobs_b);
    const int32_t* dg = (const int32_t*)(dbase + args_b + 3 * off_b + cls_b + jobs_b + ioff_b);
    const size_t cp_at = args_b + 3 * off_b + cls_b + jobs_b + ioff_b + sizeof(int32_t) * (glist.size() + 1);
    int32_t* hcp = (int32_t*)((char*)h_stage + cp_at);
    const int32_t* dcp = nchunks5 > 0 ? (const int32_t*)(dbase + cp_at) : nullptr;
    if (!clsops.empty()) std::memcpy(hcls, clsops.data(), cls_b);
    if (!ijobs.empty()) std::memcpy(hjobs, ijobs.data(), jobs_b);
    std::memcpy(hioff, ioff.data(), ioff_b);
    const int64_t n_infer = ioff.back();
    if (use_ops) CUDA_TRY(B.d_ops.ensure(sizeof(uint32_t) * tpk::kOpWords * (size_t)std::max<int64_t>(n_infer, 1)));
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
      if (use_ops) {
        ha[j].oplists = (const uint32_t*)B.d_ops.p;
        ha[j].cls_ops = dcls + clsops_at[k];
      }
      if (gspan[k].second >= 2) {
        ha[j].group = dg + gspan[k].first;
        ha[j].group_n = gspan[k].second;
      }
      uo[j + 1] = uo[j] + x.units;
      io[j + 1] = io[j] + x.items;
      to[j + 1] = to[j] + x.a.tables_len;
    }
    for (int j = 0; j < m && nchunks5 > 0; ++j)  // chunk c starts in plan j iff kUC5 c in [uo[j], uo[j+1])
      for (int64_t c = (uo[j] + kUC5 - 1) / kUC5; c < (uo[j + 1] + kUC5 - 1) / kUC5; ++c) hcp[c] = j;
    {  // callers map the kernel's per-plan outputs (error slots) in args order
      std::vector<int> l2(m);
      for (int j = 0; j < m; ++j) l2[j] = live[ord[j]];
      live.swap(l2);
    }
    if (uo[m] >= (1ll << 30) || io[m] >= (1ll << 30))
      return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "too many work items in one batch");
    CUDA_TRY(cudaMemcpyAsync(B.d_args[slot].p, h_stage, total, cudaMemcpyHostToDevice, s));
    if (!B.copied[slot]) CUDA_TRY(cudaEventCreateWithFlags(&B.copied[slot], cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(B.copied[slot], s));
    CUDA_TRY(B.d_hdr.ensure(sizeof(BatchHdr)));
    if (!B.hdr_clean) {
      CUDA_TRY(cudaMemsetAsync(B.d_hdr.p, 0, sizeof(BatchHdr), s));
      B.hdr_clean = true;
    }
    const int64_t blocks_needed = std::max<int64_t>(io[m], (uo[m] + 7) / 8);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(blocks_needed, B.resident));
    if (B.prof_start) CUDA_TRY(cudaEventRecord(B.prof_start, s));  // the launches follow back to back
    if (use_ops && n_infer > 0) {  // the batch's inference pass, before the build
      infer_kernel<<<(unsigned)((n_infer + 127) / 128), 128, 0, s>>>(djobs, (int)ijobs.size(), dioff,
                                                                    (uint32_t*)B.d_ops.p);
      CUDA_TRY(cudaGetLastError());
    }
    const FusedArgs* da = (const FusedArgs*)B.d_args[slot].p;
    const int64_t* duo = (const int64_t*)((const char*)B.d_args[slot].p + args_b);
    static const int wide = getenv("TP_BATCH_WIDE") ? atoi(getenv("TP_BATCH_WIDE")) : 0;  // measured: 4 CTAs/SM with spills beats 2 without
    const int form = nwarp == m ? 1 : (nwarp == 0 ? (use_ops ? bmode : (wide ? 3 : 2)) : 0);
    const dim3 gd((unsigned)std::min<int64_t>(grid, form == 3 ? B.resident_wide : B.resident)), bd(kFusedThreads);
    const int64_t* dio = duo + (m + 1);
    const int64_t* dto = duo + 2 * (m + 1);
    BatchHdr* hd = (BatchHdr*)B.d_hdr.p;
    if (form == 1) fused_batch_kernel<1><<<gd, bd, 0, s>>>(da, m, duo, dio, dto, hd, err_dev, nullptr);
    else if (form == 2) fused_batch_kernel<2><<<gd, bd, kMsecBytes, s>>>(da, m, duo, dio, dto, hd, err_dev, nullptr);
    else if (form == 3) fused_batch_kernel<3><<<gd, bd, kMsecBytes, s>>>(da, m, duo, dio, dto, hd, err_dev, nullptr);
    else if (form == 4) fused_batch_kernel<4><<<gd, bd, 0, s>>>(da, m, duo, dio, dto, hd, err_dev, nullptr);
    else if (form == 5) {  // the tables, then the fan-out (ordered by the launch boundary)
      const dim3 g1((unsigned)std::max<int64_t>(1, std::min<int64_t>((uo[m] + 15) / 16, B.resident)));
      const dim3 g2((unsigned)std::max<int64_t>(1, std::min<int64_t>(io[m], B.resident)));
      fused_batch_kernel<5, 1><<<g1, bd, 0, s>>>(da, m, duo, dio, dto, hd, err_dev, dcp);
      fused_batch_kernel<5, 2><<<g2, bd, 0, s>>>(da, m, duo, dio, dto, hd, err_dev, nullptr);
    }
    else fused_batch_kernel<0><<<gd, bd, kMsecBytes, s>>>(da, m, duo, dio, dto, hd, err_dev, nullptr);
    if (B.prof_stop) CUDA_TRY(cudaEventRecord(B.prof_stop, s));
    B.last_launches = (use_ops && n_infer > 0 ? 1 : 0) + (form == 5 ? 2 : 1);
    if (prof && n >= 32)
      fprintf(stderr, "[tp batch launch] %d plans: prepare %.0f us, class keys %.0f, staging + launches %.0f\n", n,
              tp1 - tp0, tp2 - tp1, now_us() - tp2);
    if (cudaPeekAtLastError() != cudaSuccess) {
      B.hdr_clean = false;
      for (int k : live) plans[k]->arena->sched_clean = false;
    }
    for (int k : live) {
      after_launch(plans[k]);
      plans[k]->last_grid = grid;
      if (use_ops) plans[k]->arena->tables_dirty = true;
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
  DeviceGuard dg;
  return execute_batch_impl(plans, n, device_outs, stream, nullptr, nullptr);
}

tp_status tp_batch_set_profile_events(int32_t device, void* start_event, void* stop_event) {
  if (device < 0 || device >= 64) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "device ordinal out of range");
  g_batch[device].prof_start = (cudaEvent_t)start_event;
  g_batch[device].prof_stop = (cudaEvent_t)stop_event;
  return TP_OK;
}

int64_t tp_batch_last_launches(int32_t device) {
  return device >= 0 && device < 64 ? g_batch[device].last_launches : 0;
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
  DeviceGuard dg;
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
  DeviceGuard dg;
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

}  // extern "C"

namespace {
// The smallest error key of the plan's last execute (device slot, host
// analysis); ~0 = none. Synchronises the plan's stream.
tp_status plan_error_key(tp_plan* p, uint64_t& key) {
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
  key = std::min<uint64_t>(dev, p->host_err);
  return TP_OK;
}

tp_status status_of_key(uint64_t key) {
  if (key == ~0ull) return TP_OK;
  const int kind = (int)(key & 63);
  return set_err(status_of_kind(kind), kind, kind_text(kind));
}
}  // namespace

extern "C" {

tp_status tp_plan_check_errors(tp_plan* p) {
  DeviceGuard dg;
  if (!p) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null plan");
  uint64_t key = ~0ull;
  tp_status st = plan_error_key(p, key);
  if (st) return st;
  return status_of_key(key);
}

}  // extern "C"

namespace {
// tp_plan_execute_host; with key_out the smallest error key is returned
// there instead of as a status (the multi-device build combines its devices').
thread_local char p_exec_detail[256];
bool prof_host() {
  static const bool prof = getenv("TP_PROFILE_HOST") != nullptr;
  return prof;
}

tp_status execute_host_impl(tp_plan* p, const tp_build_opts* opts, tp_aux_index* index_out,
                            tp_cost_tensors* host_out, uint64_t* key_out) {
  if (!p) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null plan");
  const double tx0 = prof_host() ? now_us() : 0;
  tp_status st = ensure_stream(p);
  if (st) return st;
  if (!p->uploaded) {
    st = tp_plan_upload(p, nullptr);
    if (st) return st;
  }
  const double tx0b = prof_host() ? now_us() : 0;
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
  d.edge_pair_min_cost_s = (double*)dev(b[9], h.edge_pair_min_cost_s, e1 - e0, 8);
  d.edge_pair_min_volume_bytes = (double*)dev(b[10], h.edge_pair_min_volume_bytes, e1 - e0, 8);
  if (oom) return set_err(TP_ERR_CUDA, 0, "device allocation for the outputs failed");
  const double tx1 = prof_host() ? now_us() : 0;
  tp_build_opts o = opts ? *opts : tp_build_opts{0, -1, 0, -1, nullptr};
  o.stream = nullptr;
  st = tp_plan_execute(p, &o, &d);
  if (st) return st;
  const double tx2 = prof_host() ? now_us() : 0;
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
  ce = ce ? ce : back(h.edge_pair_min_cost_s, d.edge_pair_min_cost_s, e1 - e0, 8);
  ce = ce ? ce : back(h.edge_pair_min_volume_bytes, d.edge_pair_min_volume_bytes, e1 - e0, 8);
  const double tx3 = prof_host() ? now_us() : 0;
  if (key_out) st = plan_error_key(p, *key_out);  // synchronises the stream
  else st = tp_plan_check_errors(p);
  if (prof_host())
    snprintf(p_exec_detail, sizeof(p_exec_detail), "upload %.0f, outputs %.0f, execute enqueue %.0f, copies enqueue %.0f, wait %.0f",
             tx0b - tx0, tx1 - tx0b, tx2 - tx1, tx3 - tx2, now_us() - tx3);
  if (ce != cudaSuccess) return set_err(TP_ERR_CUDA, 0, cudaGetErrorString(ce));
  if (st) return st;
  if (index_out) tp_plan_index(p, index_out);
  return TP_OK;
}
}  // namespace

extern "C" {

tp_status tp_plan_execute_host(tp_plan* p, const tp_build_opts* opts, tp_aux_index* index_out,
                               tp_cost_tensors* host_out) {
  DeviceGuard dg;
  return execute_host_impl(p, opts, index_out, host_out, nullptr);
}

tp_status tp_plan_execute_host_scratch(tp_plan* p, const tp_build_opts* opts, tp_aux_index* index_out,
                                       tp_cost_tensors* host_out) {
  DeviceGuard dg;
  if (!p) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null plan");
  if (p->arena) return execute_host_impl(p, opts, index_out, host_out, nullptr);
  // borrow the thread's one-shot arena for this (synchronous) call: its
  // descriptors are this plan's only until the call returns
  p->arena = thread_arena(p->device);
  if (!p->arena) return execute_host_impl(p, opts, index_out, host_out, nullptr);  // (no such device: owns one)
  p->owns_arena = false;
  p->uploaded = false;
  p->range_key = {{-1, -1, -1, -1}};
  const tp_status st = execute_host_impl(p, opts, index_out, host_out, nullptr);
  if (p->arena->stream) cudaStreamSynchronize(p->arena->stream);
  p->arena = nullptr;
  p->owns_arena = true;
  p->uploaded = false;
  p->range_key = {{-1, -1, -1, -1}};
  return st;
}

tp_status tp_build_cost_tensors(const tp_graph_desc* graph, const tp_topology_desc* topo,
                                const tp_build_opts* opts, tp_aux_index* index_out,
                                tp_cost_tensors* host_out) {
  DeviceGuard dg;
  static const bool prof = getenv("TP_PROFILE_HOST") != nullptr;
  const double t0 = prof ? now_us() : 0;
  tp_plan* p = nullptr;
  tp_status st = tp_plan_create(graph, topo, opts ? opts->device : -1, &p);
  if (st) return st;
  const double t1 = prof ? now_us() : 0;
  p->arena = thread_arena(p->device);  // reused across one-shot calls
  p->owns_arena = p->arena == nullptr;
  st = tp_plan_execute_host(p, opts, index_out, host_out);
  const double t2 = prof ? now_us() : 0;
  tp_plan_destroy(p);
  if (prof)
    fprintf(stderr, "[tp one-shot] create %.0f us, execute_host %.0f us (%s), destroy %.0f us\n", t1 - t0, t2 - t1,
            p_exec_detail, now_us() - t2);
  return st;
}

}  // extern "C"

namespace {
// A copy of an analysed plan for another device (the multi-device build):
// the host analysis is device-independent; arenas, uploads and launch state
// are not copied.
tp_plan* clone_for_device(const tp_plan* p, int device) {
  tp_plan* q = new tp_plan(*p);
  q->device = device;
  q->arena = nullptr;
  q->owns_arena = true;
  q->d_terms = nullptr;
  q->uploaded = false;
  q->range_key = {{-1, -1, -1, -1}};
  q->last_stream = nullptr;
  q->prof_start = q->prof_stop = nullptr;
  q->timeline = false;
  q->last_parity = -1;
  q->resident_blocks = 0;
  q->shards.clear();
  return q;
}

// Contiguous graph-edge ranges, one per device, balanced by aux edges
// (sum |Su| x |Sw|, the edge_base differences).
std::vector<int32_t> edge_split(const tp_plan* p, int n) {
  const int32_t E = p->valid_edges;
  std::vector<int32_t> b(n + 1, 0);
  b[n] = E;
  const int64_t a0 = p->edge_base[0], total = p->edge_base[E] - a0;
  for (int r = 1; r < n; ++r) {
    const double target = (double)a0 + (double)total * r / n;
    int32_t e = b[r - 1];
    while (e < E && (double)p->edge_base[e] + 0.5 * (double)(p->edge_base[e + 1] - p->edge_base[e]) <= target) ++e;
    b[r] = e;
  }
  return b;
}

// Every device of `devices` builds its edge range of plan p (device 0 of the
// list also the per-node tensors) and copies its slice straight into the
// caller's host arrays at the range's offsets. borrow: shards take pooled
// arenas for the call (the one-shot entry) instead of owning one.
tp_status execute_host_multi(tp_plan* p, const int32_t* devices, int32_t n, tp_aux_index* index_out,
                             tp_cost_tensors* host_out, bool borrow) {
  if (!p || !devices || n < 1 || !host_out) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "bad multi-device arguments");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_err(TP_ERR_CUDA, 0, "no CUDA device: the engine has no CPU path");
  for (int i = 0; i < n; ++i) {
    if (devices[i] < 0 || devices[i] >= ndev || devices[i] >= 64)
      return set_err(TP_ERR_INVALID_ARGUMENT, 0, "device ordinal out of range");
    for (int j = 0; j < i; ++j)
      if (devices[j] == devices[i]) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "device listed twice");
  }
  // per-device copies of the analysed plan, cached on it
  if ((int)p->shards.size() < n) p->shards.resize(n, nullptr);
  for (int i = 0; i < n; ++i) {
    tp_plan*& q = p->shards[i];
    if (q && q->device != devices[i]) {
      tp_plan_destroy(q);
      q = nullptr;
    }
    if (!q) q = clone_for_device(p, devices[i]);
    if (q->env.intra != p->env.intra || q->env.inter != p->env.inter) {  // tp_plan_set_bandwidth reaches the shards
      q->env = p->env;
      q->uploaded = false;
    }
  }
  const std::vector<int32_t> b = edge_split(p, n);
  std::vector<tp_status> st(n, TP_OK);
  std::vector<std::string> msg(n);
  std::vector<int> kinds(n, 0);
  std::vector<uint64_t> keys(n, ~0ull);
  auto work = [&](int i) {
    tp_plan* q = p->shards[i];
    cudaSetDevice(q->device);
    if (borrow && !q->arena) {
      q->arena = arena_pool_get(q->device);
      q->owns_arena = false;
      q->uploaded = false;
    }
    const int32_t e0 = b[i], e1 = b[i + 1];
    const int64_t off = q->edge_base[e0] - q->edge_base[0];
    const int64_t roff = q->row_base[e0] - q->row_base[0];
    tp_cost_tensors h = *host_out;
    if (i) h.node_intra_cost_s = h.node_intra_volume_bytes = h.node_memory_bytes = nullptr;
    auto sh = [](double* x, int64_t o) { return x ? x + o : nullptr; };
    h.edge_cost_s = sh(h.edge_cost_s, off);
    h.edge_volume_bytes = sh(h.edge_volume_bytes, off);
    h.edge_memory_bytes = sh(h.edge_memory_bytes, off);
    if (h.aux_edge_records) h.aux_edge_records = (char*)h.aux_edge_records + 40 * off;
    h.row_min_cost_s = sh(h.row_min_cost_s, roff);
    h.row_min_volume_bytes = sh(h.row_min_volume_bytes, roff);
    h.edge_pair_min_cost_s = sh(h.edge_pair_min_cost_s, e0);
    h.edge_pair_min_volume_bytes = sh(h.edge_pair_min_volume_bytes, e0);
    const tp_build_opts o{e0, e1, i != 0, q->device, nullptr};
    st[i] = execute_host_impl(q, &o, nullptr, &h, &keys[i]);
    if (st[i]) {
      msg[i] = g_err;
      kinds[i] = g_err_kind;
    }
    if (borrow && !q->owns_arena) {
      arena_pool_put(q->arena);
      q->arena = nullptr;
      q->owns_arena = true;
      q->uploaded = false;
      q->range_key = {{-1, -1, -1, -1}};
    }
  };
  run_pool(n, n, [&](int i, int) { work(i); });  // one pool worker per device (no thread spawns per call)
  for (int i = 0; i < n; ++i)
    if (st[i]) return set_err(st[i], kinds[i], msg[i]);
  uint64_t key = ~0ull;
  for (uint64_t k : keys) key = std::min(key, k);
  tp_status r = status_of_key(key);
  if (r) return r;
  if (index_out) tp_plan_index(p, index_out);
  g_err[0] = 0;
  g_err_kind = 0;
  return TP_OK;
}
}  // namespace

extern "C" {

tp_status tp_plan_execute_host_multi(tp_plan* p, const int32_t* devices, int32_t num_devices,
                                     tp_aux_index* index_out, tp_cost_tensors* host_out) {
  DeviceGuard dg;
  return execute_host_multi(p, devices, num_devices, index_out, host_out, false);
}

tp_status tp_build_cost_tensors_multi(const tp_graph_desc* graph, const tp_topology_desc* topo,
                                      const int32_t* devices, int32_t num_devices, tp_aux_index* index_out,
                                      tp_cost_tensors* host_out) {
  DeviceGuard dg;
  if (!devices || num_devices < 1) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "empty device list");
  tp_plan* p = nullptr;
  tp_status st = tp_plan_create(graph, topo, devices[0], &p);
  if (st) return st;
  st = execute_host_multi(p, devices, num_devices, index_out, host_out, true);
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

}  // extern "C"

namespace {
// One enqueued host batch (a whole call, or one chunk of a pipelined sweep).
struct HostBatch {
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};  // TP_PROFILE_HOST: compute start, built, drained
  tp_plan* const* plans = nullptr;
  int n = 0;
  std::vector<char> borrowed;
  std::vector<int> live;
  std::vector<BatchErr> errs;
  int64_t err_base = 0;  // this batch's error slots in B.d_err / B.h_err
  double t[4] = {0, 0, 0, 0};
  int64_t d2h_bytes = 0;
  void give_back() {
    for (int i = 0; i < n; ++i) {
      if (!borrowed[i]) continue;
      tp_plan* p = plans[i];
      p->arena = nullptr;
      p->owns_arena = true;
      p->uploaded = false;
      p->range_key = {{-1, -1, -1, -1}};
    }
  }
};


// Enqueue a batch of plans of one device without waiting for it: every
// plan's descriptors uploaded (borrowed arenas: ONE packed copy and two
// set-up launches) and the batched build on B.stream into the output staging
// of `slot`; the copies back (one per tensor kind where the caller's slices
// are contiguous) on B.copy_stream once the build is done. `slot` selects
// the staging halves, `arena_base` the first borrowed arena, `err_base` the
// error slots.
// `pre` (the pipelined sweep): every plan already on its borrowed arena with
// its descriptors prepared (upload_prepare with range length `min_range`).
tp_status host_batch_enqueue(BatchCtx& B, int device, tp_plan* const* plans, int32_t n, tp_cost_tensors* host_outs,
                             int32_t host_threads, int slot, int64_t arena_base, int64_t err_base, HostBatch& H,
                             std::vector<UploadPrep>* pre = nullptr, int64_t min_range = 0) {
  static const bool prof = getenv("TP_PROFILE_HOST") != nullptr;
  H.plans = plans;
  H.n = n;
  H.err_base = err_base;
  H.borrowed.assign(n, pre ? 1 : 0);
  H.errs.assign(n, BatchErr{});
  H.t[0] = prof ? now_us() : 0;
  while ((int64_t)B.host_arenas.size() < arena_base + n) {
    Arena* a = new Arena();
    a->device = device;
    B.host_arenas.push_back(a);
  }
  for (int i = 0; i < n && !pre; ++i) {
    tp_plan* p = plans[i];
    if (p->arena) continue;
    p->arena = B.host_arenas[arena_base + i];
    p->owns_arena = false;
    p->uploaded = false;
    H.borrowed[i] = 1;
  }
  if (!B.stream) CUDA_TRY(cudaStreamCreateWithFlags(&B.stream, cudaStreamNonBlocking));
  if (!B.copy_stream) CUDA_TRY(cudaStreamCreateWithFlags(&B.copy_stream, cudaStreamNonBlocking));
  for (int q = 0; q < 2; ++q) {
    if (!B.built[q]) CUDA_TRY(cudaEventCreateWithFlags(&B.built[q], cudaEventDisableTiming));
    if (!B.drained[q]) CUDA_TRY(cudaEventCreateWithFlags(&B.drained[q], cudaEventDisableTiming));
  }
  cudaStream_t s = B.stream;
  for (int i = 0; i < n; ++i) {
    tp_status st = ensure_stream(plans[i]);
    if (st) return st;
  }
  // uploads: plans on their own arenas the usual way; the borrowed ones in
  // ONE packed copy (descriptors packed by the workers) and two set-up launches
  for (int i = 0; i < n; ++i)
    if (!H.borrowed[i] && !plans[i]->uploaded) H.errs[i].take(tp_plan_upload(plans[i], s));
  std::vector<int> todo;
  for (int i = 0; i < n; ++i)
    if (H.borrowed[i]) todo.push_back(i);
  // as execute_batch_impl will decide (same outputs): with op lists no pair records are read
  const bool direct = batch_mode_of(plans, n, host_outs) != 0;
  std::vector<UploadPrep> U_own;
  const int64_t brange =
      min_range > 0 ? min_range : (direct ? batch_range_len(plans, n) : kFusedThreads * kFanPer);  // as execute_batch_impl
  if (!pre) {
    U_own.resize(todo.size());
    run_pool((int)todo.size(), host_threads,
             [&](int j, int) { H.errs[todo[j]].take(upload_prepare(plans[todo[j]], U_own[j], brange)); }, device);
  }
  std::vector<UploadPrep>& U = pre ? *pre : U_own;
  for (int i = 0; i < n; ++i)
    if (H.errs[i].st) return H.errs[i].st;
  if (!todo.empty()) {
    const int m = (int)todo.size();
    std::vector<size_t> off(m + 1, 0);
    for (int j = 0; j < m; ++j) off[j + 1] = off[j] + U[j].pk.total();
    const size_t jobs_at = (off[m] + 255) & ~(size_t)255;
    const size_t total = jobs_at + sizeof(UpJob) * m + 2 * sizeof(int64_t) * (m + 1);
    if (B.packed[slot]) CUDA_TRY(cudaEventSynchronize(B.packed[slot]));  // h_pack[slot] free again
    if (B.h_pack_cap[slot] < total) {
      if (B.h_pack[slot]) cudaFreeHost(B.h_pack[slot]);
      B.h_pack[slot] = nullptr;
      B.h_pack_cap[slot] = 0;
      CUDA_TRY(cudaMallocHost(&B.h_pack[slot], total));
      B.h_pack_cap[slot] = total;
    }
    CUDA_TRY(B.d_pack[slot].ensure(total));
    char* hp = (char*)B.h_pack[slot];
    char* dp = (char*)B.d_pack[slot].p;
    run_pool(
        m, host_threads,
        [&](int j, int) {
          tp_plan* p = plans[todo[j]];
          upload_stage(U[j], hp + off[j], dp + off[j]);
          H.errs[todo[j]].take(upload_finish(p, U[j]));
        },
        device);
    for (int i = 0; i < n; ++i)
      if (H.errs[i].st) return H.errs[i].st;
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
    if (!B.packed[slot]) CUDA_TRY(cudaEventCreateWithFlags(&B.packed[slot], cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(B.packed[slot], s));
    for (int j = 0; j < m; ++j) {
      tp_status st = upload_tables(plans[todo[j]], U[j], s);
      if (st) return st;
    }
    const UpJob* dj = (const UpJob*)(dp + jobs_at);
    const int64_t* dso = (const int64_t*)(dp + jobs_at + sizeof(UpJob) * m);
    if (so[m] > 0) batch_side_kernel<<<(unsigned)((so[m] + 127) / 128), 128, 0, s>>>(dj, m, dso);
    // a batch priced from op lists reads layouts through the descriptors, not pair records
    if (po[m] > 0 && !direct)
      batch_pair_rec_kernel<<<(unsigned)((po[m] + 127) / 128), 128, 0, s>>>(dj, m, dso + (m + 1));
    CUDA_TRY(cudaGetLastError());
  }
  H.t[1] = prof ? now_us() : 0;
  // outputs: device staging of this slot, drained by the copy stream
  std::vector<int64_t> nn(n), ne(n);
  int64_t tn = 0, te = 0;
  for (int i = 0; i < n; ++i) {
    nn[i] = plans[i]->num_aux_nodes;
    ne[i] = plans[i]->edge_base[plans[i]->valid_edges] - plans[i]->edge_base[0];
    tn += nn[i];
    te += ne[i];
  }
  auto host_ptr = [&](int i, int k) -> double* {
    const tp_cost_tensors& h = host_outs[i];
    double* const v[6] = {h.node_intra_cost_s, h.node_intra_volume_bytes, h.node_memory_bytes,
                          h.edge_cost_s,       h.edge_volume_bytes,       h.edge_memory_bytes};
    return v[k];
  };
  H.d2h_bytes = 0;
  for (int k = 0; k < 6; ++k)
    for (int i = 0; i < n; ++i)
      if (host_ptr(i, k)) H.d2h_bytes += (int64_t)sizeof(double) * (k < 3 ? nn[i] : ne[i]);
  // the build may write this half only after the copy stream drained its last use
  CUDA_TRY(cudaStreamWaitEvent(s, B.drained[slot], 0));
  if (prof) {
    for (auto& e : H.ev) CUDA_TRY(cudaEventCreate(&e));
    CUDA_TRY(cudaEventRecord(H.ev[0], s));
  }
  std::vector<tp_cost_tensors> dev(n);
  bool want[6];
  double* h_of[6];
  for (int k = 0; k < 6; ++k) {
    want[k] = false;
    for (int i = 0; i < n; ++i) want[k] |= host_ptr(i, k) != nullptr;
    const int64_t tot = k < 3 ? tn : te;
    if (want[k]) CUDA_TRY(B.out[slot][k].ensure(sizeof(double) * (size_t)std::max<int64_t>(tot, 1)));
    h_of[k] = (double*)B.out[slot][k].p;
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
  tp_status st = execute_batch_impl(plans, n, dev.data(), s, (unsigned long long*)B.d_err.p + err_base, &H.live, slot,
                                    min_range);
  if (st) return st;
  CUDA_TRY(cudaEventRecord(B.built[slot], s));
  H.t[2] = prof ? now_us() : 0;
  // back to the host on the copy stream: one copy per tensor kind where the caller's slices are contiguous
  cudaStream_t c = B.copy_stream;
  CUDA_TRY(cudaStreamWaitEvent(c, B.built[slot], 0));
  for (int k = 0; k < 6; ++k) {
    if (!want[k]) continue;
    bool contiguous = true;
    for (int i = 0; contiguous && i < n; ++i) {
      contiguous = host_ptr(i, k) != nullptr;
      if (contiguous && i + 1 < n) contiguous = host_ptr(i + 1, k) == host_ptr(i, k) + (k < 3 ? nn[i] : ne[i]);
    }
    const int64_t tot = k < 3 ? tn : te;
    if (contiguous) {
      if (tot > 0) CUDA_TRY(cudaMemcpyAsync(host_ptr(0, k), h_of[k], sizeof(double) * tot, cudaMemcpyDeviceToHost, c));
      continue;
    }
    int64_t off = 0;
    for (int i = 0; i < n; ++i) {
      const int64_t cnt = k < 3 ? nn[i] : ne[i];
      if (host_ptr(i, k) && cnt > 0)
        CUDA_TRY(cudaMemcpyAsync(host_ptr(i, k), h_of[k] + off, sizeof(double) * cnt, cudaMemcpyDeviceToHost, c));
      off += cnt;
    }
  }
  if (!H.live.empty())
    CUDA_TRY(cudaMemcpyAsync(B.h_err + err_base, (unsigned long long*)B.d_err.p + err_base,
                             sizeof(unsigned long long) * H.live.size(), cudaMemcpyDeviceToHost, c));
  CUDA_TRY(cudaEventRecord(B.drained[slot], c));
  if (prof) {
    CUDA_TRY(cudaEventRecord(H.ev[1], s));
    CUDA_TRY(cudaEventRecord(H.ev[2], c));
  }
  H.t[3] = prof ? now_us() : 0;
  return TP_OK;
}

// After the stream has passed the batch: statuses, index outputs, arenas back.
void host_batch_finish(BatchCtx& B, HostBatch& H, tp_aux_index* index_outs) {
  std::vector<unsigned long long> slot(H.n, 0);
  for (size_t k = 0; k < H.live.size(); ++k) slot[H.live[k]] = B.h_err[H.err_base + k];
  for (int i = 0; i < H.n; ++i) {
    if (!H.errs[i].st) H.errs[i].take(status_from_slot(H.plans[i], slot[i]));
    if (index_outs) tp_plan_index(H.plans[i], &index_outs[i]);
  }
  H.give_back();
}

tp_status ensure_err_slots(BatchCtx& B, int64_t n) {
  CUDA_TRY(B.d_err.ensure(sizeof(unsigned long long) * std::max<int64_t>(n, 1)));
  if (B.h_err_cap < (size_t)n) {
    if (B.h_err) cudaFreeHost(B.h_err);
    B.h_err = nullptr;
    B.h_err_cap = 0;
    CUDA_TRY(cudaMallocHost(&B.h_err, sizeof(unsigned long long) * std::max<int64_t>(n, 1)));
    B.h_err_cap = n;
  }
  return TP_OK;
}

bool needs_each(tp_plan* const* plans, int32_t n, const tp_cost_tensors* host_outs) {
  bool one_device = plans[0] != nullptr;
  for (int i = 0; one_device && i < n; ++i) one_device = plans[i] && plans[i]->device == plans[0]->device;
  // the batched launch writes the six SoA tensors only: AuxEdge records and
  // the solver minima go through one tp_plan_execute_host per plan
  bool extra = false;
  for (int i = 0; i < n; ++i) {
    const tp_cost_tensors& h = host_outs[i];
    extra |= h.aux_edge_records || h.row_min_cost_s || h.row_min_volume_bytes || h.edge_pair_min_cost_s ||
             h.edge_pair_min_volume_bytes;
  }
  return !one_device || extra || plans[0]->device < 0 || plans[0]->device >= 64;
}
}  // namespace

extern "C" {

tp_status tp_plan_execute_host_batch(tp_plan* const* plans, int32_t n, tp_aux_index* index_outs,
                                     tp_cost_tensors* host_outs, int32_t host_threads, int32_t* status_out) {
  DeviceGuard dg;
  if (n < 0 || (n > 0 && (!plans || !host_outs))) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null batch arrays");
  if (n == 0) return TP_OK;
  if (needs_each(plans, n, host_outs)) return execute_host_each(plans, n, index_outs, host_outs, host_threads, status_out);
  const int device = plans[0]->device;
  CUDA_TRY(cudaSetDevice(device));
  BatchCtx& B = g_batch[device];
  std::lock_guard<std::mutex> hl(B.host_mu);
  static const bool prof = getenv("TP_PROFILE_HOST") != nullptr;
  tp_status st = ensure_err_slots(B, n);
  if (st) return st;
  HostBatch H;
  st = host_batch_enqueue(B, device, plans, n, host_outs, host_threads, 0, 0, 0, H);
  if (st) {  // a failed upload is its plan's status; anything else fails the call
    cudaStreamSynchronize(B.stream);
    if (B.copy_stream) cudaStreamSynchronize(B.copy_stream);
    H.give_back();
    for (const BatchErr& e : H.errs)
      if (e.st) return batch_status(H.errs, status_out);
    return st;
  }
  CUDA_TRY(cudaStreamSynchronize(B.stream));
  CUDA_TRY(cudaStreamSynchronize(B.copy_stream));
  if (prof)
    fprintf(stderr, "[tp batch] %d plans: uploads %.0f us, launch prep %.0f, copies enqueued %.0f, wait %.0f\n", n,
            H.t[1] - H.t[0], H.t[2] - H.t[1], H.t[3] - H.t[2], now_us() - H.t[3]);
  host_batch_finish(B, H, index_outs);
  return batch_status(H.errs, status_out);
}

tp_status tp_build_cost_tensors_batch(const tp_graph_desc* const* graphs, const tp_topology_desc* const* topos,
                                      int32_t n, int32_t device, int32_t host_threads, tp_aux_index* index_outs,
                                      tp_cost_tensors* host_outs, int32_t* status_out) {
  DeviceGuard dg;
  if (n < 0 || (n > 0 && (!graphs || !topos || !host_outs)))
    return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null batch arrays");
  if (n == 0) return TP_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_err(TP_ERR_CUDA, 0, "no CUDA device: the engine has no CPU path");
  if (device < 0) CUDA_TRY(cudaGetDevice(&device));
  if (device >= ndev || device >= 64) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "device ordinal out of range");
  CUDA_TRY(cudaSetDevice(device));
  static const bool prof = getenv("TP_PROFILE_HOST") != nullptr;
  const double t0 = prof ? now_us() : 0;
  // Chunks of scenarios in a pipeline: the host analysis of chunk k + 1 (a
  // thread pool) runs while the GPU builds chunk k and streams it into the
  // caller's pinned memory; chunk k + 1's uploads queue behind it.
  static const int env_chunks = getenv("TP_SWEEP_CHUNKS") ? atoi(getenv("TP_SWEEP_CHUNKS")) : 0;
  // a few big scenarios (a sweep of one large graph under several bandwidths): one chunk each
  const int K = std::max(1, std::min<int>(n, env_chunks > 0 ? env_chunks
                                                            : (n <= 12 ? n : std::min(24, std::max(2, n / 40)))));
  // the first two chunks a quarter and a half of the others: the device and
  // the host link start after a short first analysis
  std::vector<int> cb(K + 1, 0);
  if (K >= 4) {
    const double unit = (double)n / (K - 2 + 0.75);
    cb[1] = std::max(1, (int)(0.25 * unit));
    cb[2] = std::max(cb[1] + 1, (int)(0.75 * unit));
    for (int k = 3; k <= K; ++k) cb[k] = cb[2] + (int)((int64_t)(n - cb[2]) * (k - 2) / (K - 2));
  } else {
    for (int k = 0; k <= K; ++k) cb[k] = (int)((int64_t)n * k / K);
  }
  std::vector<tp_plan*> plans(n, nullptr);
  std::vector<BatchErr> errs(n);
  BatchCtx& B = g_batch[device];
  std::lock_guard<std::mutex> hl(B.host_mu);
  tp_status st = ensure_err_slots(B, n);
  if (st) return st;
  while ((int64_t)B.host_arenas.size() < n) {  // scenario i borrows arena i
    Arena* a = new Arena();
    a->device = device;
    B.host_arenas.push_back(a);
  }
  // The analysis of a scenario also puts it on its arena and prepares its
  // descriptor pack (a fixed range length for the whole sweep, so the pack's
  // range table is the one the launch uses); chunk k's enqueue then only
  // copies the packs and launches.
  constexpr int64_t kSweepRange = 1024;
  std::vector<UploadPrep> prep(n);
  // Analysis threads: up to 8 (TP_SWEEP_THREADS to override). More finish
  // the analysis sooner but slow the host link and this thread's enqueues
  // (measured on cfg5, 16 cores: 15 threads 11.1-11.4 ms, 8 threads 10.0-10.1,
  // 4 threads 10.4-11.0).
  static const int env_threads = getenv("TP_SWEEP_THREADS") ? atoi(getenv("TP_SWEEP_THREADS")) : 0;
  const int analysis_threads =
      host_threads > 0 ? host_threads
      : env_threads > 0 ? env_threads
                        : std::max(2, std::min(8, (int)std::thread::hardware_concurrency() / 2));
  auto create = [&](int k) {
    run_pool(
        cb[k + 1] - cb[k], analysis_threads,
        [&](int j, int) {
          const int i = cb[k] + j;
          tp_plan* p = nullptr;
          errs[i].take(tp_plan_create(graphs[i], topos[i], device, &p));
          if (p) {
            p->arena = B.host_arenas[i];
            p->owns_arena = false;
            p->uploaded = false;
            tp_status s2 = ensure_stream(p);
            if (!s2) s2 = upload_prepare(p, prep[i], kSweepRange);
            if (!s2) class_keys(p);  // cached for the batch's inference dedup
            if (s2) {
              errs[i].take(s2);
              p->arena = nullptr;
              p->owns_arena = true;
              tp_plan_destroy(p);
              p = nullptr;
            }
          }
          plans[i] = p;
        },
        device);
  };
  std::vector<HostBatch> H(K);
  std::vector<char> enq(K, 0);
  // per chunk: the analysed plans (a failed analysis keeps its status)
  std::vector<std::vector<int>> ok_idx(K);
  std::vector<std::vector<tp_plan*>> ok_plans(K);
  std::vector<std::vector<tp_cost_tensors>> outs(K);
  std::vector<std::vector<UploadPrep>> preps(K);
  double t_create = 0;
  std::vector<double> tk(2 * K + 2, 0);  // per chunk: analysed, enqueued (TP_PROFILE_HOST)
  // The analysis runs ahead on its own thread (holding the worker pool) while
  // this thread enqueues the analysed chunks in order -- their set-up then
  // runs inline here instead of waiting for the pool.
  std::mutex amu;
  std::condition_variable acv;
  int analysed = 0;  // chunks [0, analysed) are ready
  bool stop = false;
  // retire[k]: chunk k's statuses taken and its plans destroyed (by the
  // analyser once its copies completed, overlapping the later chunks)
  std::vector<char> retired(K, 0);
  std::vector<cudaEvent_t> done(K, nullptr);
  for (auto& e : done) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  bool main_done = false, failed = false;
  auto destroy_chunk = [&](int k) {
    run_pool(cb[k + 1] - cb[k], host_threads, [&](int j, int) {
      tp_plan*& p = plans[cb[k] + j];
      tp_plan_destroy(p);
      p = nullptr;
    }, device);
  };
  std::thread analyser([&] {
    cudaSetDevice(device);
    for (int k = 0; k < K; ++k) {
      {
        std::lock_guard<std::mutex> lk(amu);
        if (stop) break;
      }
      const double c0 = prof ? now_us() : 0;
      create(k);
      std::lock_guard<std::mutex> lk(amu);
      if (prof) {
        t_create += now_us() - c0;
        tk[2 * k] = now_us() - t0;
      }
      analysed = k + 1;
      acv.notify_all();
    }
    for (int k = 0; k < K; ++k) {  // then retire the chunks as their copies complete
      {
        std::unique_lock<std::mutex> lk(amu);
        acv.wait(lk, [&] { return enq[k] || main_done; });
        if (!enq[k] || failed) break;
      }
      if (cudaEventSynchronize(done[k]) != cudaSuccess) break;
      host_batch_finish(B, H[k], nullptr);
      for (size_t j = 0; j < ok_idx[k].size(); ++j) {
        errs[ok_idx[k][j]] = H[k].errs[j];
        if (index_outs) tp_plan_index(plans[ok_idx[k][j]], &index_outs[ok_idx[k][j]]);
      }
      destroy_chunk(k);
      std::vector<UploadPrep>().swap(preps[k]);  // its packs went up with the chunk
      retired[k] = 1;
    }
  });
  for (int k = 0; k < K; ++k) {
    {
      std::unique_lock<std::mutex> lk(amu);
      acv.wait(lk, [&] { return analysed > k; });
    }
    for (int i = cb[k]; i < cb[k + 1]; ++i)
      if (plans[i]) {
        ok_idx[k].push_back(i);
        ok_plans[k].push_back(plans[i]);
        outs[k].push_back(host_outs[i]);
        preps[k].push_back(std::move(prep[i]));
      }
    bool queued = false;
    if (!ok_plans[k].empty()) {
      const int m = (int)ok_plans[k].size();
      if (needs_each(ok_plans[k].data(), m, outs[k].data())) {
        st = set_err(TP_ERR_INVALID_ARGUMENT, 0, "tp_build_cost_tensors_batch writes the six SoA tensors only");
        break;
      }
      // the pool is the analyser's while it analyses (then this chunk's set-up runs inline)
      st = host_batch_enqueue(B, device, ok_plans[k].data(), m, outs[k].data(), host_threads, k & 1, cb[k], cb[k],
                              H[k], &preps[k], kSweepRange);
      queued = true;
    } else {
      H[k].plans = ok_plans[k].data();  // nothing analysed in this chunk: nothing to finish
      H[k].n = 0;
    }
    if (st == TP_OK) {
      const cudaError_t ce = cudaEventRecord(done[k], B.copy_stream ? B.copy_stream : B.stream);
      if (ce != cudaSuccess) st = set_err(TP_ERR_CUDA, 0, cudaGetErrorString(ce));
    }
    {
      std::lock_guard<std::mutex> lk(amu);
      if (st) failed = true;
      enq[k] = queued || st == TP_OK;
      acv.notify_all();
    }
    if (prof) tk[2 * k + 1] = now_us() - t0;
    if (st) break;
  }
  {
    std::lock_guard<std::mutex> lk(amu);
    stop = true;
    main_done = true;
    acv.notify_all();
  }
  analyser.join();
  const double t_sync = prof ? now_us() : 0;
  cudaError_t ce = cudaStreamSynchronize(B.stream);
  const cudaError_t ce2 = B.copy_stream ? cudaStreamSynchronize(B.copy_stream) : cudaSuccess;
  if (ce == cudaSuccess) ce = ce2;
  for (int k = 0; k < K; ++k) {
    if (retired[k]) continue;
    if (enq[k] && H[k].n > 0) {
      if (st == TP_OK && ce == cudaSuccess) {
        host_batch_finish(B, H[k], nullptr);
        for (size_t j = 0; j < ok_idx[k].size(); ++j) {
          errs[ok_idx[k][j]] = H[k].errs[j];
          if (index_outs) tp_plan_index(plans[ok_idx[k][j]], &index_outs[ok_idx[k][j]]);
        }
      } else {
        H[k].give_back();
      }
    }
  }
  for (auto& e : done) cudaEventDestroy(e);
  run_pool(n, host_threads, [&](int i, int) { tp_plan_destroy(plans[i]); }, device);  // what is left
  if (prof) {
    fprintf(stderr, "[tp sweep] %d scenarios in %d chunks: %.0f us (analysis thread %.0f us; sync wait %.0f us)\n",
            n, K, now_us() - t0, t_create, now_us() - t_sync);
    for (int k = 0; k < K; ++k) {
      float a = -1, b = -1, c = -1;
      if (H[k].ev[0] && H[0].ev[0]) {
        cudaEventElapsedTime(&a, H[0].ev[0], H[k].ev[0]);
        cudaEventElapsedTime(&b, H[0].ev[0], H[k].ev[1]);
        cudaEventElapsedTime(&c, H[0].ev[0], H[k].ev[2]);
      }
      fprintf(stderr, "  chunk %d: analysed at %.0f us, enqueued at %.0f (uploads %.0f, launch prep %.0f, copies %.0f); "
              "device (from chunk 0 start): compute %.0f, built %.0f, drained %.0f us; %.1f MB\n", k, tk[2 * k],
              tk[2 * k + 1], H[k].t[1] - H[k].t[0], H[k].t[2] - H[k].t[1], H[k].t[3] - H[k].t[2], a * 1e3, b * 1e3,
              c * 1e3, H[k].d2h_bytes / 1e6);
    }
    for (auto& h : H)
      for (auto& e : h.ev)
        if (e) cudaEventDestroy(e);
  }
  if (st) return st;
  if (ce != cudaSuccess) return set_err(TP_ERR_CUDA, 0, cudaGetErrorString(ce));
  return batch_status(errs, status_out);
}

tp_status tp_plan_price_assignments(tp_plan* p, const tp_cost_tensors* t, const int32_t* assignments, int32_t k,
                                    double* cost_s, double* volume_bytes, double* memory_bytes, void* stream) {
  DeviceGuard dg;
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

tp_status tp_plan_export_lp(const tp_plan* p, const tp_cost_tensors* h, int32_t mode_volume, double device_memory,
                            const char* path, int64_t* bytes_out) {
  if (!p || !h || !path) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "null argument");
  if (p->host_err != ~0ull) return set_err(TP_ERR_INVALID_ARGUMENT, 0, "the plan's build has an error");
  if (!h->node_intra_cost_s || !h->node_intra_volume_bytes || !h->node_memory_bytes || !h->edge_cost_s ||
      !h->edge_volume_bytes || !h->edge_memory_bytes)
    return set_err(TP_ERR_INVALID_ARGUMENT, 0, "all six host cost tensors are needed");
  FILE* f = std::fopen(path, "wb");
  if (!f) return set_err(TP_ERR_INVALID_ARGUMENT, 0, std::string("cannot write '") + path + "'");
  taps_b200::LpInput in{p->num_ops,        p->num_edges,           p->node_base.data(),     p->edge_base.data(),
                        p->edge_from_op.data(), p->edge_to_op.data(), p->in_deg.data(),      p->out_deg.data(),
                        h->node_intra_cost_s, h->node_intra_volume_bytes, h->node_memory_bytes, h->edge_cost_s,
                        h->edge_volume_bytes, h->edge_memory_bytes};
  int64_t total = 0;
  bool ok = true;
  auto sink = [&](const char* d, size_t n) {
    ok = ok && std::fwrite(d, 1, n, f) == n;
    total += (int64_t)n;
  };
  taps_b200::write_lp(in, mode_volume != 0, device_memory, sink);
  ok = std::fclose(f) == 0 && ok;
  if (!ok) return set_err(TP_ERR_INVALID_ARGUMENT, 0, std::string("write to '") + path + "' failed");
  if (bytes_out) *bytes_out = total;
  return TP_OK;
}

tp_status tp_enumerate_strategies(int32_t p, int64_t total_devices, int64_t* count, int64_t* degrees,
                                  int32_t* device_map, int64_t* matrix_dims, int32_t* matrix_depth) {
  DeviceGuard dg;
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
  DeviceGuard dg;
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
