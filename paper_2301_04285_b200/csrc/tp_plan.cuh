// tp_plan.cuh — host side of a plan: device buffers, the descriptor pack,
// arenas, tp_plan, the host analysis (Builder) and the batch worker pool.
// Part of the single translation unit tp_engine.cu (included from there, in order).
#pragma once

namespace {

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
  DevBuf out[11];  // one-shot staging of the requested outputs
  DevBuf d_desc;  // the descriptor pack
  void* h_stage = nullptr;  // pinned staging of the pack
  size_t h_stage_cap = 0;
  cudaEvent_t stage_done = nullptr;  // the last pack copy out of h_stage
  bool sched_clean = false;  // Sched zero (set up, or left so by the last launch)
  bool tables_dirty = false; // a launch priced in the fan-out left the class tables un-reset
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
  std::vector<std::pair<uint64_t, std::vector<int64_t>>> class_keys;  // batches: op-list keys (cached)
  std::vector<tp_plan*> shards;  // per-device copies of a multi-device build (owned)
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


// Layout ids of a side's strategies (layout_tables): a pure function of the
// strategy table (p, log2 N) and the slicing, memoised for the process.
struct SideMemoKey {
  uint64_t a, b;
  bool operator==(const SideMemoKey& o) const { return a == o.a && b == o.b; }
};
struct SideMemoHash {
  size_t operator()(const SideMemoKey& k) const { return (size_t)((k.a * 0x9e3779b97f4a7c15ull) ^ k.b); }
};
std::mutex g_side_memo_mu;
std::unordered_map<SideMemoKey, std::pair<std::vector<int32_t>, std::vector<int32_t>>, SideMemoHash> g_side_memo;

bool side_memo_get(const uint64_t* k, std::vector<int32_t>& uid, std::vector<int32_t>& reps) {
  std::lock_guard<std::mutex> lk(g_side_memo_mu);
  auto it = g_side_memo.find(SideMemoKey{k[0], k[1]});
  if (it == g_side_memo.end()) return false;
  uid = it->second.first;
  reps = it->second.second;
  return true;
}

void side_memo_put(const uint64_t* k, const std::vector<int32_t>& uid, const std::vector<int32_t>& reps) {
  std::lock_guard<std::mutex> lk(g_side_memo_mu);
  if (g_side_memo.size() < 4096) g_side_memo.emplace(SideMemoKey{k[0], k[1]}, std::make_pair(uid, reps));
}

double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// The host analysis of one graph runs its per-op / per-edge passes on the
// worker pool from this many ops / edges on (TP_HOST_WORKERS: how many
// workers, default all).
// TP_HOST_PAR_MIN overrides the threshold (tests force the parallel passes).
const int kParallelItems = getenv("TP_HOST_PAR_MIN") ? std::max(1, atoi(getenv("TP_HOST_PAR_MIN"))) : 8192;
// workers for the host analysis of one graph (TP_HOST_WORKERS, default all)
int host_workers() {
  static const int w = getenv("TP_HOST_WORKERS") ? atoi(getenv("TP_HOST_WORKERS")) : 0;
  return w;
}

int pool_size(int n, int host_threads) {
  int t = host_threads > 0 ? host_threads : (int)std::min(32u, std::max(1u, std::thread::hardware_concurrency()));
  return std::max(1, std::min(t, n));
}

// A persistent pool of host workers: a sweep calls run_pool several times
// per chunk, and spawning 16 threads costs ~0.5 ms each time. Workers sleep
// on a condition variable between jobs. One job at a time: a caller that finds
// the pool busy (another device's batch on another thread) or that is itself
// a worker runs its items inline.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool* p = new HostPool();  // never destroyed: no join at process exit
    return *p;
  }
  int size() const { return (int)th_.size() + 1; }
  // fn(item, worker) over [0, n) on min(workers, size()) threads (the caller is worker 0)
  void run(int n, int workers, const std::function<void(int, int)>& fn, int device) {
    std::unique_lock<std::mutex> busy(run_mu_, std::try_to_lock);
    if (!busy.owns_lock() || t_in_worker) {
      for (int i = 0; i < n; ++i) fn(i, 0);
      return;
    }
    workers = std::max(1, std::min(workers, size()));
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      n_ = n;
      device_ = device;
      next_.store(0);
      want_ = workers - 1;
      running_ = workers - 1;
      ++gen_;
    }
    cv_.notify_all();
    for (int i = next_.fetch_add(1); i < n; i = next_.fetch_add(1)) fn(i, 0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return running_ == 0; });
    fn_ = nullptr;
  }

 private:
  HostPool() {
    const int hw = (int)std::min(32u, std::max(1u, std::thread::hardware_concurrency()));
    for (int w = 1; w < hw; ++w) th_.emplace_back([this, w] { loop(w); });
  }
  void loop(int w) {
    t_in_worker = true;
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      if (w > want_) continue;  // not needed for this job
      const std::function<void(int, int)>* fn = fn_;
      const int n = n_, device = device_;
      lk.unlock();
      // a new host thread starts on device 0, and a job may have switched it
      if (device >= 0) cudaSetDevice(device);
      for (int i = next_.fetch_add(1); i < n; i = next_.fetch_add(1)) (*fn)(i, w);
      lk.lock();
      if (--running_ == 0) done_.notify_all();
    }
  }
  static thread_local bool t_in_worker;
  std::vector<std::thread> th_;
  std::mutex run_mu_, mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int, int)>* fn_ = nullptr;
  int n_ = 0, device_ = -1, want_ = 0, running_ = 0;
  uint64_t gen_ = 0;
  std::atomic<int> next_{0};
};
thread_local bool HostPool::t_in_worker = false;

// fn(item, worker) over items [0, n), items claimed one at a time, on up to
// `workers` pool threads (pool_size) with `device` current.
template <typename F>
void run_pool(int n, int workers, F&& fn, int device = -1) {
  workers = pool_size(n, workers);
  if (workers <= 1) {
    for (int i = 0; i < n; ++i) fn(i, 0);
    return;
  }
  const std::function<void(int, int)> f = [&](int i, int w) { fn(i, w); };
  HostPool::get().run(n, workers, f, device);
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

// 64-bit key hash -> the first id with that hash (open addressing; callers
// chain equal hashes themselves and compare the keys)
struct HashIndex {
  std::vector<uint64_t> key;
  std::vector<int32_t> val;
  uint64_t mask = 0;
  void init(int n) {
    size_t cap = 16;
    while (cap < 2 * (size_t)std::max(n, 1)) cap <<= 1;
    key.assign(cap, 0);
    val.assign(cap, -1);
    mask = cap - 1;
  }
  // the head for hash h (-1 when new; assign to insert)
  int32_t& at(uint64_t h) {
    for (uint64_t i = (h ^ (h >> 31)) & mask;; i = (i + 1) & mask) {
      if (val[i] < 0) {
        key[i] = h;
        return val[i];
      }
      if (key[i] == h) return val[i];
    }
  }
};

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
  // the last occurrence's spec winning (layout.hpp:339-347). Op i's slots sit
  // at its first tensor index op_tensor_begin[i] (at most one slot per
  // tensor), slot_cnt[i] of them, so every op fills its own span in parallel.
  std::vector<int32_t> slot_cnt, slot_name, slot_spec;
  std::vector<std::array<int8_t, tpk::kMaxR>> slot_sa;  // tensor dim -> slicing axis, per slot
  int find_slot(int op, int nm) const {  // local slot index of tensor name nm, or -1
    const int b = g->op_tensor_begin[op], e = b + slot_cnt[op];
    for (int i = b; i < e; ++i)
      if (slot_name[i] == nm) return i - b;
    return -1;
  }
  int spec_of(int op, int k) const { return slot_spec[g->op_tensor_begin[op] + k]; }
  const std::array<int8_t, tpk::kMaxR>& sa_of(int op, int k) const { return slot_sa[g->op_tensor_begin[op] + k]; }
  std::map<int, int64_t> table_of_p;
  // node classes by key hash: first class with a hash, then a chain per class
  HashIndex class_head;
  std::vector<int32_t> class_next;
  std::vector<int32_t> class_nslot;
  // every op's node-class key parts, where build_op puts them: slice checks
  // at the op's first slice index, slot descriptors and occurrences at its
  // first tensor index; with the key's hash
  std::vector<SliceChk> chk_all;
  std::vector<SlotDesc> slots_all;
  std::vector<Occ> occ_all;
  std::vector<uint64_t> op_hash;
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
    const int nops = g->num_ops;
    wrow_of_op.assign(nops, 0);
    p.op_row.assign(nops, 0);
    // In operator order: the aux node ids, the strategy tables, and where the
    // reference would stop (a non-power-of-two mesh or an op without axes ends
    // the node phase; a capacity limit fails the call after the ops before it).
    int64_t nodes = 0;
    int lim = nops, lim_ek = 0;
    BatchErr lim_err;
    for (int i = 0; i < nops; ++i) {
      p.node_base[i] = nodes;
      const int np = g->op_axis_begin[i + 1] - g->op_axis_begin[i];
      const int ek = !pow2 ? tpk::kNotPow2 : (np < 1 ? tpk::kNoAxes : 0);
      if (ek) {
        lim = i;
        lim_ek = ek;
        break;
      }
      if (np > tpk::kMaxAxes) {
        lim = i;
        lim_err.take(set_err(TP_ERR_CAPACITY, tpk::kCapacity, "operator with more than 8 axes"));
        break;
      }
      const int64_t S = tpk::strategy_count(np, p.n_log2);
      if (S > (1 << 20)) {
        lim = i;
        lim_err.take(set_err(TP_ERR_CAPACITY, tpk::kCapacity, "more than 2^20 strategies per operator"));
        break;
      }
      if (!table_of_p.count(np)) {
        table_of_p[np] = p.table_total;
        p.tabs.push_back(TableDesc{p.table_total, S, np, p.n_log2});
        p.table_total += S;
      }
      nodes += S;
    }
    for (int i = lim; i <= nops; ++i) p.node_base[i] = nodes;
    // every op's slots and class key, independently (in parallel for big graphs)
    {
      const int nt = num_tensors();
      const int nslices = nops > 0 && g->op_axis_begin[nops] > 0 ? g->axis_slice_begin[g->op_axis_begin[nops]] : 0;
      slot_cnt.assign(nops, 0);
      slot_name.resize(nt);
      slot_spec.resize(nt);
      slot_sa.resize(nt);
      chk_all.resize(nslices);
      slots_all.resize(nt);
      occ_all.resize(nt);
      op_hash.resize(nops);
      std::vector<BatchErr> op_err(lim);
      // (measured: the pool's dispatch costs more than it saves below a few
      // thousand ops -- cfg4's 1,152 ops take ~155 us on one thread)
      const int kOpsPerItem = std::max(1, std::min(256, kParallelItems / 32));
      const bool par = lim >= kParallelItems && lim > kOpsPerItem;
      run_pool(par ? (lim + kOpsPerItem - 1) / kOpsPerItem : 1, host_workers(), [&](int it, int) {
        const int i1 = par ? std::min(lim, (it + 1) * kOpsPerItem) : lim;
        for (int i = par ? it * kOpsPerItem : 0; i < i1; ++i)
          op_err[i].take(build_op(i, g->op_axis_begin[i + 1] - g->op_axis_begin[i]));
      });
      for (int i = 0; i < lim; ++i)  // the first failing op, in order
        if (op_err[i].st) return set_err(op_err[i].st, op_err[i].kind, op_err[i].msg);
    }
    if (lim_err.st) return set_err(lim_err.st, lim_err.kind, lim_err.msg);
    if (lim_ek) p.host_err = ekey(1 + (uint64_t)nodes * 2, lim_ek);
    p.valid_ops = lim;
    // node classes, in operator order (first member first)
    class_head.init(lim);
    for (int i = 0; i < lim; ++i) add_to_class(i, g->op_axis_begin[i + 1] - g->op_axis_begin[i],
                                               p.node_base[i + 1] - p.node_base[i], p.node_base[i]);
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
    HashIndex sig_head;  // key hash -> first class; chains below
    std::vector<int32_t> sig_next, sig_pu, sig_pw;
    std::vector<int64_t> sig_shape;  // kMaxR extents per class
    std::vector<int32_t> sig_of_edge;
    const int kEdgesPerItem = std::max(1, std::min(512, kParallelItems / 16));
    if (p.host_err == ~0ull) {
      // every edge's slots, checks and class-key hash, independently (in
      // parallel for big graphs); then the classes and aux ids in edge order
      struct EdgePre {
        int32_t ku, kw, tu, R, pu, pw, tab_u, tab_w;
        int64_t Su, Sw;
        double bytes;
        uint64_t h;
        int32_t stop;  // 0, or why the reference stops at this edge (1 dangling, 2 tensor missing, 3 shape, 4 capacity)
      };
      const int ne = g->num_edges;
      std::vector<EdgePre> pre(ne);
      sig_of_edge.resize(ne);
      auto edge_pre = [&](int e) {
        EdgePre& x = pre[e];
        x.stop = 0;
        const int u = p.edge_from_op[e], w = p.edge_to_op[e];
        if (u < 0 || w < 0) {
          x.stop = 1;
          return;
        }
        x.ku = find_slot(u, g->edge_tensor[e]);
        x.kw = find_slot(w, g->edge_tensor[e]);
        if (x.ku < 0 || x.kw < 0) {
          x.stop = 2;
          return;
        }
        const int tu = spec_of(u, x.ku), tw = spec_of(w, x.kw);
        const int R = rank_of(tu);
        bool same_shape = R == rank_of(tw);
        for (int d = 0; same_shape && d < R; ++d) same_shape = shape_of(tu)[d] == shape_of(tw)[d];
        if (!same_shape) {
          x.stop = 3;
          return;
        }
        x.tu = tu;
        x.R = R;
        x.pu = g->op_axis_begin[u + 1] - g->op_axis_begin[u];
        x.pw = g->op_axis_begin[w + 1] - g->op_axis_begin[w];
        x.tab_u = (int32_t)table_of_p.find(x.pu)->second;
        x.tab_w = (int32_t)table_of_p.find(x.pw)->second;
        x.Su = p.node_base[u + 1] - p.node_base[u];
        x.Sw = p.node_base[w + 1] - p.node_base[w];
        if (x.Su * x.Sw >= ((int64_t)1 << 31) - 4096) {
          x.stop = 4;
          return;
        }
        int64_t elements = 1;
        for (int d = 0; d < R; ++d) elements *= shape_of(tu)[d];
        x.bytes = (double)elements * g->tensor_element_size[tu];  // graph.hpp:52-54
        // edge class key (the reference's memo key, aux_graph.hpp:257-271, plus
        // the bytes and axis counts): hashed, compared field by field on a hit
        int64_t bbits;
        std::memcpy(&bbits, &x.bytes, 8);
        uint64_t h = hash_words(0x51ed27f3c6a8b9d1ull ^ ((uint64_t)x.pu << 40) ^ ((uint64_t)x.pw << 20) ^ (uint64_t)R,
                                &bbits, 8);
        h = hash_words(h, shape_of(tu), sizeof(int64_t) * R);
        h = hash_words(h, sa_of(u, x.ku).data(), R);
        x.h = hash_words(h, sa_of(w, x.kw).data(), R);
      };
      if (ne >= kParallelItems)
        run_pool((ne + kEdgesPerItem - 1) / kEdgesPerItem, host_workers(), [&](int it, int) {
          for (int e = it * kEdgesPerItem; e < std::min(ne, (it + 1) * kEdgesPerItem); ++e) edge_pre(e);
        });
      else
        for (int e = 0; e < ne; ++e) edge_pre(e);
      sig_head.init(ne);
      p.edges.reserve(ne);
      p.valid_edges = ne;
      for (int e = 0; e < ne; ++e) {
        p.edge_base[e] = aux;
        p.row_base[e] = rows;
        const EdgePre& x = pre[e];
        if (x.stop) {
          if (x.stop == 4) return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "more than 2^31 pairs on one edge");
          p.host_err = ekey(kEdgePhase + (uint64_t)aux * 2 + (x.stop == 3 ? 1 : 0),
                            x.stop == 1 ? tpk::kDangling : (x.stop == 2 ? tpk::kEdgeTensorMissing : tpk::kShapeMismatch));
          p.valid_edges = e;
          break;
        }
        const int u = p.edge_from_op[e], w = p.edge_to_op[e];
        const int ku = x.ku, kw = x.kw, tu = x.tu, R = x.R, pu = x.pu, pw = x.pw;
        const int64_t Su = x.Su, Sw = x.Sw;
        const double bytes = x.bytes;
        const auto& sau = sa_of(u, ku);
        const auto& saw = sa_of(w, kw);
        int32_t& head = sig_head.at(x.h);
        int32_t sig = -1;
        for (int32_t c = head; c >= 0; c = sig_next[c]) {
          const SigDesc& o = p.sigs[c];
          if (o.R == R && o.tab_u == x.tab_u && o.tab_w == x.tab_w &&
              sig_pu[c] == pu && sig_pw[c] == pw && !std::memcmp(&o.bytes, &bytes, 8) &&
              !std::memcmp(sig_shape.data() + (size_t)c * tpk::kMaxR, shape_of(tu), sizeof(int64_t) * R) &&
              !std::memcmp(o.sa_u, sau.data(), R) && !std::memcmp(o.sa_w, saw.data(), R)) {
            sig = c;
            break;
          }
        }
        if (sig < 0) {
          sig = (int32_t)p.sigs.size();
          sig_next.push_back(head);
          head = sig;
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
          sd.tab_u = x.tab_u;
          sd.tab_w = x.tab_w;
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
          p.total_pairs += Su * Sw;
        }
        sig_of_edge[e] = sig;
        aux += Su * Sw;
        rows += Su;
      }
      for (int e = p.valid_edges; e <= g->num_edges; ++e) {
        p.edge_base[e] = aux;
        p.row_base[e] = rows;
      }
      // the edge descriptors (independent per edge)
      const int nv = p.valid_edges;
      p.edges.resize(nv);
      auto edge_desc = [&](int e) {
        EdgeDesc ed{};
        const int u = p.edge_from_op[e], w = p.edge_to_op[e];
        ed.aux_base = p.edge_base[e];
        ed.nb_u = p.node_base[u];
        ed.nb_w = p.node_base[w];
        ed.wrow = wrow_of_op[w];
        ed.sig = sig_of_edge[e];
        ed.e = e;
        p.edges[e] = ed;
      };
      if (nv >= kParallelItems)
        run_pool((nv + kEdgesPerItem - 1) / kEdgesPerItem, host_workers(), [&](int it, int) {
          for (int e = it * kEdgesPerItem; e < std::min(nv, (it + 1) * kEdgesPerItem); ++e) edge_desc(e);
        });
      else
        for (int e = 0; e < nv; ++e) edge_desc(e);
      // edges by class, edge order within (counting sort)
      p.sig_edge_begin.assign(p.sigs.size() + 1, 0);
      for (int e = 0; e < nv; ++e) ++p.sig_edge_begin[sig_of_edge[e] + 1];
      for (size_t c = 0; c < p.sigs.size(); ++c) p.sig_edge_begin[c + 1] += p.sig_edge_begin[c];
      p.sig_edges.resize(nv);
      std::vector<int32_t> fill(p.sig_edge_begin.begin(), p.sig_edge_begin.end() - 1);
      for (int e = 0; e < nv; ++e) p.sig_edges[fill[sig_of_edge[e]]++] = e;
    }
    p.num_aux_edges = aux;
    p.num_rows = rows;
    if (p.sig_edge_begin.empty()) p.sig_edge_begin.push_back(0);
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
    p.fsegs.resize(p.edges.size());
    auto fan_seg = [&](size_t e) {
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
      f.bytes = bs.bytes;
      f.ovr = bs.has_override;
      p.fsegs[e] = f;
    };
    const int nseg = (int)p.edges.size();
    if (nseg >= kParallelItems)
      run_pool((nseg + kEdgesPerItem - 1) / kEdgesPerItem, host_workers(), [&](int it, int) {
        for (int e = it * kEdgesPerItem; e < std::min(nseg, (it + 1) * kEdgesPerItem); ++e) fan_seg(e);
      });
    else
      for (int e = 0; e < nseg; ++e) fan_seg(e);
    const double tc7 = prof ? clk() : 0;
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
      fprintf(stderr, "[tp host] check %.0f us, graph %.0f, node phase %.0f, edge phase %.0f, memo %.0f, tables %.0f, "
              "fan-out segments %.0f, rest %.0f\n", tc1 - tc0, tc2 - tc1, tc3 - tc2, tc4 - tc3, tc5 - tc4, tc6 - tc5,
              tc7 - tc6, clk() - tc7);
    p.h2d_bytes = (int64_t)(p.tabs.size() * sizeof(TableDesc) + p.classes.size() * sizeof(ClassDesc) +
                            p.members.size() * sizeof(int64_t) + p.chks.size() * sizeof(SliceChk) +
                            p.slots.size() * sizeof(SlotDesc) + p.occs.size() * sizeof(Occ) +
                            p.sigs.size() * sizeof(SigDesc) + p.edges.size() * sizeof(EdgeDesc) +
                            p.side_jobs.size() * sizeof(SideJob) +
                            p.overrides.size() * sizeof(double) + p.maps.size() * sizeof(int32_t) +
                            (p.pair_sig.size() + p.row_cls.size()) * sizeof(int32_t));
    return st;
  }

  // Slots, slice checks, occurrences of op i and the hash of its node-class
  // key, each written into the op's own spans (no shared state: ops run in
  // parallel). The first error in the reference's order is returned.
  tp_status build_op(int i, int np) {
    const tp_plan& p = *P;
    const int t0 = g->op_tensor_begin[i], t1 = g->op_tensor_begin[i + 1];
    int32_t* nm = slot_name.data() + t0;
    int32_t* sp = slot_spec.data() + t0;
    int n = 0;
    for (int t = t0; t < t1; ++t) {
      int k = -1;
      for (int x = 0; x < n; ++x)
        if (nm[x] == g->tensor_name[t]) k = x;
      if (k < 0) {
        k = n++;
        nm[k] = g->tensor_name[t];
      }
      sp[k] = t;
      if (rank_of(t) > tpk::kMaxR) return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "tensor rank above 8");
      for (int d = 0; d < rank_of(t); ++d)
        if (shape_of(t)[d] < 1) return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "tensor extent < 1 is unsupported");
    }
    if (n > 32000) return set_err(TP_ERR_CAPACITY, tpk::kCapacity, "too many tensors per op");
    slot_cnt[i] = n;
    std::array<int8_t, tpk::kMaxR>* sa = slot_sa.data() + t0;
    for (int k = 0; k < n; ++k) sa[k].fill(-1);
    const int a0 = g->op_axis_begin[i];
    const int s0 = np > 0 ? g->axis_slice_begin[a0] : 0;
    const int s1 = np > 0 ? g->axis_slice_begin[a0 + np] : 0;
    SliceChk* chk = chk_all.data() + s0;
    for (int a = 0; a < np; ++a) {
      for (int s = g->axis_slice_begin[a0 + a]; s < g->axis_slice_begin[a0 + a + 1]; ++s) {
        const int k = find_slot(i, g->slice_tensor[s]);
        SliceChk c{};
        c.axis = (int8_t)a;
        c.slot = (int16_t)k;
        c.v = 0;
        if (k >= 0) {
          const int dim = g->slice_dim[s];
          const int tk = sp[k];
          if (dim < 0 || dim >= rank_of(tk))
            return set_err(TP_ERR_INVALID_ARGUMENT, 0, "slice dimension out of range");
          c.v = (int8_t)v2_capped(shape_of(tk)[dim]);
          sa[k][dim] = (int8_t)a;  // later slices overwrite (layout.hpp:366)
        }
        chk[s - s0] = c;
      }
    }
    SlotDesc* slots = slots_all.data() + t0;
    for (int k = 0; k < n; ++k) {
      SlotDesc sd{};
      const int tk = sp[k];
      int64_t el = 1;
      for (int d = 0; d < rank_of(tk); ++d) el *= shape_of(tk)[d];
      sd.elements = el;
      sd.es = g->tensor_element_size[tk];
      sd.R = (int8_t)rank_of(tk);
      for (int d = 0; d < tpk::kMaxR; ++d) sd.sa[d] = sa[k][d];
      slots[k] = sd;
    }
    Occ* occ = occ_all.data() + t0;
    const int nin = g->op_num_inputs[i];
    const int32_t* fed0 = fed_list.data() + fed_begin[op_key[i]];
    const int32_t* fed1 = fed_list.data() + fed_begin[op_key[i] + 1];
    for (int t = t0; t < t1; ++t) {
      Occ oc{};
      const int name = g->tensor_name[t];
      oc.slot = (int16_t)find_slot(i, name);
      uint8_t mask = 0;
      for (int a = 0; a < np; ++a) {
        bool slices = false;
        for (int s = g->axis_slice_begin[a0 + a]; s < g->axis_slice_begin[a0 + a + 1]; ++s)
          slices |= g->slice_tensor[s] == name;
        if (!slices) mask |= (uint8_t)(1u << a);
      }
      oc.nonslicing = mask;
      if (t - t0 < nin) {
        bool fed = false;  // aux_graph.hpp:155-162
        for (const int32_t* x = fed0; x < fed1; ++x) fed |= *x == name;
        oc.in_memory = !fed;
      } else {
        oc.in_memory = 1;
      }
      occ[t - t0] = oc;
    }
    // node class key: everything the per-node costs depend on -- the axis
    // count, the in-degree and the slice checks, slots and occurrences (POD,
    // padding zeroed), hashed as words and compared bytewise on a hit
    const size_t nchk = (size_t)(s1 - s0), nocc = (size_t)(t1 - t0);
    uint64_t h = hash_words(0x9e3779b97f4a7c15ull ^ ((uint64_t)np << 32) ^ (uint64_t)(uint32_t)p.in_deg[i], chk,
                            nchk * sizeof(SliceChk));
    h = hash_words(h ^ nchk, slots, (size_t)n * sizeof(SlotDesc));
    op_hash[i] = hash_words(h ^ (size_t)n, occ, nocc * sizeof(Occ));
    return TP_OK;
  }

  // Op i (aux nodes [nb, nb + S)) joins its node class, a new one if no
  // earlier op had an equal key.
  void add_to_class(int i, int np, int64_t S, int64_t nb) {
    tp_plan& p = *P;
    const int t0 = g->op_tensor_begin[i];
    const int s0 = np > 0 ? g->axis_slice_begin[g->op_axis_begin[i]] : 0;
    const int nchk = np > 0 ? g->axis_slice_begin[g->op_axis_begin[i] + np] - s0 : 0;
    const int nslot = slot_cnt[i], nocc = g->op_tensor_begin[i + 1] - t0;
    const SliceChk* chk = chk_all.data() + s0;
    const SlotDesc* slots = slots_all.data() + t0;
    const Occ* occ = occ_all.data() + t0;
    int32_t& head = class_head.at(op_hash[i]);
    int32_t cls = -1;
    for (int32_t c = head; c >= 0; c = class_next[c]) {
      const ClassDesc& cd = p.classes[c];
      if (cd.p == np && cd.indeg == (double)p.in_deg[i] && cd.chk_end - cd.chk_begin == nchk &&
          class_nslot[c] == nslot && cd.occ_end - cd.occ_begin == nocc &&
          !std::memcmp(p.chks.data() + cd.chk_begin, chk, nchk * sizeof(SliceChk)) &&
          !std::memcmp(p.slots.data() + cd.slot_begin, slots, nslot * sizeof(SlotDesc)) &&
          !std::memcmp(p.occs.data() + cd.occ_begin, occ, nocc * sizeof(Occ))) {
        cls = c;
        break;
      }
    }
    if (cls < 0) {
      cls = (int32_t)p.classes.size();
      class_next.push_back(head);
      head = cls;
      class_nslot.push_back(nslot);
      ClassDesc cd{};
      cd.row_base = p.total_rows;
      cd.first_node = nb;
      cd.indeg = (double)p.in_deg[i];
      cd.S = (int32_t)S;
      cd.p = np;
      cd.table = (int32_t)table_of_p[np];
      cd.chk_begin = (int32_t)p.chks.size();
      p.chks.insert(p.chks.end(), chk, chk + nchk);
      cd.chk_end = (int32_t)p.chks.size();
      cd.slot_begin = (int32_t)p.slots.size();
      p.slots.insert(p.slots.end(), slots, slots + nslot);
      cd.occ_begin = (int32_t)p.occs.size();
      p.occs.insert(p.occs.end(), occ, occ + nocc);
      cd.occ_end = (int32_t)p.occs.size();
      p.classes.push_back(cd);
      class_members.emplace_back();
      p.total_rows += S;
    }
    class_members[cls].push_back(nb);
    wrow_of_op[i] = p.classes[cls].row_base;
    p.op_row[i] = p.classes[cls].row_base;
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
        // a pure function of (p, log2 N, the slicing): memoised process-wide
        // (sweeps repeat a handful of sides over many scenarios)
        uint64_t ck[2] = {(uint64_t)td->p | ((uint64_t)td->n << 8) | ((uint64_t)R << 16), 0};
        for (int d = 0; d < R; ++d) ck[1] |= (uint64_t)(uint8_t)sa[d] << (8 * d);
        if (side_memo_get(ck, uid, reps)) goto have_maps;
        {
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
        }
        side_memo_put(ck, uid, reps);
      } else {
        for (int32_t s = 0; s < S; ++s) uid[s] = s, reps.push_back(s);
      }
    have_maps:
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

}  // namespace

