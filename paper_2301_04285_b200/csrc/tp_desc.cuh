// tp_desc.cuh — error plumbing and the device descriptors of a plan
// (host-built, uploaded once).
// Part of the single translation unit tp_engine.cu (included from there, in order).
#pragma once

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

// Every entry point that may switch the current device restores the caller's
// on return (a PyTorch caller's current device must not follow the plan's).
// It also drops a stale runtime error left by an earlier unrelated call (the
// launches below check cudaGetLastError, which would report it as theirs).
struct DeviceGuard {
  int dev = -1;
  DeviceGuard() {
    (void)cudaGetLastError();
    if (cudaGetDevice(&dev) != cudaSuccess) dev = -1;
  }
  ~DeviceGuard() {
    int now = -1;
    if (dev >= 0 && cudaGetDevice(&now) == cudaSuccess && now != dev) cudaSetDevice(dev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

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
  // batches priced in the fan-out (op lists): the base class's bytes and
  // whether they come per entry from the overrides; the op lists of the base
  // class start at opb (filled in shared memory by the kernel)
  double bytes;
  int32_t ovr, pad;
  int64_t opb;
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
#ifndef TP_BATCH_FAN_PER
#define TP_BATCH_FAN_PER 4  // the same for a batch's second launch (fused_batch_kernel<5, 2>)
#endif

}  // namespace
