// Host compilation of the engine's per-thread algorithms (tp_core.cuh) — a
// development check only: lets the CPU test suite exercise the kernel logic
// against the oracle without a GPU. The product never runs this code on the
// host; the engine library has no CPU path.
#include <cstring>
#include "../../include/taps_b200.h"
#include "../../paper_2301_04285_b200/csrc/tp_core.cuh"

extern "C" int core_redistribute(const tp_redist_query* q, tp_redist_result* r) {
  std::memset(r, 0, sizeof(*r));
  tpk::QueryPOD p{};
  p.rank = q->rank;
  p.fdepth = q->from_depth;
  p.tdepth = q->to_depth;
  p.local = q->local_device_num;
  if (q->rank > tpk::kMaxR || q->from_depth > tpk::kMaxD || q->to_depth > tpk::kMaxD) return r->status = tpk::kCapacity;
  for (int i = 0; i < q->rank; ++i) { p.shape[i] = q->shape[i]; p.fmap[i] = q->from_map[i]; p.tmap[i] = q->to_map[i]; }
  for (int k = 0; k < q->from_depth; ++k) p.fdims[k] = q->from_dims[k];
  for (int k = 0; k < q->to_depth; ++k) p.tdims[k] = q->to_dims[k];
  p.bytes = q->tensor_bytes; p.intra = q->intra_bandwidth; p.inter = q->inter_bandwidth;
  r->status = tpk::run_query(p, *r);
  return r->status;
}

extern "C" int core_unrank(int p, int n, long long s, int* deg, int* dmap, int* mx, int* depth) {
  tpk::Strat st;
  tpk::unrank_strategy(p, n, s, st);
  for (int a = 0; a < p; ++a) { deg[a] = st.deg[a]; dmap[a] = st.dmap[a]; mx[a] = st.mx[a]; }
  *depth = st.depth;
  return 0;
}

#include "../../paper_2301_04285_b200/csrc/tp_fast.cuh"

// The register-resident pair path the kernels run (tp_fast.cuh).
extern "C" int core_redistribute_fast(const tp_redist_query* q, tp_redist_result* r) {
  std::memset(r, 0, sizeof(*r));
  tpk::QueryPOD p{};
  p.rank = q->rank;
  p.fdepth = q->from_depth;
  p.tdepth = q->to_depth;
  p.local = q->local_device_num;
  if (q->rank > tpk::kMaxR || q->from_depth > tpk::kMaxD || q->to_depth > tpk::kMaxD) return r->status = tpk::kCapacity;
  for (int i = 0; i < q->rank; ++i) { p.shape[i] = q->shape[i]; p.fmap[i] = q->from_map[i]; p.tmap[i] = q->to_map[i]; }
  for (int k = 0; k < q->from_depth; ++k) p.fdims[k] = q->from_dims[k];
  for (int k = 0; k < q->to_depth; ++k) p.tdims[k] = q->to_dims[k];
  p.bytes = q->tensor_bytes; p.intra = q->intra_bandwidth; p.inter = q->inter_bandwidth;
  tpk::FastTabs none{nullptr, nullptr};
  if (q->local_device_num == 2) {  // also exercise the table path
    static double bw[65], sc[17 * 17];
    const tpk::Env env{p.intra, p.inter, (int64_t)p.local};
    for (int ct = 0; ct < 65; ++ct) bw[ct] = tpk::eff_bw(ct, env);
    for (int ke = 0; ke < 17; ++ke)
      for (int pe = 0; pe < 17; ++pe)
        sc[ke * 17 + pe] = ke < pe ? (double)(1ll << ke) * (double)((1ll << pe) - (1ll << ke)) / (double)((1ll << pe) - 1) : 0.0;
    none = tpk::FastTabs{bw, sc};
  }
  r->status = tpk::run_query_fast(p, *r, none);
  return r->status;
}
