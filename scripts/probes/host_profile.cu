// Host-analysis probe: the engine's Builder on a dumped graph, no GPU needed.
#include "../../paper_2301_04285_b200/csrc/tp_engine.cu"
#include <cstdlib>
#include <vector>
template <typename T>
std::vector<T> rd(FILE* f) {
  int64_t n = 0;
  if (fread(&n, 8, 1, f) != 1) exit(2);
  std::vector<T> v(n);
  if (n && fread(v.data(), sizeof(T), n, f) != (size_t)n) exit(2);
  return v;
}
int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  int64_t hdr[4];
  double bw[3];
  if (fread(hdr, 8, 4, f) != 4 || fread(bw, 8, 3, f) != 3) return 2;
  auto op_id = rd<int32_t>(f), op_tb = rd<int32_t>(f), op_nin = rd<int32_t>(f), op_ab = rd<int32_t>(f),
       t_name = rd<int32_t>(f), t_sb = rd<int32_t>(f);
  auto shape = rd<int64_t>(f);
  auto t_es = rd<int32_t>(f), a_sb = rd<int32_t>(f), s_t = rd<int32_t>(f), s_d = rd<int32_t>(f),
       e_f = rd<int32_t>(f), e_t = rd<int32_t>(f), e_n = rd<int32_t>(f);
  tp_graph_desc g{(int32_t)hdr[0], op_id.data(), op_tb.data(), op_nin.data(), op_ab.data(), t_name.data(),
                  t_sb.data(), shape.data(), t_es.data(), a_sb.data(), s_t.data(), s_d.data(), (int32_t)hdr[1],
                  e_f.data(), e_t.data(), e_n.data()};
  tp_topology_desc t{(int32_t)hdr[2], (int32_t)hdr[3], bw[0], bw[1], bw[2]};
  const int reps = argc > 2 ? atoi(argv[2]) : 20;
  double best = 1e30;
  for (int r = 0; r < reps; ++r) {
    auto t0 = std::chrono::steady_clock::now();
    tp_plan* p = new tp_plan();
    Builder b{&g, &t, p};
    if (b.run() != TP_OK) return 3;
    auto t1 = std::chrono::steady_clock::now();
    best = std::min(best, std::chrono::duration<double, std::micro>(t1 - t0).count());
    delete p;
  }
  printf("best Builder::run %.0f us\n", best);
  return 0;
}
