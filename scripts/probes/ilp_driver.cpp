// Offline driver for the exact selection solver (csrc/host/ilp.cpp): reads
// an instance written by STITCH_ILP_DUMP and solves it, printing the
// selection, the canonical total, the search statistics and the time.
//
//   make -C paper_1911_11576_b200/csrc
//   g++ -O2 -std=c++17 -Ipaper_1911_11576_b200/csrc scripts/probes/ilp_driver.cpp \
//       paper_1911_11576_b200/csrc/build/{ilp,ir,json}.o -o /tmp/ilp_driver
//   /tmp/ilp_driver /tmp/bert_ilp.8.txt [node_budget]
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "host/ilp.hpp"

using namespace stitch;

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s instance.txt [node_budget]\n", argv[0]);
    return 2;
  }
  FILE* f = std::fopen(argv[1], "r");
  if (!f) return 2;
  IlpInstance inst;
  size_t np = 0, nc = 0, nh = 0;
  if (std::fscanf(f, "%d %d %zu %zu %zu", &inst.num_vars, &inst.num_nodes, &np, &nc, &nh) != 5) return 3;
  inst.scores.resize(inst.num_vars);
  for (double& s : inst.scores)
    if (std::fscanf(f, "%la", &s) != 1) return 3;
  if (inst.num_nodes > 0) {
    inst.node_sets.resize(inst.num_vars);
    for (auto& ns : inst.node_sets) {
      size_t k = 0;
      if (std::fscanf(f, "%zu", &k) != 1) return 3;
      ns.resize(k);
      for (int& x : ns)
        if (std::fscanf(f, "%d", &x) != 1) return 3;
    }
  }
  inst.pairs.resize(np);
  for (auto& pc : inst.pairs)
    if (std::fscanf(f, "%d %d", &pc.u, &pc.v) != 2) return 3;
  inst.cycles.resize(nc);
  for (auto& cc : inst.cycles) {
    size_t k = 0;
    if (std::fscanf(f, "%zu", &k) != 1) return 3;
    cc.pattern_indices.resize(k);
    for (int& v : cc.pattern_indices)
      if (std::fscanf(f, "%d", &v) != 1) return 3;
  }
  inst.clique_hint.resize(nh);
  for (int& c : inst.clique_hint)
    if (std::fscanf(f, "%d", &c) != 1) return 3;
  std::fclose(f);
  if (argc > 2) set_ilp_node_budget(std::atoll(argv[2]));
  const auto t0 = std::chrono::steady_clock::now();
  FusionPlan p = solve(inst);
  const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const SolveStats& st = last_solve_stats();
  std::printf("vars %d nodes %d cycles %zu | selected %zu total %a (%.9f) | %.2fs nodes %lld queries %lld truncated %d "
              "lp_gap %.6f\n",
              inst.num_vars, inst.num_nodes, inst.cycles.size(), p.selected.size(), p.total_score, p.total_score, sec,
              (long long)st.nodes, (long long)st.queries, (int)st.truncated, st.lp_gap);
  for (int v : p.selected) std::printf("%d ", v);
  std::printf("\n");
  return 0;
}
