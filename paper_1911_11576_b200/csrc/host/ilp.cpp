// Exact 0/1 selection with cycle elimination.
//
// Answer contract (reference proj/src/ilp_solver.cpp:139 solve):
//   optimum  = max over feasible selections S of canonical(S), where
//              canonical(S) sums scores in ascending variable order;
//   selected = lexicographically smallest feasible S with canonical(S) ==
//              optimum, built index by index preferring "stop here", then
//              "include", then "exclude" (ilp_solver.cpp:153-167).
// Cycle elimination (ilp_solver.cpp:175) adds sum_{i in witness} X_i <= |S|-1
// for the patterns on contract_plan's witness cycle and re-solves.
#include "ilp.hpp"

#include <algorithm>
#include <chrono>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <limits>
#include <map>
#include <numeric>

namespace stitch {

namespace {

thread_local SolveStats g_stats;
constexpr double kNegInf = -std::numeric_limits<double>::infinity();

// Node prices y >= 0 with sum_{x in P} y_x >= s_P for every pattern P: a
// feasible dual of the set-packing LP  max s.x, sum_{P covers x} x_P <= 1,
// so any feasible selection of the patterns totals at most sum_x y_x (and
// any sub-selection avoiding some nodes at most the sum over the rest).
// Solved with a revised primal simplex (Dantzig pricing, Bland's rule after
// degenerate stalls); the duals are then repaired so feasibility holds
// exactly whatever the floating-point error. Instances here are small (one
// connected component: hundreds of nodes, thousands of patterns), and the
// LP relaxation is usually integral, so the bound closes the search at once.
std::vector<double> lp_node_prices(const std::vector<std::vector<int>>& sets, const std::vector<double>& s, int num_nodes,
                                   std::vector<double>* primal = nullptr) {
  // Revised simplex with an explicit dense basis inverse (m x m, m = graph
  // nodes touched) and sparse 0/1 columns: O(m^2 + nnz) per pivot.
  std::vector<int> rows;
  std::vector<int> row_of(num_nodes, -1);
  for (const auto& p : sets)
    for (int x : p)
      if (row_of[x] < 0) {
        row_of[x] = static_cast<int>(rows.size());
        rows.push_back(x);
      }
  const int m = static_cast<int>(rows.size()), n = static_cast<int>(sets.size());
  std::vector<double> y(num_nodes, 0.0);
  auto ratio_prices = [&]() {
    std::fill(y.begin(), y.end(), 0.0);
    for (int j = 0; j < n; ++j)
      for (int x : sets[j]) y[x] = std::max(y[x], s[j] / std::max<size_t>(1, sets[j].size()));
    if (primal) primal->assign(n, 0.0);
  };
  if (m == 0 || n == 0 || m > 4096) {
    ratio_prices();
    return y;
  }
  std::vector<std::vector<int>> col(n);
  for (int j = 0; j < n; ++j)
    for (int x : sets[j]) col[j].push_back(row_of[x]);
  // Right-hand side perturbed per row (1 + 1e-7 .. 2e-7): set-packing LPs
  // are massively primal-degenerate and the unperturbed simplex stalls for
  // hundreds of thousands of pivots; on the perturbed one every ratio test
  // makes progress. The final basis is re-evaluated on the true b = 1.
  std::vector<double> Binv(static_cast<size_t>(m) * m, 0.0), xb(m, 1.0), cb(m, 0.0), dual(m, 0.0), d(m);
  for (int i = 0; i < m; ++i) xb[i] = 1.0 + 1e-7 * (1.0 + ((i * 2654435761u) % 1024) / 1024.0);
  for (int i = 0; i < m; ++i) Binv[static_cast<size_t>(i) * m + i] = 1.0;
  std::vector<int> basis(m);
  for (int i = 0; i < m; ++i) basis[i] = n + i;  // slacks
  const double eps = 1e-9;
  int stall = 0;
  bool optimal = false;
  // Iteration cap: degenerate whole-graph LPs can pivot for a long time; on
  // a miss the max-ratio prices (weaker, still valid) are used instead.
  int lp_iters = 0;
  for (int iter = 0; iter < 20 * m + 2000; ++iter, ++lp_iters) {
    // duals: dual = cb^T Binv
    for (int k = 0; k < m; ++k) dual[k] = 0.0;
    for (int i = 0; i < m; ++i)
      if (cb[i] != 0.0) {
        const double* bi = &Binv[static_cast<size_t>(i) * m];
        for (int k = 0; k < m; ++k) dual[k] += cb[i] * bi[k];
      }
    // pricing (Dantzig; Bland's lowest index while degenerate pivots stall)
    int e = -1;
    double best = eps;
    for (int j = 0; j < n; ++j) {
      double r = s[j];
      for (int k : col[j]) r -= dual[k];
      if (r > best) {
        best = r;
        e = j;
        if (stall >= 50) break;
      }
    }
    if (e < 0)
      for (int k = 0; k < m; ++k)
        if (-dual[k] > eps) {  // slack k enters
          e = n + k;
          break;
        }
    if (e < 0) {
      optimal = true;
      break;
    }
    // d = Binv a_e
    if (e < n) {
      std::fill(d.begin(), d.end(), 0.0);
      for (int k : col[e])
        for (int i = 0; i < m; ++i) d[i] += Binv[static_cast<size_t>(i) * m + k];
    } else {
      for (int i = 0; i < m; ++i) d[i] = Binv[static_cast<size_t>(i) * m + (e - n)];
    }
    int r = -1;
    double ratio = 0.0;
    for (int i = 0; i < m; ++i)
      if (d[i] > eps) {
        const double q = xb[i] / d[i];
        if (r < 0 || q < ratio - 1e-12 || (std::fabs(q - ratio) <= 1e-12 && basis[i] < basis[r])) r = i, ratio = q;
      }
    if (r < 0) break;
    stall = ratio <= 1e-12 ? stall + 1 : 0;
    const double piv = d[r];
    double* br = &Binv[static_cast<size_t>(r) * m];
    for (int k = 0; k < m; ++k) br[k] /= piv;
    for (int i = 0; i < m; ++i) {
      if (i == r || d[i] == 0.0) continue;
      double* bi = &Binv[static_cast<size_t>(i) * m];
      const double f = d[i];
      for (int k = 0; k < m; ++k) bi[k] -= f * br[k];
      xb[i] -= f * ratio;
    }
    xb[r] = ratio;
    basis[r] = e;
    cb[r] = e < n ? s[e] : 0.0;
  }
  if (std::getenv("STITCH_ILP_TRACE"))
    std::fprintf(stderr, "[ilp]   LP m=%d n=%d iterations=%d optimal=%d\n", m, n, lp_iters, (int)optimal);
  if (!optimal) {
    ratio_prices();
    return y;
  }
  for (int k = 0; k < m; ++k) y[rows[k]] = std::max(0.0, dual[k]);
  if (primal) {
    // primal values of the optimal basis for b = 1
    primal->assign(n, 0.0);
    for (int i = 0; i < m; ++i) {
      if (basis[i] >= n) continue;
      const double* bi = &Binv[static_cast<size_t>(i) * m];
      double xi = 0.0;
      for (int k = 0; k < m; ++k) xi += bi[k];
      (*primal)[basis[i]] = xi;
    }
  }
  // repair: make every pattern constraint hold (with a relative margin)
  for (int j = 0; j < n; ++j) {
    double t = 0.0;
    for (int x : sets[j]) t += y[x];
    const double need = s[j] * (1.0 + 1e-12) + 1e-12;
    if (t < need && !sets[j].empty()) {
      const double add = (need - t) / sets[j].size();
      for (int x : sets[j]) y[x] += add;
    }
  }
  return y;
}

// Near-optimality window delta: every selection S whose canonical total can
// equal the canonical optimum has a real total within delta of the real
// optimum R*. Recursive summation of k >= 0 terms errs by at most
// gamma_{k-1} * sum (gamma_k = k u / (1 - k u), u = 2^-53), so
// canonical(S) >= canonical(S*) >= R*(1 - gamma) and
// canonical(S) <= R(S)(1 + gamma) give R(S) >= R* - 2 gamma R*; the window
// is 8 gamma_K R_up (4x headroom for the approximate running totals the
// search compares), with K the largest possible selection (node-disjoint
// patterns: at most one per covered node) and R_up the fractional
// node-price bound sum_x max_{P covers x} s_P / |P| >= R*.
double selection_window(const IlpInstance& inst) {
  const int n = inst.num_vars;
  const bool nodes = static_cast<int>(inst.node_sets.size()) == n && inst.num_nodes > 0;
  double rup = 0.0;
  long long k = 0;
  if (nodes) {
    std::vector<double> best(inst.num_nodes, 0.0);
    std::vector<char> used(inst.num_nodes, 0);
    for (int v = 0; v < n; ++v) {
      if (inst.scores[v] <= 0.0) continue;
      if (inst.node_sets[v].empty()) {
        rup += inst.scores[v];
        ++k;
        continue;
      }
      const double r = inst.scores[v] / inst.node_sets[v].size();
      for (int x : inst.node_sets[v]) {
        best[x] = std::max(best[x], r);
        used[x] = 1;
      }
    }
    for (int x = 0; x < inst.num_nodes; ++x) {
      rup += best[x] * (1.0 + 1e-12);
      k += used[x];
    }
  } else {
    for (double sv : inst.scores)
      if (sv > 0.0) {
        rup += sv;
        ++k;
      }
  }
  const double u = std::ldexp(1.0, -53);
  const double kk = static_cast<double>(k + 2);
  const double gamma = kk * u / (1.0 - kk * u);
  return 8.0 * gamma * rup * (1.0 + 1e-9);
}

class Search {
 public:
  explicit Search(const IlpInstance& inst, double window = -1.0)
      : in_(inst), n_(inst.num_vars), window_(window >= 0.0 ? window : selection_window(inst)) {
    // Conflicts either as explicit pairs or implied by shared graph nodes
    // (planner instances: pair lists grow quadratically with overlap).
    node_mode_ = inst.pairs.empty() && static_cast<int>(inst.node_sets.size()) == n_ && inst.num_nodes > 0;
    adj_.resize(n_);
    for (const PairConstraint& pc : inst.pairs) {
      adj_[pc.u].push_back(pc.v);
      adj_[pc.v].push_back(pc.u);
    }
    limit_.resize(inst.cycles.size());
    cycles_of_.resize(n_);
    for (size_t c = 0; c < inst.cycles.size(); ++c) {
      limit_[c] = static_cast<int>(inst.cycles[c].pattern_indices.size()) - 1;
      for (int v : inst.cycles[c].pattern_indices) cycles_of_[v].push_back(static_cast<int>(c));
    }
    order_.resize(n_);
    std::iota(order_.begin(), order_.end(), 0);
    std::stable_sort(order_.begin(), order_.end(), [&](int a, int b) { return in_.scores[a] > in_.scores[b]; });
    build_cliques();
    use_frac_ = static_cast<int>(inst.node_sets.size()) == n_ && inst.num_nodes > 0;
    if (use_frac_) {
      ratio_.resize(n_);
      for (int v = 0; v < n_; ++v)
        ratio_[v] = inst.node_sets[v].empty() ? inst.scores[v] : inst.scores[v] / inst.node_sets[v].size();
      std::vector<std::vector<int>> pos_sets;
      std::vector<double> pos_scores;
      for (int v = 0; v < n_; ++v)
        if (inst.scores[v] > 0.0 && !inst.node_sets[v].empty()) {
          pos_sets.push_back(inst.node_sets[v]);
          pos_scores.push_back(inst.scores[v]);
        }
      std::vector<double> xlp;
      lp_price_ = lp_node_prices(pos_sets, pos_scores, inst.num_nodes, &xlp);
      // Reduced-cost fixing. With y the (repaired, feasible) duals,
      // s.x = sum(y) - sum_i y_i slack_i + sum_j r_j x_j and r_j <= 0, so a
      // selection within `gap + delta` of the incumbent (the LP primal when it
      // is integral and satisfies the cycle constraints) never uses a
      // variable with r_j < -(gap + delta): those are excluded from branching.
      {
        double ysum = 0.0;
        for (double yv : lp_price_) ysum += yv;
        lp_bound_ = ysum;
        std::vector<int> inc;
        bool integral = !xlp.empty();
        int k2 = 0;
        for (int v = 0; v < n_ && integral; ++v)
          if (inst.scores[v] > 0.0 && !inst.node_sets[v].empty()) {
            const double xv = xlp[k2++];
            if (xv > 1e-7 && xv < 1.0 - 1e-7) integral = false;
            else if (xv < -1e-7 || xv > 1.0 + 1e-7) integral = false;
            else if (xv >= 0.5) inc.push_back(v);
          }
        // the incumbent must be a feasible packing (the LP basis was chosen on
        // a perturbed right-hand side)
        if (integral) {
          std::vector<char> hit(inst.num_nodes, 0);
          for (int v : inc)
            for (int x : inst.node_sets[v]) {
              if (hit[x]) integral = false;
              hit[x] = 1;
            }
        }
        if (integral) {
          std::vector<int> cc(inst.cycles.size(), 0);
          for (int v : inc)
            for (size_t c = 0; c < inst.cycles.size(); ++c)
              if (std::find(inst.cycles[c].pattern_indices.begin(), inst.cycles[c].pattern_indices.end(), v) !=
                  inst.cycles[c].pattern_indices.end())
                ++cc[c];
          for (size_t c = 0; c < inst.cycles.size(); ++c)
            if (cc[c] > static_cast<int>(inst.cycles[c].pattern_indices.size()) - 1) integral = false;
        }
        if (integral) {
          // r_j x_j summed over a selection within the window of the
          // incumbent is at least -(ysum - incumbent + window); the
          // floating-point error of ysum, the incumbent and each r_j is
          // below (m + |P| + k + 3) eps (ysum + s_P), covered 4x.
          double incumbent = 0.0;
          for (int v : inc) incumbent += inst.scores[v];
          size_t maxp = 0;
          for (int v = 0; v < n_; ++v) maxp = std::max(maxp, inst.node_sets[v].size());
          const double eps = std::numeric_limits<double>::epsilon();
          const double fp = 4.0 * (inst.num_nodes + maxp + inc.size() + 3) * eps * 2.0 * (ysum + 1.0);
          const double margin = (ysum - incumbent) + window_ + fp;
          rc_out_.assign(n_, 0);
          for (int v = 0; v < n_; ++v) {
            if (inst.scores[v] <= 0.0 || inst.node_sets[v].empty()) continue;
            double r = inst.scores[v];
            for (int x : inst.node_sets[v]) r -= lp_price_[x];
            if (r < -margin) rc_out_[v] = 1;
          }
        }
        if (const char* rp = std::getenv("STITCH_ILP_REDUCED")) {
          // the variables reduced-cost fixing keeps, with their node sets and
          // reduced costs, and the node prices (solver development aid)
          if (FILE* f = std::fopen(rp, "w")) {
            for (int v = 0; v < n_; ++v) {
              if (inst.scores[v] <= 0.0 || inst.node_sets[v].empty() || (!rc_out_.empty() && rc_out_[v])) continue;
              double r = inst.scores[v];
              for (int x : inst.node_sets[v]) r -= lp_price_[x];
              std::fprintf(f, "v %d %a %a", v, inst.scores[v], r);
              for (int x : inst.node_sets[v]) std::fprintf(f, " %d", x);
              std::fprintf(f, "\n");
            }
            for (int x = 0; x < inst.num_nodes; ++x) std::fprintf(f, "y %d %a\n", x, lp_price_[x]);
            std::fclose(f);
          }
        }
        if (std::getenv("STITCH_ILP_TRACE")) {
          int out = 0;
          for (char c : rc_out_) out += c;
          std::fprintf(stderr, "[ilp]   LP bound %.6f integral=%d incumbent vars=%zu fixed-out=%d of %d\n", ysum,
                       (int)integral, inc.size(), out, n_);
        }
      }
      lp_stamp_.assign(inst.num_nodes, 0);
      node_vars_.assign(inst.num_nodes, {});
      for (int v = 0; v < n_; ++v)
        if (inst.scores[v] > 0.0)
          for (int x : inst.node_sets[v]) node_vars_[x].push_back(v);
      avail_.assign(n_, 0);
      ystamp_.assign(inst.num_nodes, 0);
      y_.assign(inst.num_nodes, 0.0);
      // LP-guided branching: variables the LP sets to 1 first (an integral
      // LP optimum is then found by the first dive), then by score
      std::vector<double> xv(n_, 0.0);
      int k = 0;
      for (int v = 0; v < n_; ++v)
        if (inst.scores[v] > 0.0 && !inst.node_sets[v].empty()) xv[v] = k < static_cast<int>(xlp.size()) ? xlp[k++] : 0.0;
      std::stable_sort(order_.begin(), order_.end(), [&](int a, int b) {
        const bool ia = xv[a] > 0.5, ib = xv[b] > 0.5;
        if (ia != ib) return ia;
        return in_.scores[a] > in_.scores[b];
      });
    }
    words_ = (n_ + 63) / 64;
    double total = 0.0;
    for (double s : inst.scores) total += s;
    // Relative slack covering the rounding of any partial sum the search
    // forms: <= n terms in general; with node sets and the node clique hint
    // every sum (selection, clique cover, node prices) has at most one term
    // per graph node (+ the patterns covering none).
    long long terms = n_;
    if (use_frac_ && static_cast<int>(inst.clique_hint.size()) == n_) {
      terms = inst.num_nodes;
      for (int v = 0; v < n_; ++v) terms += inst.node_sets[v].empty() ? 1 : 0;
    }
    slack_ = 4.0 * (terms + 2) * std::numeric_limits<double>::epsilon();
    (void)total;
  }

  // Best canonical total consistent with `fixed` (-1 free, 0 out, 1 in);
  // -inf when the fixed-in set is itself infeasible. With `target`, stops at
  // the first selection reaching it. The witness is kept in best_bits().
  double query(const std::vector<signed char>& fixed, double target = std::numeric_limits<double>::quiet_NaN()) {
    ++g_stats.queries;
    chosen_.assign(words_, 0);
    block_.assign(n_, 0);
    cover_.assign(node_mode_ ? in_.num_nodes : 0, 0);
    ccount_.assign(limit_.size(), 0);
    approx_ = 0.0;
    for (int v = 0; v < n_; ++v) {
      if (fixed[v] != 1) continue;
      if (!takeable(v)) return kNegInf;
      take(v);
    }
    free_.clear();
    // Zero-score variables never branch "in": adding 0.0 leaves every
    // canonical total unchanged, and excluding a variable never makes a
    // selection infeasible, so any total reachable with them is reachable
    // without them. (They still join the lexicographic answer through the
    // index-by-index extraction in solve(), as in the reference.)
    for (int v : order_)
      if (fixed[v] == -1 && in_.scores[v] > 0.0 && (rc_out_.empty() || !rc_out_[v])) free_.push_back(v);
    best_ = kNegInf;
    target_ = target;
    done_ = false;
    best_bits_ = chosen_;
    cm_.assign(nclique_, 0.0);
    cm_stamp_.assign(nclique_, 0);
    price_.assign(in_.num_nodes, 0.0);
    price_stamp_.assign(in_.num_nodes, 0);
    stamp_ = 0;
    dfs(0);
    return best_;
  }

  bool in_best(int v) const { return (best_bits_[v >> 6] >> (v & 63)) & 1; }
  // Variables reduced-cost fixing proved absent from every selection within
  // the window of the optimum (empty when the LP was not integral).
  const std::vector<char>& fixed_out() const { return rc_out_; }

  // Every feasible selection of positive-score variables whose total is
  // within `delta` of the optimum (approximate totals; the caller re-sums
  // canonically). Returns false when more than `cap` were found.
  bool collect_near_optimal(double delta, size_t cap, std::vector<std::vector<int>>* out) {
    collect_ = true;
    delta_ = delta;
    cap_ = cap;
    overflow_ = false;
    cands_.clear();
    std::vector<signed char> fixed(n_, -1);
    query(fixed);
    collect_ = false;
    if (overflow_) return false;
    if (truncated_ && cands_.empty()) return false;
    out->clear();
    for (const auto& [tot, bits] : cands_) {
      if (tot < best_ - delta_) continue;
      std::vector<int> sel;
      for (int v = 0; v < n_; ++v)
        if ((bits[v >> 6] >> (v & 63)) & 1) sel.push_back(v);
      out->push_back(std::move(sel));
    }
    return true;
  }

 private:
  void build_cliques() {
    clique_.assign(n_, -1);
    if (static_cast<int>(in_.clique_hint.size()) == n_) {
      clique_ = in_.clique_hint;
    } else {
      // Greedy clique cover from the pair list (small instances only).
      std::vector<std::vector<int>> members;
      if (n_ <= 4096) {
        std::vector<std::vector<char>> conflict(n_, std::vector<char>(n_, 0));
        for (int v = 0; v < n_; ++v)
          for (int w : adj_[v]) conflict[v][w] = 1;
        for (int v : order_) {
          int home = -1;
          for (size_t c = 0; c < members.size() && home < 0; ++c) {
            bool all = true;
            for (int w : members[c]) all = all && conflict[v][w];
            if (all) home = static_cast<int>(c);
          }
          if (home < 0) {
            home = static_cast<int>(members.size());
            members.emplace_back();
          }
          members[home].push_back(v);
          clique_[v] = home;
        }
      } else {
        std::iota(clique_.begin(), clique_.end(), 0);
      }
    }
    nclique_ = 0;
    for (int c : clique_) nclique_ = std::max(nclique_, c + 1);
  }

  bool takeable(int v) const {
    if (node_mode_) {
      for (int x : in_.node_sets[v])
        if (cover_[x]) return false;
    } else if (block_[v]) {
      return false;
    }
    for (int c : cycles_of_[v])
      if (ccount_[c] + 1 > limit_[c]) return false;
    return true;
  }
  void take(int v) {
    chosen_[v >> 6] |= uint64_t{1} << (v & 63);
    if (node_mode_)
      for (int x : in_.node_sets[v]) ++cover_[x];
    else
      for (int w : adj_[v]) ++block_[w];
    for (int c : cycles_of_[v]) ++ccount_[c];
    approx_ += in_.scores[v];
  }
  void drop(int v, double saved) {
    chosen_[v >> 6] &= ~(uint64_t{1} << (v & 63));
    if (node_mode_)
      for (int x : in_.node_sets[v]) --cover_[x];
    else
      for (int w : adj_[v]) --block_[w];
    for (int c : cycles_of_[v]) --ccount_[c];
    approx_ = saved;
  }
  double canonical() const {
    double t = 0.0;
    for (int wi = 0; wi < words_; ++wi) {
      uint64_t m = chosen_[wi];
      while (m) {
        int b = __builtin_ctzll(m);
        t += in_.scores[wi * 64 + b];
        m &= m - 1;
      }
    }
    return t;
  }

  void dfs(size_t pos) {
    if (done_) return;
    ++g_stats.nodes;
    if (node_budget_ > 0 && ++budget_used_ > node_budget_) {
      truncated_ = true;
      done_ = true;
      return;
    }
    // The current selection is feasible on its own (everything after `pos`
    // excluded): score it exactly when it can matter.
    if (collect_) {
      if (approx_ >= best_ - delta_) {
        cands_.push_back({approx_, chosen_});
        if (approx_ > best_) {
          best_ = approx_;
          // drop candidates that fell out of the window
          size_t w = 0;
          for (size_t i = 0; i < cands_.size(); ++i)
            if (cands_[i].first >= best_ - delta_) {
              if (w != i) cands_[w] = std::move(cands_[i]);
              ++w;
            }
          cands_.resize(w);
        }
        if (cands_.size() > cap_) {
          overflow_ = true;
          done_ = true;
          return;
        }
      }
    } else if (approx_ * (1.0 + slack_) >= best_ || best_ == kNegInf) {
      double c = canonical();
      if (c > best_) {
        best_ = c;
        best_bits_ = chosen_;
        if (c == target_) {
          done_ = true;
          return;
        }
      }
    }
    // Clique-cover bound over the still-takeable free variables.
    ++stamp_;
    double extra = 0.0;
    size_t first = free_.size();
    for (size_t i = pos; i < free_.size(); ++i) {
      int v = free_[i];
      if (!takeable(v)) continue;
      if (first == free_.size()) first = i;
      int c = clique_[v];
      double s = in_.scores[v];
      if (cm_stamp_[c] != stamp_) {
        cm_stamp_[c] = stamp_;
        cm_[c] = s;
        extra += s;
      } else if (s > cm_[c]) {
        extra += s - cm_[c];
        cm_[c] = s;
      }
    }
    if (first == free_.size()) return;
    if (use_frac_) {
      // fractional node-price bound over the same takeable free variables
      double frac = 0.0;
      for (size_t i = pos; i < free_.size() && frac < extra; ++i) {
        int v = free_[i];
        if (!takeable(v)) continue;
        const double r = ratio_[v];
        for (int x : in_.node_sets[v]) {
          if (price_stamp_[x] != stamp_) {
            price_stamp_[x] = stamp_;
            price_[x] = r;
            frac += r;
          } else if (r > price_[x]) {
            frac += r - price_[x];
            price_[x] = r;
          }
        }
      }
      extra = std::min(extra, frac);
      // LP-dual bound: the static optimal node prices over the nodes the
      // takeable free variables can still cover
      double lpb = 0.0;
      for (size_t i = pos; i < free_.size() && lpb < extra; ++i) {
        int v = free_[i];
        if (!takeable(v)) continue;
        for (int x : in_.node_sets[v])
          if (lp_stamp_[x] != stamp_) {
            lp_stamp_[x] = stamp_;
            lpb += lp_price_[x];
          }
      }
      extra = std::min(extra, lpb);
      // Adaptive dual: when the static prices cannot prune, lower each
      // coverable node's price as far as the still-available patterns allow
      // (one coordinate-descent pass; the prices stay dual-feasible for the
      // subproblem, so the sum stays a valid bound). Excluding an LP-basic
      // pattern frees slack exactly here.
      const double cutoff = collect_ ? best_ - delta_ : (std::isnan(target_) ? best_ : target_);
      // (quadratic in pattern size per node: only for moderate components)
      if (n_ <= 8000 && (approx_ + extra) * (1.0 + slack_) >= cutoff && best_ != kNegInf) {
        ++avail_stamp_;
        std::vector<int>& cov = cov_scratch_;
        cov.clear();
        for (size_t i = pos; i < free_.size(); ++i) {
          int v = free_[i];
          if (!takeable(v)) continue;
          avail_[v] = avail_stamp_;
          // every node of every available pattern (not only those the
          // early-exiting static pass above reached: a pattern's constraint
          // must see current prices on all of its nodes)
          for (int x : in_.node_sets[v])
            if (ystamp_[x] != avail_stamp_) {
              ystamp_[x] = avail_stamp_;
              y_[x] = lp_price_[x];
              cov.push_back(x);
            }
        }
        double ysum = 0.0;
        for (int x : cov) {
          double need = 0.0;
          for (int v : node_vars_[x]) {
            if (avail_[v] != avail_stamp_) continue;
            double rest = in_.scores[v];
            for (int z : in_.node_sets[v])
              if (z != x) rest -= y_[z];
            need = std::max(need, rest);
          }
          y_[x] = std::min(y_[x], need * (1.0 + 1e-12) + 1e-12);
          ysum += y_[x];
        }
        extra = std::min(extra, ysum);
      }
    }
    double bound = (approx_ + extra) * (1.0 + slack_);
    if (collect_) {
      if (bound < best_ - delta_) return;
    } else if (std::isnan(target_) ? bound <= best_ : bound < target_) {
      return;
    }
    int v = free_[first];
    double saved = approx_;
    take(v);
    dfs(first + 1);
    drop(v, saved);
    dfs(first + 1);
  }

  const IlpInstance& in_;
  int n_;
  double window_;
  std::vector<std::vector<int>> adj_;
  std::vector<int> limit_;
  std::vector<std::vector<int>> cycles_of_;
  std::vector<int> order_, clique_, free_;
  int nclique_ = 0, words_ = 0;
  bool use_frac_ = false;
  bool collect_ = false, overflow_ = false;
 public:
  long long node_budget_ = 0, budget_used_ = 0;
  bool truncated_ = false;
  double lp_bound_ = 0.0;
 private:
  double delta_ = 0.0;
  size_t cap_ = 0;
  std::vector<std::pair<double, std::vector<uint64_t>>> cands_;
  double slack_ = 0.0;

  std::vector<uint64_t> chosen_, best_bits_;
  std::vector<int> block_, ccount_, cover_;
  bool node_mode_ = false;
  double approx_ = 0.0, best_ = kNegInf, target_ = 0.0;
  bool done_ = false;
  std::vector<double> cm_;
  std::vector<unsigned> cm_stamp_;
  std::vector<double> price_;
  std::vector<unsigned> price_stamp_;
  std::vector<double> ratio_;  // s_P / |P|
  std::vector<char> rc_out_;   // reduced-cost fixed to 0
  std::vector<double> lp_price_;  // LP dual node prices (static, valid for every subproblem)
  std::vector<unsigned> lp_stamp_;
  std::vector<std::vector<int>> node_vars_;  // graph node -> variables covering it
  std::vector<unsigned> avail_, ystamp_;
  std::vector<double> y_;
  std::vector<int> cov_scratch_;
  unsigned avail_stamp_ = 0;
  unsigned stamp_ = 0;
};

}  // namespace

const SolveStats& last_solve_stats() { return g_stats; }

namespace {
thread_local long long g_node_budget = -1;
}

void set_ilp_node_budget(long long nodes) { g_node_budget = nodes; }

long long ilp_node_budget() {
  if (g_node_budget >= 0) return g_node_budget;
  static const long long b = [] {
    const char* e = std::getenv("STITCH_ILP_NODE_BUDGET");
    return e ? std::atoll(e) : 300000LL;
  }();
  return b;
}

std::vector<PairConstraint> build_conflicts(const std::vector<FusionPattern>& patterns) {
  std::map<std::string, std::vector<int>> holders;
  for (size_t i = 0; i < patterns.size(); ++i)
    for (const std::string& id : patterns[i].node_ids) holders[id].push_back(static_cast<int>(i));
  std::vector<std::pair<int, int>> pairs;
  for (const auto& [id, hs] : holders)
    for (size_t a = 0; a < hs.size(); ++a)
      for (size_t b = a + 1; b < hs.size(); ++b) pairs.push_back({hs[a], hs[b]});
  std::sort(pairs.begin(), pairs.end());
  pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
  std::vector<PairConstraint> out;
  out.reserve(pairs.size());
  for (auto [u, v] : pairs) out.push_back({u, v});
  return out;
}

namespace {

FusionPlan solve_monolithic(const IlpInstance& inst);

// Exact solve by decomposition (same answer contract as solve_monolithic).
//
// Variables split into components that share no pair or cycle constraint.
// A selection's real total is the sum of its components' totals, and its
// canonical (ascending-order double) total differs from the real one by at
// most (n-1) eps sum|s| <= delta/4; so every selection whose canonical total
// can reach the canonical optimum has, in every component, a real total
// within delta of that component's optimum. Those near-optimal component
// selections are enumerated, their combinations re-summed canonically (the
// optimum is then exactly the reference's), and the lexicographic
// extraction is replayed over the optimal family F, with zero-score
// variables added exactly where the reference's index-by-index probe would
// add them. Returns false (caller falls back) when an enumeration cap trips.
bool solve_decomposed(const IlpInstance& inst, FusionPlan* plan) {
  const int n = inst.num_vars;
  std::vector<int> parent(n);
  std::iota(parent.begin(), parent.end(), 0);
  std::function<int(int)> find = [&](int x) { return parent[x] == x ? x : parent[x] = find(parent[x]); };
  for (const PairConstraint& pc : inst.pairs) parent[find(pc.u)] = find(pc.v);
  const bool node_mode = inst.pairs.empty() && static_cast<int>(inst.node_sets.size()) == n && inst.num_nodes > 0;
  if (node_mode) {
    std::vector<int> owner(inst.num_nodes, -1);
    for (int v = 0; v < n; ++v)
      for (int x : inst.node_sets[v]) {
        if (owner[x] < 0) owner[x] = v;
        else parent[find(v)] = find(owner[x]);
      }
  }
  for (const CycleConstraint& cc : inst.cycles)
    for (size_t i = 1; i < cc.pattern_indices.size(); ++i) parent[find(cc.pattern_indices[i])] = find(cc.pattern_indices[0]);
  std::map<int, std::vector<int>> comps;
  double total = 0.0;
  for (int v = 0; v < n; ++v) {
    comps[find(v)].push_back(v);
    total += inst.scores[v];
  }
  (void)total;
  const double delta = selection_window(inst);

  // Near-optimal selections per component (global indices).
  std::vector<std::vector<std::vector<int>>> per;
  static const bool trace = std::getenv("STITCH_ILP_TRACE") != nullptr;
  // Sub-instance over `vars` (global indices, ascending).
  auto restrict_to = [&](const std::vector<int>& vars) {
    std::map<int, int> local;
    for (size_t i = 0; i < vars.size(); ++i) local[vars[i]] = static_cast<int>(i);
    IlpInstance sub;
    sub.num_vars = static_cast<int>(vars.size());
    for (int v : vars) sub.scores.push_back(inst.scores[v]);
    for (const PairConstraint& pc : inst.pairs)
      if (local.count(pc.u) && local.count(pc.v)) sub.pairs.push_back({local[pc.u], local[pc.v]});
    // a cycle constraint with a member outside `vars` (fixed to 0) holds
    for (const CycleConstraint& cc : inst.cycles) {
      bool all = true;
      for (int v : cc.pattern_indices) all = all && local.count(v);
      if (!all) continue;
      CycleConstraint c2;
      for (int v : cc.pattern_indices) c2.pattern_indices.push_back(local[v]);
      sub.cycles.push_back(c2);
    }
    if (static_cast<int>(inst.clique_hint.size()) == n)
      for (int v : vars) sub.clique_hint.push_back(inst.clique_hint[v]);
    if (static_cast<int>(inst.node_sets.size()) == n) {
      sub.num_nodes = inst.num_nodes;
      for (int v : vars) sub.node_sets.push_back(inst.node_sets[v]);
    }
    return sub;
  };
  // Collects the component's near-optimal selections into `per`; false when
  // a cap or the node budget trips.
  std::function<bool(const std::vector<int>&, int)> collect = [&](const std::vector<int>& vars, int depth) -> bool {
    bool any_pos = false;
    for (int v : vars) any_pos = any_pos || inst.scores[v] > 0.0;
    if (!any_pos) return true;
    IlpInstance sub = restrict_to(vars);
    if (trace) std::fprintf(stderr, "[ilp] %*ssolving component vars=%zu\n", 2 * depth, "", vars.size());
    const auto tc0 = std::chrono::steady_clock::now();
    Search search(sub, delta);
    if (trace)
      std::fprintf(stderr, "[ilp]   setup+LP %.2fs\n",
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - tc0).count());
    // Reduced-cost fixing leaves only the variables a near-optimal selection
    // can use; those often fall apart into independent pieces (an LP with
    // many zero-reduced-cost columns), and searching the pieces jointly
    // multiplies their trees. Split and collect each piece on its own (the
    // window applies per piece for the same reason it applies per
    // component); the combination step below takes their product.
    const std::vector<char>& out = search.fixed_out();
    if (!out.empty() && depth < 32) {
      std::vector<int> kept;
      for (size_t i = 0; i < vars.size(); ++i)
        if (!out[i]) kept.push_back(vars[i]);
      std::vector<int> par(kept.size());
      std::iota(par.begin(), par.end(), 0);
      std::function<int(int)> fd = [&](int x) { return par[x] == x ? x : par[x] = fd(par[x]); };
      std::map<int, int> pos;
      for (size_t i = 0; i < kept.size(); ++i) pos[kept[i]] = static_cast<int>(i);
      if (node_mode || static_cast<int>(inst.node_sets.size()) == n) {
        std::map<int, int> owner;
        for (size_t i = 0; i < kept.size(); ++i)
          for (int x : inst.node_sets[kept[i]]) {
            auto it = owner.emplace(x, static_cast<int>(i)).first;
            par[fd(static_cast<int>(i))] = fd(it->second);
          }
      }
      for (const PairConstraint& pc : inst.pairs)
        if (pos.count(pc.u) && pos.count(pc.v)) par[fd(pos[pc.u])] = fd(pos[pc.v]);
      for (const CycleConstraint& cc : inst.cycles) {
        bool all = true;
        for (int v : cc.pattern_indices) all = all && pos.count(v);
        if (all)
          for (size_t i = 1; i < cc.pattern_indices.size(); ++i)
            par[fd(pos[cc.pattern_indices[i]])] = fd(pos[cc.pattern_indices[0]]);
      }
      std::map<int, std::vector<int>> pieces;
      for (size_t i = 0; i < kept.size(); ++i) pieces[fd(static_cast<int>(i))].push_back(kept[i]);
      // recurse while the pieces shrink: a fresh LP over fewer columns fixes
      // more of them
      if (pieces.size() > 1 || kept.size() < vars.size()) {
        if (trace)
          std::fprintf(stderr, "[ilp]   reduced to %zu variables in %zu pieces\n", kept.size(), pieces.size());
        for (auto& [r, pv] : pieces) {
          (void)r;
          if (!collect(pv, depth + 1)) return false;
        }
        return true;
      }
    }
    search.node_budget_ = ilp_node_budget();
    std::vector<std::vector<int>> cands;
    const long long n0 = g_stats.nodes;
    const bool ok = search.collect_near_optimal(delta, 64, &cands);
    if (search.truncated_) {
      ++g_stats.truncated;
      double inc = 0.0;
      if (!cands.empty())
        for (int v : cands.front()) inc += sub.scores[v];
      g_stats.lp_gap += std::max(0.0, search.lp_bound_ - inc);
    }
    if (trace)
      std::fprintf(stderr, "[ilp] %*scomponent vars=%zu candidates=%zu nodes=%lld%s%s\n", 2 * depth, "", vars.size(),
                   cands.size(), g_stats.nodes - n0, ok ? "" : " (cap: fallback)",
                   search.truncated_ ? " (node budget: incumbent)" : "");
    if (!ok) return false;
    for (auto& c : cands)
      for (int& v : c) v = vars[v];
    per.push_back(std::move(cands));
    return true;
  };
  for (auto& [root, vars] : comps) {
    (void)root;
    if (!collect(vars, 0)) return false;
  }
  // Canonical optimum over the combinations.
  size_t combos = 1;
  for (const auto& c : per) {
    combos *= std::max<size_t>(1, c.size());
    if (combos > 4096) return false;
  }
  std::vector<std::vector<int>> family;
  double optimum = 0.0;
  std::vector<size_t> idx(per.size(), 0);
  for (size_t k = 0; k < combos; ++k) {
    std::vector<int> sel;
    for (size_t i = 0; i < per.size(); ++i) sel.insert(sel.end(), per[i][idx[i]].begin(), per[i][idx[i]].end());
    std::sort(sel.begin(), sel.end());
    double canon = 0.0;
    for (int v : sel) canon += inst.scores[v];
    if (family.empty() || canon > optimum) {
      optimum = canon;
      family.clear();
    }
    if (canon == optimum) family.push_back(std::move(sel));
    for (size_t i = 0; i < per.size(); ++i) {
      if (++idx[i] < per[i].size()) break;
      idx[i] = 0;
    }
  }
  if (family.empty()) family.push_back({});
  // Replay the reference's extraction (ilp_solver.cpp:153-167) over F:
  // index by index, stop once the prefix reaches the optimum, else include
  // v when some optimal completion of the decisions so far contains it.
  // alive[f]: family member f is still consistent with every decision.
  std::vector<std::vector<int>> adj(n);
  for (const PairConstraint& pc : inst.pairs) {
    adj[pc.u].push_back(pc.v);
    adj[pc.v].push_back(pc.u);
  }
  std::vector<std::vector<int>> cycles_of(n);
  for (size_t c = 0; c < inst.cycles.size(); ++c)
    for (int v : inst.cycles[c].pattern_indices) cycles_of[v].push_back(static_cast<int>(c));
  const size_t F = family.size();
  // node mode: graph nodes covered by each family member and by the zeros
  std::vector<std::vector<char>> fcover(node_mode ? F : 0, std::vector<char>(node_mode ? inst.num_nodes : 0, 0));
  std::vector<char> zcover(node_mode ? inst.num_nodes : 0, 0);
  if (node_mode)
    for (size_t f = 0; f < F; ++f)
      for (int w : family[f])
        for (int x : inst.node_sets[w]) fcover[f][x] = 1;
  std::vector<std::vector<char>> member(F, std::vector<char>(n, 0));
  std::vector<std::vector<int>> ccount(F, std::vector<int>(inst.cycles.size(), 0));
  for (size_t f = 0; f < F; ++f)
    for (int w : family[f]) {
      member[f][w] = 1;
      for (int c : cycles_of[w]) ++ccount[f][c];
    }
  std::vector<char> alive(F, 1), zero_in(n, 0);
  // zero v joins member f's completion: no conflict with f's set or the zeros
  // already selected, and every cycle constraint keeps a free slot
  auto zero_fits = [&](size_t f, int v) {
    if (node_mode) {
      for (int x : inst.node_sets[v])
        if (fcover[f][x] || zcover[x]) return false;
    }
    for (int w : adj[v])
      if (member[f][w] || zero_in[w]) return false;
    for (int c : cycles_of[v])
      if (ccount[f][c] + 1 > static_cast<int>(inst.cycles[c].pattern_indices.size()) - 1) return false;
    return true;
  };
  plan->selected.clear();
  double prefix = 0.0;
  for (int v = 0; v < n; ++v) {
    if (prefix == optimum) break;
    const bool pos = inst.scores[v] > 0.0;
    bool keep = false;
    for (size_t f = 0; f < F && !keep; ++f)
      if (alive[f]) keep = pos ? member[f][v] != 0 : zero_fits(f, v);
    if (keep) {
      for (size_t f = 0; f < F; ++f) {
        if (!alive[f]) continue;
        if (pos ? !member[f][v] : !zero_fits(f, v)) {
          alive[f] = 0;
        } else if (!pos) {
          for (int c : cycles_of[v]) ++ccount[f][c];
        }
      }
      if (!pos) {
        zero_in[v] = 1;
        if (node_mode)
          for (int x : inst.node_sets[v]) zcover[x] = 1;
      }
      plan->selected.push_back(v);
      prefix = 0.0;
      for (int w : plan->selected) prefix += inst.scores[w];
    } else if (pos) {
      for (size_t f = 0; f < F; ++f)
        if (member[f][v]) alive[f] = 0;
    }
  }
  plan->total_score = prefix;
  return true;
}

// STITCH_ILP_DUMP=<prefix>: every instance solved is written to
// <prefix>.<k>.txt (scores as hex floats, node sets, pairs, cycles) for the
// offline solver driver scripts/probes/ilp_driver.cpp.
void dump_instance(const IlpInstance& inst) {
  static const char* prefix = std::getenv("STITCH_ILP_DUMP");
  if (!prefix) return;
  static int k = 0;
  const std::string path = std::string(prefix) + "." + std::to_string(k++) + ".txt";
  FILE* f = std::fopen(path.c_str(), "w");
  if (!f) return;
  std::fprintf(f, "%d %d %zu %zu %zu\n", inst.num_vars, inst.num_nodes, inst.pairs.size(), inst.cycles.size(),
               inst.clique_hint.size());
  for (double s : inst.scores) std::fprintf(f, "%a\n", s);
  for (int v = 0; v < inst.num_vars && inst.num_nodes > 0; ++v) {
    std::fprintf(f, "%zu", inst.node_sets[v].size());
    for (int x : inst.node_sets[v]) std::fprintf(f, " %d", x);
    std::fprintf(f, "\n");
  }
  for (const PairConstraint& pc : inst.pairs) std::fprintf(f, "%d %d\n", pc.u, pc.v);
  for (const CycleConstraint& cc : inst.cycles) {
    std::fprintf(f, "%zu", cc.pattern_indices.size());
    for (int v : cc.pattern_indices) std::fprintf(f, " %d", v);
    std::fprintf(f, "\n");
  }
  for (int c : inst.clique_hint) std::fprintf(f, "%d\n", c);
  std::fclose(f);
}

}  // namespace

FusionPlan solve(const IlpInstance& inst) {
  if (static_cast<int>(inst.scores.size()) != inst.num_vars)
    throw GraphError("ILP instance: one score per variable required");
  for (double s : inst.scores)
    if (s < 0) throw GraphError("ILP instance requires non-negative scores");
  dump_instance(inst);
  static const char* method = std::getenv("STITCH_ILP_METHOD");
  if (!(method && std::string(method) == "monolithic")) {
    FusionPlan plan;
    if (solve_decomposed(inst, &plan)) return plan;
  }
  return solve_monolithic(inst);
}

namespace {

FusionPlan solve_monolithic(const IlpInstance& inst) {
  const int n = inst.num_vars;
  Search search(inst);
  std::vector<signed char> fixed(n, -1);
  static const bool trace = std::getenv("STITCH_ILP_TRACE") != nullptr;
  const double optimum = search.query(fixed);
  if (trace) std::fprintf(stderr, "[ilp] n=%d pairs=%zu optimum=%.6f nodes=%lld\n", n, inst.pairs.size(), optimum, g_stats.nodes);
  std::vector<char> witness(n, 0);
  for (int v = 0; v < n; ++v) witness[v] = search.in_best(v);

  FusionPlan plan;
  double prefix = 0.0;
  for (int v = 0; v < n; ++v) {
    if (prefix == optimum) break;  // stopping here is lexicographically smallest
    fixed[v] = 1;
    bool keep = witness[v];
    const long long before = g_stats.nodes;
    if (!keep && search.query(fixed, optimum) == optimum) {
      keep = true;
      for (int w = 0; w < n; ++w) witness[w] = search.in_best(w);
    }
    if (trace && g_stats.nodes - before > 100000)
      std::fprintf(stderr, "[ilp] extraction v=%d took %lld nodes\n", v, g_stats.nodes - before);
    if (keep) {
      plan.selected.push_back(v);
      prefix = 0.0;
      for (int w : plan.selected) prefix += inst.scores[w];
    } else {
      fixed[v] = 0;
    }
  }
  plan.total_score = prefix;
  return plan;
}

}  // namespace

FusionPlan solve_with_cycle_elimination(const Graph& g, const std::vector<FusionPattern>& patterns,
                                        const std::vector<double>& scores) {
  IlpInstance inst;
  inst.num_vars = static_cast<int>(patterns.size());
  inst.scores = scores;
  // conflicts are implied by shared nodes (inst.node_sets below); no O(k^2) pair list
  // Clique hint: each pattern joins the clique of its most-shared node.
  std::map<std::string, int> holders;
  for (const FusionPattern& p : patterns)
    for (const std::string& id : p.node_ids) ++holders[id];
  std::map<std::string, int> clique_id;
  inst.clique_hint.resize(patterns.size());
  for (size_t i = 0; i < patterns.size(); ++i) {
    const std::string* home = nullptr;
    for (const std::string& id : patterns[i].node_ids)
      if (!home || holders[id] > holders[*home]) home = &id;
    if (!home) {
      inst.clique_hint[i] = -1;
      continue;
    }
    auto it = clique_id.emplace(*home, static_cast<int>(clique_id.size())).first;
    inst.clique_hint[i] = it->second;
  }
  int next = static_cast<int>(clique_id.size());
  for (int& c : inst.clique_hint)
    if (c < 0) c = next++;
  std::map<std::string, int> node_index;
  inst.node_sets.resize(patterns.size());
  for (size_t i = 0; i < patterns.size(); ++i)
    for (const std::string& id : patterns[i].node_ids) {
      auto it = node_index.emplace(id, static_cast<int>(node_index.size())).first;
      inst.node_sets[i].push_back(it->second);
    }
  inst.num_nodes = static_cast<int>(node_index.size());

  SolveStats total;
  for (int round = 0; round < 10000; ++round) {
    g_stats = SolveStats{};
    FusionPlan plan = solve(inst);
    total.nodes += g_stats.nodes;
    total.queries += g_stats.queries;
    total.truncated = g_stats.truncated;
    total.lp_gap = g_stats.lp_gap;
    total.rounds = round + 1;
    std::vector<FusionPattern> chosen;
    for (int idx : plan.selected) {
      FusionPattern p = patterns[idx];
      p.pattern_id = idx;
      chosen.push_back(std::move(p));
    }
    ContractResult r = contract_plan(g, chosen);
    if (std::getenv("STITCH_ILP_TRACE")) {
      std::fprintf(stderr, "[ilp] round %d total %.17g selected", round, plan.total_score);
      for (int v : plan.selected) std::fprintf(stderr, " %d", v);
      std::fprintf(stderr, "%s\n", r.cycle ? " (cycle)" : "");
    }
    if (!r.cycle) {
      g_stats = total;
      return plan;
    }
    if (r.cycle->pattern_ids.empty()) throw InternalError("contraction cycle without any pattern on it");
    inst.cycles.push_back({r.cycle->pattern_ids});
  }
  throw GraphError("cycle elimination did not converge within 10000 rounds");
}

}  // namespace stitch
