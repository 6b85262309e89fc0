// Control plane: link graph, MWU tree packing, ILP tree-count minimisation,
// one-hop switch trees, weight-proportional split and chunking.
//
//   Graph model ............ P:338 (Sec. 3.1)
//   MWU packing ............ P:363-367 (Sec. 3.2), Garg-Koenemann step (R#4)
//   ILP + relaxation ....... P:371-393 (Sec. 3.2.1, Eqs. 4-7; R#5, R#6)
//   AllReduce trees ........ P:395-398 (Sec. 3.3): undirected packing,
//                            per-tree root = centre (R#9)
//   One-hop switch trees ... P:440-442 (Sec. 3.5); switch Broadcast (R#10)
//   Split / chunking ....... P:477-478 (Sec. 4.1; R#11), P:510-517 (a8)
//
// This is host code only; it never touches a GPU.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <numeric>
#include <set>
#include <sstream>

#include "blink_internal.h"

namespace blink {

int esize_of(blink_dtype_t d) {
  switch (d) {
    case BLINK_FLOAT32: return 4;
    case BLINK_BFLOAT16: return 2;
    case BLINK_INT32: return 4;
  }
  return 0;
}

// ============================================================== graph
blink_result_t build_graph(const blink_graph_t* g, int nranks, Graph* out, std::string* err) {
  out->n = nranks;
  out->cap.assign(nranks, std::vector<double>(nranks, 0.0));
  if (g == nullptr) {  // NVSwitch model: uniform K_m
    out->switch_model = true;
    return BLINK_SUCCESS;
  }
  if (g->num_nodes < nranks) {
    *err = "graph has " + std::to_string(g->num_nodes) + " nodes but the comm has " +
           std::to_string(nranks) + " ranks (nodes 0..nranks-1 must be the ranks' GPUs)";
    return BLINK_ERR_TOPOLOGY;
  }
  if (g->num_links < 0 || (g->num_links > 0 && g->links == nullptr)) {
    *err = "graph.links is NULL";
    return BLINK_ERR_INVALID_ARGUMENT;
  }
  auto kind = [&](int v) { return g->kinds ? g->kinds[v] : BLINK_NODE_GPU; };
  for (int v = 0; v < nranks; ++v)
    if (kind(v) != BLINK_NODE_GPU) {
      *err = "node " + std::to_string(v) + " is a rank but not a GPU node";
      return BLINK_ERR_TOPOLOGY;
    }
  for (int v = nranks; v < g->num_nodes; ++v)
    if (kind(v) == BLINK_NODE_GPU) {
      *err = "GPU node " + std::to_string(v) + " is not one of the " + std::to_string(nranks) +
             " ranks (pass the induced sub-allocation, P:320)";
      return BLINK_ERR_TOPOLOGY;
    }
  bool any_switch = false;
  std::vector<int> on_switch(nranks, 0);
  for (int k = 0; k < g->num_links; ++k) {
    const blink_link_t& L = g->links[k];
    char buf[160];
    if (L.src < 0 || L.src >= g->num_nodes || L.dst < 0 || L.dst >= g->num_nodes) {
      snprintf(buf, sizeof buf, "link %d (%d->%d) has a dangling endpoint", k, L.src, L.dst);
      *err = buf;
      return BLINK_ERR_TOPOLOGY;
    }
    if (!(L.capacity > 0.0) || !std::isfinite(L.capacity)) {
      snprintf(buf, sizeof buf, "link %d (%d->%d) has nonpositive capacity %g", k, L.src, L.dst,
               L.capacity);
      *err = buf;
      return BLINK_ERR_TOPOLOGY;
    }
    if (L.src == L.dst) {
      snprintf(buf, sizeof buf, "link %d is a self-loop on node %d", k, L.src);
      *err = buf;
      return BLINK_ERR_TOPOLOGY;
    }
    bool ss = kind(L.src) == BLINK_NODE_SWITCH, ds = kind(L.dst) == BLINK_NODE_SWITCH;
    if (ss || ds) {
      any_switch = true;
      if (ss && ds) continue;  // switch fabric
      on_switch[ss ? L.dst : L.src] = 1;
      continue;
    }
    out->cap[L.src][L.dst] += L.capacity;
    if (L.bidirectional) out->cap[L.dst][L.src] += L.capacity;
  }
  bool any_direct = false;
  for (int u = 0; u < nranks; ++u)
    for (int v = 0; v < nranks; ++v)
      if (out->cap[u][v] > 0) any_direct = true;
  if (any_switch && !any_direct) {
    for (int v = 0; v < nranks; ++v)
      if (!on_switch[v] && nranks > 1) {
        *err = "GPU " + std::to_string(v) + " is not attached to any switch (disconnected)";
        return BLINK_ERR_TOPOLOGY;
      }
    out->switch_model = true;
    return BLINK_SUCCESS;
  }
  if (any_switch) {
    // NEXT-4: servers = components of the GPU-GPU links, joined
    // by the network switch; every server needs a network attachment
    out->switch_model = false;
    out->multi_server = true;
    std::vector<int> comp(nranks, -1);
    for (int s0 = 0; s0 < nranks; ++s0) {
      if (comp[s0] >= 0) continue;
      const int id = int(out->servers.size());
      out->servers.push_back({});
      std::vector<int> st{s0};
      comp[s0] = id;
      while (!st.empty()) {
        int u = st.back();
        st.pop_back();
        out->servers[id].push_back(u);
        for (int v = 0; v < nranks; ++v)
          if (comp[v] < 0 && (out->cap[u][v] > 0 || out->cap[v][u] > 0)) {
            comp[v] = id;
            st.push_back(v);
          }
      }
      std::sort(out->servers[id].begin(), out->servers[id].end());
      bool attached = false;
      for (int v : out->servers[id]) attached = attached || on_switch[v];
      if (!attached) {
        std::string ids;
        for (int v : out->servers[id]) ids += (ids.empty() ? "" : ",") + std::to_string(v);
        *err = "server {" + ids + "} has no link to the network switch (disconnected)";
        return BLINK_ERR_TOPOLOGY;
      }
    }
    return BLINK_SUCCESS;
  }
  out->switch_model = false;
  // weak connectivity: report one disconnected partition
  std::vector<int> seen(nranks, 0);
  std::vector<int> st{0};
  seen[0] = 1;
  while (!st.empty()) {
    int u = st.back();
    st.pop_back();
    for (int v = 0; v < nranks; ++v)
      if (!seen[v] && (out->cap[u][v] > 0 || out->cap[v][u] > 0)) {
        seen[v] = 1;
        st.push_back(v);
      }
  }
  std::string part;
  for (int v = 0; v < nranks; ++v)
    if (!seen[v]) part += (part.empty() ? "" : ",") + std::to_string(v);
  if (!part.empty()) {
    *err = "allocation is disconnected: GPUs {" + part + "} are unreachable from GPU 0";
    return BLINK_ERR_TOPOLOGY;
  }
  return BLINK_SUCCESS;
}

// ============================================================== MWU inner oracles
namespace {

struct WEdge {
  int u, v;
  double w;
  int key;  // lexicographic (src, dst) tie-break
};

// Chu-Liu / Edmonds minimum arborescence.  Returns, for every vertex, the key
// of its chosen in-edge (-1 at the root).  Written as an explicit contraction
// loop with a stack of levels that is unwound afterwards.
std::vector<int> min_arborescence(int n, int root, const std::vector<WEdge>& edges0) {
  struct Level {
    int n, root;
    std::vector<WEdge> edges;        // edges of this level (key = index into parent level's edges)
    std::vector<int> best;           // chosen in-edge index per vertex
    std::vector<int> comp;           // vertex -> contracted id
  };
  std::vector<Level> levels;
  Level cur;
  cur.n = n;
  cur.root = root;
  cur.edges = edges0;
  // Work on indices: edge identity at level L is its position in levels[L].edges.
  std::vector<std::vector<int>> origin;  // origin[L][j] = index of edge j of level L+1 in level L
  while (true) {
    const int N = cur.n;
    cur.best.assign(N, -1);
    for (int j = 0; j < int(cur.edges.size()); ++j) {
      const WEdge& e = cur.edges[j];
      if (e.v == cur.root || e.u == e.v) continue;
      int b = cur.best[e.v];
      if (b < 0 || e.w < cur.edges[b].w || (e.w == cur.edges[b].w && e.key < cur.edges[b].key))
        cur.best[e.v] = j;
    }
    for (int v = 0; v < N; ++v)
      if (v != cur.root && cur.best[v] < 0) return {};  // unreachable
    // cycle search
    cur.comp.assign(N, -1);
    std::vector<int> mark(N, -1);
    int nc = 0;
    bool cyc = false;
    for (int v = 0; v < N; ++v) {
      int x = v;
      while (x != cur.root && mark[x] < 0 && cur.comp[x] < 0) {
        mark[x] = v;
        x = cur.edges[cur.best[x]].u;
      }
      if (x != cur.root && mark[x] == v && cur.comp[x] < 0) {
        cyc = true;
        int y = x;
        do {
          cur.comp[y] = nc;
          y = cur.edges[cur.best[y]].u;
        } while (y != x);
        ++nc;
      }
    }
    if (!cyc) break;
    for (int v = 0; v < N; ++v)
      if (cur.comp[v] < 0) cur.comp[v] = nc++;
    Level nxt;
    nxt.n = nc;
    nxt.root = cur.comp[cur.root];
    std::vector<int> org;
    for (int j = 0; j < int(cur.edges.size()); ++j) {
      const WEdge& e = cur.edges[j];
      int cu = cur.comp[e.u], cv = cur.comp[e.v];
      if (cu == cv || e.v == cur.root) continue;
      nxt.edges.push_back({cu, cv, e.w - cur.edges[cur.best[e.v]].w, e.key});
      org.push_back(j);
    }
    levels.push_back(std::move(cur));
    origin.push_back(std::move(org));
    cur = std::move(nxt);
  }
  // Unwind: chosen edge indices at the deepest level, mapped upwards.
  std::vector<int> chosen;  // edge indices at the current level
  for (int v = 0; v < cur.n; ++v)
    if (v != cur.root) chosen.push_back(cur.best[v]);
  for (int L = int(levels.size()) - 1; L >= 0; --L) {
    Level& lv = levels[L];
    std::vector<int> in_of(lv.n, -1);  // vertex -> chosen in-edge (level L index)
    for (int j : chosen) {
      int jj = origin[L][j];
      in_of[lv.edges[jj].v] = jj;
    }
    std::vector<int> up;
    for (int v = 0; v < lv.n; ++v) {
      if (v == lv.root) continue;
      up.push_back(in_of[v] >= 0 ? in_of[v] : lv.best[v]);
    }
    chosen.swap(up);
    cur = std::move(lv);
  }
  std::vector<int> parent(n, -1);
  for (int j : chosen) parent[edges0[j].v] = edges0[j].u;
  return parent;
}

// Kruskal over undirected pairs (u < v); ties (w, u, v) ascending, or (w,
// -u, -v) with `desc` (the alternate MWU run).  Returns pair indices.
std::vector<int> min_spanning_tree(int n, const std::vector<std::pair<int, int>>& pairs,
                                   const std::vector<double>& w, bool desc = false) {
  std::vector<int> idx(pairs.size());
  std::iota(idx.begin(), idx.end(), 0);
  std::sort(idx.begin(), idx.end(), [&](int a, int b) {
    if (w[a] != w[b]) return w[a] < w[b];
    return desc ? pairs[b] < pairs[a] : pairs[a] < pairs[b];
  });
  std::vector<int> uf(n);
  std::iota(uf.begin(), uf.end(), 0);
  std::function<int(int)> find = [&](int x) { return uf[x] == x ? x : uf[x] = find(uf[x]); };
  std::vector<int> out;
  for (int j : idx) {
    int a = find(pairs[j].first), b = find(pairs[j].second);
    if (a != b) {
      uf[a] = b;
      out.push_back(j);
    }
  }
  if (int(out.size()) != n - 1) return {};
  std::sort(out.begin(), out.end());
  return out;
}

// Garg-Koenemann MWU (R#4) over `ne` resources with capacities `c`.  The
// callback returns the resource list of the minimum-length tree under the
// normalised lengths, or an empty list on failure.
struct MwuResult {
  std::map<std::vector<int>, double> x;  // tree (sorted resource list) -> weight
  double rate = 0;
  int iters = 0;
};
bool run_mwu(const std::vector<double>& c, double eps,
             const std::function<std::vector<int>(const std::vector<double>&)>& tree_of,
             MwuResult* out) {
  const int ne = int(c.size());
  const double log_delta = std::log1p(eps) - (1.0 / eps) * std::log((1.0 + eps) * ne);
  std::vector<double> logl(ne);
  for (int e = 0; e < ne; ++e) logl[e] = log_delta - std::log(c[e]);
  std::vector<double> len(ne);
  std::map<std::vector<int>, double> x;
  int it = 0;
  for (;; ++it) {
    if (it > 5000000) return false;
    double mx = *std::max_element(logl.begin(), logl.end());
    for (int e = 0; e < ne; ++e) len[e] = std::exp(logl[e] - mx);
    std::vector<int> T = tree_of(len);
    if (T.empty()) return false;
    // sum_{e in T} l_e >= 1 <=> logsumexp(logl[T]) >= 0
    double m2 = -INFINITY;
    for (int e : T) m2 = std::max(m2, logl[e]);
    double s = 0;
    for (int e : T) s += std::exp(logl[e] - m2);
    if (m2 + std::log(s) >= 0.0) break;
    double cmin = INFINITY;
    for (int e : T) cmin = std::min(cmin, c[e]);
    x[T] += cmin;
    for (int e : T) logl[e] += std::log1p(eps * cmin / c[e]);
  }
  std::vector<double> load(ne, 0.0);
  for (auto& kv : x)
    for (int e : kv.first) load[e] += kv.second;
  double lam = 0;
  for (int e = 0; e < ne; ++e) lam = std::max(lam, load[e] / c[e]);
  out->x.clear();
  out->rate = 0;
  for (auto& kv : x) {
    out->x[kv.first] = kv.second / lam;
    out->rate += kv.second / lam;
  }
  out->iters = it;
  return true;
}

// ============================================================== ILP (Eqs. 4-7)
struct IlpCand {
  std::vector<int> res;  // resources used (each once)
  int depth;
  double x;              // MWU weight (search order / rounding seed)
  int prio = 0;          // 1: exact/peeled integral candidate, tried first
  int lovasz = 0;        // from the exact integral arborescence packing
  int mult[5] = {0, 0, 0, 0, 0};  // peel multiplicity at grid 1, 2, 4, 8, 16
  int paper = 1;         // 1: returned by an MWU run (P:390's candidate set)
};
struct IlpSol {
  std::vector<int> z;
  int64_t sumz = -1;
  int ntrees = 0;
  int maxdepth = 0;
  int64_t sumdepth = 0;
};
// Lexicographic ILP objective: maximise sum z, then fewest trees, then the
// smallest maximum depth, then the least total depth (R#21: depth adds
// pipeline latency).
bool sol_better(int64_t sz, int nt, int md, int64_t sd, const IlpSol& b) {
  if (sz != b.sumz) return sz > b.sumz;
  if (nt != b.ntrees) return nt < b.ntrees;
  if (md != b.maxdepth) return md < b.maxdepth;
  return sd < b.sumdepth;
}

// ------------------------------------------------------------ LP-based B&B
// Bounded-variable primal simplex: max c^T x s.t. A x <= b, 0 <= x <= u, with
// b >= 0 (the slack basis is feasible).  Dense tableau; the problems here are
// tiny (rows = links, <= ~120; columns = candidate trees).  Dantzig pricing,
// switching to Bland's rule after a run of degenerate pivots (no cycling).
struct BoundedLp {
  int m = 0, n = 0;
  std::vector<double> A;  // m x n, row-major
  std::vector<double> b, c, u;
  // returns the optimum; x gets the primal solution
  double solve(std::vector<double>* x) const {
    const int N = n + m;
    const double tol = 1e-9;
    std::vector<double> T(size_t(m) * N, 0.0);
    for (int i = 0; i < m; ++i) {
      for (int j = 0; j < n; ++j) T[size_t(i) * N + j] = A[size_t(i) * n + j];
      T[size_t(i) * N + n + i] = 1.0;
    }
    std::vector<double> beta(b), rc(N, 0.0), ub(N, INFINITY);
    for (int j = 0; j < n; ++j) {
      rc[j] = c[j];
      ub[j] = u[j];
    }
    std::vector<int> basis(m), at_upper(N, 0), row_of(N, -1);
    for (int i = 0; i < m; ++i) {
      basis[i] = n + i;
      row_of[n + i] = i;
    }
    int degenerate = 0;
    for (int it = 0; it < 50000; ++it) {
      int e = -1;
      double bestrc = tol;
      const bool bland = degenerate > 50;
      for (int j = 0; j < N; ++j) {
        if (row_of[j] >= 0 || ub[j] <= 0) continue;
        const double d = at_upper[j] ? -rc[j] : rc[j];
        if (d > bestrc) {
          bestrc = d;
          e = j;
          if (bland) break;
        }
      }
      if (e < 0) break;
      const double dir = at_upper[e] ? -1.0 : 1.0;
      double t = ub[e];
      int r = -1;
      bool leave_upper = false;
      for (int i = 0; i < m; ++i) {
        const double al = dir * T[size_t(i) * N + e];
        if (al > tol) {
          const double lim = std::max(0.0, beta[i]) / al;
          if (lim < t - 1e-12 || (r >= 0 && lim <= t + 1e-12 && basis[i] < basis[r])) {
            t = lim;
            r = i;
            leave_upper = false;
          }
        } else if (al < -tol && std::isfinite(ub[basis[i]])) {
          const double lim = std::max(0.0, ub[basis[i]] - beta[i]) / -al;
          if (lim < t - 1e-12 || (r >= 0 && lim <= t + 1e-12 && basis[i] < basis[r])) {
            t = lim;
            r = i;
            leave_upper = true;
          }
        }
      }
      if (!std::isfinite(t)) break;  // unbounded (cannot happen: A >= 0, x bounded)
      degenerate = t < 1e-12 ? degenerate + 1 : 0;
      for (int i = 0; i < m; ++i) beta[i] -= dir * t * T[size_t(i) * N + e];
      if (r < 0) {  // bound flip
        at_upper[e] ^= 1;
        continue;
      }
      const double enter_val = (at_upper[e] ? ub[e] : 0.0) + dir * t;
      const int lv = basis[r];
      row_of[lv] = -1;
      at_upper[lv] = leave_upper ? 1 : 0;
      basis[r] = e;
      row_of[e] = r;
      at_upper[e] = 0;
      beta[r] = enter_val;
      const double piv = T[size_t(r) * N + e];
      double* R = &T[size_t(r) * N];
      for (int j = 0; j < N; ++j) R[j] /= piv;
      for (int i = 0; i < m; ++i) {
        if (i == r) continue;
        const double f = T[size_t(i) * N + e];
        if (f == 0.0) continue;
        double* Ri = &T[size_t(i) * N];
        for (int j = 0; j < N; ++j) Ri[j] -= f * R[j];
      }
      const double f = rc[e];
      for (int j = 0; j < N; ++j) rc[j] -= f * R[j];
    }
    x->assign(n, 0.0);
    for (int j = 0; j < n; ++j)
      (*x)[j] = row_of[j] >= 0 ? beta[row_of[j]] : (at_upper[j] ? ub[j] : 0.0);
    double v = 0;
    for (int j = 0; j < n; ++j) v += c[j] * (*x)[j];
    return v;
  }
};

// Eqs. 4-7 on one relaxation grid g by LP-based branch and bound: maximise
// sum z (z_T in {0..g u_T}, sum_{T contains e} z_T <= g c_e), then -- among
// solutions of that sum -- the tie-breaks of sol_better.  The LP relaxation
// bounds every node; integral LP vertices have at most |E| trees, so the
// search also finds few-tree solutions.  Minimum depth: the search is rerun
// with the candidates restricted to depth <= D for each D; fewer trees: a
// local search drops one used tree at a time and re-solves.
class IlpBB {
 public:
  const int kDives = [] {
    const char* e = getenv("BLINK_ILP_DIVES");
    return e ? std::max(2, atoi(e)) : 18;
  }();
  IlpBB(const std::vector<IlpCand>& cand, const std::vector<double>& c, int g, bool multiplicity,
        int64_t node_limit)
      : cand_(cand), g_(g), node_limit_(node_limit) {
    K_ = int(cand.size());
    E_ = int(c.size());
    cap_.resize(E_);
    for (int e = 0; e < E_; ++e) cap_[e] = int64_t(std::floor(g * c[e] + 1e-9));
    ub_.resize(K_);
    for (int j = 0; j < K_; ++j) {
      int64_t uu = 1;
      if (multiplicity) {
        double bmin = 1e30;
        for (int e : cand[j].res) bmin = std::min(bmin, c[e]);
        uu = std::max<int64_t>(1, int64_t(std::floor(bmin + 1e-9)));
      }
      ub_[j] = g * uu;
    }
  }
  int64_t nodes() const { return nodes_; }
  // max sum z (the paper's ILP objective) by LP-based branch and bound
  IlpSol solve_sum() {
    std::vector<int> all(K_);
    std::iota(all.begin(), all.end(), 0);
    return max_sum(all);
  }
  // tie-breaks at that sum: few and shallow trees.  LP diving under every
  // depth bound D (the candidates restricted to depth <= D), then a local
  // search that bans one used tree at a time and dives again; best by
  // sol_better.
  IlpSol refine(IlpSol best) {
    if (best.sumz <= 0) return best;
    const int64_t zstar = best.sumz;
    std::set<int> depths;
    for (int j = 0; j < K_; ++j) depths.insert(cand_[j].depth);
    for (int D : depths) {
      if (D > best.maxdepth) break;
      std::vector<int> sub;
      for (int j = 0; j < K_; ++j)
        if (cand_[j].depth <= D) sub.push_back(j);
      for (int variant = 0; variant < kDives; ++variant) {
        IlpSol s = dive(sub, zstar, variant);
        if (s.sumz == zstar && sol_better(s.sumz, s.ntrees, s.maxdepth, s.sumdepth, best)) best = s;
      }
    }
    for (int round = 0; round < 16; ++round) {
      std::vector<std::pair<int, int>> used;
      for (int j = 0; j < K_; ++j)
        if (best.z[j] > 0) used.push_back({best.z[j], j});
      std::sort(used.begin(), used.end());
      bool improved = false;
      for (auto& uj : used) {
        std::vector<int> sub;
        for (int j = 0; j < K_; ++j)
          if (j != uj.second && cand_[j].depth <= best.maxdepth) sub.push_back(j);
        for (int variant = 0; variant < kDives && !improved; ++variant) {
          IlpSol s = dive(sub, zstar, variant);
          if (s.sumz == zstar && sol_better(s.sumz, s.ntrees, s.maxdepth, s.sumdepth, best)) {
            best = s;
            improved = true;
          }
        }
        if (improved) break;
      }
      if (!improved) break;
    }
    return best;
  }

 private:
  // max sum z over the candidates in `sub` (others fixed at 0).  `target` > 0:
  // stop at the first solution reaching it.
  IlpSol max_sum(const std::vector<int>& sub, int64_t target = -1) {
    best_ = IlpSol();
    best_.z.assign(K_, 0);
    best_.sumz = 0;
    sub_ = sub;
    target_ = target;
    nodes_ = 0;
    // greedy incumbent (heaviest MWU weight first)
    std::vector<int> ord = sub;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return cand_[a].x > cand_[b].x; });
    std::vector<int64_t> res = cap_;
    std::vector<int> z(K_, 0);
    for (int j : ord) {
      int64_t m = ub_[j];
      for (int e : cand_[j].res) m = std::min(m, res[e]);
      if (m <= 0) continue;
      z[j] = int(m);
      for (int e : cand_[j].res) res[e] -= m;
    }
    consider(z);
    std::vector<int64_t> lo(K_, 0), hi(K_, 0);
    for (int j : sub) hi[j] = ub_[j];
    node(lo, hi);
    return best_;
  }
  // LP diving toward few trees: repeatedly solve the LP over the free
  // candidates and fix the one with the largest LP value at its rounded value
  // (variant 1: rounded down), until the LP vertex is integral.  Stops
  // without a solution if the target sum becomes unreachable.
  IlpSol dive(const std::vector<int>& sub, int64_t zstar, int variant) {
    IlpSol out;
    // variants >= 2 perturb the LP objective (deterministic hash noise of
    // 1e-4 per unit) so that different vertices, hence tree sets, come out
    std::vector<double> cost(K_, 1.0);
    if (variant >= 2)
      for (int j = 0; j < K_; ++j) {
        uint64_t h = uint64_t(j + 1) * 0x9E3779B97F4A7C15ull ^ uint64_t(variant) * 0xBF58476D1CE4E5B9ull;
        h ^= h >> 31;
        h *= 0x94D049BB133111EBull;
        h ^= h >> 29;
        cost[j] = 1.0 + 1e-4 * double(h >> 11) / double(1ull << 53);
      }
    std::vector<int64_t> lo(K_, 0), hi(K_, 0);
    for (int j : sub) hi[j] = ub_[j];
    for (int step = 0; step <= K_; ++step) {
      std::vector<int64_t> res = cap_;
      int64_t base = 0;
      for (int j : sub)
        if (lo[j] > 0) {
          base += lo[j];
          for (int e : cand_[j].res) res[e] -= lo[j];
        }
      std::vector<int> cols;
      for (int j : sub)
        if (hi[j] > lo[j]) cols.push_back(j);
      std::vector<double> x;
      lp_over(cols, res, lo, hi, &x, &cost);
      double v = 0;
      for (double xq : x) v += xq;
      if (base + int64_t(std::floor(v + 1e-7)) < zstar) return out;
      int pick = -1;
      bool integral = true;
      for (size_t q = 0; q < cols.size(); ++q) {
        const double f = x[q] - std::floor(x[q] + 1e-9);
        if (std::min(f, 1.0 - f) > 1e-6) integral = false;
        if (x[q] > 1e-6 && lo[cols[q]] == 0 &&
            (pick < 0 || x[q] > x[pick] + 1e-9 ||
             (x[q] > x[pick] - 1e-9 && cand_[cols[q]].depth < cand_[cols[pick]].depth)))
          pick = int(q);
      }
      if (integral) {
        std::vector<int> z(K_, 0);
        int64_t sz = 0, sd = 0;
        int nt = 0, md = 0;
        for (int j : sub) z[j] = int(lo[j]);
        for (size_t q = 0; q < cols.size(); ++q) z[cols[q]] += int(std::llround(x[q]));
        for (int j = 0; j < K_; ++j)
          if (z[j] > 0) {
            sz += z[j];
            ++nt;
            sd += cand_[j].depth;
            md = std::max(md, cand_[j].depth);
          }
        if (sz < zstar) return out;
        out.z = z;
        out.sumz = sz;
        out.ntrees = nt;
        out.maxdepth = md;
        out.sumdepth = sd;
        return out;
      }
      if (pick < 0) return out;
      const int j = cols[pick];
      int64_t val = variant == 1 ? int64_t(std::floor(x[pick] + 1e-9)) : int64_t(std::llround(x[pick]));
      val = std::max<int64_t>(1, std::min<int64_t>(val, hi[j]));
      lo[j] = hi[j] = val;  // fixed
      // every other candidate the LP already puts at a positive integer stays
      // there (fewer LP solves per dive)
      for (size_t q = 0; q < cols.size(); ++q) {
        const int jj = cols[q];
        if (jj == j || lo[jj] > 0 || x[q] < 1.0 - 1e-6) continue;
        const double f = x[q] - std::floor(x[q] + 1e-9);
        if (std::min(f, 1.0 - f) > 1e-6) continue;
        lo[jj] = hi[jj] = int64_t(std::llround(x[q]));
      }
    }
    return out;
  }
  double lp_over(const std::vector<int>& cols, const std::vector<int64_t>& res,
                 const std::vector<int64_t>& lo, const std::vector<int64_t>& hi,
                 std::vector<double>* x, const std::vector<double>* cost = nullptr) const {
    BoundedLp L;
    L.m = E_;
    L.n = int(cols.size());
    if (L.n == 0) {
      x->clear();
      return 0.0;
    }
    L.A.assign(size_t(L.m) * L.n, 0.0);
    L.b.resize(E_);
    for (int e = 0; e < E_; ++e) L.b[e] = double(std::max<int64_t>(res[e], 0));
    L.c.assign(L.n, 1.0);
    L.u.resize(L.n);
    for (int q = 0; q < L.n; ++q) {
      const int j = cols[q];
      for (int e : cand_[j].res) L.A[size_t(e) * L.n + q] += 1.0;
      L.u[q] = double(hi[j] - lo[j]);
      if (cost) L.c[q] = (*cost)[j];
    }
    return L.solve(x);
  }
  void consider(const std::vector<int>& z) {
    int64_t sz = 0, sd = 0;
    int nt = 0, md = 0;
    for (int j = 0; j < K_; ++j)
      if (z[j] > 0) {
        sz += z[j];
        ++nt;
        sd += cand_[j].depth;
        md = std::max(md, cand_[j].depth);
      }
    if (sol_better(sz, nt, md, sd, best_)) {
      best_.z = z;
      best_.sumz = sz;
      best_.ntrees = nt;
      best_.maxdepth = md;
      best_.sumdepth = sd;
    }
  }
  bool done() const { return nodes_ > node_limit_ || (target_ > 0 && best_.sumz >= target_); }
  void node(std::vector<int64_t>& lo, std::vector<int64_t>& hi) {
    if (done()) return;
    ++nodes_;
    std::vector<int64_t> res = cap_;
    int64_t base = 0;
    for (int j : sub_)
      if (lo[j] > 0) {
        base += lo[j];
        for (int e : cand_[j].res) res[e] -= lo[j];
      }
    for (int e = 0; e < E_; ++e)
      if (res[e] < 0) return;  // infeasible
    // LP over the free parts x' = z - lo
    std::vector<int> cols;
    for (int j : sub_)
      if (hi[j] > lo[j]) cols.push_back(j);
    std::vector<double> x;
    const double v = lp_over(cols, res, lo, hi, &x);
    const int64_t bound = base + int64_t(std::floor(v + 1e-7));
    if (bound <= best_.sumz) return;  // ties are the business of refine()
    // integral?
    int br = -1;
    double bfrac = 0;
    for (int q = 0; q < int(cols.size()); ++q) {
      const double f = x[q] - std::floor(x[q] + 1e-9);
      const double d = std::min(f, 1.0 - f);
      if (d > 1e-6 && d > bfrac) {
        bfrac = d;
        br = q;
      }
    }
    if (br < 0) {
      std::vector<int> z(K_, 0);
      for (int j : sub_) z[j] = int(lo[j]);
      for (size_t q = 0; q < cols.size(); ++q) z[cols[q]] += int(std::llround(x[q]));
      consider(z);
      return;
    }
    const int j = cols[br];
    const int64_t fl = lo[j] + int64_t(std::floor(x[br] + 1e-9));
    const int64_t olo = lo[j], ohi = hi[j];
    lo[j] = fl + 1;  // up branch first
    node(lo, hi);
    lo[j] = olo;
    if (done()) return;
    hi[j] = fl;
    node(lo, hi);
    hi[j] = ohi;
  }
  const std::vector<IlpCand>& cand_;
  int g_, K_ = 0, E_ = 0;
  int64_t node_limit_, nodes_ = 0, target_ = -1;
  std::vector<int64_t> cap_, ub_;
  std::vector<int> sub_;
  IlpSol best_;
};

// The relaxation ladder of P:390 over one candidate set: g = 1, 2, 4, 8, 16,
// accept the first g whose rate sum z / g reaches (1 - gap) * opt; otherwise
// the best rate seen (not accepted).
struct Ladder {
  IlpSol sol;
  int g = 1;
  bool accepted = false;
  double rate() const { return sol.sumz < 0 ? -1.0 : double(sol.sumz) / g; }
};
Ladder run_ladder(const std::vector<IlpCand>& cands, const std::vector<double>& caps, double threshold,
                  bool multiplicity, bool integral_first) {
  Ladder best;
  for (int gi = 0; gi < 5; ++gi) {
    const int gg = 1 << gi;
    std::vector<IlpCand> cg = cands;
    if (integral_first)  // the exact packing (Broadcast) or this grid's peeling seed the incumbent
      for (auto& c : cg) {
        if (c.lovasz) c.x = 2.0;
        if (c.mult[gi] > 0) c.x = 1.0 + double(c.mult[gi]) / gg;
      }
    IlpBB bb(cg, caps, gg, multiplicity, 2000);
    IlpSol s = bb.solve_sum();
    const double r = double(s.sumz) / gg;
    if (getenv("BLINK_PLAN_DEBUG"))
      fprintf(stderr, "ladder g=%d cands=%zu sum=%lld trees=%d nodes=%lld\n", gg, cands.size(),
              (long long)s.sumz, s.ntrees, (long long)bb.nodes());
    if (r >= threshold - 1e-12) return Ladder{bb.refine(s), gg, true};
    if (r > best.rate() + 1e-12) best = Ladder{s, gg, false};
  }
  if (best.sol.sumz > 0) {
    std::vector<IlpCand> cg = cands;
    best.sol = IlpBB(cg, caps, best.g, multiplicity, 2000).refine(best.sol);
  }
  return best;
}

// Max flow (Edmonds-Karp) on a small dense integer capacity matrix.
int64_t maxflow(std::vector<std::vector<int64_t>> c, int s, int t) {
  const int n = int(c.size());
  int64_t flow = 0;
  while (true) {
    std::vector<int> prev(n, -1);
    prev[s] = s;
    std::vector<int> q{s};
    for (size_t h = 0; h < q.size() && prev[t] < 0; ++h)
      for (int v = 0; v < n; ++v)
        if (prev[v] < 0 && c[q[h]][v] > 0) {
          prev[v] = q[h];
          q.push_back(v);
        }
    if (prev[t] < 0) return flow;
    int64_t b = INT64_MAX;
    for (int v = t; v != s; v = prev[v]) b = std::min(b, c[prev[v]][v]);
    for (int v = t; v != s; v = prev[v]) {
      c[prev[v]][v] -= b;
      c[v][prev[v]] += b;
    }
    flow += b;
  }
}

// Max flow over real capacities (Edmonds-Karp on the directed edge list):
// Edmonds' theorem gives the optimal Broadcast rate.
double maxflow_real(const std::vector<double>& caps, const std::vector<WEdge>& edges, int n, int s,
                    int t) {
  std::vector<std::vector<double>> c(n, std::vector<double>(n, 0.0));
  for (size_t j = 0; j < edges.size(); ++j) c[edges[j].u][edges[j].v] += caps[j];
  double flow = 0;
  while (true) {
    std::vector<int> prev(n, -1);
    prev[s] = s;
    std::vector<int> q{s};
    for (size_t h = 0; h < q.size() && prev[t] < 0; ++h)
      for (int v = 0; v < n; ++v)
        if (prev[v] < 0 && c[q[h]][v] > 1e-12) {
          prev[v] = q[h];
          q.push_back(v);
        }
    if (prev[t] < 0) return flow;
    double b = INFINITY;
    for (int v = t; v != s; v = prev[v]) b = std::min(b, c[prev[v]][v]);
    for (int v = t; v != s; v = prev[v]) {
      c[prev[v]][v] -= b;
      c[v][prev[v]] += b;
    }
    flow += b;
  }
}

// Nash-Williams / Tutte: the optimal fractional spanning-tree packing of an
// undirected graph is min over partitions P (|P| >= 2) of cross(P) / (|P| - 1).
// Partitions enumerated as restricted growth strings (Bell(8) = 4140).
double nash_williams(int n, const std::vector<std::pair<int, int>>& pairs,
                     const std::vector<double>& caps) {
  std::vector<int> a(n, 0), mx(n, 0);
  double best = INFINITY;
  while (true) {
    const int k = *std::max_element(a.begin(), a.end()) + 1;
    if (k >= 2) {
      double cross = 0;
      for (size_t j = 0; j < pairs.size(); ++j)
        if (a[pairs[j].first] != a[pairs[j].second]) cross += caps[j];
      best = std::min(best, cross / (k - 1));
    }
    int i = n - 1;  // next restricted growth string
    while (i > 0 && a[i] == mx[i - 1] + 1) --i;
    if (i == 0) return best;
    ++a[i];
    for (int j = i + 1; j < n; ++j) a[j] = 0;
    for (int j = i; j < n; ++j) mx[j] = std::max(mx[j - 1], a[j]);
  }
}

// Integral arborescence packing by Lovasz's constructive proof of Edmonds'
// theorem: with k = min_v lambda(r, v), grow each arborescence one
// edge (u in S, v not in S) at a time, taking an edge only if the remaining
// graph keeps lambda(r, v) >= k - t.  Edges are tried in BFS order (shallow
// trees).  Used to enrich the ILP's candidate set (SURVEY 7 "hard parts" 8).
std::vector<std::vector<int>> lovasz_packing(std::vector<std::vector<int64_t>> cap, int root) {
  const int n = int(cap.size());
  int64_t k = INT64_MAX;
  for (int v = 0; v < n; ++v)
    if (v != root) k = std::min(k, maxflow(cap, root, v));
  std::vector<std::vector<int>> out;
  for (int64_t t = 1; t <= k; ++t) {
    std::vector<int> parent(n, -2), depth(n, 0);
    parent[root] = -1;
    int in_s = 1;
    while (in_s < n) {
      bool grown = false;
      // candidate edges ordered by (depth of u, u, v)
      std::vector<std::pair<int, std::pair<int, int>>> cand;
      for (int u = 0; u < n; ++u)
        if (parent[u] != -2)
          for (int v = 0; v < n; ++v)
            if (parent[v] == -2 && cap[u][v] > 0) cand.push_back({depth[u], {u, v}});
      std::sort(cand.begin(), cand.end());
      for (auto& ce : cand) {
        int u = ce.second.first, v = ce.second.second;
        cap[u][v] -= 1;
        if (maxflow(cap, root, v) >= k - t) {
          parent[v] = u;
          depth[v] = depth[u] + 1;
          ++in_s;
          grown = true;
          break;
        }
        cap[u][v] += 1;
      }
      if (!grown) return out;  // cannot happen for integral capacities (lemma)
    }
    out.push_back(parent);
  }
  return out;
}

int tree_depth(const std::vector<int>& parent);

// hop distances from root over positive integer capacities
std::vector<int> bfs_depths(int n, const std::vector<std::vector<int64_t>>& cap, int root) {
  std::vector<int> d(n, 0), seen(n, 0), q{root};
  seen[root] = 1;
  for (size_t h = 0; h < q.size(); ++h)
    for (int v = 0; v < n; ++v)
      if (!seen[v] && cap[q[h]][v] > 0) {
        seen[v] = 1;
        d[v] = d[q[h]] + 1;
        q.push_back(v);
      }
  return d;
}

// Shallow integral Broadcast packing (product heuristic, R#21): for depth
// bounds D from the root's eccentricity up to below `cur_depth`, sample random
// arborescences of depth <= D (random growth: an edge from the tree to a new
// vertex, its tail at depth < D, chosen uniformly) and look for k of them
// that fit the integer capacities (the ILP at grid 1 over the samples).
// Returns the first (shallowest) such packing, or nothing.  Shallow trees
// shorten every chunk's pipeline fill.  Graphs up to 16 ranks.
std::vector<std::vector<int>> sample_shallow_packing(const std::vector<std::vector<int64_t>>& cap, int root,
                                                     int64_t k, int cur_depth) {
  const int n = int(cap.size());
  if (k <= 0 || n > 16) return {};
  std::vector<int> d0 = bfs_depths(n, cap, root);
  int ecc = 0;
  for (int x : d0) ecc = std::max(ecc, x);
  std::vector<std::pair<int, int>> elist;
  std::vector<double> ecap;
  std::map<std::pair<int, int>, int> eid;
  for (int u = 0; u < n; ++u)
    for (int v = 0; v < n; ++v)
      if (cap[u][v] > 0) {
        eid[{u, v}] = int(elist.size());
        elist.push_back({u, v});
        ecap.push_back(double(cap[u][v]));
      }
  uint32_t st = 0x9e3779b9u;
  auto rnd = [&]() {
    st ^= st << 13;
    st ^= st >> 17;
    st ^= st << 5;
    return st;
  };
  for (int D = ecc; D < cur_depth; ++D) {
    std::map<std::vector<int>, int> seen;
    std::vector<IlpCand> cands;
    std::vector<std::vector<int>> pars;
    for (int s = 0; s < 1500; ++s) {
      std::vector<int> parent(n, -2), depth(n, 0);
      parent[root] = -1;
      int in_t = 1;
      bool ok = true;
      while (in_t < n && ok) {
        std::vector<std::pair<int, int>> opts;
        for (int u = 0; u < n; ++u)
          if (parent[u] != -2 && depth[u] < D)
            for (int v = 0; v < n; ++v)
              if (parent[v] == -2 && cap[u][v] > 0) opts.push_back({u, v});
        if (opts.empty()) {
          ok = false;
          break;
        }
        const auto e = opts[rnd() % opts.size()];
        parent[e.second] = e.first;
        depth[e.second] = depth[e.first] + 1;
        ++in_t;
      }
      if (!ok) continue;
      std::vector<int> res;
      for (int v = 0; v < n; ++v)
        if (parent[v] >= 0) res.push_back(eid[{parent[v], v}]);
      std::sort(res.begin(), res.end());
      if (seen.count(res)) continue;
      seen[res] = 1;
      IlpCand c{res, tree_depth(parent), 1.0};
      cands.push_back(c);
      pars.push_back(parent);
    }
    // plus the trees of MWU runs whose tree oracle is a depth-bounded greedy
    // (Prim-like: the shortest edge from the tree to a new vertex whose tail
    // has depth < D) -- the same Garg-Koenemann loop as the paper's MWU,
    // restricted to shallow trees
    for (double eps : {0.1, 0.05}) {
      MwuResult mr;
      auto tree_of = [&](const std::vector<double>& len) {
        std::vector<int> parent(n, -2), depth(n, 0), res;
        parent[root] = -1;
        for (int step = 1; step < n; ++step) {
          int be = -1;
          for (size_t j = 0; j < elist.size(); ++j) {
            const int u = elist[j].first, v = elist[j].second;
            if (parent[u] == -2 || parent[v] != -2 || depth[u] >= D) continue;
            if (be < 0 || len[j] < len[be]) be = int(j);
          }
          if (be < 0) return std::vector<int>();
          parent[elist[be].second] = elist[be].first;
          depth[elist[be].second] = depth[elist[be].first] + 1;
          res.push_back(be);
        }
        std::sort(res.begin(), res.end());
        return res;
      };
      if (!run_mwu(ecap, eps, tree_of, &mr)) continue;
      for (auto& kv : mr.x) {
        if (seen.count(kv.first)) continue;
        seen[kv.first] = 1;
        std::vector<int> parent(n, -1);
        for (int e : kv.first) parent[elist[e].second] = elist[e].first;
        IlpCand c{kv.first, tree_depth(parent), kv.second};
        cands.push_back(c);
        pars.push_back(parent);
      }
    }
    if (int64_t(cands.size()) < k) continue;
    IlpBB bb(cands, ecap, 1, false, 3000);
    IlpSol sol = bb.solve_sum();
    if (sol.sumz >= k) {
      std::vector<std::vector<int>> out;
      for (size_t j = 0; j < cands.size(); ++j)
        if (sol.z[j] > 0) out.push_back(pars[j]);
      return out;
    }
  }
  return {};
}

// Greedy integral peeling of undirected spanning trees: Kruskal preferring
// links with the largest RELATIVE residual capacity (balances single and
// parallel links); candidates for the AllReduce ILP.
std::vector<std::vector<int>> peel_spanning(int n, const std::vector<std::pair<int, int>>& pairs,
                                            std::vector<int64_t> res) {
  std::vector<std::vector<int>> out;
  const std::vector<int64_t> cap0 = res;
  while (true) {
    std::vector<double> len(pairs.size());
    for (size_t j = 0; j < pairs.size(); ++j)
      len[j] = res[j] > 0 ? double(cap0[j]) / double(res[j]) : 1e30;
    std::vector<int> t = min_spanning_tree(n, pairs, len);
    if (t.empty()) break;
    bool ok = true;
    for (int j : t) ok = ok && res[j] > 0;
    if (!ok) break;
    for (int j : t) res[j] -= 1;
    out.push_back(t);
  }
  return out;
}

int tree_depth(const std::vector<int>& parent) {
  int best = 0;
  for (size_t v = 0; v < parent.size(); ++v) {
    int d = 0, x = int(v);
    while (parent[x] >= 0 && d <= int(parent.size())) {
      x = parent[x];
      ++d;
    }
    best = std::max(best, d);
  }
  return best;
}

// Orient an undirected tree (edge list) away from `root`.
std::vector<int> orient(int n, const std::vector<std::pair<int, int>>& edges, int root) {
  std::vector<std::vector<int>> adj(n);
  for (auto& e : edges) {
    adj[e.first].push_back(e.second);
    adj[e.second].push_back(e.first);
  }
  std::vector<int> parent(n, -2);
  parent[root] = -1;
  std::vector<int> st{root};
  while (!st.empty()) {
    int u = st.back();
    st.pop_back();
    for (int w : adj[u])
      if (parent[w] == -2) {
        parent[w] = u;
        st.push_back(w);
      }
  }
  return parent;
}

// Tree centre: minimum eccentricity, ties -> lowest rank (R#9).
int centre(int n, const std::vector<std::pair<int, int>>& edges) {
  int best = 0, bestecc = 1 << 30;
  for (int s = 0; s < n; ++s) {
    int e = tree_depth(orient(n, edges, s));
    if (e < bestecc) {
      bestecc = e;
      best = s;
    }
  }
  return best;
}

void sort_trees(std::vector<Tree>* trees, const std::vector<std::vector<std::pair<int, int>>>& keys) {
  std::vector<int> idx(trees->size());
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
    const Tree &A = (*trees)[a], &B = (*trees)[b];
    // weight descending: A.wnum/A.wden > B.wnum/B.wden
    __int128 l = (__int128)A.wnum * B.wden, r = (__int128)B.wnum * A.wden;
    if (l != r) return l > r;
    return keys[a] < keys[b];
  });
  std::vector<Tree> out;
  for (int i : idx) out.push_back((*trees)[i]);
  trees->swap(out);
}

int64_t gcd64(int64_t a, int64_t b) { return b == 0 ? a : gcd64(b, a % b); }

}  // namespace

// NEXT-4: three-phase multi-server AllReduce as spanning trees.
// Partition p (K = min over servers of the local packing's tree count, equal
// weights, R#24) uses local tree T_{s,p} on every server s with server-local
// root r_{s,p} (minimum eccentricity among GPUs not yet a root of this
// server, R#25: "Each data partition has a distinct server-local root",
// P:404).  Sub-slice q of partition p is the tree made of every T_{s,p}
// oriented to r_{s,p} plus the cross-server star r_{s,p} -> r_{q,p}
// ("n one-hop cross-server trees").  Reduce then broadcast along it
// runs phases 1-3, pipelined per chunk.
blink_result_t make_multiserver_plan(const Graph& g, const blink_config_t& cfg, Plan* out,
                                     std::string* err) {
  const int ns = int(g.servers.size());
  std::vector<Plan> local(ns);
  int K = 1 << 30;
  for (int s = 0; s < ns; ++s) {
    const std::vector<int>& ids = g.servers[s];
    const int k = int(ids.size());
    if (k == 1) continue;
    Graph lg;
    lg.n = k;
    lg.switch_model = false;
    lg.cap.assign(k, std::vector<double>(k, 0.0));
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) lg.cap[a][b] = g.cap[ids[a]][ids[b]];
    blink_result_t r = make_plan(lg, kAllReduce, -1, cfg, &local[s], err);
    if (r != BLINK_SUCCESS) return r;
    K = std::min(K, int(local[s].trees.size()));
  }
  if (K == (1 << 30)) K = 1;
  K = std::max(1, std::min(K, kMaxTrees / std::max(1, ns)));
  if (ns > kMaxTrees) {
    *err = "too many servers";
    return BLINK_ERR_UNSUPPORTED;
  }
  // per server, per partition: undirected global edges + local root
  std::vector<std::vector<std::vector<std::pair<int, int>>>> edges(ns, std::vector<std::vector<std::pair<int, int>>>(K));
  std::vector<std::vector<int>> root(ns, std::vector<int>(K, -1));
  for (int s = 0; s < ns; ++s) {
    const std::vector<int>& ids = g.servers[s];
    const int k = int(ids.size());
    std::vector<int> used(k, 0);
    for (int p = 0; p < K; ++p) {
      if (k == 1) {
        root[s][p] = ids[0];
        continue;
      }
      const Tree& t = local[s].trees[p];
      std::vector<std::pair<int, int>> le;
      for (int v = 0; v < k; ++v)
        if (t.parent[v] >= 0) le.push_back({t.parent[v], v});
      int best = -1, bestecc = 1 << 30, fallback = -1, fbecc = 1 << 30;
      for (int v = 0; v < k; ++v) {
        int e = tree_depth(orient(k, le, v));
        if (e < fbecc) {
          fbecc = e;
          fallback = v;
        }
        if (!used[v] && e < bestecc) {
          bestecc = e;
          best = v;
        }
      }
      if (best < 0) best = fallback;
      used[best] = 1;
      root[s][p] = ids[best];
      for (auto& e : le) edges[s][p].push_back({ids[e.first], ids[e.second]});
    }
  }
  out->trees.clear();
  for (int p = 0; p < K; ++p)
    for (int q = 0; q < ns; ++q) {
      std::vector<std::pair<int, int>> all;
      for (int s = 0; s < ns; ++s) all.insert(all.end(), edges[s][p].begin(), edges[s][p].end());
      for (int s = 0; s < ns; ++s)
        if (s != q) all.push_back({root[s][p], root[q][p]});
      Tree t;
      t.root = root[q][p];
      t.parent = orient(g.n, all, t.root);
      t.depth = tree_depth(t.parent);
      out->trees.push_back(t);
    }
  out->rate_num = K;
  out->rate_den = 1;
  out->grid = 1;
  return BLINK_SUCCESS;
}

// ============================================================== plans
blink_result_t make_plan(const Graph& g, int coll, int root, const blink_config_t& cfg, Plan* out,
                         std::string* err) {
  const int n = g.n;
  *out = Plan();
  out->coll = coll;
  out->root = coll == kBroadcast ? root : -1;
  out->nranks = n;
  out->switch_model = g.switch_model;
  if (n <= 0 || n > kMaxRanks) {
    *err = "nranks must be in [1, " + std::to_string(kMaxRanks) + "]";
    return BLINK_ERR_UNSUPPORTED;
  }
  if (coll == kBroadcast && (root < 0 || root >= n)) {
    *err = "root " + std::to_string(root) + " out of range [0," + std::to_string(n) + ")";
    return BLINK_ERR_INVALID_ARGUMENT;
  }
  if (n == 1) {
    Tree t;
    t.root = 0;
    t.parent = {-1};
    out->trees.push_back(t);
    out->rate_num = 1;
    return BLINK_SUCCESS;
  }
  if (g.switch_model) {
    if (coll == kAllReduce) {
      // m one-hop stars, star j rooted at j, weight 1/2 in K_m link units
      for (int j = 0; j < n; ++j) {
        Tree t;
        t.root = j;
        t.parent.assign(n, j);
        t.parent[j] = -1;
        t.wnum = 1;
        t.wden = 2;
        t.depth = 1;
        out->trees.push_back(t);
      }
      out->rate_num = n % 2 == 0 ? n / 2 : n;
      out->rate_den = n % 2 == 0 ? 1 : 2;
      out->grid = 2;
    } else {
      // R#10: m-1 two-level trees r -> k -> others (Edmonds optimum m-1); the
      // one-hop variant is selected per call size in size_plan.
      for (int k = 0; k < n; ++k) {
        if (k == root) continue;
        Tree t;
        t.root = root;
        t.parent.assign(n, k);
        t.parent[root] = -1;
        t.parent[k] = root;
        t.depth = n > 2 ? 2 : 1;
        out->trees.push_back(t);
      }
      out->rate_num = n - 1;
    }
    return BLINK_SUCCESS;
  }

  if (g.multi_server) {
    if (coll != kAllReduce) {
      *err = "multi-server graphs support AllReduce only (three-phase protocol, P:448-456)";
      return BLINK_ERR_UNSUPPORTED;
    }
    return make_multiserver_plan(g, cfg, out, err);
  }

  // ---------------- explicit link graph: MWU runs, then the ILP ladder
  double cmin = INFINITY;
  for (int u = 0; u < n; ++u)
    for (int v = 0; v < n; ++v)
      if (g.cap[u][v] > 0) cmin = std::min(cmin, g.cap[u][v]);
  const double eps = cfg.mwu_eps > 0 ? cfg.mwu_eps : 0.1;
  const double gap = cfg.ilp_gap > 0 ? cfg.ilp_gap : 0.05;
  // P:390's candidates: the trees of several MWU runs (the configured eps and
  // eps / 2, each with ascending and descending tie-breaks; SURVEY 7 hard
  // part 8); c* = the best MWU rate.  Same runs as oracle/packing.py mwu_runs.
  const double run_eps[4] = {eps, eps, eps / 2, eps / 2};
  const bool run_desc[4] = {false, true, false, true};

  std::vector<IlpCand> cands;
  std::vector<std::vector<int>> cand_parent;
  std::vector<double> caps;
  double c_star = 0, opt = 0;
  std::map<std::vector<int>, int> cand_of;  // resource list -> candidate index
  auto add_cand = [&](const std::vector<int>& res, const std::vector<int>& par, double x) -> int {
    auto it = cand_of.find(res);
    if (it != cand_of.end()) {
      cands[it->second].x = std::max(cands[it->second].x, x);
      return it->second;
    }
    cand_of[res] = int(cands.size());
    cands.push_back({res, tree_depth(par), x});
    cand_parent.push_back(par);
    return int(cands.size()) - 1;
  };
  if (coll == kBroadcast) {
    // resources = directed edges, capacities in units of the smallest link
    std::vector<WEdge> edges;
    for (int u = 0; u < n; ++u)
      for (int v = 0; v < n; ++v)
        if (g.cap[u][v] > 0) {
          edges.push_back({u, v, 0.0, u * n + v});
          caps.push_back(g.cap[u][v] / cmin);
        }
    // reachability from the root
    std::vector<int> seen(n, 0);
    std::vector<int> st{root};
    seen[root] = 1;
    while (!st.empty()) {
      int u = st.back();
      st.pop_back();
      for (auto& e : edges)
        if (e.u == u && !seen[e.v]) {
          seen[e.v] = 1;
          st.push_back(e.v);
        }
    }
    for (int v = 0; v < n; ++v)
      if (!seen[v]) {
        *err = "GPU " + std::to_string(v) + " is unreachable from root " + std::to_string(root);
        return BLINK_ERR_TOPOLOGY;
      }
    std::map<int, int> key_to_res;
    for (size_t j = 0; j < edges.size(); ++j) key_to_res[edges[j].u * n + edges[j].v] = int(j);
    for (int run = 0; run < 4; ++run) {
      for (auto& e : edges) e.key = run_desc[run] ? n * n - (e.u * n + e.v) : e.u * n + e.v;
      MwuResult mr;
      auto tree_of = [&](const std::vector<double>& len) {
        for (size_t j = 0; j < edges.size(); ++j) edges[j].w = len[j];
        std::vector<int> par = min_arborescence(n, root, edges);
        std::vector<int> res;
        if (par.empty()) return res;
        for (int v = 0; v < n; ++v)
          if (par[v] >= 0) res.push_back(key_to_res[par[v] * n + v]);
        std::sort(res.begin(), res.end());
        return res;
      };
      if (!run_mwu(caps, run_eps[run], tree_of, &mr)) {
        *err = "MWU failed to converge";
        return BLINK_ERR_INTERNAL;
      }
      c_star = std::max(c_star, mr.rate);
      for (auto& kv : mr.x) {
        std::vector<int> par(n, -1);
        for (int e : kv.first) par[edges[e].v] = edges[e].u;
        add_cand(kv.first, par, kv.second);
      }
    }
    // Edmonds' theorem: the optimal rate is min_v maxflow(root -> v)
    opt = INFINITY;
    for (int v = 0; v < n; ++v)
      if (v != root) opt = std::min(opt, maxflow_real(caps, edges, n, root, v));
    // product extra: exact integral candidates (Lovasz), weight 1 each, plus
    // shallow integral packings (sample_shallow_packing)
    {
      std::vector<std::vector<int64_t>> ic(n, std::vector<int64_t>(n, 0));
      for (size_t j = 0; j < edges.size(); ++j)
        ic[edges[j].u][edges[j].v] = int64_t(std::floor(caps[j] + 1e-9));
      std::vector<std::vector<int>> lv = lovasz_packing(ic, root);
      int cur_d = 0;
      for (auto& par : lv) cur_d = std::max(cur_d, tree_depth(par));
      for (auto& c : cands) cur_d = std::max(cur_d, c.depth);
      std::vector<std::vector<int>> sh = sample_shallow_packing(ic, root, int64_t(lv.size()), cur_d);
      lv.insert(lv.end(), sh.begin(), sh.end());
      for (auto& par : lv) {
        std::vector<int> res;
        for (int v = 0; v < n; ++v)
          if (par[v] >= 0) res.push_back(key_to_res[par[v] * n + v]);
        std::sort(res.begin(), res.end());
        const bool known = cand_of.count(res) > 0;
        const int j = add_cand(res, par, 0.0);
        cands[j].lovasz = 1;
        if (!known) cands[j].paper = 0;
      }
    }
  } else {
    // undirected pairs; every link needs its reverse
    std::vector<std::pair<int, int>> pairs;
    for (int u = 0; u < n; ++u)
      for (int v = u + 1; v < n; ++v) {
        bool f = g.cap[u][v] > 0, b = g.cap[v][u] > 0;
        if (f != b) {
          *err = "link " + std::to_string(f ? u : v) + "->" + std::to_string(f ? v : u) +
                 " has no reverse edge (AllReduce needs bidirectional links, P:397)";
          return BLINK_ERR_TOPOLOGY;
        }
        if (f) {
          pairs.push_back({u, v});
          caps.push_back(std::min(g.cap[u][v], g.cap[v][u]) / cmin);
        }
      }
    for (int run = 0; run < 4; ++run) {
      MwuResult mr;
      const bool desc = run_desc[run];
      auto tree_of = [&](const std::vector<double>& len) { return min_spanning_tree(n, pairs, len, desc); };
      if (!run_mwu(caps, run_eps[run], tree_of, &mr)) {
        *err = "MWU failed (graph disconnected?)";
        return BLINK_ERR_TOPOLOGY;
      }
      c_star = std::max(c_star, mr.rate);
      for (auto& kv : mr.x) {
        std::vector<std::pair<int, int>> te;
        for (int e : kv.first) te.push_back(pairs[e]);
        add_cand(kv.first, orient(n, te, centre(n, te)), kv.second);
      }
    }
    // Nash-Williams: the optimal undirected packing rate, by partition
    // enumeration up to 8 GPUs; larger allocations use the MWU rate
    opt = n <= 8 ? nash_williams(n, pairs, caps) : c_star;
    // product extra: greedy integral peelings at the grid scales
    for (int gi = 0; gi < 4; ++gi) {
      const int gg = 1 << gi;
      std::vector<int64_t> res(caps.size());
      for (size_t j = 0; j < caps.size(); ++j) res[j] = int64_t(std::floor(gg * caps[j] + 1e-9));
      std::map<std::vector<int>, int> mult;
      for (auto& t : peel_spanning(n, pairs, res)) mult[t]++;
      for (auto& kv : mult) {
        std::vector<std::pair<int, int>> te;
        for (int e : kv.first) te.push_back(pairs[e]);
        const bool known = cand_of.count(kv.first) > 0;
        const int j = add_cand(kv.first, orient(n, te, centre(n, te)), 0.0);
        cands[j].mult[gi] += kv.second;
        if (!known) cands[j].paper = 0;
      }
    }
  }
  out->c_star = c_star;
  out->opt = opt;

  // the ILP over the MWU candidates with the relaxation ladder,
  // accepted within `gap` of the optimal rate (R#3).  Product heuristics
  // (R#21: Lovasz / peeled candidates; R#26: multiplicity) run afterwards and
  // replace the paper's plan only when it missed the threshold or when they
  // reach it with fewer trees / shallower trees.
  const double threshold = (1.0 - gap) * opt;
  std::vector<IlpCand> paper_cands;
  std::vector<int> paper_idx;
  for (size_t j = 0; j < cands.size(); ++j)
    if (cands[j].paper) {
      paper_cands.push_back(cands[j]);
      paper_idx.push_back(int(j));
    }
  Ladder lp = run_ladder(paper_cands, caps, threshold, false, false);
  // map the paper solution onto the full candidate list
  IlpSol best;
  best.z.assign(cands.size(), 0);
  for (size_t q = 0; q < paper_idx.size(); ++q)
    if (!lp.sol.z.empty()) best.z[paper_idx[q]] = lp.sol.z[q];
  best.sumz = lp.sol.sumz;
  best.ntrees = lp.sol.ntrees;
  best.maxdepth = lp.sol.maxdepth;
  best.sumdepth = lp.sol.sumdepth;
  int bestg = lp.g;
  bool accepted = lp.accepted;
  for (int pass = 0; pass < 2; ++pass) {  // pass 1: multiplicity fallback (R#26)
    if (pass == 1 && accepted) break;
    Ladder lx = run_ladder(cands, caps, threshold, pass == 1, true);
    bool take;
    if (lx.accepted != accepted) {
      take = lx.accepted;
    } else if (!accepted) {
      take = lx.rate() > double(best.sumz) / bestg + 1e-12;
    } else {  // both accepted: fewer trees, then shallower, then higher rate
      const IlpSol& a = lx.sol;
      if (a.ntrees != best.ntrees) take = a.ntrees < best.ntrees;
      else if (a.maxdepth != best.maxdepth) take = a.maxdepth < best.maxdepth;
      else if (a.sumdepth != best.sumdepth) take = a.sumdepth < best.sumdepth;
      else take = lx.rate() > double(best.sumz) / bestg + 1e-12;
    }
    if (take) {
      best = lx.sol;
      bestg = lx.g;
      accepted = lx.accepted;
    }
  }
  out->accepted = accepted;
  std::vector<std::vector<std::pair<int, int>>> keys;
  for (size_t j = 0; j < cands.size(); ++j) {
    if (best.z.empty() || best.z[j] == 0) continue;
    Tree t;
    t.parent = cand_parent[j];
    for (int v = 0; v < n; ++v)
      if (t.parent[v] < 0) t.root = v;
    int64_t gd = gcd64(best.z[j], bestg);
    t.wnum = best.z[j] / gd;
    t.wden = bestg / gd;
    t.depth = cands[j].depth;
    out->trees.push_back(t);
    std::vector<std::pair<int, int>> k;
    for (int v = 0; v < n; ++v)
      if (t.parent[v] >= 0) {
        if (coll == kBroadcast)
          k.push_back({t.parent[v], v});
        else
          k.push_back({std::min(t.parent[v], v), std::max(t.parent[v], v)});
      }
    std::sort(k.begin(), k.end());
    keys.push_back(k);
  }
  if (out->trees.empty()) {
    *err = "ILP found no tree";
    return BLINK_ERR_INTERNAL;
  }
  if (int(out->trees.size()) > kMaxTrees) {
    *err = "plan needs " + std::to_string(out->trees.size()) + " trees (max " +
           std::to_string(kMaxTrees) + ")";
    return BLINK_ERR_UNSUPPORTED;
  }
  sort_trees(&out->trees, keys);
  out->grid = bestg;
  out->rate_num = best.sumz;
  out->rate_den = bestg;
  int64_t gd = gcd64(out->rate_num, out->rate_den);
  out->rate_num /= gd;
  out->rate_den /= gd;
  return BLINK_SUCCESS;
}

// ============================================================== latency plan
// R#27: calls at or below cfg.shallow_max_bytes on a link graph run on ONE
// minimum-depth tree.  Small calls are latency-bound: a chunk waits for the
// whole chunk at every hop, so time grows with depth, and
// the paper's answer on the switch is the depth-1 tree.  The
// tree: BFS distances d(v) from the root over links of positive capacity
// (Broadcast: directed u -> v; AllReduce: both directions present), and
// parent(v) = the lowest-rank u with d(u) = d(v) - 1 and a link u -> v.
// AllReduce roots it at the graph centre (minimum BFS eccentricity, ties ->
// lowest rank, as R#9 does per tree).
namespace {
std::vector<int> bfs_dist(const Graph& g, int src, bool undirected) {
  std::vector<int> d(g.n, -1);
  std::vector<int> q{src};
  d[src] = 0;
  for (size_t h = 0; h < q.size(); ++h) {
    const int u = q[h];
    for (int v = 0; v < g.n; ++v) {
      const bool link = g.cap[u][v] > 0 && (!undirected || g.cap[v][u] > 0);
      if (link && d[v] < 0) {
        d[v] = d[u] + 1;
        q.push_back(v);
      }
    }
  }
  return d;
}
}  // namespace

bool use_shallow_plan(const Graph& g, int coll, size_t bytes, const blink_config_t& cfg) {
  // bytes == 0: plan introspection (blink_get_plan / blink_plan_json with
  // count 0) shows the size-independent packed plan
  return !g.switch_model && !g.multi_server && g.n > 2 && bytes > 0 && bytes <= cfg.shallow_max_bytes &&
         (coll == kBroadcast || coll == kAllReduce);
}

blink_result_t make_shallow_plan(const Graph& g, int coll, int root, Plan* out, std::string* err) {
  const int n = g.n;
  const bool und = coll == kAllReduce;
  *out = Plan();
  out->coll = coll;
  out->root = coll == kBroadcast ? root : -1;
  out->nranks = n;
  if (coll == kBroadcast && (root < 0 || root >= n)) {
    *err = "root " + std::to_string(root) + " out of range [0," + std::to_string(n) + ")";
    return BLINK_ERR_INVALID_ARGUMENT;
  }
  if (und)  // every link needs its reverse, as for the packed plan
    for (int u = 0; u < n; ++u)
      for (int v = u + 1; v < n; ++v)
        if ((g.cap[u][v] > 0) != (g.cap[v][u] > 0)) {
          const bool f = g.cap[u][v] > 0;
          *err = "link " + std::to_string(f ? u : v) + "->" + std::to_string(f ? v : u) +
                 " has no reverse edge (AllReduce needs bidirectional links, P:397)";
          return BLINK_ERR_TOPOLOGY;
        }
  int r = root;
  if (und) {  // centre: minimum eccentricity, ties -> lowest rank
    int best = 1 << 30;
    for (int s = 0; s < n; ++s) {
      const std::vector<int> d = bfs_dist(g, s, true);
      int ecc = 0;
      for (int v = 0; v < n; ++v) ecc = d[v] < 0 ? (1 << 29) : std::max(ecc, d[v]);
      if (ecc < best) {
        best = ecc;
        r = s;
      }
    }
  }
  const std::vector<int> d = bfs_dist(g, r, und);
  Tree t;
  t.root = r;
  t.parent.assign(n, -1);
  for (int v = 0; v < n; ++v) {
    if (d[v] < 0) {
      *err = "rank " + std::to_string(v) + " is not reachable from rank " + std::to_string(r) +
             (und ? " over bidirectional links" : "");
      return BLINK_ERR_TOPOLOGY;
    }
    if (v == r) continue;
    for (int u = 0; u < n; ++u)
      if (d[u] == d[v] - 1 && g.cap[u][v] > 0 && (!und || g.cap[v][u] > 0)) {
        t.parent[v] = u;
        break;
      }
    t.depth = std::max(t.depth, d[v]);
  }
  out->trees.push_back(t);
  out->rate_num = 1;
  out->rate_den = 1;
  return BLINK_SUCCESS;
}

// ============================================================== NEXT-3 on link graphs
// "Gather is the inverse of Broadcast, and AllGather is AllReduce
// without using a reduction function."  Block plans (Plan::blocks): tree j
// covers block j of the m-block buffer.
//  AllGather: block j is broadcast from rank j down one spanning arborescence
//    rooted at j -- the AllReduce pattern (every rank's contribution reaches
//    every rank) with concatenation instead of a combine.  Each arborescence
//    is a minimum-depth (BFS) tree, as R#27's small-call tree; among the
//    vertices one level up with a link to v, v's parent is the one whose link
//    is least loaded relative to its capacity after the roots before j
//    (ties: lowest rank), so the m trees spread over the links.
//  ReduceScatter: block j reduces toward rank j along the same kind of tree
//    over bidirectional links (the reduce half of AllReduce); inner
//    ranks keep their partials in a block-sized relay area.
//  Gather to r: the minimum-depth Broadcast tree of r, reversed ("the inverse
//    of Broadcast").  Block j travels along j's path to r; tree j is that
//    chain rooted at j, and ranks off the chain are not members (-2).  Tree r
//    is r alone (its own block).  Parents are chosen deepest level first so
//    that subtree sizes are known: v joins the candidate whose resulting
//    subtree, over the capacity of the link that carries it on toward r,
//    is smallest (ties: lowest rank).
blink_result_t make_block_plan(const Graph& g, int coll, int root, Plan* out, std::string* err) {
  const int n = g.n;
  *out = Plan();
  out->coll = coll;
  out->root = coll == kGather ? root : -1;
  out->nranks = n;
  out->blocks = true;
  auto cap = [&](int u, int v) { return g.cap[u][v]; };
  const bool rs = coll == kReduceScatter;
  if (rs)  // reduce toward root j and the acks back down need both directions
    for (int u = 0; u < n; ++u)
      for (int v = u + 1; v < n; ++v)
        if ((g.cap[u][v] > 0) != (g.cap[v][u] > 0)) {
          const bool f = g.cap[u][v] > 0;
          *err = "link " + std::to_string(f ? u : v) + "->" + std::to_string(f ? v : u) +
                 " has no reverse edge (ReduceScatter needs bidirectional links, P:397)";
          return BLINK_ERR_TOPOLOGY;
        }
  if (coll == kAllGather || rs) {
    // AllGather: block j broadcast down the arborescence rooted at j.
    // ReduceScatter: block j reduced up the same shape of tree toward j (the
    // reduce half of AllReduce), partials relayed by inner ranks.
    std::vector<std::vector<double>> load(n, std::vector<double>(n, 0.0));
    for (int j = 0; j < n; ++j) {
      const std::vector<int> d = bfs_dist(g, j, rs);
      Tree t;
      t.root = j;
      t.parent.assign(n, -1);
      int maxd = 0;
      for (int v = 0; v < n; ++v) maxd = std::max(maxd, d[v]);
      for (int v = 0; v < n; ++v) {
        if (d[v] < 0) {
          *err = "rank " + std::to_string(v) + " is not reachable from rank " + std::to_string(j);
          return BLINK_ERR_TOPOLOGY;
        }
      }
      for (int lvl = 1; lvl <= maxd; ++lvl)
        for (int v = 0; v < n; ++v) {
          if (d[v] != lvl) continue;
          int best = -1;
          double bs = INFINITY;
          for (int u = 0; u < n; ++u)
            if (d[u] == lvl - 1 && cap(u, v) > 0) {
              const double sc = (load[u][v] + 1.0) / cap(u, v);
              if (sc < bs - 1e-12) {
                bs = sc;
                best = u;
              }
            }
          t.parent[v] = best;
          load[best][v] += 1.0;
        }
      t.depth = maxd;
      out->trees.push_back(t);
    }
  } else {
    if (root < 0 || root >= n) {
      *err = "root " + std::to_string(root) + " out of range [0," + std::to_string(n) + ")";
      return BLINK_ERR_INVALID_ARGUMENT;
    }
    // distances TO the root over links v -> u (the reversed Broadcast tree)
    Graph rg = g;
    for (int u = 0; u < n; ++u)
      for (int v = 0; v < n; ++v) rg.cap[u][v] = g.cap[v][u];
    const std::vector<int> d = bfs_dist(rg, root, false);
    int maxd = 0;
    for (int v = 0; v < n; ++v) {
      if (d[v] < 0) {
        *err = "rank " + std::to_string(v) + " cannot reach the gather root " + std::to_string(root);
        return BLINK_ERR_TOPOLOGY;
      }
      maxd = std::max(maxd, d[v]);
    }
    std::vector<int> up(n, -1), sub(n, 1);  // next hop toward the root, subtree size
    for (int lvl = maxd; lvl >= 1; --lvl)
      for (int v = 0; v < n; ++v) {
        if (d[v] != lvl) continue;
        int best = -1;
        double bs = INFINITY;
        for (int u = 0; u < n; ++u)
          if (d[u] == lvl - 1 && cap(v, u) > 0) {
            const double c = lvl == 1 ? cap(v, u) : (d[u] == 1 ? cap(u, root) : cap(v, u));
            const double sc = double(sub[u] + sub[v]) / c;
            if (sc < bs - 1e-12) {
              bs = sc;
              best = u;
            }
          }
        up[v] = best;
        sub[best] += sub[v];
      }
    for (int j = 0; j < n; ++j) {
      Tree t;
      t.root = j;
      t.parent.assign(n, -2);
      t.parent[j] = -1;
      int hops = 0;
      for (int v = j; v != root; v = up[v], ++hops) t.parent[up[v]] = v;
      t.depth = hops;
      out->trees.push_back(t);
    }
  }
  out->rate_num = 1;
  out->rate_den = 1;
  return BLINK_SUCCESS;
}

// ============================================================== split + chunks
blink_result_t size_plan(const Plan& p, size_t count, int esize, const blink_config_t& cfg,
                         int ctas_hint, std::vector<TreeRange>* out, std::string* err) {
  out->clear();
  const int k = int(p.trees.size());
  const size_t S = count * size_t(esize) * (p.blocks ? size_t(k) : 1);
  // R#11: b_i = floor(G * sum_{j<i} w_j / W) with exact rationals
  int64_t L = 1;
  for (const Tree& t : p.trees) L = L / gcd64(L, t.wden) * t.wden;
  std::vector<int64_t> wi(k);
  int64_t W = 0;
  for (int i = 0; i < k; ++i) {
    wi[i] = p.trees[i].wnum * (L / p.trees[i].wden);
    W += wi[i];
  }
  const int64_t G = int64_t(S / kGrain);
  int64_t acc = 0;
  std::vector<int64_t> b(k + 1);
  for (int i = 0; i < k; ++i) {
    b[i] = int64_t((__int128)G * acc / W);
    acc += wi[i];
  }
  b[k] = G;
  for (int i = 0; i < k; ++i) {
    TreeRange r;
    int64_t lo = b[i] * kGrain, hi = (i == k - 1) ? int64_t(S) : b[i + 1] * kGrain;
    if (p.blocks) {  // RS / AG: block i = [i*count, (i+1)*count) elements
      lo = int64_t(i) * int64_t(count) * esize;
      hi = lo + int64_t(count) * esize;
    }
    r.lo = lo / esize;
    r.hi = hi / esize;
    int64_t bytes = hi - lo;
    // a8: static chunk table.  Aim for >= `per_cta` chunks per CTA of the
    // channel (deeper trees pipeline better with more chunks: (c+h-1)/c,
    // P:511-513), chunks >= 16 KiB (BLINK_MIN_CHUNK) unless the range is
    // smaller, <= 4 MiB.
    int64_t cb;
    if (cfg.chunk_bytes > 0) {
      cb = int64_t(cfg.chunk_bytes);
    } else {
      // ~32 chunks per CTA (>= 16 KiB each): deeper trees pipeline
      // and dynamic chunk grabbing balances CTAs to the last
      // chunk (A/B in profiles/README.md; BLINK_CHUNKS_PER_CTA overrides)
      static const int per_cta_env = [] {
        const char* e = getenv("BLINK_CHUNKS_PER_CTA");
        return e ? std::max(1, atoi(e)) : 0;
      }();
      int per_cta = per_cta_env ? per_cta_env : 32;
      int64_t want = int64_t(std::max(1, ctas_hint)) * per_cta;
      cb = (bytes + want - 1) / want;
      static const int64_t min_chunk = [] {
        const char* e = getenv("BLINK_MIN_CHUNK");
        return e ? std::max<int64_t>(16, atoll(e)) : int64_t(16 << 10);
      }();
      // multi-hop trees signal every chunk (flags + a store drain): keep
      // their chunks larger, but a small tree needs enough chunks to
      // pipeline over its hops ((c+h-1)/c): the floor grows with
      // the tree's range, bytes/16 (Broadcast) or bytes/8 (AllReduce: twice
      // the signals per chunk) clamped to [16 KiB, cap] (A/B in
      // profiles/README.md; BLINK_MIN_CHUNK_DEEP fixes it)
      static const int64_t min_chunk_deep_env = [] {
        const char* e = getenv("BLINK_MIN_CHUNK_DEEP");
        return e ? std::max<int64_t>(16, atoll(e)) : int64_t(0);
      }();
      // cap of that floor: 96 KiB on link graphs, 64 KiB on the switch's
      // two-level Broadcast trees (A/B per call, 64 MiB: 3-GPU chains 69.6
      // -> 64.5 us, DGX-1V Broadcast 173.5 -> 159.5 us, DGX-1V AllReduce
      // 396 -> 358 us; switch Broadcast 2% slower with 96 KiB)
      static const int64_t deep_cap_env = [] {
        const char* e = getenv("BLINK_DEEP_CAP");
        return e ? std::max<int64_t>(16 << 10, atoll(e)) : int64_t(0);
      }();
      const int64_t deep_cap = deep_cap_env ? deep_cap_env : (p.switch_model ? (64 << 10) : (96 << 10));
      const int64_t min_chunk_deep =
          min_chunk_deep_env ? min_chunk_deep_env
                             : std::min<int64_t>(deep_cap, std::max<int64_t>(16 << 10,
                                                                             bytes / (p.coll == kBroadcast ? 16 : 8)));
      cb = std::max<int64_t>(cb, p.trees[i].depth >= 2 ? std::max(min_chunk, min_chunk_deep) : min_chunk);
      cb = std::min<int64_t>(cb, 4 << 20);
    }
    cb = (cb + kGrain - 1) / kGrain * kGrain;
    if (cb <= 0) cb = kGrain;
    int64_t nch = bytes > 0 ? (bytes + cb - 1) / cb : 0;
    if (nch > kMaxChunks) {
      cb = ((bytes + kMaxChunks - 1) / kMaxChunks + kGrain - 1) / kGrain * kGrain;
      nch = (bytes + cb - 1) / cb;
    }
    if (nch > kMaxChunks) {
      *err = "too many chunks";
      return BLINK_ERR_INTERNAL;
    }
    r.chunk = cb / esize;
    r.nchunks = int(nch);
    out->push_back(r);
  }
  return BLINK_SUCCESS;
}

std::string plan_to_json(const Plan& p, size_t count, int esize, const std::vector<TreeRange>& r,
                         int ctas) {
  std::ostringstream o;
  o.precision(17);
  static const char* names[] = {"broadcast", "allreduce", "reduce_scatter", "allgather", "gather"};
  o << "{\"coll\":\"" << names[p.coll] << "\",\"root\":"
    << p.root << ",\"nranks\":" << p.nranks << ",\"count\":" << count << ",\"esize\":" << esize
    << ",\"switch\":" << (p.switch_model ? "true" : "false") << ",\"rate\":[" << p.rate_num << ","
    << p.rate_den << "],\"c_star\":" << p.c_star << ",\"opt\":" << p.opt
    << ",\"accepted\":" << (p.accepted ? "true" : "false") << ",\"grid\":" << p.grid << ",\"ctas\":" << ctas
    << ",\"trees\":[";
  for (size_t i = 0; i < p.trees.size(); ++i) {
    const Tree& t = p.trees[i];
    o << (i ? "," : "") << "{\"root\":" << t.root << ",\"parent\":[";
    for (size_t v = 0; v < t.parent.size(); ++v) o << (v ? "," : "") << t.parent[v];
    o << "],\"weight\":[" << t.wnum << "," << t.wden << "],\"depth\":" << t.depth;
    if (i < r.size())
      o << ",\"lo\":" << r[i].lo << ",\"hi\":" << r[i].hi << ",\"chunk\":" << r[i].chunk
        << ",\"nchunks\":" << r[i].nchunks;
    o << "}";
  }
  o << "]}";
  return o.str();
}

}  // namespace blink

// Eq. 8 (Sec. 3.4): the PCIe / NVLink data split that makes
// T_PCIe + T_dpa = T_NVL; D_PCIe clamped to [0, D_total] (R#31), rounded
// down to the 16-byte grain (R#11).  Host-only planning: the hybrid data
// path is out of scope on B200 (PCIe Gen5 << NVLink 5, DESIGN 7).
extern "C" blink_result_t blink_hybrid_split(size_t d_total, double bw_pcie, double bw_nvl, double t_dpa,
                                             size_t* d_pcie, size_t* d_nvl) {
  if (!d_pcie || !d_nvl || !(bw_pcie > 0) || !(bw_nvl > 0) || !(t_dpa >= 0))
    return BLINK_ERR_INVALID_ARGUMENT;
  const double s = bw_pcie + bw_nvl;
  double x = double(d_total) * bw_pcie / s - t_dpa * bw_pcie * bw_nvl / s;
  if (!(x > 0)) x = 0;
  if (x > double(d_total)) x = double(d_total);
  size_t p = size_t(x);
  p = p / blink::kGrain * blink::kGrain;
  *d_pcie = p;
  *d_nvl = d_total - p;
  return BLINK_SUCCESS;
}
