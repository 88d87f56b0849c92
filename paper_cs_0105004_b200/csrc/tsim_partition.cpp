// tsim_partition.cpp -- multilevel k-way graph partitioning of the road
// network (the paper uses METIS, a
// multilevel partitioner, and compares it with ORB).  Host code, no device.
//
// Graph: one vertex per node (weight = its load, e.g. half of the attached
// links' cells x lanes); one edge per undirected node pair
// joined by links, weight = lanes of those links (every lane of a split link
// is one strip per exchange, so the edge weight is the communication
// volume a cut there costs).
//
// 1. Coarsening: heavy-edge matching in a seeded random vertex order, then
//    contraction, until the graph has <= max(20 k, 64) vertices or stops
//    shrinking.
// 2. Initial partition: orthogonal recursive bisection of the coarsest
//    vertices (weighted centroids), the method of PAPER.md:568-583.
// 3. Uncoarsening with refinement: at every level, passes over the boundary
//    vertices moving each to the neighbouring domain with the largest
//    positive cut gain (or zero gain and better balance) while every domain
//    stays within (1 + eps) of the average load (greedy Fiduccia-Mattheyses
//    style, no negative-gain moves).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <unordered_map>
#include <vector>

#include "../../include/tsim.h"

namespace {

struct Graph {
  int n = 0;
  std::vector<double> vw;         // vertex weights
  std::vector<double> cx, cy;     // weighted coordinates (for ORB)
  std::vector<int64_t> off;       // CSR
  std::vector<int32_t> adj;
  std::vector<double> ew;
};

// splitmix64: seeded permutation source
uint64_t mix(uint64_t &s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

Graph build_graph(int32_t n_nodes, const int64_t *x, const int64_t *y, int32_t n_links,
                  const int32_t *from, const int32_t *to, const int32_t *lanes,
                  const double *node_weight) {
  Graph g;
  g.n = n_nodes;
  g.vw.assign(n_nodes, 1.0);
  if (node_weight)
    for (int i = 0; i < n_nodes; i++) g.vw[i] = std::max(1e-9, node_weight[i]);
  g.cx.resize(n_nodes);
  g.cy.resize(n_nodes);
  for (int i = 0; i < n_nodes; i++) {
    g.cx[i] = (double)x[i];
    g.cy[i] = (double)y[i];
  }
  std::vector<std::unordered_map<int32_t, double>> nb(n_nodes);
  for (int j = 0; j < n_links; j++) {
    const int a = from[j], b = to[j];
    if (a == b) continue;
    const double w = lanes ? std::max(1, lanes[j]) : 1;
    nb[a][b] += w;
    nb[b][a] += w;
  }
  g.off.assign(n_nodes + 1, 0);
  for (int i = 0; i < n_nodes; i++) g.off[i + 1] = g.off[i] + (int64_t)nb[i].size();
  g.adj.resize(g.off[n_nodes]);
  g.ew.resize(g.off[n_nodes]);
  for (int i = 0; i < n_nodes; i++) {
    std::vector<std::pair<int32_t, double>> e(nb[i].begin(), nb[i].end());
    std::sort(e.begin(), e.end());
    int64_t p = g.off[i];
    for (auto &q : e) {
      g.adj[p] = q.first;
      g.ew[p++] = q.second;
    }
  }
  return g;
}

// heavy-edge matching + contraction; cmap[v] = coarse vertex of v
Graph coarsen(const Graph &g, std::vector<int32_t> &cmap, uint64_t &seed) {
  std::vector<int32_t> order(g.n), match(g.n, -1);
  std::iota(order.begin(), order.end(), 0);
  for (int i = g.n - 1; i > 0; i--) std::swap(order[i], order[mix(seed) % (uint64_t)(i + 1)]);
  const double wmax = 1.5 * std::accumulate(g.vw.begin(), g.vw.end(), 0.0) / std::max(1, g.n / 2);
  for (int v : order) {
    if (match[v] >= 0) continue;
    int best = -1;
    double bw = -1;
    for (int64_t p = g.off[v]; p < g.off[v + 1]; p++) {
      const int u = g.adj[p];
      if (match[u] >= 0 || g.vw[u] + g.vw[v] > wmax) continue;
      if (g.ew[p] > bw) {
        bw = g.ew[p];
        best = u;
      }
    }
    match[v] = best >= 0 ? best : v;
    if (best >= 0) match[best] = v;
  }
  cmap.assign(g.n, -1);
  int nc = 0;
  for (int v = 0; v < g.n; v++) {
    if (cmap[v] >= 0) continue;
    cmap[v] = nc;
    if (match[v] != v) cmap[match[v]] = nc;
    nc++;
  }
  Graph c;
  c.n = nc;
  c.vw.assign(nc, 0.0);
  c.cx.assign(nc, 0.0);
  c.cy.assign(nc, 0.0);
  for (int v = 0; v < g.n; v++) {
    c.vw[cmap[v]] += g.vw[v];
    c.cx[cmap[v]] += g.vw[v] * g.cx[v];
    c.cy[cmap[v]] += g.vw[v] * g.cy[v];
  }
  for (int i = 0; i < nc; i++) {
    c.cx[i] /= c.vw[i];
    c.cy[i] /= c.vw[i];
  }
  std::vector<std::unordered_map<int32_t, double>> nb(nc);
  for (int v = 0; v < g.n; v++)
    for (int64_t p = g.off[v]; p < g.off[v + 1]; p++) {
      const int a = cmap[v], b = cmap[g.adj[p]];
      if (a != b) nb[a][b] += g.ew[p];
    }
  c.off.assign(nc + 1, 0);
  for (int i = 0; i < nc; i++) c.off[i + 1] = c.off[i] + (int64_t)nb[i].size();
  c.adj.resize(c.off[nc]);
  c.ew.resize(c.off[nc]);
  for (int i = 0; i < nc; i++) {
    std::vector<std::pair<int32_t, double>> e(nb[i].begin(), nb[i].end());
    std::sort(e.begin(), e.end());
    int64_t p = c.off[i];
    for (auto &q : e) {
      c.adj[p] = q.first;
      c.ew[p++] = q.second;
    }
  }
  return c;
}

// ORB on weighted centroids
void orb(const Graph &g, std::vector<int32_t> &idx, size_t lo, size_t hi, int k, int d0, bool vert,
         std::vector<int32_t> &part) {
  if (k == 1) {
    for (size_t i = lo; i < hi; i++) part[idx[i]] = d0;
    return;
  }
  const std::vector<double> &c = vert ? g.cx : g.cy;
  std::stable_sort(idx.begin() + lo, idx.begin() + hi,
                   [&](int a, int b) { return c[a] < c[b] || (c[a] == c[b] && a < b); });
  const int kl = (k + 1) / 2, kr = k - kl;
  double tot = 0;
  for (size_t i = lo; i < hi; i++) tot += g.vw[idx[i]];
  const double target = tot * kl / k;
  double acc = 0, best = 1e300;
  size_t cut = lo + (size_t)kl;
  for (size_t i = lo; i < hi; i++) {
    acc += g.vw[idx[i]];
    const size_t c1 = i + 1;
    if (c1 - lo < (size_t)kl || hi - c1 < (size_t)kr) continue;
    if (std::fabs(acc - target) < best) {
      best = std::fabs(acc - target);
      cut = c1;
    }
  }
  orb(g, idx, lo, cut, kl, d0, !vert, part);
  orb(g, idx, cut, hi, kr, d0 + kl, !vert, part);
}

// greedy boundary refinement under the balance bound
void refine(const Graph &g, int k, double eps, std::vector<int32_t> &part, int passes) {
  std::vector<double> load(k, 0.0);
  for (int v = 0; v < g.n; v++) load[part[v]] += g.vw[v];
  const double tot = std::accumulate(load.begin(), load.end(), 0.0);
  const double cap = (1.0 + eps) * tot / k;
  std::vector<double> conn(k, 0.0);
  std::vector<int> touched;
  for (int pass = 0; pass < passes; pass++) {
    int moves = 0;
    for (int v = 0; v < g.n; v++) {
      const int a = part[v];
      touched.clear();
      bool boundary = false;
      for (int64_t p = g.off[v]; p < g.off[v + 1]; p++) {
        const int b = part[g.adj[p]];
        if (conn[b] == 0.0) touched.push_back(b);
        conn[b] += g.ew[p];
        boundary |= b != a;
      }
      if (boundary) {
        int best = a;
        double bgain = 0.0;
        for (int b : touched) {
          if (b == a || load[b] + g.vw[v] > cap) continue;
          const double gain = conn[b] - conn[a];
          const bool better_balance = gain == 0.0 && load[b] + g.vw[v] < load[a];
          // never empty a domain
          if (load[a] - g.vw[v] <= 0.0) continue;
          if (gain > bgain || (gain == bgain && best == a && better_balance)) {
            bgain = gain;
            best = b;
          }
        }
        if (best != a) {
          load[a] -= g.vw[v];
          load[best] += g.vw[v];
          part[v] = best;
          moves++;
        }
      }
      for (int b : touched) conn[b] = 0.0;
    }
    if (!moves) break;
  }
}

}  // namespace

extern "C" int ts_multilevel_partition(int32_t n_nodes, const int64_t *node_x_mm,
                                       const int64_t *node_y_mm, int32_t n_links,
                                       const int32_t *from, const int32_t *to,
                                       const int32_t *lanes, const double *node_weight, int32_t k,
                                       double imbalance, uint64_t seed, int32_t *domain_of_node) {
  if (n_nodes < 1 || k < 1 || k > n_nodes || !node_x_mm || !node_y_mm || !domain_of_node ||
      imbalance < 0.0)
    return TS_EINVAL;
  for (int j = 0; j < n_links; j++)
    if (from[j] < 0 || from[j] >= n_nodes || to[j] < 0 || to[j] >= n_nodes) return TS_EINVAL;
  std::vector<Graph> levels;
  std::vector<std::vector<int32_t>> maps;
  levels.push_back(build_graph(n_nodes, node_x_mm, node_y_mm, n_links, from, to, lanes, node_weight));
  uint64_t s = seed;
  const int target = std::max(20 * k, 64);
  while (levels.back().n > target) {
    std::vector<int32_t> cmap;
    Graph c = coarsen(levels.back(), cmap, s);
    if (c.n > 0.95 * levels.back().n) break;  // no longer shrinking
    maps.push_back(std::move(cmap));
    levels.push_back(std::move(c));
  }
  const Graph &cg = levels.back();
  std::vector<int32_t> part(cg.n, 0), idx(cg.n);
  std::iota(idx.begin(), idx.end(), 0);
  orb(cg, idx, 0, cg.n, k, 0, true, part);
  refine(cg, k, imbalance, part, 8);
  for (int lv = (int)levels.size() - 2; lv >= 0; lv--) {
    const std::vector<int32_t> &cm = maps[lv];
    std::vector<int32_t> fine(levels[lv].n);
    for (int v = 0; v < levels[lv].n; v++) fine[v] = part[cm[v]];
    part.swap(fine);
    refine(levels[lv], k, imbalance, part, 8);
  }
  for (int i = 0; i < n_nodes; i++) domain_of_node[i] = part[i];
  return TS_OK;
}

// ------------------------------------------------- adaptive load balancing
// PAPER.md:726-735 (§7): "we collect the execution time of each link and
// each intersection (node)" during a run and feed it to the partitioner.
// Here a domain's measured device time over a window (ts_busy_time) is
// apportioned to its links and nodes in proportion to their work counts
// over the same window (ts_get_load: vehicle updates per link, lanes in
// range + crossings per node; one unit of either counts alike).
extern "C" int ts_load_times(double domain_ms, int32_t n_links, const int64_t *link_work,
                             int32_t n_nodes, const int64_t *node_work, double *link_time,
                             double *node_time) {
  if (n_links < 0 || n_nodes < 0 || !(domain_ms >= 0.0)) return TS_EINVAL;
  if ((n_links && (!link_work || !link_time)) || (n_nodes && node_work && !node_time))
    return TS_EINVAL;
  double tot = 0.0;
  for (int32_t j = 0; j < n_links; j++) {
    if (link_work[j] < 0) return TS_EINVAL;
    tot += (double)link_work[j];
  }
  if (node_work)
    for (int32_t i = 0; i < n_nodes; i++) {
      if (node_work[i] < 0) return TS_EINVAL;
      tot += (double)node_work[i];
    }
  if (tot <= 0.0) return TS_OK;  // an idle domain: no time to apportion
  const double per = domain_ms / tot;
  for (int32_t j = 0; j < n_links; j++) link_time[j] += per * (double)link_work[j];
  if (node_work)
    for (int32_t i = 0; i < n_nodes; i++) node_time[i] += per * (double)node_work[i];
  return TS_OK;
}

// Node weights for the next partition from the per-link and per-node times
// (node weight = its own time + half of every attached
// link's time; links without measured work keep a floor of 1e-3 of their
// static share cells x lanes, so empty regions still count), then a new
// k-way partition: method 0 = ORB, 1 = multilevel
// (PAPER.md:585-636).
extern "C" int ts_orb_partition(int32_t n_nodes, const int64_t *node_x_mm, const int64_t *node_y_mm,
                                const double *node_weight, int32_t k, int32_t *domain_of_node);

extern "C" int ts_rebalance(int32_t n_nodes, const int64_t *node_x_mm, const int64_t *node_y_mm,
                            int32_t n_links, const int32_t *from, const int32_t *to,
                            const int32_t *lanes, const int64_t *length_mm,
                            const double *link_time, const double *node_time, int32_t k,
                            int32_t method, double imbalance, uint64_t seed,
                            double *node_weight_out, int32_t *domain_of_node_out) {
  if (n_nodes < 1 || n_links < 0 || k < 1 || k > n_nodes || !node_x_mm || !node_y_mm ||
      !link_time || !domain_of_node_out || (method != 0 && method != 1))
    return TS_EINVAL;
  double lsum = 0.0, ssum = 0.0;
  std::vector<double> stat(n_links);
  for (int32_t j = 0; j < n_links; j++) {
    if (from[j] < 0 || from[j] >= n_nodes || to[j] < 0 || to[j] >= n_nodes || length_mm[j] <= 0 ||
        !(link_time[j] >= 0.0))
      return TS_EINVAL;
    const int64_t cells = std::max<int64_t>(1, (length_mm[j] + 3750) / 7500);  // R1
    stat[j] = (double)cells * lanes[j];
    ssum += stat[j];
    lsum += link_time[j];
  }
  const double fl = ssum > 0.0 ? 1e-3 * std::max(lsum, 1e-12) / ssum : 0.0;
  std::vector<double> w(n_nodes, 1e-9);
  if (node_time)
    for (int32_t i = 0; i < n_nodes; i++) w[i] += std::max(0.0, node_time[i]);
  for (int32_t j = 0; j < n_links; j++) {
    const double lt = link_time[j] + fl * stat[j];
    w[from[j]] += 0.5 * lt;
    w[to[j]] += 0.5 * lt;
  }
  if (node_weight_out) std::copy(w.begin(), w.end(), node_weight_out);
  if (method == 0)
    return ts_orb_partition(n_nodes, node_x_mm, node_y_mm, w.data(), k, domain_of_node_out);
  return ts_multilevel_partition(n_nodes, node_x_mm, node_y_mm, n_links, from, to, lanes, w.data(),
                                 k, imbalance, seed, domain_of_node_out);
}
