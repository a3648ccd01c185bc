// Canonical labeling by individualization-refinement.
//
// The labeling must be IDENTICAL to the reference's (proj/src/graph_canon.cpp)
// for every graph, because it fixes the canonical form and every sigma map.
// The decisions that determine it are reproduced exactly:
//   * initial cells: one per colour value, ascending, members in node order
//     (graph_canon.cpp:219-224);
//   * refinement is simultaneous: each round splits every cell by the counts of
//     out-neighbours per cell followed by in-neighbours per cell, computed from
//     one snapshot of the partition; subcells ordered by DESCENDING signature,
//     members keep their order; repeat until stable (:82-114);
//   * branch on the first cell of maximum size > 1, trying its members in order,
//     the chosen node becoming a singleton cell in front of the rest (:151-208);
//   * leaf certificate = row-major adjacency bits of the relabeled graph, MSB
//     first in 64-bit words, compared lexicographically; the FIRST leaf with the
//     minimum certificate wins (:116-137).
// Orbit pruning by automorphisms found at equal leaves (:138-189) only skips
// subtrees that are images of already-explored ones, so it never changes which
// leaf is the first minimum; it is kept because it bounds the search.
//
// Data structures differ from the reference: partitions are flat (node order +
// cell starts), signatures are sparse (cell, count) runs compared with the
// dense-vector order, certificates are built from adjacency lists in O(E).
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <utility>
#include <vector>

#include "feinsum/core.hpp"
#include "feinsum/graph_canon.hpp"

namespace feinsum {

ColoredDigraph ColoredDigraph::empty(int n_nodes) {
  ColoredDigraph g;
  g.n = n_nodes;
  g.adj.assign(static_cast<size_t>(n_nodes) * static_cast<size_t>(n_nodes), 0);
  g.colors.assign(static_cast<size_t>(n_nodes), 1);
  return g;
}

std::vector<int> Relabeling::inverse() const {
  std::vector<int> inv(perm.size());
  for (size_t v = 0; v < perm.size(); ++v) inv[static_cast<size_t>(perm[v])] = static_cast<int>(v);
  return inv;
}

ColoredDigraph apply_relabeling(const ColoredDigraph& g, const Relabeling& r) {
  if (static_cast<int>(r.perm.size()) != g.n)
    throw error(errc::domain, "relabeling size does not match graph");
  ColoredDigraph h = ColoredDigraph::empty(g.n);
  for (int i = 0; i < g.n; ++i) {
    h.colors[r.perm[i]] = g.colors[i];
    const std::uint8_t* row = &g.adj[static_cast<size_t>(i) * g.n];
    for (int j = 0; j < g.n; ++j)
      if (row[j]) h.set_edge(r.perm[i], r.perm[j]);
  }
  return h;
}

namespace {

// Ordered partition: cells are contiguous ranges of `order`.
struct Partition {
  std::vector<int> order;   // nodes, cell by cell
  std::vector<int> starts;  // start offset of each cell; size = #cells
  int cells() const { return static_cast<int>(starts.size()); }
  int begin(int c) const { return starts[c]; }
  int end(int c) const {
    return c + 1 < cells() ? starts[c + 1] : static_cast<int>(order.size());
  }
  int size(int c) const { return end(c) - begin(c); }
};

class UnionFind {
 public:
  explicit UnionFind(int n) : parent_(static_cast<size_t>(n)) {
    std::iota(parent_.begin(), parent_.end(), 0);
  }
  int root(int x) {
    while (parent_[x] != x) {
      parent_[x] = parent_[parent_[x]];
      x = parent_[x];
    }
    return x;
  }
  void join(int a, int b) { parent_[root(a)] = root(b); }

 private:
  std::vector<int> parent_;
};

// Sparse signature: (position, count) runs over the virtual dense vector
// [out-counts per cell | in-counts per cell]; positions strictly increasing.
using Sig = std::vector<std::pair<int, int>>;

// Lexicographic order of the dense vectors the runs stand for.
bool sig_less(const Sig& a, const Sig& b) {
  size_t i = 0;
  for (; i < a.size() && i < b.size(); ++i) {
    if (a[i].first != b[i].first) return a[i].first > b[i].first;  // b nonzero first
    if (a[i].second != b[i].second) return a[i].second < b[i].second;
  }
  return a.size() < b.size();
}

class IRSearch {
 public:
  explicit IRSearch(const ColoredDigraph& g) : n_(g.n), out_(g.n), in_(g.n), cell_of_(g.n) {
    for (int i = 0; i < n_; ++i) {
      const std::uint8_t* row = &g.adj[static_cast<size_t>(i) * n_];
      for (int j = 0; j < n_; ++j)
        if (row[j]) {
          out_[i].push_back(j);
          in_[j].push_back(i);
        }
    }
    words_ = (static_cast<size_t>(n_) * n_ + 63) / 64;
  }

  // adds a candidate automorphism after checking it on the adjacency lists
  bool seed(const ColoredDigraph& g, const std::vector<int>& a) {
    if (static_cast<int>(a.size()) != n_) return false;
    std::vector<char> hit(static_cast<size_t>(n_), 0);
    bool identity = true;
    for (int v = 0; v < n_; ++v) {
      const int w = a[v];
      if (w < 0 || w >= n_ || hit[w] || g.colors[w] != g.colors[v]) return false;
      hit[w] = 1;
      identity = identity && w == v;
    }
    if (identity) return false;
    std::size_t edges = 0;
    for (int v = 0; v < n_; ++v) {
      const std::uint8_t* row = &g.adj[static_cast<size_t>(a[v]) * n_];
      for (int u : out_[v]) {
        if (!row[a[u]]) return false;
        ++edges;
      }
    }
    (void)edges;  // a bijection mapping every edge onto an edge preserves the edge set
    autos_.push_back(a);
    return true;
  }

  std::vector<int> run(const ColoredDigraph& g) {
    // initial partition by colour value, ascending
    std::vector<int> nodes(static_cast<size_t>(n_));
    std::iota(nodes.begin(), nodes.end(), 0);
    std::stable_sort(nodes.begin(), nodes.end(),
                     [&](int a, int b) { return g.colors[a] < g.colors[b]; });
    Partition p;
    p.order = nodes;
    for (int i = 0; i < n_; ++i)
      if (i == 0 || g.colors[nodes[i]] != g.colors[nodes[i - 1]]) p.starts.push_back(i);
    descend(std::move(p));
    return best_label_;
  }

 private:
  int n_;
  size_t words_;
  std::vector<std::vector<int>> out_, in_;
  std::vector<int> cell_of_;

  bool have_best_ = false;
  std::vector<std::uint64_t> best_cert_;
  std::vector<int> best_label_;
  std::vector<std::vector<int>> autos_;
  std::vector<int> path_;

  void signature(int v, int k, Sig& s) {
    // counts per cell, out then in, as sorted runs
    s.clear();
    for (int u : out_[v]) s.emplace_back(cell_of_[u], 1);
    for (int u : in_[v]) s.emplace_back(k + cell_of_[u], 1);
    std::sort(s.begin(), s.end());
    size_t w = 0;
    for (size_t r = 0; r < s.size(); ++r) {
      if (w > 0 && s[w - 1].first == s[r].first)
        ++s[w - 1].second;
      else
        s[w++] = s[r];
    }
    s.resize(w);
  }

  void refine(Partition& p) {
    std::vector<Sig> sig;
    std::vector<int> idx;
    for (;;) {
      const int k = p.cells();
      for (int c = 0; c < k; ++c)
        for (int t = p.begin(c); t < p.end(c); ++t) cell_of_[p.order[t]] = c;

      Partition q;
      q.order.reserve(p.order.size());
      q.starts.reserve(static_cast<size_t>(k) + 4);
      bool split = false;
      for (int c = 0; c < k; ++c) {
        const int b = p.begin(c), e = p.end(c), m = e - b;
        if (m == 1) {
          q.starts.push_back(static_cast<int>(q.order.size()));
          q.order.push_back(p.order[b]);
          continue;
        }
        sig.resize(static_cast<size_t>(m));
        idx.resize(static_cast<size_t>(m));
        for (int t = 0; t < m; ++t) {
          signature(p.order[b + t], k, sig[t]);
          idx[t] = t;
        }
        // descending signature, members in original order within a group
        std::stable_sort(idx.begin(), idx.end(),
                         [&](int x, int y) { return sig_less(sig[y], sig[x]); });
        for (int t = 0; t < m; ++t) {
          if (t == 0 || sig[idx[t]] != sig[idx[t - 1]]) {
            if (t > 0) split = true;
            q.starts.push_back(static_cast<int>(q.order.size()));
          }
          q.order.push_back(p.order[b + idx[t]]);
        }
      }
      p = std::move(q);
      if (!split) return;
    }
  }

  std::vector<std::uint64_t> certificate(const std::vector<int>& label) const {
    std::vector<std::uint64_t> cert(words_, 0);
    for (int u = 0; u < n_; ++u) {
      const size_t rowbase = static_cast<size_t>(label[u]) * n_;
      for (int w : out_[u]) {
        const size_t bit = rowbase + static_cast<size_t>(label[w]);
        cert[bit >> 6] |= std::uint64_t{1} << (63 - (bit & 63));
      }
    }
    return cert;
  }

  void at_leaf(const Partition& p) {
    std::vector<int> label(static_cast<size_t>(n_));
    for (int c = 0; c < p.cells(); ++c) label[p.order[p.begin(c)]] = c;
    std::vector<std::uint64_t> cert = certificate(label);
    if (!have_best_ || cert < best_cert_) {
      have_best_ = true;
      best_cert_ = std::move(cert);
      best_label_ = std::move(label);
      return;
    }
    if (cert != best_cert_) return;
    // equal leaves differ by an automorphism: v -> best^-1(label(v))
    std::vector<int> best_inv(static_cast<size_t>(n_));
    for (int v = 0; v < n_; ++v) best_inv[best_label_[v]] = v;
    std::vector<int> gamma(static_cast<size_t>(n_));
    bool identity = true;
    for (int v = 0; v < n_; ++v) {
      gamma[v] = best_inv[label[v]];
      identity = identity && gamma[v] == v;
    }
    if (!identity) autos_.push_back(std::move(gamma));
  }

  void descend(Partition p) {
    refine(p);
    int target = -1, widest = 1;
    for (int c = 0; c < p.cells(); ++c)
      if (p.size(c) > widest) {
        widest = p.size(c);
        target = c;
      }
    if (target < 0) {
      at_leaf(p);
      return;
    }

    const int tb = p.begin(target), te = p.end(target);
    const std::vector<int> members(p.order.begin() + tb, p.order.begin() + te);
    std::vector<int> tried;
    size_t absorbed = 0;
    UnionFind orbit(n_);
    for (int v : members) {
      if (!tried.empty()) {
        for (; absorbed < autos_.size(); ++absorbed) {
          const std::vector<int>& a = autos_[absorbed];
          bool fixes = true;
          for (int w : path_)
            if (a[w] != w) {
              fixes = false;
              break;
            }
          if (fixes)
            for (int x = 0; x < n_; ++x) orbit.join(x, a[x]);
        }
        const int rv = orbit.root(v);
        bool same = false;
        for (int u : tried)
          if (orbit.root(u) == rv) {
            same = true;
            break;
          }
        if (same) continue;
      }
      tried.push_back(v);

      // child: target cell -> {v} followed by the remaining members
      Partition child;
      child.order = p.order;
      child.order[tb] = v;
      int w = tb + 1;
      for (int x : members)
        if (x != v) child.order[w++] = x;
      child.starts.reserve(p.starts.size() + 1);
      for (int c = 0; c < p.cells(); ++c) {
        child.starts.push_back(p.starts[c]);
        if (c == target) child.starts.push_back(tb + 1);
      }
      path_.push_back(v);
      descend(std::move(child));
      path_.pop_back();
    }
  }
};

}  // namespace

Relabeling canonical_labeling(const ColoredDigraph& g) { return canonical_labeling(g, {}); }

Relabeling canonical_labeling(const ColoredDigraph& g, const std::vector<std::vector<int>>& known_automorphisms) {
  if (g.n == 0) return Relabeling{{}};
  if (static_cast<int>(g.colors.size()) != g.n ||
      g.adj.size() != static_cast<size_t>(g.n) * static_cast<size_t>(g.n))
    throw error(errc::domain, "malformed colored digraph");
  IRSearch s(g);
  for (const auto& a : known_automorphisms) s.seed(g, a);
  return Relabeling{s.run(g)};
}

}  // namespace feinsum
