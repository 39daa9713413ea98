// ORACLE / TEST INFRASTRUCTURE ONLY.  Restatement of Eigen's SimplicialLLT
// (up-looking simplicial LL^T after a fill-reducing symmetric permutation) as
// used by the reference coarse solver (coarse_solver.hpp:16-47).  Ordering is
// a generic graph nested dissection (BFS level-set separators) in place of
// Eigen's AMD; both are exact factorizations, so only roundoff differs.
#pragma once

#include <functional>
#include <numeric>

#include "shim_core.hpp"

namespace Eigen {
namespace shim {

// Nested-dissection order (new -> old) of the symmetric graph (ptr, idx).
inline std::vector<Index> nested_dissection(Index n, const std::vector<Index>& ptr,
                                            const std::vector<Index>& idx) {
  std::vector<Index> order;
  order.reserve((size_t)n);
  std::vector<int64_t> stamp((size_t)n, -1);
  std::vector<Index> level((size_t)n, -1);
  int64_t next_stamp = 0;
  const size_t leaf = 64;

  // BFS inside the stamped set; returns visit order, fills level[].
  auto bfs = [&](Index start, int64_t st, std::vector<Index>& visit) {
    visit.clear();
    visit.push_back(start);
    level[(size_t)start] = 0;
    stamp[(size_t)start] = st + 1;  // visited marker within this set
    for (size_t h = 0; h < visit.size(); ++h) {
      Index v = visit[h];
      for (Index p = ptr[(size_t)v]; p < ptr[(size_t)v + 1]; ++p) {
        Index w = idx[(size_t)p];
        if (stamp[(size_t)w] == st) {
          stamp[(size_t)w] = st + 1;
          level[(size_t)w] = level[(size_t)v] + 1;
          visit.push_back(w);
        }
      }
    }
  };

  std::function<void(std::vector<Index>&)> dissect = [&](std::vector<Index>& set) {
    if (set.size() <= leaf) {
      order.insert(order.end(), set.begin(), set.end());
      return;
    }
    int64_t st = next_stamp;
    next_stamp += 2;
    for (Index v : set) stamp[(size_t)v] = st;
    std::vector<Index> visit;
    bfs(set[0], st, visit);
    if (visit.size() < set.size()) {
      // Disconnected: split into the reached component and the remainder.
      std::vector<Index> rest;
      for (Index v : set)
        if (stamp[(size_t)v] == st) rest.push_back(v);
      std::vector<Index> comp(visit);
      dissect(comp);
      dissect(rest);
      return;
    }
    // Pseudo-peripheral start: restart from the farthest node a few times.
    Index far = visit.back();
    for (int rep = 0; rep < 2; ++rep) {
      for (Index v : set) stamp[(size_t)v] = st;
      bfs(far, st, visit);
      far = visit.back();
    }
    Index nlev = level[(size_t)visit.back()] + 1;
    if (nlev < 3) {
      order.insert(order.end(), set.begin(), set.end());
      return;
    }
    Index mid = nlev / 2;
    std::vector<Index> a, b, sep;
    for (Index v : visit) {
      Index l = level[(size_t)v];
      if (l < mid)
        a.push_back(v);
      else if (l > mid)
        b.push_back(v);
      else
        sep.push_back(v);
    }
    set.clear();
    set.shrink_to_fit();
    dissect(a);
    dissect(b);
    order.insert(order.end(), sep.begin(), sep.end());
  };

  std::vector<Index> all((size_t)n);
  std::iota(all.begin(), all.end(), Index(0));
  dissect(all);
  return order;
}

}  // namespace shim

template <class MatrixType>
class SimplicialLLT {
 public:
  void analyzePattern(const MatrixType& a) {
    n_ = a.cols();
    const auto& cp = a.col_ptr();
    const auto& ri = a.row_idx();
    // Symmetrized adjacency without the diagonal.
    std::vector<Index> deg((size_t)n_, 0);
    for (Index j = 0; j < n_; ++j)
      for (Index p = cp[(size_t)j]; p < cp[(size_t)j + 1]; ++p)
        if (ri[(size_t)p] != j) {
          ++deg[(size_t)j];
          ++deg[(size_t)ri[(size_t)p]];
        }
    std::vector<Index> ptr((size_t)n_ + 1, 0);
    for (Index j = 0; j < n_; ++j) ptr[(size_t)j + 1] = ptr[(size_t)j] + deg[(size_t)j];
    std::vector<Index> idx((size_t)ptr.back()), pos(ptr.begin(), ptr.end() - 1);
    for (Index j = 0; j < n_; ++j)
      for (Index p = cp[(size_t)j]; p < cp[(size_t)j + 1]; ++p) {
        Index i = ri[(size_t)p];
        if (i == j) continue;
        idx[(size_t)pos[(size_t)j]++] = i;
        idx[(size_t)pos[(size_t)i]++] = j;
      }
    perm_ = shim::nested_dissection(n_, ptr, idx);
    path_.assign((size_t)n_ + 1, 0);
    pinv_.assign((size_t)n_, 0);
    for (Index k = 0; k < n_; ++k) pinv_[(size_t)perm_[(size_t)k]] = k;

    // Upper triangle of P A P^T, column-compressed (pattern only here).
    build_upper(a, /*values=*/false);
    // Elimination tree.
    parent_.assign((size_t)n_, -1);
    std::vector<Index> ancestor((size_t)n_, -1);
    for (Index k = 0; k < n_; ++k)
      for (Index p = cptr_[(size_t)k]; p < cptr_[(size_t)k + 1]; ++p) {
        Index i = crow_[(size_t)p];
        while (i != -1 && i < k) {
          Index inext = ancestor[(size_t)i];
          ancestor[(size_t)i] = k;
          if (inext == -1) parent_[(size_t)i] = k;
          i = inext;
        }
      }
    // Column counts of L via row patterns (ereach).
    std::vector<Index> counts((size_t)n_, 1), stack((size_t)n_), mark((size_t)n_, -1);
    for (Index k = 0; k < n_; ++k) {
      Index top = ereach(k, stack, mark);
      for (Index t = top; t < n_; ++t) ++counts[(size_t)stack[(size_t)t]];
    }
    lptr_.assign((size_t)n_ + 1, 0);
    for (Index j = 0; j < n_; ++j) lptr_[(size_t)j + 1] = lptr_[(size_t)j] + counts[(size_t)j];
    lrow_.assign((size_t)lptr_.back(), 0);
    lval_.assign((size_t)lptr_.back(), 0.0);
    analyzed_ = true;
  }

  void factorize(const MatrixType& a) {
    if (!analyzed_) analyzePattern(a);
    build_upper(a, /*values=*/true);
    info_ = Success;
    std::vector<Index> next(lptr_.begin(), lptr_.end() - 1), stack((size_t)n_),
        mark((size_t)n_, -1);
    std::vector<double> x((size_t)n_, 0.0);
    for (Index k = 0; k < n_; ++k) {
      Index top = ereach(k, stack, mark);
      x[(size_t)k] = 0.0;
      for (Index p = cptr_[(size_t)k]; p < cptr_[(size_t)k + 1]; ++p)
        if (crow_[(size_t)p] <= k) x[(size_t)crow_[(size_t)p]] += cval_[(size_t)p];
      double d = x[(size_t)k];
      x[(size_t)k] = 0.0;
      for (; top < n_; ++top) {
        Index i = stack[(size_t)top];
        double lki = x[(size_t)i] / lval_[(size_t)lptr_[(size_t)i]];
        x[(size_t)i] = 0.0;
        for (Index p = lptr_[(size_t)i] + 1; p < next[(size_t)i]; ++p)
          x[(size_t)lrow_[(size_t)p]] -= lval_[(size_t)p] * lki;
        d -= lki * lki;
        Index p = next[(size_t)i]++;
        lrow_[(size_t)p] = k;
        lval_[(size_t)p] = lki;
      }
      if (!(d > 0.0)) {
        info_ = NumericalIssue;
        return;
      }
      Index p = next[(size_t)k]++;
      lrow_[(size_t)p] = k;
      lval_[(size_t)p] = std::sqrt(d);
    }
  }

  ComputationInfo info() const { return info_; }

  VectorXd solve(const Map<const VectorXd>& b) const {
    std::vector<double> y((size_t)n_);
    for (Index k = 0; k < n_; ++k) y[(size_t)k] = b(perm_[(size_t)k]);
    // L y = P b (column-oriented forward substitution).
    for (Index j = 0; j < n_; ++j) {
      y[(size_t)j] /= lval_[(size_t)lptr_[(size_t)j]];
      for (Index p = lptr_[(size_t)j] + 1; p < lptr_[(size_t)j + 1]; ++p)
        y[(size_t)lrow_[(size_t)p]] -= lval_[(size_t)p] * y[(size_t)j];
    }
    // L^T z = y.
    for (Index j = n_ - 1; j >= 0; --j) {
      for (Index p = lptr_[(size_t)j] + 1; p < lptr_[(size_t)j + 1]; ++p)
        y[(size_t)j] -= lval_[(size_t)p] * y[(size_t)lrow_[(size_t)p]];
      y[(size_t)j] /= lval_[(size_t)lptr_[(size_t)j]];
    }
    VectorXd x(n_);
    for (Index k = 0; k < n_; ++k) x(perm_[(size_t)k]) = y[(size_t)k];
    return x;
  }

 private:
  // Upper triangle (row <= col) of P A P^T in CSC.
  void build_upper(const MatrixType& a, bool values) {
    const auto& cp = a.col_ptr();
    const auto& ri = a.row_idx();
    const auto& va = a.vals();
    std::vector<Index> cnt((size_t)n_ + 1, 0);
    for (Index j = 0; j < n_; ++j)
      for (Index p = cp[(size_t)j]; p < cp[(size_t)j + 1]; ++p) {
        Index i2 = pinv_[(size_t)ri[(size_t)p]], j2 = pinv_[(size_t)j];
        if (i2 <= j2) ++cnt[(size_t)j2 + 1];
      }
    for (Index j = 0; j < n_; ++j) cnt[(size_t)j + 1] += cnt[(size_t)j];
    cptr_ = cnt;
    crow_.assign((size_t)cnt.back(), 0);
    if (values) cval_.assign((size_t)cnt.back(), 0.0);
    std::vector<Index> pos(cnt.begin(), cnt.end() - 1);
    for (Index j = 0; j < n_; ++j)
      for (Index p = cp[(size_t)j]; p < cp[(size_t)j + 1]; ++p) {
        Index i2 = pinv_[(size_t)ri[(size_t)p]], j2 = pinv_[(size_t)j];
        if (i2 > j2) continue;
        Index q = pos[(size_t)j2]++;
        crow_[(size_t)q] = i2;
        if (values) cval_[(size_t)q] = va[(size_t)p];
      }
  }

  // Nonzero pattern of row k of L in topological order: stack[top..n).
  Index ereach(Index k, std::vector<Index>& stack, std::vector<Index>& mark) const {
    Index top = n_;
    mark[(size_t)k] = k;
    for (Index p = cptr_[(size_t)k]; p < cptr_[(size_t)k + 1]; ++p) {
      Index i = crow_[(size_t)p];
      if (i > k) continue;
      Index len = 0;
      std::vector<Index>& s = stack;
      // Climb the etree until a marked node, recording the path.
      while (mark[(size_t)i] != k) {
        path_[(size_t)len++] = i;
        mark[(size_t)i] = k;
        i = parent_[(size_t)i];
      }
      while (len > 0) s[(size_t)--top] = path_[(size_t)--len];
    }
    return top;
  }

 public:
  SimplicialLLT() = default;

 private:
  Index n_ = 0;
  bool analyzed_ = false;
  ComputationInfo info_ = Success;
  std::vector<Index> perm_, pinv_, parent_, cptr_, crow_, lptr_, lrow_;
  std::vector<double> cval_, lval_;
  mutable std::vector<Index> path_;
};

}  // namespace Eigen
