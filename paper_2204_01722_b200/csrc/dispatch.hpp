// Runtime (p, q) -> compile-time (P, Q) dispatch over the supported pairs.
#pragma once

#include <type_traits>

#include "common.hpp"

namespace hxg {

template <int V>
using IC = std::integral_constant<int, V>;

// Calls f(IC<P>{}, IC<Q>{}) for the supported pair or throws.
template <class F>
void dispatch_pq(int p, int q, F&& f) {
  switch (p * 10 + q) {
    case 12: f(IC<1>{}, IC<2>{}); return;
    case 13: f(IC<1>{}, IC<3>{}); return;
    case 14: f(IC<1>{}, IC<4>{}); return;
    case 15: f(IC<1>{}, IC<5>{}); return;
    case 23: f(IC<2>{}, IC<3>{}); return;
    case 24: f(IC<2>{}, IC<4>{}); return;
    case 25: f(IC<2>{}, IC<5>{}); return;
    case 34: f(IC<3>{}, IC<4>{}); return;
    case 35: f(IC<3>{}, IC<5>{}); return;
    case 45: f(IC<4>{}, IC<5>{}); return;
    default:
      throw Error(HXG_ERR_UNSUPPORTED, "unsupported (order, quadrature) pair (" +
                                           std::to_string(p) + ", " + std::to_string(q) +
                                           "); supported: p in 1..4, q in p+1..5");
  }
}

template <class F>
void dispatch_p(int p, F&& f) {
  switch (p) {
    case 1: f(IC<1>{}); return;
    case 2: f(IC<2>{}); return;
    case 3: f(IC<3>{}); return;
    case 4: f(IC<4>{}); return;
    default:
      throw Error(HXG_ERR_UNSUPPORTED, "unsupported order " + std::to_string(p));
  }
}

template <class F>
void dispatch_q(int q, F&& f) {
  switch (q) {
    case 2: f(IC<2>{}); return;
    case 3: f(IC<3>{}); return;
    case 4: f(IC<4>{}); return;
    case 5: f(IC<5>{}); return;
    default:
      throw Error(HXG_ERR_UNSUPPORTED, "unsupported quadrature size " + std::to_string(q));
  }
}

inline int grid_for(long long work, int block, int max_blocks = 148 * 16) {
  long long g = (work + block - 1) / block;
  if (g > max_blocks) g = max_blocks;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace hxg
