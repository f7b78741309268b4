// refelem.cpp -- LGL nodes, weights and differentiation matrix in 64-bit.
// Same numerical recipe as the reference (core/src/reference_element.cpp:
// 11-138: three-term Legendre recurrence, safeguarded Newton on
// (1-x^2) P_N'(x) bracketed by Chebyshev-Lobatto midpoints, x >= 0 half
// mirrored, barycentric D with the diagonal as negative row sum) so the
// operators the GPU consumes equal the reference's to the last bit
// (tests/test_host_mirror.py checks it against oracle/_ref).
#include <cmath>
#include <limits>

#include "host_types.hpp"

namespace esdg_b200 {
namespace host {

namespace {

struct PN {
  double value, deriv;
};

PN legendre_pn(int n, double x) {
  if (n == 0) return {1.0, 0.0};
  double prev = 1.0, cur = x;
  for (int k = 2; k <= n; ++k) {
    const double next = ((2.0 * k - 1.0) * x * cur - (k - 1.0) * prev) / k;
    prev = cur;
    cur = next;
  }
  double deriv;
  if (std::abs(x) == 1.0) {
    const double edge = n * (n + 1) / 2.0;
    deriv = (x == 1.0) ? edge : ((n % 2 == 0) ? -1.0 : 1.0) * edge;
  } else {
    deriv = n * (x * cur - prev) / (x * x - 1.0);
  }
  return {cur, deriv};
}

double lobatto_q(int n, double x) { return (1.0 - x * x) * legendre_pn(n, x).deriv; }

bool interior_node(int n, double a, double b, double& x_out) {
  double qa = lobatto_q(n, a), qb = lobatto_q(n, b);
  for (int widen = 0; widen < 8 && ((qa > 0) == (qb > 0)); ++widen) {
    const double w = 0.25 * (b - a);
    a = std::max(a - w, -1.0 + 1e-14);
    b = std::min(b + w, 1.0 - 1e-14);
    qa = lobatto_q(n, a);
    qb = lobatto_q(n, b);
  }
  if ((qa > 0) == (qb > 0)) return false;
  double x = 0.5 * (a + b);
  for (int it = 0; it < 200; ++it) {
    const double qx = lobatto_q(n, x);
    if (qx == 0.0) break;
    if ((qx > 0) == (qa > 0)) {
      a = x;
      qa = qx;
    } else {
      b = x;
    }
    // q'(x) = -N (N+1) P_N(x)
    const double slope = -double(n) * (n + 1) * legendre_pn(n, x).value;
    double next = (slope != 0.0) ? x - qx / slope : x;
    if (!(next > a && next < b)) next = 0.5 * (a + b);
    if (next == x) break;
    x = next;
    if (b - a <= 2.0 * std::abs(x) * std::numeric_limits<double>::epsilon()) break;
  }
  x_out = x;
  return true;
}

} // namespace

bool RefElement::build(int order, RefElement& r) {
  if (order < 1 || order > 32) return false;
  const int nq = order + 1;
  r.order = order;
  r.nq = nq;
  r.nodes.assign(size_t(nq), 0.0);
  r.weights.assign(size_t(nq), 0.0);
  r.nodes.front() = -1.0;
  r.nodes.back() = 1.0;
  std::vector<double> cgl(static_cast<size_t>(nq));
  for (int i = 0; i < nq; ++i) cgl[size_t(i)] = -std::cos(M_PI * i / order);
  const int first = nq / 2 + nq % 2;
  for (int i = first; i < nq - 1; ++i) {
    double a = 0.5 * (cgl[size_t(i) - 1] + cgl[size_t(i)]);
    const double b = 0.5 * (cgl[size_t(i)] + cgl[size_t(i) + 1]);
    if (i == first && nq % 2 == 0) a = 0.0;
    double x;
    if (!interior_node(order, a, b, x)) return false;
    r.nodes[size_t(i)] = x;
    r.nodes[size_t(nq - 1 - i)] = -x;
  }
  if (nq % 2 == 1) r.nodes[size_t(nq / 2)] = 0.0;

  const double wf = 2.0 / (double(order) * (order + 1));
  for (int i = (nq + 1) / 2; i < nq; ++i) {
    const double p = legendre_pn(order, r.nodes[size_t(i)]).value;
    r.weights[size_t(i)] = wf / (p * p);
    r.weights[size_t(nq - 1 - i)] = r.weights[size_t(i)];
  }
  if (nq % 2 == 1) {
    const double p = legendre_pn(order, 0.0).value;
    r.weights[size_t(nq / 2)] = wf / (p * p);
  }

  // barycentric differentiation matrix, diagonal = -(row sum)
  std::vector<double> bary(static_cast<size_t>(nq), 1.0);
  for (int i = 0; i < nq; ++i)
    for (int j = 0; j < nq; ++j)
      if (j != i) bary[size_t(i)] /= (r.nodes[size_t(i)] - r.nodes[size_t(j)]);
  r.diff.assign(size_t(nq) * size_t(nq), 0.0);
  for (int i = 0; i < nq; ++i) {
    double sum = 0.0;
    for (int j = 0; j < nq; ++j) {
      if (j == i) continue;
      const double dij = (bary[size_t(j)] / bary[size_t(i)]) /
                         (r.nodes[size_t(i)] - r.nodes[size_t(j)]);
      r.diff[size_t(i) * size_t(nq) + size_t(j)] = dij;
      sum += dij;
    }
    r.diff[size_t(i) * size_t(nq) + size_t(i)] = -sum;
  }
  return true;
}

void lsrk_coefficients(double a[5], double b[5], double c[5]) {
  // Carpenter-Kennedy LSRK(5,4), 2N storage (time_integration.hpp:17-37)
  static const double A[5] = {0.0, -567301805773.0 / 1357537059087.0,
                              -2404267990393.0 / 2016746695238.0,
                              -3550918686646.0 / 2091501179385.0,
                              -1275806237668.0 / 842570457699.0};
  static const double B[5] = {1432997174477.0 / 9575080441755.0,
                              5161836677717.0 / 13612068292357.0,
                              1720146321549.0 / 2090206949498.0,
                              3134564353537.0 / 4481467310338.0,
                              2277821191437.0 / 14882151754819.0};
  static const double C[5] = {0.0, 1432997174477.0 / 9575080441755.0,
                              2526269341429.0 / 6820363962896.0,
                              2006345519317.0 / 3224310063776.0,
                              2802321613138.0 / 2924317926251.0};
  for (int s = 0; s < 5; ++s) {
    a[s] = A[s];
    b[s] = B[s];
    c[s] = C[s];
  }
}

} // namespace host
} // namespace esdg_b200
