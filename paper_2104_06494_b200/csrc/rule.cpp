// Host-side construction of the degree-7 rule and its null rules.
//
// Restates /root/reference/proj/src/rule.cpp:166-349 (build_rule).  The
// weights are least-squares / Gram-Schmidt outputs in x87 long double, so the
// only way to reproduce the reference's doubles bit-for-bit is to perform the
// same long double operations in the same order; this file does exactly that
// (tests/test_rule.py compares all 25 orbit weights for n = 1..16 against the
// reference library).  Compiled by g++ with -ffp-contract=off (x87 has no FMA
// anyway), never by nvcc.

#include "rule.hpp"

#include <array>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <vector>

namespace pgn {
namespace {

using ld = long double;
using Vec = std::array<ld, kOrbits>;

enum Orbit { kCenter = 0, kNear = 1, kFar = 2, kPairs = 3, kCorners = 4 };

// rule.cpp:14-17 generator magnitudes (half-width units)
const ld kL2 = std::sqrt(9.0L / 70.0L);
const ld kL3 = std::sqrt(9.0L / 10.0L);
const ld kL4 = std::sqrt(9.0L / 10.0L);
const ld kL5 = std::sqrt(9.0L / 19.0L);
// rule.cpp:26-27 (double constants promoted to long double at use)
constexpr double kNullScaleDeg3 = 1e-2;
constexpr double kNullScaleDeg1 = 1e-4;

// An even monomial x_{a1}^{e1} x_{a2}^{e2} x_{a3}^{e3} on distinct axes.
struct Mono {
  int k;
  int e[3];
};

struct Geom {
  ld mag[kOrbits];
  int64_t size[kOrbits];
};

Geom geometry(int n) {
  Geom g{};
  const ld mags[kOrbits] = {0.0L, kL2, kL3, kL4, kL5};
  const int64_t sizes[kOrbits] = {1, 2 * n, 2 * n, int64_t{2} * n * (n - 1),
                                  int64_t{1} << n};
  for (int o = 0; o < kOrbits; ++o) {
    g.mag[o] = mags[o];
    g.size[o] = sizes[o];
  }
  return g;
}

// Sum of a monomial over the points of one orbit (rule.cpp:38-57).
ld orbit_moment(int orbit, ld mag, int n, const Mono& p) {
  auto pw = [&](int e) { return std::pow(mag, static_cast<ld>(e)); };
  if (orbit == kCenter) return p.k == 0 ? 1.0L : 0.0L;
  if (orbit == kNear || orbit == kFar) {
    if (p.k == 0) return 2.0L * n;
    return p.k == 1 ? 2.0L * pw(p.e[0]) : 0.0L;
  }
  if (orbit == kPairs) {
    if (p.k == 0) return 2.0L * n * (n - 1);
    if (p.k == 1) return 4.0L * (n - 1) * pw(p.e[0]);
    return p.k == 2 ? 4.0L * pw(p.e[0] + p.e[1]) : 0.0L;
  }
  return std::pow(2.0L, static_cast<ld>(n)) * pw(p.e[0] + p.e[1] + p.e[2]);
}

// Mean of the monomial over [-1,1]^n (rule.cpp:60-64).
ld cube_moment(const Mono& p) {
  ld t = 1.0L;
  for (int i = 0; i < p.k; ++i) t /= static_cast<ld>(p.e[i] + 1);
  return t;
}

std::vector<Mono> monomials(int n, int max_deg) {  // rule.cpp:177-191
  std::vector<Mono> v{{0, {0, 0, 0}}};
  if (max_deg >= 2) v.push_back({1, {2, 0, 0}});
  if (max_deg >= 4) {
    v.push_back({1, {4, 0, 0}});
    if (n >= 2) v.push_back({2, {2, 2, 0}});
  }
  if (max_deg >= 6) {
    v.push_back({1, {6, 0, 0}});
    if (n >= 2) v.push_back({2, {4, 2, 0}});
    if (n >= 3) v.push_back({3, {2, 2, 2}});
  }
  return v;
}

// Least-squares solve of the moment system through the normal equations with
// partial pivoting, then a residual check of the full system (rule.cpp:68-111).
Vec solve_normal(const std::vector<Vec>& A, const std::vector<ld>& b,
                 const std::vector<int>& cols) {
  const int k = static_cast<int>(cols.size());
  ld M[kOrbits][kOrbits] = {};
  ld r[kOrbits] = {};
  for (size_t row = 0; row < A.size(); ++row)
    for (int i = 0; i < k; ++i) {
      r[i] += A[row][cols[i]] * b[row];
      for (int j = 0; j < k; ++j) M[i][j] += A[row][cols[i]] * A[row][cols[j]];
    }
  for (int c = 0; c < k; ++c) {
    int piv = c;
    for (int q = c + 1; q < k; ++q)
      if (std::fabs(M[q][c]) > std::fabs(M[piv][c])) piv = q;
    if (piv != c) {
      for (int j = 0; j < k; ++j) std::swap(M[c][j], M[piv][j]);
      std::swap(r[c], r[piv]);
    }
    if (M[c][c] == 0.0L) throw std::logic_error("rule moments: singular system");
    for (int q = c + 1; q < k; ++q) {
      const ld f = M[q][c] / M[c][c];
      for (int j = c; j < k; ++j) M[q][j] -= f * M[c][j];
      r[q] -= f * r[c];
    }
  }
  Vec x{};
  for (int c = k - 1; c >= 0; --c) {
    ld s = r[c];
    for (int j = c + 1; j < k; ++j) s -= M[c][j] * x[cols[j]];
    x[cols[c]] = s / M[c][c];
  }
  for (size_t row = 0; row < A.size(); ++row) {
    ld res = -b[row];
    for (int i = 0; i < k; ++i) res += A[row][cols[i]] * x[cols[i]];
    if (std::fabs(res) > 1e-12L) throw std::logic_error("rule moments: inconsistent system");
  }
  return x;
}

// Point-weighted inner product over orbit vectors (rule.cpp:127-132).
ld pdot(const Vec& u, const Vec& v, const Geom& g) {
  ld s = 0.0L;
  for (int o = 0; o < kOrbits; ++o) s += static_cast<ld>(g.size[o]) * u[o] * v[o];
  return s;
}

// Modified Gram-Schmidt against a growing orthonormal set (rule.cpp:135-158).
struct GramSchmidt {
  const Geom& g;
  std::vector<Vec> basis;
  bool project_out(Vec v, Vec& out) const {
    for (const Vec& q : basis) {
      const ld c = pdot(v, q, g);
      for (int o = 0; o < kOrbits; ++o) v[o] -= c * q[o];
    }
    const ld nn = pdot(v, v, g);
    if (nn < 1e-18L) return false;
    const ld inv = 1.0L / std::sqrt(nn);
    for (int o = 0; o < kOrbits; ++o) out[o] = v[o] * inv;
    return true;
  }
  bool push(const Vec& v) {
    Vec q;
    if (!project_out(v, q)) return false;
    basis.push_back(q);
    return true;
  }
};

}  // namespace

int64_t rule_point_count(int n) {
  return (int64_t{1} << n) + int64_t{2} * n * (n - 1) + 4 * n + 1;
}

RuleOrbits build_rule_orbits(int n) {
  if (n < 1 || n > kMaxDim) throw std::invalid_argument("build_rule: dimension out of range");
  const Geom g = geometry(n);
  std::vector<int> cols7, cols5;
  for (int o = 0; o < kOrbits; ++o)
    if (g.size[o] > 0) cols7.push_back(o);
  for (int o = 0; o < kOrbits - 1; ++o)
    if (g.size[o] > 0) cols5.push_back(o);

  auto system = [&](const std::vector<Mono>& ps, std::vector<Vec>& A, std::vector<ld>& b) {
    A.assign(ps.size(), Vec{});
    b.assign(ps.size(), 0.0L);
    for (size_t r = 0; r < ps.size(); ++r) {
      for (int o = 0; o < kOrbits; ++o)
        A[r][o] = g.size[o] ? orbit_moment(o, g.mag[o], n, ps[r]) : 0.0L;
      b[r] = cube_moment(ps[r]);
    }
  };
  std::vector<Vec> A7, A5;
  std::vector<ld> b7, b5;
  system(monomials(n, 6), A7, b7);
  const Vec w7 = solve_normal(A7, b7, cols7);
  system(monomials(n, 4), A5, b5);
  const Vec w5 = solve_normal(A5, b5, cols5);

  Vec u1{};
  for (int o = 0; o < kOrbits; ++o) u1[o] = w7[o] - w5[o];
  const ld u1_norm = std::sqrt(pdot(u1, u1, g));

  auto per_point = [&](const Mono& p) {  // rule.cpp:216-222
    Vec v{};
    for (int o = 0; o < kOrbits; ++o)
      if (g.size[o]) v[o] = orbit_moment(o, g.mag[o], n, p) / static_cast<ld>(g.size[o]);
    return v;
  };
  // rule.cpp:224-242: seeds e_o orthogonalised against the annihilated
  // moments and the rules found so far.
  auto nulls_against = [&](const std::vector<Mono>& kill, const std::vector<Vec>& prior,
                           int want) {
    GramSchmidt gs{g, {}};
    for (const Mono& p : kill) gs.push(per_point(p));
    for (const Vec& u : prior) gs.push(u);
    std::vector<Vec> got;
    for (int o = 0; o < kOrbits && static_cast<int>(got.size()) < want; ++o) {
      if (!g.size[o]) continue;
      Vec seed{};
      seed[o] = 1.0L;
      Vec q;
      if (gs.project_out(seed, q)) {
        got.push_back(q);
        gs.push(q);
      }
    }
    return got;
  };
  const std::vector<Mono> deg1 = {{0, {0, 0, 0}}};
  const std::vector<Mono> deg3 = {{0, {0, 0, 0}}, {1, {2, 0, 0}}};
  std::vector<Vec> d3 = nulls_against(deg3, {u1}, 2);
  std::vector<Vec> prior = {u1};
  prior.insert(prior.end(), d3.begin(), d3.end());
  std::vector<Vec> d1 = nulls_against(deg1, prior, 1);
  if (d1.empty()) throw std::logic_error("build_rule: degree-1 null rule not found");

  std::vector<Vec> nulls = {u1};
  for (Vec u : d3) {
    for (int o = 0; o < kOrbits; ++o) u[o] *= u1_norm * static_cast<ld>(kNullScaleDeg3);
    nulls.push_back(u);
  }
  for (Vec u : d1) {
    for (int o = 0; o < kOrbits; ++o) u[o] *= u1_norm * static_cast<ld>(kNullScaleDeg1);
    nulls.push_back(u);
  }
  while (nulls.size() < 4) nulls.push_back(nulls.back());

  // Annihilation self-check (rule.cpp:267-279).
  const std::vector<Mono> deg5 = monomials(n, 4);
  const size_t n3 = d3.size();
  for (size_t k = 0; k < nulls.size(); ++k) {
    const std::vector<Mono>& kill = k == 0 ? deg5 : (k <= n3 ? deg3 : deg1);
    for (const Mono& p : kill) {
      ld s = 0.0L;
      for (int o = 0; o < kOrbits; ++o)
        if (g.size[o]) s += nulls[k][o] * orbit_moment(o, g.mag[o], n, p);
      if (std::fabs(s) > 1e-13L) throw std::logic_error("build_rule: null rule fails annihilation");
    }
  }

  RuleOrbits r;
  r.dim = n;
  r.point_count = rule_point_count(n);
  for (int o = 0; o < kOrbits; ++o) {
    r.w[0][o] = static_cast<double>(w7[o]);
    for (int k = 1; k < 5; ++k) r.w[k][o] = static_cast<double>(nulls[k - 1][o]);
  }
  r.gen[0] = static_cast<double>(kL2);
  r.gen[1] = static_cast<double>(kL3);
  r.gen[2] = static_cast<double>(kL4);
  r.gen[3] = static_cast<double>(kL5);
  // The degree-5 rule has no corner orbit, so the first null rule's corner
  // weight is w7's exactly (u1 = w7 - 0).  k_evaluate_sep relies on it: one
  // product w * f serves the corner points' S[0] and S[1] sums.
  if (n >= 2 && std::memcmp(&r.w[0][kCorners], &r.w[1][kCorners], sizeof(double)) != 0)
    throw std::logic_error("build_rule: corner weights of the rule and its first null rule differ");
  return r;
}

void expand_rule(const RuleOrbits& r, double* points, double* weight_sets) {
  const int n = r.dim;
  const int64_t N = r.point_count;
  int64_t p = 0;
  auto put = [&](int orbit, int a, double ga, int b, double gb) {
    if (points) {
      for (int i = 0; i < n; ++i) points[p * n + i] = 0.0;
      if (a >= 0) points[p * n + a] = ga;
      if (b >= 0) points[p * n + b] = gb;
    }
    if (weight_sets)
      for (int k = 0; k < 5; ++k) weight_sets[k * N + p] = r.w[k][orbit];
    ++p;
  };
  put(kCenter, -1, 0, -1, 0);
  for (int orbit = kNear; orbit <= kFar; ++orbit) {
    const double l = r.gen[orbit - 1];
    for (int a = 0; a < n; ++a)
      for (int s = 0; s < 2; ++s) put(orbit, a, s ? l : -l, -1, 0);
  }
  const double l4 = r.gen[2], l5 = r.gen[3];
  for (int a = 0; a < n; ++a)
    for (int b = a + 1; b < n; ++b)
      for (int sa = 0; sa < 2; ++sa)
        for (int sb = 0; sb < 2; ++sb) put(kPairs, a, sa ? l4 : -l4, b, sb ? l4 : -l4);
  for (int64_t mask = 0; mask < (int64_t{1} << n); ++mask) {
    if (points)
      for (int i = 0; i < n; ++i) points[p * n + i] = ((mask >> i) & 1) ? l5 : -l5;
    if (weight_sets)
      for (int k = 0; k < 5; ++k) weight_sets[k * N + p] = r.w[k][kCorners];
    ++p;
  }
}

}  // namespace pgn
