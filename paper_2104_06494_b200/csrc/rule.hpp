// Degree-7 fully symmetric rule + embedded null rules (host side).
#pragma once

#include <cstdint>

namespace pgn {

constexpr int kMaxDim = 16;  // geometry.hpp:8
constexpr int kOrbits = 5;   // center, axis-near, axis-far, face pairs, corners

// The rule collapsed to what the kernels need: weights are constant per
// orbit, so 5 weight sets x 5 orbits = 25 doubles plus 4 generator
// magnitudes describe all N(n) points (rule.cpp:281-337).
struct RuleOrbits {
  int dim = 0;
  int64_t point_count = 0;
  double w[5][kOrbits] = {};  // w[k][o]: k = 0 integral (deg 7), 1..4 null rules
  double gen[4] = {};         // l2, l3, l4, l5 as doubles (rule.cpp:302-303)
};

// rule.cpp:162-164
int64_t rule_point_count(int n);

// rule.cpp:166-349, bit-identical (x87 long double, same operation order).
// Throws std::invalid_argument / std::logic_error like the reference.
RuleOrbits build_rule_orbits(int n);

// Expands to the reference's point-major tables (rule.cpp:281-337):
// points N x n, weight_sets 5 x N.  Either pointer may be null.
void expand_rule(const RuleOrbits& r, double* points, double* weight_sets);

}  // namespace pgn
