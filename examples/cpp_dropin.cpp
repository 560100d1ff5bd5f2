// A reference-style caller (cf. bfcub_cli.cpp:69-101) compiled against the
// B200 library: only the include and the namespace alias differ.
#define PAGANI_BFCUB_ALIAS
#include <cstdio>
#include <cstring>

#include "pagani.hpp"

int main(int argc, char** argv) {
  const bool run = argc > 1 && std::strcmp(argv[1], "run") == 0;
  bfcub::Config cfg;
  cfg.tau_rel = 1e-3;
  std::printf("digits=%d d(8)=%d N(8)=%lld\n", cfg.convergence_digits(),
              bfcub::initial_subdivisions(8, cfg.init_target),
              static_cast<long long>(bfcub::rule_point_count(8)));
  std::printf("reference_value(f4, 5) = %.17g\n", bfcub::reference_value("f4", 5));
  if (!run) return 0;
  const auto res = bfcub::integrate(bfcub::integrand_by_id("f4"), bfcub::Bounds::unit_cube(5), cfg);
  std::printf("f4 5D: %.17g +- %.3g %s it=%d regions=%lld\n", res.estimate, res.errorest,
              bfcub::to_string(res.status).c_str(), res.iterations,
              static_cast<long long>(res.regions_generated));
  const auto seq = bfcub::integrate_sequential(bfcub::integrand_by_id("f4"),
                                               bfcub::Bounds::unit_cube(3), 1e-3);
  std::printf("sequential f4 3D: %.17g %s steps=%d\n", seq.estimate,
              bfcub::to_string(seq.status).c_str(), seq.iterations);
  return 0;
}
