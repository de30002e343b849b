// ORACLE — test infrastructure, not product code.
//
// Seeded random streams for restating the reference's test fixtures
// (proj/tests/test_solver.cpp:14-57, acceptance.cpp:100-142,
// kernel_bench.cpp:15-29).  The reference draws std::mt19937 +
// std::uniform_real_distribution<double> from libstdc++; this file uses the same
// engine and distribution (and the same Vec3(u(rng), u(rng), u(rng))
// construction, whose argument evaluation order the compiler fixes) so the
// fixtures reproduce the reference's numbers.
#include <random>

#include "wfo.h"

namespace {
struct Vec3c {
  double x, y, z;
  Vec3c(double a, double b, double c) : x(a), y(b), z(c) {}
};
}  // namespace

struct wfo_rng {
  std::mt19937 eng;
};

extern "C" {

wfo_rng* wfo_rng_new(uint32_t seed) {
  auto* r = new wfo_rng;
  r->eng.seed(seed);
  return r;
}
void wfo_rng_free(wfo_rng* r) { delete r; }
double wfo_rng_uniform(wfo_rng* r, double lo, double hi) {
  std::uniform_real_distribution<double> u(lo, hi);
  return u(r->eng);
}
void wfo_rng_vec3(wfo_rng* r, double lo, double hi, double out[3]) {
  std::uniform_real_distribution<double> u(lo, hi);
  auto& rng = r->eng;
  const Vec3c v(u(rng), u(rng), u(rng));
  out[0] = v.x;
  out[1] = v.y;
  out[2] = v.z;
}
int wfo_rng_int(wfo_rng* r, int lo, int hi) {
  std::uniform_int_distribution<int> u(lo, hi);
  return u(r->eng);
}
/* n draws of Vec3(u, u, u) in sequence (e.g. the per-point jitter loop of
 * kernel_bench.cpp:24-27) */
void wfo_rng_vec3_array(wfo_rng* r, double lo, double hi, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) wfo_rng_vec3(r, lo, hi, out + 3 * i);
}

}  // extern "C"
