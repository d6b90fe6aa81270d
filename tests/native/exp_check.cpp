// Bit-for-bit check of sgdb::libm::exp (paper_1802_08800_b200/csrc/libm_exp.hpp)
// against the host libm's exp. Built and run by tests/test_libm_exp.py with
// -ffp-contract=off so that every non-fma step of the restatement is one
// IEEE operation. Prints "<checked> <mismatches> [first mismatch]".
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "libm_exp.hpp"

int main(int argc, char** argv) {
  const uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1000000;
  std::mt19937_64 rng(12345);
  std::uniform_real_distribution<double> wide(-760.0, 720.0), mid(-40.0, 40.0),
      small(-1.0, 1.0);
  std::uniform_int_distribution<int> ex(-70, 10);
  uint64_t checked = 0, bad = 0;
  auto one = [&](double x) {
    const double a = sgdb::libm::exp(x), b = std::exp(x);
    ++checked;
    if (std::memcmp(&a, &b, sizeof a) != 0 && !(std::isnan(a) && std::isnan(b))) {
      if (bad < 4) std::printf("first mismatch x=%a ours=%a libm=%a\n", x, a, b);
      ++bad;
    }
  };
  const double specials[] = {0.0, -0.0, 1.0, -1.0, 0x1p-54, -0x1p-54, 0x1p-55, 512.0, -512.0,
                             709.78, 709.79, -708.39, -708.4, -744.4, -745.1, -745.2, 1024.0,
                             -1024.0, INFINITY, -INFINITY, NAN, 1e-300, -1e-300, 5e-324};
  for (double s : specials) one(s);
  for (uint64_t i = 0; i < n; ++i) {
    one(wide(rng));
    one(mid(rng));
    one(small(rng));
    one(std::ldexp(small(rng), ex(rng)));
    // neighbours of k ln2/128 boundaries
    const double k = std::floor(mid(rng) * 128.0 / 0.6931471805599453);
    one(std::nextafter(k * 0.6931471805599453 / 128.0 + 0.0027, 0.0));
  }
  std::printf("%llu %llu\n", (unsigned long long)checked, (unsigned long long)bad);
  return bad != 0;
}
