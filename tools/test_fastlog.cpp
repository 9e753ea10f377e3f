// Accuracy of dev::fastlog vs long-double logl (host build of the same code).
#include <cstdio>
#include <cmath>
#include <random>
#include "../paper_2006_14602_b200/csrc/fastlog.cuh"
static double ulp_err(double got, long double ref) {
  if (ref == 0) return got == 0 ? 0 : 1e9;
  double r = (double)ref;
  double u = std::nextafter(std::fabs(r), INFINITY) - std::fabs(r);
  return (double)(std::fabs((long double)got - ref) / u);
}
int main() {
  std::mt19937_64 g(1);
  double worst = 0, wx = 0; long n = 0, bad = 0;
  auto check = [&](double x) {
    double a = ddpma::dev::fastlog(x);
    long double ref = logl((long double)x);
    double e = ulp_err(a, ref);
    if (e > worst) { worst = e; wx = x; }
    if (e > 0.5) bad++;
    n++;
  };
  std::uniform_real_distribution<double> u01(0.0, 1.0);
  for (int i = 0; i < 4000000; ++i) check(std::exp(u01(g) * 80 - 40));
  for (int i = 0; i < 2000000; ++i) check(1.0 + (u01(g) - 0.5) * 0.1);
  for (int i = 0; i < 2000000; ++i) check(u01(g) * 3);
  for (int i = 0; i < 100000; ++i) check(std::ldexp(1.0 + u01(g), -1060));   // subnormal
  std::printf("n=%ld worst=%.4f ulp at x=%.17g  (>0.5ulp: %.4f%%)\n", n, worst, wx, 100.0 * bad / n);
  std::printf("log(1)=%g log(0)=%g log(-1)=%g log(inf)=%g log(2)=%.17g (ref %.17g)\n",
              ddpma::dev::fastlog(1.0), ddpma::dev::fastlog(0.0), ddpma::dev::fastlog(-1.0),
              ddpma::dev::fastlog(INFINITY), ddpma::dev::fastlog(2.0), std::log(2.0));
  return worst < 1.0 ? 0 : 1;
}
