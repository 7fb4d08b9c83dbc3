// Host-side scalar constants of the method (product path, independent of the oracle).
//   chi2_{p,u} quantile  — cut-off c_p^2 and the univariate
//                          reweighting cut-off chi2_{1,0.975};
//   c(alpha, p) = alpha / F_{chi2_{p+2}}(chi2_{p,alpha}) — consistency factor
//                          (reading R1).
// F is the regularised lower incomplete gamma P(a, x) (series below a+1,
// Lentz continued fraction above); the quantile is found by bisection to the
// last representable double.
#include <cmath>
#include <atomic>
#include <cstdlib>

namespace rtd {

static std::atomic<long long> g_launches{0}, g_sorts{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void count_sort() { g_sorts.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(); }
long long sort_count() { return g_sorts.load(); }

bool debug_sync() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("RTD_DEBUG_SYNC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

static double gamma_p(double a, double x) {
  if (x <= 0.0) return 0.0;
  const double lg = std::lgamma(a);
  if (x < a + 1.0) {
    double ap = a, sum = 1.0 / a, del = sum;
    for (int n = 0; n < 100000; n++) {
      ap += 1.0;
      del *= x / ap;
      sum += del;
      if (std::fabs(del) < std::fabs(sum) * 1e-17) break;
    }
    return sum * std::exp(-x + a * std::log(x) - lg);
  }
  // continued fraction for Q(a, x)
  const double tiny = 1e-300;
  double b = x + 1.0 - a, c = 1.0 / tiny, d = 1.0 / b, h = d;
  for (int i = 1; i < 100000; i++) {
    double an = -i * (i - a);
    b += 2.0;
    d = an * d + b;
    if (std::fabs(d) < tiny) d = tiny;
    c = b + an / c;
    if (std::fabs(c) < tiny) c = tiny;
    d = 1.0 / d;
    double del = d * c;
    h *= del;
    if (std::fabs(del - 1.0) < 1e-17) break;
  }
  return 1.0 - std::exp(-x + a * std::log(x) - lg) * h;
}

double chi2_cdf(double x, int dof) { return gamma_p(0.5 * dof, 0.5 * x); }

double chi2_quantile(double prob, int dof) {
  double lo = 0.0, hi = std::fmax(1.0, (double)dof);
  while (chi2_cdf(hi, dof) < prob) hi *= 2.0;
  for (int it = 0; it < 2000; it++) {
    double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (chi2_cdf(mid, dof) < prob) lo = mid; else hi = mid;
  }
  // pick the endpoint whose CDF is closer to prob
  return std::fabs(chi2_cdf(lo, dof) - prob) <= std::fabs(chi2_cdf(hi, dof) - prob) ? lo : hi;
}

double consistency_factor(double alpha, int p) {
  if (alpha >= 1.0) return 1.0;
  return alpha / chi2_cdf(chi2_quantile(alpha, p), p + 2);
}

}  // namespace rtd
