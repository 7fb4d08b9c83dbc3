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
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

namespace rtd {

static std::atomic<long long> g_launches{0}, g_sorts{0};
// RTD_TRACE_HOST=1: host timestamp and call site of every launch, the last TRACE_N printed at exit as deltas
// (where the host spends its time between launches on a latency-bound fit)
static constexpr int TRACE_N = 4096;
struct TraceEnt {
  long long ns;
  const char* file;
  int line;
};
static TraceEnt g_trace[TRACE_N];
static std::atomic<long long> g_ntrace{0};
static void dump_trace() {
  const long long n = g_ntrace.load(), n0 = n > 400 ? n - 400 : 0;
  for (long long i = n0 + 1; i < n; i++) {
    const TraceEnt& a = g_trace[(i - 1) % TRACE_N];
    const TraceEnt& b = g_trace[i % TRACE_N];
    std::fprintf(stderr, "[trace] %8.1f us  %s:%d\n", (b.ns - a.ns) * 1e-3, std::strrchr(b.file, '/') ? std::strrchr(b.file, '/') + 1 : b.file, b.line);
  }
}
static bool trace_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("RTD_TRACE_HOST");
    v = (e && e[0] == '1') ? 1 : 0;
    if (v) std::atexit(dump_trace);
  }
  return v == 1;
}
void count_launch(const char* file, int line) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (trace_on()) {
    const long long k = g_ntrace.fetch_add(1);
    g_trace[k % TRACE_N] = {std::chrono::duration_cast<std::chrono::nanoseconds>(
                                std::chrono::steady_clock::now().time_since_epoch()).count(), file, line};
  }
}
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

// The quantile and the consistency factor are memoised per argument pair: a bisection to the last double over
// the incomplete-gamma series costs tens of microseconds, and a fit asks for the same few values every call
// (on a latency-bound 20,000-row fit that host time left the GPU idle between launches).
static double chi2_quantile_raw(double prob, int dof);
static std::mutex g_memo_mu;
static std::map<std::pair<double, int>, double> g_q_memo, g_c_memo;
double chi2_quantile(double prob, int dof) {
  {
    std::lock_guard<std::mutex> lk(g_memo_mu);
    auto it = g_q_memo.find({prob, dof});
    if (it != g_q_memo.end()) return it->second;
  }
  const double v = chi2_quantile_raw(prob, dof);
  std::lock_guard<std::mutex> lk(g_memo_mu);
  g_q_memo[{prob, dof}] = v;
  return v;
}

static double chi2_quantile_raw(double prob, int dof) {
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
  {
    std::lock_guard<std::mutex> lk(g_memo_mu);
    auto it = g_c_memo.find({alpha, p});
    if (it != g_c_memo.end()) return it->second;
  }
  const double v = alpha / chi2_cdf(chi2_quantile(alpha, p), p + 2);
  std::lock_guard<std::mutex> lk(g_memo_mu);
  g_c_memo[{alpha, p}] = v;
  return v;
}

}  // namespace rtd
