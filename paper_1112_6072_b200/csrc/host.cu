// host.cu — host-side parts of libsperm.so: errors, primes, CRT (Garner),
// the improved Step 3 scheduler and the kernel timing registry.
#include <cmath>
#include <algorithm>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace sperm {

static thread_local std::string g_err;

int set_error(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_check(cudaError_t e, const char* what) {
  return set_error(SPERM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

static std::atomic<long long> g_launches{0};
void count_launch(int k) { g_launches += k; }

// The library's scratch buffers come from the device's default stream-ordered pool
// (cudaMallocAsync).  With the default release threshold (0) the pool returns its memory to
// the driver at every synchronization, so the next allocation has to map pages again; keep it.
void keep_pool_memory() {
  static std::atomic<unsigned> done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 32) return;
  const unsigned bit = 1u << dev;
  if (done.load() & bit) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t threshold = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
  }
  done.fetch_or(bit);
}

int sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || cached <= 0)
      cached = 148;
  }
  return cached;
}

// ------------------------------------------------------------------ timing
namespace {
struct TimingEntry {
  double ms = 0.0;
  int64_t launches = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
};
std::mutex g_tmu;
std::map<std::string, TimingEntry> g_timing;
bool g_timing_on = false;
std::vector<cudaEvent_t> g_event_pool;

cudaEvent_t get_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

TimingScope::TimingScope(const char* name, cudaStream_t s) : name_(name), s_(s), ev0_(nullptr), ev1_(nullptr) {
  std::lock_guard<std::mutex> lk(g_tmu);
  if (!g_timing_on) return;
  cudaEvent_t e0 = get_event(), e1 = get_event();
  ev0_ = e0;
  ev1_ = e1;
  cudaEventRecord(e0, s);
}

TimingScope::~TimingScope() {
  if (!ev0_) return;
  cudaEventRecord((cudaEvent_t)ev1_, s_);
  std::lock_guard<std::mutex> lk(g_tmu);
  g_timing[name_].pending.emplace_back((cudaEvent_t)ev0_, (cudaEvent_t)ev1_);
}

}  // namespace sperm

using namespace sperm;

extern "C" {

int sperm_version(void) { return 1; }

// Primes needed to reconstruct per(A) of one host matrix: |per(A)| <= min(prod of row abs
// sums, prod of column abs sums) and, for a 0/1 matrix, the Bregman-Minc bound
// prod_i (r_i!)^(1/r_i) (by rows and by columns).  Logarithms with a safety margin.
int sperm_bound_primes(const int32_t* h_mat, int n, int* h_k) {
  if (!h_k || n < 0 || (n > 0 && !h_mat)) return set_error(SPERM_ERR_ARG, "sperm_bound_primes: bad arguments");
  double lr = 0, lc = 0, br = 0, bc = 0;
  bool binary = true, zero = false;
  for (int i = 0; i < n; ++i) {
    double r = 0, c = 0;
    for (int j = 0; j < n; ++j) {
      const int32_t u = h_mat[(size_t)i * n + j];
      if (u != 0 && u != 1) binary = false;
      r += std::fabs((double)u);
      c += std::fabs((double)h_mat[(size_t)j * n + i]);
    }
    if (r == 0 || c == 0) zero = true;
    if (r > 0) { lr += std::log2(r); br += std::lgamma(r + 1.0) / (r * std::log(2.0)); }
    if (c > 0) { lc += std::log2(c); bc += std::lgamma(c + 1.0) / (c * std::log(2.0)); }
  }
  double lb = std::min(lr, lc);
  if (binary) lb = std::min(lb, std::min(br, bc));
  if (zero) lb = -1.0;
  const double need = lb + 1.0 + 1e-9 * std::fabs(lb) + 1e-6;  // prod p > 2 * bound
  int k = 1;
  while (k <= SPERM_KMAX && 30.99999 * k <= need) ++k;
  if (k > SPERM_KMAX) return set_error(SPERM_ERR_PRIMES, "sperm_bound_primes: bound needs more than 8 primes");
  *h_k = k;
  return SPERM_OK;
}

int64_t sperm_launch_count(int reset) {
  const long long v = reset ? g_launches.exchange(0) : g_launches.load();
  return (int64_t)v;
}

const char* sperm_last_error(void) { return g_err.c_str(); }

uint32_t sperm_prime(int i) { return (i >= 0 && i < SPERM_KMAX) ? kPrimes[i] : 0u; }

void sperm_timing_enable(int on) {
  std::lock_guard<std::mutex> lk(g_tmu);
  g_timing_on = on != 0;
}

void sperm_timing_reset(void) {
  std::lock_guard<std::mutex> lk(g_tmu);
  for (auto& kv : g_timing) {
    for (auto& pr : kv.second.pending) {
      cudaEventSynchronize(pr.second);
      g_event_pool.push_back(pr.first);
      g_event_pool.push_back(pr.second);
    }
  }
  g_timing.clear();
}

int sperm_timing_get(const char* name, double* h_ms, int64_t* h_launches) {
  if (!name || !h_ms || !h_launches) return set_error(SPERM_ERR_ARG, "sperm_timing_get: NULL argument");
  std::lock_guard<std::mutex> lk(g_tmu);
  auto it = g_timing.find(name);
  if (it == g_timing.end()) {
    *h_ms = 0.0;
    *h_launches = 0;
    return SPERM_OK;
  }
  TimingEntry& t = it->second;
  for (auto& pr : t.pending) {
    cudaError_t e = cudaEventSynchronize(pr.second);
    if (e != cudaSuccess) return cuda_check(e, "cudaEventSynchronize");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pr.first, pr.second);
    t.ms += ms;
    t.launches += 1;
    g_event_pool.push_back(pr.first);
    g_event_pool.push_back(pr.second);
  }
  t.pending.clear();
  *h_ms = t.ms;
  *h_launches = t.launches;
  return SPERM_OK;
}

// ------------------------------------------------------------------ CRT
// Garner's algorithm: mixed-radix digits v_i with x = v_0 + p_0 (v_1 + p_1 (v_2 + ...)),
// then x is expanded into base-2^32 limbs; the symmetric representative is taken.
int sperm_crt_batch(const uint32_t* h_residues, int64_t count, int stride, const int32_t* h_k, int k_all,
                    uint32_t* h_mag, int limbs, int* h_sign) {
  if (count < 0 || (count > 0 && (!h_residues || !h_mag || !h_sign)) || stride < 1)
    return set_error(SPERM_ERR_ARG, "sperm_crt_batch: bad arguments");
  for (int64_t r = 0; r < count; ++r) {
    const int k = h_k ? h_k[r] : k_all;
    const int rc = sperm_crt(h_residues + r * stride, k, h_mag + r * limbs, limbs, h_sign + r);
    if (rc != SPERM_OK) return rc;
  }
  return SPERM_OK;
}

namespace {
// inv[j][i] = p_j^-1 mod p_i (j < i), Fermat, computed once
struct CrtTables {
  uint64_t inv[SPERM_KMAX][SPERM_KMAX];
  CrtTables() {
    for (int i = 0; i < SPERM_KMAX; ++i)
      for (int j = 0; j < SPERM_KMAX; ++j) {
        const uint64_t p = kPrimes[i];
        uint64_t r = 1, b = kPrimes[j] % p, e = p - 2;
        while (e) {
          if (e & 1) r = r * b % p;
          b = b * b % p;
          e >>= 1;
        }
        inv[j][i] = r;
      }
  }
};
const CrtTables& crt_tables() {
  static const CrtTables t;
  return t;
}
}  // namespace

int sperm_crt(const uint32_t* h_residues, int k, uint32_t* h_mag, int limbs, int* h_sign) {
  if (!h_residues || !h_mag || !h_sign || k < 1 || k > SPERM_KMAX || limbs < k + 1)
    return set_error(SPERM_ERR_ARG, "sperm_crt: bad arguments");
  // Garner: mixed-radix digits v_i with x = v_0 + p_0 (v_1 + p_1 (v_2 + ...))
  const CrtTables& T = crt_tables();
  uint64_t v[SPERM_KMAX];
  for (int i = 0; i < k; ++i) {
    const uint64_t p = kPrimes[i];
    uint64_t x = h_residues[i] % p;
    for (int j = 0; j < i; ++j) x = (x + p - v[j] % p) % p * T.inv[j][i] % p;
    v[i] = x;
  }
  // x = Horner over the mixed radix, in limbs (k + 2 limbs hold 2x and M: every p_i < 2^31)
  constexpr int LW = SPERM_KMAX + 2;
  uint32_t X[LW] = {0}, M[LW] = {0}, X2[LW];
  const int nl = k + 2;
  auto mul_add = [&](uint32_t* a, uint32_t m, uint32_t add) {
    uint64_t carry = add;
    for (int t = 0; t < nl; ++t) {
      const uint64_t cur = (uint64_t)a[t] * m + carry;
      a[t] = (uint32_t)cur;
      carry = cur >> 32;
    }
  };
  X[0] = (uint32_t)v[k - 1];
  for (int i = k - 2; i >= 0; --i) mul_add(X, kPrimes[i], (uint32_t)v[i]);
  M[0] = 1;
  for (int i = 0; i < k; ++i) mul_add(M, kPrimes[i], 0);
  // compare 2X with M
  for (int t = 0; t < nl; ++t) X2[t] = X[t];
  mul_add(X2, 2, 0);
  int cmp = 0;
  for (int t = nl - 1; t >= 0 && cmp == 0; --t)
    if (X2[t] != M[t]) cmp = X2[t] > M[t] ? 1 : -1;
  int sign = 1;
  if (cmp > 0) {  // x - M < 0: magnitude M - X
    int64_t borrow = 0;
    for (int t = 0; t < nl; ++t) {
      const int64_t d = (int64_t)M[t] - X[t] - borrow;
      borrow = d < 0;
      X[t] = (uint32_t)(d + (borrow ? (int64_t)1 << 32 : 0));
    }
    sign = -1;
  }
  for (int t = limbs; t < nl; ++t)
    if (X[t] != 0) return set_error(SPERM_ERR_ARG, "sperm_crt: too few limbs");
  bool zero = true;
  for (int t = 0; t < limbs; ++t) {
    h_mag[t] = t < nl ? X[t] : 0u;
    if (t < nl && X[t]) zero = false;
  }
  *h_sign = zero ? 0 : sign;
  return SPERM_OK;
}

// ------------------------------------------------------------------ schedule
// The improved Step 3: order jobs by non-increasing weight and
// give each to the currently least-loaded machine (LPT); or the
// natural order of Algorithm PH Step 3; or a seeded random order.
int sperm_schedule(const double* h_weights, int64_t count, int machines, int policy, uint64_t seed,
                   int32_t* h_machine, int32_t* h_order, double* h_loads) {
  if (count < 0 || machines < 1 || (count > 0 && (!h_weights || !h_machine || !h_order)))
    return set_error(SPERM_ERR_ARG, "sperm_schedule: bad arguments");
  std::vector<int32_t> order(count);
  for (int64_t i = 0; i < count; ++i) order[i] = (int32_t)i;
  if (policy == 0) {
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
      return h_weights[a] > h_weights[b];  // stable: ties keep the lower job id first
    });
  } else if (policy == 2) {
    uint64_t s = seed;
    auto next = [&]() {
      uint64_t z = (s += 0x9E3779B97F4A7C15ull);
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      return z ^ (z >> 31);
    };
    for (int64_t i = count - 1; i > 0; --i) {
      int64_t j = (int64_t)(next() % (uint64_t)(i + 1));
      std::swap(order[i], order[j]);
    }
  } else if (policy != 1) {
    return set_error(SPERM_ERR_ARG, "sperm_schedule: unknown policy");
  }
  std::vector<double> loads(machines, 0.0);
  for (int64_t r = 0; r < count; ++r) {
    int32_t j = order[r];
    int best = 0;
    for (int m = 1; m < machines; ++m)
      if (loads[m] < loads[best]) best = m;
    h_machine[j] = best;
    loads[best] += h_weights[j];
    h_order[r] = j;
  }
  if (h_loads)
    for (int m = 0; m < machines; ++m) h_loads[m] = loads[m];
  return SPERM_OK;
}

// Algorithm LS replayed with the jobs' actual costs: jobs taken in the given
// order, each to the machine whose accumulated cost is currently least (ties: lowest id) — Step 3
// of Algorithm PH as it runs ("the currently least loaded processor")
// when the job costs are known afterwards (Tables 5-7's natural / exact / estimated orders).
int sperm_list_schedule(const double* h_cost, const int32_t* h_order, int64_t count, int machines,
                        int32_t* h_machine, double* h_loads) {
  if (count < 0 || machines < 1 || (count > 0 && (!h_cost || !h_order)) || !h_loads)
    return set_error(SPERM_ERR_ARG, "sperm_list_schedule: bad arguments");
  std::vector<double> loads(machines, 0.0);
  std::vector<char> seen(count, 0);
  for (int64_t r = 0; r < count; ++r) {
    const int32_t j = h_order[r];
    if (j < 0 || j >= count || seen[j]) return set_error(SPERM_ERR_ARG, "sperm_list_schedule: order is not a permutation");
    seen[j] = 1;
    int best = 0;
    for (int m = 1; m < machines; ++m)
      if (loads[m] < loads[best]) best = m;
    loads[best] += h_cost[j];
    if (h_machine) h_machine[j] = best;
  }
  for (int m = 0; m < machines; ++m) h_loads[m] = loads[m];
  return SPERM_OK;
}

// ------------------------------------------------------------------ interpolation
// Coefficients of the polynomial P of degree < npts through (x_j, P(x_j) mod p_q), modulo each of
// the first k CRT primes: Newton divided differences, then the Newton form expanded into the
// monomial basis (Horner on polynomials), all in exact uint64 arithmetic mod p.  Used for the
// permanental polynomial per(xI - A) (Eq. (11)) from its values at npts points.
static uint64_t powmod(uint64_t b, uint64_t e, uint64_t p) {
  uint64_t r = 1;
  b %= p;
  while (e) {
    if (e & 1) r = r * b % p;
    b = b * b % p;
    e >>= 1;
  }
  return r;
}

int sperm_interpolate_mod(const uint32_t* h_values, int stride, const int64_t* h_x, int npts, int k,
                          uint32_t* h_coef, int coef_stride) {
  if (npts < 1 || k < 1 || k > SPERM_KMAX || stride < k || coef_stride < k || !h_values || !h_x || !h_coef)
    return set_error(SPERM_ERR_ARG, "sperm_interpolate_mod: bad arguments");
  for (int q = 0; q < k; ++q) {
    const uint64_t p = kPrimes[q];
    std::vector<uint64_t> xs(npts), d(npts);
    for (int j = 0; j < npts; ++j) {
      const int64_t xm = h_x[j] % (int64_t)p;
      xs[j] = (uint64_t)(xm < 0 ? xm + (int64_t)p : xm);
      d[j] = h_values[(size_t)j * stride + q] % p;
    }
    for (int j = 0; j < npts; ++j)
      for (int i = 0; i < j; ++i)
        if (xs[i] == xs[j]) return set_error(SPERM_ERR_ARG, "sperm_interpolate_mod: points not distinct mod p");
    // divided differences: d[j] = f[x_0..x_j]
    for (int lvl = 1; lvl < npts; ++lvl)
      for (int j = npts - 1; j >= lvl; --j) {
        const uint64_t num = (d[j] + p - d[j - 1]) % p;
        const uint64_t den = (xs[j] + p - xs[j - lvl]) % p;
        d[j] = num * powmod(den, p - 2, p) % p;
      }
    // P = d0 + (x - x0)(d1 + (x - x1)(d2 + ...)): Horner from the innermost term
    std::vector<uint64_t> c(npts, 0);
    c[0] = d[npts - 1];
    int deg = 0;
    for (int j = npts - 2; j >= 0; --j) {
      // c := c * (x - x_j) + d[j]
      ++deg;
      for (int t = deg; t >= 1; --t) c[t] = (c[t - 1] + (p - xs[j]) * c[t] % p) % p;
      c[0] = ((p - xs[j]) * c[0] % p + d[j]) % p;
    }
    for (int t = 0; t < npts; ++t) h_coef[(size_t)t * coef_stride + q] = (uint32_t)c[t];
  }
  return SPERM_OK;
}

// ------------------------------------------------------------------ Kendall tau
// Kendall's rank correlation with the tie correction of Eq. (10), in
// O(m log m): sort the pairs by (x, y); S = concordant - discordant pairs = P0 - T - U + W - 2 D
// with P0 = m(m-1)/2 pairs, T / U = pairs tied in x / in y (Eqs. (8), (9)), W = pairs tied in
// both, and D = discordant pairs = inversions of the y sequence (in (x, y) order), counted by
// a bottom-up merge sort.  Every count is an exact int64.
int sperm_kendall_tau(const double* h_x, const double* h_y, int64_t m, double* h_tau, int64_t* h_counts) {
  if (m < 0 || (m > 0 && (!h_x || !h_y)) || !h_tau) return set_error(SPERM_ERR_ARG, "sperm_kendall_tau: bad arguments");
  for (int64_t i = 0; i < m; ++i)
    if (std::isnan(h_x[i]) || std::isnan(h_y[i])) return set_error(SPERM_ERR_ARG, "sperm_kendall_tau: NaN input");
  std::vector<int64_t> idx(m);
  for (int64_t i = 0; i < m; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) {
    return h_x[a] != h_x[b] ? h_x[a] < h_x[b] : h_y[a] < h_y[b];
  });
  const int64_t P0 = m * (m - 1) / 2;
  int64_t T = 0, W = 0;
  for (int64_t i = 0; i < m;) {  // runs of equal x, and within them runs of equal (x, y)
    int64_t j = i;
    while (j < m && h_x[idx[j]] == h_x[idx[i]]) ++j;
    T += (j - i) * (j - i - 1) / 2;
    for (int64_t a = i; a < j;) {
      int64_t b = a;
      while (b < j && h_y[idx[b]] == h_y[idx[a]]) ++b;
      W += (b - a) * (b - a - 1) / 2;
      a = b;
    }
    i = j;
  }
  std::vector<double> y(m), tmp(m);
  for (int64_t i = 0; i < m; ++i) y[i] = h_y[idx[i]];
  int64_t D = 0;  // strict inversions y[i] > y[j], i < j (equal y are not discordant)
  for (int64_t w = 1; w < m; w *= 2) {
    for (int64_t lo = 0; lo < m; lo += 2 * w) {
      const int64_t mid = std::min(lo + w, m), hi = std::min(lo + 2 * w, m);
      int64_t a = lo, b = mid, k = lo;
      while (a < mid && b < hi) {
        if (y[a] <= y[b]) tmp[k++] = y[a++];
        else { D += mid - a; tmp[k++] = y[b++]; }
      }
      while (a < mid) tmp[k++] = y[a++];
      while (b < hi) tmp[k++] = y[b++];
    }
    std::swap(y, tmp);
  }
  int64_t U = 0;  // y is now sorted: runs of equal y
  for (int64_t i = 0; i < m;) {
    int64_t j = i;
    while (j < m && y[j] == y[i]) ++j;
    U += (j - i) * (j - i - 1) / 2;
    i = j;
  }
  const int64_t S = P0 - T - U + W - 2 * D;
  const double den = std::sqrt((double)(P0 - T)) * std::sqrt((double)(P0 - U));
  *h_tau = den > 0.0 ? (double)S / den : std::nan("");
  if (h_counts) {
    h_counts[0] = S;
    h_counts[1] = T;
    h_counts[2] = U;
    h_counts[3] = P0;
  }
  return SPERM_OK;
}

}  // extern "C"
