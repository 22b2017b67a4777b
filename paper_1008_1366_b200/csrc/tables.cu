// tables.cu -- twiddle-table cache, see tables.cuh.
#include "tables.cuh"

#include "fft_dev.cuh"

#include <cmath>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

namespace idc {

namespace {
std::mutex g_mu;
std::map<std::pair<int, int>, double2*> g_tables;  // (device, N) -> table
std::map<std::pair<int, long>, double2*> g_ptables;  // (device, N * 65536 + E) -> pass table

// exp(2 pi i k / N) with k reduced to the first octant so that cosl/sinl see
// arguments in [0, pi/4] (symmetries are exact).
void root(long k, long N, double* c, double* s) {
  k %= N;
  if (k < 0) k += N;
  // angle = 2 pi k / N.  Work in units of N/8 (octants) using 8k.
  const long double two_pi = 6.283185307179586476925286766559005768L;
  long k8 = 8 * k;
  int oct = (int)(k8 / N);            // 0..7
  long rem = k8 - (long)oct * N;      // 0 <= rem < N, angle within octant = 2pi*rem/(8N)
  long double a = two_pi * (long double)rem / (8.0L * (long double)N);  // [0, pi/4)
  // for odd octants use the complementary angle: pi/4 - a = 2pi*(N-rem)/(8N)
  long double ca, sa;
  if (oct & 1) {
    long double b = two_pi * (long double)(N - rem) / (8.0L * (long double)N);
    // angle = (oct+1)*pi/4 - b
    ca = cosl(b);
    sa = sinl(b);
    // rotate: base (oct+1)*pi/4 is a multiple of pi/2 for odd oct
    int q = (oct + 1) / 2;  // quarter turns (1..4)
    // exp(i(q pi/2 - b)) = i^q * (cos b - i sin b)
    long double re = ca, im = -sa;
    for (int t = 0; t < (q & 3); ++t) {  // multiply by i
      long double tmp = re;
      re = -im;
      im = tmp;
    }
    *c = (double)re;
    *s = (double)im;
  } else {
    ca = cosl(a);
    sa = sinl(a);
    int q = oct / 2;  // quarter turns (0..3)
    long double re = ca, im = sa;
    for (int t = 0; t < q; ++t) {
      long double tmp = re;
      re = -im;
      im = tmp;
    }
    *c = (double)re;
    *s = (double)im;
  }
}
}  // namespace

const double2* zeta_table(int N) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(dev, N);
  auto it = g_tables.find(key);
  if (it != g_tables.end()) return it->second;
  std::vector<double2> h(N);
  for (int k = 0; k < N; ++k) {
    double c, s;
    root(k, N, &c, &s);
    h[k] = make_double2(c, s);
  }
  double2* d = nullptr;
  if (cudaMalloc(&d, sizeof(double2) * (size_t)N) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, h.data(), sizeof(double2) * (size_t)N, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {   // a pageable upload may return before its DMA lands;
    cudaFree(d);                                  // launches on non-blocking streams are not ordered after it
    return nullptr;
  }
  g_tables[key] = d;
  return d;
}

const double2* pass_table(int N, int E) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  if (E > N) E = N;
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(dev, (long)N * 65536 + E);
  auto it = g_ptables.find(key);
  if (it != g_ptables.end()) return it->second;
  std::vector<double2> h;
  for (int NS = 1; NS < N;) {
    const int R = pass_radix(N, E, NS);
    if (NS > 1) {
      const int Q = pass_q(R);
      const long STEP = N / ((long)NS * R);
      auto put = [&](long mult) {
        for (int j = 0; j < NS; ++j) {
          double c, s;
          root(mult * j * STEP, N, &c, &s);
          h.push_back(make_double2(c, s));
        }
      };
#if IDC_FOLD_TW
      (void)Q;
      for (int l = 0; (1 << l) < R; ++l) put(1L << l);
#else
      for (int c = 1; c < Q; ++c) put(c);
      for (int a = 1; a < R / Q; ++a) put((long)Q * a);
#endif
    }
    NS *= R;
  }
  if (h.empty()) h.push_back(make_double2(1.0, 0.0));
  double2* d = nullptr;
  if (cudaMalloc(&d, sizeof(double2) * h.size()) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, h.data(), sizeof(double2) * h.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {   // see zeta_table
    cudaFree(d);
    return nullptr;
  }
  g_ptables[key] = d;
  return d;
}

}  // namespace idc
