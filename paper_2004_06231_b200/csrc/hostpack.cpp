// Host packing of float64 batches (the reference caller's type: trainer.py:104
// up-casts every batch to float64; image datasets are v / 255 in float64,
// modelio.py:145-166). The bytes that cross PCIe are the smallest exact form
// of the batch: when every value is v / 255 (or a raw count v) for a byte v,
// one byte per value -- the device decode (k_decode_u8, io.cu) restores
// exactly the fp32 value the host cast would give -- else fp32 (round to
// nearest). All host threads; a thread that meets an off-grid value stops the
// others. Host code only (g++; AVX2 path chosen at run time).
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace einet {

namespace {

constexpr double kRound = 6755399441055744.0;  // 1.5 * 2^52: round to nearest even by shift

// Exact-grid test of one value: r = x * div clamped to [0, 255] (NaN -> 0)
// and rounded to nearest; x must equal r / div (correctly rounded, as the
// device decode computes it) and carry no sign bit (negative zero's fp32 cast
// keeps the sign, the decoded byte would not).
inline bool pack1(double x, double div, uint8_t &out) {
  double y = x * div;
  y = y > 0.0 ? y : 0.0;
  y = y < 255.0 ? y : 255.0;
  const double r = (y + kRound) - kRound;
  uint64_t bits;
  std::memcpy(&bits, &x, 8);
  out = (uint8_t)(int)r;
  return (r / div == x) & ((bits >> 63) == 0);
}

bool pack_run_scalar(const double *__restrict__ x, uint8_t *__restrict__ u8, int64_t n,
                     double div) {
  bool ok = true;
  for (int64_t i = 0; i < n; ++i) ok &= pack1(x[i], div, u8[i]);
  return ok;
}

// The same test four values at a time: MAXPD returns its second operand for
// a NaN first operand (NaN -> 0), the quotient is the IEEE division, an
// unordered compare flags NaN, the sign bits come from MOVMSKPD.
__attribute__((target("avx2"))) bool pack_run_avx2(const double *__restrict__ x,
                                                   uint8_t *__restrict__ u8, int64_t n,
                                                   double div) {
  const __m256d vdiv = _mm256_set1_pd(div), zero = _mm256_setzero_pd(),
                top = _mm256_set1_pd(255.0), mag = _mm256_set1_pd(kRound);
  const __m128i pick = _mm_setr_epi8(0, 4, 8, 12, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1);
  __m256d bad = zero;
  int sign = 0;
  int64_t i = 0;
  for (; i + 4 <= n; i += 4) {
    const __m256d xv = _mm256_loadu_pd(x + i);
    __m256d y = _mm256_max_pd(_mm256_mul_pd(xv, vdiv), zero);
    y = _mm256_min_pd(y, top);
    const __m256d r = _mm256_sub_pd(_mm256_add_pd(y, mag), mag);
    bad = _mm256_or_pd(bad, _mm256_cmp_pd(_mm256_div_pd(r, vdiv), xv, _CMP_NEQ_UQ));
    sign |= _mm256_movemask_pd(xv);
    const __m128i b = _mm_shuffle_epi8(_mm256_cvttpd_epi32(r), pick);
    const int32_t w = _mm_cvtsi128_si32(b);
    std::memcpy(u8 + i, &w, 4);
  }
  bool ok = _mm256_movemask_pd(bad) == 0 && sign == 0;
  for (; i < n; ++i) ok &= pack1(x[i], div, u8[i]);
  return ok;
}

bool pack_run(const double *x, uint8_t *u8, int64_t n, double div) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  return avx2 ? pack_run_avx2(x, u8, n, div) : pack_run_scalar(x, u8, n, div);
}

template <class F>
void host_parallel(int64_t n, int threads, F &&body) {
  const int64_t min_per = 1 << 18;  // values per thread worth a thread
  int t = (int)std::min<int64_t>(threads, std::max<int64_t>(1, n / min_per));
  if (t <= 1) {
    body(0, n);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(t - 1);
  for (int i = 1; i < t; ++i) pool.emplace_back([&, i] { body(n * i / t, n * (i + 1) / t); });
  body(0, n / t);
  for (auto &th : pool) th.join();
}

}  // namespace

int host_pack_f64(const double *x, int64_t n, uint8_t *u8, float *f32, int threads) {
  if (threads <= 0) threads = (int)std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  for (const double div : {255.0, 1.0}) {
    std::atomic<bool> off{false};
    host_parallel(n, threads, [&](int64_t lo, int64_t hi) {
      constexpr int64_t kStep = 4096;  // poll the stop flag every 4096 values
      for (int64_t b = lo; b < hi; b += kStep) {
        if (off.load(std::memory_order_relaxed)) return;
        if (!pack_run(x + b, u8 + b, std::min(hi, b + kStep) - b, div)) {
          off.store(true, std::memory_order_relaxed);
          return;
        }
      }
    });
    if (!off.load()) return (int)div;
  }
  if (!f32) return -1;
  host_parallel(n, threads, [&](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) f32[i] = (float)x[i];
  });
  return 0;
}

}  // namespace einet
