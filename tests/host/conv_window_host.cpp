// Host build of the device converter in paper_1905_13415_b200/csrc/parpa_convert.cuh (shims below),
// checked against libc strtod / strtoll on random short numeric strings.  Exercised by
// tests/test_convert_host.py; no GPU needed.
#include <algorithm>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#define __device__
#define __host__
#define __forceinline__ inline
#define __noinline__
#define __constant__
static inline int __ffs(uint32_t x) { return __builtin_ffs(x); }
static inline int __popc(uint32_t x) { return __builtin_popcount(x); }
static inline int __ffsll(long long x) { return __builtin_ffsll(x); }
static inline double __ddiv_rn(double a, double b) { return a / b; }
static inline double __dmul_rn(double a, double b) { return a * b; }
static inline double __fma_rn(double a, double b, double c) { return __builtin_fma(a, b, c); }
static inline long long __double_as_longlong(double d) { long long r; memcpy(&r, &d, 8); return r; }
static inline double __longlong_as_double(long long x) { double r; memcpy(&r, &x, 8); return r; }
static inline unsigned long long __umul64hi(unsigned long long a, unsigned long long b) {
  return (unsigned long long)(((unsigned __int128)a * b) >> 64);
}
using std::min;
using std::max;
#include "../../paper_1905_13415_b200/csrc/parpa_convert.cuh"

int main(int argc, char **argv) {
  const long iters = argc > 1 ? atol(argv[1]) : 2000000;
  std::mt19937_64 r(12345);
  long bad = 0, n = 0, n8 = 0;
  const char *fixed[] = {"12.5", "1234.567", "123.4567", ".5", "5.", "-0.0", "+7", "-73.987654", "0.001", "100",
                         "9007199254740993", "1.2.3", "-", ".", "1e5", "1234567.12345678", "99999999999999.9",
                         "-.5", "+.", "0", "-0", "007", "1234", "12345", "123456789012345"};
  const int nfixed = sizeof(fixed) / sizeof(fixed[0]);
  for (long it = 0; it < iters + nfixed; it++) {
    std::string f;
    if (it < nfixed) {
      f = fixed[it];
    } else {
      const int L = 1 + (int)(r() % 16);
      const char al[] = "0123456789.-+eE";
      for (int i = 0; i < L; i++) f += (r() % 10 < 8) ? char('0' + r() % 10) : al[r() % 15];
    }
    char buf[32] = {0};
    memcpy(buf, f.data(), f.size());
    uint32_t x[4];
    memcpy(x, buf, 16);
    for (int isf = 0; isf < 2; isf++) {
      long long out = 0;
      int res = parpa::conv_window(x[0], x[1], x[2], x[3], (uint32_t)f.size(), isf != 0, out);
      if (f.size() <= 8) {                         // the 8-character window must agree where both accept
        unsigned long long x8;
        memcpy(&x8, buf, 8);
        long long out8 = 0;
        const int res8 = parpa::conv_window8(x8, (uint32_t)f.size(), isf != 0, out8);
        if (f.size() <= 4) {                       // and the 4-character one
          uint32_t x4;
          memcpy(&x4, buf, 4);
          long long out4 = 0;
          const int res4 = parpa::conv_window4(x4, (uint32_t)f.size(), isf != 0, out4);
          if (res4 != res8 || (res4 == 1 && out4 != out8)) { if (bad < 10) printf("BAD4 '%s' isf=%d %d %d\n", buf, isf, res4, res8); bad++; }
        }
        if (res8 == 1 && res == 2) { res = 1; out = out8; n8++; }
        else if (res8 == 1 && out8 != out) { if (bad < 10) printf("BAD8 '%s' isf=%d %lld %lld\n", buf, isf, out8, out); bad++; }
        else if (res8 == 1) n8++;
      }
      if (res == 2) continue;                      // deferred to the exact converters
      char *e;
      bool ok;
      long long ref;
      errno = 0;
      if (isf) {
        const double v = strtod(buf, &e);
        ok = *e == 0 && f.find_first_of("eExXnNiI") == std::string::npos;
        memcpy(&ref, &v, 8);
      } else {
        ref = strtoll(buf, &e, 10);
        ok = *e == 0 && errno == 0;
      }
      if (res != 1 || !ok || ref != out) {
        if (bad < 10) printf("BAD '%s' isf=%d res=%d ok=%d out=%lld ref=%lld\n", buf, isf, res, ok, out, ref);
        bad++;
      }
      n++;
    }
  }
  // div_pow10 against the correctly rounded quotient (strtod of "m e-k") over random m <= 2^53, k <= 22
  for (long it = 0; it < iters; it++) {
    const unsigned long long m = 1 + (r() % 4 == 0 ? r() % 100000 : r() % (1ull << 53));
    const uint32_t k = 1 + (uint32_t)(r() % 22);
    char buf[64];
    snprintf(buf, sizeof buf, "%llue-%u", m, k);
    const double ref = strtod(buf, nullptr), got = parpa::div_pow10((double)m, k);
    if (memcmp(&ref, &got, 8) != 0) {
      if (bad < 20) printf("BAD div_pow10 %s got %.17g ref %.17g\n", buf, got, ref);
      bad++;
    }
    n++;
  }
  printf("checked %ld fast-path conversions (%ld by the 8-character window), %ld mismatches\n", n, n8, bad);
  return bad != 0;
}
