// parpa_convert.cuh — type conversion of field values on the device.
//
// Thread tier (inside the emit kernels): int64 exact; float64 by Clinger's fast path — with at
// most 19 significant digits m <= 2^53 and a decimal exponent |e| <= 22, the value m·10^e is one
// correctly rounded IEEE division or multiplication of two exact doubles.  Everything else is
// deferred to the device tier (k_deferred), which runs an exact decimal-to-binary algorithm: the
// digits are held as a decimal (up to 800 digits + a "truncated nonzero" flag), scaled by powers
// of two until they lie in [1/2, 1), shifted by 53 bits and rounded half-to-even.  That is the
// "simple decimal conversion" scheme (as in Go's strconv); it is exact for every input.
// Grammar (reading R15): [+-]?([0-9]+(\.[0-9]*)?|\.[0-9]+)([eE][+-]?[0-9]+)?; int64 (R14):
// [+-]?[0-9]+ within [-2^63, 2^63-1].  Sources yield the field's DATA bytes one at a time.
#pragma once
#include <stdint.h>

namespace parpa {

__constant__ double c_pow10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                   1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
// RN(10^-k): the compiler rounds each decimal literal correctly
__constant__ double c_rpow10[23] = {1e-0,  1e-1,  1e-2,  1e-3,  1e-4,  1e-5,  1e-6,  1e-7,  1e-8,  1e-9,  1e-10, 1e-11,
                                    1e-12, 1e-13, 1e-14, 1e-15, 1e-16, 1e-17, 1e-18, 1e-19, 1e-20, 1e-21, 1e-22};

// Correctly rounded m / 10^k for an exact double m (0 < m <= 2^53) and 1 <= k <= 22 with three FP64
// operations instead of a full division: y = RN(1/b) (table), q = RN(m·y) is within an ulp of m/b, the
// residual r = m - q·b is exact in one FMA, and RN(q + r·y) is then the correctly rounded quotient
// (Markstein's theorem; no over/underflow is possible in this range).  Verified against libc strtod
// by tests/test_convert_host.py.
__device__ __forceinline__ double div_pow10(double m, uint32_t k) {
  const double b = c_pow10[k], y = c_rpow10[k];
  const double q = __dmul_rn(m, y);
  const double r = __fma_rn(-q, b, m);
  return __fma_rn(r, y, q);
}

// returns 1 valid, 0 invalid
template <class Src>
__device__ int conv_int64(Src &s, long long &out) {
  uint8_t c;
  if (!s.next(c)) return 0;
  bool neg = false;
  if (c == '+' || c == '-') {
    neg = c == '-';
    if (!s.next(c)) return 0;
  }
  unsigned long long acc = 0;
  int nsig = 0;
  while (true) {
    unsigned d = (unsigned)c - '0';
    if (d > 9) return 0;
    if (nsig || d) {
      if (++nsig > 19) return 0;                 // >= 10^19 > 2^63: overflow
      acc = acc * 10ull + d;
    }
    if (!s.next(c)) break;
  }
  unsigned long long lim = neg ? 0x8000000000000000ull : 0x7FFFFFFFFFFFFFFFull;
  if (acc > lim) return 0;
  out = neg ? (long long)(0ull - acc) : (long long)acc;
  return 1;
}

// returns 1 valid (bits set), 0 invalid grammar, 2 valid but outside the exact fast path
template <class Src>
__device__ int conv_float64_fast(Src &s, long long &bits) {
  uint8_t c;
  bool more = s.next(c);
  if (!more) return 0;
  bool neg = false;
  if (c == '+' || c == '-') {
    neg = c == '-';
    more = s.next(c);
  }
  unsigned long long m = 0;
  int nsig = 0, e10 = 0, ndig = 0;
  bool dropped = false;
  while (more && (unsigned)(c - '0') <= 9u) {
    unsigned d = c - '0';
    ndig++;
    if (nsig || d) {
      if (nsig < 19) { m = m * 10ull + d; nsig++; }
      else { e10++; dropped |= d != 0; }
    }
    more = s.next(c);
  }
  if (more && c == '.') {
    more = s.next(c);
    while (more && (unsigned)(c - '0') <= 9u) {
      unsigned d = c - '0';
      ndig++;
      if (nsig || d) {
        if (nsig < 19) { m = m * 10ull + d; nsig++; e10--; }
        else dropped |= d != 0;
      } else {
        e10--;
      }
      more = s.next(c);
    }
  }
  if (ndig == 0) return 0;
  if (more && (c == 'e' || c == 'E')) {
    bool eneg = false;
    int ex = 0, nex = 0;
    more = s.next(c);
    if (more && (c == '+' || c == '-')) {
      eneg = c == '-';
      more = s.next(c);
    }
    while (more && (unsigned)(c - '0') <= 9u) {
      if (ex < 100000) ex = ex * 10 + (c - '0');
      nex++;
      more = s.next(c);
    }
    if (nex == 0) return 0;
    e10 += eneg ? -ex : ex;
  }
  if (more) return 0;                             // trailing bytes outside the grammar
  if (m == 0) {
    bits = neg ? (long long)0x8000000000000000ull : 0;
    return 1;
  }
  if (dropped || m > (1ull << 53) || e10 < -22 || e10 > 22) return 2;
  double v = (double)m;
  v = e10 < 0 ? __ddiv_rn(v, c_pow10[-e10]) : __dmul_rn(v, c_pow10[e10]);
  if (neg) v = -v;
  bits = __double_as_longlong(v);
  return 1;
}

// ---- register-window fast path (thread tier, both types in one instruction stream) -----------------
// x0..x3 = the field's first 16 bytes (byte i of the 128-bit value = field byte i), 1 <= L <= 16.
// Accepts [+-]?digits with at most one '.' (float64 only) — the common shapes; anything else
// (exponents, stray bytes, empty digit strings, > 2^53 significands) returns 2 and goes to the
// byte-at-a-time converters above, which decide validity exactly.  int64 and float64 share the
// instruction stream so that lanes of different numeric columns do not diverge.
// Four characters per step (SWAR): classify digits / '.' with carry-free byte arithmetic, turn the
// sign into a leading zero digit and drop the '.' (shift the bytes before it up by one, so that it
// becomes a leading zero of the step, which then contributes one digit less), right-align the step's
// characters and fold them as four decimal digits.
__device__ __forceinline__ uint32_t digits4(uint32_t d) {          // byte 0 = most significant digit
  const uint32_t t = d * 10u + (d >> 8);                           // bytes 0, 2: two-digit pairs
  return (t & 0xFFu) * 100u + ((t >> 16) & 0xFFu);
}
__device__ __forceinline__ int conv_window(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3, uint32_t L,
                                           bool isf, long long &out) {
  const uint32_t c0 = x0 & 0xFFu;
  const bool neg = c0 == '-';
  const uint32_t sgn = (c0 == '-' || c0 == '+') ? 1u : 0u;
  if (sgn) x0 = (x0 & 0xFFFFFF00u) | 0x30u;                        // sign -> leading '0'
  const uint32_t xs[4] = {x0, x1, x2, x3};
  unsigned long long m = 0;
  uint32_t bad = 0, ndots = 0, dotpos = 0;
#pragma unroll
  for (int w = 0; w < 4; w++) {
    if (4u * w >= L) break;
    const uint32_t k = min(4u, L - 4u * w);                        // characters of the field in this step
    const uint32_t x = xs[w];
    uint32_t d = x ^ 0x30303030u;                                  // digits -> 0..9
    const uint32_t t = x ^ 0x2E2E2E2Eu;                            // '.' -> 0
    const uint32_t vm = k == 4u ? 0x80808080u : (0x80808080u & ((1u << (8u * k)) - 1u));
    const uint32_t dotm = ~(((t & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | t) & vm;
    const uint32_t ndm = (((d & 0x7F7F7F7Fu) + 0x76767676u) | d) & vm;
    bad |= ndm & ~dotm;
    uint32_t kd = k;                                               // digits this step contributes
    if (dotm) {
      const uint32_t q = ((uint32_t)__ffs(dotm) - 1u) >> 3;       // byte of the '.'
      ndots += (uint32_t)__popc(dotm);
      dotpos = 4u * w + q;
      const uint32_t lo = (1u << (8u * q)) - 1u;                   // bytes before the '.'
      const uint32_t hi = q == 3u ? 0u : (0xFFFFFFFFu << (8u * (q + 1u)));
      d = ((d & lo) << 8) | (d & hi);                              // drop it: a leading zero of the step
      kd--;
    }
    if (k < 4u) d <<= 8u * (4u - k);                               // right-align (zeros lead)
    const uint32_t p10 = kd == 4u ? 10000u : kd == 3u ? 1000u : kd == 2u ? 100u : kd == 1u ? 10u : 1u;
    m = m * p10 + digits4(d);
  }
  const uint32_t nd = L - sgn - ndots;
  if (bad || ndots > 1u || nd == 0u || (ndots && !isf)) return 2;
  if (!isf) {
    out = neg ? (long long)(0ull - m) : (long long)m;              // < 10^16: no overflow
    return 1;
  }
  if (m == 0) {
    out = neg ? (long long)0x8000000000000000ull : 0;
    return 1;
  }
  if (m > (1ull << 53)) return 2;
  const uint32_t frac = ndots ? L - 1u - dotpos : 0u;
  double v = (double)m;
  if (frac) v = div_pow10(v, frac);                                // Clinger: one correctly rounded op
  if (neg) v = -v;
  out = __double_as_longlong(v);
  return 1;
}

// ---- four- / eight-character windows (the common case: every numeric field of the taxi / yelp / clf
// shapes) ---------------------------------------------------------------------------------------------
// x = the field's first 4 / 8 bytes (byte i = field byte i), 1 <= L <= 4 / 8.  The same grammar subset as
// conv_window, in one 32- / 64-bit word: the sign becomes a leading '0', the '.' is squeezed out (the bytes
// after it move down one place), the n remaining characters are checked to be digits in one carry-free
// test, shifted up so that 4 - n / 8 - n zero digits lead, and folded pairwise (1+1, 2+2, 4+4 digits).
// Returns 1 (converted) or 2 ("not handled here": the byte-wise converters decide validity exactly).
// parse_window4/8 yield the significand m < 10^8, the digits after the '.' (frac <= 7) and the sign;
// finish_window turns them into int64 or float64 bits (m / 10^frac, one correctly rounded division).
__device__ __forceinline__ int parse_window4(uint32_t x, uint32_t L, bool isf, uint32_t &m, uint32_t &frac, bool &neg) {
  const uint32_t c0 = x & 0xFFu;
  neg = c0 == '-';
  const uint32_t sgn = (c0 == '-' || c0 == '+') ? 1u : 0u;
  const uint32_t vm = 0xFFFFFFFFu >> (32u - 8u * L);
  uint32_t d = (x ^ 0x30303030u) & vm;
  if (sgn) d &= 0xFFFFFF00u;                                     // sign -> leading zero digit
  uint32_t n = L;
  frac = 0;
  if (isf) {                                                     // (an int64 '.' fails the digit test)
    const uint32_t t = d ^ 0x1E1E1E1Eu;                          // '.' (0x2E ^ 0x30) -> 0
    const uint32_t dotm = ~(((t & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | t) & 0x80808080u & vm;
    if (dotm) {
      const uint32_t q = (uint32_t)(__ffs(dotm) - 1) >> 3;      // byte of the first '.'
      const uint32_t lo = (1u << (8u * q)) - 1u;
      d = (d & lo) | ((d >> 8) & ~lo);                           // squeeze it out
      n = L - 1u;
      frac = n - q;
    }
  }
  if (n <= sgn) return 2;                                        // no digit
  const uint32_t nm = 0xFFFFFFFFu >> (32u - 8u * n);
  if ((((d & 0x7F7F7F7Fu) + 0x76767676u) | d) & 0x80808080u & nm) return 2;   // stray byte / 2nd '.'
  d <<= 8u * (4u - n);                                           // right-align: 4 - n leading zeros
  d = (d * 10u + (d >> 8)) & 0x00FF00FFu;
  m = (d & 0xFFFFu) * 100u + (d >> 16);
  return 1;
}
__device__ __forceinline__ int parse_window8(unsigned long long x, uint32_t L, bool isf, uint32_t &m, uint32_t &frac,
                                             bool &neg) {
  const uint32_t c0 = (uint32_t)x & 0xFFu;
  neg = c0 == '-';
  const uint32_t sgn = (c0 == '-' || c0 == '+') ? 1u : 0u;
  const unsigned long long H = 0x8080808080808080ull, M7 = 0x7F7F7F7F7F7F7F7Full;
  const unsigned long long vm = L >= 8u ? ~0ull : (1ull << (8u * L)) - 1ull;
  unsigned long long d = (x ^ 0x3030303030303030ull) & vm;
  if (sgn) d &= ~0xFFull;
  uint32_t n = L;
  frac = 0;
  if (isf) {
    const unsigned long long t = d ^ 0x1E1E1E1E1E1E1E1Eull;
    const unsigned long long dotm = ~(((t & M7) + M7) | t) & H & vm;
    if (dotm) {
      const uint32_t q = (uint32_t)(__ffsll((long long)dotm) - 1) >> 3;
      const unsigned long long lo = (1ull << (8u * q)) - 1ull;
      d = (d & lo) | ((d >> 8) & ~lo);
      n = L - 1u;
      frac = n - q;
    }
  }
  if (n <= sgn) return 2;
  const unsigned long long nm = n >= 8u ? ~0ull : (1ull << (8u * n)) - 1ull;
  if ((((d & M7) + 0x7676767676767676ull) | d) & H & nm) return 2;
  d <<= 8u * (8u - n);
  d = (d * 10u + (d >> 8)) & 0x00FF00FF00FF00FFull;
  d = (d * 100u + (d >> 16)) & 0x0000FFFF0000FFFFull;
  m = (uint32_t)((d * 10000u + (d >> 32)) & 0xFFFFFFFFull);
  return 1;
}
__device__ __forceinline__ long long finish_window(uint32_t m, uint32_t frac, bool neg, bool isf) {
  if (!isf) return neg ? -(long long)m : (long long)m;
  double v = (double)m;
  if (frac) v = div_pow10(v, frac);
  if (neg) v = -v;
  return __double_as_longlong(v);
}
__device__ __forceinline__ int conv_window4(uint32_t x, uint32_t L, bool isf, long long &out) {
  uint32_t m, frac;
  bool neg;
  if (parse_window4(x, L, isf, m, frac, neg) != 1) return 2;
  out = finish_window(m, frac, neg, isf);
  return 1;
}
__device__ __forceinline__ int conv_window8(unsigned long long x, uint32_t L, bool isf, long long &out) {
  uint32_t m, frac;
  bool neg;
  if (parse_window8(x, L, isf, m, frac, neg) != 1) return 2;
  out = finish_window(m, frac, neg, isf);
  return 1;
}

// ---- timestamps (reading R29)----------------------------------------------------------
// Seconds since 1970-01-01T00:00:00Z of an ISO "YYYY-MM-DD HH:MM:SS" ('T' also accepted) or CLF
// "DD/Mon/YYYY:HH:MM:SS +HHMM" datetime (the zone offset is subtracted); proleptic Gregorian, no
// leap seconds, exact lengths 19 / 26, fields range-checked, anything else invalid.  Day count:
// 365 days per year plus the leap years before it (y/4 - y/100 + y/400, years shifted by one
// 400-year cycle so that every quantity is positive), plus the days before the month from the
// closed form (367 M - 362) / 12 minus 2 (1 in a leap year) after February, plus the day.
__device__ __forceinline__ bool ts_leap(int y) { return (y % 4 == 0 && y % 100 != 0) || y % 400 == 0; }
__host__ __device__ constexpr long long ts_days_shifted(int Y, int M, int D, bool leap) {
  return 365LL * (Y + 400) + (Y + 399) / 4 - (Y + 399) / 100 + (Y + 399) / 400 + (367 * M - 362) / 12 -
         (M <= 2 ? 0 : (leap ? 1 : 2)) + D - 1;
}
constexpr long long TS_EPOCH_DAYS = ts_days_shifted(1970, 1, 1, false);
__device__ __forceinline__ int ts_dig(uint8_t c, int &bad) {
  const int d = (int)c - '0';
  bad |= (unsigned)d > 9u;
  return d;
}
// x = the field's bytes packed little-endian (byte i = bits 8(i%4).. of x[i/4]); n = length.  Every
// byte index below is a compile-time constant, so x stays in registers.
#define TSB(i) ((uint8_t)(x[(i) >> 2] >> (8 * ((i) & 3))))
__device__ __forceinline__ int conv_timestamp_words(const uint32_t (&x)[7], int n, long long &out) {
  int bad = 0, Y, M, D, h, mi, sec, zoff = 0;
  if (n == 19) {
    bad |= TSB(4) != '-' || TSB(7) != '-' || (TSB(10) != ' ' && TSB(10) != 'T') || TSB(13) != ':' || TSB(16) != ':';
    Y = ts_dig(TSB(0), bad) * 1000 + ts_dig(TSB(1), bad) * 100 + ts_dig(TSB(2), bad) * 10 + ts_dig(TSB(3), bad);
    M = ts_dig(TSB(5), bad) * 10 + ts_dig(TSB(6), bad);
    D = ts_dig(TSB(8), bad) * 10 + ts_dig(TSB(9), bad);
    h = ts_dig(TSB(11), bad) * 10 + ts_dig(TSB(12), bad);
    mi = ts_dig(TSB(14), bad) * 10 + ts_dig(TSB(15), bad);
    sec = ts_dig(TSB(17), bad) * 10 + ts_dig(TSB(18), bad);
  } else if (n == 26) {
    bad |= TSB(2) != '/' || TSB(6) != '/' || TSB(11) != ':' || TSB(14) != ':' || TSB(17) != ':' || TSB(20) != ' ' ||
           (TSB(21) != '+' && TSB(21) != '-');
    const uint32_t key = (uint32_t)TSB(3) | ((uint32_t)TSB(4) << 8) | ((uint32_t)TSB(5) << 16);
    switch (key) {
      case 'J' | 'a' << 8 | 'n' << 16: M = 1; break;
      case 'F' | 'e' << 8 | 'b' << 16: M = 2; break;
      case 'M' | 'a' << 8 | 'r' << 16: M = 3; break;
      case 'A' | 'p' << 8 | 'r' << 16: M = 4; break;
      case 'M' | 'a' << 8 | 'y' << 16: M = 5; break;
      case 'J' | 'u' << 8 | 'n' << 16: M = 6; break;
      case 'J' | 'u' << 8 | 'l' << 16: M = 7; break;
      case 'A' | 'u' << 8 | 'g' << 16: M = 8; break;
      case 'S' | 'e' << 8 | 'p' << 16: M = 9; break;
      case 'O' | 'c' << 8 | 't' << 16: M = 10; break;
      case 'N' | 'o' << 8 | 'v' << 16: M = 11; break;
      case 'D' | 'e' << 8 | 'c' << 16: M = 12; break;
      default: M = 0; bad = 1;
    }
    D = ts_dig(TSB(0), bad) * 10 + ts_dig(TSB(1), bad);
    Y = ts_dig(TSB(7), bad) * 1000 + ts_dig(TSB(8), bad) * 100 + ts_dig(TSB(9), bad) * 10 + ts_dig(TSB(10), bad);
    h = ts_dig(TSB(12), bad) * 10 + ts_dig(TSB(13), bad);
    mi = ts_dig(TSB(15), bad) * 10 + ts_dig(TSB(16), bad);
    sec = ts_dig(TSB(18), bad) * 10 + ts_dig(TSB(19), bad);
    const int zh = ts_dig(TSB(22), bad) * 10 + ts_dig(TSB(23), bad);
    const int zm = ts_dig(TSB(24), bad) * 10 + ts_dig(TSB(25), bad);
    bad |= zh > 23 || zm > 59;
    zoff = (zh * 3600 + zm * 60) * (TSB(21) == '-' ? -1 : 1);
  } else {
    return 0;
  }
  if (bad || M < 1 || M > 12 || D < 1 || h > 23 || mi > 59 || sec > 59) return 0;
  const bool leap = ts_leap(Y);
  const int dim = M == 2 ? 28 + (leap ? 1 : 0) : 30 + ((M + (M >> 3)) & 1);
  if (D > dim) return 0;
  out = (ts_days_shifted(Y, M, D, leap) - TS_EPOCH_DAYS) * 86400LL + h * 3600 + mi * 60 + sec - zoff;
  return 1;
}
#undef TSB
// byte-source form (the rare paths: fields outside a register window, device tier)
template <class Src>
__device__ __noinline__ int conv_timestamp(Src &s, long long &out) {
  uint32_t x[7] = {0, 0, 0, 0, 0, 0, 0};
  int n = 0;
  uint8_t c;
#pragma unroll 1
  while (s.next(c)) {
    if (n >= 26) return 0;                                 // longer than any accepted shape
    x[n >> 2] |= (uint32_t)c << (8 * (n & 3));
    n++;
  }
  return conv_timestamp_words(x, n, out);
}

// ---- exact slow path ------------------------------------------------------------------------
// The multi-precision decimal below (dec_* : digit shifts, round-half-even, float bits) follows the
// structure of the Go standard library's strconv "decimal" conversion (decimal.go / atof.go), written
// anew in C++ for this device tier.  That code's notice, reproduced as its license requires:
//
//   Copyright (c) 2009 The Go Authors. All rights reserved.
//
//   Redistribution and use in source and binary forms, with or without modification, are permitted
//   provided that the following conditions are met:
//     * Redistributions of source code must retain the above copyright notice, this list of
//       conditions and the following disclaimer.
//     * Redistributions in binary form must reproduce the above copyright notice, this list of
//       conditions and the following disclaimer in the documentation and/or other materials provided
//       with the distribution.
//     * Neither the name of Google Inc. nor the names of its contributors may be used to endorse or
//       promote products derived from this software without specific prior written permission.
//
//   THIS SOFTWARE IS PROVIDED BY THE COPYRIGHT HOLDERS AND CONTRIBUTORS "AS IS" AND ANY EXPRESS OR
//   IMPLIED WARRANTIES, INCLUDING, BUT NOT LIMITED TO, THE IMPLIED WARRANTIES OF MERCHANTABILITY AND
//   FITNESS FOR A PARTICULAR PURPOSE ARE DISCLAIMED. IN NO EVENT SHALL THE COPYRIGHT OWNER OR
//   CONTRIBUTORS BE LIABLE FOR ANY DIRECT, INDIRECT, INCIDENTAL, SPECIAL, EXEMPLARY, OR CONSEQUENTIAL
//   DAMAGES (INCLUDING, BUT NOT LIMITED TO, PROCUREMENT OF SUBSTITUTE GOODS OR SERVICES; LOSS OF USE,
//   DATA, OR PROFITS; OR BUSINESS INTERRUPTION) HOWEVER CAUSED AND ON ANY THEORY OF LIABILITY, WHETHER
//   IN CONTRACT, STRICT LIABILITY, OR TORT (INCLUDING NEGLIGENCE OR OTHERWISE) ARISING IN ANY WAY OUT
//   OF THE USE OF THIS SOFTWARE, EVEN IF ADVISED OF THE POSSIBILITY OF SUCH DAMAGE.
constexpr int DEC_MAX = 800;
constexpr long long EXP_SAT = 100000000000ll;     // exponent accumulation stops at >= 10^11 (12 digits)
struct Decimal {
  uint8_t d[DEC_MAX];            // digit values 0..9, most significant first; value = 0.d × 10^dp
  int nd, dp;
  bool neg, trunc;
};

__device__ inline void dec_trim(Decimal &a) {
  while (a.nd > 0 && a.d[a.nd - 1] == 0) a.nd--;
  if (a.nd == 0) a.dp = 0;
}

__device__ inline void dec_rshift(Decimal &a, int k) {          // divide by 2^k, k <= 60
  int r = 0, w = 0;
  unsigned long long n = 0;
  for (; (n >> k) == 0; r++) {
    if (r >= a.nd) {
      if (n == 0) { a.nd = 0; return; }
      while ((n >> k) == 0) { n = n * 10; r++; }
      break;
    }
    n = n * 10 + a.d[r];
  }
  a.dp -= r - 1;
  unsigned long long mask = (1ull << k) - 1;
  for (; r < a.nd; r++) {
    unsigned long long dig = n >> k;
    n &= mask;
    a.d[w++] = (uint8_t)dig;
    n = n * 10 + a.d[r];
  }
  while (n > 0) {
    unsigned long long dig = n >> k;
    n &= mask;
    if (w < DEC_MAX) a.d[w++] = (uint8_t)dig;
    else if (dig > 0) a.trunc = true;
    n = n * 10;
  }
  a.nd = w;
  dec_trim(a);
}

__device__ inline void dec_lshift(Decimal &a, int k) {          // multiply by 2^k, k <= 60
  uint8_t t[DEC_MAX + 24];
  int w = DEC_MAX + 24;
  unsigned long long n = 0;
  for (int r = a.nd - 1; r >= 0; r--) {
    n += (unsigned long long)a.d[r] << k;
    unsigned long long q = n / 10;
    t[--w] = (uint8_t)(n - 10 * q);
    n = q;
  }
  while (n > 0) {
    unsigned long long q = n / 10;
    t[--w] = (uint8_t)(n - 10 * q);
    n = q;
  }
  int newnd = DEC_MAX + 24 - w;
  int delta = newnd - a.nd;
  int cnt = newnd < DEC_MAX ? newnd : DEC_MAX;
  for (int i = 0; i < cnt; i++) a.d[i] = t[w + i];
  for (int i = cnt; i < newnd; i++)
    if (t[w + i]) a.trunc = true;
  a.nd = cnt;
  a.dp += delta;
  dec_trim(a);
}

__device__ inline void dec_shift(Decimal &a, int k) {
  if (a.nd == 0) return;
  if (k > 0) {
    while (k > 60) { dec_lshift(a, 60); k -= 60; }
    dec_lshift(a, k);
  } else if (k < 0) {
    while (k < -60) { dec_rshift(a, 60); k += 60; }
    dec_rshift(a, -k);
  }
}

__device__ inline bool dec_round_up(const Decimal &a, int nd) {
  if (nd < 0 || nd >= a.nd) return false;
  if (a.d[nd] == 5 && nd + 1 == a.nd) {          // exactly halfway -> round to even
    if (a.trunc) return true;
    return nd > 0 && (a.d[nd - 1] & 1);
  }
  return a.d[nd] >= 5;
}

__device__ inline unsigned long long dec_rounded_integer(const Decimal &a) {
  if (a.dp > 20) return 0xFFFFFFFFFFFFFFFFull;
  int i;
  unsigned long long n = 0;
  for (i = 0; i < a.dp && i < a.nd; i++) n = n * 10 + a.d[i];
  for (; i < a.dp; i++) n *= 10;
  if (dec_round_up(a, a.dp)) n++;
  return n;
}

__device__ inline unsigned long long dec_float_bits(Decimal &a) {
  const int mantbits = 52, bias = -1023;
  const int powtab[9] = {1, 3, 6, 9, 13, 16, 19, 23, 26};
  int exp = 0;
  unsigned long long mant = 0;
  bool overflow = false;
  if (a.nd == 0) { exp = bias; goto out; }
  if (a.dp > 310) { overflow = true; goto out; }
  if (a.dp < -330) { exp = bias; goto out; }
  while (a.dp > 0) {
    int n = a.dp >= 9 ? 27 : powtab[a.dp];
    dec_shift(a, -n);
    exp += n;
  }
  while (a.dp < 0 || (a.dp == 0 && a.d[0] < 5)) {
    int n = -a.dp >= 9 ? 27 : powtab[-a.dp];
    dec_shift(a, n);
    exp -= n;
  }
  exp--;                                           // range [0.5, 1) -> [1, 2)
  if (exp < bias + 1) {
    int n = bias + 1 - exp;
    dec_shift(a, -n);
    exp += n;
  }
  if (exp - bias >= (1 << 11) - 1) { overflow = true; goto out; }
  dec_shift(a, 1 + mantbits);
  mant = dec_rounded_integer(a);
  if (mant == (2ull << mantbits)) {
    mant >>= 1;
    exp++;
    if (exp - bias >= (1 << 11) - 1) { overflow = true; goto out; }
  }
  if ((mant & (1ull << mantbits)) == 0) exp = bias;  // denormal
out:
  if (overflow) { mant = 0; exp = (1 << 11) - 1 + bias; }
  unsigned long long b = mant & ((1ull << mantbits) - 1);
  b |= (unsigned long long)((exp - bias) & ((1 << 11) - 1)) << mantbits;
  if (a.neg) b |= 1ull << 63;
  return b;
}

// exact float64 from any valid grammar; returns 1 / 0
template <class Src>
__device__ int conv_float64_exact(Src &s, long long &bits) {
  Decimal a;
  a.nd = 0; a.dp = 0; a.neg = false; a.trunc = false;
  uint8_t c;
  bool more = s.next(c);
  if (!more) return 0;
  if (c == '+' || c == '-') {
    a.neg = c == '-';
    more = s.next(c);
  }
  bool sawdot = false, sawdigits = false;
  long long ntot = 0;                              // significant digits seen (stored or not)
  long long dp = 0;
  while (more) {
    if (c == '.') {
      if (sawdot) return 0;
      sawdot = true;
      dp = ntot;
    } else if ((unsigned)(c - '0') <= 9u) {
      sawdigits = true;
      if (c == '0' && ntot == 0) {
        dp--;                                      // leading zero (matters only after the point)
      } else {
        if (a.nd < DEC_MAX) a.d[a.nd++] = (uint8_t)(c - '0');
        else if (c != '0') a.trunc = true;
        ntot++;
      }
    } else {
      break;
    }
    more = s.next(c);
  }
  if (!sawdigits) return 0;
  if (!sawdot) dp = ntot;
  if (more && (c == 'e' || c == 'E')) {
    bool eneg = false;
    long long ex = 0;
    int nex = 0;
    more = s.next(c);
    if (more && (c == '+' || c == '-')) {
      eneg = c == '-';
      more = s.next(c);
    }
    while (more && (unsigned)(c - '0') <= 9u) {
      if (ex < EXP_SAT) ex = ex * 10 + (c - '0');   // saturates beyond any significand's reach (< 2^32
      nex++;                                        // digits), so the clamp below decides correctly
      more = s.next(c);
    }
    if (nex == 0) return 0;
    dp += eneg ? -ex : ex;
  }
  if (more) return 0;
  if (dp > 100000) dp = 100000;
  if (dp < -100000) dp = -100000;
  a.dp = (int)dp;
  dec_trim(a);
  bits = (long long)dec_float_bits(a);
  return 1;
}

}  // namespace parpa
