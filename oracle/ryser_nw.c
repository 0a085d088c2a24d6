/* oracle/ryser_nw.c — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Ryser's formula with the Nijenhuis-Wilf refinement and Gray-code order
 * ("R-NW"), evaluated in exact integer arithmetic:
 *
 *   w_i(S) = 2 a_{i,n-1} - sum_j a_ij + 2 sum_{j in S} a_ij      (doubled x_i)
 *   per(A) = (-1)^{n-1} 2^{1-n} sum_{S subset [n-1]} (-1)^{|S|} prod_i w_i(S)
 *
 * Subsets are visited in binary-reflected Gray order g(t) = t ^ (t >> 1);
 * going from t-1 to t flips column ctz(t).  Every term's product is formed in
 * full as an exact multi-limb integer and added to a 64*LIMBS-bit two's
 * complement accumulator.  No modular arithmetic, no blocking, no reuse of
 * partial products: a plain transcription of the formula.
 *
 * ryser_nw_range(n, a, t0, t1, acc) adds the terms t in [t0, t1) into acc
 * (LIMBS little-endian uint64 words, two's complement).  The Python wrapper
 * (cryser.py) applies the (-1)^{n-1} 2^{1-n} factor.  Returns 0 on success,
 * -1 if n is out of range or a row sum does not fit in 32 bits.
 */
#include <stdint.h>
#include <string.h>

#define LIMBS 12 /* 768-bit accumulator */

static void add_mag(uint64_t* acc, const uint64_t* mag, int nl, int negative) {
  unsigned __int128 carry = 0;
  if (!negative) {
    for (int k = 0; k < LIMBS; ++k) {
      unsigned __int128 s = (unsigned __int128)acc[k] + (k < nl ? mag[k] : 0) + carry;
      acc[k] = (uint64_t)s;
      carry = s >> 64;
    }
  } else {
    uint64_t borrow = 0;
    for (int k = 0; k < LIMBS; ++k) {
      uint64_t m = k < nl ? mag[k] : 0;
      uint64_t d = acc[k] - m - borrow;
      borrow = (acc[k] < m) || (acc[k] - m < borrow);
      acc[k] = d;
    }
  }
}

int ryser_nw_range(int n, const int64_t* a, uint64_t t0, uint64_t t1, uint64_t* acc) {
  if (n < 1 || n > 62) return -1;
  int64_t w[64];
  for (int i = 0; i < n; ++i) {
    int64_t s = 0;
    for (int j = 0; j < n; ++j) s += a[i * n + j];
    w[i] = 2 * a[i * n + (n - 1)] - s;
  }
  uint64_t g = t0 ^ (t0 >> 1);
  for (int j = 0; j < n - 1; ++j)
    if ((g >> j) & 1)
      for (int i = 0; i < n; ++i) w[i] += 2 * a[i * n + j];
  uint64_t mag[LIMBS];
  for (uint64_t t = t0; t < t1; ++t) {
    if (t != t0) {
      int j = __builtin_ctzll(t);
      g ^= (uint64_t)1 << j;
      int64_t sgn = ((g >> j) & 1) ? 2 : -2;
      for (int i = 0; i < n; ++i) w[i] += sgn * a[i * n + j];
    }
    /* product of the n row sums, magnitude in limbs, sign separately */
    memset(mag, 0, sizeof(mag));
    mag[0] = 1;
    int nl = 1, neg = __builtin_popcountll(g) & 1, zero = 0;
    for (int i = 0; i < n; ++i) {
      int64_t v = w[i];
      if (v == 0) { zero = 1; break; }
      if (v < 0) { neg ^= 1; v = -v; }
      if (v >= ((int64_t)1 << 32)) return -1;
      unsigned __int128 carry = 0;
      for (int k = 0; k < nl; ++k) {
        unsigned __int128 p = (unsigned __int128)mag[k] * (uint64_t)v + carry;
        mag[k] = (uint64_t)p;
        carry = p >> 64;
      }
      if (carry) {
        if (nl == LIMBS) return -1;
        mag[nl++] = (uint64_t)carry;
      }
    }
    if (!zero) add_mag(acc, mag, nl, neg);
  }
  return 0;
}

int ryser_nw_limbs(void) { return LIMBS; }
