// Division of 32-bit unsigned integers by a divisor fixed for a launch
// (pixel counts, crop width, sample counts, bin counts) with one multiply-high,
// an add and two shifts instead of the ~15-instruction emulated udiv whose
// reciprocal runs on the XU pipe (the MUFU/conversion pipe that the DARTS
// vertex already loads to ~60 %; profiles/README.md).
//
// Method: Granlund & Montgomery, "Division by invariant integers using
// multiplication" (PLDI 1994), Fig. 4.1: for 1 <= d < 2^32 let
// l = ceil(log2 d) and m = floor(2^32 (2^l - d) / d) + 1 (fits 32 bits); then
// for every 0 <= n < 2^32
//   t = mulhi(m, n),  n / d = (t + ((n - t) >> 1)) >> (l - 1)
// (d = 1 is carried as m = 0 with shifts 0 and 0: t = 0, n / d = n).
// Checked exhaustively over edge cases and randomly in tests/test_fastdiv.py.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define DTS_HD __host__ __device__ __forceinline__
#else
#define DTS_HD static inline
#endif

struct FastDiv {
  uint32_t d;   // the divisor
  uint32_t m;   // magic multiplier
  uint32_t s1;  // 1 (0 for d = 1)
  uint32_t s2;  // l - 1 (0 for d = 1)
};

DTS_HD FastDiv fastdiv_make(uint32_t d) {
  FastDiv f;
  f.d = d;
  if (d <= 1) {
    f.m = 0; f.s1 = 0; f.s2 = 0;
    return f;
  }
  uint32_t l = 0;
  while (l < 32 && (1ull << l) < (uint64_t)d) ++l;  // ceil(log2 d), 1..32
  f.m = (uint32_t)((((1ull << l) - d) << 32) / d + 1);
  f.s1 = 1;
  f.s2 = l - 1;
  return f;
}

DTS_HD uint32_t fastdiv_mulhi(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

DTS_HD uint32_t fastdiv_div(uint32_t n, const FastDiv& f) {
  const uint32_t t = fastdiv_mulhi(f.m, n);
  return (t + ((n - t) >> f.s1)) >> f.s2;
}

// quotient and remainder
DTS_HD uint32_t fastdiv_divmod(uint32_t n, const FastDiv& f, uint32_t& r) {
  const uint32_t q = fastdiv_div(n, f);
  r = n - q * f.d;
  return q;
}
