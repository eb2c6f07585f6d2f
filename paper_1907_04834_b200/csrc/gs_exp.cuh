// gs_exp.cuh -- exp(x) for x <= 0 in FP64, for the Gaussian weights of the FP64
// kernels: G = exp(-r^2 / (2 s)) (kernel_exact.cpp:7-9, bh_kernel.cpp). A
// table-driven Cody-Waite reduction: x = (64 e + j) ln2/64 + r, |r| <= ln2/128,
// exp(x) = 2^e * 2^(j/64) * exp(r) with a degree-5 Taylor polynomial (truncation
// 3.5e-17 relative): 10 DP operations instead of libdevice exp's ~17 and no
// slow path. Accuracy: a few ulp for x >= -708; exp(x) < 3.4e-308 (x < -708)
// returns 0 (an absolute change below 3.4e-308 in a sum of O(1) terms).
#pragma once

namespace gsb {

// 2^(j/64), j = 0..63, correctly rounded (generated with 60-digit decimal arithmetic)
static __device__ const double kExp2Tab64[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0,
};

__device__ __forceinline__ double exp_nonpos(double x, const double* __restrict__ tab) {
  const double kL2E64 = 0x1.71547652b82fep+6;     // 64 / ln 2
  const double kShift = 0x1.8p52;                 // rint by addition
  const double kLn2Hi = 0x1.62e42fee00000p-7;     // (ln 2)/64, high 32 bits (exact k * hi)
  const double kLn2Lo = 0x1.a39ef35793c76p-39;    // (ln 2)/64 - kLn2Hi
  const bool tiny = x < -708.0;
  x = tiny ? -708.0 : x;
  double kd = fma(x, kL2E64, kShift);
  const int k = __double2loint(kd);  // rint(x * 64 / ln 2), two's complement in the low word
  kd -= kShift;
  double r = fma(kd, -kLn2Hi, x);
  r = fma(kd, -kLn2Lo, r);
  double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  p = fma(p, r, 1.0 / 6.0);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double t = tab[k & 63];
  // 2^e * t: add e = k >> 6 (>= -1022 for x >= -708) to t's exponent field
  const double s = __hiloint2double(__double2hiint(t) + ((k >> 6) << 20), __double2loint(t));
  return tiny ? 0.0 : s * p;
}

}  // namespace gsb
