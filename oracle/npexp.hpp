// SPDX-License-Identifier: BSD-3-Clause (SVML-derived; see NOTICE)
// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// numpy's float64 exp as the reference host evaluates it.  numpy 2.3 on an
// AVX512_SKX CPU dispatches np.exp (arrays and numpy scalars) to
// DOUBLE_exp_AVX512_SKX -> Intel SVML __svml_exp8_ha, which differs from
// glibc's exp in the last bit on ~4.5 % of inputs.  Restated from numpy's
// binary (constants from __svml_dexp_ha_data_internal_avx512); pinned by
// tests/test_oracle_residuals.py against the reference's own residual values.
// |x| >= 707.7 (SVML's scalar rare path) uses glibc's exp instead.
#pragma once
#include <cfenv>
#include <cmath>
#include <cstdint>
#include <cstring>

namespace oracle {

inline double svml_exp(double x) {
  static const double TH[16] = {0x1.0000000000000p+0, 0x1.0b5586cf9890fp+0, 0x1.172b83c7d517bp+0,
      0x1.2387a6e756238p+0, 0x1.306fe0a31b715p+0, 0x1.3dea64c123422p+0, 0x1.4bfdad5362a27p+0,
      0x1.5ab07dd485429p+0, 0x1.6a09e667f3bcdp+0, 0x1.7a11473eb0187p+0, 0x1.8ace5422aa0dbp+0,
      0x1.9c49182a3f090p+0, 0x1.ae89f995ad3adp+0, 0x1.c199bdd85529cp+0, 0x1.d5818dcfba487p+0,
      0x1.ea4afa2a490dap+0};
  static const double TL[16] = {0x0.0p+0, 0x1.79aa65d837b6dp-54, -0x1.01b15eaa59348p-55,
      0x1.68efde3a8a894p-54, 0x1.34d754db0abb6p-55, 0x1.59f48a72a4c6dp-55, 0x1.690cebb7aafb0p-56,
      0x1.063e1e21c5409p-54, -0x1.3b3efbf5e2228p-54, -0x1.b32dcb94da51dp-56, 0x1.db72fc1f0eab4p-55,
      0x1.1affc2b91ce27p-56, 0x1.c1a7792cb3387p-55, 0x1.36eae30af0cb3p-56, 0x1.4a385a63d07a7p-56,
      -0x1.ff7128fd391f0p-55};
  if (!(std::fabs(x) < 0x1.61da04cbafe44p+9)) return std::exp(x);
  const int old = std::fegetround();
  std::fesetround(FE_TOWARDZERO);  // first SVML op is {rz-sae}
  volatile double s = std::fma(x, 0x1.71547652b82fep+0, 0x1.8000000003ff0p+48);
  std::fesetround(old);
  const double n = s - 0x1.8000000003ff0p+48;
  uint64_t sb;
  double sv = s;
  std::memcpy(&sb, &sv, 8);
  const int j = static_cast<int>(sb & 15);
  double r = std::fma(-n, 0x1.62e42fefa39efp-1, x);
  r = std::fma(-n, 0x1.abc9e3b39803fp-56, r);
  uint64_t rb;
  std::memcpy(&rb, &r, 8);
  rb &= 0xbfffffffffffffffull;
  std::memcpy(&r, &rb, 8);
  const double r2 = r * r;
  const double p1 = std::fma(0x1.7411836940c04p-10, r, 0x1.1101cbbc265c0p-7);
  const double p2 = std::fma(0x1.55557242d68fep-5, r, 0x1.5555553939732p-3);
  const double p3 = std::fma(0x1.000000000d008p-1, r, 0x1.fffffffffff70p-1);
  double P = std::fma(p1, r2, p2);
  P = std::fma(P, r2, p3);
  const double q = std::fma(P, r, TL[j]);
  const double y = std::fma(q, TH[j], TH[j]);
  return std::ldexp(y, static_cast<int>(std::floor(n)));
}

}  // namespace oracle
