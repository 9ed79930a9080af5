// SPDX-License-Identifier: BSD-3-Clause (SVML-derived; see NOTICE)
// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// numpy's float64 arctan as the reference host evaluates it: numpy 2.3 on an
// AVX512_SKX CPU dispatches np.arctan (arrays and numpy scalars) to Intel SVML
// __svml_atan8_ha, which differs from glibc's atan in ~0.17 % of inputs (the
// reference's helical_valley float residual, problems.py:70-81, calls it; its
// Dual path calls math.atan = glibc).  Restated from numpy's binary (tables
// __svml_datan_ha_data_internal_avx512; the VRCP14PD seed reproduced by the
// table tools/extract_rcp14.c measured on the reference host).  Pinned by
// tests/test_glibc_ports.py (device port) and tests/test_oracle_residuals.py.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>

namespace oracle {

#define NLK_RCP14_TABLE static const uint16_t kRcp14[65536]
#include "../paper_2403_16341_b200/csrc/nlk_rcp14_table.inc"
#undef NLK_RCP14_TABLE

inline uint64_t atan_bits(double d) { uint64_t u; std::memcpy(&u, &d, 8); return u; }
inline double atan_from(uint64_t u) { double d; std::memcpy(&d, &u, 8); return d; }

inline double svml_atan(double x) {
  static const double HI[32] = {0x0.0p+0, 0x1.f5b75f92c80ddp-3, 0x1.dac670561bb4fp-2,
      0x1.4978fa3269ee1p-1, 0x1.921fb54442d18p-1, 0x1.cac7c57846f9ep-1, 0x1.f730bd281f69bp-1,
      0x1.0d38f2c5ba09fp+0, 0x1.1b6e192ebbe44p+0, 0x1.270ef55a53a25p+0, 0x1.30b6d796a4da8p+0,
      0x1.38d6a6ce13353p+0, 0x1.3fc176b7a8560p+0, 0x1.45b54837351a0p+0, 0x1.4ae10fc6589a5p+0,
      0x1.4f68dea672617p+0, 0x1.5368c951e9cfdp+0, 0x1.56f6f33a3e6a7p+0, 0x1.5a25052114e60p+0,
      0x1.5d013c41adabdp+0, 0x1.5f97315254857p+0, 0x1.61f06c6a92b89p+0, 0x1.6414d44094c7cp+0,
      0x1.660b02c736a06p+0, 0x1.67d8863bc99bdp+0, 0x1.698213a9d5053p+0, 0x1.6b0bae830c070p+0,
      0x1.6c78c7edeb195p+0, 0x1.6dcc57bb565fdp+0, 0x1.6f08f07435fecp+0, 0x1.7030cf9403197p+0,
      0x1.7145eac2088a4p+0};
  static const double LO[32] = {0x0.0p+0, 0x1.8ab6e3cf7afbdp-57, 0x1.a2b7f222f65e2p-56,
      0x1.2419a87f2a458p-56, 0x1.1a62633145c07p-55, 0x1.0dae13ad18a6bp-55, 0x1.007887af0cbbdp-56,
      -0x1.bd0dc231bfd70p-54, 0x1.b1b466a88828ep-54, -0x1.a66b1af5f84fbp-54, 0x1.6254cb03bb199p-54,
      -0x1.12c77e8a80f5cp-55, -0x1.441a3bd3f1084p-59, 0x1.9e4a72eedacc4p-56, -0x1.3b03e8a27f555p-54,
      0x1.934f9f2b0020ep-54, -0x1.96f47948a99f1p-54, -0x1.df6edd6f1ec3bp-56, 0x1.8c2d0c89de218p-56,
      0x1.f82bba194dd5dp-54, -0x1.31151a43b51cap-55, -0x1.487d50bceb1a5p-55, -0x1.c5f60a65c7397p-54,
      -0x1.acb6afb332a0fp-56, -0x1.9b7bd2e1e8c9cp-54, -0x1.b9839085189e3p-54, -0x1.7d1ab82ffb70bp-54,
      0x1.9239ad620ffe2p-54, -0x1.29c86447928e7p-54, -0x1.957a7170df016p-55, -0x1.cbe1896221608p-56,
      -0x1.fda5797b32a0bp-54};
  const double S = 0x1.8p50, S4 = 0x1.8000000000010p50;
  const double ax = std::fabs(x);
  const bool in_table = ax < 7.875;  // else the pi/2 - atan(1/x) branch
  const double sh = ax + S;
  const double b = sh - S;  // ax rounded to a quarter (vreducepd 0x28 complement)
  const double t = in_table ? ax - b : -1.0;
  const int idx = static_cast<int>(atan_bits(sh) & 15) + (sh >= S4 ? 16 : 0);
  const double den = in_table ? std::fma(b, ax, 1.0) : (0x1p128 < ax ? 0x1p128 : ax);
  // VRCP14PD seed
  const uint64_t u = atan_bits(den);
  const uint32_t e = static_cast<uint32_t>(u >> 52) & 0x7ffu, m16 = static_cast<uint32_t>(u >> 36) & 0xffffu;
  const double r0 = atan_from((static_cast<uint64_t>((m16 == 0 ? 2046u : 2045u) - e) << 52) |
                              (static_cast<uint64_t>(kRcp14[m16]) << 36));
  const double dlo = std::fma(b, ax, -(den - 1.0));
  const double ee = std::fma(-r0, den, 1.0);
  double r = std::fma(ee, r0, r0);
  r = std::fma(ee * ee, r, r);
  const double q = r * t;
  double c = std::fma(-r, den, 1.0);
  c = std::fma(q, c, std::fma(r, t, -q));
  if (in_table) c = std::fma(-(dlo * r), q, c);
  const double hi = in_table ? HI[idx] : 0x1.921fb54442d18p+0;
  const double lo = in_table ? LO[idx] : 0x1.1a62633145c07p-54;
  const double q2 = q * q, q4 = q2 * q2, q3 = q2 * q;
  double p = std::fma(0x1.2e9b9f5c4fe97p-4, q2, -0x1.74257c46790ccp-4);
  p = std::fma(q4, p, std::fma(0x1.c71bfeff916a0p-4, q2, -0x1.249248eef04dap-3));
  p = std::fma(q4, p, std::fma(0x1.999999998741ep-3, q2, -0x1.555555555554dp-2));
  const double s = hi + q;
  const double low = (c + lo) + (q - (s - hi));
  const double res = std::fma(q3, p, low) + s;
  return atan_from(atan_bits(res) ^ (atan_bits(x) & 0x8000000000000000ull));
}

}  // namespace oracle
