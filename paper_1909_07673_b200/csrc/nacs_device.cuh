// nacs_device.cuh — device helpers shared by the CTA kernels (nacs_kernels.cu) and the
// warp-per-request kernel (nacs_warp.cu).
#pragma once
#include <cfloat>
#include <climits>
#include <cstdint>

#include "nacs_internal.h"

namespace nacs {

#ifndef NACS_FULL
#define NACS_FULL 0xffffffffu
#endif

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// s * d rounded once, for an integer 0 <= d < 2^23: (2^23 + d) is exact in FP32 and
// fma(s, 2^23 + d, -s*2^23) = round(s * d).  s2p23 = s * 2^23 (exact).
__device__ __forceinline__ float scaled_diff(float s, float s2p23, int d) {
  return fmaf(s, __int_as_float(0x4B000000 | d), -s2p23);
}
// x / h for x < 2^24 with magic = ceil(2^32 / h); h = 1 (k = 2) has no 32-bit magic and is
// stored as magic = 0
__device__ __forceinline__ unsigned div_h(unsigned x, unsigned magic) { return magic ? __umulhi(x, magic) : x; }

// FP32 error-bound constants.  u = 2^-24.
// TOPSIS: |r32 - r| <= 20u; ambiguous top-2 gap <= 2^-17 (> 4 x 40u).
constexpr float kTopsisDelta = 7.62939453125e-06f;  // 2^-17

// TOPSIS parameters of one pod step (statistics over the feasible set F).
struct TopsisP {
  float sf[4], s2p23[4];
  float p2sq[2], m2sq[2];  // Fragmentation (f_u in {0,1}): squared weighted distances by f_u
  int mx[4], mn[4];
  int mxb[4], mnb[4];  // 0x4B000000 + mx, 0x4B000000 - mn: the bits of 2^23 + d in one integer add
  double sd[4];
};

// a5T: closeness of one server in FP32 (R12-R13): v_c = w_c x_c / ||x_c||; Ed+ = ||v - A+||,
// Ed- = ||v - A-||, A+ = max, A- = min over F; differences taken in exact integers.
__device__ __forceinline__ float topsis32(const TopsisP& t, int x0, int x1, int x2, int x3) {
  float p0 = scaled_diff(t.sf[0], t.s2p23[0], t.mx[0] - x0);
  float m0 = scaled_diff(t.sf[0], t.s2p23[0], x0 - t.mn[0]);
  float p1 = scaled_diff(t.sf[1], t.s2p23[1], t.mx[1] - x1);
  float m1 = scaled_diff(t.sf[1], t.s2p23[1], x1 - t.mn[1]);
  float p3 = scaled_diff(t.sf[3], t.s2p23[3], t.mx[3] - x3);
  float m3 = scaled_diff(t.sf[3], t.s2p23[3], x3 - t.mn[3]);
  // f_u in {0,1}: its weighted distances are 0 or sf[2], squared once per pod step
  float ep2 = fmaf(p3, p3, fmaf(p1, p1, fmaf(p0, p0, x2 ? t.p2sq[1] : t.p2sq[0])));
  float em2 = fmaf(m3, m3, fmaf(m1, m1, fmaf(m0, m0, x2 ? t.m2sq[1] : t.m2sq[0])));
  float ep = ep2 > 0.f ? __fmul_rn(ep2, rsqrt_approx(ep2)) : 0.f;
  float em = em2 > 0.f ? __fmul_rn(em2, rsqrt_approx(em2)) : 0.f;
  float den = __fadd_rn(ep, em);
  return den > 0.f ? __fmul_rn(em, rcp_approx(den)) : 0.f;
}

// The closeness r = Ed-/(Ed+ + Ed-) = 1 / (1 + sqrt(q)) with q = Ed+^2 / Ed-^2 is a
// decreasing function of q, so an argmax of r is an argmin of q: one reciprocal instead
// of two square roots and a division.  q = +inf when Ed- = 0 (r = 0).  FP32 relative
// error of q <= 19u (Ed+^2, Ed-^2 8u each, reciprocal 2u, product u).
__device__ __forceinline__ float topsis_q32(const TopsisP& t, int x0, int x1, int x2, int x3) {
  float p0 = scaled_diff(t.sf[0], t.s2p23[0], t.mx[0] - x0);
  float m0 = scaled_diff(t.sf[0], t.s2p23[0], x0 - t.mn[0]);
  float p1 = scaled_diff(t.sf[1], t.s2p23[1], t.mx[1] - x1);
  float m1 = scaled_diff(t.sf[1], t.s2p23[1], x1 - t.mn[1]);
  float p3 = scaled_diff(t.sf[3], t.s2p23[3], t.mx[3] - x3);
  float m3 = scaled_diff(t.sf[3], t.s2p23[3], x3 - t.mn[3]);
  float ep2 = fmaf(p3, p3, fmaf(p1, p1, fmaf(p0, p0, x2 ? t.p2sq[1] : t.p2sq[0])));
  float em2 = fmaf(m3, m3, fmaf(m1, m1, fmaf(m0, m0, x2 ? t.m2sq[1] : t.m2sq[0])));
  return em2 > 0.f ? __fmul_rn(ep2, rcp_approx(em2)) : __int_as_float(0x7f800000);
}
// Same q for the scan: (2^23 + d) as one integer add on pre-biased bounds (d >= 0 on F; off
// F the value is finite garbage that the feasibility mask drops), and no Ed- = 0 guard:
// Ed+ = Ed- = 0 only when every feasible server is identical (q = NaN for all, never
// selected; the caller's FP64 re-decision then sees q1 = q2 = inf and decides).  f_u is
// bit 0 of x2 (the warp kernel's layout keeps the server index in the other bits).
__device__ __forceinline__ float topsis_q32_scan(const TopsisP& t, int x0, int x1, int x2, int x3) {
  float p0 = fmaf(t.sf[0], __int_as_float(t.mxb[0] - x0), -t.s2p23[0]);
  float m0 = fmaf(t.sf[0], __int_as_float(x0 + t.mnb[0]), -t.s2p23[0]);
  float p1 = fmaf(t.sf[1], __int_as_float(t.mxb[1] - x1), -t.s2p23[1]);
  float m1 = fmaf(t.sf[1], __int_as_float(x1 + t.mnb[1]), -t.s2p23[1]);
  float p3 = fmaf(t.sf[3], __int_as_float(t.mxb[3] - x3), -t.s2p23[3]);
  float m3 = fmaf(t.sf[3], __int_as_float(x3 + t.mnb[3]), -t.s2p23[3]);
  float ep2 = fmaf(p3, p3, fmaf(p1, p1, fmaf(p0, p0, (x2 & 1) ? t.p2sq[1] : t.p2sq[0])));
  float em2 = fmaf(m3, m3, fmaf(m1, m1, fmaf(m0, m0, (x2 & 1) ? t.m2sq[1] : t.m2sq[0])));
  return __fmul_rn(ep2, rcp_approx(em2));
}
constexpr float kTopsisDeltaQ = 1.52587890625e-05f;  // 2^-16 relative (> 6 x 2 x 19u)

__device__ __forceinline__ double topsis64(const TopsisP& t, int x0, int x1, int x2, int x3) {
  int x[4] = {x0, x1, x2, x3};
  double ep = 0, em = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double p = t.sd[c] * (double)(t.mx[c] - x[c]);
    double m = t.sd[c] * (double)(x[c] - t.mn[c]);
    ep += p * p;
    em += m * m;
  }
  ep = sqrt(ep);
  em = sqrt(em);
  return (ep + em) > 0 ? em / (ep + em) : 0.0;
}

// TOPSIS parameters from the per-criterion scales sd_c = w_c / ||x_c|| (mx, mn already set).
__device__ __forceinline__ void topsis_params_sd(TopsisP& t, const double sdv[4]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double sd = sdv[c];
    t.sd[c] = sd;
    t.sf[c] = (float)sd;
    t.s2p23[c] = (float)sd * 8388608.0f;
    t.mxb[c] = 0x4B000000 + t.mx[c];
    t.mnb[c] = 0x4B000000 - t.mn[c];
  }
  const float q2 = __fmul_rn(t.sf[2], t.sf[2]);
  t.p2sq[0] = t.mx[2] - 0 ? q2 : 0.f;
  t.p2sq[1] = t.mx[2] - 1 ? q2 : 0.f;
  t.m2sq[0] = 0 - t.mn[2] ? q2 : 0.f;
  t.m2sq[1] = 1 - t.mn[2] ? q2 : 0.f;
}

// Statistics -> TOPSIS parameters (R12): ||x_c|| = sqrt(sum over F of x_c^2), exact sums.
__device__ __forceinline__ void topsis_params(TopsisP& t, const double w[4], const unsigned long long sq[4]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double N = sqrt((double)sq[c]);
    double sd = N > 0 ? w[c] / N : 0.0;
    t.sd[c] = sd;
    t.sf[c] = (float)sd;
    t.s2p23[c] = (float)sd * 8388608.0f;
    t.mxb[c] = 0x4B000000 + t.mx[c];
    t.mnb[c] = 0x4B000000 - t.mn[c];
  }
  const float q2 = __fmul_rn(t.sf[2], t.sf[2]);
  t.p2sq[0] = t.mx[2] - 0 ? q2 : 0.f;
  t.p2sq[1] = t.mx[2] - 1 ? q2 : 0.f;
  t.m2sq[0] = 0 - t.mn[2] ? q2 : 0.f;
  t.m2sq[1] = 1 - t.mn[2] ? q2 : 0.f;
}

__device__ __forceinline__ unsigned long long score_key(float r, int u) {
  return ((unsigned long long)__float_as_uint(r) << 32) | (0xFFFFFFFFu - (unsigned)u);
}
__device__ __forceinline__ void top2_insert(unsigned long long& k1, unsigned long long& k2,
                                            unsigned long long k) {
  if (k > k1) { k2 = k1; k1 = k; }
  else if (k > k2) { k2 = k; }
}
__device__ __forceinline__ void top2_merge(unsigned long long& a1, unsigned long long& a2,
                                           unsigned long long b1, unsigned long long b2) {
  unsigned long long hi = a1 > b1 ? a1 : b1;
  unsigned long long lo = a1 > b1 ? b1 : a1;
  unsigned long long s2 = a2 > b2 ? a2 : b2;
  a1 = hi;
  a2 = lo > s2 ? lo : s2;
}
__device__ __forceinline__ void warp_top2(unsigned long long& k1, unsigned long long& k2) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long b1 = __shfl_xor_sync(NACS_FULL, k1, o);
    unsigned long long b2 = __shfl_xor_sync(NACS_FULL, k2, o);
    top2_merge(k1, k2, b1, b2);
  }
}
__device__ __forceinline__ void warp_argmax64(double& v, int& j) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double bv = __shfl_xor_sync(NACS_FULL, v, o);
    int bj = __shfl_xor_sync(NACS_FULL, j, o);
    if (bv > v || (bv == v && (unsigned)bj < (unsigned)j)) { v = bv; j = bj; }
  }
}
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(NACS_FULL, x, o);
  return x;
}

}  // namespace nacs
