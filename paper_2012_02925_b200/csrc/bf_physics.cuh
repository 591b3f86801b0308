// bf_physics.cuh — point physics of the reference, as device functions.
//
// EXACT build (BF_EXACT=1, -fmad=false): every expression is written in the
// reference's left-to-right evaluation order (C++ and Python associate
// + - * / identically); CUDA's double / and sqrt are IEEE correctly rounded,
// so the results are numpy's bit for bit.
// FAST build (BF_EXACT=0): FMA contraction plus strength reduction — one
// reciprocal per state instead of one division per use, rsqrt for 1/a,
// multiplications by precomputed 1/gamma and 1/(2(g^2-1)), and the kappa=-1
// zero terms dropped.  Each replacement changes a result by a few ulp; the
// 1e-12 parity bar is checked in tests/test_gpu_parity.py.
// Citations: blockflow/physics.py and blockflow/solver.py.
#pragma once
#include "bf_internal.h"

#ifndef BF_NS
#error "define BF_NS (bf_exact / bf_fast) before including bf_physics.cuh"
#endif

namespace bf {
namespace BF_NS {

struct St {
  double r, u, v, w, p;
};

#define BF_DEV __device__ __forceinline__

#if !BF_EXACT
// FAST build: branch-free reciprocal / reciprocal square root.  The MUFU
// seed (rcp/rsqrt.approx.ftz.f64, ~2^-22 relative) is refined by ONE
// third-order step to ~1 ulp (residual e ~2^-22, truncation ~e^3 ~2^-66):
//   1/x:       r + r (e + e^2),           e = 1 - x r
//   1/sqrt(x): y + y e (1/2 + 3/8 e),     e = 1 - x y^2
// (three and five fp64 ops, dependency depth three and four, against four and
// seven / four and six for two Newton steps); no special-case slow path (all
// operands here are normal, positive, finite numbers; non-physical states are
// flagged separately).
BF_DEV double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
#ifdef BF_NEWTON2
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
#else
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
#endif
}
BF_DEV double frsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#ifdef BF_NEWTON2
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  return y * fma(-hx * y, y, 1.5);
#else
  const double e = fma(-x * y, y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
#endif
}
BF_DEV double fsqrt(double x) {       // x * rsqrt(x), one residual correction
  const double y = frsqrt(x);
  const double s = x * y;
  return fma(fma(-s, s, x), 0.5 * y, s);
}
BF_DEV double fdiv(double a, double b) {
  const double r = frcp(b);
  const double q = a * r;
  return fma(fma(-b, q, a), r, q);
}
#define BF_RCP(x) frcp(x)
#define BF_DIV(a, b) fdiv((a), (b))
#define BF_SQRT(x) fsqrt(x)
#else
#define BF_RCP(x) (1.0 / (x))
#define BF_DIV(a, b) ((a) / (b))
#define BF_SQRT(x) sqrt(x)
#endif

// physics.py:169-175.  rinv = 1/rho (FAST only).
BF_DEV void euler_flux(const St& s, double nx, double ny, double nz, const Consts& c,
                       double F[5], double rinv) {
  const double vn = s.u * nx + s.v * ny + s.w * nz;
  const double ke = 0.5 * (s.u * s.u + s.v * s.v + s.w * s.w);
#if BF_EXACT
  (void)rinv;
  const double ht = c.gog1 * s.p / s.r + ke;
#else
  const double ht = c.gog1 * s.p * rinv + ke;
#endif
  const double m = s.r * vn;
  F[0] = m;
  F[1] = m * s.u + nx * s.p;
  F[2] = m * s.v + ny * s.p;
  F[3] = m * s.w + nz * s.p;
  F[4] = m * ht;
}

BF_DEV void euler_flux(const St& s, double nx, double ny, double nz, const Consts& c,
                       double F[5]) {
#if BF_EXACT
  euler_flux(s, nx, ny, nz, c, F, 0.0);
#else
  euler_flux(s, nx, ny, nz, c, F, frcp(s.r));
#endif
}

// physics.py:183-187.  half_inv = 1/(2*delta) (FAST only).
BF_DEV double harten_abs(double lam, double delta, double half_inv) {
  const double mag = fabs(lam);
#if BF_EXACT
  (void)half_inv;
  const double safe = delta > 0.0 ? delta : 1.0;
  return mag < delta ? (lam * lam + delta * delta) / (2.0 * safe) : mag;
#else
  return mag < delta ? (lam * lam + delta * delta) * half_inv : mag;
#endif
}

// physics.py:190-255.  Returns false when the Roe average has a2 <= 0.
BF_DEV bool roe_flux(const St& L, const St& R, double nx, double ny, double nz,
                     const Consts& c, double F[5]) {
  double fl[5], fr[5];
#if BF_EXACT
  euler_flux(L, nx, ny, nz, c, fl, 0.0);
  euler_flux(R, nx, ny, nz, c, fr, 0.0);
  const double hl = c.gog1 * L.p / L.r + 0.5 * (L.u * L.u + L.v * L.v + L.w * L.w);
  const double hr = c.gog1 * R.p / R.r + 0.5 * (R.u * R.u + R.v * R.v + R.w * R.w);
  const double rt = sqrt(R.r / L.r);
  const double wf = 1.0 / (1.0 + rt);
#else
  const double rli = frcp(L.r), rri = frcp(R.r);
  euler_flux(L, nx, ny, nz, c, fl, rli);
  euler_flux(R, nx, ny, nz, c, fr, rri);
  const double hl = c.gog1 * L.p * rli + 0.5 * (L.u * L.u + L.v * L.v + L.w * L.w);
  const double hr = c.gog1 * R.p * rri + 0.5 * (R.u * R.u + R.v * R.v + R.w * R.w);
  const double rt = fsqrt(R.r * rli);
  const double wf = frcp(1.0 + rt);
#endif
  const double rho = rt * L.r;
  const double u = (L.u + rt * R.u) * wf;
  const double v = (L.v + rt * R.v) * wf;
  const double w = (L.w + rt * R.w) * wf;
  const double h = (hl + rt * hr) * wf;
  const double a2 = c.gm1 * (h - 0.5 * (u * u + v * v + w * w));
  const bool ok = !(a2 <= 0.0);
  const double a = BF_SQRT(a2);
  const double vn = u * nx + v * ny + w * nz;
  const double dr = R.r - L.r;
  const double dp = R.p - L.p;
  const double du = R.u - L.u;
  const double dv = R.v - L.v;
  const double dw = R.w - L.w;
  const double dvn = du * nx + dv * ny + dw * nz;
  const double delta = c.efix * (fabs(vn) + a);
#if BF_EXACT
  const double l1 = harten_abs(vn - a, delta, 0.0);
  const double l2 = harten_abs(vn, delta, 0.0);
  const double l5 = harten_abs(vn + a, delta, 0.0);
  const double al1 = (dp - rho * a * dvn) / (2.0 * a2);
  const double al2 = dr - dp / a2;
  const double al5 = (dp + rho * a * dvn) / (2.0 * a2);
#else
  const double hinv = 0.5 * frcp(delta > 0.0 ? delta : 1.0);
  const double l1 = harten_abs(vn - a, delta, hinv);
  const double l2 = harten_abs(vn, delta, hinv);
  const double l5 = harten_abs(vn + a, delta, hinv);
  const double ia2 = frcp(a2);
  const double al1 = (dp - rho * a * dvn) * (0.5 * ia2);
  const double al2 = dr - dp * ia2;
  const double al5 = (dp + rho * a * dvn) * (0.5 * ia2);
#endif
  const double su = du - dvn * nx;
  const double sv = dv - dvn * ny;
  const double sw = dw - dvn * nz;
  const double ke = 0.5 * (u * u + v * v + w * w);
  const double d0 = l1 * al1 + l2 * al2 + l5 * al5;
  const double d1 = l1 * al1 * (u - a * nx) + l2 * (al2 * u + rho * su) + l5 * al5 * (u + a * nx);
  const double d2 = l1 * al1 * (v - a * ny) + l2 * (al2 * v + rho * sv) + l5 * al5 * (v + a * ny);
  const double d3 = l1 * al1 * (w - a * nz) + l2 * (al2 * w + rho * sw) + l5 * al5 * (w + a * nz);
  const double d4 = l1 * al1 * (h - a * vn) + l2 * (al2 * ke + rho * (u * su + v * sv + w * sw)) +
                    l5 * al5 * (h + a * vn);
  F[0] = 0.5 * (fl[0] + fr[0]) - 0.5 * d0;
  F[1] = 0.5 * (fl[1] + fr[1]) - 0.5 * d1;
  F[2] = 0.5 * (fl[2] + fr[2]) - 0.5 * d2;
  F[3] = 0.5 * (fl[3] + fr[3]) - 0.5 * d3;
  F[4] = 0.5 * (fl[4] + fr[4]) - 0.5 * d4;
  return ok;
}

// physics.py:267-290: one side of the Van Leer splitting.  The reference
// evaluates all branches and selects with np.where; evaluating only the
// selected branch gives the same doubles.
BF_DEV void van_leer_half(const St& s, double nx, double ny, double nz, const Consts& c,
                          double sign, double F[5]) {
  const double vn = s.u * nx + s.v * ny + s.w * nz;
#if BF_EXACT
  const double a = sqrt(c.gamma * s.p / s.r);
  const double mn = vn / a;
  const double rinv = 0.0;
#else
  const double rinv = frcp(s.r);
  const double a2 = c.gamma * s.p * rinv;
  const double ainv = frsqrt(a2);
  const double a = a2 * ainv;
  const double mn = vn * ainv;
  {
    // branch-free: both forms, then select (lets the two halves of a face
    // interleave instead of serialising behind data-dependent branches)
    double full[5];
    euler_flux(s, nx, ny, nz, c, full, rinv);
    const double ke = 0.5 * (s.u * s.u + s.v * s.v + s.w * s.w);
    const double sh = mn + sign;
    const double fm = sign * 0.25 * s.r * a * (sh * sh);
    const double et = c.gm1 * vn + sign * 2.0 * a;
    const double fac = (-vn + sign * 2.0 * a) * c.inv_gamma;
    const double ee = et * et * c.inv_vlc + ke - 0.5 * vn * vn;
    const double part[5] = {fm, fm * (s.u + nx * fac), fm * (s.v + ny * fac),
                            fm * (s.w + nz * fac), fm * ee};
    const bool up = sign * mn >= 1.0, down = sign * mn <= -1.0;
#pragma unroll
    for (int e = 0; e < 5; ++e) F[e] = up ? full[e] : (down ? 0.0 : part[e]);
    return;
  }
#endif
  if (sign * mn >= 1.0) {
    euler_flux(s, nx, ny, nz, c, F, rinv);
    return;
  }
  if (sign * mn <= -1.0) {
    F[0] = F[1] = F[2] = F[3] = F[4] = 0.0;
    return;
  }
  const double ke = 0.5 * (s.u * s.u + s.v * s.v + s.w * s.w);
  const double sh = mn + sign;
  const double fm = sign * 0.25 * s.r * a * (sh * sh);
  const double et = c.gm1 * vn + sign * 2.0 * a;
#if BF_EXACT
  const double fac = (-vn + sign * 2.0 * a) / c.gamma;
  const double ee = et * et / c.vl_c + ke - 0.5 * vn * vn;
#else
  const double fac = (-vn + sign * 2.0 * a) * c.inv_gamma;
  const double ee = et * et * c.inv_vlc + ke - 0.5 * vn * vn;
#endif
  F[0] = fm;
  F[1] = fm * (s.u + nx * fac);
  F[2] = fm * (s.v + ny * fac);
  F[3] = fm * (s.w + nz * fac);
  F[4] = fm * ee;
}

// physics.py:293-297
BF_DEV void van_leer_flux(const St& L, const St& R, double nx, double ny, double nz,
                          const Consts& c, double F[5]) {
  double fp[5], fm[5];
  van_leer_half(L, nx, ny, nz, c, 1.0, fp);
  van_leer_half(R, nx, ny, nz, c, -1.0, fm);
#pragma unroll
  for (int e = 0; e < 5; ++e) F[e] = fp[e] + fm[e];
}

// solver.py:138-171, (nx, ny, nz) is the OUTWARD unit normal.  Boundary faces
// only (a small fraction of the work): reference form in both builds.
BF_DEV St farfield_state(const St& s, double nx, double ny, double nz, const Consts& c) {
  const double g = c.gamma;
  const double ai = sqrt(g * s.p / s.r);
  const double vni = s.u * nx + s.v * ny + s.w * nz;
  const double vnf = c.fs_u * nx + c.fs_v * ny + c.fs_w * nz;
  const double rout = vni + 2.0 * ai / c.gm1;
  const double rin = vnf - c.ff_two_af_gm1;
  const double vnb = 0.5 * (rout + rin);
  const double ab = c.ff_qgm1 * (rout - rin);
  const bool out = vnb > 0.0;
  const double sb = out ? s.p / pow(s.r, g) : c.ff_sf;
  const double ut = out ? s.u - vni * nx : c.fs_u - vnf * nx;
  const double vt = out ? s.v - vni * ny : c.fs_v - vnf * ny;
  const double wt = out ? s.w - vni * nz : c.fs_w - vnf * nz;
  const double rb = pow(ab * ab / (g * sb), c.ff_exp);
  const double pb = rb * ab * ab / g;
  const bool so = vnb >= ab;
  const bool si = vnb <= -ab;
  St o;
  o.r = so ? s.r : (si ? c.fs_rho : rb);
  o.u = so ? s.u : (si ? c.fs_u : ut + vnb * nx);
  o.v = so ? s.v : (si ? c.fs_v : vt + vnb * ny);
  o.w = so ? s.w : (si ? c.fs_w : wt + vnb * nz);
  o.p = so ? s.p : (si ? c.fs_p : pb);
  return o;
}

// solver.py:105-131.  np.maximum / np.minimum NaN semantics kept.
template <int LIM>
BF_DEV double limiter(double a, double b) {
  if constexpr (LIM == LIM_NONE) {
    return 1.0;
  } else if constexpr (LIM == LIM_VAN_ALBADA) {
    const double x = BF_DIV(2.0 * a * b + 1e-12, a * a + b * b + 1e-12);
    return (0.0 >= x) ? 0.0 : x;
  } else if constexpr (LIM == LIM_MINMOD) {
    const double r = BF_DIV(a, b);
    return (a * b > 0.0) ? ((1.0 <= r) ? 1.0 : r) : 0.0;
  } else {
    const double r = BF_DIV(a, b);
    const double val = BF_DIV(2.0 * r, 1.0 + r);
    return (a * b > 0.0) ? val : 0.0;
  }
}

// Number of stored limiter arrays per (cell, direction, var): Van Albada is
// bitwise symmetric in (a, b) — (2a)b == (2b)a exactly, a*a+b*b commutes —
// so psi+ == psi- and one evaluation serves both; "none" is identically 1.
template <int LIM>
__host__ __device__ constexpr int psi_count() {
  return LIM == LIM_NONE ? 0 : (LIM == LIM_VAN_ALBADA ? 1 : 2);
}

}  // namespace BF_NS
}  // namespace bf
