// bf_vl.cuh — FAST-build Van Leer stage kernel in the cell-split form
// (included by bf_kernels.cu inside namespace bf::bf_fast).
//
// Why a second kernel: with flux-vector splitting the face flux is
//   F_{c+1/2} = F+(qL_{c+1/2}) + F-(qR_{c+1/2})        (physics.py:293-297)
// and both MUSCL states are functions of ONE cell's stencil
//   qL_{c+1/2} = w_c + (eps/4)[(1-k) Psi+_c D-_c + (1+k) Psi-_c D+_c]
//   qR_{c-1/2} = w_c - (eps/4)[(1+k) Psi+_c D-_c + (1-k) Psi-_c D+_c]
// (solver.py:437-474 with f = c+1 resp. f = c), where Psi+-_c are the cell's
// limiters (solver.py:413-435).  So every cell computes, per direction, the
// half flux F+ of its high face and F- of its low face (already times the
// face area), and the residual needs only the neighbours' halves:
//   R_c = sum_d [F+_c + F-_{c+1}]_d - [F+_{c-1} + F-_c]_d .
// No limiter arrays, no face loop, no per-face load imbalance: x neighbours
// are lanes of the same warp (shuffles), y neighbours go through shared
// memory, z neighbours stay in registers while the CTA marches in k.
// Tile-edge cells outside the tile (2*TJ in x, 2*TI in y per plane) are extra
// half-flux items done by the last warps (warp 0 issues the TMA groups).
//
// Per k-plane: B0 barrier | phase A: halves of plane k (x, y) and the z halves
// of cell k+1 (own column) | AB barrier | phase B: residual, stage-0 dt and
// sum(R^2), RK update, decode.  TMA traffic: the haloed 5-variable plane k+2
// and the geometry group of plane k+1 are issued at the AB barrier of plane k
// (phase B needs no geometry: halves are pre-scaled and wall/farfield
// overwrites are applied in phase A); Q0/dt of plane k at B0.
//
// Used for FAST precision, Van Leer flux, limiters computed (not frozen);
// the reference-order kernel (bf_stage.cuh) covers EXACT, Roe and the
// limiter-freeze steps.  Different FP association than the reference (area
// scaling per half, FMA, Newton reciprocals): held to the 1e-12 bar.
#pragma once

// In-kernel ghost push (PushRule): compiled in with -DBF_VL_PUSH=1 only; on
// C4 it is slower than the separate ghost launch.
#ifndef BF_VL_PUSH
#define BF_VL_PUSH 0
#endif
// The tile's block record (DevBlock) in shared memory instead of a register
// copy: C4 stage 1.158 -> 1.115 ms (S1 spills 32/52 B -> 0; the k loop reloaded
// spilled invariants from local memory every plane).  -DBF_VL_SMEM_BLOCK=0: copy.
#ifndef BF_VL_SMEM_BLOCK
#define BF_VL_SMEM_BLOCK 1
#endif
#ifndef BF_VL2D_MINB
#define BF_VL2D_MINB 2
#endif

BF_DEV void tma_prefetch4(const void* tmap, int x, int y, int z, int s) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                   reinterpret_cast<unsigned long long>(tmap)),
               "r"(x), "r"(y), "r"(z), "r"(s)
               : "memory");
}

// 1/b of the Van Albada limiter quotient.  Default: the ~1 ulp reciprocal
// (frcp).  -DBF_VA_RCP1: MUFU seed (~2^-22) and one Newton step (~2^-44
// relative), 2.9% faster on C4 but its error, (error) x (eps/4) x D in the
// face states, shifts long runs: C1 FAST vs EXACT after 250 / 1000 / 2000
// steps 1.3e-12 / 1.0e-11 / 1.1e-11 of the freestream pressure, against
// 9.6e-14 / 7.2e-13 / 1.8e-12 with frcp (profiles/r02_fast_drift_c1.jsonl).
BF_DEV double frcp1(double b) {
#ifndef BF_VA_RCP1
  return frcp(b);
#endif
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  return fma(r, fma(-b, r, 1.0), r);
}

// a / b with a single-Newton reciprocal and one quotient correction (~1 ulp)
BF_DEV double fdiv1(double a, double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  r = fma(r, fma(-b, r, 1.0), r);
  const double q = a * r;
  return fma(fma(-b, q, a), r, q);
}

// max(x, 0) on the bit pattern (sign mask): three integer ops instead of the
// DSETP/FSEL/SEL/LOP3 sequence of fmax's NaN handling
BF_DEV double dpos(double x) {
  const int hi = __double2hiint(x);
  const int m = ~(hi >> 31);
  return __hiloint2double(hi & m, __double2loint(x) & m);
}

// Positivity pre-filter on the high words: a double x <= 0 has hi(x) <= 0 as a
// signed int (sign bit set, or +0); the converse only adds values below 2^-1042.
// Integer min on the high halves keeps the common case off the fp64 pipe; the
// exact double comparisons run only when the filter fires.
BF_DEV bool maybe_nonpos(double a, double b, double c, double d) {
  return min(min(__double2hiint(a), __double2hiint(b)), min(__double2hiint(c), __double2hiint(d))) <= 0;
}

template <int LIM>
BF_DEV double vl_limiter(double a, double b) {
  if constexpr (LIM == LIM_NONE) {
    return 1.0;
  } else if constexpr (LIM == LIM_VAN_ALBADA) {
    // denominator > 0: max(num, 0) / den == max(num / den, 0)
    return fdiv1(dpos(fma(2.0 * a, b, 1e-12)), fma(a, a, fma(b, b, 1e-12)));
  } else if constexpr (LIM == LIM_MINMOD) {
    const double r = fdiv1(a, b);
    return (a * b > 0.0) ? ((1.0 <= r) ? 1.0 : r) : 0.0;
  } else {
    const double r = fdiv1(a, b);
    const double val = fdiv1(2.0 * r, 1.0 + r);
    return (a * b > 0.0) ? val : 0.0;
  }
}

// Both MUSCL states of one cell from its stencil (wm, w0, wp) along a direction:
// qL at the cell's high face, qR at its low face.  K1: eps = 1, kappa = -1.
template <int LIM, bool K1>
BF_DEV void vl_recon(double wm, double w0, double wp, const Consts& c, double& qL, double& qR) {
  const double dm = w0 - wm, dp = wp - w0;
  if constexpr (K1 && LIM == LIM_VAN_ALBADA) {
    // (eps/4)(1-k) Psi = Psi/2 = (ab + 1e-12/2) / (a^2 + b^2 + 1e-12), a = D+, b = D-
    // (the denominator is positive, so max(num, 0) * (1/den) == max(num/den, 0))
    const double t = dpos(fma(dp, dm, c.lim_eps_half)) * frcp1(fma(dp, dp, fma(dm, dm, c.lim_eps)));
    qL = fma(t, dm, w0);
    qR = fma(-t, dp, w0);
    return;
  }
  const double pp = vl_limiter<LIM>(dp, dm);
  const double pm = (psi_count<LIM>() == 2) ? vl_limiter<LIM>(dm, dp) : pp;
  if constexpr (K1) {
    qL = fma(0.5 * pp, dm, w0);
    qR = fma(-0.5 * pm, dp, w0);
  } else {
    qL = w0 + c.quarter * fma(c.omk * pp, dm, c.opk * pm * dp);
    qR = w0 - c.quarter * fma(c.opk * pp, dm, c.omk * pm * dp);
  }
}

// One side of the Van Leer splitting (physics.py:267-290) times the face area:
// vl_sub is the subsonic form, valid as arithmetic for any state; vl_super
// replaces it where |M| >= 1.  Subsonic test |vn| / a < 1 as vn^2 rho < g p
// (the branch condition does not wait for the reciprocal square root; the two
// forms agree at |M| = 1).
BF_DEV bool vl_subsonic(const double q[5], double nx, double ny, double nz, const Consts& c) {
  const double vn = fma(q[1], nx, fma(q[2], ny, q[3] * nz));
  return vn * vn * q[0] < c.gamma * q[4];
}

// y = 1/sqrt(g p rho) of a state: a = g p y and 1/a = rho y
BF_DEV double vl_rsq(const double q[5], const Consts& c) { return frsqrt(c.gamma * q[4] * q[0]); }

BF_DEV void vl_sub(const double q[5], double y, double nx, double ny, double nz, double A,
                   double sign, const Consts& c, double F[5]) {
  const double gp = c.gamma * q[4];
  const double a = gp * y;
  const double ainv = q[0] * y;
  const double vn = fma(q[1], nx, fma(q[2], ny, q[3] * nz));
  const double mn = vn * ainv;
  const double sh = mn + sign;
  const double fm = q[0] * (a * ((0.25 * sign) * A)) * (sh * sh);
  const double ta = (2.0 * sign) * a;
  const double et = fma(c.gm1, vn, ta);
  const double fac = (ta - vn) * c.inv_gamma;
  // e = et^2 / (2 (g^2-1)) + ke - vn^2 / 2
  const double s2 = fma(q[1], q[1], fma(q[2], q[2], fma(q[3], q[3], -vn * vn)));
  const double ee = fma(et * et, c.inv_vlc, 0.5 * s2);
  F[0] = fm;
  F[1] = fm * fma(nx, fac, q[1]);
  F[2] = fm * fma(ny, fac, q[2]);
  F[3] = fm * fma(nz, fac, q[3]);
  F[4] = fm * ee;
}

BF_DEV void vl_super(const double q[5], double nx, double ny, double nz, double A,
                     double sign, const Consts& c, double F[5]) {
  const double vn = fma(q[1], nx, fma(q[2], ny, q[3] * nz));
  if (sign * vn > 0.0) {   // the whole flux goes to this side
    const double m = q[0] * vn * A;
    const double pA = q[4] * A;
    F[0] = m;
    F[1] = fma(m, q[1], nx * pA);
    F[2] = fma(m, q[2], ny * pA);
    F[3] = fma(m, q[3], nz * pA);
    const double ke = 0.5 * fma(q[1], q[1], fma(q[2], q[2], q[3] * q[3]));
    F[4] = m * fma(c.gog1 * q[4], frcp(q[0]), ke);
  } else {
    F[0] = F[1] = F[2] = F[3] = F[4] = 0.0;
  }
}

BF_DEV void vl_half(const double q[5], double nx, double ny, double nz, double A, double sign,
                    const Consts& c, double F[5]) {
  vl_sub(q, vl_rsq(q, c), nx, ny, nz, A, sign, c, F);
  if (!vl_subsonic(q, nx, ny, nz, c)) vl_super(q, nx, ny, nz, A, sign, c, F);
}

// F+ of the high face (state qp, geometry gp) and F- of the low face (qm, gm)
// of one cell, gp/gm = {nx, ny, nz, A} at stride gs.  The two reciprocal
// square roots go first (two independent MUFU + refinement chains: 1.137 ->
// 1.099 ms); computing both whole subsonic forms as one straight-line block
// with a joint fallback measured slower (register pressure).
BF_DEV void vl_pair(const double qp[5], const double* gp, const double qm[5], const double* gm,
                    int gs, const Consts& c, double Fp[5], double Fm[5]) {
  // both reciprocal square roots first: two independent MUFU + refinement chains
  const double yp = vl_rsq(qp, c), ym = vl_rsq(qm, c);
  vl_sub(qp, yp, gp[0], gp[gs], gp[2 * gs], gp[3 * gs], 1.0, c, Fp);
  if (!vl_subsonic(qp, gp[0], gp[gs], gp[2 * gs], c))
    vl_super(qp, gp[0], gp[gs], gp[2 * gs], gp[3 * gs], 1.0, c, Fp);
  vl_sub(qm, ym, gm[0], gm[gs], gm[2 * gs], gm[3 * gs], -1.0, c, Fm);
  if (!vl_subsonic(qm, gm[0], gm[gs], gm[2 * gs], c))
    vl_super(qm, gm[0], gm[gs], gm[2 * gs], gm[3 * gs], -1.0, c, Fm);
}

// local-time-step term (solver.py:709-716) of one face
// sound speed sqrt(g p / rho) = g p / sqrt(g p rho): one reciprocal square root
BF_DEV double sound_speed(double rho, double p, const Consts& c) {
  const double gp = c.gamma * p;
  return gp * frsqrt(gp * rho);
}

BF_DEV double lam_term(double u, double v, double w, double snd, double nx, double ny, double nz,
                       double A) {
  return (fabs(fma(u, nx, fma(v, ny, w * nz))) + snd) * A;
}

// Ghost push (PushRule, bf_internal.h): cell (i, j, k) got its new state
// (r, u, v, w, p) in W[cur ^ 1]; write every ghost value of W[cur ^ 1] that the
// next ghost update would derive from this cell.  Rare (cells within `g`
// layers of a face) and kept out of line; the block's rules sit in shared
// memory and the block scalars come by value, so a call has no global-load
// dependency chain before its stores.
struct PushSmem {
  int range[6][2];
  PushRule rules[PUSH_MAX_RULES];
};

__device__ __noinline__ void push_ghosts(const PushSmem* ps, double* base, long long sy,
                                         long long sz, long long fsz, int n0, int n1, int n2,
                                         int g, int ndim, int out, const Consts& c, int i, int j,
                                         int k, double r, double u, double v, double w,
                                         double p) {
  const double T = BF_DIV(p, r * c.R);
  const int cell[3] = {i, j, k};
  const int nn[3] = {n0, n1, n2};
  const long long st[3] = {1, sy, sz};
  const long long o = i + sy * (long long)j + sz * (long long)k;
  double* const W = base + (long long)fw(out, 0) * fsz;
  for (int f = 0; f < 2 * ndim; ++f) {
    const int ax = f >> 1, side = f & 1;
    const int n = nn[ax], co = cell[ax];
    if (side == 0 ? co >= g : co < n - g) continue;
    for (int q = ps->range[f][0]; q < ps->range[f][1]; ++q) {
      const PushRule& R = ps->rules[q];
      if (i < R.lo[0] || i >= R.hi[0] || j < R.lo[1] || j >= R.hi[1] || k < R.lo[2] ||
          k >= R.hi[2])
        continue;
      if (R.kind == PK_COPY || R.kind == PK_PACK) {
        const long long d = R.base + (long long)(i - R.lo[0]) * R.coef[0] +
                            (long long)(j - R.lo[1]) * R.coef[1] +
                            (long long)(k - R.lo[2]) * R.coef[2];
        const long long fs = R.dst_fsz;
        if (R.kind == PK_COPY) {   // partner block's ghosts (halo.py:70-106)
          double* D = R.dst + (long long)fw(out, 0) * fs;
          D[d] = r;
          D[fs + d] = u;
          D[2 * fs + d] = v;
          if (R.nfields == 6) D[3 * fs + d] = w;
          D[4 * fs + d] = p;
          D[5 * fs + d] = T;
        } else {                   // message buffer (halo.py:47-67), fields packed in order
          double* B = R.dst;
          int e = 0;
          B[(e++) * fs + d] = r;
          B[(e++) * fs + d] = u;
          B[(e++) * fs + d] = v;
          if (R.nfields == 6) B[(e++) * fs + d] = w;
          B[(e++) * fs + d] = p;
          B[(e++) * fs + d] = T;
        }
        continue;
      }
      // physical patch (solver.py:281-403): ghost layer L sits at -1-L / n+L
      const int layer = side == 0 ? co : n - 1 - co;
      auto gofs = [&](int L) { return o + (long long)((side == 0 ? -1 - L : n + L) - co) * st[ax]; };
      auto put = [&](long long og, double r_, double u_, double v_, double w_, double p_,
                     double T_) {
        W[og] = r_;
        W[fsz + og] = u_;
        W[2 * fsz + og] = v_;
        W[3 * fsz + og] = w_;
        W[4 * fsz + og] = p_;
        W[5 * fsz + og] = T_;
      };
      if (R.kind == PK_OUTFLOW) {
        for (int L = 0; L < g; ++L) put(gofs(L), r, u, v, w, p, T);
        continue;
      }
      // outward unit normal of the boundary face at this tangential position
      const long long fo = o + (long long)((side == 0 ? 0 : n) - co) * st[ax];
      const double sg = side == 0 ? -1.0 : 1.0;
      const double* fn = base + (long long)ffn(ax, 0) * fsz + fo;
      const double nx = sg * fn[0], ny = sg * fn[fsz], nz = sg * fn[2 * fsz];
      if (R.kind == PK_FARFIELD) {
        const St qb = farfield_state(St{r, u, v, w, p}, nx, ny, nz, c);
        const double tb = qb.p / (qb.r * c.R);
        for (int L = 0; L < g; ++L) put(gofs(L), qb.r, qb.u, qb.v, qb.w, qb.p, tb);
        continue;
      }
      double ug, vg, wg;
      if (R.kind == PK_SLIP) {
        const double vn = u * nx + v * ny + w * nz;
        ug = u - 2.0 * vn * nx;
        vg = v - 2.0 * vn * ny;
        wg = w - 2.0 * vn * nz;
      } else {
        ug = -u;
        vg = -v;
        wg = -w;
      }
      const double tg = (R.kind == PK_NOSLIP && c.has_tw) ? 2.0 * c.tw - T : T;
      put(gofs(layer), p / (c.R * tg), ug, vg, wg, p, tg);
    }
  }
}

template <int NDIM, int LIM>
struct VCfg {
  static constexpr int TJ = Cfg<NDIM, LIM>::TJ;   // same tiles as the reference-order kernel
  static constexpr int NT = TI * TJ;
  static constexpr int PW = TI + 2 * HALO;
  static constexpr int PH = TJ + 2 * HALO;
  static constexpr int PLANE = PW * PH;
  static constexpr int NS = (NDIM == 3) ? NSLOT : 1;
  static constexpr int NFX = GXW * TJ;             // x geometry [4][TJ][GXW]
  static constexpr int NFY = TI * (TJ + 1);        // y geometry [4][TJ+1][TI]
  static constexpr int NHY = TI * (TJ + 1);        // y halves  [5][TJ+1][TI]
  static constexpr int NH = 2 * TJ + 2 * TI;       // tile-edge half-flux items per plane
  static constexpr int r16(int x) { return (x + 15) / 16 * 16; }
  static constexpr int OW = 0;
  static constexpr int OHP = r16(OW + NS * 5 * PLANE);   // F+_y of rows -1..TJ-1 (index row+1)
  static constexpr int OHM = r16(OHP + 5 * NHY);         // F-_y of rows 0..TJ   (index row)
  static constexpr int OXH = r16(OHM + 5 * NHY);         // [2][5][TJ]: F+ of cell -1, F- of cell TI
  static constexpr int OFX = r16(OXH + 10 * TJ);
  static constexpr int OFY = r16(OFX + 4 * NFX);
  static constexpr int OZG = r16(OFY + 4 * NFY);         // [2][4][TJ][TI] z faces (3D)
  // 2 CTAs per SM (TJ <= 8, 3D): Q0 / dt/V are read from L2 (prefetched) instead
  // of staged, to fit two CTAs' shared memory
  static constexpr bool QLDG = NDIM == 3 && TJ <= 8;
  // 2D: one plane per CTA, latency-bound: several CTAs per SM (register cap)
  static constexpr int MINB = QLDG ? 2 : (NDIM == 2 ? BF_VL2D_MINB : 1);
  static constexpr int OQ = r16(OZG + (NDIM == 3 ? 8 * NT : 0));   // [6][TJ][TI] Q0, dt/V
  static constexpr int OPS = r16(OQ + (QLDG ? 5 * (NT / 32) : 6 * NT));   // PushSmem
  static constexpr int OBAR = r16(OPS + (BF_VL_PUSH ? (int)((sizeof(PushSmem) + 7) / 8) : 0));
  static constexpr int OBLK = OBAR + 8;                  // the tile's DevBlock (BF_VL_SMEM_BLOCK)
  static constexpr int TOTAL = OBLK + (int)(sizeof(DevBlock) + 7) / 8;
  static constexpr size_t BYTES = sizeof(double) * TOTAL;
  static constexpr unsigned WBYTES = 5u * PLANE * 8u;
  static constexpr unsigned GYZBYTES = (4u * NFY + (NDIM == 3 ? 4u * NT : 0u)) * 8u;
  static constexpr unsigned GXBYTES = 4u * NFX * 8u;
  BF_DEV static int pidx(int ii, int jj) { return (jj + HALO) * PW + (ii + HALO); }
};

template <int NDIM, int LIM, bool K1, bool S0>
__global__ void __launch_bounds__(VCfg<NDIM, LIM>::NT, VCfg<NDIM, LIM>::MINB) vl_stage_kernel(const __grid_constant__ StageArgs a) {
  pdl_trigger();   // the next kernel may be dispatched (it waits in pdl_wait for this one)
  using K = VCfg<NDIM, LIM>;
  constexpr int NT = K::NT, TJ = K::TJ, PLANE = K::PLANE, PW = K::PW;
  extern __shared__ __align__(128) double smem[];
  // fused ghost fill (StageArgs::fill_chunks): fill-only CTAs first, then the
  // tiles — interior first; the boundary tiles wait for the whole fill
  const bool fused = a.fill_chunks > 0;
  const int nworkers = a.fill_ctas * (NT / 32);
  const unsigned parties = (unsigned)(nworkers + a.ntiles - a.n_interior);
  if (fused && (int)blockIdx.x < a.fill_ctas) {
    pdl_wait();
    if (a.stop && *a.stop) return;   // batched iterate stopped (RunState)
    fill_work(a.fill, a.fill_chunks, (int)(blockIdx.x * (NT / 32) + threadIdx.x / 32), nworkers,
              a.fill_sync, parties, reinterpret_cast<GhostTask*>(smem) + threadIdx.x / 32);
    return;
  }
  const int cta = fused ? (int)blockIdx.x - a.fill_ctas : (int)blockIdx.x;
  const bool wait_fill = fused && cta >= a.n_interior;
  constexpr int NFX = K::NFX, NFY = K::NFY, NHY = K::NHY;
  double* const sW = smem + K::OW;
  double* const sHP = smem + K::OHP;
  double* const sHM = smem + K::OHM;
  double* const sXH = smem + K::OXH;
  double* const sFX = smem + K::OFX;
  double* const sFY = smem + K::OFY;
  double* const sZG = smem + K::OZG;
  double* const sQ = smem + K::OQ;
  unsigned long long* const bars = reinterpret_cast<unsigned long long*>(smem + K::OBAR);
  PushSmem* const sPS = reinterpret_cast<PushSmem*>(smem + K::OPS);
  // bars[0..2]: plane ring, bars[3]: geometry group, bars[4]: Q0 / dt group

  const int tile_id = a.tile_list ? a.tile_list[cta] : cta;
  const Tile t = a.tiles[tile_id];
#if BF_VL_SMEM_BLOCK
  // the block record in shared memory: its fields are re-read with LDS instead
  // of being held in registers across the k loop (or spilled to local memory)
  DevBlock* const sBk = reinterpret_cast<DevBlock*>(smem + K::OBLK);
  if (threadIdx.x < sizeof(DevBlock) / 8)
    reinterpret_cast<unsigned long long*>(sBk)[threadIdx.x] =
        reinterpret_cast<const unsigned long long*>(a.blocks + t.block)[threadIdx.x];
  __syncthreads();
  const DevBlock& b = *sBk;
#else
  const DevBlock b = a.blocks[t.block];
#endif
  const Consts& c = a.c;
  const unsigned char* const tm = a.tmaps + (size_t)t.block * NTMAP * 128;
  const int tid = threadIdx.x;
  const int tx = tid % TI, ty = tid / TI;
  const int i0 = t.i0, j0 = t.j0, k0 = t.k0, kc = t.kc;
  const int ni = b.n[0], nj = b.n[1], nk = (NDIM == 3) ? b.n[2] : 1;
  const long long sy = b.sy, sz = b.sz, fsz = b.fsz;
  const int i = i0 + tx, j = j0 + ty;
  const bool in_i = i < ni, in_j = j < nj;
  const bool cell_on = in_i && in_j;
  const int flags = a.flags;
  constexpr bool stage0 = S0;   // first RK stage: dt/V and sum(R^2)
  const bool last = flags & F_LAST;
  const int stage = a.stage;
  const double* const Win = b.base + (long long)fw(a.cur, 0) * fsz;
  double* const Wout = b.base + (long long)fw(a.cur ^ 1, 0) * fsz;
  const long long colofs = i + sy * (long long)j;
  const int s0 = K::pidx(tx, ty);
  const unsigned FULL = 0xffffffffu;

  auto slot_of = [&](int k) -> double* {
    if constexpr (NDIM == 3) return sW + ((k - k0) % NSLOT) * 5 * PLANE;
    else return sW;
  };
  auto bar_of = [&](int k) { return bars + ((NDIM == 3) ? (k - k0) % NSLOT : 0); };
  auto par_of = [&](int k) { return (unsigned)(((NDIM == 3) ? (k - k0) / NSLOT : 0) & 1); };
  auto zslot = [&](int face) -> double* {   // z face `face` lives in slot (face - k0) & 1
    return sZG + ((face - k0) & 1) * 4 * NT;
  };

  auto issue_plane = [&](int k) {
    unsigned long long* bar = bar_of(k);
    mbar_expect_tx(bar, K::WBYTES);
    tma_load4(slot_of(k), tm + 0 * 128, b.ox + i0 - HALO, b.oy + j0 - HALO,
              (NDIM == 3) ? b.oz + k : 0, fw(a.cur, 0), bar);
  };
  auto issue_geo_yz = [&](int k) {   // y face geometry of plane k, z face k+2 (phase A)
    unsigned long long* bar = bars + 3;
    const int z = (NDIM == 3) ? b.oz + k : 0;
    mbar_expect_tx(bar, K::GYZBYTES);
    tma_load4(sFY, tm + 2 * 128, b.ox + i0, b.oy + j0, z, ffn(1, 0), bar);
    if constexpr (NDIM == 3) tma_load4(zslot(k + 2), tm + 5 * 128, b.ox + i0, b.oy + j0, z + 2,
                                       ffn(2, 0), bar);
  };
  auto issue_b = [&](int k) {        // x face geometry, Q0 (and dt/V) of plane k (phase B)
    unsigned long long* bar = bars + 4;
    const int z = (NDIM == 3) ? b.oz + k : 0;
    if constexpr (K::QLDG) {
      mbar_expect_tx(bar, K::GXBYTES);
      tma_load4(sFX, tm + 1 * 128, b.ox + i0, b.oy + j0, z, ffn(0, 0), bar);
      tma_prefetch4(tm + 3 * 128, b.ox + i0, b.oy + j0, z, FQ);
      if (!stage0) tma_prefetch4(tm + 4 * 128, b.ox + i0, b.oy + j0, z, FDTV);
    } else {
      mbar_expect_tx(bar, K::GXBYTES + (stage0 ? 5u : 6u) * NT * 8u);
      tma_load4(sFX, tm + 1 * 128, b.ox + i0, b.oy + j0, z, ffn(0, 0), bar);
      tma_load4(sQ, tm + 3 * 128, b.ox + i0, b.oy + j0, z, FQ, bar);
      if (!stage0) tma_load4(sQ + 5 * NT, tm + 4 * 128, b.ox + i0, b.oy + j0, z, FDTV, bar);
    }
  };
  auto prefetch_l2 = [&](int k) {    // geometry and Q0 of plane k into L2
    const int z = (NDIM == 3) ? b.oz + k : 0;
    tma_prefetch4(tm + 1 * 128, b.ox + i0, b.oy + j0, z, ffn(0, 0));
    tma_prefetch4(tm + 2 * 128, b.ox + i0, b.oy + j0, z, ffn(1, 0));
    if constexpr (NDIM == 3) tma_prefetch4(tm + 5 * 128, b.ox + i0, b.oy + j0, z + 2, ffn(2, 0));
    tma_prefetch4(tm + 3 * 128, b.ox + i0, b.oy + j0, z, FQ);
  };

  auto face_err = [&](int d, int kind, unsigned long long lin) {
    record_error(a.err, make_err_key(stage, 0, b.order, d, kind, lin));
  };
  // C-order linear face index of the reference's face arrays (solver.py:501-506)
  auto lin_x = [&](int f, int jj, int k) {
    return ((unsigned long long)f * nj + jj) * (unsigned long long)nk + (NDIM == 3 ? k : 0);
  };
  auto lin_y = [&](int ii, int f, int k) {
    return ((unsigned long long)ii * (nj + 1) + f) * (unsigned long long)nk + (NDIM == 3 ? k : 0);
  };
  auto lin_z = [&](int ii, int jj, int f) {
    return ((unsigned long long)ii * nj + jj) * (unsigned long long)(nk + 1) + f;
  };
  // wall / farfield flux of a boundary face (solver.py:526-580); wv[0..3] are
  // the var-0 pointers of cells f-2..f+1 (stride vs)
  // wall / farfield flux (times A) of a boundary face (solver.py:526-580).
  // in1 / in2: first / second interior cell, gh: the ghost cell across the
  // face.  For a farfield patch the ghost fill already stored
  // farfield_state(in1, outward n) in every ghost layer (solver.py:138-171,
  // ghost_kernel BC_FARFIELD), so the overwrite flux is its Euler flux.
  auto overwrite = [&](int bk, const double* in1, const double* in2, const double* gh, int vs,
                       const double* g, int gs, double F[5]) {
    const double nx = g[0], ny = g[gs], nz = g[2 * gs], A = g[3 * gs];
    if (bk == BFACE_WALL) {
      const double pw = fma(1.5, in1[4 * vs], -0.5 * in2[4 * vs]) * A;
      F[0] = 0.0;
      F[1] = nx * pw;
      F[2] = ny * pw;
      F[3] = nz * pw;
      F[4] = 0.0;
    } else {
      const St q{gh[0], gh[vs], gh[2 * vs], gh[3 * vs], gh[4 * vs]};
      euler_flux(q, nx, ny, nz, c, F);
#pragma unroll
      for (int e = 0; e < 5; ++e) F[e] = F[e] * A;
    }
  };

  // ---- state carried along k (3D) ---------------------------------------------------
  double hpz[5] = {0, 0, 0, 0, 0};   // F+_z of cell k (times A_{k+1/2})
  double fzl[5] = {0, 0, 0, 0, 0};   // z flux of face k (times A), the low face of cell k
  double lamz = 0.0;                 // z part of the stage-0 lambda of cell k
  double rsum[5] = {0.0, 0.0, 0.0, 0.0, 0.0};

  // static tables (tile, block, tensor maps) are read before the wait: up to
  // here the CTA overlaps the previous kernel's drain
  if (tid < NTMAP) asm volatile("prefetch.tensormap [%0];" ::"l"(tm + tid * 128) : "memory");
  pdl_wait();                      // the previous kernel's writes are complete and visible
  if (a.stop && *a.stop) return;   // batched iterate stopped (RunState)
  if (tid == 0) {
    for (int q = 0; q < 5; ++q) mbar_init(bars + q, 1);
    fence_mbar_init();
    if (wait_fill) {   // the fill workers' ghost stores, published by the barrier below
      fill_wait(a.fill_sync, nworkers);
      fill_arrive(a.fill_sync, 1u, parties);
    }
  }
  if (BF_VL_PUSH && a.push) {   // this block's ghost-push rules -> shared memory
    const int* rg = a.push_range + t.block * 12;
    const int r0 = rg[0], r1 = rg[11];
    if (tid < 12) (&sPS->range[0][0])[tid] = rg[tid] - r0;
    constexpr int RW = (int)(sizeof(PushRule) / 8);
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(a.push_rules + r0);
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(sPS->rules);
    for (int q = tid; q < (r1 - r0) * RW; q += NT) dst[q] = src[q];
  }
  __syncthreads();
  if (tid == 0) {
    if constexpr (NDIM == 3) {
      issue_plane(k0);
      issue_plane(k0 + 1);
      issue_plane(k0 + 2);
    } else {
      issue_plane(0);
    }
    issue_geo_yz(k0);
  }

  // z half fluxes of cell kc (own column): w[0..2] = W(kc-1), W(kc), W(kc+1);
  // glo / ghi: geometry of faces kc, kc+1 (stride gs)
  auto z_halves = [&](int kcell, const double wa[5], const double wb[5], const double wc[5],
                      const double* glo, const double* ghi, int gs, double hp[5], double hm[5],
                      bool want_hp) {
    double qL[5], qR[5];
#pragma unroll
    for (int v = 0; v < 5; ++v) vl_recon<LIM, K1>(wa[v], wb[v], wc[v], c, qL[v], qR[v]);
    vl_pair(qL, ghi, qR, glo, gs, c, hp, hm);
    if (maybe_nonpos(qL[0], qL[4], qR[0], qR[4])) {
      const bool bL = (qL[0] <= 0.0) | (qL[4] <= 0.0), bR = (qR[0] <= 0.0) | (qR[4] <= 0.0);
      // qL belongs to face kcell+1 (valid while kcell <= nk-1), qR to face kcell
      if (want_hp && bL && kcell <= nk - 1) face_err(2, ERR_FACE_LEFT, lin_z(i, j, kcell + 1));
      if (bR && kcell >= 0) face_err(2, ERR_FACE_RIGHT, lin_z(i, j, kcell));
    }
  };

  if constexpr (NDIM == 3) {
    // ---- prologue: F+_z(k0-1), F-_z(k0), F+_z(k0), z flux of face k0 ----------------
    double wa[5], wb[5], wc[5], wd[5];
    double g0[4] = {0, 0, 0, 0}, g1[4] = {0, 0, 0, 0};
    if (cell_on) {
      const long long o = colofs + sz * (long long)(k0 - 2);
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        wa[v] = Win[v * fsz + o];
        wb[v] = Win[v * fsz + o + sz];
      }
      const double* fn = b.base + (long long)ffn(2, 0) * fsz + colofs + sz * (long long)k0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        g0[q] = __ldg(fn + q * fsz);
        g1[q] = __ldg(fn + q * fsz + sz);
      }
    }
    // face k0+1 geometry for iteration 0 (slot of face k0+1)
#pragma unroll
    for (int q = 0; q < 4; ++q) zslot(k0 + 1)[q * NT + tid] = g1[q];
    mbar_wait(bar_of(k0), par_of(k0));
    mbar_wait(bar_of(k0 + 1), par_of(k0 + 1));
    if (cell_on) {
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        wc[v] = slot_of(k0)[v * PLANE + s0];
        wd[v] = slot_of(k0 + 1)[v * PLANE + s0];
      }
      double hp_prev[5], hm0[5];
      {   // cell k0-1: only its F+ (face k0) is needed
        double qL[5], qR[5];
#pragma unroll
        for (int v = 0; v < 5; ++v) vl_recon<LIM, K1>(wa[v], wb[v], wc[v], c, qL[v], qR[v]);
        vl_half(qL, g0[0], g0[1], g0[2], g0[3], 1.0, c, hp_prev);
        if ((qL[0] <= 0.0) | (qL[4] <= 0.0)) face_err(2, ERR_FACE_LEFT, lin_z(i, j, k0));
      }
      z_halves(k0, wb, wc, wd, g0, g1, 1, hpz, hm0, true);
#pragma unroll
      for (int v = 0; v < 5; ++v) fzl[v] = hp_prev[v] + hm0[v];
      if (k0 == 0) {
        const int bk = b.bface[4][i + ni * j];
        if (bk != BFACE_NONE) {
          overwrite(bk, wc, wd, wb, 1, g0, 1, fzl);
        }
      }
      if (stage0) {
        const double snd = sound_speed(wc[0], wc[4], c);
        lamz = lam_term(wc[1], wc[2], wc[3], snd, g0[0], g0[1], g0[2], g0[3]) +
               lam_term(wc[1], wc[2], wc[3], snd, g1[0], g1[1], g1[2], g1[3]);
      }
    }
  }

  for (int kk = 0; kk < kc; ++kk) {
    const int k = k0 + kk;
    const long long kofs = (NDIM == 3) ? sz * (long long)k : 0;
    const double* const pk = slot_of(k);
    const double* const w = pk + s0;

    // boundary-face kinds of this cell's x / y faces (2 bits each: x lo, x hi,
    // y lo, y hi), loaded ahead of the B0 barrier so phase A hides the latency
    unsigned bfk = 0;
    {
      const int kz = (NDIM == 3) ? k : 0;
      if (in_j && i == 0) bfk = b.bface[0][j + nj * kz];
      if (in_j && i == ni - 1) bfk |= (unsigned)b.bface[1][j + nj * kz] << 2;
      if (in_i && j == 0) bfk |= (unsigned)b.bface[2][i + ni * kz] << 4;
      if (in_i && j == nj - 1) bfk |= (unsigned)b.bface[3][i + ni * kz] << 6;
    }
    __syncthreads();   // B0: plane k-1 retired (its ring slot, x geometry, y halves, Q0)
    if (tid == 0) {
      fence_async_smem();
      issue_b(k);
      if constexpr (NDIM == 3) {
        if (kk > 0) issue_plane(k + 2);   // into the slot of plane k-1
        // plane k+3 into L2 now, so next iteration's TMA of it is an L2 hit
        if (kk + 1 < kc)
          tma_prefetch4(tm, b.ox + i0 - HALO, b.oy + j0 - HALO, b.oz + k + 3, fw(a.cur, 0));
      }
    }
    mbar_wait(bars + 3, (unsigned)(kk & 1));
    mbar_wait(bar_of(k), par_of(k));

    // ---- phase A1: tile-edge half fluxes ----------------------------------------------
#ifndef BF_ABLATE_HALO
#define BF_ABLATE_HALO 0
#endif
    // tile-edge items on the LAST warps: warp 0 also issues the TMA groups
    if (!BF_ABLATE_HALO && tid >= NT - K::NH) {
      const int h = tid - (NT - K::NH);
      int cx, cy, st, d, fo;
      double sg;
      double g[4];
      double* out;
      int os;
      bool valid;
      unsigned long long lin;
      if (h < 2 * TJ) {   // x: F+ of cell -1 (face i0), F- of cell TI (face i0+TI)
        const int row = h % TJ, hi = h / TJ;
        cx = hi ? TI : -1;
        cy = row;
        st = 1;
        d = 0;
        sg = hi ? -1.0 : 1.0;
        fo = hi ? TI : 0;
        out = sXH + hi * 5 * TJ + row;
        os = TJ;
        valid = (j0 + row < nj) && (i0 + fo <= ni);
        lin = lin_x(i0 + fo, j0 + row, k);
        // x geometry of plane k is staged only for phase B: read these two faces directly
        const double* fn =
            b.base + (long long)ffn(0, 0) * fsz + (i0 + fo) + sy * (long long)(j0 + row) + kofs;
#pragma unroll
        for (int q = 0; q < 4; ++q) g[q] = valid ? __ldg(fn + q * fsz) : 0.0;
      } else {            // y: F+ of row -1 (face j0), F- of row TJ (face j0+TJ)
        const int e = h - 2 * TJ;
        const int col = e % TI, hi = e / TI;
        cx = col;
        cy = hi ? TJ : -1;
        st = PW;
        d = 1;
        sg = hi ? -1.0 : 1.0;
        fo = hi ? TJ : 0;
        out = hi ? sHM + TJ * TI + col : sHP + col;
        os = NHY;
        valid = (i0 + col < ni) && (j0 + fo <= nj);
        lin = lin_y(i0 + col, j0 + fo, k);
        const double* gy = sFY + fo * TI + col;
#pragma unroll
        for (int q = 0; q < 4; ++q) g[q] = gy[q * NFY];
      }
      const double* wh = pk + K::pidx(cx, cy);
      double q5[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        const double wm = wh[v * PLANE - st], w0 = wh[v * PLANE], wp = wh[v * PLANE + st];
        if constexpr (K1 && LIM == LIM_VAN_ALBADA) {   // only the side this item needs
          const double dm = w0 - wm, dp = wp - w0;
          const double t =
              dpos(fma(dp, dm, c.lim_eps_half)) * frcp1(fma(dp, dp, fma(dm, dm, c.lim_eps)));
          q5[v] = fma(t, sg > 0.0 ? dm : -dp, w0);
        } else {
          double qL, qR;
          vl_recon<LIM, K1>(wm, w0, wp, c, qL, qR);
          q5[v] = sg > 0.0 ? qL : qR;
        }
      }
      double F[5];
      vl_half(q5, g[0], g[1], g[2], g[3], sg, c, F);
#pragma unroll
      for (int v = 0; v < 5; ++v) out[v * os] = F[v];
      if (valid && maybe_nonpos(q5[0], q5[4], q5[0], q5[4]) && ((q5[0] <= 0.0) | (q5[4] <= 0.0)))
        face_err(d, sg > 0.0 ? ERR_FACE_LEFT : ERR_FACE_RIGHT, lin);
    }

    // ---- phase A2: y halves -> shared memory -------------------------------------------
    // residual (face fluxes already times A); the y part is split as
    //   (F+_j - F-_j) [own halves, here] + F-_{j+1} - F+_{j-1} [neighbours, phase B2]
    double R[5];
    bool ylo_ovw = false, yhi_ovw = false;
    double lam = 0.0;   // stage 0: y and z parts of lambda of cell k
    double snd = 0.0;   // stage 0: sound speed of cell k (phases A2 and B1)
    {
      double qL[5], qR[5];
#pragma unroll
      for (int v = 0; v < 5; ++v)
        vl_recon<LIM, K1>(w[v * PLANE - PW], w[v * PLANE], w[v * PLANE + PW], c, qL[v], qR[v]);
      const double* gl = sFY + ty * TI + tx;   // face j (low); face j+1 at gl + TI
      double hp[5], hm[5];
      vl_pair(qL, gl + TI, qR, gl, NFY, c, hp, hm);
      if (maybe_nonpos(qL[0], qL[4], qR[0], qR[4]) && in_i) {
        const bool bL = (qL[0] <= 0.0) | (qL[4] <= 0.0), bR = (qR[0] <= 0.0) | (qR[4] <= 0.0);
        if (bL && in_j) face_err(1, ERR_FACE_LEFT, lin_y(i, j + 1, k));
        if (bR && j <= nj) face_err(1, ERR_FACE_RIGHT, lin_y(i, j, k));
      }
      if (in_i && (j == 0 || j == nj - 1)) {
        if (j == 0) {   // whole face flux into the F- slot; phase B drops the F+ half
          const int bk = (bfk >> 4) & 3u;
          if (bk != BFACE_NONE) {
            overwrite(bk, w, w + PW, w - PW, PLANE, gl, NFY, hm);
            ylo_ovw = true;
          }
        }
        if (j == nj - 1) {   // whole face flux into the F+ slot
          const int bk = (bfk >> 6) & 3u;
          if (bk != BFACE_NONE) {
            overwrite(bk, w, w - PW, w + PW, PLANE, gl + TI, NFY, hp);
            yhi_ovw = true;
          }
        }
      }
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        sHP[v * NHY + (ty + 1) * TI + tx] = hp[v];
        sHM[v * NHY + ty * TI + tx] = hm[v];
        R[v] = hp[v] - hm[v];
      }
      if (stage0 && cell_on) {
        snd = sound_speed(w[0], w[4 * PLANE], c);
        lam = lam_term(w[PLANE], w[2 * PLANE], w[3 * PLANE], snd, gl[0], gl[NFY], gl[2 * NFY],
                       gl[3 * NFY]) +
              lam_term(w[PLANE], w[2 * PLANE], w[3 * PLANE], snd, gl[TI], gl[NFY + TI],
                       gl[2 * NFY + TI], gl[3 * NFY + TI]);
        if constexpr (NDIM == 3) lam += lamz;
      }
    }

    // ---- phase A3 (3D): z halves of cell k+1, z flux of face k+1 ----------------------
    if constexpr (NDIM == 3) {
      mbar_wait(bar_of(k + 2), par_of(k + 2));
      if (cell_on) {
        const double* p1 = slot_of(k + 1) + s0;
        const double* p2 = slot_of(k + 2) + s0;
        double w0[5], wc[5], wz2[5];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          w0[v] = w[v * PLANE];
          wc[v] = p1[v * PLANE];
          wz2[v] = p2[v * PLANE];
        }
        const double* glo = zslot(k + 1) + tid;
        const double* ghi = zslot(k + 2) + tid;
        double hp1[5], hm1[5], fhi[5];
        z_halves(k + 1, w0, wc, wz2, glo, ghi, NT, hp1, hm1, true);
#pragma unroll
        for (int v = 0; v < 5; ++v) fhi[v] = hpz[v] + hm1[v];
        if (k == nk - 1) {
          const int bk = b.bface[5][i + ni * j];
          if (bk != BFACE_NONE) {
            double wm1[5] = {0, 0, 0, 0, 0};   // W(k-1): walls only (plane k-1 has left the ring)
            if (bk == BFACE_WALL) wm1[4] = Win[4 * fsz + colofs + sz * (long long)(k - 1)];
            overwrite(bk, w0, wm1, wc, 1, glo, NT, fhi);
          }
        }
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          R[v] += fhi[v] - fzl[v];
          fzl[v] = fhi[v];
          hpz[v] = hp1[v];
        }
        if (stage0) {
          const double snd1 = sound_speed(wc[0], wc[4], c);
          lamz = lam_term(wc[1], wc[2], wc[3], snd1, glo[0], glo[NT], glo[2 * NT], glo[3 * NT]) +
                 lam_term(wc[1], wc[2], wc[3], snd1, ghi[0], ghi[NT], ghi[2 * NT], ghi[3 * NT]);

        }
      }
    }

    __syncthreads();   // AB: y halves and tile-edge halves of plane k complete
    if (tid == 32) {   // (warp 1: warp 0 issued the B0 group)
      fence_async_smem();
      if (kk + 1 < kc) issue_geo_yz(k + 1);
      if (kk + 2 < kc) prefetch_l2(k + 2);
    }

    // ---- phase B1: x halves of cell (i, j, k); neighbours by shuffle --------------------
    mbar_wait(bars + 4, (unsigned)(kk & 1));   // x geometry, Q0 (dt/V) of plane k
    bool xlo_halo = tx == 0, xhi_halo = tx == TI - 1;
    {
      double qL[5], qR[5];
#pragma unroll
      for (int v = 0; v < 5; ++v)
        vl_recon<LIM, K1>(w[v * PLANE - 1], w[v * PLANE], w[v * PLANE + 1], c, qL[v], qR[v]);
      const double* gl = sFX + ty * GXW + tx;   // face i (low); face i+1 at gl + 1
      double hp[5], hm[5];
      vl_pair(qL, gl + 1, qR, gl, NFX, c, hp, hm);
      if (maybe_nonpos(qL[0], qL[4], qR[0], qR[4]) && in_j) {
        const bool bL = (qL[0] <= 0.0) | (qL[4] <= 0.0), bR = (qR[0] <= 0.0) | (qR[4] <= 0.0);
        if (bL && in_i) face_err(0, ERR_FACE_LEFT, lin_x(i + 1, j, k));
        if (bR && i <= ni) face_err(0, ERR_FACE_RIGHT, lin_x(i, j, k));
      }
      double fhi[5], flo[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        const double hmn = __shfl_down_sync(FULL, hm[v], 1);
        const double hpp = __shfl_up_sync(FULL, hp[v], 1);
        // the tile-edge lanes complete these with the tile-edge halves below
        fhi[v] = xhi_halo ? hp[v] : hp[v] + hmn;
        flo[v] = xlo_halo ? hm[v] : hpp + hm[v];
      }
      if (in_j && (i == 0 || i == ni - 1)) {
        if (i == 0) {
          const int bk = (bfk >> 0) & 3u;
          if (bk != BFACE_NONE) {
            overwrite(bk, w, w + 1, w - 1, PLANE, gl, NFX, flo);
            xlo_halo = false;
          }
        }
        if (i == ni - 1) {
          const int bk = (bfk >> 2) & 3u;
          if (bk != BFACE_NONE) {
            overwrite(bk, w, w - 1, w + 1, PLANE, gl + 1, NFX, fhi);
            xhi_halo = false;
          }
        }
      }
#pragma unroll
      for (int v = 0; v < 5; ++v) R[v] += fhi[v] - flo[v];
      if (stage0 && cell_on) {
        lam += lam_term(w[PLANE], w[2 * PLANE], w[3 * PLANE], snd, gl[0], gl[NFX], gl[2 * NFX],
                        gl[3 * NFX]) +
               lam_term(w[PLANE], w[2 * PLANE], w[3 * PLANE], snd, gl[1], gl[NFX + 1],
                        gl[2 * NFX + 1], gl[3 * NFX + 1]);
      }
    }

    // ---- phase B2: residual, update of cell (i, j, k) -----------------------------------
    if (cell_on) {
      const int hi = (ty + 1) * TI + tx, lo = ty * TI + tx;
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        const double* HP = sHP + v * NHY;
        const double* HM = sHM + v * NHY;
        double r = R[v];
        if (!yhi_ovw) r += HM[hi];   // overwritten faces: the whole flux is the own half
        if (!ylo_ovw) r -= HP[lo];
        if (xlo_halo) r -= sXH[v * TJ + ty];
        if (xhi_halo) r += sXH[5 * TJ + v * TJ + ty];
        R[v] = r;
      }
      const long long co = colofs + kofs;
      if (flags & F_SOURCE) {
#pragma unroll
        for (int v = 0; v < 5; ++v) R[v] = R[v] - b.base[(long long)(FSRC + v) * fsz + co];
      }
      double dtv;
      if (stage0) {
#pragma unroll
        for (int v = 0; v < 5; ++v) rsum[v] = fma(R[v], R[v], rsum[v]);
        dtv = c.cfl * frcp(lam);
        b.base[(long long)FDTV * fsz + co] = dtv;
      } else {
        dtv = K::QLDG ? b.base[(long long)FDTV * fsz + co] : sQ[5 * NT + tid];
      }
      const double adt = a.alpha * dtv;
      double qn[5];
#pragma unroll
      for (int v = 0; v < 5; ++v)
        qn[v] = fma(-adt, R[v], K::QLDG ? b.base[(long long)(FQ + v) * fsz + co] : sQ[v * NT + tid]);
      const double rq = frcp(qn[0]);
      const double uu = qn[1] * rq, vv = qn[2] * rq, ww = qn[3] * rq;
      const double pp = c.gm1 * fma(-0.5, fma(qn[1], uu, fma(qn[2], vv, qn[3] * ww)), qn[4]);
      if (maybe_nonpos(qn[0], pp, qn[0], pp) && (qn[0] <= 0.0 || pp <= 0.0)) {
        const unsigned long long lin =
            ((unsigned long long)i * nj + j) * (unsigned long long)nk + (NDIM == 3 ? k : 0);
        record_error(a.err, make_err_key(stage, 1, b.order, 0, 0, lin));
      }
      Wout[co] = qn[0];
      Wout[fsz + co] = uu;
      Wout[2 * fsz + co] = vv;
      Wout[3 * fsz + co] = ww;
      Wout[4 * fsz + co] = pp;
      if (last) {
#pragma unroll
        for (int v = 0; v < 5; ++v) b.base[(long long)(FQ + v) * fsz + co] = qn[v];
      }
#if BF_VL_PUSH
      if (a.push) {
        const int g = b.g;
        const bool near = i < g || i >= ni - g || j < g || j >= nj - g ||
                          (NDIM == 3 && (k < g || k >= nk - g));
        if (near)
          push_ghosts(sPS, b.base, sy, sz, fsz, ni, nj, nk, g, NDIM, a.cur ^ 1, c, i, j, k, qn[0],
                      uu, vv, ww, pp);
      }
#endif
    }
  }

  // ---- deterministic per-tile sum(R^2) ----------------------------------------
  if (stage0) {
    __syncthreads();
    double* red = sQ;   // free after the last phase B: [NT/32][5]
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      double x = rsum[v];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(FULL, x, off);
      if ((tid & 31) == 0) red[(tid >> 5) * 5 + v] = x;
    }
    __syncthreads();
    if (tid < 5) {
      double x = 0.0;
      for (int q = 0; q < NT / 32; ++q) x += red[q * 5 + tid];
      a.partial[(long long)tile_id * 5 + tid] = x;
    }
  }
}

template <int NDIM, int LIM, bool K1, bool S0>
static cudaError_t launch_vl_s(const StageArgs& a, cudaStream_t s) {
  using K = VCfg<NDIM, LIM>;
  auto k = vl_stage_kernel<NDIM, LIM, K1, S0>;
  static unsigned long long attr_done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_done & (1ull << dev))) {
    cudaError_t e =
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::BYTES);
    if (e != cudaSuccess) return e;
    attr_done |= (1ull << dev);
  }
  if (a.ntiles == 0) return cudaSuccess;
  return launch_pdl(k, (unsigned)(a.ntiles + (a.fill_chunks ? a.fill_ctas : 0)), (unsigned)K::NT, K::BYTES, s, a);
}

template <int NDIM, int LIM, bool K1>
static cudaError_t launch_vl_t(const StageArgs& a, cudaStream_t s) {
  return (a.flags & F_STAGE0) ? launch_vl_s<NDIM, LIM, K1, true>(a, s)
                              : launch_vl_s<NDIM, LIM, K1, false>(a, s);
}

template <int NDIM, bool K1>
static cudaError_t launch_vl_l(int lim, const StageArgs& a, cudaStream_t s) {
  switch (lim) {
    case LIM_NONE: return launch_vl_t<NDIM, LIM_NONE, K1>(a, s);
    case LIM_VAN_LEER: return launch_vl_t<NDIM, LIM_VAN_LEER, K1>(a, s);
    case LIM_VAN_ALBADA: return launch_vl_t<NDIM, LIM_VAN_ALBADA, K1>(a, s);
    default: return launch_vl_t<NDIM, LIM_MINMOD, K1>(a, s);
  }
}

static cudaError_t launch_vl(int ndim, int lim, const StageArgs& a, cudaStream_t s) {
  const bool k1 = a.c.muscl_k1 != 0;
  if (ndim == 3) return k1 ? launch_vl_l<3, true>(lim, a, s) : launch_vl_l<3, false>(lim, a, s);
  return k1 ? launch_vl_l<2, true>(lim, a, s) : launch_vl_l<2, false>(lim, a, s);
}
