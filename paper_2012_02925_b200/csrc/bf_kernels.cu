// bf_kernels.cu — the per-RK-stage device pipeline.
//
// Compiled twice by build.py: -DBF_EXACT=1 -fmad=false (namespace bf_exact,
// bitwise reference arithmetic) and -DBF_EXACT=0 (namespace bf_fast, FMA and
// strength reduction).
//
//   stage_kernel   fused limiter + MUSCL + face flux + boundary-flux overwrite
//                  + residual + (stage 0) local dt and sum(R^2) + RK update +
//                  decode (solver.py:413-753).  2.5-D k-streaming: a CTA owns a
//                  TI x TJ column tile and marches KC cells in k; the 5
//                  primitive planes k..k+2 sit in a 4-slot shared-memory ring
//                  filled by cp.async one plane ahead, so every W value is read
//                  from HBM once per tile (plus the 2-cell i/j halo).
//   ghost_kernel   physical-BC ghost fill (solver.py:281-403), same-device
//                  connected copies and message pack/unpack (halo.py:47-115)
//                  for every block of the rank in ONE launch.
//   reduce_kernel  fixed-order per-block sum of the per-tile sum(R^2) partials.
#include <cuda_runtime.h>

#include "bf_internal.h"

#if BF_EXACT
#define BF_NS bf_exact
#else
#define BF_NS bf_fast
#endif
#include "bf_physics.cuh"

namespace bf {
namespace BF_NS {

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
BF_DEV void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
BF_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
BF_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
BF_DEV void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

BF_DEV void record_error(unsigned long long* err, unsigned long long key) {
  if (key < *reinterpret_cast<volatile unsigned long long*>(err)) atomicMin(err, key);
}

// Compile-time tile geometry and shared-memory layout (in doubles).
template <int NDIM, int LIM>
struct Cfg {
  static constexpr int PC = psi_count<LIM>();
  static constexpr int TJ = (NDIM == 3 && PC < 2) ? TJ_3D : TJ_2D;
  static constexpr int NT = TI * TJ;
  static constexpr int PW = TI + 2 * HALO;                // plane row pitch
  static constexpr int PH = TJ + 2 * HALO;
  static constexpr int PLANE = PW * PH;                   // cells per plane
  static constexpr int NS = (NDIM == 3) ? NSLOT : 1;
  static constexpr int NPX = (TI + 2) * TJ;               // psi_x cells: i = -1..TI
  static constexpr int NPY = TI * (TJ + 2);               // psi_y cells: j = -1..TJ
  static constexpr int NFX = (TI + 1) * TJ;               // x faces
  static constexpr int NFY = TI * (TJ + 1);               // y faces
  static constexpr int OW = 0;                            // [NS][5][PLANE]
  static constexpr int OPX = OW + NS * 5 * PLANE;         // [PC][5][NPX]
  static constexpr int OPY = OPX + PC * 5 * NPX;          // [PC][5][NPY]
  static constexpr int OFX = OPY + PC * 5 * NPY;          // [5][NFX]
  static constexpr int OFY = OFX + 5 * NFX;               // [5][NFY]
  static constexpr int OQ = OFY + 5 * NFY;                // [6][NT] Q0 + dt/V (or V)
  static constexpr int TOTAL = OQ + 6 * NT;
  static constexpr size_t BYTES = sizeof(double) * TOTAL;
  static constexpr int NITEM = NFX + NFY;                 // x/y face items per plane
  static constexpr int MAXIT = (NITEM + NT - 1) / NT;
  static constexpr int NLIM = NPX + NPY;
  BF_DEV static int pidx(int ii, int jj) { return (jj + HALO) * PW + (ii + HALO); }
};

// psi+ / psi- of one cell from its three stencil values (solver.py:419-435):
// psi+_c = phi(D_{c+1}, D_c), psi-_c = phi(D_c, D_{c+1}).
template <int LIM>
BF_DEV void cell_limiter(double wm, double w0, double wp, double& pp, double& pm) {
  const double lo = w0 - wm;
  const double hi = wp - w0;
  pp = limiter<LIM>(hi, lo);
  if constexpr (psi_count<LIM>() == 2) pm = limiter<LIM>(lo, hi);
  else pm = pp;
}

// MUSCL face states (solver.py:437-474) + flux (physics.py) + area scaling
// (solver.py:519) + boundary overwrite (solver.py:526-580) for one face.
// c0..c3: var-0 pointers of cells f-2, f-1, f, f+1 (var stride vs).
// ppl/pml: psi+/psi- of cell f-1, ppr/pmr: of cell f (var stride ps).
template <int FLUX, int LIM>
BF_DEV int face_flux(const double* c0, const double* c1, const double* c2, const double* c3, int vs,
                     const double* ppl, const double* pml, const double* ppr, const double* pmr,
                     int ps, double nx, double ny, double nz, double A, int bkind,
                     double side_sign, const Consts& c, double F[5]) {
  double qL[5], qR[5];
#pragma unroll
  for (int v = 0; v < 5; ++v) {
    const double wl = c1[v * vs];
    const double wr = c2[v * vs];
    if (c.eps0) {
      qL[v] = wl;
      qR[v] = wr;
    } else {
      const double dm = wl - c0[v * vs];
      const double d0 = wr - wl;
      const double dp = c3[v * vs] - wr;
      double a_pl = 1.0, a_ml = 1.0, a_pr = 1.0, a_mr = 1.0;
      if constexpr (psi_count<LIM>() > 0) {
        a_pl = ppl[v * ps];
        a_pr = ppr[v * ps];
        a_ml = pml[v * ps];
        a_mr = pmr[v * ps];
      }
#if BF_EXACT
      qL[v] = wl + c.quarter * (c.omk * a_pl * dm + c.opk * a_ml * d0);
      qR[v] = wr - c.quarter * (c.opk * a_pr * d0 + c.omk * a_mr * dp);
#else
      if (c.kappa_m1) {
        qL[v] = wl + c.quarter * (c.omk * a_pl * dm);
        qR[v] = wr - c.quarter * (c.omk * a_mr * dp);
      } else {
        qL[v] = wl + c.quarter * (c.omk * a_pl * dm + c.opk * a_ml * d0);
        qR[v] = wr - c.quarter * (c.opk * a_pr * d0 + c.omk * a_mr * dp);
      }
#endif
    }
  }
  int err = 0;
  if (qL[0] <= 0.0 || qL[4] <= 0.0) err = ERR_FACE_LEFT;
  else if (qR[0] <= 0.0 || qR[4] <= 0.0) err = ERR_FACE_RIGHT;
  const St L{qL[0], qL[1], qL[2], qL[3], qL[4]};
  const St R{qR[0], qR[1], qR[2], qR[3], qR[4]};
  if constexpr (FLUX == FLUX_ROE) {
    if (!roe_flux(L, R, nx, ny, nz, c, F) && err == 0) err = ERR_ROE_A2;
  } else {
    van_leer_flux(L, R, nx, ny, nz, c, F);
  }
#pragma unroll
  for (int e = 0; e < 5; ++e) F[e] = F[e] * A;
  if (bkind != BFACE_NONE) {
    // first / second interior cells next to the boundary plane
    const double* in1 = (side_sign < 0.0) ? c2 : c1;
    const double* in2 = (side_sign < 0.0) ? c3 : c0;
    if (bkind == BFACE_WALL) {
      const double pw = 1.5 * in1[4 * vs] - 0.5 * in2[4 * vs];
      F[0] = 0.0;
      F[1] = nx * pw * A;
      F[2] = ny * pw * A;
      F[3] = nz * pw * A;
      F[4] = 0.0;
    } else {
      const St s1{in1[0], in1[vs], in1[2 * vs], in1[3 * vs], in1[4 * vs]};
      const St qb = farfield_state(s1, side_sign * nx, side_sign * ny, side_sign * nz, c);
      double Fb[5];
      euler_flux(qb, nx, ny, nz, c, Fb);
#pragma unroll
      for (int e = 0; e < 5; ++e) F[e] = Fb[e] * A;
    }
  }
  return err;
}

// Geometry and boundary code of one face, loaded early (ahead of its use).
struct FaceGeo {
  double nx, ny, nz, A;
  int bk;
  double sgn;
};

BF_DEV void load_geo(FaceGeo& g, const DevBlock& b, int d, long long off, bool on, int bface,
                     int bk_side) {
  if (on) {
    const double* fn = b.base + (long long)ffn(d, 0) * b.fsz + off;
    g.nx = __ldg(fn);
    g.ny = __ldg(fn + b.fsz);
    g.nz = __ldg(fn + 2 * b.fsz);
    g.A = __ldg(fn + 3 * b.fsz);
  } else {
    g.nx = g.ny = g.nz = 0.0;
    g.A = 0.0;
  }
  g.bk = BFACE_NONE;
  g.sgn = 1.0;
  if (on && bk_side >= 0) {
    g.bk = b.bface[2 * d + bk_side][bface];
    g.sgn = bk_side == 0 ? -1.0 : 1.0;
  }
}

// ---------------------------------------------------------------------------
// the fused stage kernel
// ---------------------------------------------------------------------------
template <int NDIM, int FLUX, int LIM>
__global__ void __launch_bounds__(Cfg<NDIM, LIM>::NT, 1) stage_kernel(const StageArgs a) {
  using K = Cfg<NDIM, LIM>;
  constexpr int NT = K::NT, TJ = K::TJ, PLANE = K::PLANE, PW = K::PW, PC = K::PC;
  extern __shared__ __align__(16) double smem[];
  double* const sW = smem + K::OW;
  double* const sPX = smem + K::OPX;
  double* const sPY = smem + K::OPY;
  double* const sFX = smem + K::OFX;
  double* const sFY = smem + K::OFY;
  double* const sQ = smem + K::OQ;

  const Tile t = a.tiles[blockIdx.x];
  const DevBlock b = a.blocks[t.block];     // local copy: no aliasing reloads
  const Consts& c = a.c;
  const int tid = threadIdx.x;
  const int tx = tid % TI, ty = tid / TI;
  const int i0 = t.i0, j0 = t.j0, k0 = t.k0;
  const int ni = b.n[0], nj = b.n[1], nk = b.n[2];
  const long long sy = b.sy, sz = b.sz, fsz = b.fsz;
  const int i = i0 + tx, j = j0 + ty;
  const bool col_on = (i < ni) && (j < nj);
  const int flags = a.flags;
  const bool stage0 = flags & F_STAGE0;
  const bool last = flags & F_LAST;
  const bool psi_load = (PC > 0) && (flags & F_PSI_LOAD);
  const bool psi_store = (PC > 0) && (flags & F_PSI_STORE);
  const int stage = a.stage;
  const double* const Win = b.base + (long long)fw(a.cur, 0) * fsz;
  double* const Wout = b.base + (long long)fw(a.cur ^ 1, 0) * fsz;
  const long long colofs = i + sy * (long long)j;

  auto slot = [&](int k) -> double* {
    if constexpr (NDIM == 3) return sW + ((k - k0 + 4 * NSLOT) % NSLOT) * 5 * PLANE;
    else return sW;
  };
  auto psi_ptr = [&](int d, int pm, int v) -> double* {
    return b.base + (long long)(b.psi0 + 10 * d + 5 * pm + v) * fsz;
  };

  // issue the cp.async copies of one plane (tile + 2-cell i/j halo, cross shape)
  auto load_plane = [&](int k) {
    if (NDIM == 3 && (k < -HALO || k >= nk + HALO)) return;
    double* dst = slot(k);
    const long long kofs = (NDIM == 3) ? sz * (long long)k : 0;
    constexpr int ROWS_FULL = TJ * PW;
    constexpr int ROWS_HALO = 2 * HALO * TI;
    for (int q = tid; q < ROWS_FULL + ROWS_HALO; q += NT) {
      int ii, jj;
      if (q < ROWS_FULL) {
        jj = q / PW;
        ii = q % PW - HALO;
      } else {
        const int r = (q - ROWS_FULL) / TI;
        ii = (q - ROWS_FULL) % TI;
        jj = (r < HALO) ? r - HALO : TJ + r - HALO;
      }
      const int gi = i0 + ii, gj = j0 + jj;
      if (gi < -HALO || gi >= ni + HALO || gj < -HALO || gj >= nj + HALO) continue;
      const double* src = Win + gi + sy * (long long)gj + kofs;
      const int s = K::pidx(ii, jj);
#pragma unroll
      for (int v = 0; v < 5; ++v) cp_async8(dst + v * PLANE + s, src + v * fsz);
    }
  };
  // Q0 (+ dt/V or V) of the own cell, staged per thread
  auto load_q = [&](int k) {
    if (!col_on) return;
    const long long o = colofs + ((NDIM == 3) ? sz * (long long)k : 0);
    const double* q = b.base + (long long)FQ * fsz + o;
#pragma unroll
    for (int v = 0; v < 5; ++v) cp_async8(sQ + v * NT + tid, q + v * fsz);
    const double* dv = b.base + (long long)(stage0 ? FVOL : FDTV) * fsz + o;
    cp_async8(sQ + 5 * NT + tid, dv);
  };

  // ---- x/y face items of this thread (fixed for all k) ----------------------
  // item q < NFX: x face (row = q / (TI+1), f = q % (TI+1)); else y face
  int it_q[K::MAXIT];
#pragma unroll
  for (int r = 0; r < K::MAXIT; ++r) it_q[r] = tid + r * NT;

  double rsum[5] = {0.0, 0.0, 0.0, 0.0, 0.0};

  // ---- z-direction carried state (3D) -------------------------------------------
  double wm1[5] = {0, 0, 0, 0, 0};  // W(k-1), own column
  double pzp[5], pzm[5];            // psi+/psi- of cell k
  double fz[5];                     // flux at face k
#pragma unroll
  for (int v = 0; v < 5; ++v) pzp[v] = pzm[v] = fz[v] = 0.0;

  if constexpr (NDIM == 3) {
    if (col_on) {
      const long long o = colofs + sz * (long long)(k0 - 2);
#pragma unroll
      for (int v = 0; v < 5; ++v) wm1[v] = Win[v * fsz + o];
    }
    load_plane(k0 - 1);
    load_plane(k0);
    load_plane(k0 + 1);
    cp_async_commit();
  } else {
    load_plane(0);
    load_q(0);
    cp_async_commit();
  }

  const int kfirst = (NDIM == 3) ? -1 : 0;
  for (int kk = kfirst; kk < t.kc; ++kk) {
    const int k = k0 + kk;
    const bool xy = kk >= 0;
    const long long kofs = (NDIM == 3) ? sz * (long long)k : 0;
    cp_async_wait_all();
    __syncthreads();   // B0: planes k..k+2 resident; everyone done with iteration k-1
    if constexpr (NDIM == 3) {
      if (xy) load_q(k);
      cp_async_commit();
      if (kk + 1 < t.kc) load_plane(k + 3);
      cp_async_commit();
    }
    const double* pk = slot(k);
    const int s0 = K::pidx(tx, ty);

    // early geometry loads for this iteration's faces
    FaceGeo gz;
    if constexpr (NDIM == 3) {
      const int fk = k + 1;
      load_geo(gz, b, 2, colofs + sz * (long long)fk, col_on, i + ni * j,
               fk == 0 ? 0 : (fk == nk ? 1 : -1));
    }
    FaceGeo gi_[K::MAXIT];
#pragma unroll
    for (int r = 0; r < K::MAXIT; ++r) {
      const int q = it_q[r];
      if (!xy || q >= K::NITEM) {
        gi_[r].A = 0.0;
        continue;
      }
      if (q < K::NFX) {
        const int row = q / (TI + 1), f = q % (TI + 1);
        const int gi = i0 + f, gj = j0 + row;
        const bool on = gi <= ni && gj < nj;
        load_geo(gi_[r], b, 0, gi + sy * (long long)gj + kofs, on, gj + nj * (NDIM == 3 ? k : 0),
                 gi == 0 ? 0 : (gi == ni ? 1 : -1));
      } else {
        const int q2 = q - K::NFX;
        const int f = q2 / TI, col = q2 % TI;
        const int gi = i0 + col, gj = j0 + f;
        const bool on = gj <= nj && gi < ni;
        load_geo(gi_[r], b, 1, gi + sy * (long long)gj + kofs, on, gi + ni * (NDIM == 3 ? k : 0),
                 gj == 0 ? 0 : (gj == nj ? 1 : -1));
      }
    }

    // ---- P1: x / y limiters of plane k -> smem -------------------------------------
    if (xy && PC > 0) {
      for (int q = tid; q < K::NLIM; q += NT) {
        int gi, gj, d, o, sc, step;
        if (q < K::NPX) {
          const int row = q / (TI + 2), cc = q % (TI + 2) - 1;    // cell cc in [-1, TI]
          gi = i0 + cc;
          gj = j0 + row;
          d = 0;
          o = q;
          sc = K::pidx(cc, row);
          step = 1;
        } else {
          const int q2 = q - K::NPX;
          const int row = q2 / TI - 1, cc = q2 % TI;             // row in [-1, TJ]
          gi = i0 + cc;
          gj = j0 + row;
          d = 1;
          o = q2;
          sc = K::pidx(cc, row);
          step = PW;
        }
        double* dstp = (d == 0) ? sPX + o : sPY + o;
        const int vstride = (d == 0) ? K::NPX : K::NPY;
        const bool in_range = (d == 0) ? (gi >= -1 && gi <= ni && gj < nj)
                                       : (gj >= -1 && gj <= nj && gi < ni);
        const long long go = gi + sy * (long long)gj + kofs;
        if (psi_load) {
          if (in_range) {
#pragma unroll
            for (int v = 0; v < 5; ++v) {
              dstp[v * vstride] = psi_ptr(d, 0, v)[go];
              if constexpr (PC == 2) dstp[(5 + v) * vstride] = psi_ptr(d, 1, v)[go];
            }
          }
        } else {
#pragma unroll
          for (int v = 0; v < 5; ++v) {
            double pp, pm;
            cell_limiter<LIM>(pk[v * PLANE + sc - step], pk[v * PLANE + sc],
                              pk[v * PLANE + sc + step], pp, pm);
            dstp[v * vstride] = pp;
            if constexpr (PC == 2) dstp[(5 + v) * vstride] = pm;
            if (psi_store && in_range) {
              psi_ptr(d, 0, v)[go] = pp;
              psi_ptr(d, 1, v)[go] = pm;
            }
          }
        }
      }
    }

    // ---- z limiter of cell k+1 and z face k+1 (own column, registers) ------------
    double Fz[5] = {0, 0, 0, 0, 0};
    if constexpr (NDIM == 3) {
      const double* p0 = slot(k);
      const double* p1 = slot(k + 1);
      const double* p2 = slot(k + 2);
      double nzp[5], nzm[5];
      const long long cz = colofs + sz * (long long)(k + 1);
      if (kk == kfirst) {
        // psi_z of cell k (= k0-1) from W(k-1) (regs), W(k), W(k+1)
        const long long czk = colofs + sz * (long long)k;
        if (psi_load) {
#pragma unroll
          for (int v = 0; v < 5; ++v) {
            pzp[v] = col_on ? psi_ptr(2, 0, v)[czk] : 0.0;
            pzm[v] = (PC == 2) ? (col_on ? psi_ptr(2, 1, v)[czk] : 0.0) : pzp[v];
          }
        } else {
#pragma unroll
          for (int v = 0; v < 5; ++v) {
            cell_limiter<LIM>(wm1[v], p0[v * PLANE + s0], p1[v * PLANE + s0], pzp[v], pzm[v]);
            if (psi_store && col_on && k >= -1) {
              psi_ptr(2, 0, v)[czk] = pzp[v];
              psi_ptr(2, 1, v)[czk] = pzm[v];
            }
          }
        }
      }
      if (psi_load) {
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          nzp[v] = col_on ? psi_ptr(2, 0, v)[cz] : 0.0;
          nzm[v] = (PC == 2) ? (col_on ? psi_ptr(2, 1, v)[cz] : 0.0) : nzp[v];
        }
      } else {
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          cell_limiter<LIM>(p0[v * PLANE + s0], p1[v * PLANE + s0], p2[v * PLANE + s0], nzp[v],
                            nzm[v]);
          if (psi_store && col_on && k + 1 <= nk) {
            psi_ptr(2, 0, v)[cz] = nzp[v];
            psi_ptr(2, 1, v)[cz] = nzm[v];
          }
        }
      }
      // z face k+1 from a unit-stride copy of the own-column stencil
      {
        double st[4][5];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          st[0][v] = wm1[v];
          st[1][v] = p0[v * PLANE + s0];
          st[2][v] = p1[v * PLANE + s0];
          st[3][v] = p2[v * PLANE + s0];
        }
        const int ez = face_flux<FLUX, LIM>(st[0], st[1], st[2], st[3], 1, pzp, pzm, nzp, nzm, 1,
                                            gz.nx, gz.ny, gz.nz, gz.A, gz.bk, gz.sgn, c, Fz);
        if (ez && col_on) {
          const int fk = k + 1;
          const unsigned long long lin =
              ((unsigned long long)i * nj + j) * (unsigned long long)(nk + 1) + fk;
          record_error(a.err, make_err_key(stage, 0, b.order, 2, ez, lin));
        }
      }
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        pzp[v] = nzp[v];
        pzm[v] = nzm[v];
      }
      if (kk == kfirst) {
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          fz[v] = Fz[v];
          wm1[v] = p0[v * PLANE + s0];
        }
        continue;   // prologue iteration: z only
      }
    }

    __syncthreads();   // B1: psi of plane k complete

    // ---- P2: x / y face fluxes of plane k -> smem ----------------------------------
#pragma unroll
    for (int r = 0; r < K::MAXIT; ++r) {
      const int q = it_q[r];
      if (q >= K::NITEM) continue;
      double Fq[5];
      if (q < K::NFX) {
        const int row = q / (TI + 1), f = q % (TI + 1);
        const int sc = K::pidx(f, row);
        const int po = row * (TI + 2) + f;          // psi of cell f-1 (index (f-1)+1)
        const int e = face_flux<FLUX, LIM>(pk + sc - 2, pk + sc - 1, pk + sc, pk + sc + 1, PLANE,
                                           sPX + po, sPX + (PC == 2 ? 5 * K::NPX : 0) + po,
                                           sPX + po + 1, sPX + (PC == 2 ? 5 * K::NPX : 0) + po + 1,
                                           K::NPX, gi_[r].nx, gi_[r].ny, gi_[r].nz, gi_[r].A,
                                           gi_[r].bk, gi_[r].sgn, c, Fq);
        const int gi = i0 + f, gj = j0 + row;
        if (e && gi <= ni && gj < nj) {
          const unsigned long long lin =
              ((unsigned long long)gi * nj + gj) * (unsigned long long)(NDIM == 3 ? nk : 1) +
              (NDIM == 3 ? k : 0);
          record_error(a.err, make_err_key(stage, 0, b.order, 0, e, lin));
        }
#pragma unroll
        for (int v = 0; v < 5; ++v) sFX[v * K::NFX + q] = Fq[v];
      } else {
        const int q2 = q - K::NFX;
        const int f = q2 / TI, col = q2 % TI;
        const int sc = K::pidx(col, f);
        const int po = f * TI + col;                // psi of row f-1 (index (f-1)+1)
        const int e = face_flux<FLUX, LIM>(pk + sc - 2 * PW, pk + sc - PW, pk + sc, pk + sc + PW,
                                           PLANE, sPY + po, sPY + (PC == 2 ? 5 * K::NPY : 0) + po,
                                           sPY + po + TI, sPY + (PC == 2 ? 5 * K::NPY : 0) + po + TI,
                                           K::NPY, gi_[r].nx, gi_[r].ny, gi_[r].nz, gi_[r].A,
                                           gi_[r].bk, gi_[r].sgn, c, Fq);
        const int gi = i0 + col, gj = j0 + f;
        if (e && gj <= nj && gi < ni) {
          const unsigned long long lin =
              ((unsigned long long)gi * (nj + 1) + gj) * (unsigned long long)(NDIM == 3 ? nk : 1) +
              (NDIM == 3 ? k : 0);
          record_error(a.err, make_err_key(stage, 0, b.order, 1, e, lin));
        }
#pragma unroll
        for (int v = 0; v < 5; ++v) sFY[v * K::NFY + q2] = Fq[v];
      }
    }
    if constexpr (NDIM == 3) cp_async_wait_1();   // own Q0 / dt staging landed
    else cp_async_wait_all();
    __syncthreads();   // B2: face fluxes of plane k complete

    // ---- P3: residual, dt, update of cell (i, j, k) --------------------------------
    if (col_on) {
      double R[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        const int ox = ty * (TI + 1) + tx;
        const double dx = sFX[v * K::NFX + ox + 1] - sFX[v * K::NFX + ox];
        const double dy = sFY[v * K::NFY + (ty + 1) * TI + tx] - sFY[v * K::NFY + ty * TI + tx];
        if constexpr (NDIM == 3) R[v] = ((0.0 + dx) + dy) + (Fz[v] - fz[v]);
        else R[v] = (0.0 + dx) + dy;
      }
      const long long co = colofs + kofs;
      if (flags & F_SOURCE) {
#pragma unroll
        for (int v = 0; v < 5; ++v) R[v] = R[v] - b.base[(long long)(FSRC + v) * fsz + co];
      }
      double dtv;
      if (stage0) {
#pragma unroll
        for (int v = 0; v < 5; ++v) rsum[v] += R[v] * R[v];
        const double rho = pk[s0], u = pk[PLANE + s0], v = pk[2 * PLANE + s0],
                     w = pk[3 * PLANE + s0], p = pk[4 * PLANE + s0];
        const double snd = sqrt(c.gamma * p / rho);
        double lam = 0.0;
#pragma unroll
        for (int d = 0; d < NDIM; ++d) {
#pragma unroll
          for (int hi = 0; hi < 2; ++hi) {
            const long long fo = co + (hi ? (d == 0 ? 1 : (d == 1 ? sy : sz)) : 0);
            const double* fn = b.base + (long long)ffn(d, 0) * fsz + fo;
            const double nx = __ldg(fn), ny = __ldg(fn + fsz), nz = __ldg(fn + 2 * fsz),
                         A = __ldg(fn + 3 * fsz);
            lam = lam + (fabs(u * nx + v * ny + w * nz) + snd) * A;
          }
        }
        const double vol = sQ[5 * NT + tid];
#if BF_EXACT
        dtv = c.cfl * vol / lam / vol;
#else
        dtv = c.cfl / lam;
#endif
        b.base[(long long)FDTV * fsz + co] = dtv;
      } else {
        dtv = sQ[5 * NT + tid];
      }
      double qn[5];
      const double adt = a.alpha * dtv;
#pragma unroll
      for (int v = 0; v < 5; ++v) qn[v] = sQ[v * NT + tid] - adt * R[v];
#if BF_EXACT
      const double uu = qn[1] / qn[0], vv = qn[2] / qn[0], ww = qn[3] / qn[0];
#else
      const double rq = 1.0 / qn[0];
      const double uu = qn[1] * rq, vv = qn[2] * rq, ww = qn[3] * rq;
#endif
      const double pp = c.gm1 * (qn[4] - 0.5 * (qn[1] * uu + qn[2] * vv + qn[3] * ww));
      if (qn[0] <= 0.0 || pp <= 0.0) {
        const unsigned long long lin =
            ((unsigned long long)i * nj + j) * (unsigned long long)(NDIM == 3 ? nk : 1) +
            (NDIM == 3 ? k : 0);
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
    }
    if constexpr (NDIM == 3) {
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        fz[v] = Fz[v];
        wm1[v] = pk[v * PLANE + s0];
      }
    }
  }

  // ---- deterministic per-tile sum(R^2) ----------------------------------------
  if (stage0) {
    cp_async_wait_all();
    __syncthreads();
    double* red = smem;   // reuse the plane ring: [NT/32][5]
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      double x = rsum[v];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
      if ((tid & 31) == 0) red[(tid >> 5) * 5 + v] = x;
    }
    __syncthreads();
    if (tid < 5) {
      double x = 0.0;
      for (int w = 0; w < NT / 32; ++w) x += red[w * 5 + tid];
      a.partial[(long long)blockIdx.x * 5 + tid] = x;
    }
  }
}

// ---------------------------------------------------------------------------
// ghost fill / pack / unpack (one launch per stage, all blocks)
// ---------------------------------------------------------------------------
BF_DEV double interior_T(const double* W, long long fsz, long long o, int t_derived,
                         const Consts& c) {
  return t_derived ? W[4 * fsz + o] / (W[o] * c.R) : W[5 * fsz + o];
}

__global__ void __launch_bounds__(256) ghost_kernel(const GhostArgs a) {
  const long long item = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= a.total_items) return;
  int lo = 0, hi = a.ntasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.tasks[mid].begin <= item) lo = mid;
    else hi = mid - 1;
  }
  const GhostTask& t = a.tasks[lo];
  const long long m = item - t.begin;
  if (m >= t.items) return;
  const Consts& c = a.c;

  if (t.kind == GK_COPY) {
    const int o0 = (int)(m % t.n[0]);
    const long long r = m / t.n[0];
    const int o1 = (int)(r % t.n[1]);
    const int o2 = (int)(r / t.n[1]);
    const long long doff = t.dst_origin + o0 * t.dst_stride[0] + o1 * t.dst_stride[1] +
                           o2 * t.dst_stride[2];
    const long long soff = t.src_origin + o0 * t.src_stride[0] + o1 * t.src_stride[1] +
                           o2 * t.src_stride[2];
    double val[6];
    if (t.src_block >= 0) {
      const DevBlock& sb = a.blocks[t.src_block];
      const double* W = sb.base + (long long)fw(a.cur, 0) * sb.fsz;
      int f = 0;
      val[f++] = W[soff];
      val[f++] = W[sb.fsz + soff];
      val[f++] = W[2 * sb.fsz + soff];
      if (t.nfields == 6) val[f++] = W[3 * sb.fsz + soff];
      val[f++] = W[4 * sb.fsz + soff];
      val[f++] = interior_T(W, sb.fsz, soff, a.t_derived, c);
    } else {
      for (int f = 0; f < t.nfields; ++f) val[f] = t.src_buf[f * t.buf_cells + soff];
    }
    if (t.block >= 0) {
      const DevBlock& db = a.blocks[t.block];
      double* W = db.base + (long long)fw(a.cur, 0) * db.fsz;
      int f = 0;
      W[doff] = val[f++];
      W[db.fsz + doff] = val[f++];
      W[2 * db.fsz + doff] = val[f++];
      if (t.nfields == 6) W[3 * db.fsz + doff] = val[f++];
      W[4 * db.fsz + doff] = val[f++];
      W[5 * db.fsz + doff] = val[f++];
    } else {
      for (int f = 0; f < t.nfields; ++f) t.dst_buf[f * t.buf_cells + doff] = val[f];
    }
    return;
  }

  // ---- physical patch: one tangential position, all ghost layers ----------
  const DevBlock& b = a.blocks[t.block];
  const long long fsz = b.fsz;
  double* W = b.base + (long long)fw(a.cur, 0) * fsz;
  const int u0 = (int)(m % t.tn[0]), u1 = (int)(m / t.tn[0]);
  int cell[3] = {0, 0, 0};
  cell[t.ta] = t.tlo[0] + u0;
  cell[t.tb] = t.tlo[1] + u1;
  const int d = t.axis;
  const long long st[3] = {1, b.sy, b.sz};
  cell[d] = 0;
  const long long base = cell[0] + b.sy * (long long)cell[1] + b.sz * (long long)cell[2];
  const int n = b.n[d];
  // ghost position / mirror interior position of layer L (solver.py:300-304)
  auto gpos = [&](int L) { return t.side == 0 ? -1 - L : n + L; };
  auto ipos = [&](int L) { return t.side == 0 ? L : n - 1 - L; };
  const int bc = t.bc_type;
  if (bc == BC_INFLOW) {
    for (int L = 0; L < t.depth; ++L) {
      const long long o = base + st[d] * gpos(L);
      W[o] = c.fs_rho;
      W[fsz + o] = c.fs_u;
      W[2 * fsz + o] = c.fs_v;
      W[3 * fsz + o] = c.fs_w;
      W[4 * fsz + o] = c.fs_p;
      W[5 * fsz + o] = c.fs_T;
    }
  } else if (bc == BC_OUTFLOW) {
    const long long oi = base + st[d] * ipos(0);
    const double v0 = W[oi], v1 = W[fsz + oi], v2 = W[2 * fsz + oi], v3 = W[3 * fsz + oi],
                 v4 = W[4 * fsz + oi];
    const double v5 = interior_T(W, fsz, oi, a.t_derived, c);
    for (int L = 0; L < t.depth; ++L) {
      const long long o = base + st[d] * gpos(L);
      W[o] = v0;
      W[fsz + o] = v1;
      W[2 * fsz + o] = v2;
      W[3 * fsz + o] = v3;
      W[4 * fsz + o] = v4;
      W[5 * fsz + o] = v5;
    }
  } else if (bc == BC_SLIP || bc == BC_NOSLIP) {
    const long long fo = base + st[d] * (t.side == 0 ? 0 : n);
    const double sg = t.side == 0 ? -1.0 : 1.0;
    const double* fn = b.base + (long long)ffn(d, 0) * fsz + fo;
    const double nx = sg * fn[0], ny = sg * fn[fsz], nz = sg * fn[2 * fsz];
    for (int L = 0; L < t.depth; ++L) {
      const long long og = base + st[d] * gpos(L);
      const long long oi = base + st[d] * ipos(L);
      const double u = W[fsz + oi], v = W[2 * fsz + oi], w = W[3 * fsz + oi];
      if (bc == BC_SLIP) {
        const double vn = u * nx + v * ny + w * nz;
        W[fsz + og] = u - 2.0 * vn * nx;
        W[2 * fsz + og] = v - 2.0 * vn * ny;
        W[3 * fsz + og] = w - 2.0 * vn * nz;
      } else {
        W[fsz + og] = -u;
        W[2 * fsz + og] = -v;
        W[3 * fsz + og] = -w;
      }
      const double pg = W[4 * fsz + oi];
      W[4 * fsz + og] = pg;
      const double ti = interior_T(W, fsz, oi, a.t_derived, c);
      const double tg = (bc == BC_NOSLIP && c.has_tw) ? 2.0 * c.tw - ti : ti;
      W[5 * fsz + og] = tg;
      W[og] = pg / (c.R * tg);
    }
  } else if (bc == BC_FARFIELD) {
    const long long fo = base + st[d] * (t.side == 0 ? 0 : n);
    const double sg = t.side == 0 ? -1.0 : 1.0;
    const double* fn = b.base + (long long)ffn(d, 0) * fsz + fo;
    const double nx = sg * fn[0], ny = sg * fn[fsz], nz = sg * fn[2 * fsz];
    const long long oi = base + st[d] * ipos(0);
    const St s{W[oi], W[fsz + oi], W[2 * fsz + oi], W[3 * fsz + oi], W[4 * fsz + oi]};
    const St q = farfield_state(s, nx, ny, nz, c);
    const double tb = q.p / (q.r * c.R);
    for (int L = 0; L < t.depth; ++L) {
      const long long o = base + st[d] * gpos(L);
      W[o] = q.r;
      W[fsz + o] = q.u;
      W[2 * fsz + o] = q.v;
      W[3 * fsz + o] = q.w;
      W[4 * fsz + o] = q.p;
      W[5 * fsz + o] = tb;
    }
  } else {   // mms_dirichlet: cached exact values
    const long long nt = (long long)t.tn[0] * t.tn[1];
    for (int L = 0; L < t.depth; ++L) {
      const long long o = base + st[d] * gpos(L);
      const double* src = t.dirichlet + (long long)L * 6 * nt + m;
      for (int f = 0; f < 6; ++f) W[f * fsz + o] = src[f * nt];
    }
  }
}

// Fixed-order per-block reduction of the per-tile partial sums.
__global__ void __launch_bounds__(256) reduce_kernel(const double* partial, const int* tile_begin,
                                                     int nblocks, double* out) {
  __shared__ double red[256 * 5];
  const int blk = blockIdx.x;
  if (blk >= nblocks) return;
  const int tb = tile_begin[blk], te = tile_begin[blk + 1];
  double x[5] = {0, 0, 0, 0, 0};
  for (int t = tb + threadIdx.x; t < te; t += blockDim.x) {
#pragma unroll
    for (int v = 0; v < 5; ++v) x[v] += partial[(long long)t * 5 + v];
  }
#pragma unroll
  for (int v = 0; v < 5; ++v) red[threadIdx.x * 5 + v] = x[v];
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
#pragma unroll
      for (int v = 0; v < 5; ++v) red[threadIdx.x * 5 + v] += red[(threadIdx.x + s) * 5 + v];
    }
    __syncthreads();
  }
  if (threadIdx.x < 5) out[blk * 5 + threadIdx.x] = red[threadIdx.x];
}

// ---------------------------------------------------------------------------
// launchers (called by the runtime)
// ---------------------------------------------------------------------------
template <int NDIM, int FLUX, int LIM>
static cudaError_t launch_stage_t(const StageArgs& a, cudaStream_t s) {
  using K = Cfg<NDIM, LIM>;
  auto k = stage_kernel<NDIM, FLUX, LIM>;
  static unsigned long long attr_done = 0;   // one bit per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_done & (1ull << dev))) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)K::BYTES);
    if (e != cudaSuccess) return e;
    attr_done |= (1ull << dev);
  }
  if (a.ntiles == 0) return cudaSuccess;
  k<<<a.ntiles, K::NT, K::BYTES, s>>>(a);
  return cudaGetLastError();
}

template <int NDIM, int FLUX>
static cudaError_t launch_stage_l(int lim, const StageArgs& a, cudaStream_t s) {
  switch (lim) {
    case LIM_NONE: return launch_stage_t<NDIM, FLUX, LIM_NONE>(a, s);
    case LIM_VAN_LEER: return launch_stage_t<NDIM, FLUX, LIM_VAN_LEER>(a, s);
    case LIM_VAN_ALBADA: return launch_stage_t<NDIM, FLUX, LIM_VAN_ALBADA>(a, s);
    default: return launch_stage_t<NDIM, FLUX, LIM_MINMOD>(a, s);
  }
}

cudaError_t launch_stage(int ndim, int flux, int lim, const StageArgs& a, cudaStream_t s) {
  if (ndim == 3)
    return flux == FLUX_ROE ? launch_stage_l<3, FLUX_ROE>(lim, a, s)
                            : launch_stage_l<3, FLUX_VAN_LEER>(lim, a, s);
  return flux == FLUX_ROE ? launch_stage_l<2, FLUX_ROE>(lim, a, s)
                          : launch_stage_l<2, FLUX_VAN_LEER>(lim, a, s);
}

// Tile rows used by the stage kernel for a (ndim, limiter) pair (the runtime
// cuts tiles to match).
int stage_tile_rows(int ndim, int lim) {
  if (ndim == 2) return TJ_2D;
  return lim == LIM_VAN_LEER || lim == LIM_MINMOD ? TJ_2D : TJ_3D;
}

cudaError_t launch_ghost(const GhostArgs& a, cudaStream_t s) {
  if (a.total_items == 0) return cudaSuccess;
  const long long nb = (a.total_items + 255) / 256;
  ghost_kernel<<<(unsigned)nb, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_reduce(const double* partial, const int* tile_begin, int nblocks, double* out,
                          cudaStream_t s) {
  if (nblocks == 0) return cudaSuccess;
  reduce_kernel<<<nblocks, 256, 0, s>>>(partial, tile_begin, nblocks, out);
  return cudaGetLastError();
}

}  // namespace BF_NS
}  // namespace bf
