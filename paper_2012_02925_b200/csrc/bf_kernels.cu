// bf_kernels.cu — the per-RK-stage device pipeline.
//
// Compiled twice by build.py: -DBF_EXACT=1 -fmad=false (namespace bf_exact,
// bitwise reference arithmetic) and -DBF_EXACT=0 (namespace bf_fast, FMA).
//
//   ghost_kernel   physical-BC ghost fill (solver.py:281-403), same-device
//                  connected copies and message pack/unpack (halo.py:47-115)
//                  for every block of the rank in ONE launch;
//   stage_kernel   fused limiter + MUSCL + face flux + boundary-flux
//                  overwrite + residual + (stage 0) local dt and sum(R^2) +
//                  RK update + decode (solver.py:413-753), 2.5-D k-streaming
//                  over TIxTJ column tiles, plane ring in shared memory filled
//                  by cp.async;
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
// small helpers
// ---------------------------------------------------------------------------
BF_DEV void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
BF_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
BF_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

BF_DEV void record_error(unsigned long long* err, unsigned long long key) {
  if (key < *reinterpret_cast<volatile unsigned long long*>(err)) atomicMin(err, key);
}

// Shared-memory layout of the stage kernel (doubles).
template <int NDIM>
struct Smem {
  static constexpr int NS = (NDIM == 3) ? NSLOT : 1;
  static constexpr int W = 0;                                   // [NS][5][PLANE]
  static constexpr int PX = W + NS * 5 * PLANE;                 // [2][5][TJ][TI+2]
  static constexpr int PY = PX + 2 * 5 * TJ * (TI + 2);         // [2][5][TJ+2][TI]
  static constexpr int FX = PY + 2 * 5 * (TJ + 2) * TI;         // [5][TJ][TI+1]
  static constexpr int FY = FX + 5 * TJ * (TI + 1);             // [5][TJ+1][TI]
  static constexpr int TOTAL = FY + 5 * (TJ + 1) * TI;
  static constexpr size_t BYTES = sizeof(double) * TOTAL;
};

BF_DEV int pidx(int ii, int jj) { return (jj + HALO) * PW + (ii + HALO); }

// Issue the cp.async copies of one k-plane (cross-shaped region: the tile
// plus a 2-cell halo in i and in j) of the 5 primitive fields.
template <int NDIM>
BF_DEV void load_plane(double* sw, const DevBlock& b, const double* const* W, int i0, int j0,
                       int k) {
  if (NDIM == 3 && (k < -HALO || k >= b.n[2] + HALO)) return;
  const long long kofs = (NDIM == 3) ? b.sz * (long long)k : 0;
  constexpr int ROWS_FULL = TJ * PW;              // rows 0..TJ-1, ii = -2..TI+1
  constexpr int ROWS_HALO = 2 * HALO * TI;        // rows -2,-1,TJ,TJ+1, ii = 0..TI-1
  for (int q = threadIdx.x; q < ROWS_FULL + ROWS_HALO; q += NT) {
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
    if (gi < -HALO || gi >= b.n[0] + HALO || gj < -HALO || gj >= b.n[1] + HALO) continue;
    const long long off = gi + b.sy * (long long)gj + kofs;
    const int s = pidx(ii, jj);
#pragma unroll
    for (int v = 0; v < 5; ++v) cp_async8(sw + v * PLANE + s, W[v] + off);
  }
}

BF_DEV St load_st(const double* p, int stride) {
  St s;
  s.r = p[0];
  s.u = p[stride];
  s.v = p[2 * stride];
  s.w = p[3 * stride];
  s.p = p[4 * stride];
  return s;
}

// psi+ / psi- of one cell from its three stencil values (solver.py:419-435):
// psi+_c = phi(D_{c+1}, D_c), psi-_c = phi(D_c, D_{c+1}).
template <int LIM>
BF_DEV void cell_limiter(double wm, double w0, double wp, double& pp, double& pm) {
  const double lo = w0 - wm;
  const double hi = wp - w0;
  pp = limiter<LIM>(hi, lo);
  pm = limiter<LIM>(lo, hi);
}

// MUSCL face states (solver.py:437-474) + flux (physics.py) + area scaling
// (solver.py:519) + boundary overwrite (solver.py:526-580) for one face.
// c0..c3 point at var 0 of cells f-2, f-1, f, f+1 (var stride vs); pl/ml and
// pr/mr at var 0 of psi+/psi- of cells f-1 and f (var stride ps).
// Returns an error kind (0 ok).
template <int FLUX>
BF_DEV int face_flux(const double* c0, const double* c1, const double* c2, const double* c3,
                     int vs, const double* pl, const double* ml, const double* pr,
                     const double* mr, int ps, double nx, double ny, double nz, double A,
                     int bkind, double side_sign, const Consts& c, double F[5]) {
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
      qL[v] = wl + c.quarter * (c.omk * pl[v * ps] * dm + c.opk * ml[v * ps] * d0);
      qR[v] = wr - c.quarter * (c.opk * pr[v * ps] * d0 + c.omk * mr[v * ps] * dp);
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
      const St s1 = load_st(in1, vs);
      const St qb = farfield_state(s1, side_sign * nx, side_sign * ny, side_sign * nz, c);
      double Fb[5];
      euler_flux(qb, nx, ny, nz, c, Fb);
#pragma unroll
      for (int e = 0; e < 5; ++e) F[e] = Fb[e] * A;
    }
  }
  return err;
}

// ---------------------------------------------------------------------------
// the fused stage kernel
// ---------------------------------------------------------------------------
template <int NDIM, int FLUX, int LIM>
__global__ void __launch_bounds__(NT, 1) stage_kernel(const StageArgs a) {
  using S = Smem<NDIM>;
  extern __shared__ __align__(16) double smem[];
  double* sW = smem + S::W;
  double* sPX = smem + S::PX;
  double* sPY = smem + S::PY;
  double* sFX = smem + S::FX;
  double* sFY = smem + S::FY;
  constexpr int PXS = 5 * TJ * (TI + 2);      // plus->minus offset
  constexpr int PYS = 5 * (TJ + 2) * TI;

  const Tile t = a.tiles[blockIdx.x];
  const DevBlock& b = a.blocks[t.block];
  const Consts& c = a.c;
  const int tx = threadIdx.x % TI, ty = threadIdx.x / TI;
  const int i0 = t.i0, j0 = t.j0, k0 = t.k0;
  const int ni = b.n[0], nj = b.n[1], nk = b.n[2];
  const int i = i0 + tx, j = j0 + ty;
  const bool col_on = (i < ni) && (j < nj);
  const bool stage0 = a.flags & F_STAGE0;
  const bool last = a.flags & F_LAST;
  const bool psi_load = a.flags & F_PSI_LOAD;
  const bool psi_store = a.flags & F_PSI_STORE;
  const double* const* Win = b.W[a.cur];
  double* const* Wout = b.W[a.cur ^ 1];
  const int stage = a.stage;

  double rsum[5] = {0.0, 0.0, 0.0, 0.0, 0.0};

  // plane slot of k (ring of NS planes)
  auto slot = [&](int k) -> double* {
    if constexpr (NDIM == 3) return sW + (((k - k0 + 2 * NSLOT) % NSLOT) * 5 * PLANE);
    else return sW;
  };

  // z-direction carried state (NDIM == 3)
  double pzp[5], pzm[5];    // psi+/psi- at cell k (own column)
  double fz[5];             // flux at face k (own column)

  const int kfirst = (NDIM == 3) ? -1 : 0;
  if constexpr (NDIM == 3) {
    // prologue: planes k0-2 .. k0+1
    for (int k = k0 - 2; k <= k0 + 1; ++k) load_plane<3>(slot(k), b, Win, i0, j0, k);
    cp_async_commit();
  } else {
    load_plane<2>(sW, b, Win, i0, j0, 0);
    cp_async_commit();
  }

  for (int kk = kfirst; kk < t.kc; ++kk) {
    const int k = k0 + kk;
    cp_async_wait_all();
    __syncthreads();
    if constexpr (NDIM == 3) {
      if (kk + 1 < t.kc) load_plane<3>(slot(k + 3), b, Win, i0, j0, k + 3);
      cp_async_commit();
    }
    const bool xy = (kk >= 0);
    const long long kofs = (NDIM == 3) ? b.sz * (long long)k : 0;
    const double* pk = slot(k);

    // ---- P1: limiters -------------------------------------------------------
    if constexpr (NDIM == 3) {
      // psi_z of cell k+1 (and, in the prologue iteration, of cell k = k0-1)
      const double* pm1 = slot(k - 1);
      const double* p0 = slot(k);
      const double* p1 = slot(k + 1);
      const double* p2 = slot(k + 2);
      const int s = pidx(tx, ty);
      const long long cz = i + b.sy * (long long)j;
      if (kk == kfirst) {
        if (psi_load) {
          if (col_on) {
#pragma unroll
            for (int v = 0; v < 5; ++v) {
              pzp[v] = b.psi[2][0][v][cz + b.sz * (long long)k];
              pzm[v] = b.psi[2][1][v][cz + b.sz * (long long)k];
            }
          }
        } else {
#pragma unroll
          for (int v = 0; v < 5; ++v)
            cell_limiter<LIM>(pm1[v * PLANE + s], p0[v * PLANE + s], p1[v * PLANE + s], pzp[v],
                              pzm[v]);
          if (psi_store && col_on && k >= -1) {
#pragma unroll
            for (int v = 0; v < 5; ++v) {
              b.psi[2][0][v][cz + b.sz * (long long)k] = pzp[v];
              b.psi[2][1][v][cz + b.sz * (long long)k] = pzm[v];
            }
          }
        }
      }
      // psi of cell k+1 stored in registers as "next"
      double nzp[5], nzm[5];
      if (psi_load) {
        if (col_on) {
#pragma unroll
          for (int v = 0; v < 5; ++v) {
            nzp[v] = b.psi[2][0][v][cz + b.sz * (long long)(k + 1)];
            nzm[v] = b.psi[2][1][v][cz + b.sz * (long long)(k + 1)];
          }
        }
      } else {
#pragma unroll
        for (int v = 0; v < 5; ++v)
          cell_limiter<LIM>(p0[v * PLANE + s], p1[v * PLANE + s], p2[v * PLANE + s], nzp[v],
                            nzm[v]);
        if (psi_store && col_on && k + 1 <= nk) {
#pragma unroll
          for (int v = 0; v < 5; ++v) {
            b.psi[2][0][v][cz + b.sz * (long long)(k + 1)] = nzp[v];
            b.psi[2][1][v][cz + b.sz * (long long)(k + 1)] = nzm[v];
          }
        }
      }
      // z face k+1: cells k-1, k, k+1, k+2; psi of cells k and k+1
      {
        const int fk = k + 1;
        double F[5];
        const long long fo = cz + b.sz * (long long)fk;
        double nx = 0, ny = 0, nz = 0, A = 0;
        if (col_on) {
          nx = b.fn[2][0][fo];
          ny = b.fn[2][1][fo];
          nz = b.fn[2][2][fo];
          A = b.fn[2][3][fo];
        }
        int bk = BFACE_NONE;
        double sgn = 1.0;
        if (col_on && fk == 0) {
          bk = b.bface[4][i + ni * j];
          sgn = -1.0;
        } else if (col_on && fk == nk) {
          bk = b.bface[5][i + ni * j];
        }
        const int e = face_flux<FLUX>(pm1 + s, p0 + s, p1 + s, p2 + s, PLANE, pzp, pzm, nzp,
                                      nzm, 1, nx, ny, nz, A, bk, sgn, c, F);
        if (e && col_on) {
          const unsigned long long lin =
              ((unsigned long long)i * nj + j) * (unsigned long long)(nk + 1) + fk;
          record_error(a.err, make_err_key(stage, 0, b.order, 2, e, lin));
        }
        if (kk == kfirst) {
#pragma unroll
          for (int v = 0; v < 5; ++v) fz[v] = F[v];
        }
        // carry limiter state
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          pzp[v] = nzp[v];
          pzm[v] = nzm[v];
        }
        if (kk == kfirst) continue;   // prologue iteration: z only
        // x / y limiters for plane k
        if (!psi_load) {
          for (int q = threadIdx.x; q < TJ * (TI + 2) + (TJ + 2) * TI; q += NT) {
            if (q < TJ * (TI + 2)) {
              const int row = q / (TI + 2), cc = q % (TI + 2) - 1;   // cell cc in [-1, TI]
              const int sc = pidx(cc, row);
              const int o = row * (TI + 2) + (cc + 1);
#pragma unroll
              for (int v = 0; v < 5; ++v)
                cell_limiter<LIM>(pk[v * PLANE + sc - 1], pk[v * PLANE + sc],
                                  pk[v * PLANE + sc + 1], sPX[v * TJ * (TI + 2) + o],
                                  sPX[PXS + v * TJ * (TI + 2) + o]);
              const int gi = i0 + cc, gj = j0 + row;
              if (psi_store && gi >= -1 && gi <= ni && gj < nj) {
                const long long go = gi + b.sy * (long long)gj + kofs;
#pragma unroll
                for (int v = 0; v < 5; ++v) {
                  b.psi[0][0][v][go] = sPX[v * TJ * (TI + 2) + o];
                  b.psi[0][1][v][go] = sPX[PXS + v * TJ * (TI + 2) + o];
                }
              }
            } else {
              const int q2 = q - TJ * (TI + 2);
              const int row = q2 / TI - 1, cc = q2 % TI;            // row in [-1, TJ]
              const int sc = pidx(cc, row);
              const int o = (row + 1) * TI + cc;
#pragma unroll
              for (int v = 0; v < 5; ++v)
                cell_limiter<LIM>(pk[v * PLANE + sc - PW], pk[v * PLANE + sc],
                                  pk[v * PLANE + sc + PW], sPY[v * (TJ + 2) * TI + o],
                                  sPY[PYS + v * (TJ + 2) * TI + o]);
              const int gi = i0 + cc, gj = j0 + row;
              if (psi_store && gj >= -1 && gj <= nj && gi < ni) {
                const long long go = gi + b.sy * (long long)gj + kofs;
#pragma unroll
                for (int v = 0; v < 5; ++v) {
                  b.psi[1][0][v][go] = sPY[v * (TJ + 2) * TI + o];
                  b.psi[1][1][v][go] = sPY[PYS + v * (TJ + 2) * TI + o];
                }
              }
            }
          }
        } else {
          for (int q = threadIdx.x; q < TJ * (TI + 2) + (TJ + 2) * TI; q += NT) {
            int gi, gj, o, d;
            if (q < TJ * (TI + 2)) {
              const int row = q / (TI + 2), cc = q % (TI + 2) - 1;
              gi = i0 + cc;
              gj = j0 + row;
              o = row * (TI + 2) + (cc + 1);
              d = 0;
              if (gi < -1 || gi > ni || gj >= nj) continue;
            } else {
              const int q2 = q - TJ * (TI + 2);
              const int row = q2 / TI - 1, cc = q2 % TI;
              gi = i0 + cc;
              gj = j0 + row;
              o = (row + 1) * TI + cc;
              d = 1;
              if (gj < -1 || gj > nj || gi >= ni) continue;
            }
            const long long go = gi + b.sy * (long long)gj + kofs;
            double* dp = (d == 0) ? sPX : sPY;
            const int stride = (d == 0) ? TJ * (TI + 2) : (TJ + 2) * TI;
            const int ms = (d == 0) ? PXS : PYS;
#pragma unroll
            for (int v = 0; v < 5; ++v) {
              dp[v * stride + o] = b.psi[d][0][v][go];
              dp[ms + v * stride + o] = b.psi[d][1][v][go];
            }
          }
        }
        __syncthreads();
        // ---- P2: x / y face fluxes of plane k ------------------------------------
        for (int q = threadIdx.x; q < TJ * (TI + 1) + (TJ + 1) * TI; q += NT) {
          double Fq[5];
          if (q < TJ * (TI + 1)) {
            const int row = q / (TI + 1), f = q % (TI + 1);      // face f: cells f-1 | f
            const int gi = i0 + f, gj = j0 + row;
            const bool on = gi <= ni && gj < nj;
            double nx = 0, ny = 0, nz = 0, A = 0;
            int bk = BFACE_NONE;
            double sgn = 1.0;
            if (on) {
              const long long fo = gi + b.sy * (long long)gj + kofs;
              nx = b.fn[0][0][fo];
              ny = b.fn[0][1][fo];
              nz = b.fn[0][2][fo];
              A = b.fn[0][3][fo];
              if (gi == 0) {
                bk = b.bface[0][gj + nj * (NDIM == 3 ? k : 0)];
                sgn = -1.0;
              } else if (gi == ni) {
                bk = b.bface[1][gj + nj * (NDIM == 3 ? k : 0)];
              }
            }
            const int sc = pidx(f, row);
            const int po = row * (TI + 2) + f;      // psi cell f-1 at index (f-1)+1
            const int e = face_flux<FLUX>(pk + sc - 2, pk + sc - 1, pk + sc, pk + sc + 1, PLANE,
                                          sPX + po, sPX + PXS + po, sPX + po + 1,
                                          sPX + PXS + po + 1, TJ * (TI + 2), nx, ny, nz, A, bk,
                                          sgn, c, Fq);
            if (e && on) {
              const unsigned long long lin =
                  ((unsigned long long)gi * nj + gj) * (unsigned long long)(NDIM == 3 ? nk : 1) +
                  (NDIM == 3 ? k : 0);
              record_error(a.err, make_err_key(stage, 0, b.order, 0, e, lin));
            }
#pragma unroll
            for (int v = 0; v < 5; ++v) sFX[v * TJ * (TI + 1) + row * (TI + 1) + f] = Fq[v];
          } else {
            const int q2 = q - TJ * (TI + 1);
            const int f = q2 / TI, col = q2 % TI;          // face row f: cells f-1 | f
            const int gi = i0 + col, gj = j0 + f;
            const bool on = gj <= nj && gi < ni;
            double nx = 0, ny = 0, nz = 0, A = 0;
            int bk = BFACE_NONE;
            double sgn = 1.0;
            if (on) {
              const long long fo = gi + b.sy * (long long)gj + kofs;
              nx = b.fn[1][0][fo];
              ny = b.fn[1][1][fo];
              nz = b.fn[1][2][fo];
              A = b.fn[1][3][fo];
              if (gj == 0) {
                bk = b.bface[2][gi + ni * (NDIM == 3 ? k : 0)];
                sgn = -1.0;
              } else if (gj == nj) {
                bk = b.bface[3][gi + ni * (NDIM == 3 ? k : 0)];
              }
            }
            const int sc = pidx(col, f);
            const int po = f * TI + col;             // psi row f-1 at index ((f-1)+1)*TI
            const int e = face_flux<FLUX>(pk + sc - 2 * PW, pk + sc - PW, pk + sc, pk + sc + PW,
                                          PLANE, sPY + po, sPY + PYS + po, sPY + po + TI,
                                          sPY + PYS + po + TI, (TJ + 2) * TI, nx, ny, nz, A, bk,
                                          sgn, c, Fq);
            if (e && on) {
              const unsigned long long lin =
                  ((unsigned long long)gi * (nj + 1) + gj) *
                      (unsigned long long)(NDIM == 3 ? nk : 1) +
                  (NDIM == 3 ? k : 0);
              record_error(a.err, make_err_key(stage, 0, b.order, 1, e, lin));
            }
#pragma unroll
            for (int v = 0; v < 5; ++v) sFY[v * (TJ + 1) * TI + f * TI + col] = Fq[v];
          }
        }
        __syncthreads();
        // ---- P3: residual, dt, update of cell (i, j, k) ----------------------------
        if (col_on) {
          double R[5];
#pragma unroll
          for (int v = 0; v < 5; ++v) {
            const double fxl = sFX[v * TJ * (TI + 1) + ty * (TI + 1) + tx];
            const double fxh = sFX[v * TJ * (TI + 1) + ty * (TI + 1) + tx + 1];
            const double fyl = sFY[v * (TJ + 1) * TI + ty * TI + tx];
            const double fyh = sFY[v * (TJ + 1) * TI + (ty + 1) * TI + tx];
            R[v] = ((0.0 + (fxh - fxl)) + (fyh - fyl)) + (F[v] - fz[v]);
          }
          const long long co = i + b.sy * (long long)j + kofs;
          if (a.flags & F_SOURCE) {
#pragma unroll
            for (int v = 0; v < 5; ++v) R[v] = R[v] - b.src[v][co];
          }
          double dtv;
          const int s0 = pidx(tx, ty);
          if (stage0) {
#pragma unroll
            for (int v = 0; v < 5; ++v) rsum[v] += R[v] * R[v];
            const double rho = pk[s0], u = pk[PLANE + s0], v = pk[2 * PLANE + s0],
                         w = pk[3 * PLANE + s0], p = pk[4 * PLANE + s0];
            const double snd = sqrt(c.gamma * p / rho);
            double lam = 0.0;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
#pragma unroll
              for (int hi = 0; hi < 2; ++hi) {
                const long long fo = co + (hi ? (d == 0 ? 1 : (d == 1 ? b.sy : b.sz)) : 0);
                const double nx = b.fn[d][0][fo], ny = b.fn[d][1][fo], nz = b.fn[d][2][fo],
                             A = b.fn[d][3][fo];
                lam = lam + (fabs(u * nx + v * ny + w * nz) + snd) * A;
              }
            }
            const double vol = b.vol[co];
            dtv = c.cfl * vol / lam / vol;
            b.dtv[co] = dtv;
          } else {
            dtv = b.dtv[co];
          }
          double qn[5];
          const double adt = a.alpha * dtv;
#pragma unroll
          for (int v = 0; v < 5; ++v) qn[v] = b.Q[v][co] - adt * R[v];
          const double uu = qn[1] / qn[0], vv = qn[2] / qn[0], ww = qn[3] / qn[0];
          const double pp = c.gm1 * (qn[4] - 0.5 * (qn[1] * uu + qn[2] * vv + qn[3] * ww));
          if (qn[0] <= 0.0 || pp <= 0.0) {
            const unsigned long long lin = ((unsigned long long)i * nj + j) * nk + k;
            record_error(a.err, make_err_key(stage, 1, b.order, 0, 0, lin));
          }
          Wout[0][co] = qn[0];
          Wout[1][co] = uu;
          Wout[2][co] = vv;
          Wout[3][co] = ww;
          Wout[4][co] = pp;
          if (last) {
#pragma unroll
            for (int v = 0; v < 5; ++v) b.Q[v][co] = qn[v];
          }
        }
#pragma unroll
        for (int v = 0; v < 5; ++v) fz[v] = F[v];
      }
    } else {
      // ------------------------------ 2D --------------------------------------
      if (!psi_load) {
        for (int q = threadIdx.x; q < TJ * (TI + 2) + (TJ + 2) * TI; q += NT) {
          if (q < TJ * (TI + 2)) {
            const int row = q / (TI + 2), cc = q % (TI + 2) - 1;
            const int sc = pidx(cc, row);
            const int o = row * (TI + 2) + (cc + 1);
#pragma unroll
            for (int v = 0; v < 5; ++v)
              cell_limiter<LIM>(pk[v * PLANE + sc - 1], pk[v * PLANE + sc], pk[v * PLANE + sc + 1],
                                sPX[v * TJ * (TI + 2) + o], sPX[PXS + v * TJ * (TI + 2) + o]);
            const int gi = i0 + cc, gj = j0 + row;
            if (psi_store && gi >= -1 && gi <= ni && gj < nj) {
              const long long go = gi + b.sy * (long long)gj;
#pragma unroll
              for (int v = 0; v < 5; ++v) {
                b.psi[0][0][v][go] = sPX[v * TJ * (TI + 2) + o];
                b.psi[0][1][v][go] = sPX[PXS + v * TJ * (TI + 2) + o];
              }
            }
          } else {
            const int q2 = q - TJ * (TI + 2);
            const int row = q2 / TI - 1, cc = q2 % TI;
            const int sc = pidx(cc, row);
            const int o = (row + 1) * TI + cc;
#pragma unroll
            for (int v = 0; v < 5; ++v)
              cell_limiter<LIM>(pk[v * PLANE + sc - PW], pk[v * PLANE + sc],
                                pk[v * PLANE + sc + PW], sPY[v * (TJ + 2) * TI + o],
                                sPY[PYS + v * (TJ + 2) * TI + o]);
            const int gi = i0 + cc, gj = j0 + row;
            if (psi_store && gj >= -1 && gj <= nj && gi < ni) {
              const long long go = gi + b.sy * (long long)gj;
#pragma unroll
              for (int v = 0; v < 5; ++v) {
                b.psi[1][0][v][go] = sPY[v * (TJ + 2) * TI + o];
                b.psi[1][1][v][go] = sPY[PYS + v * (TJ + 2) * TI + o];
              }
            }
          }
        }
      } else {
        for (int q = threadIdx.x; q < TJ * (TI + 2) + (TJ + 2) * TI; q += NT) {
          int gi, gj, o, d;
          if (q < TJ * (TI + 2)) {
            const int row = q / (TI + 2), cc = q % (TI + 2) - 1;
            gi = i0 + cc;
            gj = j0 + row;
            o = row * (TI + 2) + (cc + 1);
            d = 0;
            if (gi < -1 || gi > ni || gj >= nj) continue;
          } else {
            const int q2 = q - TJ * (TI + 2);
            const int row = q2 / TI - 1, cc = q2 % TI;
            gi = i0 + cc;
            gj = j0 + row;
            o = (row + 1) * TI + cc;
            d = 1;
            if (gj < -1 || gj > nj || gi >= ni) continue;
          }
          const long long go = gi + b.sy * (long long)gj;
          double* dp = (d == 0) ? sPX : sPY;
          const int stride = (d == 0) ? TJ * (TI + 2) : (TJ + 2) * TI;
          const int ms = (d == 0) ? PXS : PYS;
#pragma unroll
          for (int v = 0; v < 5; ++v) {
            dp[v * stride + o] = b.psi[d][0][v][go];
            dp[ms + v * stride + o] = b.psi[d][1][v][go];
          }
        }
      }
      __syncthreads();
      for (int q = threadIdx.x; q < TJ * (TI + 1) + (TJ + 1) * TI; q += NT) {
        double Fq[5];
        if (q < TJ * (TI + 1)) {
          const int row = q / (TI + 1), f = q % (TI + 1);
          const int gi = i0 + f, gj = j0 + row;
          const bool on = gi <= ni && gj < nj;
          double nx = 0, ny = 0, nz = 0, A = 0;
          int bk = BFACE_NONE;
          double sgn = 1.0;
          if (on) {
            const long long fo = gi + b.sy * (long long)gj;
            nx = b.fn[0][0][fo];
            ny = b.fn[0][1][fo];
            nz = b.fn[0][2][fo];
            A = b.fn[0][3][fo];
            if (gi == 0) {
              bk = b.bface[0][gj];
              sgn = -1.0;
            } else if (gi == ni) {
              bk = b.bface[1][gj];
            }
          }
          const int sc = pidx(f, row);
          const int po = row * (TI + 2) + f;
          const int e = face_flux<FLUX>(pk + sc - 2, pk + sc - 1, pk + sc, pk + sc + 1, PLANE,
                                        sPX + po, sPX + PXS + po, sPX + po + 1, sPX + PXS + po + 1,
                                        TJ * (TI + 2), nx, ny, nz, A, bk, sgn, c, Fq);
          if (e && on) {
            const unsigned long long lin = (unsigned long long)gi * nj + gj;
            record_error(a.err, make_err_key(stage, 0, b.order, 0, e, lin));
          }
#pragma unroll
          for (int v = 0; v < 5; ++v) sFX[v * TJ * (TI + 1) + row * (TI + 1) + f] = Fq[v];
        } else {
          const int q2 = q - TJ * (TI + 1);
          const int f = q2 / TI, col = q2 % TI;
          const int gi = i0 + col, gj = j0 + f;
          const bool on = gj <= nj && gi < ni;
          double nx = 0, ny = 0, nz = 0, A = 0;
          int bk = BFACE_NONE;
          double sgn = 1.0;
          if (on) {
            const long long fo = gi + b.sy * (long long)gj;
            nx = b.fn[1][0][fo];
            ny = b.fn[1][1][fo];
            nz = b.fn[1][2][fo];
            A = b.fn[1][3][fo];
            if (gj == 0) {
              bk = b.bface[2][gi];
              sgn = -1.0;
            } else if (gj == nj) {
              bk = b.bface[3][gi];
            }
          }
          const int sc = pidx(col, f);
          const int po = f * TI + col;
          const int e = face_flux<FLUX>(pk + sc - 2 * PW, pk + sc - PW, pk + sc, pk + sc + PW,
                                        PLANE, sPY + po, sPY + PYS + po, sPY + po + TI,
                                        sPY + PYS + po + TI, (TJ + 2) * TI, nx, ny, nz, A, bk,
                                        sgn, c, Fq);
          if (e && on) {
            const unsigned long long lin = (unsigned long long)gi * (nj + 1) + gj;
            record_error(a.err, make_err_key(stage, 0, b.order, 1, e, lin));
          }
#pragma unroll
          for (int v = 0; v < 5; ++v) sFY[v * (TJ + 1) * TI + f * TI + col] = Fq[v];
        }
      }
      __syncthreads();
      if (col_on) {
        double R[5];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          const double fxl = sFX[v * TJ * (TI + 1) + ty * (TI + 1) + tx];
          const double fxh = sFX[v * TJ * (TI + 1) + ty * (TI + 1) + tx + 1];
          const double fyl = sFY[v * (TJ + 1) * TI + ty * TI + tx];
          const double fyh = sFY[v * (TJ + 1) * TI + (ty + 1) * TI + tx];
          R[v] = (0.0 + (fxh - fxl)) + (fyh - fyl);
        }
        const long long co = i + b.sy * (long long)j;
        if (a.flags & F_SOURCE) {
#pragma unroll
          for (int v = 0; v < 5; ++v) R[v] = R[v] - b.src[v][co];
        }
        double dtv;
        const int s0 = pidx(tx, ty);
        if (stage0) {
#pragma unroll
          for (int v = 0; v < 5; ++v) rsum[v] += R[v] * R[v];
          const double rho = pk[s0], u = pk[PLANE + s0], v = pk[2 * PLANE + s0],
                       w = pk[3 * PLANE + s0], p = pk[4 * PLANE + s0];
          const double snd = sqrt(c.gamma * p / rho);
          double lam = 0.0;
#pragma unroll
          for (int d = 0; d < 2; ++d) {
#pragma unroll
            for (int hi = 0; hi < 2; ++hi) {
              const long long fo = co + (hi ? (d == 0 ? 1 : b.sy) : 0);
              const double nx = b.fn[d][0][fo], ny = b.fn[d][1][fo], nz = b.fn[d][2][fo],
                           A = b.fn[d][3][fo];
              lam = lam + (fabs(u * nx + v * ny + w * nz) + snd) * A;
            }
          }
          const double vol = b.vol[co];
          dtv = c.cfl * vol / lam / vol;
          b.dtv[co] = dtv;
        } else {
          dtv = b.dtv[co];
        }
        double qn[5];
        const double adt = a.alpha * dtv;
#pragma unroll
        for (int v = 0; v < 5; ++v) qn[v] = b.Q[v][co] - adt * R[v];
        const double uu = qn[1] / qn[0], vv = qn[2] / qn[0], ww = qn[3] / qn[0];
        const double pp = c.gm1 * (qn[4] - 0.5 * (qn[1] * uu + qn[2] * vv + qn[3] * ww));
        if (qn[0] <= 0.0 || pp <= 0.0) {
          const unsigned long long lin = (unsigned long long)i * nj + j;
          record_error(a.err, make_err_key(stage, 1, b.order, 0, 0, lin));
        }
        Wout[0][co] = qn[0];
        Wout[1][co] = uu;
        Wout[2][co] = vv;
        Wout[3][co] = ww;
        Wout[4][co] = pp;
        if (last) {
#pragma unroll
          for (int v = 0; v < 5; ++v) b.Q[v][co] = qn[v];
        }
      }
    }
  }

  // ---- deterministic per-tile sum(R^2) ----------------------------------------
  if (stage0) {
    __syncthreads();
    double* red = smem;   // reuse the plane ring: [NT/32][5]
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      double x = rsum[v];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
      if ((threadIdx.x & 31) == 0) red[(threadIdx.x >> 5) * 5 + v] = x;
    }
    __syncthreads();
    if (threadIdx.x < 5) {
      double x = 0.0;
      for (int w = 0; w < NT / 32; ++w) x += red[w * 5 + threadIdx.x];
      a.partial[(long long)blockIdx.x * 5 + threadIdx.x] = x;
    }
  }
}

// ---------------------------------------------------------------------------
// ghost fill / pack / unpack (one launch per stage, all blocks)
// ---------------------------------------------------------------------------
BF_DEV double interior_T(const DevBlock& b, const double* const* W, long long o, int t_derived,
                         const Consts& c) {
  return t_derived ? W[4][o] / (W[0][o] * c.R) : W[5][o];
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
    // field list: rho u v [w] p T
    double val[6];
    if (t.src_block >= 0) {
      const DevBlock& sb = a.blocks[t.src_block];
      const double* const* W = sb.W[a.cur];
      int f = 0;
      val[f++] = W[0][soff];
      val[f++] = W[1][soff];
      val[f++] = W[2][soff];
      if (t.nfields == 6) val[f++] = W[3][soff];
      val[f++] = W[4][soff];
      val[f++] = interior_T(sb, W, soff, a.t_derived, c);
    } else {
      for (int f = 0; f < t.nfields; ++f) val[f] = t.src_buf[f * t.buf_cells + soff];
    }
    if (t.block >= 0) {
      double* const* W = a.blocks[t.block].W[a.cur];
      int f = 0;
      W[0][doff] = val[f++];
      W[1][doff] = val[f++];
      W[2][doff] = val[f++];
      if (t.nfields == 6) W[3][doff] = val[f++];
      W[4][doff] = val[f++];
      W[5][doff] = val[f++];
    } else {
      for (int f = 0; f < t.nfields; ++f) t.dst_buf[f * t.buf_cells + doff] = val[f];
    }
    return;
  }

  // ---- physical patch: one tangential position, all ghost layers ----------
  const DevBlock& b = a.blocks[t.block];
  double* const* W = b.W[a.cur];
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
      W[0][o] = c.fs_rho;
      W[1][o] = c.fs_u;
      W[2][o] = c.fs_v;
      W[3][o] = c.fs_w;
      W[4][o] = c.fs_p;
      W[5][o] = c.fs_T;
    }
  } else if (bc == BC_OUTFLOW) {
    const long long oi = base + st[d] * ipos(0);
    const double v0 = W[0][oi], v1 = W[1][oi], v2 = W[2][oi], v3 = W[3][oi], v4 = W[4][oi];
    const double v5 = interior_T(b, W, oi, a.t_derived, c);
    for (int L = 0; L < t.depth; ++L) {
      const long long o = base + st[d] * gpos(L);
      W[0][o] = v0;
      W[1][o] = v1;
      W[2][o] = v2;
      W[3][o] = v3;
      W[4][o] = v4;
      W[5][o] = v5;
    }
  } else if (bc == BC_SLIP || bc == BC_NOSLIP) {
    // outward unit normal on the boundary face plane
    const long long fo = base + st[d] * (t.side == 0 ? 0 : n);
    const double sg = t.side == 0 ? -1.0 : 1.0;
    const double nx = sg * b.fn[d][0][fo], ny = sg * b.fn[d][1][fo], nz = sg * b.fn[d][2][fo];
    for (int L = 0; L < t.depth; ++L) {
      const long long og = base + st[d] * gpos(L);
      const long long oi = base + st[d] * ipos(L);
      const double u = W[1][oi], v = W[2][oi], w = W[3][oi];
      if (bc == BC_SLIP) {
        const double vn = u * nx + v * ny + w * nz;
        W[1][og] = u - 2.0 * vn * nx;
        W[2][og] = v - 2.0 * vn * ny;
        W[3][og] = w - 2.0 * vn * nz;
      } else {
        W[1][og] = -u;
        W[2][og] = -v;
        W[3][og] = -w;
      }
      const double pg = W[4][oi];
      W[4][og] = pg;
      const double ti = interior_T(b, W, oi, a.t_derived, c);
      const double tg = (bc == BC_NOSLIP && c.has_tw) ? 2.0 * c.tw - ti : ti;
      W[5][og] = tg;
      W[0][og] = pg / (c.R * tg);
    }
  } else if (bc == BC_FARFIELD) {
    const long long fo = base + st[d] * (t.side == 0 ? 0 : n);
    const double sg = t.side == 0 ? -1.0 : 1.0;
    const double nx = sg * b.fn[d][0][fo], ny = sg * b.fn[d][1][fo], nz = sg * b.fn[d][2][fo];
    const long long oi = base + st[d] * ipos(0);
    const St s{W[0][oi], W[1][oi], W[2][oi], W[3][oi], W[4][oi]};
    const St q = farfield_state(s, nx, ny, nz, c);
    const double tb = q.p / (q.r * c.R);
    for (int L = 0; L < t.depth; ++L) {
      const long long o = base + st[d] * gpos(L);
      W[0][o] = q.r;
      W[1][o] = q.u;
      W[2][o] = q.v;
      W[3][o] = q.w;
      W[4][o] = q.p;
      W[5][o] = tb;
    }
  } else {   // mms_dirichlet: cached exact values
    const long long nt = (long long)t.tn[0] * t.tn[1];
    for (int L = 0; L < t.depth; ++L) {
      const long long o = base + st[d] * gpos(L);
      const double* src = t.dirichlet + (long long)L * 6 * nt + m;
      for (int f = 0; f < 6; ++f) W[f][o] = src[f * nt];
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
  auto k = stage_kernel<NDIM, FLUX, LIM>;
  const size_t bytes = Smem<NDIM>::BYTES;
  static unsigned long long attr_done = 0;   // one bit per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_done & (1ull << dev))) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)bytes);
    if (e != cudaSuccess) return e;
    attr_done |= (1ull << dev);
  }
  if (a.ntiles == 0) return cudaSuccess;
  k<<<a.ntiles, NT, bytes, s>>>(a);
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

size_t stage_smem_bytes(int ndim) { return ndim == 3 ? Smem<3>::BYTES : Smem<2>::BYTES; }

}  // namespace BF_NS
}  // namespace bf
