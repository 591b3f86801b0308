// bf_stage.cuh — the fused per-stage kernel (included by bf_kernels.cu inside
// namespace bf::BF_NS).
//
// One CTA owns a TI x TJ column tile of one block and marches KC cells in k.
// Per k-plane, three barrier-separated phases, each balanced across threads:
//   P1  every (cell, variable) limiter value of the plane's x and y stencils
//       (a flat loop: each thread gets the same number +-1 of scalar items),
//       stored to shared memory;
//   P2  face fluxes: own x-low face, own y-low face (+ one tile-edge face for
//       TI+TJ threads), then the own-column z face k+1 and its limiter; each
//       face's geometry was staged by cp.async into the very shared-memory
//       slot its flux is written to;
//   P3  residual, stage-0 local dt / sum(R^2), RK update and decode.
// Shared memory: a 4-slot ring of 5-variable primitive planes (k..k+2 resident,
// k+3 in flight, cp.async), limiter arrays, face slots, and per-cell Q0 + dt/V
// staging.  HBM is touched once per cell per stage for W, Q0, dt/V and the
// face geometry (plus the 2-cell i/j halo reads, mostly L2 hits).
#pragma once

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
  static constexpr int NLIM = NPX + NPY;
  static constexpr int NFX = (TI + 1) * TJ;               // x faces: f = 0..TI per row
  static constexpr int NFY = TI * (TJ + 1);               // y faces: rows f = 0..TJ
  static constexpr int NEXTRA = TI + TJ;                  // tile-edge faces (f = TI, row TJ)
  static constexpr int OW = 0;                            // [NS][5][PLANE]
  static constexpr int OPX = OW + NS * 5 * PLANE;         // [PC][5][NPX]
  static constexpr int OPY = OPX + PC * 5 * NPX;          // [PC][5][NPY]
  static constexpr int OFX = OPY + PC * 5 * NPY;          // [5][NFX] geometry, then flux
  static constexpr int OFY = OFX + 5 * NFX;               // [5][NFY]
  static constexpr int OQ = OFY + 5 * NFY;                // [6][NT] Q0 + dt/V (or V)
  static constexpr int TOTAL = OQ + 6 * NT;
  static constexpr size_t BYTES = sizeof(double) * TOTAL;
  BF_DEV static int pidx(int ii, int jj) { return (jj + HALO) * PW + (ii + HALO); }
};

template <int NDIM, int FLUX, int LIM>
__global__ void __launch_bounds__(Cfg<NDIM, LIM>::NT, 1) stage_kernel(const StageArgs a) {
  using K = Cfg<NDIM, LIM>;
  constexpr int NT = K::NT, TJ = K::TJ, PLANE = K::PLANE, PW = K::PW, PC = K::PC;
  constexpr int NFX = K::NFX, NFY = K::NFY, NPX = K::NPX, NPY = K::NPY;
  extern __shared__ __align__(16) double smem[];
  double* const sW = smem + K::OW;
  double* const sPX = smem + K::OPX;
  double* const sPY = smem + K::OPY;
  double* const sFX = smem + K::OFX;
  double* const sFY = smem + K::OFY;
  double* const sQ = smem + K::OQ;

  const Tile t = a.tiles[blockIdx.x];
  const DevBlock b = a.blocks[t.block];     // by value: no aliasing reloads
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

  // ---- cp.async producers -------------------------------------------------------
  auto load_plane = [&](int k) {   // tile + 2-cell i/j halo (cross shape), 5 vars
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
  // this thread's x/y faces of plane k: geometry (nx ny nz A) into their slots
  // (slot components 0..3; the flux later overwrites components 0..4)
  const int qx = ty * (TI + 1) + tx;                       // own x-low face
  const int qy = ty * TI + tx;                             // own y-low face
  const int ex = tid < TJ ? tid : -1;                      // extra x face f=TI, row tid
  const int ey = (tid >= TJ && tid < TJ + TI) ? tid - TJ : -1;   // extra y face row TJ
  auto face_on_x = [&](int f, int row) { return i0 + f <= ni && j0 + row < nj; };
  auto face_on_y = [&](int f, int col) { return j0 + f <= nj && i0 + col < ni; };
  auto stage_geo = [&](int k) {
    const long long kofs = (NDIM == 3) ? sz * (long long)k : 0;
    auto put = [&](double* slotbase, int q, int nq, int d, long long off) {
      const double* src = b.base + (long long)ffn(d, 0) * fsz + off;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) cp_async8(slotbase + cc * nq + q, src + cc * fsz);
    };
    if (face_on_x(tx, ty)) put(sFX, qx, NFX, 0, colofs + kofs);
    if (face_on_y(ty, tx)) put(sFY, qy, NFY, 1, colofs + kofs);
    if (ex >= 0 && face_on_x(TI, ex))
      put(sFX, ex * (TI + 1) + TI, NFX, 0, (i0 + TI) + sy * (long long)(j0 + ex) + kofs);
    if (ey >= 0 && face_on_y(TJ, ey))
      put(sFY, TJ * TI + ey, NFY, 1, (i0 + ey) + sy * (long long)(j0 + TJ) + kofs);
  };
  auto stage_q = [&](int k) {      // own cell's Q0 and dt/V (V at stage 0)
    if (!col_on) return;
    const long long o = colofs + ((NDIM == 3) ? sz * (long long)k : 0);
    const double* q = b.base + (long long)FQ * fsz + o;
#pragma unroll
    for (int v = 0; v < 5; ++v) cp_async8(sQ + v * NT + tid, q + v * fsz);
    cp_async8(sQ + 5 * NT + tid, b.base + (long long)(stage0 ? FVOL : FDTV) * fsz + o);
  };

  double rsum[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  // z-direction carried state (3D, own column)
  double wm1[5] = {0, 0, 0, 0, 0};  // W(k-1)
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
    stage_geo(0);
    stage_q(0);
    cp_async_commit();
  }

  // z limiter of cell kc from the own-column values of kc-1, kc, kc+1
  auto z_limiter = [&](int kc, double wm_[5], const double* p0, const double* p1, double pp[5],
                       double pm[5]) {
    const int s0 = K::pidx(tx, ty);
    const long long cz = colofs + sz * (long long)kc;
    if (psi_load) {
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        pp[v] = col_on ? psi_ptr(2, 0, v)[cz] : 0.0;
        pm[v] = (PC == 2) ? (col_on ? psi_ptr(2, 1, v)[cz] : 0.0) : pp[v];
      }
      return;
    }
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      cell_limiter<LIM>(wm_[v], p0[v * PLANE + s0], p1[v * PLANE + s0], pp[v], pm[v]);
      if (psi_store && col_on && kc >= -1 && kc <= nk) {
        psi_ptr(2, 0, v)[cz] = pp[v];
        psi_ptr(2, 1, v)[cz] = pm[v];
      }
    }
  };

  const int kfirst = (NDIM == 3) ? -1 : 0;
  for (int kk = kfirst; kk < t.kc; ++kk) {
    const int k = k0 + kk;
    const bool xy = kk >= 0;
    const long long kofs = (NDIM == 3) ? sz * (long long)k : 0;
    cp_async_wait_all();
    __syncthreads();   // B0: planes k..k+2 resident; iteration k-1 fully retired
    // producers for this iteration: [geometry + Q0 of plane k], [plane k+3]
    if constexpr (NDIM == 3) {
      if (xy) {
        stage_geo(k);
        stage_q(k);
      }
      cp_async_commit();
      if (kk + 1 < t.kc) load_plane(k + 3);
      cp_async_commit();
    }
    const double* pk = slot(k);
    const int s0 = K::pidx(tx, ty);

    if constexpr (NDIM == 3) {
      if (kk == kfirst) {
        // prologue: psi_z(k0-1), psi_z(k0) and the z face k0; no x/y work
        double nzp[5], nzm[5], Fz[5];
        z_limiter(k, wm1, slot(k), slot(k + 1), pzp, pzm);
        double w0[5];
#pragma unroll
        for (int v = 0; v < 5; ++v) w0[v] = slot(k)[v * PLANE + s0];
        z_limiter(k + 1, w0, slot(k + 1), slot(k + 2), nzp, nzm);
        double st[4][5];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          st[0][v] = wm1[v];
          st[1][v] = w0[v];
          st[2][v] = slot(k + 1)[v * PLANE + s0];
          st[3][v] = slot(k + 2)[v * PLANE + s0];
        }
        const int fk = k + 1;
        const long long fo = colofs + sz * (long long)fk;
        const double* fn = b.base + (long long)ffn(2, 0) * fsz + fo;
        double gnx = 0, gny = 0, gnz = 0, gA = 0;
        int bk = BFACE_NONE;
        double sg = 1.0;
        if (col_on) {
          gnx = __ldg(fn);
          gny = __ldg(fn + fsz);
          gnz = __ldg(fn + 2 * fsz);
          gA = __ldg(fn + 3 * fsz);
          if (fk == 0) {
            bk = b.bface[4][i + ni * j];
            sg = -1.0;
          } else if (fk == nk) {
            bk = b.bface[5][i + ni * j];
          }
        }
        const int ez = face_flux<FLUX, LIM>(st[0], st[1], st[2], st[3], 1, pzp, pzm, nzp, nzm, 1,
                                            gnx, gny, gnz, gA, bk, sg, c, Fz);
        if (ez && col_on) {
          const unsigned long long lin =
              ((unsigned long long)i * nj + j) * (unsigned long long)(nk + 1) + fk;
          record_error(a.err, make_err_key(stage, 0, b.order, 2, ez, lin));
        }
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          pzp[v] = nzp[v];
          pzm[v] = nzm[v];
          fz[v] = Fz[v];
          wm1[v] = w0[v];
        }
        continue;
      }
    }

    // ---- P1: every (cell, var) limiter value of the x and y stencils of plane k --
    if constexpr (PC > 0) {
      int v = 0, q = tid;
      while (q >= K::NLIM) {
        q -= K::NLIM;
        ++v;
      }
      for (; v < 5;) {
        int gi, gj, d, sc, step;
        double* dst;
        int vstride;
        if (q < NPX) {
          const int row = q / (TI + 2), cc = q % (TI + 2) - 1;    // cell cc in [-1, TI]
          gi = i0 + cc;
          gj = j0 + row;
          d = 0;
          sc = K::pidx(cc, row);
          step = 1;
          dst = sPX + q;
          vstride = NPX;
        } else {
          const int q2 = q - NPX;
          const int row = q2 / TI - 1, cc = q2 % TI;             // row in [-1, TJ]
          gi = i0 + cc;
          gj = j0 + row;
          d = 1;
          sc = K::pidx(cc, row);
          step = PW;
          dst = sPY + q2;
          vstride = NPY;
        }
        const bool in_range = (d == 0) ? (gi >= -1 && gi <= ni && gj < nj)
                                       : (gj >= -1 && gj <= nj && gi < ni);
        const long long go = gi + sy * (long long)gj + kofs;
        if (psi_load) {
          if (in_range) {
            dst[v * vstride] = psi_ptr(d, 0, v)[go];
            if constexpr (PC == 2) dst[(5 + v) * vstride] = psi_ptr(d, 1, v)[go];
          }
        } else {
          double pp, pm;
          const double* w = pk + v * PLANE + sc;
          cell_limiter<LIM>(w[-step], w[0], w[step], pp, pm);
          dst[v * vstride] = pp;
          if constexpr (PC == 2) dst[(5 + v) * vstride] = pm;
          if (psi_store && in_range) {
            psi_ptr(d, 0, v)[go] = pp;
            psi_ptr(d, 1, v)[go] = pm;
          }
        }
        q += NT;
        while (q >= K::NLIM) {
          q -= K::NLIM;
          ++v;
        }
      }
    }
    cp_async_wait_1();   // own geometry + Q0 staging landed (plane k+3 may be in flight)
    __syncthreads();     // B1: limiters and staged geometry visible

    // ---- stage 0: local time step of the own cell (solver.py:696-731) -------------
    double dtv = 0.0;
    if (stage0) {
      if (col_on) {
        const double rho = pk[s0], u = pk[PLANE + s0], v = pk[2 * PLANE + s0],
                     w = pk[3 * PLANE + s0], p = pk[4 * PLANE + s0];
        const double snd = BF_SQRT(BF_DIV(c.gamma * p, rho));
        double lam = 0.0;
        auto term = [&](double nx, double ny, double nz, double A) {
          lam = lam + (fabs(u * nx + v * ny + w * nz) + snd) * A;
        };
        term(sFX[qx], sFX[NFX + qx], sFX[2 * NFX + qx], sFX[3 * NFX + qx]);
        term(sFX[qx + 1], sFX[NFX + qx + 1], sFX[2 * NFX + qx + 1], sFX[3 * NFX + qx + 1]);
        term(sFY[qy], sFY[NFY + qy], sFY[2 * NFY + qy], sFY[3 * NFY + qy]);
        term(sFY[qy + TI], sFY[NFY + qy + TI], sFY[2 * NFY + qy + TI], sFY[3 * NFY + qy + TI]);
        if constexpr (NDIM == 3) {
          const long long co = colofs + kofs;
          for (int hi = 0; hi < 2; ++hi) {
            const double* fn = b.base + (long long)ffn(2, 0) * fsz + co + (hi ? sz : 0);
            term(__ldg(fn), __ldg(fn + fsz), __ldg(fn + 2 * fsz), __ldg(fn + 3 * fsz));
          }
        }
        const double vol = sQ[5 * NT + tid];
#if BF_EXACT
        dtv = c.cfl * vol / lam / vol;
#else
        dtv = c.cfl * BF_RCP(lam);
#endif
        b.base[(long long)FDTV * fsz + colofs + kofs] = dtv;
      }
      __syncthreads();   // geometry slots are about to be overwritten by fluxes
    }

    // ---- P2: x / y faces of plane k (geometry slot -> flux slot) --------------------
    auto x_face = [&](int f, int row) {
      const int q = row * (TI + 1) + f;
      const int gi = i0 + f, gj = j0 + row;
      const bool on = face_on_x(f, row);
      int bk = BFACE_NONE;
      double sg = 1.0;
      if (on && gi == 0) {
        bk = b.bface[0][gj + nj * (NDIM == 3 ? k : 0)];
        sg = -1.0;
      } else if (on && gi == ni) {
        bk = b.bface[1][gj + nj * (NDIM == 3 ? k : 0)];
      }
      const int sc = K::pidx(f, row);
      const int po = row * (TI + 2) + f;            // psi of cell f-1 (index (f-1)+1)
      double F[5];
      const int e = face_flux<FLUX, LIM>(pk + sc - 2, pk + sc - 1, pk + sc, pk + sc + 1, PLANE,
                                         sPX + po, sPX + (PC == 2 ? 5 * NPX : 0) + po,
                                         sPX + po + 1, sPX + (PC == 2 ? 5 * NPX : 0) + po + 1,
                                         NPX, sFX[q], sFX[NFX + q], sFX[2 * NFX + q],
                                         on ? sFX[3 * NFX + q] : 0.0, bk, sg, c, F);
      if (e && on) {
        const unsigned long long lin =
            ((unsigned long long)gi * nj + gj) * (unsigned long long)(NDIM == 3 ? nk : 1) +
            (NDIM == 3 ? k : 0);
        record_error(a.err, make_err_key(stage, 0, b.order, 0, e, lin));
      }
#pragma unroll
      for (int v = 0; v < 5; ++v) sFX[v * NFX + q] = F[v];
    };
    auto y_face = [&](int f, int col) {
      const int q = f * TI + col;
      const int gi = i0 + col, gj = j0 + f;
      const bool on = face_on_y(f, col);
      int bk = BFACE_NONE;
      double sg = 1.0;
      if (on && gj == 0) {
        bk = b.bface[2][gi + ni * (NDIM == 3 ? k : 0)];
        sg = -1.0;
      } else if (on && gj == nj) {
        bk = b.bface[3][gi + ni * (NDIM == 3 ? k : 0)];
      }
      const int sc = K::pidx(col, f);
      const int po = f * TI + col;                  // psi of row f-1 (index (f-1)+1)
      double F[5];
      const int e = face_flux<FLUX, LIM>(pk + sc - 2 * PW, pk + sc - PW, pk + sc, pk + sc + PW,
                                         PLANE, sPY + po, sPY + (PC == 2 ? 5 * NPY : 0) + po,
                                         sPY + po + TI, sPY + (PC == 2 ? 5 * NPY : 0) + po + TI,
                                         NPY, sFY[q], sFY[NFY + q], sFY[2 * NFY + q],
                                         on ? sFY[3 * NFY + q] : 0.0, bk, sg, c, F);
      if (e && on) {
        const unsigned long long lin =
            ((unsigned long long)gi * (nj + 1) + gj) * (unsigned long long)(NDIM == 3 ? nk : 1) +
            (NDIM == 3 ? k : 0);
        record_error(a.err, make_err_key(stage, 0, b.order, 1, e, lin));
      }
#pragma unroll
      for (int v = 0; v < 5; ++v) sFY[v * NFY + q] = F[v];
    };
    x_face(tx, ty);
    y_face(ty, tx);
    if (ex >= 0) x_face(TI, ex);
    if (ey >= 0) y_face(TJ, ey);

    // z limiter of cell k+1 and the z face k+1 (own column, registers)
    double Fz[5] = {0, 0, 0, 0, 0};
    if constexpr (NDIM == 3) {
      double nzp[5], nzm[5];
      double w0[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) w0[v] = pk[v * PLANE + s0];
      z_limiter(k + 1, w0, slot(k + 1), slot(k + 2), nzp, nzm);
      double st[4][5];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        st[0][v] = wm1[v];
        st[1][v] = w0[v];
        st[2][v] = slot(k + 1)[v * PLANE + s0];
        st[3][v] = slot(k + 2)[v * PLANE + s0];
      }
      const int fk = k + 1;
      const double* fn = b.base + (long long)ffn(2, 0) * fsz + colofs + sz * (long long)fk;
      double gnx = 0, gny = 0, gnz = 0, gA = 0;
      int bk = BFACE_NONE;
      double sg = 1.0;
      if (col_on) {
        gnx = __ldg(fn);
        gny = __ldg(fn + fsz);
        gnz = __ldg(fn + 2 * fsz);
        gA = __ldg(fn + 3 * fsz);
        if (fk == nk) bk = b.bface[5][i + ni * j];
      }
      (void)sg;
      const int ez = face_flux<FLUX, LIM>(st[0], st[1], st[2], st[3], 1, pzp, pzm, nzp, nzm, 1,
                                          gnx, gny, gnz, gA, bk, 1.0, c, Fz);
      if (ez && col_on) {
        const unsigned long long lin =
            ((unsigned long long)i * nj + j) * (unsigned long long)(nk + 1) + fk;
        record_error(a.err, make_err_key(stage, 0, b.order, 2, ez, lin));
      }
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        pzp[v] = nzp[v];
        pzm[v] = nzm[v];
        wm1[v] = w0[v];
      }
    }
    if constexpr (NDIM == 2) cp_async_wait_all();
    __syncthreads();   // B2: face fluxes of plane k complete

    // ---- P3: residual, update of cell (i, j, k) ---------------------------------------
    if (col_on) {
      double R[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        const double dx = sFX[v * NFX + qx + 1] - sFX[v * NFX + qx];
        const double dy = sFY[v * NFY + qy + TI] - sFY[v * NFY + qy];
        if constexpr (NDIM == 3) R[v] = ((0.0 + dx) + dy) + (Fz[v] - fz[v]);
        else R[v] = (0.0 + dx) + dy;
      }
      const long long co = colofs + kofs;
      if (flags & F_SOURCE) {
#pragma unroll
        for (int v = 0; v < 5; ++v) R[v] = R[v] - b.base[(long long)(FSRC + v) * fsz + co];
      }
      if (stage0) {
#pragma unroll
        for (int v = 0; v < 5; ++v) rsum[v] += R[v] * R[v];
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
      const double rq = BF_RCP(qn[0]);
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
#pragma unroll
    for (int v = 0; v < 5; ++v) fz[v] = Fz[v];
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
