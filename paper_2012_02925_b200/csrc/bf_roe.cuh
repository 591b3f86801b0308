// bf_roe.cuh — FAST-build Roe stage kernel in the face-owner form
// (included by bf_kernels.cu after bf_vl.cuh, inside namespace bf::bf_fast).
//
// Roe's flux-difference splitting (physics.py:190-255) needs BOTH MUSCL states
// of a face at once, so the cell-split trick of bf_vl.cuh does not apply.
// Instead every cell OWNS its high face in each direction and computes its
// flux; the low face's flux is the neighbour's high face:
//   x: the cell reconstructs both of its x states; the right state of face
//      i+1/2 (cell i+1's low-side state) comes from lane+1 by shuffle, and the
//      finished flux goes back to lane+1 by shuffle;
//   y: the cell reconstructs its own high-side state and cell j+1's low-side
//      state directly from the staged plane (ghost depth 2 covers j+2), so no
//      exchange precedes the flux; the flux is handed to row j+1 through
//      shared memory across the existing AB barrier;
//   z: the high-side state of cell k is carried in registers while the CTA
//      marches in k; cell k+1's low-side state is reconstructed when plane k+2
//      lands, so face k+1/2's flux is computed in iteration k and carried as
//      the low-face flux of iteration k+1.
// Faces on the tile's low x / low y edges and its high x edge are extra items
// on the last two warps (64 per plane for 32 x 16 tiles).  Same two barriers
// per plane, TMA ring, geometry staging and epilogue as bf_vl.cuh.
//
// FAST arithmetic for the flux: one rsqrt(rho_L rho_R) gives 1/rho_L,
// 1/rho_R and sqrt(rho_R / rho_L); one rsqrt(a^2) gives a and 1/a^2; one
// reciprocal each for 1/(1 + sqrt(rho_R/rho_L)) and the Harten threshold
// (four MUFU seeds, each refined to ~1 ulp); FMA contraction.  Held to the
// 1e-12 bar against the oracle (tests/test_gpu_roe_split.py).
#pragma once

// Roe flux times the face area (physics.py:190-255 + solver.py:519).  Returns
// false when the Roe-averaged a^2 <= 0 (physics.py:213-217).
BF_DEV bool roe_face(const double L[5], const double Rr[5], double nx, double ny, double nz,
                     double A, const Consts& c, double F[5]) {
  const double rl = L[0], ul = L[1], vl = L[2], wl = L[3], pl = L[4];
  const double rr = Rr[0], ur = Rr[1], vr = Rr[2], wr = Rr[3], pr = Rr[4];
  const double y = frsqrt(rl * rr);
  const double yy = y * y;
  const double rli = rr * yy, rri = rl * yy;          // 1/rho_L, 1/rho_R
  const double rt = rr * y;                           // sqrt(rho_R / rho_L)
  const double wf = frcp(1.0 + rt);
  const double kel = 0.5 * fma(ul, ul, fma(vl, vl, wl * wl));
  const double ker = 0.5 * fma(ur, ur, fma(vr, vr, wr * wr));
  const double hl = fma(c.gog1 * pl, rli, kel);
  const double hr = fma(c.gog1 * pr, rri, ker);
  const double rho = rt * rl;
  const double u = fma(rt, ur, ul) * wf;
  const double v = fma(rt, vr, vl) * wf;
  const double w = fma(rt, wr, wl) * wf;
  const double h = fma(rt, hr, hl) * wf;
  const double ke = 0.5 * fma(u, u, fma(v, v, w * w));
  const double a2 = c.gm1 * (h - ke);
  const bool ok = !(a2 <= 0.0);
  const double ra = frsqrt(a2);
  const double a = a2 * ra;
  const double ia2h = 0.5 * (ra * ra);                // 1 / (2 a^2)
  const double vn = fma(u, nx, fma(v, ny, w * nz));
  const double vnl = fma(ul, nx, fma(vl, ny, wl * nz));
  const double vnr = fma(ur, nx, fma(vr, ny, wr * nz));
  const double dr = rr - rl, dp = pr - pl;
  const double du = ur - ul, dv = vr - vl, dw = wr - wl;
  const double dvn = vnr - vnl;
  // Harten's fix (physics.py:183-187): |lam| < delta -> (lam^2 + delta^2) / (2 delta)
  const double delta = c.efix * (fabs(vn) + a);
  const double hinv = 0.5 * frcp(delta);
  const double dd = delta * delta;
  auto habs = [&](double lam) {
    const double m = fabs(lam);
    return m < delta ? fma(lam, lam, dd) * hinv : m;
  };
  const double l1 = habs(vn - a), l2 = habs(vn), l5 = habs(vn + a);
  const double rad = rho * a * dvn;
  const double a1 = l1 * ((dp - rad) * ia2h);          // lam1 alpha1
  const double a5 = l5 * ((dp + rad) * ia2h);          // lam5 alpha5
  const double a2c = fma(-dp, 2.0 * ia2h, dr);         // alpha2
  const double l2r = l2 * rho;
  const double su = fma(-dvn, nx, du), sv = fma(-dvn, ny, dv), sw = fma(-dvn, nz, dw);
  const double s15 = a1 + a5, d15 = a5 - a1;           // combinations of the acoustic waves
  const double l2a = l2 * a2c;
  const double d0 = s15 + l2a;
  const double d1 = fma(s15, u, fma(d15 * a, nx, fma(l2a, u, l2r * su)));
  const double d2 = fma(s15, v, fma(d15 * a, ny, fma(l2a, v, l2r * sv)));
  const double d3 = fma(s15, w, fma(d15 * a, nz, fma(l2a, w, l2r * sw)));
  const double d4 = fma(s15, h, fma(d15 * a, vn, fma(l2a, ke, l2r * fma(u, su, fma(v, sv, w * sw)))));
  // 0.5 (F_L + F_R - D) A
  const double ml = rl * vnl, mr = rr * vnr;
  const double hA = 0.5 * A;
  F[0] = hA * (ml + mr - d0);
  F[1] = hA * (fma(ml, ul, fma(mr, ur, nx * (pl + pr))) - d1);
  F[2] = hA * (fma(ml, vl, fma(mr, vr, ny * (pl + pr))) - d2);
  F[3] = hA * (fma(ml, wl, fma(mr, wr, nz * (pl + pr))) - d3);
  F[4] = hA * (fma(ml, hl, mr * hr) - d4);
  return ok;
}

// One MUSCL state of a cell from its stencil (wm, w0, wp): the left state of
// its high face (HI) or the right state of its low face (!HI).
template <int LIM, bool K1, bool HI>
BF_DEV double recon_side(double wm, double w0, double wp, const Consts& c) {
  const double dm = w0 - wm, dp = wp - w0;
  if constexpr (K1 && LIM == LIM_VAN_ALBADA) {
    const double t = dpos(fma(dp, dm, c.lim_eps_half)) * frcp1(fma(dp, dp, fma(dm, dm, c.lim_eps)));
    return HI ? fma(t, dm, w0) : fma(-t, dp, w0);
  } else {
    double qL, qR;
    vl_recon<LIM, K1>(wm, w0, wp, c, qL, qR);
    return HI ? qL : qR;
  }
}

#ifndef BF_ROE_SMEM_BLOCK
#define BF_ROE_SMEM_BLOCK 0
#endif

template <int NDIM, int LIM>
struct RCfg {
  static constexpr int TJ = Cfg<NDIM, LIM>::TJ;   // same tiles as the other stage kernels
  static constexpr int NT = TI * TJ;
  static constexpr int PW = TI + 2 * HALO;
  static constexpr int PH = TJ + 2 * HALO;
  static constexpr int PLANE = PW * PH;
  static constexpr int NS = (NDIM == 3) ? NSLOT : 1;
  static constexpr int NFX = GXW * TJ;             // x geometry [4][TJ][GXW]
  static constexpr int NFY = TI * (TJ + 1);        // y geometry [4][TJ+1][TI]
  static constexpr int NYF = TI * (TJ + 1);        // y face fluxes [5][TJ+1][TI], row r = face j0+r
  static constexpr int NH = 2 * TJ + TI;           // tile-edge face items per plane
  static constexpr int r16(int x) { return (x + 15) / 16 * 16; }
  static constexpr int OW = 0;
  static constexpr int OYF = r16(OW + NS * 5 * PLANE);
  static constexpr int OXF = r16(OYF + 5 * NYF);         // [2][5][TJ]: faces i0, i0+TI
  static constexpr int OFX = r16(OXF + 10 * TJ);
  static constexpr int OFY = r16(OFX + 4 * NFX);
  static constexpr int OZG = r16(OFY + 4 * NFY);         // [2][4][TJ][TI] z faces (3D)
  static constexpr int OQ = r16(OZG + (NDIM == 3 ? 8 * NT : 0));   // [6][TJ][TI] Q0, dt/V
  // cell k's high-side z state (the left state of face k+1/2), thread-private:
  // carried along k in shared memory instead of 5 registers
  static constexpr int OZQ = r16(OQ + 6 * NT);
  static constexpr int ORS = r16(OZQ + (NDIM == 3 ? 5 * NT : 0));   // [NT/32][5] sum(R^2)
  static constexpr int OBAR = r16(ORS + 5 * (NT / 32));
  static constexpr int OBLK = OBAR + 8;                  // the tile's DevBlock
  static constexpr int TOTAL = OBLK + (int)(sizeof(DevBlock) + 7) / 8;
  static constexpr size_t BYTES = sizeof(double) * TOTAL;
  static constexpr int MINB = (NDIM == 2) ? BF_VL2D_MINB : 1;
  static constexpr unsigned WBYTES = 5u * PLANE * 8u;
  static constexpr unsigned GYZBYTES = (4u * NFY + (NDIM == 3 ? 4u * NT : 0u)) * 8u;
  static constexpr unsigned GXBYTES = 4u * NFX * 8u;
  BF_DEV static int pidx(int ii, int jj) { return (jj + HALO) * PW + (ii + HALO); }
};

template <int NDIM, int LIM, bool K1, bool S0>
__global__ void __launch_bounds__(RCfg<NDIM, LIM>::NT, RCfg<NDIM, LIM>::MINB)
    roe_stage_kernel(const __grid_constant__ StageArgs a) {
  pdl_trigger();                   // the next kernel may be dispatched (it waits for us)
  pdl_wait();                      // the previous kernel's writes are complete and visible
  if (a.stop && *a.stop) return;   // batched iterate stopped (RunState)
  using K = RCfg<NDIM, LIM>;
  constexpr int NT = K::NT, TJ = K::TJ, PLANE = K::PLANE, PW = K::PW;
  constexpr int NFX = K::NFX, NFY = K::NFY, NYF = K::NYF;
  extern __shared__ __align__(128) double smem[];
  double* const sW = smem + K::OW;
  double* const sYF = smem + K::OYF;
  double* const sXF = smem + K::OXF;
  double* const sFX = smem + K::OFX;
  double* const sFY = smem + K::OFY;
  double* const sZG = smem + K::OZG;
  double* const sQ = smem + K::OQ;
  double* const sZQ = smem + K::OZQ + threadIdx.x;   // [5] at stride NT
  double* const sRS = smem + K::ORS;
  unsigned long long* const bars = reinterpret_cast<unsigned long long*>(smem + K::OBAR);
  // bars[0..2]: plane ring, bars[3]: y/z geometry group, bars[4]: x geometry + Q0 / dt group

  const int tile_id = a.tile_list ? a.tile_list[blockIdx.x] : (int)blockIdx.x;
  const Tile t = a.tiles[tile_id];
#if BF_ROE_SMEM_BLOCK
  // the block record in shared memory (as in vl_stage_kernel): measured 1%
  // slower here (C4 Roe stage 1.527 vs 1.512 ms), off by default
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
  constexpr bool stage0 = S0;
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
  auto zslot = [&](int face) -> double* { return sZG + ((face - k0) & 1) * 4 * NT; };

  auto issue_plane = [&](int k) {
    unsigned long long* bar = bar_of(k);
    mbar_expect_tx(bar, K::WBYTES);
    tma_load4(slot_of(k), tm + 0 * 128, b.ox + i0 - HALO, b.oy + j0 - HALO,
              (NDIM == 3) ? b.oz + k : 0, fw(a.cur, 0), bar);
  };
  auto issue_geo_yz = [&](int k) {   // y face geometry of plane k, z face k+2
    unsigned long long* bar = bars + 3;
    const int z = (NDIM == 3) ? b.oz + k : 0;
    mbar_expect_tx(bar, K::GYZBYTES);
    tma_load4(sFY, tm + 2 * 128, b.ox + i0, b.oy + j0, z, ffn(1, 0), bar);
    if constexpr (NDIM == 3) tma_load4(zslot(k + 2), tm + 5 * 128, b.ox + i0, b.oy + j0, z + 2,
                                       ffn(2, 0), bar);
  };
  auto issue_b = [&](int k) {        // x face geometry, Q0 (and dt/V) of plane k
    unsigned long long* bar = bars + 4;
    const int z = (NDIM == 3) ? b.oz + k : 0;
    mbar_expect_tx(bar, K::GXBYTES + (stage0 ? 5u : 6u) * NT * 8u);
    tma_load4(sFX, tm + 1 * 128, b.ox + i0, b.oy + j0, z, ffn(0, 0), bar);
    tma_load4(sQ, tm + 3 * 128, b.ox + i0, b.oy + j0, z, FQ, bar);
    if (!stage0) tma_load4(sQ + 5 * NT, tm + 4 * 128, b.ox + i0, b.oy + j0, z, FDTV, bar);
  };
  auto prefetch_l2 = [&](int k) {
    const int z = (NDIM == 3) ? b.oz + k : 0;
    tma_prefetch4(tm + 1 * 128, b.ox + i0, b.oy + j0, z, ffn(0, 0));
    tma_prefetch4(tm + 2 * 128, b.ox + i0, b.oy + j0, z, ffn(1, 0));
    if constexpr (NDIM == 3) tma_prefetch4(tm + 5 * 128, b.ox + i0, b.oy + j0, z + 2, ffn(2, 0));
    tma_prefetch4(tm + 3 * 128, b.ox + i0, b.oy + j0, z, FQ);
  };

  auto face_err = [&](int d, int kind, unsigned long long lin) {
    record_error(a.err, make_err_key(stage, 0, b.order, d, kind, lin));
  };
  // face checks of one face (solver.py:501-506) and its Roe a^2 (physics.py:213-217)
  auto check_face = [&](int d, const double* qL, const double* qR, bool ok,
                        unsigned long long lin) {
    if (maybe_nonpos(qL[0], qL[4], qR[0], qR[4])) {
      if ((qL[0] <= 0.0) | (qL[4] <= 0.0)) face_err(d, ERR_FACE_LEFT, lin);
      if ((qR[0] <= 0.0) | (qR[4] <= 0.0)) face_err(d, ERR_FACE_RIGHT, lin);
    }
    if (!ok) face_err(d, ERR_ROE_A2, lin);
  };
  auto lin_x = [&](int f, int jj, int k) {
    return ((unsigned long long)f * nj + jj) * (unsigned long long)nk + (NDIM == 3 ? k : 0);
  };
  auto lin_y = [&](int ii, int f, int k) {
    return ((unsigned long long)ii * (nj + 1) + f) * (unsigned long long)nk + (NDIM == 3 ? k : 0);
  };
  auto lin_z = [&](int ii, int jj, int f) {
    return ((unsigned long long)ii * nj + jj) * (unsigned long long)(nk + 1) + f;
  };
  // wall / farfield flux (times A) of a boundary face (solver.py:526-580); the
  // ghost fill stored farfield_state(in1, outward n) in the ghost layers, so a
  // farfield overwrite is the Euler flux of the ghost cell (as bf_vl.cuh).
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
  double fzl[5] = {0, 0, 0, 0, 0};   // z flux of face k-1/2 (times A), the low face of cell k
  double lamz = 0.0;                 // z part of the stage-0 lambda of cell k

  if (tid == 0) {
    for (int q = 0; q < 5; ++q) mbar_init(bars + q, 1);
    fence_mbar_init();
  }
  if (stage0 && tid < 5 * (NT / 32)) sRS[tid] = 0.0;
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

  if constexpr (NDIM == 3) {
    // ---- prologue: face k0's flux and cell k0's high-side state ---------------------
    double wa[5], wb[5];
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
#pragma unroll
    for (int q = 0; q < 4; ++q) zslot(k0 + 1)[q * NT + tid] = g1[q];
    mbar_wait(bar_of(k0), par_of(k0));
    mbar_wait(bar_of(k0 + 1), par_of(k0 + 1));
    if (cell_on) {
      double wc[5], wd[5], qLm[5], qR0[5], zqL[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        wc[v] = slot_of(k0)[v * PLANE + s0];
        wd[v] = slot_of(k0 + 1)[v * PLANE + s0];
        qLm[v] = recon_side<LIM, K1, true>(wa[v], wb[v], wc[v], c);   // cell k0-1, high side
        vl_recon<LIM, K1>(wb[v], wc[v], wd[v], c, zqL[v], qR0[v]);    // cell k0, both sides
        sZQ[v * NT] = zqL[v];
      }
      const bool ok = roe_face(qLm, qR0, g0[0], g0[1], g0[2], g0[3], c, fzl);
      check_face(2, qLm, qR0, ok, lin_z(i, j, k0));
      if (maybe_nonpos(zqL[0], zqL[4], zqL[0], zqL[4]) && ((zqL[0] <= 0.0) | (zqL[4] <= 0.0)))
        face_err(2, ERR_FACE_LEFT, lin_z(i, j, k0 + 1));
      if (k0 == 0) {
        const int bk = b.bface[4][i + ni * j];
        if (bk != BFACE_NONE) overwrite(bk, wc, wd, wb, 1, g0, 1, fzl);
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

    unsigned bfk = 0;   // boundary-face kinds of this cell's x / y faces (2 bits each)
    {
      const int kz = (NDIM == 3) ? k : 0;
      if (in_j && i == ni - 1) bfk = (unsigned)b.bface[1][j + nj * kz] << 2;
      if (in_i && j == nj - 1) bfk |= (unsigned)b.bface[3][i + ni * kz] << 6;
    }
    __syncthreads();   // B0: plane k-1 retired (ring slot, x geometry, y fluxes, Q0)
    if (tid == 0) {
      fence_async_smem();
      issue_b(k);
      if constexpr (NDIM == 3) {
        if (kk > 0) issue_plane(k + 2);
        if (kk + 1 < kc)
          tma_prefetch4(tm, b.ox + i0 - HALO, b.oy + j0 - HALO, b.oz + k + 3, fw(a.cur, 0));
      }
    }
    mbar_wait(bars + 3, (unsigned)(kk & 1));
    mbar_wait(bar_of(k), par_of(k));

    // ---- phase A1: tile-edge faces (x: i0 and i0+TI per row; y: j0 per column) -------
    if (tid >= NT - K::NH) {
      const int h = tid - (NT - K::NH);
      int cx, cy, st, d, f;
      double g[4];
      double* out;
      int os;
      bool valid;
      unsigned long long lin;
      int bk = BFACE_NONE;
      if (h < 2 * TJ) {   // x face f = i0 (+TI): left cell cx, right cell cx+1
        const int row = h % TJ, hi = h / TJ;
        cx = hi ? TI - 1 : -1;
        cy = row;
        st = 1;
        d = 0;
        f = i0 + (hi ? TI : 0);
        out = sXF + hi * 5 * TJ + row;
        os = TJ;
        valid = (j0 + row < nj) && (f <= ni);
        lin = lin_x(f, j0 + row, k);
        const double* fn =
            b.base + (long long)ffn(0, 0) * fsz + f + sy * (long long)(j0 + row) + kofs;
#pragma unroll
        for (int q = 0; q < 4; ++q) g[q] = valid ? __ldg(fn + q * fsz) : 0.0;
        if (valid && (f == 0 || f == ni)) {
          const int kz = (NDIM == 3) ? k : 0;
          bk = b.bface[f == 0 ? 0 : 1][j0 + row + nj * kz];
        }
      } else {            // y face f = j0: left cell row -1, right cell row 0
        const int col = h - 2 * TJ;
        cx = col;
        cy = -1;
        st = PW;
        d = 1;
        f = j0;
        out = sYF + col;
        os = NYF;
        valid = (i0 + col < ni);
        lin = lin_y(i0 + col, f, k);
        const double* gy = sFY + col;
#pragma unroll
        for (int q = 0; q < 4; ++q) g[q] = gy[q * NFY];
        if (valid && f == 0) {
          const int kz = (NDIM == 3) ? k : 0;
          bk = b.bface[2][i0 + col + ni * kz];
        }
      }
      const double* wl = pk + K::pidx(cx, cy);   // left cell; right cell at wl + st
      double qL[5], qR[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        const double* wv = wl + v * PLANE;
        qL[v] = recon_side<LIM, K1, true>(wv[-st], wv[0], wv[st], c);
        qR[v] = recon_side<LIM, K1, false>(wv[0], wv[st], wv[2 * st], c);
      }
      double F[5];
      const bool ok = roe_face(qL, qR, g[0], g[1], g[2], g[3], c, F);
      if (valid) check_face(d, qL, qR, ok, lin);
      if (bk != BFACE_NONE) {   // boundary face: the reference overwrites the flux
        if (f == 0) overwrite(bk, wl + st, wl + 2 * st, wl, PLANE, g, 1, F);
        else overwrite(bk, wl, wl - st, wl + st, PLANE, g, 1, F);
      }
#pragma unroll
      for (int v = 0; v < 5; ++v) out[v * os] = F[v];
    }

    // ---- phase A2: y flux of face j+1/2 (this cell's high face) -> shared memory ------
    double R[5];
    double lam = 0.0;
    double snd = 0.0;
    {
      double qL[5], qR[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        const double* wv = w + v * PLANE;
        qL[v] = recon_side<LIM, K1, true>(wv[-PW], wv[0], wv[PW], c);
        qR[v] = recon_side<LIM, K1, false>(wv[0], wv[PW], wv[2 * PW], c);
      }
      const double* gh = sFY + (ty + 1) * TI + tx;   // face j+1
      double F[5];
      const bool ok = roe_face(qL, qR, gh[0], gh[NFY], gh[2 * NFY], gh[3 * NFY], c, F);
      if (cell_on) check_face(1, qL, qR, ok, lin_y(i, j + 1, k));
      if (cell_on && j == nj - 1) {
        const int bk = (bfk >> 6) & 3u;
        if (bk != BFACE_NONE) overwrite(bk, w, w - PW, w + PW, PLANE, gh, NFY, F);
      }
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        sYF[v * NYF + (ty + 1) * TI + tx] = F[v];
        R[v] = F[v];
      }
      if (stage0 && cell_on) {
        const double* gl = sFY + ty * TI + tx;
        snd = sound_speed(w[0], w[4 * PLANE], c);
        lam = lam_term(w[PLANE], w[2 * PLANE], w[3 * PLANE], snd, gl[0], gl[NFY], gl[2 * NFY],
                       gl[3 * NFY]) +
              lam_term(w[PLANE], w[2 * PLANE], w[3 * PLANE], snd, gh[0], gh[NFY], gh[2 * NFY],
                       gh[3 * NFY]);
        if constexpr (NDIM == 3) lam += lamz;
      }
    }

    // ---- phase A3 (3D): z flux of face k+1/2 -------------------------------------------
    if constexpr (NDIM == 3) {
      mbar_wait(bar_of(k + 2), par_of(k + 2));
      if (cell_on) {
        const double* p1 = slot_of(k + 1) + s0;
        const double* p2 = slot_of(k + 2) + s0;
        double w0[5], wc[5], qR1[5], qL1[5], zqL[5];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          w0[v] = w[v * PLANE];
          wc[v] = p1[v * PLANE];
          vl_recon<LIM, K1>(w0[v], wc[v], p2[v * PLANE], c, qL1[v], qR1[v]);   // cell k+1
          zqL[v] = sZQ[v * NT];
          sZQ[v * NT] = qL1[v];
        }
        const double* glo = zslot(k + 1) + tid;   // face k+1/2
        double fhi[5];
        const bool ok = roe_face(zqL, qR1, glo[0], glo[NT], glo[2 * NT], glo[3 * NT], c, fhi);
        check_face(2, zqL, qR1, ok, lin_z(i, j, k + 1));
        if (k + 1 <= nk - 1 && maybe_nonpos(qL1[0], qL1[4], qL1[0], qL1[4]) &&
            ((qL1[0] <= 0.0) | (qL1[4] <= 0.0)))
          face_err(2, ERR_FACE_LEFT, lin_z(i, j, k + 2));
        if (k == nk - 1) {
          const int bk = b.bface[5][i + ni * j];
          if (bk != BFACE_NONE) {
            double wm1[5] = {0, 0, 0, 0, 0};   // W(k-1): walls only (plane k-1 left the ring)
            if (bk == BFACE_WALL) wm1[4] = Win[4 * fsz + colofs + sz * (long long)(k - 1)];
            overwrite(bk, w0, wm1, wc, 1, glo, NT, fhi);
          }
        }
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          R[v] += fhi[v] - fzl[v];
          fzl[v] = fhi[v];
        }
        if (stage0) {
          const double* ghi = zslot(k + 2) + tid;
          const double snd1 = sound_speed(wc[0], wc[4], c);
          lamz = lam_term(wc[1], wc[2], wc[3], snd1, glo[0], glo[NT], glo[2 * NT], glo[3 * NT]) +
                 lam_term(wc[1], wc[2], wc[3], snd1, ghi[0], ghi[NT], ghi[2 * NT], ghi[3 * NT]);
        }
      }
    }

    __syncthreads();   // AB: y fluxes and tile-edge fluxes of plane k complete
    if (tid == 32) {
      fence_async_smem();
      if (kk + 1 < kc) issue_geo_yz(k + 1);
      if (kk + 2 < kc) prefetch_l2(k + 2);
    }

    // ---- phase B1: x flux of face i+1/2; the low face's by shuffle ---------------------
    mbar_wait(bars + 4, (unsigned)(kk & 1));
    {
      double qL[5], qR[5], qRn[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        vl_recon<LIM, K1>(w[v * PLANE - 1], w[v * PLANE], w[v * PLANE + 1], c, qL[v], qR[v]);
        qRn[v] = __shfl_down_sync(FULL, qR[v], 1);
      }
      const double* gl = sFX + ty * GXW + tx;   // face i (low); face i+1 at gl + 1
      double fhi[5];
      const bool ok = roe_face(qL, qRn, gl[1], gl[NFX + 1], gl[2 * NFX + 1], gl[3 * NFX + 1], c,
                               fhi);
      if (cell_on && tx < TI - 1) check_face(0, qL, qRn, ok, lin_x(i + 1, j, k));
      if (cell_on && i == ni - 1 && tx < TI - 1) {
        const int bk = (bfk >> 2) & 3u;
        if (bk != BFACE_NONE) overwrite(bk, w, w - 1, w + 1, PLANE, gl + 1, NFX, fhi);
      }
      double flo[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        flo[v] = __shfl_up_sync(FULL, fhi[v], 1);
        if (tx == 0) flo[v] = sXF[v * TJ + ty];
        if (tx == TI - 1) fhi[v] = sXF[5 * TJ + v * TJ + ty];
        R[v] += fhi[v] - flo[v];
      }
      if (stage0 && cell_on) {
        lam += lam_term(w[PLANE], w[2 * PLANE], w[3 * PLANE], snd, gl[0], gl[NFX], gl[2 * NFX],
                        gl[3 * NFX]) +
               lam_term(w[PLANE], w[2 * PLANE], w[3 * PLANE], snd, gl[1], gl[NFX + 1],
                        gl[2 * NFX + 1], gl[3 * NFX + 1]);
      }
    }

    // ---- phase B2: residual, update of cell (i, j, k) -----------------------------------
    if (cell_on) {
#pragma unroll
      for (int v = 0; v < 5; ++v) R[v] -= sYF[v * NYF + ty * TI + tx];
      const long long co = colofs + kofs;
      if (flags & F_SOURCE) {
#pragma unroll
        for (int v = 0; v < 5; ++v) R[v] = R[v] - b.base[(long long)(FSRC + v) * fsz + co];
      }
      double dtv;
      if (stage0) {
        dtv = c.cfl * frcp(lam);
        b.base[(long long)FDTV * fsz + co] = dtv;
      } else {
        dtv = sQ[5 * NT + tid];
      }
      const double adt = a.alpha * dtv;
      double qn[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) qn[v] = fma(-adt, R[v], sQ[v * NT + tid]);
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
    }
    if (stage0) {   // sum(R^2) of the plane: warp tree, accumulated per warp (fixed order)
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        double x = cell_on ? R[v] * R[v] : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(FULL, x, off);
        if ((tid & 31) == 0) sRS[(tid >> 5) * 5 + v] += x;
      }
    }
  }

  // ---- deterministic per-tile sum(R^2) ----------------------------------------
  if (stage0) {
    __syncthreads();
    if (tid < 5) {
      double x = 0.0;
      for (int q = 0; q < NT / 32; ++q) x += sRS[q * 5 + tid];
      a.partial[(long long)tile_id * 5 + tid] = x;
    }
  }
}

template <int NDIM, int LIM, bool K1, bool S0>
static cudaError_t launch_roe_s(const StageArgs& a, cudaStream_t s) {
  using K = RCfg<NDIM, LIM>;
  auto k = roe_stage_kernel<NDIM, LIM, K1, S0>;
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
  return launch_pdl(k, (unsigned)a.ntiles, (unsigned)K::NT, K::BYTES, s, a);
}

template <int NDIM, int LIM, bool K1>
static cudaError_t launch_roe_t(const StageArgs& a, cudaStream_t s) {
  return (a.flags & F_STAGE0) ? launch_roe_s<NDIM, LIM, K1, true>(a, s)
                              : launch_roe_s<NDIM, LIM, K1, false>(a, s);
}

template <int NDIM, bool K1>
static cudaError_t launch_roe_l(int lim, const StageArgs& a, cudaStream_t s) {
  switch (lim) {
    case LIM_NONE: return launch_roe_t<NDIM, LIM_NONE, K1>(a, s);
    case LIM_VAN_LEER: return launch_roe_t<NDIM, LIM_VAN_LEER, K1>(a, s);
    case LIM_VAN_ALBADA: return launch_roe_t<NDIM, LIM_VAN_ALBADA, K1>(a, s);
    default: return launch_roe_t<NDIM, LIM_MINMOD, K1>(a, s);
  }
}

static cudaError_t launch_roe(int ndim, int lim, const StageArgs& a, cudaStream_t s) {
  const bool k1 = a.c.muscl_k1 != 0;
  if (ndim == 3) return k1 ? launch_roe_l<3, true>(lim, a, s) : launch_roe_l<3, false>(lim, a, s);
  return k1 ? launch_roe_l<2, true>(lim, a, s) : launch_roe_l<2, false>(lim, a, s);
}
