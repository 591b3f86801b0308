// bf_stage.cuh — the fused per-stage kernel (included by bf_kernels.cu inside
// namespace bf::BF_NS).
//
// One CTA owns a TI x TJ column tile of one block and marches KC cells in k.
// All global->shared traffic is TMA: each block has a 4-D tensor map over its
// field arena (padded i, j, k, field slot), so ONE cp.async.bulk.tensor moves
// the 5 primitive variables of a haloed (TI+4) x (TJ+4) plane, ONE moves the 4
// geometry components of a face tile, ONE the 5 conserved variables; tiles at
// block edges are zero-filled by the TMA unit.  One elected thread issues,
// mbarriers carry completion.
// Per k-plane, three barrier-separated phases:
//   P1  every (cell, variable) limiter value of the plane's x and y stencils
//       (a flat loop: each thread gets the same number +-1 of scalar items);
//   P2  face fluxes: own x-low face, own y-low face (+ one tile-edge face for
//       TI+TJ threads), then the own-column z limiter and z face k+1; a face's
//       geometry sits in the shared-memory slot its flux is written to;
//   P3  residual, stage-0 local dt / sum(R^2), RK update and decode.
#pragma once

// ---- TMA / mbarrier primitives ------------------------------------------------
BF_DEV unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
BF_DEV void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
BF_DEV void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
BF_DEV void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}
BF_DEV void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
BF_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// 4-D tile load: box at coordinates (x, y, z, s) of the tensor map -> smem
BF_DEV void tma_load4(void* dst, const void* tmap, int x, int y, int z, int s,
                      unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(tmap)), "r"(x), "r"(y), "r"(z), "r"(s),
      "r"(smem_u32(bar))
      : "memory");
}

template <int NDIM, int LIM>
struct Cfg {
  static constexpr int PC = psi_count<LIM>();
  static constexpr int TJ = (NDIM == 3 && PC < 2) ? TJ_3D : TJ_2D;
  static constexpr int NT = TI * TJ;
  static constexpr int MINB = (NT <= 256) ? 2 : 1;          // CTAs per SM targeted
  static constexpr int PW = TI + 2 * HALO;                  // plane row pitch (36)
  static constexpr int PH = TJ + 2 * HALO;
  static constexpr int PLANE = PW * PH;                     // cells per plane (full rectangle)
  static constexpr int NS = (NDIM == 3) ? NSLOT : 1;
  static constexpr int NPX = (TI + 2) * TJ;                 // psi_x cells: i = -1..TI
  static constexpr int NPY = TI * (TJ + 2);                 // psi_y cells: j = -1..TJ
  static constexpr int NLIM = NPX + NPY;
  static constexpr int NFX = GXW * TJ;                      // x-face slots [row][f], f = 0..33
  static constexpr int NFY = TI * (TJ + 1);                 // y-face slots [f][col]
  static constexpr bool ZG = (NDIM == 3) && (MINB == 1);    // z geometry staged in smem
  static constexpr int r128(int x) { return (x + 15) / 16 * 16; }   // 128-byte alignment
  static constexpr int OW = 0;                                      // [NS][5][PH][PW]
  static constexpr int OPX = r128(OW + NS * 5 * PLANE);             // [PC][5][NPX]
  static constexpr int OPY = r128(OPX + PC * 5 * NPX);              // [PC][5][NPY]
  static constexpr int OFX = r128(OPY + PC * 5 * NPY);              // [5][TJ][GXW]
  static constexpr int OFY = r128(OFX + 5 * NFX);                   // [5][TJ+1][TI]
  static constexpr int OQ = r128(OFY + 5 * NFY);                    // [6][TJ][TI]
  static constexpr int OZ = r128(OQ + 6 * NT);                      // [4][TJ][TI] (ZG)
  static constexpr int NEDGE = TI + TJ;                             // tile-edge faces per plane
  static constexpr int OH = r128(OZ + (ZG ? 4 * NT : 0));           // [NEDGE][2][5] half fluxes
  static constexpr int OBAR = r128(OH + NEDGE * 10);                // mbarriers
  static constexpr int TOTAL = OBAR + 8;
  static constexpr size_t BYTES = sizeof(double) * TOTAL;
  // TMA transaction sizes
  static constexpr unsigned WBYTES = 5u * PLANE * 8u;
  static constexpr unsigned GBYTES = (4u * NFX + 4u * NFY + 5u * NT + 1u * NT +
                                      (ZG ? 4u * NT : 0u)) * 8u;
  BF_DEV static int pidx(int ii, int jj) { return (jj + HALO) * PW + (ii + HALO); }
};

template <int NDIM, int FLUX, int LIM>
__global__ void __launch_bounds__(Cfg<NDIM, LIM>::NT, Cfg<NDIM, LIM>::MINB)
    stage_kernel(const StageArgs a) {
  pdl_trigger();                   // the next kernel may be dispatched (it waits for us)
  pdl_wait();                      // the previous kernel's writes are complete and visible
  if (a.stop && *a.stop) return;   // batched iterate stopped (RunState)
  using K = Cfg<NDIM, LIM>;
  constexpr int NT = K::NT, TJ = K::TJ, PLANE = K::PLANE, PW = K::PW, PC = K::PC;
  constexpr int NFX = K::NFX, NFY = K::NFY, NPX = K::NPX, NPY = K::NPY;
  extern __shared__ __align__(128) double smem[];
  double* const sW = smem + K::OW;
  double* const sPX = smem + K::OPX;
  double* const sPY = smem + K::OPY;
  double* const sFX = smem + K::OFX;
  double* const sFY = smem + K::OFY;
  double* const sQ = smem + K::OQ;
  double* const sZ = smem + K::OZ;
  double* const sH = smem + K::OH;
  unsigned long long* const bars = reinterpret_cast<unsigned long long*>(smem + K::OBAR);
  // Van Leer faces split exactly into F+(qL) + F-(qR): the TI+TJ tile-edge
  // faces become 2*(TI+TJ) half-face items done in the limiter phase by the
  // last warps, so the flux phase has exactly three faces per thread.
  // Measured neutral on C4 (barrier stalls 16.5% -> 8.7% but +8% instructions,
  // profiles/r01_stage_kernel_v9.ncu.json), so off unless BF_SPLIT_EDGE=1.
#ifndef BF_SPLIT_EDGE
#define BF_SPLIT_EDGE 0
#endif
  constexpr bool SPLIT = BF_SPLIT_EDGE && FLUX == FLUX_VAN_LEER;
  constexpr int NHALF = SPLIT ? 2 * K::NEDGE : 0;
  constexpr int NFLAT = NT - NHALF;            // threads on the flat limiter loop
  // bars[0..2]: plane ring slots, bars[3]: per-plane geometry/Q0 group

  const int tile_id = a.tile_list ? a.tile_list[blockIdx.x] : (int)blockIdx.x;
  const Tile t = a.tiles[tile_id];
  const DevBlock b = a.blocks[t.block];     // by value: no aliasing reloads
  const Consts& c = a.c;
  const unsigned char* const tm = a.tmaps + (size_t)t.block * NTMAP * 128;
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
  double* const Wout = b.base + (long long)fw(a.cur ^ 1, 0) * fsz;
  const long long colofs = i + sy * (long long)j;
  const int s0 = K::pidx(tx, ty);

  // plane p (p = k - (k0 - 1)) lives in slot p % NS; its barrier parity is (p / NS) & 1
  auto slot_of = [&](int k) -> double* {
    if constexpr (NDIM == 3) return sW + ((k - k0 + 1) % NSLOT) * 5 * PLANE;
    else return sW;
  };
  auto bar_of = [&](int k) { return bars + ((NDIM == 3) ? (k - k0 + 1) % NSLOT : 0); };
  auto par_of = [&](int k) { return (unsigned)(((NDIM == 3) ? (k - k0 + 1) / NSLOT : 0) & 1); };
  auto psi_ptr = [&](int d, int pm, int v) -> double* {
    return b.base + (long long)(b.psi0 + 10 * d + 5 * pm + v) * fsz;
  };

  // ---- producers (thread 0) -------------------------------------------------------
  auto issue_plane = [&](int k) {
    unsigned long long* bar = bar_of(k);
    mbar_expect_tx(bar, K::WBYTES);
    tma_load4(slot_of(k), tm + 0 * 128, b.ox + i0 - HALO, b.oy + j0 - HALO,
              (NDIM == 3) ? b.oz + k : 0, fw(a.cur, 0), bar);
  };
  auto issue_group = [&](int k) {   // geometry of plane k's faces, Q0, dt/V (or V), z geometry
    unsigned long long* bar = bars + 3;
    const int z = (NDIM == 3) ? b.oz + k : 0;
    mbar_expect_tx(bar, K::GBYTES);
    tma_load4(sFX, tm + 1 * 128, b.ox + i0, b.oy + j0, z, ffn(0, 0), bar);
    tma_load4(sFY, tm + 2 * 128, b.ox + i0, b.oy + j0, z, ffn(1, 0), bar);
    tma_load4(sQ, tm + 3 * 128, b.ox + i0, b.oy + j0, z, FQ, bar);
    tma_load4(sQ + 5 * NT, tm + 4 * 128, b.ox + i0, b.oy + j0, z, stage0 ? FVOL : FDTV, bar);
    if constexpr (K::ZG) tma_load4(sZ, tm + 5 * 128, b.ox + i0, b.oy + j0, z + 1, ffn(2, 0), bar);
  };

  const int qx = ty * GXW + tx;                            // own x-low face slot
  const int qy = ty * TI + tx;                             // own y-low face slot
  const int ex = tid < TJ ? tid : -1;                      // extra x face f=TI, row tid
  const int ey = (tid >= TJ && tid < TJ + TI) ? tid - TJ : -1;   // extra y face row TJ
  auto face_on_x = [&](int f, int row) { return i0 + f <= ni && j0 + row < nj; };
  auto face_on_y = [&](int f, int col) { return j0 + f <= nj && i0 + col < ni; };

  double rsum[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  double wm1[5] = {0, 0, 0, 0, 0};  // W(k-1), own column
  double pzp[5], pzm[5];            // psi+/psi- of cell k
  double fz[5];                     // flux at face k
#pragma unroll
  for (int v = 0; v < 5; ++v) pzp[v] = pzm[v] = fz[v] = 0.0;

  if (tid == 0) {
    for (int q = 0; q < 4; ++q) mbar_init(bars + q, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if constexpr (NDIM == 3) {
    if (col_on) {
      const double* Win = b.base + (long long)fw(a.cur, 0) * fsz;
      const long long o = colofs + sz * (long long)(k0 - 2);
#pragma unroll
      for (int v = 0; v < 5; ++v) wm1[v] = Win[v * fsz + o];
    }
    if (tid == 0) {
      issue_plane(k0 - 1);
      issue_plane(k0);
      issue_plane(k0 + 1);
    }
    mbar_wait(bar_of(k0 - 1), par_of(k0 - 1));
    mbar_wait(bar_of(k0), par_of(k0));
    mbar_wait(bar_of(k0 + 1), par_of(k0 + 1));
  } else {
    if (tid == 0) {
      issue_plane(0);
      issue_group(0);
    }
    mbar_wait(bar_of(0), 0);
  }

  // z limiter of cell kc from the own-column values of kc-1, kc, kc+1
  auto z_limiter = [&](int kc, const double* wa, const double* wb, const double* wc, double pp[5],
                       double pm[5]) {
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
      cell_limiter<LIM>(wa[v], wb[v], wc[v], pp[v], pm[v]);
      if (psi_store && col_on && kc >= -1 && kc <= nk) {
        psi_ptr(2, 0, v)[cz] = pp[v];
        psi_ptr(2, 1, v)[cz] = pm[v];
      }
    }
  };
  // z face fk from own-column W(fk-2..fk+1) and psi of cells fk-1, fk
  auto z_face = [&](int fk, const double st[4][5], const double* ppl, const double* pml,
                    const double* ppr, const double* pmr, double g[4], double F[5]) {
    int bk = BFACE_NONE;
    double sg = 1.0;
    if (col_on && fk == 0) {
      bk = b.bface[4][i + ni * j];
      sg = -1.0;
    } else if (col_on && fk == nk) {
      bk = b.bface[5][i + ni * j];
    }
    const int ez = face_flux<FLUX, LIM>(st[0], st[1], st[2], st[3], 1, ppl, pml, ppr, pmr, 1, g[0],
                                        g[1], g[2], g[3], bk, sg, c, F);
    if (c.viscous && col_on) {   // F - Fv (solver.py:522-524)
      const double* fv = b.base + (long long)(b.vis0 + 27 + 8) * fsz + colofs + sz * (long long)fk;
#pragma unroll
      for (int m = 0; m < 4; ++m) F[m + 1] = F[m + 1] - fv[m * fsz];
    }
    if (ez && col_on) {
      const unsigned long long lin =
          ((unsigned long long)i * nj + j) * (unsigned long long)(nk + 1) + fk;
      record_error(a.err, make_err_key(stage, 0, b.order, 2, ez, lin));
    }
  };
  auto load_zgeo_global = [&](int fk, double g[4]) {
    if (!col_on) {
      g[0] = g[1] = g[2] = g[3] = 0.0;
      return;
    }
    const double* fn = b.base + (long long)ffn(2, 0) * fsz + colofs + sz * (long long)fk;
    g[0] = __ldg(fn);
    g[1] = __ldg(fn + fsz);
    g[2] = __ldg(fn + 2 * fsz);
    g[3] = __ldg(fn + 3 * fsz);
  };

  const int kfirst = (NDIM == 3) ? -1 : 0;
  for (int kk = kfirst; kk < t.kc; ++kk) {
    const int k = k0 + kk;
    const bool xy = kk >= 0;
    const long long kofs = (NDIM == 3) ? sz * (long long)k : 0;
    const double* pk = slot_of(k);

    if constexpr (NDIM == 3) {
      if (!xy) {
        // prologue: psi_z(k0-1), psi_z(k0) and the z face k0; no x/y work
        double st[4][5], nzp[5], nzm[5], Fz[5], g[4];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          st[0][v] = wm1[v];
          st[1][v] = slot_of(k)[v * PLANE + s0];
          st[2][v] = slot_of(k + 1)[v * PLANE + s0];
          st[3][v] = slot_of(k + 2)[v * PLANE + s0];
        }
        z_limiter(k, st[0], st[1], st[2], pzp, pzm);
        z_limiter(k + 1, st[1], st[2], st[3], nzp, nzm);
        load_zgeo_global(k + 1, g);
        z_face(k + 1, st, pzp, pzm, nzp, nzm, g, Fz);
#pragma unroll
        for (int v = 0; v < 5; ++v) {
          pzp[v] = nzp[v];
          pzm[v] = nzm[v];
          fz[v] = Fz[v];
          wm1[v] = st[1][v];
        }
        continue;
      }
    }

    __syncthreads();   // B0: iteration k-1 fully retired (smem slots free)
    if (tid == 0) {
      fence_async_smem();
      if constexpr (NDIM == 3) {
        issue_group(k);
        issue_plane(k + 2);   // into the slot of plane k-1 (its own column is in wm1)
      }
    }

    // ---- P1a (Van Leer): half fluxes of the tile-edge faces ---------------------------
    if (SPLIT && tid >= NFLAT) {
      const int hidx = tid - NFLAT;
      const int e = hidx >> 1, h = hidx & 1;           // h = 0: F+(qL), h = 1: F-(qR)
      const bool isx = e < TJ;
      const int fcol = isx ? TI : e - TJ;              // the face's cell f (right of the face)
      const int frow = isx ? e : TJ;
      const int step = isx ? 1 : PW;
      const int d = isx ? 0 : 1;
      const int gi = i0 + fcol, gj = j0 + frow;
      const bool on = isx ? face_on_x(TI, e) : face_on_y(TJ, fcol);
      double g[3] = {0.0, 0.0, 0.0};
      if (on) {
        const double* fn = b.base + (long long)ffn(d, 0) * fsz + gi + sy * (long long)gj + kofs;
        g[0] = __ldg(fn);
        g[1] = __ldg(fn + fsz);
        g[2] = __ldg(fn + 2 * fsz);
      }
      const double* wf = pk + K::pidx(fcol, frow);     // var-0 pointer of cell f
      const double* wc = h == 0 ? wf - step : wf;      // cell whose limiter this side needs
      const int lc = h == 0 ? -1 : 0;                  // its offset from f along the face normal
      double q5[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        const double* w = wc + v * PLANE;
        double pp = 1.0, pm = 1.0;
        if constexpr (PC > 0) {
          if (psi_load) {
            const int ci = gi + (isx ? lc : 0), cj = gj + (isx ? 0 : lc);
            const long long go = ci + sy * (long long)cj + kofs;
            pp = on ? psi_ptr(d, 0, v)[go] : 0.0;
            pm = (PC == 2) ? (on ? psi_ptr(d, 1, v)[go] : 0.0) : pp;
          } else {
            cell_limiter<LIM>(w[-step], w[0], w[step], pp, pm);
          }
        }
        q5[v] = h == 0 ? muscl_left(w[-step], w[0], w[step], pp, pm, c)
                       : muscl_right(w[-step], w[0], w[step], pp, pm, c);
      }
      if (on && (q5[0] <= 0.0 || q5[4] <= 0.0)) {
        const unsigned long long lin =
            isx ? ((unsigned long long)gi * nj + gj) * (unsigned long long)(NDIM == 3 ? nk : 1) +
                      (NDIM == 3 ? k : 0)
                : ((unsigned long long)gi * (nj + 1) + gj) *
                          (unsigned long long)(NDIM == 3 ? nk : 1) +
                      (NDIM == 3 ? k : 0);
        record_error(a.err, make_err_key(stage, 0, b.order, d,
                                         h == 0 ? ERR_FACE_LEFT : ERR_FACE_RIGHT, lin));
      }
      double Fh[5];
      van_leer_half(St{q5[0], q5[1], q5[2], q5[3], q5[4]}, g[0], g[1], g[2], c,
                    h == 0 ? 1.0 : -1.0, Fh);
#pragma unroll
      for (int v = 0; v < 5; ++v) sH[(e * 2 + h) * 5 + v] = Fh[v];
    }

    // ---- P1: every (cell, var) limiter value of the x and y stencils of plane k --
    if (PC > 0 && tid < NFLAT) {
      // item q in [0, NLIM): [x cells i=0..TI-1 (TI*TJ)] [x edge cells i=-1,TI (2*TJ)]
      // [y cells j=-1..TJ (TI*(TJ+2))]; all index maps are shifts/masks
      static_assert(NT < K::NLIM, "one wrap per stride");
      int v = 0, q = tid;
      for (; v < 5;) {
        int cc, row, d, o;
        if (q < TI * TJ) {
          cc = q & (TI - 1);
          row = q >> 5;
          d = 0;
          o = row * (TI + 2) + cc + 1;
        } else if (q < TI * TJ + 2 * TJ) {
          const int e = q - TI * TJ;
          row = e >> 1;
          cc = (e & 1) ? TI : -1;
          d = 0;
          o = row * (TI + 2) + cc + 1;
        } else {
          const int q2 = q - NPX;
          cc = q2 & (TI - 1);
          row = (q2 >> 5) - 1;
          d = 1;
          o = q2;
        }
        const int step = d == 0 ? 1 : PW;
        double* dst = (d == 0 ? sPX : sPY) + o;
        const int vstride = d == 0 ? NPX : NPY;
        if (psi_load | psi_store) {
          const int gi = i0 + cc, gj = j0 + row;
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
            const double* w = pk + v * PLANE + K::pidx(cc, row);
            cell_limiter<LIM>(w[-step], w[0], w[step], pp, pm);
            dst[v * vstride] = pp;
            if constexpr (PC == 2) dst[(5 + v) * vstride] = pm;
            if (in_range) {
              psi_ptr(d, 0, v)[go] = pp;
              psi_ptr(d, 1, v)[go] = pm;
            }
          }
        } else {
          double pp, pm;
          const double* w = pk + v * PLANE + K::pidx(cc, row);
          cell_limiter<LIM>(w[-step], w[0], w[step], pp, pm);
          dst[v * vstride] = pp;
          if constexpr (PC == 2) dst[(5 + v) * vstride] = pm;
        }
        q += NFLAT;
        if (q >= K::NLIM) {
          q -= K::NLIM;
          ++v;
        }
      }
    }
    if constexpr (NDIM == 3) mbar_wait(bars + 3, (unsigned)(kk & 1));
    else mbar_wait(bars + 3, 0);
    __syncthreads();     // B1: limiters complete; geometry / Q0 landed

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
          double g[4];
          load_zgeo_global(k, g);
          term(g[0], g[1], g[2], g[3]);
          if constexpr (K::ZG) {
            term(sZ[qy], sZ[NT + qy], sZ[2 * NT + qy], sZ[3 * NT + qy]);
          } else {
            load_zgeo_global(k + 1, g);
            term(g[0], g[1], g[2], g[3]);
          }
        }
        const double vol = sQ[5 * NT + tid];
        if (c.viscous) {   // viscous spectral radius (solver.py:717-730)
          const long long co = colofs + kofs;
          const double* Wc = b.base + (long long)fw(a.cur, 0) * fsz;
          const double T = a.t_derived ? p / (rho * c.R) : Wc[5 * fsz + co];
          double mu = c.mu;
          if (c.has_suth)
            mu = c.suth_mu * pow(T / c.suth_t, 1.5) * (c.suth_t + c.suth_s) / (T + c.suth_s);
          auto vterm = [&](double alo, double ahi) {
            const double abar = 0.5 * (alo + ahi);
            lam = lam + c.visc_coeff * (mu / rho) * abar * abar / vol;
          };
          vterm(sFX[3 * NFX + qx], sFX[3 * NFX + qx + 1]);
          vterm(sFY[3 * NFY + qy], sFY[3 * NFY + qy + TI]);
          if constexpr (NDIM == 3) {
            const double* fz0 = b.base + (long long)ffn(2, 3) * fsz + colofs + kofs;
            vterm(fz0[0], fz0[sz]);
          }
        }
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
      const int q = row * GXW + f;
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
      if (c.viscous && on) {
        const double* fv = b.base + (long long)(b.vis0 + 27) * fsz + gi + sy * (long long)gj + kofs;
#pragma unroll
        for (int m = 0; m < 4; ++m) F[m + 1] = F[m + 1] - fv[m * fsz];
      }
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
      if (c.viscous && on) {
        const double* fv = b.base + (long long)(b.vis0 + 27 + 4) * fsz + gi + sy * (long long)gj + kofs;
#pragma unroll
        for (int m = 0; m < 4; ++m) F[m + 1] = F[m + 1] - fv[m * fsz];
      }
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
    if constexpr (!SPLIT) {
      if (ex >= 0) x_face(TI, ex);
      if (ey >= 0) y_face(TJ, ey);
    } else if (tid >= NFLAT && ((tid - NFLAT) & 1) == 0) {
      // tile-edge face e = (F+ + F-) * A (+ wall / farfield overwrite)
      const int e = (tid - NFLAT) >> 1;
      const bool isx = e < TJ;
      const int fcol = isx ? TI : e - TJ, frow = isx ? e : TJ;
      const int q = isx ? e * GXW + TI : TJ * TI + fcol;
      double* G = isx ? sFX : sFY;
      const int nq = isx ? NFX : NFY;
      const bool on = isx ? face_on_x(TI, e) : face_on_y(TJ, fcol);
      const double nx = G[q], ny = G[nq + q], nz = G[2 * nq + q];
      const double A = on ? G[3 * nq + q] : 0.0;
      double F[5];
#pragma unroll
      for (int v = 0; v < 5; ++v) F[v] = (sH[(e * 2) * 5 + v] + sH[(e * 2 + 1) * 5 + v]) * A;
      int bk = BFACE_NONE;
      if (on && isx && i0 + TI == ni) bk = b.bface[1][(j0 + frow) + nj * (NDIM == 3 ? k : 0)];
      if (on && !isx && j0 + TJ == nj) bk = b.bface[3][(i0 + fcol) + ni * (NDIM == 3 ? k : 0)];
      if (bk != BFACE_NONE) {
        const int step = isx ? 1 : PW;
        const double* wf = pk + K::pidx(fcol, frow);
        boundary_overwrite(bk, 1.0, wf - 2 * step, wf - step, wf, wf + step, PLANE, nx, ny, nz,
                           A, c, F);
      }
#pragma unroll
      for (int v = 0; v < 5; ++v) G[v * nq + q] = F[v];
    }

    // own-column z limiter of cell k+1 and z face k+1 (plane k+2 must have landed)
    double Fz[5] = {0, 0, 0, 0, 0};
    if constexpr (NDIM == 3) {
      mbar_wait(bar_of(k + 2), par_of(k + 2));
      double st[4][5], nzp[5], nzm[5], g[4];
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        st[0][v] = wm1[v];
        st[1][v] = pk[v * PLANE + s0];
        st[2][v] = slot_of(k + 1)[v * PLANE + s0];
        st[3][v] = slot_of(k + 2)[v * PLANE + s0];
      }
      z_limiter(k + 1, st[1], st[2], st[3], nzp, nzm);
      if constexpr (K::ZG) {
        g[0] = sZ[qy];
        g[1] = sZ[NT + qy];
        g[2] = sZ[2 * NT + qy];
        g[3] = sZ[3 * NT + qy];
      } else {
        load_zgeo_global(k + 1, g);
      }
      z_face(k + 1, st, pzp, pzm, nzp, nzm, g, Fz);
#pragma unroll
      for (int v = 0; v < 5; ++v) {
        pzp[v] = nzp[v];
        pzm[v] = nzm[v];
        wm1[v] = st[1][v];
      }
    }
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
    __syncthreads();
    double* red = sQ;   // free after the last P3: [NT/32][5]
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
      a.partial[(long long)tile_id * 5 + tid] = x;
    }
  }
}
