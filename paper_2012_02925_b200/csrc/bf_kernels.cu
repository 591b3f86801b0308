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

#include <cstdlib>

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

// Programmatic dependent launch (griddepcontrol): the per-stage kernels are
// launched with programmatic stream serialization, so the next one's CTAs are
// dispatched while this one drains and wait in pdl_wait() — before anything
// that reads what the previous kernel wrote (or writes what it reads) — until
// it has completed and flushed.  pdl_trigger() lets the dependent launch be
// scheduled once every CTA of this grid has started.
BF_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
BF_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Whether this thread's launches use it (set_pdl, per context by the runtime:
// on for one-wave grids, where it takes ~2 us off a C1 step; off for large
// ones — C4 measured 1.6% slower with it).
static thread_local int t_pdl = 0;
void set_pdl(int on) { t_pdl = on; }

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                              cudaStream_t s, const Args&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = t_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
  return e != cudaSuccess ? e : cudaGetLastError();
}

BF_DEV void record_error(unsigned long long* err, unsigned long long key) {
  if (key < *reinterpret_cast<volatile unsigned long long*>(err)) atomicMin(err, key);
}

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
// MUSCL left state at face f from cells f-2, f-1, f (solver.py:468-469):
// qL = w_{f-1} + (eps/4)((1-k) psi+_{f-1} D_{f-1} + (1+k) psi-_{f-1} D_f)
BF_DEV double muscl_left(double w0, double w1, double w2, double pp, double pm, const Consts& c) {
  if (c.eps0) return w1;
  const double dm = w1 - w0;
  const double d0 = w2 - w1;
#if BF_EXACT
  return w1 + c.quarter * (c.omk * pp * dm + c.opk * pm * d0);
#else
  if (c.kappa_m1) return w1 + c.quarter * (c.omk * pp * dm);
  return w1 + c.quarter * (c.omk * pp * dm + c.opk * pm * d0);
#endif
}
// MUSCL right state at face f from cells f-1, f, f+1 (solver.py:470-471):
// qR = w_f - (eps/4)((1+k) psi+_f D_f + (1-k) psi-_f D_{f+1})
BF_DEV double muscl_right(double w1, double w2, double w3, double pp, double pm, const Consts& c) {
  if (c.eps0) return w2;
  const double d0 = w2 - w1;
  const double dp = w3 - w2;
#if BF_EXACT
  return w2 - c.quarter * (c.opk * pp * d0 + c.omk * pm * dp);
#else
  if (c.kappa_m1) return w2 - c.quarter * (c.omk * pm * dp);
  return w2 - c.quarter * (c.opk * pp * d0 + c.omk * pm * dp);
#endif
}

// Wall / farfield face flux replacing the MUSCL one (solver.py:526-580).
// c0..c3: var-0 pointers of cells f-2..f+1 (var stride vs); F already scaled by A.
BF_DEV void boundary_overwrite(int bkind, double side_sign, const double* c0, const double* c1,
                               const double* c2, const double* c3, int vs, double nx, double ny,
                               double nz, double A, const Consts& c, double F[5]) {
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

template <int FLUX, int LIM>
BF_DEV int face_flux(const double* c0, const double* c1, const double* c2, const double* c3, int vs,
                     const double* ppl, const double* pml, const double* ppr, const double* pmr,
                     int ps, double nx, double ny, double nz, double A, int bkind,
                     double side_sign, const Consts& c, double F[5]) {
  double qL[5], qR[5];
#pragma unroll
  for (int v = 0; v < 5; ++v) {
    double a_pl = 1.0, a_ml = 1.0, a_pr = 1.0, a_mr = 1.0;
    if constexpr (psi_count<LIM>() > 0) {
      a_pl = ppl[v * ps];
      a_pr = ppr[v * ps];
      a_ml = pml[v * ps];
      a_mr = pmr[v * ps];
    }
    qL[v] = muscl_left(c0[v * vs], c1[v * vs], c2[v * vs], a_pl, a_ml, c);
    qR[v] = muscl_right(c1[v * vs], c2[v * vs], c3[v * vs], a_pr, a_mr, c);
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
  if (bkind != BFACE_NONE) boundary_overwrite(bkind, side_sign, c0, c1, c2, c3, vs, nx, ny, nz, A, c, F);
  return err;
}

// Fused ghost fill (StageArgs::fill_ctas, defined after the ghost kernel below)
__device__ __noinline__ void fill_work(const GhostArgs& g, int nchunks, int worker, int nworkers,
                                       unsigned* sync, unsigned parties, GhostTask* slot);
BF_DEV void fill_arrive(unsigned* sync, unsigned n, unsigned parties);
BF_DEV void fill_wait(const unsigned* sync, int nworkers);

#include "bf_stage.cuh"
#if !BF_EXACT
#include "bf_vl.cuh"
#include "bf_roe.cuh"
#endif

// ---------------------------------------------------------------------------
// ghost fill / pack / unpack (one launch per stage, all blocks)
// ---------------------------------------------------------------------------

// Whether the cell at offset `o` (from the interior origin) is an interior cell.
// (Padded blocks hold < 2^31 cells: 32-bit division.)
BF_DEV bool is_interior(const DevBlock& b, long long o) {
  const int g3 = b.ndim == 3 ? b.g : 0;
  const unsigned s = (unsigned)(o + b.g + b.sy * b.g + b.sz * g3);   // shift coords to >= 0
  const unsigned sz = (unsigned)b.sz, sy = (unsigned)b.sy;
  const unsigned k = s / sz, r = s - k * sz;
  const unsigned j = r / sy, i = r - j * sy;
  return i >= (unsigned)b.g && i < (unsigned)(b.g + b.n[0]) && j >= (unsigned)b.g &&
         j < (unsigned)(b.g + b.n[1]) && k >= (unsigned)g3 && k < (unsigned)(g3 + b.n[2]);
}

// The stored T of a cell as the reference holds it: interior cells carry
// p/(rho R) once updated (solver.py:753, not stored by the stage kernels),
// ghost cells whatever their ghost fill wrote.
BF_DEV double cell_T(const DevBlock& b, const double* W, long long o, int t_derived,
                     const Consts& c) {
  return (t_derived && is_interior(b, o)) ? W[4 * b.fsz + o] / (W[o] * c.R)
                                          : W[5 * b.fsz + o];
}

// One ghost cell's six stored values (rho u v w p T); 2D tasks carry five
// fields (no w) in buffers, in this order (halo.py:27-32).
struct G6 {
  double r, u, v, w, p, T;
};

// Values of one COPY item (source cell -> destination ghost / buffer slot).
BF_DEV void copy_load(const GhostArgs& a, const GhostTask& t, unsigned m, G6& v, long long& doff) {
  const Consts& c = a.c;
  const unsigned n0 = (unsigned)t.n[0], n1 = (unsigned)t.n[1];
  const unsigned r = m / n0;
  const long long o0 = m - r * n0;
  const unsigned o2u = r / n1;
  const long long o1 = r - o2u * n1, o2 = o2u;
  doff = t.dst_origin + o0 * t.dst_stride[0] + o1 * t.dst_stride[1] + o2 * t.dst_stride[2];
  const long long soff = t.src_origin + o0 * t.src_stride[0] + o1 * t.src_stride[1] +
                         o2 * t.src_stride[2];
  const bool three = t.nfields == 6;
  v.w = 0.0;
  if (t.src_block >= 0) {
    const DevBlock& sb = a.blocks[t.src_block];
    const double* W = sb.base + (long long)fw(a.cur, 0) * sb.fsz;
    v.r = W[soff];
    v.u = W[sb.fsz + soff];
    v.v = W[2 * sb.fsz + soff];
    if (three) v.w = W[3 * sb.fsz + soff];
    v.p = W[4 * sb.fsz + soff];
    v.T = cell_T(sb, W, soff, a.t_derived, c);
  } else {
    const double* B = t.src_buf + soff;
    const long long bs = t.buf_cells;
    v.r = B[0];
    v.u = B[bs];
    v.v = B[2 * bs];
    if (three) {
      v.w = B[3 * bs];
      v.p = B[4 * bs];
      v.T = B[5 * bs];
    } else {
      v.p = B[3 * bs];
      v.T = B[4 * bs];
    }
  }
  if (t.live_mask) {   // round-2 fields packed by reference: read them now (halo.py:58)
    const DevBlock& lb = a.blocks[t.live_block];
    const double* W = lb.base + (long long)fw(a.cur, 0) * lb.fsz;
    const long long loff = t.live_origin + o0 * t.live_stride[0] + o1 * t.live_stride[1] +
                           o2 * t.live_stride[2];
    const int nf = t.nfields;
    if (t.live_mask & 1) v.r = W[loff];
    if (t.live_mask & (1 << (nf - 2))) v.p = W[4 * lb.fsz + loff];
    if (t.live_mask & (1 << (nf - 1))) v.T = cell_T(lb, W, loff, a.t_derived, c);
  }
}

BF_DEV void copy_store(const GhostArgs& a, const GhostTask& t, const G6& v, long long doff) {
  const bool three = t.nfields == 6;
  if (t.block >= 0) {
    const DevBlock& db = a.blocks[t.block];
    double* W = db.base + (long long)fw(a.cur, 0) * db.fsz;
    W[doff] = v.r;
    W[db.fsz + doff] = v.u;
    W[2 * db.fsz + doff] = v.v;
    if (three) W[3 * db.fsz + doff] = v.w;
    W[4 * db.fsz + doff] = v.p;
    W[5 * db.fsz + doff] = v.T;
  } else {
    double* B = t.dst_buf + doff;
    const long long bs = t.buf_cells;
    B[0] = v.r;
    B[bs] = v.u;
    B[2 * bs] = v.v;
    if (three) {
      B[3 * bs] = v.w;
      B[4 * bs] = v.p;
      B[5 * bs] = v.T;
    } else {
      B[3 * bs] = v.p;
      B[4 * bs] = v.T;
    }
  }
}

BF_DEV void bc_item(const GhostArgs& a, const GhostTask& t, unsigned m);

// One task per CUDA block; the block covers ipt x GHOST_BLOCK items of it
// (strided by GHOST_BLOCK; ipt = GHOST_ITEMS for large launches, 1 for small).  COPY items load all their values before the
// first store (GHOST_ITEMS x 6 loads in flight per thread).
#ifndef BF_GHOST_MINB
#define BF_GHOST_MINB 1
#endif
__global__ void __launch_bounds__(GHOST_BLOCK, BF_GHOST_MINB) ghost_kernel(const GhostArgs a) {
  __shared__ __align__(16) GhostTask ts;   // the task record, staged once
  pdl_trigger();
  const int2 bm = a.block_map[blockIdx.x];
  {
    static_assert(sizeof(GhostTask) % 8 == 0, "GhostTask words");
    constexpr int NW = (int)(sizeof(GhostTask) / 8);
    const unsigned long long* src =
        reinterpret_cast<const unsigned long long*>(a.tasks + bm.x);
    for (int w = threadIdx.x; w < NW; w += blockDim.x)
      reinterpret_cast<unsigned long long*>(&ts)[w] = src[w];
  }
  pdl_wait();   // static tables above; the fields below were written by the previous kernel
  if (a.stop && *a.stop) return;           // batched iterate stopped (RunState)
  __syncthreads();
  const GhostTask& t = ts;
  // items per task < 2^31 (a few face layers of one block)
  const unsigned m0 = (unsigned)bm.y + threadIdx.x;
  const unsigned items = (unsigned)t.items;
  if (t.kind == GK_COPY) {
    G6 v[GHOST_ITEMS];
    long long doff[GHOST_ITEMS];
#pragma unroll
    for (int q = 0; q < GHOST_ITEMS; ++q) {
      const unsigned m = m0 + q * GHOST_BLOCK;
      if (q < a.ipt && m < items) copy_load(a, t, m, v[q], doff[q]);
    }
#pragma unroll
    for (int q = 0; q < GHOST_ITEMS; ++q) {
      const unsigned m = m0 + q * GHOST_BLOCK;
      if (q < a.ipt && m < items) copy_store(a, t, v[q], doff[q]);
    }
    return;
  }
#pragma unroll 1
  for (int q = 0; q < a.ipt; ++q) {
    const unsigned m = m0 + q * GHOST_BLOCK;
    if (m < items) bc_item(a, t, m);
  }
}

// ---- fused ghost fill: the work of one ghost_kernel launch done by warps of a
// stage-kernel launch.  Chunk c is quarter (c & 3) of block-map entry c >> 2:
// exactly the items threads (c & 3) * 32 + lane of that ghost_kernel block take,
// so every ghost value is the same double the separate launch writes.
BF_DEV void ghost_warp_chunk(const GhostArgs& a, const GhostTask& t, int2 bm, int quarter,
                             int lane) {
  const unsigned m0 = (unsigned)bm.y + (unsigned)(quarter * 32 + lane);
  const unsigned items = (unsigned)t.items;
  if (t.kind == GK_COPY) {
    G6 v[GHOST_ITEMS];
    long long doff[GHOST_ITEMS];
#pragma unroll
    for (int q = 0; q < GHOST_ITEMS; ++q) {
      const unsigned m = m0 + q * GHOST_BLOCK;
      if (q < a.ipt && m < items) copy_load(a, t, m, v[q], doff[q]);
    }
#pragma unroll
    for (int q = 0; q < GHOST_ITEMS; ++q) {
      const unsigned m = m0 + q * GHOST_BLOCK;
      if (q < a.ipt && m < items) copy_store(a, t, v[q], doff[q]);
    }
    return;
  }
#pragma unroll 1
  for (int q = 0; q < a.ipt; ++q) {
    const unsigned m = m0 + q * GHOST_BLOCK;
    if (m < items) bc_item(a, t, m);
  }
}

// A participant is through with the counters; the last of `parties` resets them
// for the next launch (every counter operation precedes its arrival).
BF_DEV void fill_arrive(unsigned* sync, unsigned n, unsigned parties) {
  if (atomicAdd(sync + 2, n) + n == parties) {
    atomicExch(sync + 1, 0u);
    atomicExch(sync + 2, 0u);
  }
}

// Fill worker `worker` of `nworkers` (one warp): chunks worker, worker +
// nworkers, ...; the chunk's task record is staged in the warp's shared-memory
// slot (one coalesced load instead of a chain of field loads).  At the end one
// release increment of the done counter (sync[1]) — the warp's stores are
// ordered before it by __syncwarp and the cumulative __threadfence — and the
// warp's arrival.  Out of line: the ghost code's registers stay out of the
// stage kernel's allocation.
__device__ __noinline__ void fill_work(const GhostArgs& g, int nchunks, int worker, int nworkers,
                                       unsigned* sync, unsigned parties, GhostTask* slot) {
  const int lane = threadIdx.x & 31;
  constexpr int NW = (int)(sizeof(GhostTask) / 8);
  int staged = -1;
  for (int c = worker; c < nchunks; c += nworkers) {
    const int2 bm = g.block_map[c >> 2];
    if (bm.x != staged) {
      __syncwarp();
      const unsigned long long* src = reinterpret_cast<const unsigned long long*>(g.tasks + bm.x);
      for (int w = lane; w < NW; w += 32) reinterpret_cast<unsigned long long*>(slot)[w] = src[w];
      __syncwarp();
      staged = bm.x;
    }
    ghost_warp_chunk(g, *slot, bm, c & 3, lane);
  }
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    atomicAdd(sync + 1, 1u);
    fill_arrive(sync, 1u, parties);
  }
}

// Acquire: every fill worker's ghost stores are visible to this CTA (the
// acquire load invalidates stale L1 lines); the proxy fence orders them before
// the caller's TMA (async proxy) reads of the ghost cells.
BF_DEV void fill_wait(const unsigned* sync, int nworkers) {
  for (;;) {
    unsigned d;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(d) : "l"(sync + 1) : "memory");
    if ((int)d >= nworkers) break;
    __nanosleep(64);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

BF_DEV void bc_item(const GhostArgs& a, const GhostTask& t, unsigned m) {
  const Consts& c = a.c;
  // ---- physical patch: one tangential position, all ghost layers ----------
  const DevBlock& b = a.blocks[t.block];
  const long long fsz = b.fsz;
  double* W = b.base + (long long)fw(a.cur, 0) * fsz;
  const unsigned tn0 = (unsigned)t.tn[0];
  const unsigned u1 = m / tn0, u0 = m - u1 * tn0;
  auto stride = [&](int ax) -> long long { return ax == 0 ? 1 : (ax == 1 ? b.sy : b.sz); };
  const int d = t.axis;
  const long long sd = stride(d);
  const long long base =
      (long long)(t.tlo[0] + (int)u0) * stride(t.ta) + (long long)(t.tlo[1] + (int)u1) * stride(t.tb);
  const int n = b.n[d];
  // ghost position / mirror interior position of layer L (solver.py:300-304)
  auto gpos = [&](int L) { return t.side == 0 ? -1 - L : n + L; };
  auto ipos = [&](int L) { return t.side == 0 ? L : n - 1 - L; };
  const int bc = t.bc_type;
  if (bc == BC_INFLOW) {
    for (int L = 0; L < t.depth; ++L) {
      const long long o = base + sd * gpos(L);
      W[o] = c.fs_rho;
      W[fsz + o] = c.fs_u;
      W[2 * fsz + o] = c.fs_v;
      W[3 * fsz + o] = c.fs_w;
      W[4 * fsz + o] = c.fs_p;
      W[5 * fsz + o] = c.fs_T;
    }
  } else if (bc == BC_OUTFLOW) {
    const long long oi = base + sd * ipos(0);
    const double v0 = W[oi], v1 = W[fsz + oi], v2 = W[2 * fsz + oi], v3 = W[3 * fsz + oi],
                 v4 = W[4 * fsz + oi];
    const double v5 = cell_T(b, W, oi, a.t_derived, c);
    for (int L = 0; L < t.depth; ++L) {
      const long long o = base + sd * gpos(L);
      W[o] = v0;
      W[fsz + o] = v1;
      W[2 * fsz + o] = v2;
      W[3 * fsz + o] = v3;
      W[4 * fsz + o] = v4;
      W[5 * fsz + o] = v5;
    }
  } else if (bc == BC_SLIP || bc == BC_NOSLIP) {
    const long long fo = base + sd * (t.side == 0 ? 0 : n);
    const double sg = t.side == 0 ? -1.0 : 1.0;
    const double* fn = b.base + (long long)ffn(d, 0) * fsz + fo;
    const double nx = sg * fn[0], ny = sg * fn[fsz], nz = sg * fn[2 * fsz];
    // the usual two ghost layers: every mirror cell's values are loaded before
    // any ghost store (an item's ghost and interior positions never coincide),
    // so the loads of both layers are in flight together
    double pre[2][5];
    const bool two = t.depth == 2;
    if (two) {
#pragma unroll
      for (int L = 0; L < 2; ++L) {
        const long long oi = base + sd * ipos(L);
        pre[L][0] = W[fsz + oi];
        pre[L][1] = W[2 * fsz + oi];
        pre[L][2] = W[3 * fsz + oi];
        pre[L][3] = W[4 * fsz + oi];
        pre[L][4] = cell_T(b, W, oi, a.t_derived, c);
      }
    }
    for (int L = 0; L < t.depth; ++L) {
      const long long og = base + sd * gpos(L);
      const long long oi = base + sd * ipos(L);
      if (two) {
        const double u = pre[L & 1][0], v = pre[L & 1][1], w = pre[L & 1][2];
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
        const double pg = pre[L & 1][3];
        W[4 * fsz + og] = pg;
        const double ti = pre[L & 1][4];
        const double tg = (bc == BC_NOSLIP && c.has_tw) ? 2.0 * c.tw - ti : ti;
        W[5 * fsz + og] = tg;
        W[og] = pg / (c.R * tg);
        continue;
      }
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
      const double ti = cell_T(b, W, oi, a.t_derived, c);
      const double tg = (bc == BC_NOSLIP && c.has_tw) ? 2.0 * c.tw - ti : ti;
      W[5 * fsz + og] = tg;
      W[og] = pg / (c.R * tg);
    }
  } else if (bc == BC_FARFIELD) {
    const long long fo = base + sd * (t.side == 0 ? 0 : n);
    const double sg = t.side == 0 ? -1.0 : 1.0;
    const double* fn = b.base + (long long)ffn(d, 0) * fsz + fo;
    const double nx = sg * fn[0], ny = sg * fn[fsz], nz = sg * fn[2 * fsz];
    const long long oi = base + sd * ipos(0);
    const St s{W[oi], W[fsz + oi], W[2 * fsz + oi], W[3 * fsz + oi], W[4 * fsz + oi]};
    const St q = farfield_state(s, nx, ny, nz, c);
    const double tb = q.p / (q.r * c.R);
    for (int L = 0; L < t.depth; ++L) {
      const long long o = base + sd * gpos(L);
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
      const long long o = base + sd * gpos(L);
      const double* src = t.dirichlet + (long long)L * 6 * nt + m;
      for (int f = 0; f < 6; ++f) W[f * fsz + o] = src[f * nt];
    }
  }
}

// ---------------------------------------------------------------------------
// laminar viscous face fluxes (solver.py:644-692, physics.py:312-344)
// ---------------------------------------------------------------------------
// mu(T): constant or Sutherland (physics.py:79-85), reference operation order
BF_DEV double viscosity(double T, const Consts& c) {
  if (!c.has_suth) return c.mu;
  return c.suth_mu * pow(T / c.suth_t, 1.5) * (c.suth_t + c.suth_s) / (T + c.suth_s);
}

// One thread per face (f along d, interior tangential) of one block direction:
// Fv x A into the block's viscous-flux slots (vis0 + 27 + 4 d + m), the stage
// kernel subtracts them after the inviscid flux and its boundary overwrite.
__global__ void __launch_bounds__(128) viscous_kernel(const ViscArgs a) {
  const int2 bm = a.map[blockIdx.x];
  const ViscTask t = a.tasks[bm.x];
  const long long m = (long long)bm.y + threadIdx.x;
  if (m >= t.items) return;
  const DevBlock& b = a.blocks[t.block];
  const Consts& c = a.c;
  const int d = t.d;
  const int i = (int)(m % t.e[0]);
  const long long r = m / t.e[0];
  const int j = (int)(r % t.e[1]), k = (int)(r / t.e[1]);
  const long long st[3] = {1, b.sy, b.sz};
  const long long fsz = b.fsz;
  const long long hi = i + b.sy * (long long)j + b.sz * (long long)k;   // cell f (face f)
  const long long lo = hi - st[d];                                      // cell f-1
  const double* W = b.base + (long long)fw(a.cur, 0) * fsz;
  const int ndim = b.ndim;
  // field n of cell o: u, v, w (slots 1..3) or T (stored / derived)
  auto val = [&](int n, long long o) {
    return n < 3 ? W[(n + 1) * fsz + o] : cell_T(b, W, o, a.t_derived, c);
  };
  double dxi[4][3], avg[4];
#pragma unroll
  for (int n = 0; n < 4; ++n) {
    const double wl = val(n, lo), wh = val(n, hi);
    dxi[n][0] = dxi[n][1] = dxi[n][2] = 0.0;
    dxi[n][d] = wh - wl;
    for (int e = 0; e < ndim; ++e) {
      if (e == d) continue;
      const double plus = val(n, lo + st[e]) + val(n, hi + st[e]);
      const double minus = val(n, lo - st[e]) + val(n, hi - st[e]);
      dxi[n][e] = 0.25 * (plus - minus);
    }
    avg[n] = 0.5 * (wl + wh);
  }
  // physical gradients: row r = sum over e (in order) of invT[d][r][e] * dxi[e]
  const double* M = b.base + (long long)(b.vis0 + 9 * d) * fsz + hi;
  double gr[4][3];
#pragma unroll
  for (int n = 0; n < 4; ++n)
#pragma unroll
    for (int row = 0; row < 3; ++row) {
      double acc = M[(3 * row + 0) * fsz] * dxi[n][0];
      acc = acc + M[(3 * row + 1) * fsz] * dxi[n][1];
      if (ndim == 3) acc = acc + M[(3 * row + 2) * fsz] * dxi[n][2];
      gr[n][row] = acc;
    }
  const double mu = viscosity(avg[3], c);
  const double kc = mu * c.cp / c.prandtl;
  const double* fn = b.base + (long long)ffn(d, 0) * fsz + hi;
  const double nx = fn[0], ny = fn[fsz], nz = fn[2 * fsz], A = fn[3 * fsz];
  // physics.py:312-344
  const double div = gr[0][0] + gr[1][1] + gr[2][2];
  const double lam = -2.0 / 3.0 * mu;
  const double txx = 2.0 * mu * gr[0][0] + lam * div;
  const double tyy = 2.0 * mu * gr[1][1] + lam * div;
  const double tzz = 2.0 * mu * gr[2][2] + lam * div;
  const double txy = mu * (gr[0][1] + gr[1][0]);
  const double txz = mu * (gr[0][2] + gr[2][0]);
  const double tyz = mu * (gr[1][2] + gr[2][1]);
  const double fx = nx * txx + ny * txy + nz * txz;
  const double fy = nx * txy + ny * tyy + nz * tyz;
  const double fz = nx * txz + ny * tyz + nz * tzz;
  const double u = avg[0], v = avg[1], w = avg[2];
  const double qx = u * txx + v * txy + w * txz + kc * gr[3][0];
  const double qy = u * txy + v * tyy + w * tyz + kc * gr[3][1];
  const double qz = u * txz + v * tyz + w * tzz + kc * gr[3][2];
  const double fe = nx * qx + ny * qy + nz * qz;
  double* out = b.base + (long long)(b.vis0 + 27 + 4 * d) * fsz + hi;
  out[0] = fx * A;
  out[fsz] = fy * A;
  out[2 * fsz] = fz * A;
  out[3 * fsz] = fe * A;
}

// Fixed-order per-block reduction of the per-tile partial sums by the first
// GUARD_NT threads of a CTA (strided per-thread sums, then a shared-memory
// tree; the other threads only take part in the barriers): the same doubles
// whichever kernel runs it.
constexpr int GUARD_NT = 256;
BF_DEV void block_sum(const double* partial, int tb, int te, double* red, double* out5) {
  // strided per-thread sums, a shuffle tree per warp, then warp 0 over the warp
  // sums (two barriers instead of a shared-memory tree's eight); the block's five
  // sums end in out5 and red[0..4]
  constexpr int NW = GUARD_NT / 32;
  const bool on = threadIdx.x < GUARD_NT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double x[5] = {0, 0, 0, 0, 0};
  if (on)
    for (int t = tb + threadIdx.x; t < te; t += GUARD_NT) {
#pragma unroll
      for (int v = 0; v < 5; ++v) x[v] += __ldcg(partial + (long long)t * 5 + v);
    }
#pragma unroll
  for (int v = 0; v < 5; ++v)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) x[v] += __shfl_down_sync(0xffffffffu, x[v], off);
  if (on && lane == 0) {
#pragma unroll
    for (int v = 0; v < 5; ++v) red[warp * 5 + v] = x[v];
  }
  __syncthreads();
  if (threadIdx.x < 32) {
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      double y = lane < NW ? red[lane * 5 + v] : 0.0;
#pragma unroll
      for (int off = NW / 2; off > 0; off >>= 1) y += __shfl_down_sync(0xffffffffu, y, off);
      x[v] = y;
    }
  }
  __syncthreads();   // every warp's red reads are done before thread 0 overwrites red[0..4]
  if (threadIdx.x == 0) {
#pragma unroll
    for (int v = 0; v < 5; ++v) {
      red[v] = x[v];
      out5[v] = x[v];
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(GUARD_NT) reduce_kernel(const double* partial, const int* tile_begin,
                                                     int nblocks, double* out) {
  __shared__ double red[GUARD_NT * 5];
  pdl_trigger();
  pdl_wait();
  const int blk = blockIdx.x;
  if (blk >= nblocks) return;
  block_sum(partial, tile_begin[blk], tile_begin[blk + 1], red, out + blk * 5);
}

// ---------------------------------------------------------------------------
// launchers (called by the runtime)
#if !BF_EXACT
// BF_VL=0 in the environment selects the reference-order kernel for FAST Van
// Leer too (A/B measurements).
static bool vl_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BF_VL");
    v = (e && e[0] == '0') ? 1 : 0;
  }
  return v == 1;
}
#endif
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
  return launch_pdl(k, (unsigned)a.ntiles, (unsigned)K::NT, K::BYTES, s, a);
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

#if !BF_EXACT
// FAST Van Leer with limiters computed in-kernel runs the cell-split kernel
// (bf_vl.cuh), which also pushes the next stage's ghosts when a.push is set.
bool vl_push_compiled() { return BF_VL_PUSH != 0; }

bool vl_active(int flux, int flags) {
  return flux == FLUX_VAN_LEER && !(flags & (F_PSI_LOAD | F_PSI_STORE)) && !vl_disabled();
}

// FAST Roe with limiters computed in-kernel runs the face-owner kernel
// (bf_roe.cuh); BF_ROE_SPLIT=0 keeps it on the reference-order kernel.
static bool roe_split_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BF_ROE_SPLIT");
    v = (e && e[0] == '0') ? 1 : 0;
  }
  return v == 1;
}

bool roe_split_active(int flux, int flags) {
  return flux == FLUX_ROE && !(flags & (F_PSI_LOAD | F_PSI_STORE)) && !roe_split_disabled();
}
#endif

cudaError_t launch_stage(int ndim, int flux, int lim, const StageArgs& a, cudaStream_t s) {
#if !BF_EXACT
  if (vl_active(flux, a.flags) && !a.c.viscous) return launch_vl(ndim, lim, a, s);
  if (roe_split_active(flux, a.flags) && !a.c.viscous) return launch_roe(ndim, lim, a, s);
#endif
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
  if (a.total_items == 0 || a.nlaunch == 0) return cudaSuccess;
  return launch_pdl(ghost_kernel, (unsigned)a.nlaunch, (unsigned)GHOST_BLOCK, 0, s, a);
}

cudaError_t launch_viscous(const ViscArgs& a, int nlaunch, cudaStream_t s) {
  if (nlaunch == 0) return cudaSuccess;
  viscous_kernel<<<(unsigned)nlaunch, 128, 0, s>>>(a);
  return cudaGetLastError();
}

// End of a batched-iterate step (RunState, bf_internal.h), one launch instead of
// the stage-0 reduce, the D2H of the sums and the host guard: the per-block
// sums (reduce_kernel's arithmetic), the step's norms from them in block order
// (as finish_collect sums them on the host), check_history_guards
// (solver.py:836-855) as history_guard in bf_runtime.cu evaluates it, with
// numpy's NaN semantics, and the reset of the error slot for the next step.
// The guard of one batched step (red: GUARD_NT x 5 doubles of shared memory;
// every thread of the CTA calls it).
// The history guards of one step from its global Σ R² (h, the five sums) and
// error state; thread 0 of the calling CTA.  r: the run state loaded up front.
BF_DEV void guard_tail(double h[5], unsigned long long key, int bad_rank, RunState& r,
                       RunState* rs, double* hist, unsigned long long* err) {
  const int s = r.steps;
  *err = ~0ull;   // the next step's error slot (the per-step reset of bf_step)
  if ((key != ~0ull || bad_rank >= 0) && !r.ignore_errors) {   // non-physical state in this step
    rs->key = key;
    rs->bad_rank = bad_rank;   // the first rank that recorded one (multi-rank batches)
    rs->status = 3;
    rs->stop = 1;
    return;
  }
  for (int v = 0; v < 5; ++v) {
    h[v] = sqrt(h[v]);
    hist[5 * s + v] = h[v];
  }
  if (!r.has_base) {
    for (int v = 0; v < 5; ++v) rs->base[v] = r.base[v] = h[v];
    rs->has_base = 1;
  }
  rs->steps = s + 1;
  auto npmax = [](const double* x) {
    double m = x[0];
    for (int v = 1; v < 5; ++v)
      if (isnan(x[v]) || x[v] > m || isnan(m)) m = isnan(m) ? m : x[v];
    return m;
  };
  int g = 0;
  if (r.has_floor && npmax(h) <= r.floor_) {
    g = 1;
  } else {
    const double* bs = r.base;
    const double bmax = npmax(bs);
    bool any = false, bad = false;
    double rmax = 0.0;
    for (int v = 0; v < 5; ++v) {
      if (!(bs[v] > 1e-12 * bmax)) continue;
      const double q = h[v] / bs[v];
      if (!isfinite(q)) bad = true;
      rmax = any ? (q > rmax ? q : rmax) : q;
      any = true;
    }
    if (any) {
      if (bad || rmax > r.factor) g = 2;
      else if (r.has_target && rmax <= r.target) g = 1;
    }
  }
  if (g) {
    rs->status = g;
    rs->stop = 1;
  }
}

BF_DEV void guard_body(const double* partial, const int* tile_begin, int nb, double* blocksum,
                       unsigned long long* err, RunState* rs, double* hist, double* red) {
  // thread 0 loads the run state and the step's error key up front: their
  // latency overlaps the sums (one launch-bound chain less on small grids)
  RunState r;
  unsigned long long key = ~0ull;
  if (threadIdx.x == 0) {
    r = *rs;
    key = *reinterpret_cast<volatile unsigned long long*>(err);
  }
  // per-block sums exactly as reduce_kernel forms them (block_sum); the step's
  // norms from them in block order (thread 0 reads each block's sums from red[0..4]
  // before the next block_sum writes its own slots there)
  double h[5] = {0, 0, 0, 0, 0};
  for (int b = 0; b < nb; ++b) {
    block_sum(partial, tile_begin[b], tile_begin[b + 1], red, blocksum + 5 * b);
    if (threadIdx.x == 0)
      for (int v = 0; v < 5; ++v) h[v] = h[v] + red[v];
  }
  if (threadIdx.x != 0) return;
  guard_tail(h, key, -1, r, rs, hist, err);
}

// Multi-rank batches (bf_iterate over NCCL / loopback ranks): before the
// rank allgather, this rank's record [Σ over its blocks in id order (as
// finish_collect sums them), error key bits]; after it, the global sums in
// rank order (as rank_allgather sums them) and the guards, every rank alike.
__global__ void rank_record_kernel(const double* blocksum, int nb, const unsigned long long* err,
                                   double* rec6, const RunState* rs) {
  pdl_wait();
  if (rs->stop) return;
  double s[5] = {0, 0, 0, 0, 0};
  for (int b = 0; b < nb; ++b)
    for (int v = 0; v < 5; ++v) s[v] = s[v] + blocksum[5 * b + v];
  for (int v = 0; v < 5; ++v) rec6[v] = s[v];
  rec6[5] = __longlong_as_double((long long)*err);
}

__global__ void rank_guard_kernel(const double* gather, int nranks, int rank,
                                  unsigned long long* err, RunState* rs, double* hist) {
  pdl_wait();
  if (rs->stop) return;
  RunState r = *rs;
  double tot[5];
  int bad = -1;
  for (int q = 0; q < nranks; ++q) {
    for (int v = 0; v < 5; ++v) tot[v] = (q == 0) ? gather[6 * q + v] : tot[v] + gather[6 * q + v];
    const unsigned long long k = (unsigned long long)__double_as_longlong(gather[6 * q + 5]);
    if (k != ~0ull && bad < 0) bad = q;
  }
  const unsigned long long own = (unsigned long long)__double_as_longlong(gather[6 * rank + 5]);
  guard_tail(tot, own, bad, r, rs, hist, err);
}

// One CTA per block forms the block's sums (block_sum); the last CTA to finish
// (counter, reset by it) sums the blocks in id order and evaluates the guards.
__global__ void __launch_bounds__(GUARD_NT) guard_kernel(const double* partial,
                                                         const int* tile_begin, int nb,
                                                         double* blocksum,
                                                         unsigned long long* err, RunState* rs,
                                                         double* hist, unsigned* count) {
  __shared__ double red[GUARD_NT * 5];
  __shared__ int last;
  pdl_trigger();
  pdl_wait();
  if (rs->stop) return;
  if (nb == 1 || !count) {   // one block (or no counter): the whole guard in this CTA
    guard_body(partial, tile_begin, nb, blocksum, err, rs, hist, red);
    return;
  }
  const int b = blockIdx.x;
  block_sum(partial, tile_begin[b], tile_begin[b + 1], red, blocksum + 5 * b);
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(count, 1u) == (unsigned)(nb - 1);
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  *count = 0u;
  RunState r = *rs;
  const unsigned long long key = *reinterpret_cast<volatile unsigned long long*>(err);
  double h[5] = {0, 0, 0, 0, 0};
  for (int q = 0; q < nb; ++q)
    for (int v = 0; v < 5; ++v) h[v] = h[v] + __ldcg(blocksum + 5 * q + v);
  guard_tail(h, key, -1, r, rs, hist, err);
}

cudaError_t launch_guard(const double* partial, const int* tile_begin, int nb, double* blocksum,
                         unsigned long long* err, RunState* rs, double* hist, unsigned* count,
                         cudaStream_t s) {
  const unsigned grid = (nb > 1 && count) ? (unsigned)nb : 1u;
  return launch_pdl(guard_kernel, grid, (unsigned)GUARD_NT, 0, s, partial, tile_begin, nb,
                    blocksum, err, rs, hist, count);
}

cudaError_t launch_rank_record(const double* blocksum, int nb, const unsigned long long* err,
                               double* rec6, const RunState* rs, cudaStream_t s) {
  return launch_pdl(rank_record_kernel, 1u, 1u, 0, s, blocksum, nb, err, rec6, rs);
}

cudaError_t launch_rank_guard(const double* gather, int nranks, int rank,
                              unsigned long long* err, RunState* rs, double* hist,
                              cudaStream_t s) {
  return launch_pdl(rank_guard_kernel, 1u, 1u, 0, s, gather, nranks, rank, err, rs, hist);
}

cudaError_t launch_reduce(const double* partial, const int* tile_begin, int nblocks, double* out,
                          cudaStream_t s) {
  if (nblocks == 0) return cudaSuccess;
  return launch_pdl(reduce_kernel, (unsigned)nblocks, (unsigned)GUARD_NT, 0, s, partial, tile_begin,
                    nblocks, out);
}

}  // namespace BF_NS
}  // namespace bf
