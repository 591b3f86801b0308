// bf_internal.h — device-side tables shared by the runtime and the kernels.
//
// HBM layout of one block: every per-cell array (W ping-pong x 6
// fields, Q x 5, dt/V, V, face normals/areas, sources, limiter arrays) uses the
// same padded, i-fastest layout with the interior origin 32-byte aligned, so a
// single (sy, sz) pair of strides addresses all of them and the stage kernel
// computes one offset per cell.  Pointers below are pre-offset to the interior
// origin: element (i, j, k) in interior coordinates (ghosts negative) is
// ptr[i + sy*j + sz*k].
#pragma once
#include <cstdint>

namespace bf {

// Stage-kernel tile: TI x TJ threads, each owning one (i, j) column that
// marches KC cells along k (2.5-D streaming); 2D blocks use the same tile
// with a single plane.
constexpr int TI = 32;                   // tile width (one warp per row)
#ifndef BF_TJ3
#define BF_TJ3 16
#endif
constexpr int TJ_3D = BF_TJ3;            // tile rows, 3D (16: 512 threads, 1 CTA/SM; 8: 2 CTAs/SM)
constexpr int TJ_2D = 8;                 // tile rows, 2D
constexpr int HALO = 2;                  // MUSCL stencil half-width
constexpr int NSLOT = 3;                 // plane ring: k, k+1 resident, k+2 landing (TMA)
constexpr int NTMAP = 6;                 // tensor maps per block: W plane, x/y face geometry,
                                         // Q0, dt/V (or V), z face geometry
constexpr int GXW = TI + 2;              // x-face geometry box width (16-byte multiple)

// Scheme switches (bfgpu.h BF_FLUX_* / BF_LIM_*)
constexpr int FLUX_ROE = 0;
constexpr int FLUX_VAN_LEER = 1;
constexpr int LIM_NONE = 0;
constexpr int LIM_VAN_LEER = 1;
constexpr int LIM_VAN_ALBADA = 2;
constexpr int LIM_MINMOD = 3;

// Physical BC types (bfgpu.h BF_BC_*, PHYSICAL_BC_TYPES order)
constexpr int BC_INFLOW = 0;
constexpr int BC_OUTFLOW = 1;
constexpr int BC_SLIP = 2;
constexpr int BC_NOSLIP = 3;
constexpr int BC_FARFIELD = 4;
constexpr int BC_MMS = 5;

// Stage flags
constexpr int F_STAGE0 = 1;      // first RK stage: compute dt/V and sum(R^2)
constexpr int F_LAST = 2;        // last RK stage: write Q
constexpr int F_PSI_STORE = 4;   // write limiter arrays (freeze step, last stage)
constexpr int F_PSI_LOAD = 8;    // read frozen limiter arrays instead of computing
constexpr int F_SOURCE = 16;     // subtract S*V (MMS)

// Boundary-face overwrite codes (solver.py:526-580)
constexpr unsigned char BFACE_NONE = 0;
constexpr unsigned char BFACE_WALL = 1;
constexpr unsigned char BFACE_FARFIELD = 2;

// Error kinds (mirror BF_ERR_* in bfgpu.h)
constexpr int ERR_FACE_LEFT = 1;
constexpr int ERR_FACE_RIGHT = 2;
constexpr int ERR_ROE_A2 = 3;
constexpr int ERR_UPDATE = 4;

struct Consts {
  double gamma, gm1, gog1, R;              // gamma, gamma-1, gamma/(gamma-1), R
  double cfl, quarter, omk, opk, efix;     // eps/4, 1-kappa, 1+kappa, entropy fix
  double fs_rho, fs_u, fs_v, fs_w, fs_p, fs_T;
  double ff_af;                            // sqrt(g*fs.p/fs.rho)
  double ff_two_af_gm1;                    // 2*af/(g-1)
  double ff_sf;                            // fs.p / fs.rho**g  (host libm pow)
  double ff_qgm1;                          // 0.25*(g-1)
  double ff_exp;                           // 1/(g-1)
  double two_over_gm1;                     // 2/(g-1)   (fast mode only)
  double vl_c;                             // 2*(g*g-1)
  double inv_gamma, inv_vlc;               // 1/gamma, 1/vl_c (fast mode only)
  double lim_eps, lim_eps_half;            // limiter epsilon 1e-12 and 1e-12/2 (constant-bank operands)
  double tw;                               // wall temperature
  int has_tw;
  double mu, prandtl, cp;                  // viscosity law (physics.py:47-90)
  double suth_mu, suth_t, suth_s;          // Sutherland (mu_ref, T_ref, S)
  double visc_coeff;                       // 2 max(4/3, gamma/Pr) (solver.py:722)
  int has_suth;
  int viscous;
  int eps0;                                // epsilon == 0
  int kappa_m1;                            // kappa == -1 (fast mode drops the zero terms)
  int muscl_k1;                            // epsilon == 1 and kappa == -1 (cell-split kernel)
};

// Field slots of a block arena (each slot fsz doubles, same padded layout).
constexpr int FW = 0;            // W[b][f] = FW + 6*b + f   (rho u v w p T, ping-pong b)
constexpr int FQ = 12;           // Q[e]    = FQ + e
constexpr int FDTV = 17;         // dt / V
constexpr int FVOL = 18;         // V
constexpr int FFN = 19;          // face geometry FFN + 4*d + c   (nx, ny, nz, A)
constexpr int FSRC = 31;         // S*V [5] when present; limiter arrays follow
// laminar NS (DevBlock::vis0 >= 0): face gradient matrices then viscous face fluxes
//   vis0 + 9*d + 3*r + e : grad_invT[d][r][e] at face f of direction d (stored at cell f)
//   vis0 + 27 + 4*d + m  : viscous flux x area, momentum x/y/z (m = 0..2), energy (m = 3)
constexpr int NVIS = 27 + 12;
__host__ __device__ constexpr int fw(int b, int f) { return FW + 6 * b + f; }
__host__ __device__ constexpr int ffn(int d, int c) { return FFN + 4 * d + c; }

struct DevBlock {
  int n[3];
  int g;            // ghost depth along stencil axes
  int ndim;
  int order;        // position of this block in the rank's id order
  int id;
  int psi0;         // first limiter slot (psi[d][pm][v] = psi0 + 10d + 5pm + v), -1: none
  int vis0;         // first viscous slot (NVIS slots), -1: inviscid
  int ox, oy, oz;   // TMA coordinates of interior cell (0,0,0) in the arena tensor
  long long sy, sz;
  long long fsz;    // doubles per slot
  double* base;     // arena base, pre-offset to the interior origin
  const unsigned char* bface[6];   // per face, over tangential interior cells
  __host__ __device__ double* f(int slot) const { return base + (long long)slot * fsz; }
};

struct Tile {
  int block;
  int i0, j0, k0, kc;
};

// Ghost-fill work item groups (one launch per stage covers every group).
enum GhostKind : int {
  GK_BC = 0,        // physical patch: one item per tangential cell, all layers
  GK_COPY = 1,      // affine copy: block->block (local link), block->buffer (pack),
                    // buffer->block (unpack)
};

struct GhostTask {
  int kind;
  int bc_type;          // GK_BC
  int block;            // GK_BC: block; GK_COPY: destination block (-1: buffer)
  int src_block;        // GK_COPY: source block (-1: buffer)
  int axis, side;       // GK_BC
  int ta, tb;           // GK_BC: tangential axes (tb = 2 with extent 1 in 2D)
  int tlo[2], tn[2];    // GK_BC: tangential start/extent (interior cells)
  int depth;            // ghost layers
  int nfields;          // GK_COPY: 6 (3D) or 5 (2D: rho u v p T)
  int n[3];             // GK_COPY: item box extents (i-fastest)
  int pad_;
  long long items;      // number of work items
  long long begin;      // prefix offset into the launch's item space
  long long dst_origin, dst_stride[3];
  long long src_origin, src_stride[3];
  long long buf_cells;  // field stride inside a message buffer
  double* dst_buf;      // GK_COPY into a buffer (pack)
  const double* src_buf;// GK_COPY from a buffer (unpack)
  // round-2 unpack of a local link: fields whose pack was a view of the
  // sender (halo.py:58, ravel of a contiguous box) are read from the sender
  // at unpack time — bit f of live_mask (buffer field order), map below
  int live_mask;
  int live_block;
  long long live_origin, live_stride[3];
  const double* dirichlet;   // GK_BC mms: [layer][6][tn0*tn1]
};

// Ghost launches are block-aligned: CUDA block b covers items
// [block_map[b].y, +GHOST_BLOCK * ipt) of task block_map[b].x (one task per block).
constexpr int GHOST_BLOCK = 128;
#ifndef BF_GHOST_ITEMS
#define BF_GHOST_ITEMS 4
#endif
constexpr int GHOST_ITEMS = BF_GHOST_ITEMS;          // max items per thread (unrolled loads)
constexpr int GHOST_SPAN = GHOST_BLOCK * GHOST_ITEMS;  // items per CUDA block (large launches)
// Small launches (fewer items than a few full-occupancy waves of GHOST_SPAN
// blocks, e.g. 2D grids) use one item per thread: more blocks, shorter chains.
constexpr long long GHOST_SMALL_ITEMS = 148LL * 4 * GHOST_SPAN;
// Large launches: 2 items per thread (with the blocks interleaved across tasks, C4
// fill 0.091-0.095 ms at 4, 0.087 ms at 2; profiles/r02_ghost_ipt.txt).
inline int ghost_ipt(long long total_items) {
  return total_items >= GHOST_SMALL_ITEMS ? (GHOST_ITEMS < 2 ? GHOST_ITEMS : 2) : 1;
}

struct GhostArgs {
  const DevBlock* blocks;
  const GhostTask* tasks;
  const int2* block_map;
  int nlaunch;          // CUDA blocks in the launch
  int ntasks;
  int cur;              // W buffer being filled
  int t_derived;        // interior T is p/(rho R) (after the first update)
  int extended;         // GK_BC: ghost round 2 (tangential range widened, solver.py:285-305)
  int ipt;              // items per thread (1 .. GHOST_ITEMS), as the block map was cut
  long long total_items;
  const int* stop;      // batched iterate: a set flag makes the launch a no-op (null: never)
  Consts c;
};

// Device-side state of a batched iterate (bf_iterate): the guard kernel at the
// end of every step sums the per-block sum(R^2) in block order, writes the
// step's norms and evaluates check_history_guards (solver.py:836-855); a
// fired guard or a recorded non-physical state sets `stop`, which turns the
// remaining launches of the batch into no-ops.
struct RunState {
  int stop;
  int steps;            // steps of the batch completed (guard evaluated)
  int status;           // 0 running, 1 converged, 2 diverged, 3 non-physical state
  int has_base;         // base = the call's first-step norms
  unsigned long long key;   // error key of status 3
  double base[5];
  int has_target, has_floor, ignore_errors;
  int bad_rank;         // status 3 of a multi-rank batch: first rank with a recorded error
  double target, floor_, factor;
};

// Ghost values pushed by the stage kernel (bf_vl.cuh): when a cell's new
// state is written, the cells it is the source of in the NEXT stage's ghost
// layers are written too — connected copies into the partner block's
// ghosts (halo.py:47-115 with the orientation folded into `coef`), message
// packing for remote partners, and the interior-dependent physical BCs
// (solver.py:281-403).  Inflow and MMS ghosts are constant (filled once).
enum PushKind : int { PK_COPY = 0, PK_PACK = 1, PK_OUTFLOW = 2, PK_SLIP = 3, PK_NOSLIP = 4,
                      PK_FARFIELD = 5 };
constexpr int PUSH_MAX_RULES = 12;   // per block (more: ghost kernel instead)
struct PushRule {
  int kind;
  int axis, side;        // the face the rule belongs to
  int nfields;           // COPY / PACK: 6 (3D) or 5 (2D: rho u v p T)
  int lo[3], hi[3];      // source cells covered (own interior coords, [lo, hi))
  long long base;        // COPY / PACK: destination offset of source cell lo
  long long coef[3];     // destination offset per source coordinate
  long long dst_fsz;     // COPY: destination slot size; PACK: buffer field stride
  double* dst;           // COPY: destination block (interior origin); PACK: send buffer
};

// Viscous face-flux launch: one task per (block, direction), faces f = 0..N_d
// over the interior tangential range (e[d] = N_d + 1).
struct ViscTask {
  int block, d;
  int e[3];
  int pad_;
  long long items;
};
struct ViscArgs {
  const DevBlock* blocks;
  const ViscTask* tasks;
  const int2* map;      // CUDA block -> (task, first item), 128 items per block
  int cur;
  int t_derived;
  Consts c;
};

struct StageArgs {
  const DevBlock* blocks;
  const Tile* tiles;
  const int* tile_list; // CTA b runs tile tile_list[b] (null: tile b); partials by tile id
  int ntiles;
  int cur;              // read W[cur], write W[cur ^ 1]
  int stage;
  int flags;
  double alpha;
  double* partial;      // [ntiles][5] sum(R^2) partials (stage 0)
  unsigned long long* err;   // [0] = min error key, [1..] unused
  const unsigned char* tmaps;   // [nblocks][NTMAP] CUtensorMap (128 B each) in global memory
  const PushRule* push_rules;   // ghost push (bf_vl.cuh), used when push != 0
  const int* push_range;        // [nblocks][6 faces][begin, end) into push_rules
  int push;
  int t_derived;        // interior T is p/(rho R) (viscous dt reads T)
  const int* stop;      // batched iterate: a set flag makes the launch a no-op (null: never)
  // Fused ghost fill (cell-split kernel, one-rank ctx; off when fill_chunks is
  // 0): the ghosts of W[cur] — the work of one ghost_kernel launch, cut into
  // fill_chunks warp chunks, assigned round robin — are written inside the
  // launch by the warps of its first fill_ctas CTAs; then come the tiles of
  // tile_list: n_interior tiles that read no ghost cell, then the boundary
  // tiles, which wait until fill_sync[1] (fill warps done) reaches every fill
  // warp.  fill_sync[2] counts arrivals (fill warps + boundary tiles); the last
  // one zeroes the counters for the next launch.
  int fill_chunks;
  int fill_ctas;
  int n_interior;
  unsigned* fill_sync;
  GhostArgs fill;
  Consts c;
};

// Error key: most significant first
//   stage(3) | phase(1: 0 residual, 1 update) | block order(12) | dir(2) | kind(2) | index(44)
__host__ __device__ inline unsigned long long make_err_key(int stage, int phase, int order,
                                                           int dir, int kind,
                                                           unsigned long long lin) {
  return ((unsigned long long)(stage & 7) << 61) | ((unsigned long long)(phase & 1) << 60) |
         ((unsigned long long)(order & 0xFFF) << 48) | ((unsigned long long)(dir & 3) << 46) |
         ((unsigned long long)(kind & 3) << 44) | (lin & ((1ull << 44) - 1));
}

}  // namespace bf
