/*
 * bfgpu.h — C ABI of the B200-native multi-block finite-volume hot path.
 *
 * One bf_ctx owns the blocks of ONE rank on ONE GPU and runs the reference's
 * per-RK-stage pipeline on the device.  Every entry point replaces a piece
 * of the reference's Python path (file:line into /root/reference/pkg/src/
 * blockflow/); the ctypes binding a maintainer adds is in INTEGRATION.md and
 * paper_2012_02925_b200/native.py.
 *
 * Conventions
 *   - plain pointers and sizes only; host arrays are float64, Fortran
 *     (i-fastest) order, exactly the reference's numpy layouts;
 *   - every int-returning call returns 0 on success or a BF_E* code, with a
 *     message retrievable through bf_last_error();
 *   - a ctx is not thread-safe; calls on one ctx must be serialised.
 */
#ifndef BFGPU_H
#define BFGPU_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BF_API_VERSION 1

/* return codes */
#define BF_OK 0
#define BF_EINVAL 1          /* bad argument / call order (ConfigError, TopologyError)  */
#define BF_ECUDA 2           /* CUDA runtime failure                                    */
#define BF_ENONPHYSICAL 3    /* NonPhysicalStateError: see bf_error_info()              */
#define BF_ENCCL 4           /* NCCL failure                                            */
#define BF_EMETRIC 5         /* MetricError: inverted cell (mesh.py compute_metrics)     */

/* solver.py:31-32 */
#define BF_FLUX_ROE 0
#define BF_FLUX_VAN_LEER 1
#define BF_LIM_NONE 0
#define BF_LIM_VAN_LEER 1
#define BF_LIM_VAN_ALBADA 2
#define BF_LIM_MINMOD 3

/* topology.py:25-32, same order as PHYSICAL_BC_TYPES */
#define BF_BC_SUPERSONIC_INFLOW 0
#define BF_BC_SUPERSONIC_OUTFLOW 1
#define BF_BC_SLIP_WALL 2
#define BF_BC_NOSLIP_WALL 3
#define BF_BC_FARFIELD 4
#define BF_BC_MMS_DIRICHLET 5

/* topology.py:23, FACES order: i_min i_max j_min j_max k_min k_max = 0..5 */

/* bf_download / bf_upload selectors */
#define BF_FIELD_RHO 0
#define BF_FIELD_U 1
#define BF_FIELD_V 2
#define BF_FIELD_W 3
#define BF_FIELD_P 4
#define BF_FIELD_T 5
#define BF_FIELD_Q0 6        /* Q0..Q4 = 6..10: conserved variables */
#define BF_FIELD_DTV 11      /* dt / V of the last step, interior only */
#define BF_FIELD_PSI 12      /* limiter arrays: 12 + 10*d + 5*minus + var */
#define BF_FIELD_VOL 50      /* cell volumes, interior only (Fortran dims) */
#define BF_FIELD_FACE 51     /* face geometry: 51 + 4*d + (nx, ny, nz, A), faces 0..N_d along d,
                                interior tangential (solver.py:212-220 _nhat / _area) */

/* arithmetic modes */
#define BF_PRECISION_EXACT 0 /* reference evaluation order, no FMA contraction: bitwise  */
#define BF_PRECISION_FAST 1  /* FMA + strength reduction: within 1e-12 of the reference  */

/* error kinds reported by bf_error_info (NonPhysicalStateError texts, solver.py:501-506,
   740-744; physics.py:213-217) */
#define BF_ERR_FACE_LEFT 1
#define BF_ERR_FACE_RIGHT 2
#define BF_ERR_ROE_A2 3
#define BF_ERR_UPDATE 4

typedef struct bf_ctx bf_ctx;
typedef struct bf_group bf_group;
typedef struct bf_loopback bf_loopback;

typedef struct bf_gas {            /* physics.py:47-90 */
  double gamma;
  double R;
  double mu;                       /* constant viscosity (sutherland unset)      */
  double prandtl;
  int has_sutherland;              /* 1: mu(T) = Sutherland's law               */
  double sutherland[3];            /* (mu_ref, T_ref, S)                        */
} bf_gas;

typedef struct bf_freestream {     /* solver.py:74-98 */
  double rho, u, v, w, p, T;
} bf_freestream;

typedef struct bf_scheme {         /* solver.py:38-66 */
  int flux;                        /* BF_FLUX_*                      */
  int limiter;                     /* BF_LIM_*                       */
  double epsilon;                  /* 0 or 1                         */
  double kappa;                    /* [-1, 1]                        */
  int rk_stages;                   /* 1, 2 or 4                      */
  double cfl;
  int limiter_freeze_at;           /* <= 0: never freeze             */
  double entropy_fix_coeff;
  int has_wall_temperature;
  double wall_temperature;
  int precision;                   /* BF_PRECISION_*                 */
  int viscous;                     /* laminar NS (solver.py:38-71)   */
} bf_scheme;

/* --- context lifetime (replaces BlockSolver construction, solver.py:189-231,
       and build_block_solvers, solver.py:858-866) -------------------------- */
bf_ctx* bf_create(int ndim, const bf_gas* gas, const bf_scheme* scheme,
                  const bf_freestream* fs, int device, int rank, int nranks);
void bf_destroy(bf_ctx* ctx);
int bf_last_error(const bf_ctx* ctx, char* buf, size_t n);
int bf_api_version(void);

/* Register one child block owned by this rank (BlockSolver.__init__).
   dims[3]        interior cells (nk = 1 in 2D);
   face_vectors   ndim*3 pointers: direction d, component c at [3*d + c], each a
                  Fortran array of shape (N_d+1, padded tangential...) — the
                  reference's metrics.face_vectors[d][c] (mesh.py:316-331);
   volume         interior cell volumes, Fortran (dims);
   source         5 pointers to S*V (solver.py:225-231) or NULL.            */
int bf_add_block(bf_ctx* ctx, int block_id, const int dims[3], int ghost_depth,
                 const double* const* face_vectors, const double* volume,
                 const double* const* source);

/* Same, from the block's padded node coordinates (Block.nodes, mesh.py:44-119):
   nodes[c], c < ndim, dense arrays of shape (P0+1, P1+1[, P2+1]) with
   P = dims + 2*ghost, element strides node_strides[0..ndim-1] along i, j, k
   (the reference's C-ordered Block.nodes[c] is passed as it is).  Face geometry and volumes are computed on the device
   with compute_metrics' operation order (mesh.py:250-331), bitwise equal to
   the host metrics; an inverted interior cell is reported by bf_sync_blocks
   (or bf_finalize) as BF_EMETRIC with the reference's MetricError text.
   Asynchronous: the node copy (pinned `nodes` move at full link speed) and
   the metric kernels of one block overlap the next call's allocation and
   copy; `nodes` must stay valid until bf_sync_blocks / bf_finalize returns.
   Moves ndim/9 of bf_add_block's geometry bytes (one node triple per cell
   instead of nine face-vector components). */
int bf_add_block_nodes(bf_ctx* ctx, int block_id, const int dims[3], int ghost_depth,
                       const double* const* nodes, const long long node_strides[3],
                       const double* const* source);

/* Wait for the bf_add_block_nodes registrations in flight; the first block
   (in registration order) with an inverted interior cell -> BF_EMETRIC
   "block <id>: inverted cell at interior index (i, j, k)" (mesh.py
   compute_metrics' MetricError).  Called by bf_finalize as well.         */
int bf_sync_blocks(bf_ctx* ctx);

/* One physical patch (solver.py:281-403, 526-580).  box[6] = (i0,i1,j0,j1,k0,k1)
   in the block's interior cell indices (BoundarySpec.box).  dirichlet: for
   BF_BC_MMS_DIRICHLET the cached ghost values, layout [layer][6 fields][t]
   with t running i-fastest over the patch's tangential cells; else NULL.   */
int bf_add_bc_patch(bf_ctx* ctx, int block_id, int bc_type, int face, const int box[6],
                    const double* dirichlet);

/* Same as bf_add_bc_patch plus, for laminar NS (ghost round 2,
   solver.py:285-305), the MMS ghost values of the EXTENDED patch: tangential
   ranges widened by the ghost depth, layout [layer][6 fields][t] i-fastest
   over the extended tangential cells (NULL for other bc types).           */
int bf_add_bc_patch_ext(bf_ctx* ctx, int block_id, int bc_type, int face, const int box[6],
                        const double* dirichlet, const double* dirichlet_ext);

/* One connected endpoint (topology.py:90-188; halo.py:47-115).  axis_map[6] =
   (b0,s0,b1,s1,b2,s2).  peer_rank == own rank and peer_block registered in this
   ctx -> same-device copy; otherwise a message to/from peer_rank tagged `tag`. */
int bf_add_link(bf_ctx* ctx, int block_id, int face, const int box[6], const int axis_map[6],
                int peer_block, int peer_face, const int peer_box[6], int peer_rank, int tag);

/* Laminar NS: the face gradient matrices of a block (solver.py:582-642, the
   inverse-transposed computational->physical Jacobian), computed on the host
   with the reference's numpy operations.  grad_invT[9*d + 3*r + e] for
   d < ndim: Fortran array over the faces of direction d (N_d+1 along d,
   interior tangential), row r, column e; NULL entries are zero.           */
int bf_add_viscous_geometry(bf_ctx* ctx, int block_id, const double* const* grad_invT);

/* Ghost round 2 (viscous) unpack order: order[q] = position of the q-th
   bf_add_link call in the reference's exchange sequence (serial driver:
   rank-major schedule order, solver.py:869-899; distributed engine: local
   entries, then remote, exchange.py:495-521).  Default: call order.      */
int bf_set_round2_order(bf_ctx* ctx, int nlinks, const int* order);

/* Freeze the topology: device tables, tiles, buffers.  Must precede uploads. */
int bf_finalize(bf_ctx* ctx);

/* Initial state (init_uniform / init_manufactured / sync_conserved,
   solver.py:258-277): 6 padded primitive fields + 5 padded conserved fields;
   q5 = NULL derives the conserved fields on the device (encode_primitive,
   reference operation order: bitwise equal to the host conversion).      */
int bf_upload_fields(bf_ctx* ctx, int block_id, const double* const* fields6,
                     const double* const* q5);

/* --- the hot path ------------------------------------------------------ */
/* RankStepper.update_ghosts (solver.py:777-784): round-1 exchange + physical BCs. */
int bf_update_ghosts(bf_ctx* ctx);
/* RankStepper.step (solver.py:786-814).  sumsq_out[5] = sum over this rank's
   blocks in id order of sum(R^2) from the first stage; when the ctx has an NCCL
   communicator the rank-ordered sum over all ranks (exchange.py:294-309). */
int bf_step(bf_ctx* ctx, int step_index, double* sumsq_out, long long* ncells_out);
/* nsteps consecutive steps driven from C (no return to the caller between
   steps); per-step norms land in hist_out[nsteps*5] (sqrt of the rank-ordered
   sums).  Returns at the first step with a non-physical state (bf_error_info
   names it). */
int bf_run(bf_ctx* ctx, int first_step, int nsteps, double* hist_out, int* steps_done);
/* solver.iterate's loop (solver.py:914-936) driven from C: up to max_steps
   steps, after each one the history guards of solver.py:836-855 (residual floor,
   divergence factor, residual target; has_* = 0 disables a criterion).  status:
   0 ran max_steps, 1 converged at the last step, 2 diverged at the last step
   (the caller raises DivergenceError exactly as the guard does). */
int bf_iterate(bf_ctx* ctx, int first_step, int max_steps, int has_target, double target,
               int has_floor, double floor_, double divergence_factor, double* hist_out,
               int* steps_done, int* status);

/* --- state access --------------------------------------------------------- */
/* Padded Fortran array of the block's field `what` (BF_FIELD_*) exactly as the
   reference's BlockSolver would hold it after the same calls. */
int bf_download(bf_ctx* ctx, int block_id, int what, double* out);
/* Details of the last BF_ENONPHYSICAL: kind (BF_ERR_*), block id, stage,
   direction, index[3] (face or cell index in the reference's array numbering). */
int bf_error_info(const bf_ctx* ctx, int* kind, int* block_id, int* stage, int* direction,
                  long long index[3]);

/* --- multi-rank ------------------------------------------------------------ */
/* NCCL: one process per GPU.  bf_nccl_unique_id fills 128 bytes on rank 0, the
   caller broadcasts them (torch.distributed), then every rank calls
   bf_nccl_init before bf_finalize. */
int bf_nccl_unique_id(void* out128);
int bf_nccl_init(bf_ctx* ctx, const void* id128);
/* Loopback transport: the NCCL calls of the path (grouped ncclSend/ncclRecv of
   the halo messages, ncclAllGather of the residual record) served inside ONE
   process whose ranks are host threads, one bf_ctx each, on any GPUs (several
   may share one).  Same matching, ordering and completion semantics as NCCL:
   the runtime's exchange / interior-boundary overlap / rank-ordered residual
   code runs unchanged with it bound in place of libnccl (exchange.py:599-682
   runs its ranks as threads the same way).  bf_loopback_init replaces
   bf_nccl_init (before bf_finalize); the world must outlive its contexts.  A
   rank that stops calling makes its peers fail with BF_ENCCL after
   BF_LOOPBACK_TIMEOUT seconds (default 120) or at bf_loopback_abort. */
bf_loopback* bf_loopback_create(int nranks);
int bf_loopback_init(bf_ctx* ctx, bf_loopback* world);
void bf_loopback_abort(bf_loopback* world);
void bf_loopback_destroy(bf_loopback* world);
/* In-process group: several ctxs (ranks) driven in lock step by one host
   thread; remote links become device-to-device pushes into the peer's
   receive buffers (peer access over NVLink when the ctxs sit on different
   GPUs).  Used for N ranks on fewer GPUs and for single-process multi-GPU. */
bf_group* bf_group_create(bf_ctx* const* ctxs, int n);
void bf_group_destroy(bf_group* grp);
int bf_group_update_ghosts(bf_group* grp);
int bf_group_step(bf_group* grp, int step_index, double* sumsq_out, int* failed_rank);

/* --- measurement ---------------------------------------------------------- */
/* Launch on a caller-provided cudaStream_t (e.g. torch's current stream) so the
   caller's CUDA events bracket the work; NULL restores the ctx's own stream. */
int bf_set_stream(bf_ctx* ctx, void* cuda_stream);
/* Per-kernel-class CUDA-event timing: enable, then read {launches, total_ms}
   for class 0 = stage kernel (an interior/boundary split stage counts once, its span
   from the first launch to the join of both), 1 = ghost/pack kernel, 2 = unpack (and the
   viscous face-flux kernel), 3 = reduce; class 4 = every kernel launch inside those
   scopes (launches) and the sum of the four classes (total_ms). */
int bf_set_profiling(bf_ctx* ctx, int on);
int bf_kernel_stats(bf_ctx* ctx, int kernel_class, long long* launches, double* total_ms);
/* Transfer counters of the exchange engine, cumulative over the context's life
   (replaces exchange.py:83-101 TransferCounters, which RankRuntime increments as
   it moves messages, exchange.py:371-466): out = {messages, runs, bytes,
   staging_copies, waits, max_pending}.  One message per remote endpoint and
   round (all fields concatenated), runs = halo pack + unpack launches, one wait
   per grouped exchange, staging copies 0 (device buffers are sent directly). */
int bf_transfer_counters(const bf_ctx* ctx, long long out[6]);
/* Device bytes the last bf_upload_fields / bf_download moved (for e2e accounting). */
long long bf_transfer_bytes(const bf_ctx* ctx, int direction /*0 h2d, 1 d2h*/);

/* Block arenas of destroyed contexts (and the staging buffers' stream-ordered
   pool) are kept for reuse by the next context on the same device while another
   context of that device is alive (bounded; a failing arena allocation releases
   them first).  When the last context of a device is destroyed they go back to
   the driver and the default pool's release threshold is restored, unless
   BF_ARENA_CACHE=1 keeps them.  bf_release_cache hands them back explicitly:
   device >= 0 one device, < 0 all.  bf_cache_bytes: arena bytes held. */
void bf_release_cache(int device);
long long bf_cache_bytes(int device);

/* Host-only probe (no GPU needed): the order in which a rank issues its remote
   endpoints' messages inside one NCCL group (remote_links_sorted: by peer rank,
   then link tag, then own block id).  order_out[q] = index into the inputs of
   the q-th message.  Used by the CPU tests against distributed.remote_links. */
int bf_probe_remote_order(int n, const int* peer_rank, const int* tag, const int* block,
                          int* order_out);

/* Host-only lowering probe (no GPU needed): the affine index map the device
   unpack applies for one connected endpoint — for each recv-box cell (i-fastest,
   count = product of recv extents), the partner-send-box linear index it reads.
   Used by the CPU tests to prove bit-exact ghost indexing against halo.py. */
int bf_probe_unpack_map(const int own_dims[3], int ghost_depth, int ndim, int face,
                        const int box[6], const int axis_map[6], int peer_face,
                        long long* out, long long out_len);

#ifdef __cplusplus
}
#endif
#endif /* BFGPU_H */
