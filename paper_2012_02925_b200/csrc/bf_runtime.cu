// bf_runtime.cu — host runtime behind include/bfgpu.h.
//
// Owns device memory, lowers the reference's boundary model (BoundarySpec
// boxes, orientation maps, halo_regions) into device task tables, sequences
// the per-stage launches (RankStepper.step, solver.py:786-814) on one CUDA
// stream and moves halo messages with NCCL (one process per GPU) or with
// device-to-device copies between contexts of one process (bf_group).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <cstdlib>
#include <array>
#include <set>
#include <string>
#include <vector>

#include "../../include/bfgpu.h"
#include "bf_internal.h"
#include "bf_loopback.h"

namespace bf {
namespace bf_exact {
cudaError_t launch_stage(int ndim, int flux, int lim, const StageArgs& a, cudaStream_t s);
cudaError_t launch_viscous(const ViscArgs& a, int nlaunch, cudaStream_t s);
cudaError_t launch_ghost(const GhostArgs& a, cudaStream_t s);
cudaError_t launch_reduce(const double* partial, const int* tile_begin, int nblocks, double* out,
                          cudaStream_t s);
cudaError_t launch_guard(const double* partial, const int* tile_begin, int nb, double* blocksum,
                         unsigned long long* err, RunState* rs, double* hist, unsigned* count,
                         cudaStream_t s);
cudaError_t launch_rank_record(const double* blocksum, int nb, const unsigned long long* err,
                               double* rec6, const RunState* rs, cudaStream_t s);
cudaError_t launch_rank_guard(const double* gather, int nranks, int rank,
                              unsigned long long* err, RunState* rs, double* hist,
                              cudaStream_t s);
int stage_tile_rows(int ndim, int lim);
void set_pdl(int on);
}  // namespace bf_exact
namespace bf_fast {
cudaError_t launch_stage(int ndim, int flux, int lim, const StageArgs& a, cudaStream_t s);
cudaError_t launch_viscous(const ViscArgs& a, int nlaunch, cudaStream_t s);
bool vl_active(int flux, int flags);
bool vl_push_compiled();
cudaError_t launch_ghost(const GhostArgs& a, cudaStream_t s);
cudaError_t launch_reduce(const double* partial, const int* tile_begin, int nblocks, double* out,
                          cudaStream_t s);
void set_pdl(int on);
}  // namespace bf_fast
}  // namespace bf

using namespace bf;

namespace {

// NCCL is bound lazily with dlopen: the library has no load-time dependency on
// libnccl, so whichever NCCL the process already holds (e.g. torch's bundled
// one) is reused and importing libbfgpu first cannot shadow it.
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi load_nccl() {
  NcclApi a;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    a.err = dlerror() ? dlerror() : "libnccl.so.2 not found";
    return a;
  }
  auto sym = [&](const char* n) { return dlsym(h, n); };
  a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
  a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
  a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
  a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
  a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
  a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
  a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
  a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
  a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
  a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Send && a.Recv && a.GroupStart &&
         a.GroupEnd && a.AllGather && a.GetErrorString;
  if (!a.ok) a.err = "libnccl is missing required symbols";
  return a;
}

NcclApi& nccl() {
  static NcclApi api = load_nccl();
  return api;
}

// The same entry points bound to the in-process transport (bf_loopback.h).
const NcclApi& loopback_api() {
  static const NcclApi api = [] {
    NcclApi a;
    a.ok = true;
    a.Send = bf_lb::Send;
    a.Recv = bf_lb::Recv;
    a.GroupStart = bf_lb::GroupStart;
    a.GroupEnd = bf_lb::GroupEnd;
    a.AllGather = bf_lb::AllGather;
    a.GetErrorString = bf_lb::GetErrorString;
    return a;
  }();
  return api;
}

// ---- device-side set-up kernels (replace host restriding loops) -----------------
// Dense Fortran box (e0, e1, e2) -> arena slot at (o0, o1, o2) in padded-array
// coordinates relative to the slot start.
__global__ void scatter_box_kernel(double* dst, long long sy, long long sz, long long o0,
                                   long long o1, long long o2, const double* src, int e0,
                                   int e1, int e2) {
  const long long n = (long long)e0 * e1 * e2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t % e0, r = t / e0;
    const long long j = r % e1, k = r / e1;
    dst[(o0 + i) + sy * (o1 + j) + sz * (o2 + k)] = src[t];
  }
}

// Arena slot -> dense Fortran box (inverse of scatter_box_kernel).
__global__ void gather_box_kernel(double* dst, const double* src, long long sy, long long sz,
                                  long long o0, long long o1, long long o2, int e0, int e1,
                                  int e2) {
  const long long n = (long long)e0 * e1 * e2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t % e0, r = t / e0;
    const long long j = r % e1, k = r / e1;
    dst[t] = src[(o0 + i) + sy * (o1 + j) + sz * (o2 + k)];
  }
}

// Unit normals and areas of one direction's faces (solver.py:212-220) with the
// reference's IEEE operation order (explicit _rn intrinsics: no contraction).
// sv: 3 component arrays of shape in (N_d+1 along d, padded tangential), Fortran.
// Writes the interior-tangential faces f = 0..N_d into 4 slots (nx, ny, nz, A),
// face f stored at interior cell index f.
__global__ void face_normals_kernel(double* nx_slot, long long fsz, long long sy, long long sz,
                                    long long origin, const double* sv, long long ncomp_stride,
                                    int d, int e0, int e1, int e2, int in0, int in1, int g0,
                                    int g1, int g2) {
  const long long n = (long long)e0 * e1 * e2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    // e0..e2 span the padded tangential range: input index = padded index,
    // output cell = padded index - ghost (negative = tangential ghost column)
    const int ii = (int)(t % e0);
    const long long r = t / e0;
    const int jj = (int)(r % e1), kk = (int)(r / e1);
    const long long s = ii + (long long)in0 * (jj + (long long)in1 * kk);
    const int i = (d == 0) ? ii : ii - g0;
    const int j = (d == 1) ? jj : jj - g1;
    const int k = (d == 2) ? kk : kk - g2;
    const double x = sv[s], y = sv[ncomp_stride + s], z = sv[2 * ncomp_stride + s];
    const double A =
        __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
    const long long o = origin + i + sy * j + sz * k;
    nx_slot[o] = A > 0.0 ? __ddiv_rn(x, A) : 0.0;
    nx_slot[fsz + o] = A > 0.0 ? __ddiv_rn(y, A) : 0.0;
    nx_slot[2 * fsz + o] = A > 0.0 ? __ddiv_rn(z, A) : 0.0;
    nx_slot[3 * fsz + o] = A;
  }
}

// ---- device metrics (geometry.py / mesh.py:250-331), reference operation order ----------
// Nodes: 3 padded component arrays (Fortran, (P0+1) x (P1+1) [x (P2+1)]).  Explicit
// _rn intrinsics keep numpy's rounding (no contraction), so the face geometry and the
// volumes are bitwise those of compute_metrics on the host.
struct V3 {
  double x, y, z;
};
__device__ __forceinline__ V3 v_sub(V3 a, V3 b) {
  return {__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z)};
}
__device__ __forceinline__ V3 v_cross(V3 a, V3 b) {   // numpy.cross component order
  return {__dsub_rn(__dmul_rn(a.y, b.z), __dmul_rn(a.z, b.y)),
          __dsub_rn(__dmul_rn(a.z, b.x), __dmul_rn(a.x, b.z)),
          __dsub_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x))};
}
__device__ __forceinline__ V3 v_scale(double s, V3 a) {
  return {__dmul_rn(s, a.x), __dmul_rn(s, a.y), __dmul_rn(s, a.z)};
}
__device__ __forceinline__ double v_sum3_mul(V3 g, V3 t) {   // (g0 t0 + g1 t1) + g2 t2
  return __dadd_rn(__dadd_rn(__dmul_rn(g.x, t.x), __dmul_rn(g.y, t.y)), __dmul_rn(g.z, t.z));
}
struct NodeView {
  const double* x;
  const double* y;
  const double* z;      // null in 2D
  long long s0, s1, s2;  // element strides along i, j, k
  __device__ V3 at(long long a, long long b, long long c) const {
    const long long o = s0 * a + s1 * b + s2 * c;
    return {x[o], y[o], z ? z[o] : 0.0};
  }
};
// Corner orderings per face direction, normals toward +axis (mesh.py:294-298)
__constant__ int kFaceCorners[3][4][3] = {
    {{0, 0, 0}, {0, 1, 0}, {0, 1, 1}, {0, 0, 1}},
    {{0, 0, 0}, {0, 0, 1}, {1, 0, 1}, {1, 0, 0}},
    {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0}}};

// Faces f = 0..N_d of direction d over the interior tangential range: face vector,
// then unit normal and area (solver.py:212-220) into the 4 geometry slots.
// Tangential coverage is the padded range (ghost columns included): the
// boundary-face normals there serve the extended (round-2) wall / farfield
// ghosts of laminar NS runs (solver.py:310-319 reads padded _nhat).
__global__ void metrics_faces_kernel(double* nx_slot, long long fsz, long long sy, long long sz,
                                     long long origin, NodeView nv, int ndim, int d, int e0,
                                     int e1, int e2, int g, int gk, int l0, int l1, int l2) {
  const long long n = (long long)e0 * e1 * e2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % e0) + l0;
    const long long r = t / e0;
    const int j = (int)(r % e1) + l1, k = (int)(r / e1) + l2;
    const int ni = i + g, nj = j + g, nk = k + gk;   // node of the face's (0,0,0) corner
    V3 s;
    if (ndim == 3) {
      V3 c[4];
      for (int q = 0; q < 4; ++q)
        c[q] = nv.at(ni + kFaceCorners[d][q][0], nj + kFaceCorners[d][q][1],
                     nk + kFaceCorners[d][q][2]);
      s = v_scale(0.5, v_cross(v_sub(c[2], c[0]), v_sub(c[3], c[1])));
    } else if (d == 0) {   // fv_i = (dy, -dx, 0) along the j edge
      const V3 a = nv.at(ni, nj, 0), b = nv.at(ni, nj + 1, 0);
      s = {__dsub_rn(b.y, a.y), -__dsub_rn(b.x, a.x), 0.0};
    } else {               // fv_j = (-dy, dx, 0) along the i edge
      const V3 a = nv.at(ni, nj, 0), b = nv.at(ni + 1, nj, 0);
      s = {-__dsub_rn(b.y, a.y), __dsub_rn(b.x, a.x), 0.0};
    }
    const double A =
        __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(s.x, s.x), __dmul_rn(s.y, s.y)), __dmul_rn(s.z, s.z)));
    const long long o = origin + i + sy * j + sz * k;
    nx_slot[o] = A > 0.0 ? __ddiv_rn(s.x, A) : 0.0;
    nx_slot[fsz + o] = A > 0.0 ? __ddiv_rn(s.y, A) : 0.0;
    nx_slot[2 * fsz + o] = A > 0.0 ? __ddiv_rn(s.z, A) : 0.0;
    nx_slot[3 * fsz + o] = A;
  }
}

// mesh.py:287-331: (sum3(g1 t1) + sum3(g2 t2)) / 3 over the two triangles of a quad
__device__ double tri_flux(V3 c0, V3 c1, V3 c2, V3 c3) {
  const double third = 3.0;
  const V3 t1 = v_scale(0.5, v_cross(v_sub(c1, c0), v_sub(c2, c0)));
  const V3 t2 = v_scale(0.5, v_cross(v_sub(c2, c0), v_sub(c3, c0)));
  const V3 g1 = {__ddiv_rn(__dadd_rn(__dadd_rn(c0.x, c1.x), c2.x), third),
                 __ddiv_rn(__dadd_rn(__dadd_rn(c0.y, c1.y), c2.y), third),
                 __ddiv_rn(__dadd_rn(__dadd_rn(c0.z, c1.z), c2.z), third)};
  const V3 g2 = {__ddiv_rn(__dadd_rn(__dadd_rn(c0.x, c2.x), c3.x), third),
                 __ddiv_rn(__dadd_rn(__dadd_rn(c0.y, c2.y), c3.y), third),
                 __ddiv_rn(__dadd_rn(__dadd_rn(c0.z, c2.z), c3.z), third)};
  return __ddiv_rn(__dadd_rn(v_sum3_mul(g1, t1), v_sum3_mul(g2, t2)), third);
}

// Interior cell volumes into the V slot; the first inverted cell (C order over the
// interior, np.argwhere) goes to *bad as (i*nj + j)*nk + k.
__global__ void metrics_volume_kernel(double* vol, long long sy, long long sz, NodeView nv, int ndim,
                                      int e0, int e1, int e2, int g, int gk,
                                      unsigned long long* bad) {
  const long long n = (long long)e0 * e1 * e2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % e0);
    const long long r = t / e0;
    const int j = (int)(r % e1), k = (int)(r / e1);
    const int a = i + g, b = j + g, c = k + gk;
    double v;
    if (ndim == 3) {
      v = 0.0;
      for (int d = 0; d < 3; ++d) {
        V3 lo[4], hi[4];
        for (int q = 0; q < 4; ++q) {
          const int* o = kFaceCorners[d][q];
          lo[q] = nv.at(a + o[0], b + o[1], c + o[2]);
          hi[q] = nv.at(a + o[0] + (d == 0), b + o[1] + (d == 1), c + o[2] + (d == 2));
        }
        const double part = __dsub_rn(tri_flux(hi[0], hi[1], hi[2], hi[3]),
                                      tri_flux(lo[0], lo[1], lo[2], lo[3]));
        v = d == 0 ? part : __dadd_rn(v, part);
      }
    } else {   // shoelace, mesh.py:250-284
      const V3 pa = nv.at(a, b, 0), pb = nv.at(a + 1, b, 0), pc = nv.at(a + 1, b + 1, 0),
               pd = nv.at(a, b + 1, 0);
      const double t1 = __dsub_rn(__dmul_rn(pa.x, pb.y), __dmul_rn(pb.x, pa.y));
      const double t2 = __dsub_rn(__dmul_rn(pb.x, pc.y), __dmul_rn(pc.x, pb.y));
      const double t3 = __dsub_rn(__dmul_rn(pc.x, pd.y), __dmul_rn(pd.x, pc.y));
      const double t4 = __dsub_rn(__dmul_rn(pd.x, pa.y), __dmul_rn(pa.x, pd.y));
      v = __dmul_rn(0.5, __dadd_rn(__dadd_rn(__dadd_rn(t1, t2), t3), t4));
    }
    vol[i + sy * j + sz * k] = v;
    if (v <= 0.0) atomicMin(bad, ((unsigned long long)i * e1 + j) * (unsigned long long)e2 + k);
  }
}

// encode_primitive (physics.py:136-140) over a whole padded arena slot range,
// reference operation order: rho u, rho v, rho w, p/(g-1) + rho*(0.5*((uu+vv)+ww)).
__global__ void encode_kernel(double* W, double* Q, long long fsz, long long n, double gm1) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const double r = W[t], u = W[fsz + t], v = W[2 * fsz + t], w = W[3 * fsz + t],
                 p = W[4 * fsz + t];
    const double ke =
        __dmul_rn(0.5, __dadd_rn(__dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v)), __dmul_rn(w, w)));
    Q[t] = r;
    Q[fsz + t] = __dmul_rn(r, u);
    Q[2 * fsz + t] = __dmul_rn(r, v);
    Q[3 * fsz + t] = __dmul_rn(r, w);
    Q[4 * fsz + t] = __dadd_rn(__ddiv_rn(p, gm1), __dmul_rn(r, ke));
  }
}

// Laminar NS keeps the reference's single-array ghost semantics: round 2 and
// the extended BCs read edge / corner ghost cells, which in the reference still
// hold the PREVIOUS ghost update's values, while the ping-pong buffer being
// filled holds those of two updates ago.  Copy every ghost cell (6 fields)
// from the other buffer before a viscous ghost update.
__global__ void ghost_sync_kernel(double* dst, const double* src, long long fsz, long long lead,
                                  long long sy, long long sz, int P0, int P1, int P2, int g0,
                                  int g1, int g2, int n0, int n1, int n2) {
  const long long n = (long long)P0 * P1 * P2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % P0);
    const long long r = t / P0;
    const int j = (int)(r % P1), k = (int)(r / P1);
    const bool inner = i >= g0 && i < g0 + n0 && j >= g1 && j < g1 + n1 && k >= g2 && k < g2 + n2;
    if (inner) continue;
    const long long o = lead + i + sy * j + sz * k;
    for (int f = 0; f < 6; ++f) dst[f * fsz + o] = src[f * fsz + o];
  }
}

int grid_for(long long n) { return (int)std::min<long long>((n + 255) / 256, 148 * 16); }

// One padded field as the reference holds it: interior from the current W
// buffer (T derived as p/(rho R) once the state has been updated,
// solver.py:753), ghost cells from the buffer the last ghost update filled.
__global__ void merge_field_kernel(double* out, const double* cur, const double* ghost,
                                   const double* rho, const double* p, int derived, double R,
                                   long long sy, long long sz, long long lead, int g0, int g1,
                                   int g2, int n0, int n1, int n2, int P0, int P1, int P2) {
  const long long n = (long long)P0 * P1 * P2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % P0);
    const long long r = t / P0;
    const int j = (int)(r % P1), k = (int)(r / P1);
    const long long s = lead + i + sy * j + sz * k;
    const bool inner = i >= g0 && i < g0 + n0 && j >= g1 && j < g1 + n1 && k >= g2 && k < g2 + n2;
    out[t] = inner ? (derived ? __ddiv_rn(p[s], __dmul_rn(rho[s], R)) : cur[s]) : ghost[s];
  }
}

constexpr unsigned long long NO_ERROR = ~0ull;

struct HostPatch {
  int block, type, face;
  int box[6];
  std::vector<double> dirichlet;
  std::vector<double> dirichlet_ext;   // round-2 (extended) MMS ghost values
};

struct HostLink {
  int block, face;
  int box[6];
  int amap[6];
  int peer_block, peer_face;
  int peer_box[6];
  int peer_rank, tag;
  // remote only, filled at finalize
  long long cells = 0;
  int order2 = -1;           // position in the round-2 unpack sequence
  long long cells2 = 0;      // round-2 (extended) box cells
  double* send2 = nullptr;   // round-2 message buffers (remote) / snapshot buffer (local)
  double* recv2 = nullptr;
  int nfields = 0;
  double* send = nullptr;
  double* recv = nullptr;
};

struct HostBlock {
  int id = 0;
  int n[3] = {0, 0, 0};
  int g = 2, gk = 2;
  int P[3] = {0, 0, 0};      // padded dims
  long long lead = 0, sy = 0, sz = 0, origin = 0, fsz = 0;
  int nslots = 0;
  double* arena = nullptr;
  std::vector<double*> owned;  // allocations to free (the arena, back to the arena cache)
  size_t arena_bytes = 0;
  DevBlock dev{};
  std::vector<unsigned char> bface_h[6];
  unsigned char* bface_d[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  bool has_src = false;
  unsigned long long* d_bad = nullptr;   // bf_add_block_nodes: inverted-cell flag in flight
  int tile_begin = 0, tile_end = 0;
  long long cells() const { return (long long)n[0] * n[1] * n[2]; }
  long long off(int i, int j, int k) const { return i + sy * (long long)j + sz * (long long)k; }
};

struct TimerPair {
  cudaEvent_t a, b;
  int cls;
  int kernels = 1;               // kernel launches inside the timed scope
  bool owned_by_graph = false;   // recorded by a captured step: not returned to the pool
};

}  // namespace

struct bf_ctx {
  int ndim = 3;
  bf_gas gas{};
  bf_scheme sch{};
  bf_freestream fs{};
  Consts c{};
  int device = 0, rank = 0, nranks = 1;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  // halo exchange overlapped with interior tiles (bf_step): messages + unpack on
  // comm_stream while the stage kernel runs the tiles that read no remote ghost
  cudaStream_t comm_stream = nullptr;
  cudaStream_t copy_stream = nullptr;   // bf_add_block_nodes: node copies
  std::vector<std::pair<double*, size_t>> staging;   // node buffers in flight (bf_sync_blocks)
  cudaEvent_t ev_filled = nullptr, ev_unpacked = nullptr;
  cudaEvent_t ev_bd = nullptr;     // boundary tiles of the stage done (comm_stream)
  int* d_tiles_in = nullptr;       // tile ids reading no remote-received ghost cell
  int* d_tiles_bd = nullptr;       // the others (launched after the unpack)
  int n_tiles_in = 0, n_tiles_bd = 0;
  bool split_tiles = false;        // interior / boundary tile lists built
  bool split_forced = false;       // BF_SPLIT_TILES=1
  bool exchange_pending = false;   // messages + unpack queued on comm_stream this stage
  bool hide_fill = false;          // one-rank ctx: ghost fill on comm_stream beside the
                                   // interior tiles (BF_HIDE_GHOSTS=1; measured slower)
  bool fill_pending = false;       // this stage's ghost fill is queued on comm_stream
  bool no_overlap = false;         // BF_NO_OVERLAP=1: exchange in line (A/B timing)
  // fused ghost fill (StageArgs::fill_ctas): the cell-split kernel's launch fills
  // the ghosts itself; tiles ordered interior-first (reading no ghost cell)
  int* d_tiles_fused = nullptr;
  int n_fused_in = 0;
  int fused_mode = -1;             // BF_FUSED_FILL: 0 off, 1 on, unset: fused_fill_pays

  int fill_ctas_env = 0;           // BF_FILL_CTAS=n: fill-only CTAs per fused launch
  int num_sms = 148;
  int pdl_mode = -1;               // BF_PDL: 0 off, 1 on, unset: one-wave grids (use_pdl)
  bool ghost_interleave = true;    // BF_GHOST_INTERLEAVE=0: ghost blocks in task order
  unsigned* d_fill_sync = nullptr; // [1] fill warps done, [2] arrivals; [3] guard-kernel CTA counter
  bool fuse_next = false;          // the next stage launch fills the ghosts of W[cur]
  bool counted = false;           // registered in the per-device live-context count
  // one RK step as a CUDA graph (standalone Euler ctx), per starting buffer and
  // profiling mode; a profiled graph records its own timing events
  cudaGraphExec_t gexec[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  std::vector<TimerPair> gprof[2];
  // batched iterate (bf_iterate): steps whose norms and guards stay on the device;
  // their graphs end with the guard kernel instead of the per-step D2H
  cudaGraphExec_t gexec_b[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  std::vector<TimerPair> gprof_b[2];
  bool batching = false;
  // multi-rank batched iterate (NCCL / loopback ranks): per step the rank record,
  // its allgather and the guards stay on the device (rank_record / rank_guard)
  bool mr_batching = false;
  bool batch_off = false;          // BF_BATCH=0
  RunState* d_run = nullptr;
  double* d_hist = nullptr;        // [BATCH_MAX][5]
  void* h_run = nullptr;           // pinned: RunState + hist
  bool capturing = false;
  bool graph_off = false;          // BF_GRAPH=0, or a capture that did not reproduce
  long long cur_epoch = 0;         // bumped by every stage launch (buffer swap)
  long long synced_cur = -1;       // epoch whose ghosts were synced from the other buffer
  std::vector<HostBlock> blocks;
  std::map<int, int> index_of;     // block id -> position
  std::vector<HostPatch> patches;
  std::vector<HostLink> links;
  bool finalized = false;
  // device tables
  DevBlock* d_blocks = nullptr;
  unsigned char* d_tmaps = nullptr;   // [nblocks][NTMAP] CUtensorMap
  Tile* d_tiles = nullptr;
  int ntiles = 0;
  int* d_tile_begin = nullptr;
  GhostTask* d_tasks_fill = nullptr;   // BCs + local copies + packs
  int n_fill = 0;
  long long items_fill = 0;
  GhostTask* d_tasks_unpack = nullptr;
  std::vector<PushRule> h_push;
  PushRule* d_push = nullptr;      // ghost push rules (stage kernel writes next ghosts)
  int* d_push_range = nullptr;     // [nblocks][6][2]
  bool push_ok = false;            // push rules built (all blocks >= 2 ghost depths thick)
  bool pushed = false;             // ghosts of W[cur] were written by the last stage
  bool other_filled = false;       // constant ghosts (inflow, MMS) present in W[cur ^ 1]
  int2* d_map_fill = nullptr;      // ghost launch block -> (task, first item)
  int2* d_map_unpack = nullptr;
  int nmap_fill = 0, nmap_unpack = 0;
  int ipt_fill = 1, ipt_unpack = 1;   // ghost items per thread of those launches
  int n_unpack = 0;
  long long items_unpack = 0;
  std::vector<GhostTask> h_tasks_fill, h_tasks_unpack;
  // laminar NS ghost round 2 (solver.py:777-784): pack (one launch) -> messages ->
  // unpacks one launch per link in reference order -> extended BCs one launch per
  // per-block patch position
  struct GhostLaunch {
    GhostTask* d = nullptr;
    int2* map = nullptr;
    int ntasks = 0, nmap = 0;
    long long items = 0;
    int ipt = 1;
  };
  GhostLaunch r2_pack;
  std::vector<GhostLaunch> r1_bc;   // thin blocks: round-1 BCs in canonical order
  std::vector<GhostLaunch> r2_unpack, r2_bc;
  std::set<int> visc_geometry;      // blocks given their face gradient matrices
  ViscTask* d_visc = nullptr;        // viscous face-flux launch
  int2* d_visc_map = nullptr;
  int n_visc_map = 0;
  std::vector<double*> dirichlet_d;
  double* d_partial = nullptr;
  double* d_blocksum = nullptr;
  unsigned long long* d_err = nullptr;
  double* d_rank6 = nullptr;          // [6] own rank record (NCCL)
  double* d_gather = nullptr;         // [nranks][6]
  double* h_pinned = nullptr;         // blocksum + err staging
  // RunState::stop is its first member
  const int* stop_flag() const {
    return (batching || mr_batching) ? reinterpret_cast<const int*>(d_run) : nullptr;
  }
  // state
  int cur = 0;
  int ghost_buf = 0;
  int t_derived = 0;
  bool psi_valid = false;
  bool have_psi = false;
  int kc = 16;   // k-chunk per tile (32 for the FAST Van Leer kernel: profiles/r01_kc_*.json)
  // errors
  std::string msg;
  int e_kind = 0, e_block = -1, e_stage = 0, e_dir = 0;
  long long e_idx[3] = {0, 0, 0};
  // comm
  ncclComm_t comm = nullptr;
  const NcclApi* net = nullptr;    // transport bound to comm: libnccl or the loopback
  bf_lb::Rank* lb_rank = nullptr;  // loopback: what comm points to (owned)
  bf_group* group = nullptr;
  // profiling
  bool profiling = false;
  std::vector<TimerPair> pending;
  std::vector<cudaEvent_t> event_pool;
  long long prof_launches[4] = {0, 0, 0, 0};
  long long prof_kernels = 0;      // kernel launches in all timed scopes
  double prof_ms[4] = {0, 0, 0, 0};
  long long bytes_h2d = 0, bytes_d2h = 0;
  // transfer counters of the engine as it runs (exchange.py:83-101 fields):
  // messages / bytes = remote sends (one concatenated message per endpoint and
  // round), runs = halo pack + unpack kernel launches, waits = completions the
  // unpack waits on (one per grouped exchange), max_pending = messages in flight
  long long xc[6] = {0, 0, 0, 0, 0, 0};
};

struct bf_group {
  std::vector<bf_ctx*> ctxs;            // index = rank
  std::vector<cudaEvent_t> ev_packed;   // per ctx
  std::vector<cudaEvent_t> ev_unpacked; // per ctx
  bool first = true;
};

namespace {

const NcclApi& net(const bf_ctx* ctx) { return ctx && ctx->net ? *ctx->net : nccl(); }

int fail(bf_ctx* ctx, int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx) ctx->msg = buf;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(ctx, BF_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                    \
  } while (0)

#define NK(call)                                                                              \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess)                                                                    \
      return fail(ctx, BF_ENCCL, "%s failed: %s (%s:%d)", #call, net(ctx).GetErrorString(r_), \
                  __FILE__, __LINE__);                                                        \
  } while (0)

int face_axis(int face) { return face / 2; }
int face_side(int face) { return face % 2; }

// topology.py:224-257 in INTERIOR coordinates: [lo, hi) per axis.
void halo_boxes(int face, const int box[6], const int n[3], const int ghost[3], int send[6],
                int recv[6], int round_no = 1) {
  const int ax = face_axis(face);
  const int g = ghost[ax];
  for (int a = 0; a < 3; ++a) {
    if (a == ax) {
      if (face_side(face) == 0) {
        send[2 * a] = 0;
        send[2 * a + 1] = g;
        recv[2 * a] = -g;
        recv[2 * a + 1] = 0;
      } else {
        send[2 * a] = n[a] - g;
        send[2 * a + 1] = n[a];
        recv[2 * a] = n[a];
        recv[2 * a + 1] = n[a] + g;
      }
    } else {   // round 2 widens the tangential ranges by the ghost depth (topology.py:235-257)
      const int ext = round_no == 2 ? ghost[a] : 0;
      send[2 * a] = recv[2 * a] = box[2 * a] - ext;
      send[2 * a + 1] = recv[2 * a + 1] = box[2 * a + 1] + ext;
    }
  }
}

// Whether numpy's ravel(order="F") of this box of a padded Fortran array is a
// view (the box is F-contiguous, size-1 axes ignored): halo.py:58 then packs
// rho, p and T by reference, so a round-2 unpack reads them at unpack time.
bool box_is_view(const int box[6], const int P[3]) {
  long long expect = 1, stride = 1;
  for (int a = 0; a < 3; ++a) {
    const int e = box[2 * a + 1] - box[2 * a];
    if (e > 1 && stride != expect) return false;
    if (e > 1) expect *= e;
    stride *= P[a];
  }
  return true;
}

// Affine map of one endpoint's unpack (halo.py:70-106): for own recv-box
// local coords o, the partner-local send-box coords are q[perm[a]] =
// flip_a ? ext_a-1-o_a : o_a.  Returns per own axis the partner axis and flip.
void unpack_axes(int face, const int amap[6], int peer_face, int perm[3], bool flip[3]) {
  const int ax = face_axis(face);
  for (int a = 0; a < 3; ++a) {
    perm[a] = amap[2 * a];
    flip[a] = (a == ax) ? (face_side(face) == face_side(peer_face)) : (amap[2 * a + 1] < 0);
  }
}

// Process-wide cache of block arenas: bf_destroy returns a context's arenas
// here and the next context on the same device reuses them (best fit within
// 25%) instead of paying the driver's page mapping of multi-GB allocations
// again.  Bounded; bf_release_cache hands everything back to the driver, and a
// failing cudaMalloc releases the cache and retries.
struct ArenaCache {
  struct Entry {
    int dev;
    size_t bytes;
    void* p;
  };
  std::mutex m;
  std::vector<Entry> free;
  size_t held = 0;
  std::map<int, int> live;                  // contexts alive per device
  std::map<int, cuuint64_t> pool_thr;       // default pool release threshold before bf_create
};
ArenaCache& arena_cache() {
  static ArenaCache c;
  return c;
}
constexpr size_t ARENA_CACHE_MAX = 32ull << 30;

void release_arena_cache(int dev) {   // dev < 0: all devices
  ArenaCache& c = arena_cache();
  std::lock_guard<std::mutex> g(c.m);
  int cur = -1;
  cudaGetDevice(&cur);
  std::vector<ArenaCache::Entry> keep;
  for (auto& e : c.free) {
    if (dev >= 0 && e.dev != dev) {
      keep.push_back(e);
      continue;
    }
    cudaSetDevice(e.dev);
    cudaFree(e.p);
    c.held -= e.bytes;
  }
  c.free.swap(keep);
  if (cur >= 0) cudaSetDevice(cur);
}

void* arena_alloc(int dev, size_t bytes) {
  ArenaCache& c = arena_cache();
  {
    std::lock_guard<std::mutex> g(c.m);
    int best = -1;
    for (size_t q = 0; q < c.free.size(); ++q) {
      const auto& e = c.free[q];
      if (e.dev == dev && e.bytes >= bytes && e.bytes - bytes <= bytes / 4 &&
          (best < 0 || e.bytes < c.free[best].bytes))
        best = (int)q;
    }
    if (best >= 0) {
      void* p = c.free[best].p;
      c.held -= c.free[best].bytes;
      c.free.erase(c.free.begin() + best);
      return p;
    }
  }
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) == cudaSuccess) return p;
  cudaGetLastError();
  release_arena_cache(dev);
  p = nullptr;
  if (cudaMalloc(&p, bytes) == cudaSuccess) return p;
  cudaGetLastError();
  return nullptr;
}

// Opt-in (BF_ARENA_CACHE=1): keep arenas and the staging pool mapped after the
// last context of a device is destroyed.  By default the cache and the pool are
// handed back to the driver then, and the pool's release threshold is restored,
// so a caller embedding the drop-in in a larger CUDA job gets its memory back.
bool arena_cache_keep() {
  const char* e = std::getenv("BF_ARENA_CACHE");
  return e && e[0] == '1';
}

void device_ctx_opened(int dev) {
  ArenaCache& c = arena_cache();
  std::lock_guard<std::mutex> g(c.m);
  if (c.live[dev]++ == 0) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      cuuint64_t old = 0;
      if (!c.pool_thr.count(dev) &&
          cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &old) == cudaSuccess)
        c.pool_thr[dev] = old;
      // staging buffers (uploads, downloads) come from the stream-ordered pool;
      // keep its memory mapped between calls instead of releasing it at every
      // synchronisation (re-mapping 100+ MB per call dominated the transfers)
      cuuint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
}

void release_arena_cache(int dev);

void device_ctx_closed(int dev) {
  bool last = false;
  {
    ArenaCache& c = arena_cache();
    std::lock_guard<std::mutex> g(c.m);
    last = --c.live[dev] <= 0;
    if (last) c.live[dev] = 0;
  }
  if (!last || arena_cache_keep()) return;
  release_arena_cache(dev);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    ArenaCache& c = arena_cache();
    std::lock_guard<std::mutex> g(c.m);
    if (c.pool_thr.count(dev)) {
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &c.pool_thr[dev]);
      c.pool_thr.erase(dev);
    }
    cudaMemPoolTrimTo(pool, 0);
  }
}

void arena_free(int dev, void* p, size_t bytes) {
  ArenaCache& c = arena_cache();
  std::lock_guard<std::mutex> g(c.m);
  if (c.held + bytes > ARENA_CACHE_MAX) {
    cudaFree(p);
    return;
  }
  c.free.push_back({dev, bytes, p});
  c.held += bytes;
}

double* dalloc(bf_ctx* ctx, size_t n, int* err) {
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, n * sizeof(double));
  if (e != cudaSuccess) {
    *err = fail(ctx, BF_ECUDA, "cudaMalloc(%zu bytes) failed: %s", n * sizeof(double),
                cudaGetErrorString(e));
    return nullptr;
  }
  return static_cast<double*>(p);
}

cudaError_t (*stage_fn(const bf_ctx* ctx))(int, int, int, const StageArgs&, cudaStream_t) {
  return ctx->sch.precision == BF_PRECISION_EXACT ? bf_exact::launch_stage : bf_fast::launch_stage;
}
cudaError_t (*ghost_fn(const bf_ctx* ctx))(const GhostArgs&, cudaStream_t) {
  return ctx->sch.precision == BF_PRECISION_EXACT ? bf_exact::launch_ghost : bf_fast::launch_ghost;
}

cudaEvent_t take_event(bf_ctx* ctx) {
  if (!ctx->event_pool.empty()) {
    cudaEvent_t e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct ProfScope {
  bf_ctx* ctx;
  int cls;
  int kernels = 1;
  cudaEvent_t a = nullptr;
  ProfScope(bf_ctx* c, int k) : ctx(c), cls(k) {
    if (ctx->profiling) {
      a = take_event(ctx);
      record(a);
    }
  }
  // inside a step capture the records become event nodes of the graph
  void record(cudaEvent_t e) {
    cudaEventRecordWithFlags(e, ctx->stream,
                             ctx->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
  }
  ~ProfScope() {
    if (ctx->profiling) {
      cudaEvent_t b = take_event(ctx);
      record(b);
      ctx->pending.push_back({a, b, cls, kernels});
    }
  }
};

void drain_profile(bf_ctx* ctx) {
  for (auto& p : ctx->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      ctx->prof_ms[p.cls] += ms;
      ctx->prof_launches[p.cls] += 1;
      ctx->prof_kernels += p.kernels;
    }
    if (!p.owned_by_graph) {
      ctx->event_pool.push_back(p.a);
      ctx->event_pool.push_back(p.b);
    }
  }
  ctx->pending.clear();
}

// ---- finalize helpers ---------------------------------------------------------

int make_launch(bf_ctx* ctx, std::vector<GhostTask>& ts, bf_ctx::GhostLaunch& L);
int run_ghost_launch(bf_ctx* ctx, const bf_ctx::GhostLaunch& L, int extended);

int build_tables(bf_ctx* ctx) {
  const int ndim = ctx->ndim;
  // boundary-face overwrite maps (solver.py:526-580), canonical patch order
  std::vector<int> order(ctx->patches.size());
  for (size_t p = 0; p < order.size(); ++p) order[p] = (int)p;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
    const HostPatch& a = ctx->patches[x];
    const HostPatch& b = ctx->patches[y];
    if (a.block != b.block) return a.block < b.block;
    if (a.face != b.face) return a.face < b.face;
    return std::lexicographical_compare(a.box, a.box + 6, b.box, b.box + 6);
  });
  for (auto& hb : ctx->blocks) {
    for (int f = 0; f < 2 * ndim; ++f) {
      const int ax = f / 2;
      int ta = -1, tb = -1;
      for (int a = 0; a < 3; ++a)
        if (a != ax) (ta < 0 ? ta : tb) = a;
      hb.bface_h[f].assign((size_t)hb.n[ta] * hb.n[tb], BFACE_NONE);
    }
  }
  for (int p : order) {
    const HostPatch& hp = ctx->patches[p];
    unsigned char code;
    if (hp.type == BC_SLIP || hp.type == BC_NOSLIP) code = BFACE_WALL;
    else if (hp.type == BC_FARFIELD) code = BFACE_FARFIELD;
    else continue;
    HostBlock& hb = ctx->blocks[ctx->index_of[hp.block]];
    const int ax = hp.face / 2;
    int ta = -1, tb = -1;
    for (int a = 0; a < 3; ++a)
      if (a != ax) (ta < 0 ? ta : tb) = a;
    for (int u1 = hp.box[2 * tb]; u1 < hp.box[2 * tb + 1]; ++u1)
      for (int u0 = hp.box[2 * ta]; u0 < hp.box[2 * ta + 1]; ++u0)
        hb.bface_h[hp.face][(size_t)u0 + (size_t)hb.n[ta] * u1] = code;
  }
  for (auto& hb : ctx->blocks) {
    for (int f = 0; f < 2 * ndim; ++f) {
      void* p = nullptr;
      const size_t nb = std::max<size_t>(hb.bface_h[f].size(), 1);
      CK(cudaMalloc(&p, nb));
      CK(cudaMemcpy(p, hb.bface_h[f].data(), hb.bface_h[f].size(), cudaMemcpyHostToDevice));
      hb.bface_d[f] = static_cast<unsigned char*>(p);
      hb.dev.bface[f] = hb.bface_d[f];
    }
  }

  // ghost tasks: physical patches (one item per tangential cell).  A block thinner
  // than the ghost depth along an axis with physical patches has BC ghosts that
  // mirror the opposite face's ghosts, so the reference's sequential patch order
  // matters: such contexts run the BCs after the exchange, one launch per
  // per-block patch position (canonical order).
  std::vector<GhostTask>& fill = ctx->h_tasks_fill;
  std::vector<GhostTask>& unp = ctx->h_tasks_unpack;
  fill.clear();
  unp.clear();
  bool thin = false;
  for (const HostPatch& hp : ctx->patches) {
    const HostBlock& hb = ctx->blocks[ctx->index_of[hp.block]];
    if (hb.n[hp.face / 2] < hb.g) thin = true;
  }
  std::vector<std::vector<GhostTask>> bc_levels;
  std::map<int, int> bc_pos;
  std::vector<int> canon(ctx->patches.size());
  for (size_t p = 0; p < canon.size(); ++p) canon[p] = (int)p;
  for (int p : (thin ? canon : order)) {
    const HostPatch& hp = ctx->patches[p];
    const int bi = ctx->index_of[hp.block];
    const HostBlock& hb = ctx->blocks[bi];
    GhostTask t{};
    t.kind = GK_BC;
    t.bc_type = hp.type;
    t.block = bi;
    t.src_block = -1;
    t.axis = hp.face / 2;
    t.side = hp.face % 2;
    int ta = -1, tb = -1;
    for (int a = 0; a < 3; ++a)
      if (a != t.axis) (ta < 0 ? ta : tb) = a;
    t.ta = ta;
    t.tb = tb;
    t.tlo[0] = hp.box[2 * ta];
    t.tn[0] = hp.box[2 * ta + 1] - hp.box[2 * ta];
    t.tlo[1] = hp.box[2 * tb];
    t.tn[1] = hp.box[2 * tb + 1] - hp.box[2 * tb];
    t.depth = hb.g;
    t.items = (long long)t.tn[0] * t.tn[1];
    if (hp.type == BC_MMS) {
      const size_t need = (size_t)t.depth * 6 * t.items;
      if (hp.dirichlet.size() != need)
        return fail(ctx, BF_EINVAL, "mms_dirichlet patch on block %d: got %zu values, need %zu",
                    hp.block, hp.dirichlet.size(), need);
      void* d = nullptr;
      CK(cudaMalloc(&d, need * sizeof(double)));
      CK(cudaMemcpy(d, hp.dirichlet.data(), need * sizeof(double), cudaMemcpyHostToDevice));
      ctx->dirichlet_d.push_back(static_cast<double*>(d));
      t.dirichlet = static_cast<double*>(d);
    }
    if (thin) {
      const int j = bc_pos[bi]++;
      if ((int)bc_levels.size() <= j) bc_levels.resize(j + 1);
      if (t.items > 0) bc_levels[j].push_back(t);
    } else if (t.items > 0) {
      fill.push_back(t);
    }
  }
  ctx->r1_bc.clear();
  for (auto& lv : bc_levels) {
    bf_ctx::GhostLaunch L;
    int rc = make_launch(ctx, lv, L);
    if (rc) return rc;
    ctx->r1_bc.push_back(L);
  }

  // connected endpoints
  for (auto& L : ctx->links) {
    const int bi = ctx->index_of[L.block];
    const HostBlock& hb = ctx->blocks[bi];
    const int ghost[3] = {hb.g, hb.g, ndim == 3 ? hb.g : 0};
    int send[6], recv[6];
    halo_boxes(L.face, L.box, hb.n, ghost, send, recv);
    int ext[3];
    for (int a = 0; a < 3; ++a) ext[a] = recv[2 * a + 1] - recv[2 * a];
    int perm[3];
    bool flip[3];
    unpack_axes(L.face, L.amap, L.peer_face, perm, flip);
    int P[3];
    for (int a = 0; a < 3; ++a) P[perm[a]] = ext[a];
    const long long own_st[3] = {1, hb.sy, hb.sz};
    const int nf = (ndim == 3) ? 6 : 5;
    const bool local = (L.peer_rank == ctx->rank) && ctx->index_of.count(L.peer_block);
    GhostTask t{};
    t.kind = GK_COPY;
    t.nfields = nf;
    for (int a = 0; a < 3; ++a) t.n[a] = ext[a];
    t.items = (long long)ext[0] * ext[1] * ext[2];
    t.block = bi;
    t.dst_origin = hb.off(recv[0], recv[2], recv[4]);
    for (int a = 0; a < 3; ++a) t.dst_stride[a] = own_st[a];
    if (local) {
      const int pi = ctx->index_of[L.peer_block];
      const HostBlock& pb = ctx->blocks[pi];
      const int pghost[3] = {pb.g, pb.g, ndim == 3 ? pb.g : 0};
      int psend[6], precv[6];
      halo_boxes(L.peer_face, L.peer_box, pb.n, pghost, psend, precv);
      for (int a = 0; a < 3; ++a)
        if (psend[2 * a + 1] - psend[2 * a] != P[a])
          return fail(ctx, BF_EINVAL, "link tag %d: partner send box does not match", L.tag);
      const long long pst[3] = {1, pb.sy, pb.sz};
      t.src_block = pi;
      t.src_origin = pb.off(psend[0], psend[2], psend[4]);
      for (int a = 0; a < 3; ++a) {
        const long long s = pst[perm[a]];
        if (flip[a]) {
          t.src_origin += (long long)(ext[a] - 1) * s;
          t.src_stride[a] = -s;
        } else {
          t.src_stride[a] = s;
        }
      }
      if (t.items > 0) fill.push_back(t);
    } else {
      // pack: own send box -> send buffer (i-fastest over the own send box)
      L.cells = t.items;
      L.nfields = nf;
      int err = 0;
      L.send = dalloc(ctx, (size_t)nf * std::max<long long>(L.cells, 1), &err);
      if (err) return err;
      L.recv = dalloc(ctx, (size_t)nf * std::max<long long>(L.cells, 1), &err);
      if (err) return err;
      GhostTask pk{};
      pk.kind = GK_COPY;
      pk.nfields = nf;
      int sext[3];
      for (int a = 0; a < 3; ++a) sext[a] = send[2 * a + 1] - send[2 * a];
      for (int a = 0; a < 3; ++a) pk.n[a] = sext[a];
      pk.items = (long long)sext[0] * sext[1] * sext[2];
      pk.block = -1;
      pk.dst_buf = L.send;
      pk.buf_cells = L.cells;
      pk.dst_origin = 0;
      pk.dst_stride[0] = 1;
      pk.dst_stride[1] = sext[0];
      pk.dst_stride[2] = (long long)sext[0] * sext[1];
      pk.src_block = bi;
      pk.src_origin = hb.off(send[0], send[2], send[4]);
      for (int a = 0; a < 3; ++a) pk.src_stride[a] = own_st[a];
      if (pk.items > 0) fill.push_back(pk);
      // unpack: recv buffer (partner send box, partner axis order) -> own ghosts
      const long long Pst[3] = {1, P[0], (long long)P[0] * P[1]};
      t.src_block = -1;
      t.src_buf = L.recv;
      t.buf_cells = L.cells;
      t.src_origin = 0;
      for (int a = 0; a < 3; ++a) {
        const long long s = Pst[perm[a]];
        if (flip[a]) {
          t.src_origin += (long long)(ext[a] - 1) * s;
          t.src_stride[a] = -s;
        } else {
          t.src_stride[a] = s;
        }
      }
      if (t.items > 0) unp.push_back(t);
    }
  }
  long long acc = 0;
  for (auto& t : fill) {
    t.begin = acc;
    acc += t.items;
  }
  ctx->items_fill = acc;
  acc = 0;
  for (auto& t : unp) {
    t.begin = acc;
    acc += t.items;
  }
  ctx->items_unpack = acc;
  ctx->n_fill = (int)fill.size();
  ctx->n_unpack = (int)unp.size();
  auto block_map = [&](const std::vector<GhostTask>& ts, int2** dst, int* n, int ipt) -> int {
    std::vector<int2> m;
    for (size_t ti = 0; ti < ts.size(); ++ti)
      for (long long it = 0; it < ts[ti].items; it += (long long)GHOST_BLOCK * ipt)
        m.push_back(make_int2((int)ti, (int)it));
    // the tasks' CUDA blocks interleaved instead of task after task: the strided
    // i-face rows (32-byte sectors half used) and the dense j/k-face rows then
    // share the DRAM at any moment (C4 fill 0.101 -> 0.094 ms); BF_GHOST_INTERLEAVE=0:
    // task order.  Items and their values are unchanged, only the block order.
    if (ctx->ghost_interleave) {   // each task's blocks spread evenly over the launch
      std::vector<long long> cnt(ts.size(), 0), seen(ts.size(), 0);
      for (const int2& e : m) ++cnt[e.x];
      std::vector<std::pair<double, int2>> key;
      key.reserve(m.size());
      for (const int2& e : m) key.push_back({(seen[e.x]++ + 0.5) / cnt[e.x], e});
      std::stable_sort(key.begin(), key.end(),
                       [](const auto& x, const auto& y) { return x.first < y.first; });
      for (size_t q = 0; q < m.size(); ++q) m[q] = key[q].second;
    }
    *n = (int)m.size();
    if (m.empty()) return BF_OK;
    void* p = nullptr;
    CK(cudaMalloc(&p, m.size() * sizeof(int2)));
    CK(cudaMemcpy(p, m.data(), m.size() * sizeof(int2), cudaMemcpyHostToDevice));
    *dst = static_cast<int2*>(p);
    return BF_OK;
  };
  ctx->ipt_fill = ghost_ipt(ctx->items_fill);
  ctx->ipt_unpack = ghost_ipt(ctx->items_unpack);
  if (const char* e = std::getenv("BF_GHOST_IPT")) {   // A/B: items per thread of the fill
    ctx->ipt_fill = std::max(1, std::min(GHOST_ITEMS, std::atoi(e)));
  }
  if (int rc = block_map(fill, &ctx->d_map_fill, &ctx->nmap_fill, ctx->ipt_fill)) return rc;
  if (int rc = block_map(unp, &ctx->d_map_unpack, &ctx->nmap_unpack, ctx->ipt_unpack)) return rc;
  if (!fill.empty()) {
    void* p = nullptr;
    CK(cudaMalloc(&p, fill.size() * sizeof(GhostTask)));
    CK(cudaMemcpy(p, fill.data(), fill.size() * sizeof(GhostTask), cudaMemcpyHostToDevice));
    ctx->d_tasks_fill = static_cast<GhostTask*>(p);
  }
  if (!unp.empty()) {
    void* p = nullptr;
    CK(cudaMalloc(&p, unp.size() * sizeof(GhostTask)));
    CK(cudaMemcpy(p, unp.data(), unp.size() * sizeof(GhostTask), cudaMemcpyHostToDevice));
    ctx->d_tasks_unpack = static_cast<GhostTask*>(p);
  }
  return BF_OK;
}

// Ghost push rules (PushRule): for every source cell band of a block face,
// where the stage kernel writes the next stage's ghost values (bf_vl.cuh).
// Disabled (ghost kernel instead) when a block is thinner than 2 ghost depths.
// The in-kernel ghost push is measured slower on C4 than the separate ghost
// launch (stage 1.76 ms vs 1.30 + 0.11 ms: the x-face band cells run it on
// 2-4 divergent lanes on the critical path of every plane), so it is opt-in:
// build with -DBF_VL_PUSH=1 and run with BF_PUSH=1.
// Timing experiments on deliberately wrong kernel variants: BF_IGNORE_ERRORS=1
// keeps stepping past non-physical states (never set in tests or bench).
bool ignore_errors() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BF_IGNORE_ERRORS");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

bool push_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("BF_PUSH");
    v = (e && e[0] == '1' && bf_fast::vl_push_compiled()) ? 1 : 0;
  }
  return v == 1;
}

int build_push(bf_ctx* ctx) {
  const int ndim = ctx->ndim;
  const int nb = (int)ctx->blocks.size();
  ctx->push_ok = true;
  for (const HostBlock& hb : ctx->blocks)
    for (int a = 0; a < ndim; ++a)
      if (hb.n[a] < 2 * hb.g) ctx->push_ok = false;
  if (!ctx->push_ok) return BF_OK;
  std::vector<std::vector<PushRule>> per((size_t)nb * 6);
  for (const HostPatch& hp : ctx->patches) {
    int kind;
    switch (hp.type) {
      case BC_OUTFLOW: kind = PK_OUTFLOW; break;
      case BC_SLIP: kind = PK_SLIP; break;
      case BC_NOSLIP: kind = PK_NOSLIP; break;
      case BC_FARFIELD: kind = PK_FARFIELD; break;
      default: continue;   // inflow / MMS Dirichlet ghosts are constant
    }
    const int bi = ctx->index_of[hp.block];
    const HostBlock& hb = ctx->blocks[bi];
    PushRule r{};
    r.kind = kind;
    r.axis = hp.face / 2;
    r.side = hp.face % 2;
    for (int a = 0; a < 3; ++a) {
      r.lo[a] = hp.box[2 * a];
      r.hi[a] = hp.box[2 * a + 1];
    }
    const int ax = r.axis, n = hb.n[ax];
    const int layers = (kind == PK_SLIP || kind == PK_NOSLIP) ? hb.g : 1;   // source layers
    r.lo[ax] = r.side == 0 ? 0 : n - layers;
    r.hi[ax] = r.side == 0 ? layers : n;
    per[(size_t)bi * 6 + hp.face].push_back(r);
  }
  const int nf = ndim == 3 ? 6 : 5;
  for (auto& L : ctx->links) {
    const int bi = ctx->index_of[L.block];
    const HostBlock& hb = ctx->blocks[bi];
    const int ghost[3] = {hb.g, hb.g, ndim == 3 ? hb.g : 0};
    int send[6], recv[6];
    halo_boxes(L.face, L.box, hb.n, ghost, send, recv);
    const bool local = (L.peer_rank == ctx->rank) && ctx->index_of.count(L.peer_block);
    PushRule r{};
    r.nfields = nf;
    if (!local) {   // own send box -> message buffer, i-fastest over the box
      r.kind = PK_PACK;
      r.axis = L.face / 2;
      r.side = L.face % 2;
      int sext[3];
      for (int a = 0; a < 3; ++a) {
        r.lo[a] = send[2 * a];
        r.hi[a] = send[2 * a + 1];
        sext[a] = r.hi[a] - r.lo[a];
      }
      r.base = 0;
      r.coef[0] = 1;
      r.coef[1] = sext[0];
      r.coef[2] = (long long)sext[0] * sext[1];
      r.dst_fsz = L.cells;
      r.dst = L.send;
      per[(size_t)bi * 6 + L.face].push_back(r);
      continue;
    }
    // this endpoint receives from the peer block: the rule lives on the peer's face
    int ext[3];
    for (int a = 0; a < 3; ++a) ext[a] = recv[2 * a + 1] - recv[2 * a];
    int perm[3];
    bool flip[3];
    unpack_axes(L.face, L.amap, L.peer_face, perm, flip);
    const int pi = ctx->index_of[L.peer_block];
    const HostBlock& pb = ctx->blocks[pi];
    const int pghost[3] = {pb.g, pb.g, ndim == 3 ? pb.g : 0};
    int psend[6], precv[6];
    halo_boxes(L.peer_face, L.peer_box, pb.n, pghost, psend, precv);
    const long long own_st[3] = {1, hb.sy, hb.sz};
    r.kind = PK_COPY;
    r.axis = L.peer_face / 2;
    r.side = L.peer_face % 2;
    for (int b = 0; b < 3; ++b) {
      r.lo[b] = psend[2 * b];
      r.hi[b] = psend[2 * b + 1];
    }
    r.base = hb.off(recv[0], recv[2], recv[4]);
    for (int a = 0; a < 3; ++a) {
      if (flip[a]) {
        r.base += (long long)(ext[a] - 1) * own_st[a];
        r.coef[perm[a]] = -own_st[a];
      } else {
        r.coef[perm[a]] = own_st[a];
      }
    }
    r.dst_fsz = hb.fsz;
    r.dst = hb.dev.base;
    per[(size_t)pi * 6 + L.peer_face].push_back(r);
  }
  for (int bi = 0; bi < nb; ++bi) {
    size_t cnt = 0;
    for (int f = 0; f < 6; ++f) cnt += per[(size_t)bi * 6 + f].size();
    if (cnt > (size_t)PUSH_MAX_RULES) {
      ctx->push_ok = false;
      return BF_OK;
    }
  }
  std::vector<int> range((size_t)nb * 12, 0);
  ctx->h_push.clear();
  for (size_t q = 0; q < per.size(); ++q) {
    range[2 * q] = (int)ctx->h_push.size();
    for (auto& r : per[q]) ctx->h_push.push_back(r);
    range[2 * q + 1] = (int)ctx->h_push.size();
  }
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(ctx->h_push.size(), 1) * sizeof(PushRule)));
  if (!ctx->h_push.empty())
    CK(cudaMemcpy(p, ctx->h_push.data(), ctx->h_push.size() * sizeof(PushRule),
                  cudaMemcpyHostToDevice));
  ctx->d_push = static_cast<PushRule*>(p);
  CK(cudaMalloc(&p, range.size() * sizeof(int)));
  CK(cudaMemcpy(p, range.data(), range.size() * sizeof(int), cudaMemcpyHostToDevice));
  ctx->d_push_range = static_cast<int*>(p);
  return BF_OK;
}

std::vector<HostLink*> remote_links_sorted(bf_ctx* ctx);

// A ghost task list as its own launch: begin offsets and the block map.
int make_launch(bf_ctx* ctx, std::vector<GhostTask>& ts, bf_ctx::GhostLaunch& L) {
  long long acc = 0;
  for (auto& t : ts) {
    t.begin = acc;
    acc += t.items;
  }
  L.items = acc;
  L.ntasks = (int)ts.size();
  if (ts.empty()) return BF_OK;
  void* p = nullptr;
  CK(cudaMalloc(&p, ts.size() * sizeof(GhostTask)));
  CK(cudaMemcpy(p, ts.data(), ts.size() * sizeof(GhostTask), cudaMemcpyHostToDevice));
  L.d = static_cast<GhostTask*>(p);
  L.ipt = ghost_ipt(L.items);
  std::vector<int2> m;
  for (size_t ti = 0; ti < ts.size(); ++ti)
    for (long long it = 0; it < ts[ti].items; it += (long long)GHOST_BLOCK * L.ipt)
      m.push_back(make_int2((int)ti, (int)it));
  L.nmap = (int)m.size();
  CK(cudaMalloc(&p, std::max<size_t>(m.size(), 1) * sizeof(int2)));
  if (!m.empty()) CK(cudaMemcpy(p, m.data(), m.size() * sizeof(int2), cudaMemcpyHostToDevice));
  L.map = static_cast<int2*>(p);
  return BF_OK;
}

// Laminar NS ghost round 2 (solver.py:777-784; exchange.py:495-521; halo.py):
// every round-2 send box is packed before any unpack (snapshot), unpacks run
// in the reference's exchange order (their widened boxes overlap at edges and
// corners: the last writer wins), then the extended physical BCs in each
// block's canonical patch order (later patches overwrite shared corners).
int build_round2(bf_ctx* ctx) {
  const int ndim = ctx->ndim;
  const int nf = ndim == 3 ? 6 : 5;
  std::vector<GhostTask> pack;
  std::vector<std::pair<int, GhostTask>> unp;   // (order, task)
  for (size_t q = 0; q < ctx->links.size(); ++q) {
    HostLink& L = ctx->links[q];
    const int bi = ctx->index_of[L.block];
    const HostBlock& hb = ctx->blocks[bi];
    const int ghost[3] = {hb.g, hb.g, ndim == 3 ? hb.g : 0};
    int send[6], recv[6];
    halo_boxes(L.face, L.box, hb.n, ghost, send, recv, 2);
    int ext[3];
    for (int a = 0; a < 3; ++a) ext[a] = recv[2 * a + 1] - recv[2 * a];
    int perm[3];
    bool flip[3];
    unpack_axes(L.face, L.amap, L.peer_face, perm, flip);
    int P[3];   // partner send-box extents, partner axes
    for (int a = 0; a < 3; ++a) P[perm[a]] = ext[a];
    const bool local = (L.peer_rank == ctx->rank) && ctx->index_of.count(L.peer_block);
    L.cells2 = (long long)ext[0] * ext[1] * ext[2];
    int err = 0;
    L.send2 = dalloc(ctx, (size_t)nf * std::max<long long>(L.cells2, 1), &err);
    if (err) return err;
    if (!local) {
      L.recv2 = dalloc(ctx, (size_t)nf * std::max<long long>(L.cells2, 1), &err);
      if (err) return err;
    }
    // pack: the SENDER's round-2 send box, i-fastest in the sender's axes
    GhostTask pk{};
    pk.kind = GK_COPY;
    pk.nfields = nf;
    pk.block = -1;
    pk.dst_buf = L.send2;
    pk.buf_cells = L.cells2;
    pk.live_block = -1;
    int sbox[6];
    const HostBlock* sb = &hb;
    int sbi = bi;
    if (local) {
      sbi = ctx->index_of[L.peer_block];
      sb = &ctx->blocks[sbi];
      const int pg[3] = {sb->g, sb->g, ndim == 3 ? sb->g : 0};
      int precv[6];
      halo_boxes(L.peer_face, L.peer_box, sb->n, pg, sbox, precv, 2);
    } else {
      std::memcpy(sbox, send, sizeof sbox);
    }
    int sext[3];
    for (int a = 0; a < 3; ++a) sext[a] = sbox[2 * a + 1] - sbox[2 * a];
    if (local)
      for (int a = 0; a < 3; ++a)
        if (sext[a] != P[a]) return fail(ctx, BF_EINVAL, "link tag %d: round-2 boxes differ", L.tag);
    for (int a = 0; a < 3; ++a) pk.n[a] = sext[a];
    pk.items = (long long)sext[0] * sext[1] * sext[2];
    pk.dst_origin = 0;
    pk.dst_stride[0] = 1;
    pk.dst_stride[1] = sext[0];
    pk.dst_stride[2] = (long long)sext[0] * sext[1];
    pk.src_block = sbi;
    pk.src_origin = sb->off(sbox[0], sbox[2], sbox[4]);
    pk.src_stride[0] = 1;
    pk.src_stride[1] = sb->sy;
    pk.src_stride[2] = sb->sz;
    if (pk.items > 0) pack.push_back(pk);
    // unpack: buffer (partner axes, flips) -> own widened recv box
    GhostTask t{};
    t.kind = GK_COPY;
    t.nfields = nf;
    for (int a = 0; a < 3; ++a) t.n[a] = ext[a];
    t.items = L.cells2;
    t.block = bi;
    t.src_block = -1;
    t.dst_origin = hb.off(recv[0], recv[2], recv[4]);
    const long long own_st[3] = {1, hb.sy, hb.sz};
    for (int a = 0; a < 3; ++a) t.dst_stride[a] = own_st[a];
    t.src_buf = local ? L.send2 : L.recv2;
    t.buf_cells = L.cells2;
    const long long Pst[3] = {1, P[0], (long long)P[0] * P[1]};
    t.src_origin = 0;
    for (int a = 0; a < 3; ++a) {
      const long long st = Pst[perm[a]];
      if (flip[a]) {
        t.src_origin += (long long)(ext[a] - 1) * st;
        t.src_stride[a] = -st;
      } else {
        t.src_stride[a] = st;
      }
    }
    t.live_block = -1;
    t.live_mask = 0;
    if (local && box_is_view(sbox, sb->P)) {   // rho, p, T by reference (halo.py:58)
      // sbox is in interior coords; the view test needs padded coords (shift is harmless)
      t.live_mask = (1 << 0) | (1 << (nf - 2)) | (1 << (nf - 1));
      t.live_block = sbi;
      const long long pst[3] = {1, sb->sy, sb->sz};
      t.live_origin = sb->off(sbox[0], sbox[2], sbox[4]);
      for (int a = 0; a < 3; ++a) {
        const long long st = pst[perm[a]];
        if (flip[a]) {
          t.live_origin += (long long)(ext[a] - 1) * st;
          t.live_stride[a] = -st;
        } else {
          t.live_stride[a] = st;
        }
      }
    }
    const int ord = L.order2 >= 0 ? L.order2 : (int)q;
    // distributed engine: local entries first, then the remote ones (exchange.py:506-521)
    if (t.items > 0) unp.push_back({(local ? 0 : 1 << 20) + ord, t});
  }
  int rc = make_launch(ctx, pack, ctx->r2_pack);
  if (rc) return rc;
  std::stable_sort(unp.begin(), unp.end(),
                   [](const auto& a, const auto& b) { return a.first < b.first; });
  ctx->r2_unpack.clear();
  for (auto& e : unp) {
    std::vector<GhostTask> one{e.second};
    bf_ctx::GhostLaunch L;
    rc = make_launch(ctx, one, L);
    if (rc) return rc;
    ctx->r2_unpack.push_back(L);
  }
  // extended BCs: launch j = the j-th physical patch (insertion = canonical order) of
  // every block
  std::map<int, int> seen;
  std::vector<std::vector<GhostTask>> levels;
  for (const HostPatch& hp : ctx->patches) {
    const int bi = ctx->index_of[hp.block];
    const HostBlock& hb = ctx->blocks[bi];
    const int j = seen[bi]++;
    if ((int)levels.size() <= j) levels.resize(j + 1);
    GhostTask t{};
    t.kind = GK_BC;
    t.bc_type = hp.type;
    t.block = bi;
    t.src_block = -1;
    t.axis = hp.face / 2;
    t.side = hp.face % 2;
    int ta = -1, tb = -1;
    for (int a = 0; a < 3; ++a)
      if (a != t.axis) (ta < 0 ? ta : tb) = a;
    t.ta = ta;
    t.tb = tb;
    const int gg[3] = {hb.g, hb.g, ndim == 3 ? hb.g : 0};
    t.tlo[0] = hp.box[2 * ta] - gg[ta];
    t.tn[0] = hp.box[2 * ta + 1] - hp.box[2 * ta] + 2 * gg[ta];
    t.tlo[1] = hp.box[2 * tb] - gg[tb];
    t.tn[1] = hp.box[2 * tb + 1] - hp.box[2 * tb] + 2 * gg[tb];
    t.depth = hb.g;
    t.items = (long long)t.tn[0] * t.tn[1];
    if (hp.type == BC_MMS) {
      const size_t need = (size_t)t.depth * 6 * t.items;
      if (hp.dirichlet_ext.size() != need)
        return fail(ctx, BF_EINVAL, "mms_dirichlet patch on block %d: %zu extended values, need %zu",
                    hp.block, hp.dirichlet_ext.size(), need);
      void* d = nullptr;
      CK(cudaMalloc(&d, need * sizeof(double)));
      CK(cudaMemcpy(d, hp.dirichlet_ext.data(), need * sizeof(double), cudaMemcpyHostToDevice));
      ctx->dirichlet_d.push_back(static_cast<double*>(d));
      t.dirichlet = static_cast<double*>(d);
    }
    if (t.items > 0) levels[j].push_back(t);
  }
  ctx->r2_bc.clear();
  for (auto& lv : levels) {
    bf_ctx::GhostLaunch L;
    rc = make_launch(ctx, lv, L);
    if (rc) return rc;
    ctx->r2_bc.push_back(L);
  }
  return BF_OK;
}

// One of the round-2 launches on ctx->stream.
int run_ghost_launch(bf_ctx* ctx, const bf_ctx::GhostLaunch& L, int extended) {
  if (L.ntasks == 0 || L.nmap == 0) return BF_OK;
  GhostArgs g{};
  g.blocks = ctx->d_blocks;
  g.tasks = L.d;
  g.block_map = L.map;
  g.nlaunch = L.nmap;
  g.ntasks = L.ntasks;
  g.total_items = L.items;
  g.cur = ctx->cur;
  g.t_derived = ctx->t_derived;
  g.extended = extended;
  g.ipt = L.ipt;
  g.stop = ctx->stop_flag();
  g.c = ctx->c;
  CK(ghost_fn(ctx)(g, ctx->stream));
  return BF_OK;
}

int sync_ghosts_from_other(bf_ctx* ctx) {
  for (auto& hb : ctx->blocks) {
    const long long np = (long long)hb.P[0] * hb.P[1] * hb.P[2];
    ghost_sync_kernel<<<grid_for(np), 256, 0, ctx->stream>>>(
        hb.dev.f(fw(ctx->cur, 0)) - hb.origin, hb.dev.f(fw(ctx->cur ^ 1, 0)) - hb.origin,
        hb.fsz, hb.lead, hb.sy, hb.sz, hb.P[0], hb.P[1], hb.P[2], hb.g, hb.g,
        ctx->ndim == 3 ? hb.g : 0, hb.n[0], hb.n[1], hb.n[2]);
    CK(cudaGetLastError());
  }
  return BF_OK;
}

enum { XC_MESSAGES, XC_RUNS, XC_BYTES, XC_STAGING, XC_WAITS, XC_MAX_PENDING };

// One grouped exchange of `n` remote endpoints: n sends + n receives in flight,
// one pack and one unpack launch, one completion the unpack waits on.
void count_exchange(bf_ctx* ctx, long long n, long long bytes) {
  ctx->xc[XC_MESSAGES] += n;
  ctx->xc[XC_BYTES] += bytes;
  ctx->xc[XC_RUNS] += 2;
  ctx->xc[XC_WAITS] += 1;
  ctx->xc[XC_MAX_PENDING] = std::max(ctx->xc[XC_MAX_PENDING], 2 * n);
}

// Round 2 of a ghost update: packs, remote messages, ordered unpacks, extended BCs.
int ghosts_round2(bf_ctx* ctx) {
  int rc = run_ghost_launch(ctx, ctx->r2_pack, 0);
  if (rc) return rc;
  bool remote = false;
  for (auto& L : ctx->links)
    if (L.recv2) remote = true;
  if (remote) {
    if (!ctx->comm)
      return fail(ctx, BF_EINVAL, "rank %d has remote links but no communicator", ctx->rank);
    {
      long long n = 0, b = 0;
      for (HostLink* L : remote_links_sorted(ctx)) {
        ++n;
        b += (long long)sizeof(double) * L->nfields * L->cells2;
      }
      count_exchange(ctx, n, b);
    }
    NK(net(ctx).GroupStart());
    for (HostLink* L : remote_links_sorted(ctx)) {
      const size_t cnt = (size_t)L->nfields * L->cells2;
      NK(net(ctx).Send(L->send2, cnt, ncclDouble, L->peer_rank, ctx->comm, ctx->stream));
      NK(net(ctx).Recv(L->recv2, cnt, ncclDouble, L->peer_rank, ctx->comm, ctx->stream));
    }
    NK(net(ctx).GroupEnd());
  }
  for (auto& L : ctx->r2_unpack) {
    rc = run_ghost_launch(ctx, L, 0);
    if (rc) return rc;
  }
  for (auto& L : ctx->r2_bc) {
    rc = run_ghost_launch(ctx, L, 1);
    if (rc) return rc;
  }
  return BF_OK;
}

// One 4-D tensor map per (block, box shape) over the block arena:
// dims (pitch, P1, P2, field slot), strides (sy, sz, fsz) doubles.  Box shapes
// follow the stage kernel's tile (bf_stage.cuh): the 5-variable haloed plane,
// x / y face geometry, Q0, dt/V, z face geometry.
int build_tensor_maps(bf_ctx* ctx) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess)
      return fail(ctx, BF_ECUDA, "cuTensorMapEncodeTiled is unavailable");
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  const int TJ = bf_exact::stage_tile_rows(ctx->ndim, ctx->sch.limiter);
  const cuuint32_t boxes[NTMAP][4] = {
      {(cuuint32_t)(TI + 2 * HALO), (cuuint32_t)(TJ + 2 * HALO), 1, 5},   // W plane
      {(cuuint32_t)GXW, (cuuint32_t)TJ, 1, 4},                             // x-face geometry
      {(cuuint32_t)TI, (cuuint32_t)(TJ + 1), 1, 4},                        // y-face geometry
      {(cuuint32_t)TI, (cuuint32_t)TJ, 1, 5},                              // Q0
      {(cuuint32_t)TI, (cuuint32_t)TJ, 1, 1},                              // dt/V or V
      {(cuuint32_t)TI, (cuuint32_t)TJ, 1, 4}};                             // z-face geometry
  std::vector<CUtensorMap> maps(ctx->blocks.size() * NTMAP);
  for (size_t bi = 0; bi < ctx->blocks.size(); ++bi) {
    const HostBlock& hb = ctx->blocks[bi];
    const cuuint64_t dims[4] = {(cuuint64_t)hb.sy, (cuuint64_t)hb.P[1], (cuuint64_t)hb.P[2],
                                (cuuint64_t)hb.nslots};
    const cuuint64_t strides[3] = {(cuuint64_t)hb.sy * 8, (cuuint64_t)hb.sz * 8,
                                   (cuuint64_t)hb.fsz * 8};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    for (int m = 0; m < NTMAP; ++m) {
      const CUresult r = encode(&maps[bi * NTMAP + m], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4,
                                hb.arena, dims, strides, boxes[m], estr,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS)
        return fail(ctx, BF_ECUDA, "cuTensorMapEncodeTiled failed (%d) for block %d map %d",
                    (int)r, hb.id, m);
    }
  }
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(maps.size(), 1) * sizeof(CUtensorMap)));
  CK(cudaMemcpy(p, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  ctx->d_tmaps = static_cast<unsigned char*>(p);
  static_assert(sizeof(CUtensorMap) == 128, "CUtensorMap layout");
  return BF_OK;
}

int build_tiles(bf_ctx* ctx) {
  std::vector<Tile> tiles;
  std::vector<int> tb;
  for (size_t bi = 0; bi < ctx->blocks.size(); ++bi) {
    HostBlock& hb = ctx->blocks[bi];
    hb.tile_begin = (int)tiles.size();
    tb.push_back(hb.tile_begin);
    const int kc = ctx->ndim == 3 ? ctx->kc : 1;
    const int TJ = bf_exact::stage_tile_rows(ctx->ndim, ctx->sch.limiter);
    const int nk = ctx->ndim == 3 ? hb.n[2] : 1;
    for (int k0 = 0; k0 < nk; k0 += kc)
      for (int j0 = 0; j0 < hb.n[1]; j0 += TJ)
        for (int i0 = 0; i0 < hb.n[0]; i0 += TI)
          tiles.push_back(Tile{(int)bi, i0, j0, k0, std::min(kc, nk - k0)});
    hb.tile_end = (int)tiles.size();
  }
  tb.push_back((int)tiles.size());
  ctx->ntiles = (int)tiles.size();
  {
    // interior / boundary split: a tile is boundary when it touches a block face
    // carrying a remote (message) link — its halo reads ghost cells filled by the
    // unpack.  BF_SPLIT_TILES=1 forces the two-launch path on every block face
    // (exercised on one GPU by the tests).
    const char* e = std::getenv("BF_SPLIT_TILES");
    const bool force = e && e[0] == '1';
    // BF_HIDE_GHOSTS=1 (one-rank ctx): every block face carries a ghost fill
    // (connected copy or physical patch), so tiles touching any face wait for
    // the fill on the comm stream and the others run beside it.  Measured
    // slower (C4 stage span 1.257 vs 1.100 + 0.101 ms): a stage CTA holds a
    // whole SM (64K registers), so the latency-bound fill only gets the SMs
    // that retiring tiles free, one at a time — off by default.
    const char* h = std::getenv("BF_HIDE_GHOSTS");
    bool has_remote = false;
    for (auto& L : ctx->links) has_remote = has_remote || L.send != nullptr;
    ctx->hide_fill = (h && h[0] == '1') && !force && !has_remote && ctx->ndim == 3 &&
                     !ctx->sch.viscous && ctx->r1_bc.empty() && !(ctx->push_ok && push_enabled());
    std::vector<std::array<bool, 6>> remote(ctx->blocks.size());
    for (auto& r : remote) r.fill(force || ctx->hide_fill);
    bool any = force || ctx->hide_fill;
    for (auto& L : ctx->links)
      if (L.send) {
        remote[ctx->index_of[L.block]][L.face] = true;
        any = true;
      }
    std::vector<int> tin, tbd, fin, fbd;
    const int TJ = bf_exact::stage_tile_rows(ctx->ndim, ctx->sch.limiter);
    // a tile reads cells [i0 - HALO, i0 + TI + HALO) x [j0 - HALO, j0 + TJ + HALO) x
    // [k0 - HALO, k0 + kc + HALO): it reads face f's ghost cells when that range
    // crosses the face
    auto touches = [&](const Tile& t, int f) {
      const HostBlock& hb = ctx->blocks[t.block];
      switch (f) {
        case 0: return t.i0 < HALO;
        case 1: return t.i0 + TI + HALO > hb.n[0];
        case 2: return t.j0 < HALO;
        case 3: return t.j0 + TJ + HALO > hb.n[1];
        case 4: return ctx->ndim == 3 && t.k0 < HALO;
        default: return ctx->ndim == 3 && t.k0 + t.kc + HALO > hb.n[2];
      }
    };
    for (int q = 0; q < (int)tiles.size(); ++q) {
      const Tile& t = tiles[q];
      const auto& rf = remote[t.block];
      bool bd = false, any_face = false;
      for (int f = 0; f < 6; ++f) {
        const bool hit = touches(t, f);
        bd = bd || (rf[f] && hit);
        any_face = any_face || hit;
      }
      (bd ? tbd : tin).push_back(q);
      (any_face ? fbd : fin).push_back(q);
    }
    // fused ghost fill order: tiles reading no ghost cell first, then the others
    ctx->n_fused_in = (int)fin.size();
    fin.insert(fin.end(), fbd.begin(), fbd.end());
    {
      void* q = nullptr;
      CK(cudaMalloc(&q, std::max<size_t>(fin.size(), 1) * sizeof(int)));
      if (!fin.empty()) CK(cudaMemcpy(q, fin.data(), fin.size() * sizeof(int), cudaMemcpyHostToDevice));
      ctx->d_tiles_fused = static_cast<int*>(q);
      CK(cudaMalloc(&q, 4 * sizeof(unsigned)));
      CK(cudaMemset(q, 0, 4 * sizeof(unsigned)));
      ctx->d_fill_sync = static_cast<unsigned*>(q);
    }
    ctx->split_tiles = any;
    ctx->split_forced = force;
    ctx->n_tiles_in = (int)tin.size();
    ctx->n_tiles_bd = (int)tbd.size();
    if (any) {
      void* q = nullptr;
      CK(cudaMalloc(&q, std::max<size_t>(tin.size(), 1) * sizeof(int)));
      if (!tin.empty()) CK(cudaMemcpy(q, tin.data(), tin.size() * sizeof(int), cudaMemcpyHostToDevice));
      ctx->d_tiles_in = static_cast<int*>(q);
      CK(cudaMalloc(&q, std::max<size_t>(tbd.size(), 1) * sizeof(int)));
      if (!tbd.empty()) CK(cudaMemcpy(q, tbd.data(), tbd.size() * sizeof(int), cudaMemcpyHostToDevice));
      ctx->d_tiles_bd = static_cast<int*>(q);
      // high priority: when a stage-kernel CTA retires, the block scheduler hands the
      // SM to the NCCL / unpack kernels first
      int lo_prio = 0, hi_prio = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
      CK(cudaStreamCreateWithPriority(&ctx->comm_stream, cudaStreamNonBlocking, hi_prio));
      CK(cudaEventCreateWithFlags(&ctx->ev_filled, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_unpacked, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_bd, cudaEventDisableTiming));
    }
  }
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(tiles.size(), 1) * sizeof(Tile)));
  CK(cudaMemcpy(p, tiles.data(), tiles.size() * sizeof(Tile), cudaMemcpyHostToDevice));
  ctx->d_tiles = static_cast<Tile*>(p);
  CK(cudaMalloc(&p, tb.size() * sizeof(int)));
  CK(cudaMemcpy(p, tb.data(), tb.size() * sizeof(int), cudaMemcpyHostToDevice));
  ctx->d_tile_begin = static_cast<int*>(p);
  return BF_OK;
}

// ---- per-stage sequencing ------------------------------------------------------

GhostArgs ghost_args(bf_ctx* ctx, bool unpack) {
  GhostArgs g{};
  g.blocks = ctx->d_blocks;
  g.tasks = unpack ? ctx->d_tasks_unpack : ctx->d_tasks_fill;
  g.block_map = unpack ? ctx->d_map_unpack : ctx->d_map_fill;
  g.nlaunch = unpack ? ctx->nmap_unpack : ctx->nmap_fill;
  g.ntasks = unpack ? ctx->n_unpack : ctx->n_fill;
  g.total_items = unpack ? ctx->items_unpack : ctx->items_fill;
  g.ipt = unpack ? ctx->ipt_unpack : ctx->ipt_fill;
  g.cur = ctx->cur;
  g.t_derived = ctx->t_derived;
  g.stop = ctx->stop_flag();
  g.c = ctx->c;
  return g;
}

int launch_fill(bf_ctx* ctx) {
  ProfScope ps(ctx, 1);
  CK(ghost_fn(ctx)(ghost_args(ctx, false), ctx->stream));
  return BF_OK;
}

int launch_unpack(bf_ctx* ctx) {
  ProfScope ps(ctx, 2);
  CK(ghost_fn(ctx)(ghost_args(ctx, true), ctx->stream));
  return BF_OK;
}

// Message issue order of a rank's remote endpoints: (peer rank, link tag, own
// block id) — both endpoints of a link see the same (tag) and their peer's
// rank, so NCCL pairs each send with the matching receive.  Mirrored by
// distributed.remote_links (checked by tests/test_abi.py via bf_probe_remote_order).
bool remote_before(int peer_a, int tag_a, int block_a, int peer_b, int tag_b, int block_b) {
  if (peer_a != peer_b) return peer_a < peer_b;
  if (tag_a != tag_b) return tag_a < tag_b;
  return block_a < block_b;
}

std::vector<HostLink*> remote_links_sorted(bf_ctx* ctx) {
  std::vector<HostLink*> out;
  for (auto& L : ctx->links)
    if (L.send) out.push_back(&L);
  std::stable_sort(out.begin(), out.end(), [](const HostLink* a, const HostLink* b) {
    return remote_before(a->peer_rank, a->tag, a->block, b->peer_rank, b->tag, b->block);
  });
  return out;
}

int nccl_exchange(bf_ctx* ctx) {
  auto rl = remote_links_sorted(ctx);
  if (rl.empty()) return BF_OK;
  {
    long long b = 0;
    for (HostLink* L : rl) b += (long long)sizeof(double) * L->nfields * L->cells;
    count_exchange(ctx, (long long)rl.size(), b);
  }
  NK(net(ctx).GroupStart());
  for (HostLink* L : rl) {
    const size_t cnt = (size_t)L->nfields * L->cells;
    NK(net(ctx).Send(L->send, cnt, ncclDouble, L->peer_rank, ctx->comm, ctx->stream));
    NK(net(ctx).Recv(L->recv, cnt, ncclDouble, L->peer_rank, ctx->comm, ctx->stream));
  }
  NK(net(ctx).GroupEnd());
  return BF_OK;
}

// ghosts of W[cur] for a standalone / NCCL ctx
// Physical + local ghosts of W[cur] (and packed messages) unless the last
// stage kernel already pushed them; on the first fill after an upload the
// other buffer gets its constant ghosts (inflow, MMS) too, since pushes never
// write those.
int fill_ghosts(bf_ctx* ctx) {
  if (ctx->pushed) return BF_OK;
  if (!ctx->other_filled) {
    ctx->cur ^= 1;
    int rc = launch_fill(ctx);
    ctx->cur ^= 1;
    if (rc) return rc;
    ctx->other_filled = true;
  }
  return launch_fill(ctx);
}

int ghosts_solo(bf_ctx* ctx) {
  if ((ctx->sch.viscous || !ctx->r1_bc.empty()) && ctx->synced_cur != ctx->cur_epoch) {
    int r0 = sync_ghosts_from_other(ctx);
    if (r0) return r0;
    ctx->synced_cur = ctx->cur_epoch;
  }
  if (ctx->hide_fill && ctx->split_tiles && !ctx->pushed) {
    // the fill goes to comm_stream after everything queued so far (the previous
    // stage, both of its launches); the next stage's interior tiles run beside
    // it and its boundary tiles follow it there (launch_stage_kernel)
    CK(cudaEventRecord(ctx->ev_filled, ctx->stream));
    CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_filled, 0));
    cudaStream_t saved = ctx->stream;
    ctx->stream = ctx->comm_stream;
    const int rc = fill_ghosts(ctx);
    ctx->stream = saved;
    if (rc) return rc;
    ctx->fill_pending = true;
    ctx->ghost_buf = ctx->cur;
    return BF_OK;
  }
  int rc = fill_ghosts(ctx);
  if (rc) return rc;
  if (ctx->n_unpack && ctx->comm && ctx->split_tiles && !ctx->no_overlap && !ctx->sch.viscous &&
      ctx->r1_bc.empty()) {
    // messages and unpack on the comm stream; the interior tiles of the next stage
    // run meanwhile on the main stream, its boundary tiles follow the unpack on
    // the comm stream (launch_stage_kernel)
    CK(cudaEventRecord(ctx->ev_filled, ctx->stream));
    CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_filled, 0));
    cudaStream_t saved = ctx->stream;
    ctx->stream = ctx->comm_stream;
    rc = nccl_exchange(ctx);
    if (!rc) rc = launch_unpack(ctx);
    ctx->stream = saved;
    if (rc) return rc;
    CK(cudaEventRecord(ctx->ev_unpacked, ctx->comm_stream));
    ctx->exchange_pending = true;
    ctx->ghost_buf = ctx->cur;
    return BF_OK;
  }
  if (ctx->n_unpack) {
    if (!ctx->comm)
      return fail(ctx, BF_EINVAL,
                  "rank %d has remote links but no communicator (bf_nccl_init or bf_group)",
                  ctx->rank);
    rc = nccl_exchange(ctx);
    if (rc) return rc;
    rc = launch_unpack(ctx);
    if (rc) return rc;
  }
  for (auto& L : ctx->r1_bc) {   // thin blocks: BCs after the exchange, in order
    rc = run_ghost_launch(ctx, L, 0);
    if (rc) return rc;
  }
  if (ctx->sch.viscous) {   // edge / corner completion (solver.py:781-784)
    rc = ghosts_round2(ctx);
    if (rc) return rc;
  }
  ctx->ghost_buf = ctx->cur;
  return BF_OK;
}

int stage_flags(bf_ctx* ctx, int step_index, int k, int nst) {
  int flags = 0;
  if (k == 0) flags |= F_STAGE0;
  if (k == nst - 1) flags |= F_LAST;
  if (ctx->blocks.size() && ctx->blocks[0].has_src) flags |= F_SOURCE;
  const int fz = ctx->sch.limiter_freeze_at;
  if (fz > 0) {
    const bool frozen = step_index > fz;
    if (frozen) {
      if (ctx->psi_valid) flags |= F_PSI_LOAD;
      else flags |= F_PSI_STORE;   // first frozen evaluation computes and keeps them
    } else if (k == nst - 1) {
      flags |= F_PSI_STORE;        // psi of the last stage is what a freeze pins
    }
  }
  return flags;
}

// Fused ghost fill (StageArgs::fill_ctas): on a one-rank inviscid ctx the FAST
// cell-split Van Leer launch fills the ghosts of W[cur] itself — the first
// fill_ctas CTAs do the ghost_kernel's work while the tiles that read no ghost
// cell run, the boundary tiles wait for it — instead of a separate ghost launch
// before every stage.  BF_FUSED_FILL=0 / 1 forces it off / on (A/B, tests;
// default: fused_fill_pays), BF_FILL_CTAS=n sets the fill CTAs per launch (both
// read at context creation).
//
// Fill-only CTAs of a fused launch: when the tiles and one fill warp per
// chunk fit on the SMs at once, that many (latency: one chunk per warp);
// otherwise BF_FILL_CTAS (default 16), which run beside the interior tiles.
int fill_ctas_for(const bf_ctx* ctx) {
  if (ctx->fill_ctas_env > 0) return ctx->fill_ctas_env;
  const int wpc = TI * bf_exact::stage_tile_rows(ctx->ndim, ctx->sch.limiter) / 32;
  const int one_each = (4 * ctx->nmap_fill + wpc - 1) / wpc;
  if (ctx->ntiles + one_each <= ctx->num_sms) return one_each;
  return 16;
}

// Where the fused fill pays (profiles/r02_fused_fill.jsonl): a small fill —
// latency-bound, C2: 0.128 -> 0.117 ms per step — hidden behind at least a
// wave of interior tiles.  A large one (C4: ~1.2M ghost items, 0.10 ms) is
// bound by the SMs' outstanding strided-sector misses: squeezed onto a few
// fill CTAs it takes as many SM-milliseconds as the whole-GPU ghost launch
// (C4 stage 1.44-2.4 ms with 32-8 fill CTAs vs 1.20 + 0.10 ms), and with too
// few interior tiles (C1) the boundary tiles just wait for it.
bool fused_fill_pays(const bf_ctx* ctx) {
  return ctx->items_fill <= (1LL << 18) && ctx->n_fused_in >= ctx->num_sms;
}

bool fused_fill_ok(const bf_ctx* ctx, int flags) {
  const bool on = ctx->fused_mode < 0 ? fused_fill_pays(ctx) : ctx->fused_mode == 1;
  return on && ctx->sch.precision != BF_PRECISION_EXACT && !ctx->sch.viscous &&
         bf_fast::vl_active(ctx->sch.flux, flags) && ctx->nranks == 1 && !ctx->comm &&
         !ctx->group && ctx->r1_bc.empty() && ctx->n_unpack == 0 && !ctx->split_forced &&
         !ctx->hide_fill && ctx->other_filled && !ctx->pushed &&
         !(ctx->push_ok && push_enabled()) && ctx->nmap_fill > 0 && ctx->ntiles > 0 &&
         ctx->d_tiles_fused && ctx->d_fill_sync;
}

int launch_stage_kernel(bf_ctx* ctx, int k, int flags, double alpha) {
  StageArgs a{};
  a.blocks = ctx->d_blocks;
  a.tiles = ctx->d_tiles;
  a.ntiles = ctx->ntiles;
  a.cur = ctx->cur;
  a.stage = k;
  a.flags = flags;
  a.alpha = alpha;
  a.partial = ctx->d_partial;
  a.err = ctx->d_err;
  a.tmaps = ctx->d_tmaps;
  a.stop = ctx->stop_flag();
  a.c = ctx->c;
  const bool vl = ctx->sch.precision != BF_PRECISION_EXACT && !ctx->sch.viscous &&
                  bf_fast::vl_active(ctx->sch.flux, flags);
  a.t_derived = ctx->t_derived;
  if (ctx->sch.viscous) {   // Fv x A of every face from the current state (ghosts round 2)
    ProfScope ps(ctx, 2);
    ViscArgs va{};
    va.blocks = ctx->d_blocks;
    va.tasks = ctx->d_visc;
    va.map = ctx->d_visc_map;
    va.cur = ctx->cur;
    va.t_derived = ctx->t_derived;
    va.c = ctx->c;
    auto fn = ctx->sch.precision == BF_PRECISION_EXACT ? bf_exact::launch_viscous
                                                       : bf_fast::launch_viscous;
    CK(fn(va, ctx->n_visc_map, ctx->stream));
  }
  a.push = (vl && ctx->push_ok && push_enabled()) ? 1 : 0;
  a.push_rules = ctx->d_push;
  a.push_range = ctx->d_push_range;
  if (ctx->fuse_next) {   // this launch fills the ghosts of W[cur] (fused_fill_ok)
    a.fill = ghost_args(ctx, false);
    a.fill_ctas = fill_ctas_for(ctx);
    a.fill_chunks = 4 * ctx->nmap_fill;
    a.n_interior = ctx->n_fused_in;
    a.fill_sync = ctx->d_fill_sync;
    a.tile_list = ctx->d_tiles_fused;
    ctx->fuse_next = false;
  }
  // two launches only when they buy an overlap (NCCL messages in flight) or
  // when forced; the split costs tile-order L2 locality and a second tail
  const bool split = !a.fill_chunks && ctx->split_tiles &&
                     (ctx->split_forced || ctx->exchange_pending || ctx->fill_pending);
  {
    ProfScope ps(ctx, 0);
    if (!split) {
      CK(stage_fn(ctx)(ctx->ndim, ctx->sch.flux, ctx->sch.limiter, a, ctx->stream));
    } else {
      // interior tiles (no ghost they read is written this stage) on the main
      // stream; boundary tiles on the comm stream behind the ghost work queued
      // there (messages + unpack, or the hidden fill) — the two launches run
      // concurrently and join before anything that follows the stage
      if (!ctx->exchange_pending && !ctx->fill_pending) {   // forced split: ghosts in line
        CK(cudaEventRecord(ctx->ev_filled, ctx->stream));
        CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_filled, 0));
      }
      StageArgs b = a;
      b.tile_list = ctx->d_tiles_in;
      b.ntiles = ctx->n_tiles_in;
      if (b.ntiles) CK(stage_fn(ctx)(ctx->ndim, ctx->sch.flux, ctx->sch.limiter, b, ctx->stream));
      b.tile_list = ctx->d_tiles_bd;
      b.ntiles = ctx->n_tiles_bd;
      if (b.ntiles)
        CK(stage_fn(ctx)(ctx->ndim, ctx->sch.flux, ctx->sch.limiter, b, ctx->comm_stream));
      ps.kernels = (ctx->n_tiles_in > 0) + (ctx->n_tiles_bd > 0);
      CK(cudaEventRecord(ctx->ev_bd, ctx->comm_stream));
      CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_bd, 0));
      ctx->exchange_pending = false;
      ctx->fill_pending = false;
    }
  }
  if ((flags & F_STAGE0) && !ctx->batching) {   // batched: summed by the guard kernel
    ProfScope ps(ctx, 3);
    auto red = ctx->sch.precision == BF_PRECISION_EXACT ? bf_exact::launch_reduce
                                                        : bf_fast::launch_reduce;
    CK(red(ctx->d_partial, ctx->d_tile_begin, (int)ctx->blocks.size(), ctx->d_blocksum,
           ctx->stream));
  }
  if (flags & (F_PSI_STORE | F_PSI_LOAD)) ctx->psi_valid = true;
  ctx->pushed = a.push != 0;
  ctx->cur ^= 1;
  ctx->cur_epoch += 1;
  ctx->t_derived = 1;
  return BF_OK;
}

double rk_alpha(int nst, int k) {
  static const double a1[1] = {1.0};
  static const double a2[2] = {0.5, 1.0};
  static const double a4[4] = {0.25, 1.0 / 3.0, 0.5, 1.0};
  return nst == 1 ? a1[k] : (nst == 2 ? a2[k] : a4[k]);
}

// Decode the error key into the reference's numbering.
void decode_error(bf_ctx* ctx, unsigned long long key) {
  const int stage = (int)(key >> 61) & 7;
  const int phase = (int)(key >> 60) & 1;
  const int order = (int)(key >> 48) & 0xFFF;
  const int dir = (int)(key >> 46) & 3;
  const int kind = (int)(key >> 44) & 3;
  const unsigned long long lin = key & ((1ull << 44) - 1);
  const HostBlock& hb = ctx->blocks[order];
  long long sh[3] = {hb.n[0], hb.n[1], hb.n[2]};
  if (phase == 0) sh[dir] += 1;
  ctx->e_kind = phase ? BF_ERR_UPDATE : kind;
  ctx->e_block = hb.id;
  ctx->e_stage = stage;
  ctx->e_dir = dir;
  ctx->e_idx[2] = (long long)(lin % sh[2]);
  ctx->e_idx[1] = (long long)((lin / sh[2]) % sh[1]);
  ctx->e_idx[0] = (long long)(lin / sh[2] / sh[1]);
  ctx->msg = "non-physical state";
}

// Host copy of the per-block sums and the error key after a step: the copies
// (enqueue_collect, part of a captured step) and the host side (finish_collect).
int enqueue_collect(bf_ctx* ctx) {
  const int nb = (int)ctx->blocks.size();
  CK(cudaMemcpyAsync(ctx->h_pinned, ctx->d_blocksum, sizeof(double) * 5 * nb,
                     cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(ctx->h_pinned + 5 * nb, ctx->d_err, sizeof(unsigned long long),
                     cudaMemcpyDeviceToHost, ctx->stream));
  return BF_OK;
}

int finish_collect(bf_ctx* ctx, double* sumsq_out, unsigned long long* key_out);

int collect(bf_ctx* ctx, double* sumsq_out, unsigned long long* key_out) {
  int rc = enqueue_collect(ctx);
  if (rc) return rc;
  return finish_collect(ctx, sumsq_out, key_out);
}

int finish_collect(bf_ctx* ctx, double* sumsq_out, unsigned long long* key_out) {
  const int nb = (int)ctx->blocks.size();
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->profiling) drain_profile(ctx);
  double s[5] = {0, 0, 0, 0, 0};
  for (int b = 0; b < nb; ++b)
    for (int v = 0; v < 5; ++v) s[v] = s[v] + ctx->h_pinned[5 * b + v];   // id order
  for (int v = 0; v < 5; ++v) sumsq_out[v] = s[v];
  unsigned long long key;
  std::memcpy(&key, ctx->h_pinned + 5 * nb, sizeof key);
  *key_out = key;
  return BF_OK;
}

int reset_error(bf_ctx* ctx) {
  CK(cudaMemsetAsync(ctx->d_err, 0xFF, sizeof(unsigned long long), ctx->stream));
  return BF_OK;
}

int rank_allgather(bf_ctx* ctx, double* sumsq, unsigned long long* key, int* bad_rank) {
  // pack [5 sums, key bits] on the host side record, then allgather through NCCL
  double rec[6];
  for (int v = 0; v < 5; ++v) rec[v] = sumsq[v];
  std::memcpy(&rec[5], key, sizeof(double));
  CK(cudaMemcpyAsync(ctx->d_rank6, rec, sizeof rec, cudaMemcpyHostToDevice, ctx->stream));
  NK(net(ctx).AllGather(ctx->d_rank6, ctx->d_gather, 6, ncclDouble, ctx->comm, ctx->stream));
  std::vector<double> all((size_t)6 * ctx->nranks);
  CK(cudaMemcpyAsync(all.data(), ctx->d_gather, sizeof(double) * all.size(),
                     cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  double tot[5];
  for (int r = 0; r < ctx->nranks; ++r) {
    for (int v = 0; v < 5; ++v) tot[v] = (r == 0) ? all[6 * r + v] : tot[v] + all[6 * r + v];
  }
  for (int v = 0; v < 5; ++v) sumsq[v] = tot[v];
  *bad_rank = -1;
  for (int r = 0; r < ctx->nranks; ++r) {
    unsigned long long k;
    std::memcpy(&k, &all[6 * r + 5], sizeof k);
    if (k != NO_ERROR && *bad_rank < 0) *bad_rank = r;
  }
  return BF_OK;
}

}  // namespace

// =============================================================================
// C ABI
// =============================================================================
extern "C" {

int bf_api_version(void) { return BF_API_VERSION; }

bf_ctx* bf_create(int ndim, const bf_gas* gas, const bf_scheme* scheme, const bf_freestream* fs,
                  int device, int rank, int nranks) {
  if ((ndim != 2 && ndim != 3) || !gas || !scheme || !fs || nranks < 1 || rank < 0 ||
      rank >= nranks)
    return nullptr;
  auto* ctx = new bf_ctx();
  ctx->ndim = ndim;
  ctx->gas = *gas;
  ctx->sch = *scheme;
  ctx->fs = *fs;
  ctx->device = device;
  ctx->rank = rank;
  ctx->nranks = nranks;
  // k-chunk per tile: 32 for the cell-split / face-owner kernels (FAST, inviscid; C4 Van
  // Leer: 1.251 vs 1.273 ms at 16), 16 for the reference-order kernel (profiles/r01_kc_*.json)
  ctx->kc = (scheme->precision != BF_PRECISION_EXACT && !scheme->viscous) ? 32 : 16;
  if (const char* e = std::getenv("BF_KC")) ctx->kc = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("BF_NO_OVERLAP")) ctx->no_overlap = e[0] == '1';
  if (const char* e = std::getenv("BF_GRAPH")) ctx->graph_off = e[0] == '0';
  if (const char* e = std::getenv("BF_BATCH")) ctx->batch_off = e[0] == '0';
  if (const char* e = std::getenv("BF_FUSED_FILL")) ctx->fused_mode = e[0] == '0' ? 0 : 1;
  if (const char* e = std::getenv("BF_FILL_CTAS")) ctx->fill_ctas_env = std::atoi(e);
  if (const char* e = std::getenv("BF_PDL")) ctx->pdl_mode = e[0] == '0' ? 0 : 1;
  if (const char* e = std::getenv("BF_GHOST_INTERLEAVE")) ctx->ghost_interleave = e[0] != '0';
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device);
  if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&ctx->own_stream,
                                                                        cudaStreamNonBlocking) !=
                                                  cudaSuccess) {
    delete ctx;
    return nullptr;
  }
  ctx->stream = ctx->own_stream;
  device_ctx_opened(device);
  ctx->counted = true;
  // constants, in the reference's scalar evaluation order (python floats)
  Consts& c = ctx->c;
  const double g = gas->gamma;
  c.gamma = g;
  c.gm1 = g - 1.0;
  c.gog1 = g / (g - 1.0);
  c.R = gas->R;
  c.cfl = scheme->cfl;
  c.quarter = scheme->epsilon / 4.0;
  c.omk = 1.0 - scheme->kappa;
  c.opk = 1.0 + scheme->kappa;
  c.efix = scheme->entropy_fix_coeff;
  c.fs_rho = fs->rho;
  c.fs_u = fs->u;
  c.fs_v = fs->v;
  c.fs_w = fs->w;
  c.fs_p = fs->p;
  c.fs_T = fs->T;
  c.ff_af = std::sqrt(g * fs->p / fs->rho);
  c.ff_two_af_gm1 = 2.0 * c.ff_af / (g - 1.0);
  c.ff_sf = fs->p / std::pow(fs->rho, g);
  c.ff_qgm1 = 0.25 * (g - 1.0);
  c.ff_exp = 1.0 / (g - 1.0);
  c.two_over_gm1 = 2.0 / (g - 1.0);
  c.vl_c = 2.0 * (g * g - 1.0);
  c.inv_gamma = 1.0 / g;
  c.inv_vlc = 1.0 / c.vl_c;
  c.lim_eps = 1e-12;
  c.lim_eps_half = 0.5e-12;
  c.kappa_m1 = scheme->kappa == -1.0;
  c.viscous = scheme->viscous != 0;
  c.mu = gas->mu;
  c.prandtl = gas->prandtl > 0.0 ? gas->prandtl : 0.72;
  c.cp = g * gas->R / (g - 1.0);                     // physics.py:75-77
  c.has_suth = gas->has_sutherland != 0;
  c.suth_mu = gas->sutherland[0];
  c.suth_t = gas->sutherland[1];
  c.suth_s = gas->sutherland[2];
  c.visc_coeff = 2.0 * std::max(4.0 / 3.0, g / c.prandtl);   // solver.py:722
  c.tw = scheme->wall_temperature;
  c.has_tw = scheme->has_wall_temperature;
  c.eps0 = scheme->epsilon == 0.0;
  c.muscl_k1 = scheme->epsilon == 1.0 && scheme->kappa == -1.0;
  return ctx;
}

void bf_destroy(bf_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  // every stream that may still touch the arenas (an aborted overlapped step can
  // leave an unpack queued on comm_stream) drains before they are recycled
  cudaStreamSynchronize(ctx->stream);
  if (ctx->comm_stream) cudaStreamSynchronize(ctx->comm_stream);
  if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
  if (ctx->own_stream) cudaStreamSynchronize(ctx->own_stream);
  for (auto& hb : ctx->blocks)
    if (hb.d_bad) cudaFree(hb.d_bad);
  for (auto& b : ctx->staging) arena_free(ctx->device, b.first, b.second);
  ctx->staging.clear();
  for (auto& row : ctx->gexec)
    for (auto& ex : row)
      if (ex) cudaGraphExecDestroy(ex);
  for (auto& row : ctx->gexec_b)
    for (auto& ex : row)
      if (ex) cudaGraphExecDestroy(ex);
  cudaFree(ctx->d_run);
  cudaFree(ctx->d_hist);
  if (ctx->h_run) cudaFreeHost(ctx->h_run);
  for (auto& v : ctx->gprof)
    for (auto& p : v) {
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
  for (auto& v : ctx->gprof_b)
    for (auto& p : v) {
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
  // (the stream-ordered staging pool keeps its memory, like the arena cache:
  // bf_release_cache returns both)
  for (auto& hb : ctx->blocks) {
    for (double* p : hb.owned) arena_free(ctx->device, p, hb.arena_bytes);
    for (int f = 0; f < 6; ++f)
      if (hb.bface_d[f]) cudaFree(hb.bface_d[f]);
  }
  for (auto& L : ctx->links) {
    if (L.send) cudaFree(L.send);
    if (L.recv) cudaFree(L.recv);
  }
  for (double* p : ctx->dirichlet_d) cudaFree(p);
  cudaFree(ctx->d_blocks);
  cudaFree(ctx->d_tiles);
  cudaFree(ctx->d_tmaps);
  cudaFree(ctx->d_tile_begin);
  cudaFree(ctx->d_tasks_fill);
  cudaFree(ctx->d_tasks_unpack);
  cudaFree(ctx->d_map_fill);
  cudaFree(ctx->d_push);
  cudaFree(ctx->d_push_range);
  cudaFree(ctx->d_map_unpack);
  cudaFree(ctx->d_partial);
  cudaFree(ctx->d_blocksum);
  cudaFree(ctx->d_err);
  cudaFree(ctx->d_rank6);
  cudaFree(ctx->d_gather);
  if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
  for (auto& p : ctx->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  if (ctx->lb_rank) delete ctx->lb_rank;
  else if (ctx->comm) nccl().CommDestroy(ctx->comm);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->ev_filled) cudaEventDestroy(ctx->ev_filled);
  if (ctx->ev_unpacked) cudaEventDestroy(ctx->ev_unpacked);
  if (ctx->ev_bd) cudaEventDestroy(ctx->ev_bd);
  cudaFree(ctx->d_tiles_in);
  cudaFree(ctx->d_tiles_bd);
  cudaFree(ctx->d_tiles_fused);
  cudaFree(ctx->d_fill_sync);
  const int dev = ctx->device;
  const bool counted = ctx->counted;
  delete ctx;
  if (counted) device_ctx_closed(dev);
}

int bf_last_error(const bf_ctx* ctx, char* buf, size_t n) {
  if (!ctx || !buf || n == 0) return BF_EINVAL;
  std::snprintf(buf, n, "%s", ctx->msg.c_str());
  return BF_OK;
}

// A block's arenas go back to the cache on every error return of
// bf_add_block / bf_add_block_nodes until the block is committed to ctx->blocks.
struct BlockGuard {
  bf_ctx* ctx;
  HostBlock* hb;
  ~BlockGuard() {
    if (!hb || hb->owned.empty()) return;
    cudaStreamSynchronize(ctx->stream);
    for (double* p : hb->owned) arena_free(ctx->device, p, hb->arena_bytes);
    hb->owned.clear();
  }
  void commit() { hb = nullptr; }
};

// Arena allocation and device-block record shared by bf_add_block and
// bf_add_block_nodes (layout: bf_internal.h).
int add_block_arena(bf_ctx* ctx, int block_id, const int dims[3], int ghost_depth, bool has_src,
                    HostBlock& hb) {
  if (!ctx) return BF_EINVAL;
  if (ctx->finalized) return fail(ctx, BF_EINVAL, "bf_add_block after bf_finalize");
  if (ctx->index_of.count(block_id)) return fail(ctx, BF_EINVAL, "duplicate block %d", block_id);
  if (ghost_depth < 2) return fail(ctx, BF_EINVAL, "ghost_depth must be >= 2");
  const int ndim = ctx->ndim;
  if (dims[0] < 1 || dims[1] < 1 || dims[2] < 1 || (ndim == 2 && dims[2] != 1))
    return fail(ctx, BF_EINVAL, "bad dims (%d,%d,%d)", dims[0], dims[1], dims[2]);
  CK(cudaSetDevice(ctx->device));
  hb.id = block_id;
  for (int a = 0; a < 3; ++a) hb.n[a] = dims[a];
  hb.g = ghost_depth;
  hb.gk = ndim == 3 ? ghost_depth : 0;
  const int gg[3] = {hb.g, hb.g, hb.gk};
  for (int a = 0; a < 3; ++a) hb.P[a] = hb.n[a] + 2 * gg[a];
  hb.lead = (4 - hb.g % 4) % 4;
  hb.sy = ((hb.lead + hb.P[0] + 3) / 4) * 4;
  hb.sz = hb.sy * hb.P[1];
  hb.fsz = ((hb.sz * hb.P[2] + 63) / 64) * 64;
  hb.origin = hb.lead + hb.g + hb.sy * hb.g + hb.sz * hb.gk;
  hb.has_src = has_src;
  const bool want_psi = ctx->sch.limiter_freeze_at > 0;
  // arena slots (bf_internal.h): W 2x6 | Q 5 | dt/V | V | face geometry 3x4 |
  // [S*V 5] | [limiters ndim x 2 x 5]
  const int psi0 = want_psi ? FSRC + (hb.has_src ? 5 : 0) : -1;
  const bool visc = ctx->sch.viscous != 0;
  const int vis0 = visc ? FSRC + (hb.has_src ? 5 : 0) + (want_psi ? 10 * ndim : 0) : -1;
  const int nfield = FSRC + (hb.has_src ? 5 : 0) + (want_psi ? 10 * ndim : 0) + (visc ? NVIS : 0);
  int err = 0;
  hb.arena_bytes = sizeof(double) * (size_t)nfield * hb.fsz;
  hb.arena = static_cast<double*>(arena_alloc(ctx->device, hb.arena_bytes));
  if (!hb.arena)
    return fail(ctx, BF_ECUDA, "cudaMalloc(%zu bytes) failed for block %d", hb.arena_bytes,
                block_id);
  hb.owned.push_back(hb.arena);
  (void)err;
  // on the context's stream: the geometry kernels that follow run there
  CK(cudaMemsetAsync(hb.arena, 0, sizeof(double) * (size_t)nfield * hb.fsz, ctx->stream));
  DevBlock& d = hb.dev;
  for (int a = 0; a < 3; ++a) d.n[a] = hb.n[a];
  d.g = hb.g;
  d.ndim = ndim;
  d.id = block_id;
  d.sy = hb.sy;
  d.sz = hb.sz;
  d.fsz = hb.fsz;
  d.base = hb.arena + hb.origin;
  d.psi0 = psi0;
  d.vis0 = vis0;
  d.ox = (int)(hb.lead + hb.g);
  d.oy = hb.g;
  d.oz = hb.gk;
  hb.nslots = nfield;
  ctx->have_psi = want_psi;
  return BF_OK;
}

int bf_add_block(bf_ctx* ctx, int block_id, const int dims[3], int ghost_depth,
                 const double* const* face_vectors, const double* volume,
                 const double* const* source) {
  HostBlock hb;
  BlockGuard guard{ctx, &hb};
  int rc0 = add_block_arena(ctx, block_id, dims, ghost_depth, source != nullptr, hb);
  if (rc0) return rc0;
  const int ndim = ctx->ndim;
  const int gg[3] = {hb.g, hb.g, hb.gk};
  DevBlock& d = hb.dev;
  // face unit normals and areas (solver.py:212-220): the reference's face-vector
  // arrays go to the device as they are; a kernel normalises and scatters them.
  cudaStream_t st = ctx->stream;
  for (int dd = 0; dd < ndim; ++dd) {
    long long in_shape[3], ext[3];
    for (int a = 0; a < 3; ++a) {
      in_shape[a] = (a == dd) ? hb.n[a] + 1 : hb.P[a];
      ext[a] = in_shape[a];
    }
    const long long nin = in_shape[0] * in_shape[1] * in_shape[2];
    double* tmp = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), sizeof(double) * 3 * nin, st));
    for (int cc = 0; cc < 3; ++cc)
      CK(cudaMemcpyAsync(tmp + cc * nin, face_vectors[3 * dd + cc], sizeof(double) * nin,
                         cudaMemcpyHostToDevice, st));
    const long long nout = ext[0] * ext[1] * ext[2];
    face_normals_kernel<<<grid_for(nout), 256, 0, st>>>(
        d.f(ffn(dd, 0)) - hb.origin, hb.fsz, hb.sy, hb.sz, hb.origin, tmp, nin, dd, (int)ext[0],
        (int)ext[1], (int)ext[2], (int)in_shape[0], (int)in_shape[1], gg[0], gg[1], gg[2]);
    CK(cudaGetLastError());
    CK(cudaFreeAsync(tmp, st));
    ctx->bytes_h2d += 3LL * (long long)sizeof(double) * nin;
  }
  // volume + sources: interior Fortran (n0, n1, n2)
  auto put_interior = [&](double* dptr, const double* src) -> int {
    const long long n = (long long)hb.n[0] * hb.n[1] * hb.n[2];
    double* tmp = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), sizeof(double) * n, st));
    CK(cudaMemcpyAsync(tmp, src, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    scatter_box_kernel<<<grid_for(n), 256, 0, st>>>(dptr, hb.sy, hb.sz, 0, 0, 0, tmp, hb.n[0],
                                                    hb.n[1], hb.n[2]);
    CK(cudaGetLastError());
    CK(cudaFreeAsync(tmp, st));
    ctx->bytes_h2d += (long long)sizeof(double) * n;
    return BF_OK;
  };
  int rc = put_interior(d.f(FVOL), volume);
  if (rc) return rc;
  if (hb.has_src)
    for (int e = 0; e < 5; ++e) {
      rc = put_interior(d.f(FSRC + e), source[e]);
      if (rc) return rc;
    }
  CK(cudaStreamSynchronize(st));
  d.order = (int)ctx->blocks.size();
  ctx->index_of[block_id] = (int)ctx->blocks.size();
  guard.commit();
  ctx->blocks.push_back(std::move(hb));
  return BF_OK;
}

int bf_add_block_nodes(bf_ctx* ctx, int block_id, const int dims[3], int ghost_depth,
                       const double* const* nodes, const long long node_strides[3],
                       const double* const* source) {
  HostBlock hb;
  BlockGuard guard{ctx, &hb};
  {   // the strides must describe a dense array (C or Fortran order): checked
      // before anything is allocated
    if (!ctx) return BF_EINVAL;
    const int nd = ctx->ndim, g = ghost_depth;
    const long long ext[3] = {dims[0] + 2LL * g + 1, dims[1] + 2LL * g + 1,
                              nd == 3 ? dims[2] + 2LL * g + 1 : 1};
    const long long st[3] = {node_strides[0], node_strides[1], nd == 3 ? node_strides[2] : 0};
    long long span = 1;
    for (int a = 0; a < nd; ++a) span += (ext[a] - 1) * st[a];
    if (span != ext[0] * ext[1] * ext[2])
      return fail(ctx, BF_EINVAL, "node arrays must be dense (strides %lld %lld %lld)", st[0],
                  st[1], st[2]);
  }
  static const bool trace = std::getenv("BF_TRACE_BLOCKS") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "bf_add_block_nodes %d %-8s %8.3f ms\n", block_id, what,
                 std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
  int rc = add_block_arena(ctx, block_id, dims, ghost_depth, source != nullptr, hb);
  if (rc) return rc;
  mark("arena");
  const int ndim = ctx->ndim;
  DevBlock& d = hb.dev;
  cudaStream_t st = ctx->stream;
  // the node copy runs on the copy stream, beside this block's arena memset and
  // the previous block's metric kernels on ctx->stream (no host sync per block:
  // bf_sync_blocks checks the metric flags)
  if (!ctx->copy_stream) CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  cudaEvent_t ev = nullptr;
  CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  // padded node arrays (P0+1) x (P1+1) [x (P2+1)], Fortran order
  const long long N0 = hb.P[0] + 1, N1 = hb.P[1] + 1, N2 = ndim == 3 ? hb.P[2] + 1 : 1;
  const long long nn = N0 * N1 * N2;
  // node staging from the arena cache (no stream-ordered pool growth on the host
  // path of every block); back to the cache at bf_sync_blocks
  const size_t dn_bytes = sizeof(double) * ndim * nn;
  double* dn = static_cast<double*>(arena_alloc(ctx->device, dn_bytes));
  if (!dn) return fail(ctx, BF_ECUDA, "cudaMalloc(%zu bytes) failed for block %d nodes", dn_bytes, block_id);
  ctx->staging.push_back({dn, dn_bytes});
  for (int c = 0; c < ndim; ++c)
    CK(cudaMemcpyAsync(dn + c * nn, nodes[c], sizeof(double) * nn, cudaMemcpyHostToDevice,
                       ctx->copy_stream));
  mark("copy");
  CK(cudaEventRecord(ev, ctx->copy_stream));
  CK(cudaStreamWaitEvent(st, ev, 0));
  CK(cudaEventDestroy(ev));   // released once the recorded work completes
  ctx->bytes_h2d += (long long)sizeof(double) * ndim * nn;
  NodeView nv{dn, dn + nn, ndim == 3 ? dn + 2 * nn : nullptr, node_strides[0], node_strides[1],
              ndim == 3 ? node_strides[2] : 0};
  for (int dd = 0; dd < ndim; ++dd) {
    int ext[3], lo[3];
    const int gg[3] = {hb.g, hb.g, hb.gk};
    for (int a = 0; a < 3; ++a) {
      ext[a] = (a == dd) ? hb.n[a] + 1 : hb.P[a];
      lo[a] = (a == dd) ? 0 : -gg[a];
    }
    const long long nout = (long long)ext[0] * ext[1] * ext[2];
    metrics_faces_kernel<<<grid_for(nout), 256, 0, st>>>(
        d.f(ffn(dd, 0)) - hb.origin, hb.fsz, hb.sy, hb.sz, hb.origin, nv, ndim, dd, ext[0], ext[1],
        ext[2], hb.g, hb.gk, lo[0], lo[1], lo[2]);
    CK(cudaGetLastError());
  }
  unsigned long long* bad = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&bad), sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st));
  const long long ncell = (long long)hb.n[0] * hb.n[1] * hb.n[2];
  metrics_volume_kernel<<<grid_for(ncell), 256, 0, st>>>(d.f(FVOL), hb.sy, hb.sz, nv, ndim,
                                                         hb.n[0], hb.n[1], hb.n[2], hb.g, hb.gk,
                                                         bad);
  CK(cudaGetLastError());
  if (hb.has_src) {
    const long long n = ncell;
    double* tmp = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), sizeof(double) * n, st));
    for (int e = 0; e < 5; ++e) {
      CK(cudaMemcpyAsync(tmp, source[e], sizeof(double) * n, cudaMemcpyHostToDevice, st));
      scatter_box_kernel<<<grid_for(n), 256, 0, st>>>(d.f(FSRC + e), hb.sy, hb.sz, 0, 0, 0, tmp,
                                                      hb.n[0], hb.n[1], hb.n[2]);
      CK(cudaGetLastError());
      ctx->bytes_h2d += (long long)sizeof(double) * n;
    }
    CK(cudaFreeAsync(tmp, st));
  }
  mark("metrics");
  hb.d_bad = bad;   // inverted-cell flag, checked by bf_sync_blocks
  d.order = (int)ctx->blocks.size();
  ctx->index_of[block_id] = (int)ctx->blocks.size();
  guard.commit();
  ctx->blocks.push_back(std::move(hb));
  return BF_OK;
}

int bf_add_bc_patch(bf_ctx* ctx, int block_id, int bc_type, int face, const int box[6],
                    const double* dirichlet) {
  if (!ctx) return BF_EINVAL;
  if (ctx->finalized) return fail(ctx, BF_EINVAL, "bf_add_bc_patch after bf_finalize");
  if (!ctx->index_of.count(block_id)) return fail(ctx, BF_EINVAL, "unknown block %d", block_id);
  if (bc_type < 0 || bc_type > BC_MMS)
    return fail(ctx, BF_EINVAL, "unknown physical bc type %d", bc_type);
  if (face < 0 || face >= 2 * ctx->ndim) return fail(ctx, BF_EINVAL, "bad face %d", face);
  HostPatch p;
  p.block = block_id;
  p.type = bc_type;
  p.face = face;
  std::memcpy(p.box, box, sizeof p.box);
  const HostBlock& hb = ctx->blocks[ctx->index_of[block_id]];
  for (int a = 0; a < 3; ++a)
    if (box[2 * a] < 0 || box[2 * a + 1] > hb.n[a] || box[2 * a] >= box[2 * a + 1])
      return fail(ctx, BF_EINVAL, "patch box outside block %d", block_id);
  if (bc_type == BC_MMS) {
    if (!dirichlet) return fail(ctx, BF_EINVAL, "mms_dirichlet patch needs ghost values");
    const int ax = face / 2;
    long long nt = 1;
    for (int a = 0; a < 3; ++a)
      if (a != ax) nt *= box[2 * a + 1] - box[2 * a];
    p.dirichlet.assign(dirichlet, dirichlet + (size_t)hb.g * 6 * nt);
  }
  ctx->patches.push_back(std::move(p));
  return BF_OK;
}

int bf_add_bc_patch_ext(bf_ctx* ctx, int block_id, int bc_type, int face, const int box[6],
                        const double* dirichlet, const double* dirichlet_ext) {
  int rc = bf_add_bc_patch(ctx, block_id, bc_type, face, box, dirichlet);
  if (rc) return rc;
  if (bc_type == BC_MMS && dirichlet_ext) {
    const HostBlock& hb = ctx->blocks[ctx->index_of[block_id]];
    const int gg[3] = {hb.g, hb.g, ctx->ndim == 3 ? hb.g : 0};
    const int ax = face / 2;
    long long nt = 1;
    for (int a = 0; a < 3; ++a)
      if (a != ax) nt *= box[2 * a + 1] - box[2 * a] + 2 * gg[a];
    ctx->patches.back().dirichlet_ext.assign(dirichlet_ext, dirichlet_ext + (size_t)hb.g * 6 * nt);
  }
  return BF_OK;
}

int bf_add_viscous_geometry(bf_ctx* ctx, int block_id, const double* const* grad_invT) {
  if (!ctx) return BF_EINVAL;
  if (!ctx->sch.viscous) return fail(ctx, BF_EINVAL, "bf_add_viscous_geometry on an inviscid ctx");
  if (!ctx->index_of.count(block_id)) return fail(ctx, BF_EINVAL, "unknown block %d", block_id);
  CK(cudaSetDevice(ctx->device));
  HostBlock& hb = ctx->blocks[ctx->index_of[block_id]];
  DevBlock& d = hb.dev;
  cudaStream_t st = ctx->stream;
  for (int dd = 0; dd < ctx->ndim; ++dd) {
    int ext[3];
    for (int a = 0; a < 3; ++a) ext[a] = (a == dd) ? hb.n[a] + 1 : hb.n[a];
    const long long n = (long long)ext[0] * ext[1] * ext[2];
    double* tmp = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), sizeof(double) * n, st));
    for (int m = 0; m < 9; ++m) {
      const double* src = grad_invT[9 * dd + m];
      if (!src) continue;   // zero (arena is zero-initialised)
      CK(cudaMemcpyAsync(tmp, src, sizeof(double) * n, cudaMemcpyHostToDevice, st));
      scatter_box_kernel<<<grid_for(n), 256, 0, st>>>(d.f(d.vis0 + 9 * dd + m), hb.sy, hb.sz, 0, 0,
                                                      0, tmp, ext[0], ext[1], ext[2]);
      CK(cudaGetLastError());
      ctx->bytes_h2d += (long long)sizeof(double) * n;
    }
    CK(cudaFreeAsync(tmp, st));
  }
  CK(cudaStreamSynchronize(st));
  ctx->visc_geometry.insert(block_id);
  return BF_OK;
}

int bf_set_round2_order(bf_ctx* ctx, int nlinks, const int* order) {
  if (!ctx) return BF_EINVAL;
  if (ctx->finalized) return fail(ctx, BF_EINVAL, "bf_set_round2_order after bf_finalize");
  if (nlinks != (int)ctx->links.size())
    return fail(ctx, BF_EINVAL, "round-2 order for %d links, ctx has %zu", nlinks,
                ctx->links.size());
  for (int q = 0; q < nlinks; ++q) ctx->links[q].order2 = order[q];
  return BF_OK;
}

int bf_add_link(bf_ctx* ctx, int block_id, int face, const int box[6], const int axis_map[6],
                int peer_block, int peer_face, const int peer_box[6], int peer_rank, int tag) {
  if (!ctx) return BF_EINVAL;
  if (ctx->finalized) return fail(ctx, BF_EINVAL, "bf_add_link after bf_finalize");
  if (!ctx->index_of.count(block_id)) return fail(ctx, BF_EINVAL, "unknown block %d", block_id);
  if (peer_rank < 0 || peer_rank >= ctx->nranks)
    return fail(ctx, BF_EINVAL, "peer rank %d out of range", peer_rank);
  HostLink L;
  L.block = block_id;
  L.face = face;
  std::memcpy(L.box, box, sizeof L.box);
  std::memcpy(L.amap, axis_map, sizeof L.amap);
  L.peer_block = peer_block;
  L.peer_face = peer_face;
  std::memcpy(L.peer_box, peer_box, sizeof L.peer_box);
  L.peer_rank = peer_rank;
  L.tag = tag;
  bool seen[3] = {false, false, false};
  for (int a = 0; a < 3; ++a) {
    if (axis_map[2 * a] < 0 || axis_map[2 * a] > 2 || seen[axis_map[2 * a]])
      return fail(ctx, BF_EINVAL, "orientation map is not a bijection");
    seen[axis_map[2 * a]] = true;
  }
  ctx->links.push_back(L);
  return BF_OK;
}

int bf_sync_blocks(bf_ctx* ctx) {
  if (!ctx) return BF_EINVAL;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  for (auto& b : ctx->staging) arena_free(ctx->device, b.first, b.second);
  ctx->staging.clear();
  int rc = BF_OK;
  for (HostBlock& hb : ctx->blocks) {
    if (!hb.d_bad) continue;
    unsigned long long bad = ~0ull;
    CK(cudaMemcpy(&bad, hb.d_bad, sizeof bad, cudaMemcpyDeviceToHost));
    CK(cudaFree(hb.d_bad));
    hb.d_bad = nullptr;
    if (bad != ~0ull && rc == BF_OK) {
      const unsigned long long k = bad % (unsigned long long)hb.n[2];
      const unsigned long long r = bad / (unsigned long long)hb.n[2];
      const unsigned long long j = r % (unsigned long long)hb.n[1], i = r / (unsigned long long)hb.n[1];
      rc = fail(ctx, BF_EMETRIC, "block %d: inverted cell at interior index (%llu, %llu, %llu)",
                hb.id, i, j, k);
    }
  }
  return rc;
}

int bf_finalize(bf_ctx* ctx) {
  if (!ctx) return BF_EINVAL;
  if (ctx->finalized) return BF_OK;
  if (int rc0 = bf_sync_blocks(ctx)) return rc0;
  static const bool trace = std::getenv("BF_TRACE_FINALIZE") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "bf_finalize %-12s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
  CK(cudaSetDevice(ctx->device));
  if (ctx->sch.viscous)
    for (auto& hb : ctx->blocks)
      if (!ctx->visc_geometry.count(hb.id))
        return fail(ctx, BF_EINVAL, "viscous run: block %d has no bf_add_viscous_geometry", hb.id);
  int rc = build_tables(ctx);
  if (rc) return rc;
  mark("tables");
  rc = build_push(ctx);
  if (rc) return rc;
  mark("push");
  if (ctx->sch.viscous) {
    rc = build_round2(ctx);
    if (rc) return rc;
    std::vector<ViscTask> vt;
    std::vector<int2> vm;
    for (size_t bi = 0; bi < ctx->blocks.size(); ++bi)
      for (int d = 0; d < ctx->ndim; ++d) {
        const HostBlock& hb = ctx->blocks[bi];
        ViscTask t{};
        t.block = (int)bi;
        t.d = d;
        for (int a = 0; a < 3; ++a) t.e[a] = (a == d) ? hb.n[a] + 1 : hb.n[a];
        t.items = (long long)t.e[0] * t.e[1] * t.e[2];
        for (long long it = 0; it < t.items; it += 128)
          vm.push_back(make_int2((int)vt.size(), (int)it));
        vt.push_back(t);
      }
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(vt.size(), 1) * sizeof(ViscTask)));
    CK(cudaMemcpy(p, vt.data(), vt.size() * sizeof(ViscTask), cudaMemcpyHostToDevice));
    ctx->d_visc = static_cast<ViscTask*>(p);
    CK(cudaMalloc(&p, std::max<size_t>(vm.size(), 1) * sizeof(int2)));
    CK(cudaMemcpy(p, vm.data(), vm.size() * sizeof(int2), cudaMemcpyHostToDevice));
    ctx->d_visc_map = static_cast<int2*>(p);
    ctx->n_visc_map = (int)vm.size();
  }
  rc = build_tiles(ctx);
  if (rc) return rc;
  mark("tiles");
  rc = build_tensor_maps(ctx);
  if (rc) return rc;
  mark("tmaps");
  std::vector<DevBlock> devs;
  for (auto& hb : ctx->blocks) devs.push_back(hb.dev);
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(devs.size(), 1) * sizeof(DevBlock)));
  CK(cudaMemcpy(p, devs.data(), devs.size() * sizeof(DevBlock), cudaMemcpyHostToDevice));
  ctx->d_blocks = static_cast<DevBlock*>(p);
  CK(cudaMalloc(&p, sizeof(double) * 5 * std::max(ctx->ntiles, 1)));
  ctx->d_partial = static_cast<double*>(p);
  CK(cudaMalloc(&p, sizeof(double) * 5 * std::max<size_t>(ctx->blocks.size(), 1)));
  ctx->d_blocksum = static_cast<double*>(p);
  CK(cudaMalloc(&p, sizeof(unsigned long long)));
  ctx->d_err = static_cast<unsigned long long*>(p);
  CK(cudaMemset(ctx->d_err, 0xFF, sizeof(unsigned long long)));
  CK(cudaMalloc(&p, sizeof(double) * 6));
  ctx->d_rank6 = static_cast<double*>(p);
  CK(cudaMalloc(&p, sizeof(double) * 6 * ctx->nranks));
  ctx->d_gather = static_cast<double*>(p);
  CK(cudaMallocHost(&p, sizeof(double) * (5 * ctx->blocks.size() + 2)));
  ctx->h_pinned = static_cast<double*>(p);
  mark("buffers");
  ctx->finalized = true;
  return BF_OK;
}

int bf_upload_fields(bf_ctx* ctx, int block_id, const double* const* fields6,
                     const double* const* q5) {
  if (!ctx || !ctx->finalized) return fail(ctx, BF_EINVAL, "bf_upload_fields before bf_finalize");
  if (!ctx->index_of.count(block_id)) return fail(ctx, BF_EINVAL, "unknown block %d", block_id);
  CK(cudaSetDevice(ctx->device));
  HostBlock& hb = ctx->blocks[ctx->index_of[block_id]];
  // padded Fortran arrays go to the device contiguously; a kernel restrides them
  const long long np = (long long)hb.P[0] * hb.P[1] * hb.P[2];
  double* tmp = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), sizeof(double) * np, ctx->stream));
  auto put = [&](double* dptr, const double* src) -> int {
    CK(cudaMemcpyAsync(tmp, src, sizeof(double) * np, cudaMemcpyHostToDevice, ctx->stream));
    scatter_box_kernel<<<grid_for(np), 256, 0, ctx->stream>>>(
        dptr - hb.origin + hb.lead, hb.sy, hb.sz, 0, 0, 0, tmp, hb.P[0], hb.P[1], hb.P[2]);
    CK(cudaGetLastError());
    ctx->bytes_h2d += (long long)sizeof(double) * np;
    return BF_OK;
  };
  for (int f = 0; f < 6; ++f) {
    int rc = put(hb.dev.f(fw(0, f)), fields6[f]);
    if (rc) return rc;
    CK(cudaMemcpyAsync(hb.dev.f(fw(1, f)) - hb.origin, hb.dev.f(fw(0, f)) - hb.origin,
                       sizeof(double) * hb.fsz, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  if (q5) {
    for (int e = 0; e < 5; ++e) {
      int rc = put(hb.dev.f(FQ + e), q5[e]);
      if (rc) return rc;
    }
  } else {   // sync_conserved on the device (solver.py:273-277)
    encode_kernel<<<grid_for(hb.fsz), 256, 0, ctx->stream>>>(
        hb.dev.f(fw(0, 0)) - hb.origin, hb.dev.f(FQ) - hb.origin, hb.fsz, hb.fsz,
        ctx->gas.gamma - 1.0);
    CK(cudaGetLastError());
  }
  CK(cudaFreeAsync(tmp, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->cur = 0;
  ctx->ghost_buf = 0;
  ctx->t_derived = 0;
  ctx->psi_valid = false;
  ctx->pushed = false;
  ctx->other_filled = false;
  return BF_OK;
}

int bf_update_ghosts(bf_ctx* ctx) {
  if (!ctx || !ctx->finalized) return fail(ctx, BF_EINVAL, "bf_update_ghosts before bf_finalize");
  CK(cudaSetDevice(ctx->device));
  int rc = ghosts_solo(ctx);
  if (rc) return rc;
  if (ctx->exchange_pending || ctx->fill_pending) {   // ghosts still landing on comm_stream
    CK(cudaEventRecord(ctx->ev_unpacked, ctx->comm_stream));
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_unpacked, 0));
    ctx->exchange_pending = ctx->fill_pending = false;
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return BF_OK;
}

// Programmatic dependent launch for this context's kernels (bf_kernels.cu
// launch_pdl): on when the stage grid is one wave (launch latency dominates).
void use_pdl(const bf_ctx* ctx) {
  const int on = ctx->pdl_mode < 0 ? (ctx->ntiles <= ctx->num_sms ? 1 : 0) : ctx->pdl_mode;
  bf_exact::set_pdl(on);
  bf_fast::set_pdl(on);
}

// The device work of one RK step (solver.py:786-814) on ctx->stream, up to the
// copies of its residual sums and error key.
int enqueue_step(bf_ctx* ctx, int step_index) {
  const int nst = ctx->sch.rk_stages;
  use_pdl(ctx);
  // batched: the guard kernel resets it
  int rc = (ctx->batching || ctx->mr_batching) ? BF_OK : reset_error(ctx);
  if (rc) return rc;
  for (int k = 0; k < nst; ++k) {
    const int flags = stage_flags(ctx, step_index, k, nst);
    if (fused_fill_ok(ctx, flags)) {   // the stage launch fills the ghosts itself
      ctx->fuse_next = true;
      ctx->ghost_buf = ctx->cur;
    } else {
      rc = ghosts_solo(ctx);
      if (rc) return rc;
    }
    rc = launch_stage_kernel(ctx, k, flags, rk_alpha(nst, k));
    if (rc) return rc;
  }
  if (ctx->mr_batching) {   // rank record -> allgather -> global norms and guards, on the device
    ProfScope ps(ctx, 3);
    CK(bf_exact::launch_rank_record(ctx->d_blocksum, (int)ctx->blocks.size(), ctx->d_err,
                                    ctx->d_rank6, ctx->d_run, ctx->stream));
    NK(net(ctx).AllGather(ctx->d_rank6, ctx->d_gather, 6, ncclDouble, ctx->comm, ctx->stream));
    CK(bf_exact::launch_rank_guard(ctx->d_gather, ctx->nranks, ctx->rank, ctx->d_err, ctx->d_run,
                                   ctx->d_hist, ctx->stream));
    return BF_OK;
  }
  if (ctx->batching) {   // norms and guards on the device (RunState)
    ProfScope ps(ctx, 3);
    CK(bf_exact::launch_guard(ctx->d_partial, ctx->d_tile_begin, (int)ctx->blocks.size(),
                              ctx->d_blocksum, ctx->d_err, ctx->d_run, ctx->d_hist,
                              ctx->d_fill_sync ? ctx->d_fill_sync + 3 : nullptr, ctx->stream));
    return BF_OK;
  }
  return enqueue_collect(ctx);
}

// Host-side sequencing state a step advances (buffer parity, epochs).
struct StepState {
  int cur, ghost_buf, t_derived;
  long long cur_epoch;
  bool pushed, psi_valid, other_filled, exchange_pending, fill_pending;
  bool operator==(const StepState& o) const {
    return cur == o.cur && ghost_buf == o.ghost_buf && t_derived == o.t_derived &&
           cur_epoch == o.cur_epoch && pushed == o.pushed && psi_valid == o.psi_valid &&
           other_filled == o.other_filled && exchange_pending == o.exchange_pending &&
           fill_pending == o.fill_pending;
  }
};
StepState save_state(const bf_ctx* ctx) {
  return {ctx->cur, ctx->ghost_buf, ctx->t_derived, ctx->cur_epoch,
          ctx->pushed, ctx->psi_valid, ctx->other_filled, ctx->exchange_pending,
          ctx->fill_pending};
}
void load_state(bf_ctx* ctx, const StepState& st) {
  ctx->cur = st.cur;
  ctx->ghost_buf = st.ghost_buf;
  ctx->t_derived = st.t_derived;
  ctx->cur_epoch = st.cur_epoch;
  ctx->pushed = st.pushed;
  ctx->psi_valid = st.psi_valid;
  ctx->other_filled = st.other_filled;
  ctx->exchange_pending = st.exchange_pending;
  ctx->fill_pending = st.fill_pending;
}
// What a graph-eligible step does to that state: per stage, ghosts of W[cur]
// then the buffer swap.
StepState advanced(StepState st, int nst) {
  for (int k = 0; k < nst; ++k) {
    st.ghost_buf = st.cur;
    st.cur ^= 1;
    st.cur_epoch += 1;
  }
  st.t_derived = 1;
  return st;
}

// A step is replayed from a CUDA graph when its launches are the same every
// step: one rank, inviscid, no thin-block BC ordering, no limiter freeze, no
// in-kernel push or forced tile split, past the first stage (T derived, both
// buffers' constant ghosts present).
bool graph_eligible(const bf_ctx* ctx) {
  return !ctx->graph_off && ctx->nranks == 1 && !ctx->comm &&
         !ctx->group && !ctx->sch.viscous && ctx->r1_bc.empty() &&
         ctx->sch.limiter_freeze_at <= 0 && ctx->t_derived && ctx->other_filled &&
         !ctx->pushed && !(ctx->push_ok && push_enabled()) && !ctx->split_forced &&
         ctx->n_unpack == 0;
}

// Enqueue one step through its graph (captured on first use for this starting
// buffer).  Returns 1 when the caller must take the plain path instead.
int enqueue_step_graph(bf_ctx* ctx, int step_index) {
  const int nst = ctx->sch.rk_stages;
  const StepState before = save_state(ctx);
  const int c0 = ctx->cur, pr = ctx->profiling ? 1 : 0;
  auto& gexec = ctx->batching ? ctx->gexec_b : ctx->gexec;
  auto& gprof = ctx->batching ? ctx->gprof_b : ctx->gprof;
  if (!gexec[c0][pr]) {
    cudaGraph_t g = nullptr;
    const size_t npend = ctx->pending.size();
    if (cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      ctx->graph_off = true;
      return 1;
    }
    ctx->capturing = true;
    const int rc = enqueue_step(ctx, step_index);
    ctx->capturing = false;
    const cudaError_t ce = cudaStreamEndCapture(ctx->stream, &g);
    const StepState after = save_state(ctx);
    load_state(ctx, before);
    cudaGetLastError();
    cudaGraphExec_t ex = nullptr;
    const bool ok = rc == BF_OK && ce == cudaSuccess && g &&
                    after == advanced(before, nst) &&
                    cudaGraphInstantiate(&ex, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    // timing events recorded during the capture belong to the graph
    std::vector<TimerPair> captured(ctx->pending.begin() + npend, ctx->pending.end());
    ctx->pending.resize(npend);
    if (!ok) {
      cudaGetLastError();
      for (auto& p : captured) {
        ctx->event_pool.push_back(p.a);
        ctx->event_pool.push_back(p.b);
      }
      ctx->graph_off = true;
      return 1;
    }
    for (auto& p : captured) p.owned_by_graph = true;
    if (pr) gprof[c0] = captured;
    gexec[c0][pr] = ex;
  }
  CK(cudaGraphLaunch(gexec[c0][pr], ctx->stream));
  if (pr) ctx->pending.insert(ctx->pending.end(), gprof[c0].begin(), gprof[c0].end());
  load_state(ctx, advanced(before, nst));
  return BF_OK;
}

int bf_step(bf_ctx* ctx, int step_index, double* sumsq_out, long long* ncells_out) {
  if (!ctx || !ctx->finalized) return fail(ctx, BF_EINVAL, "bf_step before bf_finalize");
  CK(cudaSetDevice(ctx->device));
  int rc = 1;
  if (graph_eligible(ctx)) rc = enqueue_step_graph(ctx, step_index);
  if (rc == 1) rc = enqueue_step(ctx, step_index);
  if (rc) return rc;
  double s[5];
  unsigned long long key;
  rc = finish_collect(ctx, s, &key);
  if (rc) return rc;
  if (ctx->comm && ctx->nranks > 1) {
    int bad = -1;
    rc = rank_allgather(ctx, s, &key, &bad);
    if (rc) return rc;
    if (bad >= 0 && key == NO_ERROR)
      return fail(ctx, BF_ENONPHYSICAL, "rank %d: non-physical state", bad);
  }
  if (key != NO_ERROR && !ignore_errors()) {
    decode_error(ctx, key);
    return BF_ENONPHYSICAL;
  }
  for (int v = 0; v < 5; ++v) sumsq_out[v] = s[v];
  if (ncells_out) {
    long long n = 0;
    for (auto& hb : ctx->blocks) n += hb.cells();
    *ncells_out = n;
  }
  return BF_OK;
}

int bf_run(bf_ctx* ctx, int first_step, int nsteps, double* hist_out, int* steps_done) {
  if (!ctx || !ctx->finalized) return fail(ctx, BF_EINVAL, "bf_run before bf_finalize");
  *steps_done = 0;
  for (int s = 0; s < nsteps; ++s) {
    double ss[5];
    int rc = bf_step(ctx, first_step + s, ss, nullptr);
    if (rc) return rc;
    for (int v = 0; v < 5; ++v) hist_out[5 * s + v] = std::sqrt(ss[v]);
    *steps_done = s + 1;
  }
  return BF_OK;
}

// check_history_guards (solver.py:836-855) on the norms of step `step`:
// 0 continue, 1 converged (floor / target reached), 2 diverged (the caller
// raises).  numpy semantics: max propagates NaN, comparisons with NaN fail.
static int history_guard(const double* hist, int step, int has_target, double target,
                         int has_floor, double floor_, double factor) {
  auto npmax = [](const double* x) {
    double m = x[0];
    for (int v = 1; v < 5; ++v)
      if (std::isnan(x[v]) || x[v] > m || std::isnan(m)) m = std::isnan(m) ? m : x[v];
    return m;
  };
  const double* h = hist + 5 * (size_t)step;
  if (has_floor && npmax(h) <= floor_) return 1;
  const double* b = hist;
  const double bmax = npmax(b);
  bool any = false, bad = false;
  double rmax = 0.0;
  for (int v = 0; v < 5; ++v) {
    if (!(b[v] > 1e-12 * bmax)) continue;
    const double r = h[v] / b[v];
    if (!std::isfinite(r)) bad = true;
    rmax = any ? (r > rmax ? r : rmax) : r;
    any = true;
  }
  if (!any) return 0;
  if (bad || rmax > factor) return 2;
  return (has_target && rmax <= target) ? 1 : 0;
}

constexpr int BATCH_MAX = 256;   // steps per batch (device history rows)

// Steps first_step .. first_step + n - 1 enqueued back to back through the
// batched graphs; the guard kernel of each step stops the rest of the batch
// (RunState).  Host sequencing state follows the steps the device executed.
static int run_batch(bf_ctx* ctx, int first_step, int n, int call_step, int has_target,
                     double target, int has_floor, double floor_, double factor,
                     double* hist_out, int* done, int* status, bool multi_rank = false) {
  if (!ctx->d_run) {
    void* p = nullptr;
    CK(cudaMalloc(&p, sizeof(RunState)));
    ctx->d_run = static_cast<RunState*>(p);
    CK(cudaMalloc(&p, sizeof(double) * 5 * BATCH_MAX));
    ctx->d_hist = static_cast<double*>(p);
    CK(cudaMallocHost(&p, sizeof(RunState) + sizeof(double) * 5 * BATCH_MAX));
    ctx->h_run = p;
  }
  RunState* hr = static_cast<RunState*>(ctx->h_run);
  std::memset(hr, 0, sizeof(RunState));
  hr->has_base = call_step > 0;
  if (call_step > 0)
    for (int v = 0; v < 5; ++v) hr->base[v] = hist_out[v];
  hr->has_target = has_target;
  hr->target = target;
  hr->has_floor = has_floor;
  hr->floor_ = floor_;
  hr->factor = factor;
  hr->ignore_errors = ignore_errors() ? 1 : 0;
  CK(cudaMemcpyAsync(ctx->d_run, hr, sizeof(RunState), cudaMemcpyHostToDevice, ctx->stream));
  {   // first step of the batch (later ones: the guard kernel)
    const int r0 = reset_error(ctx);
    if (r0) return r0;
  }
  const StepState before = save_state(ctx);
  int rc = BF_OK;
  if (multi_rank) {   // every rank enqueues the same n steps: the exchanges stay matched
    ctx->mr_batching = true;
    for (int q = 0; q < n && rc == BF_OK; ++q) rc = enqueue_step(ctx, first_step + q);
    ctx->mr_batching = false;
  } else {
    ctx->batching = true;
    for (int q = 0; q < n && rc == BF_OK; ++q) {
      rc = enqueue_step_graph(ctx, first_step + q);
      if (rc == 1) rc = fail(ctx, BF_EINVAL, "batched step graph unavailable");
    }
    ctx->batching = false;
  }
  if (rc) return rc;
  double* hh = reinterpret_cast<double*>(hr + 1);
  CK(cudaMemcpyAsync(hr, ctx->d_run, sizeof(RunState), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(hh, ctx->d_hist, sizeof(double) * 5 * n, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->profiling) drain_profile(ctx);
  const int ran = hr->steps + (hr->status == 3 ? 1 : 0);   // the failing step ran too
  if (!multi_rank || ran < n) {   // host bookkeeping of the steps the device executed
    const bool filled = multi_rank ? (before.other_filled || ran > 0) : before.other_filled;
    StepState st = before;
    for (int q = 0; q < ran; ++q) st = advanced(st, ctx->sch.rk_stages);
    st.other_filled = filled;
    load_state(ctx, st);
  }
  for (int q = 0; q < hr->steps; ++q)
    for (int v = 0; v < 5; ++v) hist_out[5 * (call_step + q) + v] = hh[5 * q + v];
  *done = hr->steps;
  *status = hr->status;
  if (hr->status == 3) {
    if (hr->key == NO_ERROR)   // another rank's state (bf_step's rank_allgather message)
      return fail(ctx, BF_ENONPHYSICAL, "rank %d: non-physical state", hr->bad_rank);
    decode_error(ctx, hr->key);
    return BF_ENONPHYSICAL;
  }
  return BF_OK;
}

// Multi-rank contexts whose steps can run back to back with the norms and
// guards on the device: the rank record is allgathered on the stream (NCCL or
// loopback), every rank evaluates the same global guards, so every rank stops
// after the same step and the remaining launches of the batch are no-ops.
bool mr_batch_eligible(const bf_ctx* ctx) {
  return ctx->comm && ctx->nranks > 1 && !ctx->group && !ctx->sch.viscous &&
         ctx->r1_bc.empty() && ctx->sch.limiter_freeze_at <= 0 &&
         !(ctx->push_ok && push_enabled());
}

int bf_iterate(bf_ctx* ctx, int first_step, int max_steps, int has_target, double target,
               int has_floor, double floor_, double divergence_factor, double* hist_out,
               int* steps_done, int* status) {
  if (!ctx || !ctx->finalized) return fail(ctx, BF_EINVAL, "bf_iterate before bf_finalize");
  CK(cudaSetDevice(ctx->device));
  *steps_done = 0;
  *status = 0;
  int s = 0;
  while (s < max_steps) {
    const bool mr = !ctx->batch_off && mr_batch_eligible(ctx);
    if (!ctx->batch_off && (graph_eligible(ctx) || mr)) {
      // device-side guards: no host round trip per step
      const int n = std::min(max_steps - s, BATCH_MAX);
      int done = 0, st = 0;
      const int rc = run_batch(ctx, first_step + s, n, s, has_target, target, has_floor, floor_,
                               divergence_factor, hist_out, &done, &st, mr);
      s += done;
      *steps_done = s;
      if (rc) return rc;
      if (st) {
        *status = st;
        break;
      }
      continue;
    }
    double ss[5];
    int rc = bf_step(ctx, first_step + s, ss, nullptr);
    if (rc) return rc;
    for (int v = 0; v < 5; ++v) hist_out[5 * s + v] = std::sqrt(ss[v]);
    *steps_done = s + 1;
    const int g = history_guard(hist_out, s, has_target, target, has_floor, floor_,
                                divergence_factor);
    ++s;
    if (g) {
      *status = g;
      break;
    }
  }
  return BF_OK;
}

int bf_download(bf_ctx* ctx, int block_id, int what, double* out) {
  if (!ctx || !ctx->finalized) return fail(ctx, BF_EINVAL, "bf_download before bf_finalize");
  if (!ctx->index_of.count(block_id)) return fail(ctx, BF_EINVAL, "unknown block %d", block_id);
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  const HostBlock& hb = ctx->blocks[ctx->index_of[block_id]];
  std::vector<double> a, b;
  auto get = [&](const double* dptr, std::vector<double>& h) -> int {
    h.resize((size_t)hb.fsz);
    CK(cudaMemcpy(h.data(), dptr - hb.origin, sizeof(double) * hb.fsz, cudaMemcpyDeviceToHost));
    ctx->bytes_d2h += (long long)sizeof(double) * hb.fsz;
    return BF_OK;
  };
  auto at = [&](long long i, long long j, long long k) {   // padded coords
    return hb.lead + i + hb.sy * j + hb.sz * k;
  };
  const int gg[3] = {hb.g, hb.g, hb.gk};
  auto interior = [&](long long i, long long j, long long k) {
    return i >= gg[0] && i < gg[0] + hb.n[0] && j >= gg[1] && j < gg[1] + hb.n[1] &&
           k >= gg[2] && k < gg[2] + hb.n[2];
  };
  int rc;
  if (what >= BF_FIELD_RHO && what <= BF_FIELD_T) {
    const long long np = (long long)hb.P[0] * hb.P[1] * hb.P[2];
    double* tmp = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), sizeof(double) * np, ctx->stream));
    const int derived = (what == BF_FIELD_T && ctx->t_derived) ? 1 : 0;
    merge_field_kernel<<<grid_for(np), 256, 0, ctx->stream>>>(
        tmp, hb.dev.f(fw(ctx->cur, what)) - hb.origin,
        hb.dev.f(fw(ctx->ghost_buf, what)) - hb.origin, hb.dev.f(fw(ctx->cur, 0)) - hb.origin,
        hb.dev.f(fw(ctx->cur, 4)) - hb.origin, derived, ctx->gas.R, hb.sy, hb.sz, hb.lead, gg[0],
        gg[1], gg[2], hb.n[0], hb.n[1], hb.n[2], hb.P[0], hb.P[1], hb.P[2]);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, tmp, sizeof(double) * np, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaFreeAsync(tmp, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->bytes_d2h += (long long)sizeof(double) * np;
    (void)a;
    (void)b;
    (void)at;
    (void)interior;
    return BF_OK;
  }
  if (what >= BF_FIELD_Q0 && what <= BF_FIELD_Q0 + 4) {
    rc = get(hb.dev.f(FQ + what - BF_FIELD_Q0), a);
    if (rc) return rc;
    for (long long k = 0; k < hb.P[2]; ++k)
      for (long long j = 0; j < hb.P[1]; ++j)
        for (long long i = 0; i < hb.P[0]; ++i)
          out[i + hb.P[0] * (j + (long long)hb.P[1] * k)] = a[at(i, j, k)];
    return BF_OK;
  }
  if (what == BF_FIELD_DTV) {
    rc = get(hb.dev.f(FDTV), a);
    if (rc) return rc;
    for (long long k = 0; k < hb.n[2]; ++k)
      for (long long j = 0; j < hb.n[1]; ++j)
        for (long long i = 0; i < hb.n[0]; ++i)
          out[i + hb.n[0] * (j + (long long)hb.n[1] * k)] =
              a[hb.origin + hb.off((int)i, (int)j, (int)k)];
    return BF_OK;
  }
  if (what == BF_FIELD_VOL) {
    rc = get(hb.dev.f(FVOL), a);
    if (rc) return rc;
    for (long long k = 0; k < hb.n[2]; ++k)
      for (long long j = 0; j < hb.n[1]; ++j)
        for (long long i = 0; i < hb.n[0]; ++i)
          out[i + hb.n[0] * (j + (long long)hb.n[1] * k)] =
              a[hb.origin + hb.off((int)i, (int)j, (int)k)];
    return BF_OK;
  }
  if (what >= BF_FIELD_FACE && what < BF_FIELD_FACE + 4 * ctx->ndim) {
    const int d = (what - BF_FIELD_FACE) / 4, cc = (what - BF_FIELD_FACE) % 4;
    rc = get(hb.dev.f(ffn(d, cc)), a);
    if (rc) return rc;
    long long ext[3] = {hb.n[0], hb.n[1], hb.n[2]};
    ext[d] += 1;
    for (long long k = 0; k < ext[2]; ++k)
      for (long long j = 0; j < ext[1]; ++j)
        for (long long i = 0; i < ext[0]; ++i)
          out[i + ext[0] * (j + ext[1] * k)] = a[hb.origin + hb.off((int)i, (int)j, (int)k)];
    return BF_OK;
  }
  if (what >= BF_FIELD_PSI && what < BF_FIELD_PSI + 10 * ctx->ndim) {
    if (!ctx->have_psi) return fail(ctx, BF_EINVAL, "limiter arrays are kept only when freezing");
    const int r = what - BF_FIELD_PSI;
    const int d = r / 10, pm = (r % 10) / 5, v = r % 5;
    rc = get(hb.dev.f(hb.dev.psi0 + 10 * d + 5 * pm + v), a);
    if (rc) return rc;
    long long ext[3] = {hb.n[0], hb.n[1], hb.n[2]};
    ext[d] += 2;
    for (long long k = 0; k < ext[2]; ++k)
      for (long long j = 0; j < ext[1]; ++j)
        for (long long i = 0; i < ext[0]; ++i) {
          long long c[3] = {i, j, k};
          c[d] -= 1;
          out[i + ext[0] * (j + ext[1] * k)] = a[hb.origin + hb.off((int)c[0], (int)c[1], (int)c[2])];
        }
    return BF_OK;
  }
  return fail(ctx, BF_EINVAL, "unknown field selector %d", what);
}

int bf_error_info(const bf_ctx* ctx, int* kind, int* block_id, int* stage, int* direction,
                  long long index[3]) {
  if (!ctx) return BF_EINVAL;
  *kind = ctx->e_kind;
  *block_id = ctx->e_block;
  *stage = ctx->e_stage;
  *direction = ctx->e_dir;
  for (int a = 0; a < 3; ++a) index[a] = ctx->e_idx[a];
  return BF_OK;
}

int bf_nccl_unique_id(void* out128) {
  ncclUniqueId id;
  if (!nccl().ok || nccl().GetUniqueId(&id) != ncclSuccess) return BF_ENCCL;
  std::memcpy(out128, &id, sizeof id);
  return BF_OK;
}

int bf_nccl_init(bf_ctx* ctx, const void* id128) {
  if (!ctx) return BF_EINVAL;
  CK(cudaSetDevice(ctx->device));
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  if (!nccl().ok) return fail(ctx, BF_ENCCL, "NCCL unavailable: %s", nccl().err.c_str());
  NK(nccl().CommInitRank(&ctx->comm, ctx->nranks, id, ctx->rank));
  return BF_OK;
}

// ---- loopback transport (bf_loopback.h) -------------------------------------------

bf_loopback* bf_loopback_create(int nranks) {
  if (nranks < 1) return nullptr;
  return reinterpret_cast<bf_loopback*>(new bf_lb::World(nranks));
}

int bf_loopback_init(bf_ctx* ctx, bf_loopback* world) {
  if (!ctx || !world) return BF_EINVAL;
  auto* w = reinterpret_cast<bf_lb::World*>(world);
  if (ctx->finalized) return fail(ctx, BF_EINVAL, "bf_loopback_init after bf_finalize");
  if (ctx->comm) return fail(ctx, BF_EINVAL, "context already has a communicator");
  if (w->n != ctx->nranks)
    return fail(ctx, BF_EINVAL, "loopback world has %d ranks, context expects %d", w->n,
                ctx->nranks);
  ctx->lb_rank = new bf_lb::Rank{w, ctx->rank, 0};
  ctx->comm = reinterpret_cast<ncclComm_t>(ctx->lb_rank);
  ctx->net = &loopback_api();
  return BF_OK;
}

void bf_loopback_abort(bf_loopback* world) {
  if (world) bf_lb::abort(reinterpret_cast<bf_lb::World*>(world));
}

void bf_loopback_destroy(bf_loopback* world) { delete reinterpret_cast<bf_lb::World*>(world); }

// ---- in-process groups --------------------------------------------------------

bf_group* bf_group_create(bf_ctx* const* ctxs, int n) {
  if (!ctxs || n < 1) return nullptr;
  auto* g = new bf_group();
  g->ctxs.assign(n, nullptr);
  for (int i = 0; i < n; ++i) {
    bf_ctx* c = ctxs[i];
    if (!c || c->rank < 0 || c->rank >= n || g->ctxs[c->rank] || !c->finalized) {
      delete g;
      return nullptr;
    }
    g->ctxs[c->rank] = c;
  }
  for (bf_ctx* c : g->ctxs) {
    cudaSetDevice(c->device);
    for (bf_ctx* o : g->ctxs)
      if (o->device != c->device) cudaDeviceEnablePeerAccess(o->device, 0);
    cudaGetLastError();   // already-enabled is fine
    cudaEvent_t a, b;
    cudaEventCreateWithFlags(&a, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&b, cudaEventDisableTiming);
    g->ev_packed.push_back(a);
    g->ev_unpacked.push_back(b);
    c->group = g;
  }
  return g;
}

void bf_group_destroy(bf_group* g) {
  if (!g) return;
  for (size_t i = 0; i < g->ctxs.size(); ++i) {
    cudaSetDevice(g->ctxs[i]->device);
    cudaEventDestroy(g->ev_packed[i]);
    cudaEventDestroy(g->ev_unpacked[i]);
    g->ctxs[i]->group = nullptr;
  }
  delete g;
}

}  // extern "C"

namespace {

// One ghost update of every member: fill+pack on each, push messages into the
// peers' receive buffers, then unpack on each (lock step from one host thread).
int group_ghosts(bf_group* g) {
  const int n = (int)g->ctxs.size();
  for (int r = 0; r < n; ++r) {
    bf_ctx* ctx = g->ctxs[r];
    CK(cudaSetDevice(ctx->device));
    if (!g->first) {
      // do not overwrite a peer's receive buffers before it consumed them
      for (int q = 0; q < n; ++q)
        if (q != r) CK(cudaStreamWaitEvent(ctx->stream, g->ev_unpacked[q], 0));
    }
    if ((ctx->sch.viscous || !ctx->r1_bc.empty()) && ctx->synced_cur != ctx->cur_epoch) {
      int r0 = sync_ghosts_from_other(ctx);
      if (r0) return r0;
      ctx->synced_cur = ctx->cur_epoch;
    }
    int rc = fill_ghosts(ctx);
    if (rc) return rc;
    {
      long long n = 0, b = 0;
      for (auto& L : ctx->links)
        if (L.send) {
          ++n;
          b += (long long)sizeof(double) * L.nfields * L.cells;
        }
      if (n) count_exchange(ctx, n, b);
    }
    for (auto& L : ctx->links) {
      if (!L.send) continue;
      bf_ctx* peer = g->ctxs[L.peer_rank];
      HostLink* match = nullptr;
      for (auto& M : peer->links)
        if (M.send && M.tag == L.tag && M.peer_rank == ctx->rank && M.block == L.peer_block) {
          match = &M;
          break;
        }
      if (!match) return fail(ctx, BF_EINVAL, "link tag %d has no partner on rank %d", L.tag,
                              L.peer_rank);
      CK(cudaMemcpyAsync(match->recv, L.send, sizeof(double) * L.nfields * L.cells,
                         cudaMemcpyDefault, ctx->stream));
    }
    CK(cudaEventRecord(g->ev_packed[r], ctx->stream));
  }
  for (int r = 0; r < n; ++r) {
    bf_ctx* ctx = g->ctxs[r];
    CK(cudaSetDevice(ctx->device));
    for (int q = 0; q < n; ++q)
      if (q != r) CK(cudaStreamWaitEvent(ctx->stream, g->ev_packed[q], 0));
    if (ctx->n_unpack) {
      int rc = launch_unpack(ctx);
      if (rc) return rc;
    }
    for (auto& L : ctx->r1_bc) {
      int rc = run_ghost_launch(ctx, L, 0);
      if (rc) return rc;
    }
    CK(cudaEventRecord(g->ev_unpacked[r], ctx->stream));
    ctx->ghost_buf = ctx->cur;
  }
  if (g->ctxs[0]->sch.viscous) {
    // round 2 (viscous): packs everywhere, messages as peer copies, then ordered
    // unpacks and the extended BCs on each member
    for (int r = 0; r < n; ++r) {
      bf_ctx* ctx = g->ctxs[r];
      CK(cudaSetDevice(ctx->device));
      for (int q = 0; q < n; ++q)
        if (q != r) CK(cudaStreamWaitEvent(ctx->stream, g->ev_unpacked[q], 0));
      int rc = run_ghost_launch(ctx, ctx->r2_pack, 0);
      if (rc) return rc;
      {
        long long n = 0, b = 0;
        for (auto& L : ctx->links)
          if (L.recv2) {
            ++n;
            b += (long long)sizeof(double) * L.nfields * L.cells2;
          }
        if (n) count_exchange(ctx, n, b);
      }
      for (auto& L : ctx->links) {
        if (!L.recv2) continue;
        bf_ctx* peer = g->ctxs[L.peer_rank];
        HostLink* match = nullptr;
        for (auto& M : peer->links)
          if (M.recv2 && M.tag == L.tag && M.peer_rank == ctx->rank && M.block == L.peer_block) {
            match = &M;
            break;
          }
        if (!match) return fail(ctx, BF_EINVAL, "link tag %d has no round-2 partner", L.tag);
        CK(cudaMemcpyAsync(match->recv2, L.send2, sizeof(double) * L.nfields * L.cells2,
                           cudaMemcpyDefault, ctx->stream));
      }
      CK(cudaEventRecord(g->ev_packed[r], ctx->stream));
    }
    for (int r = 0; r < n; ++r) {
      bf_ctx* ctx = g->ctxs[r];
      CK(cudaSetDevice(ctx->device));
      for (int q = 0; q < n; ++q)
        if (q != r) CK(cudaStreamWaitEvent(ctx->stream, g->ev_packed[q], 0));
      for (auto& L : ctx->r2_unpack) {
        int rc = run_ghost_launch(ctx, L, 0);
        if (rc) return rc;
      }
      for (auto& L : ctx->r2_bc) {
        int rc = run_ghost_launch(ctx, L, 1);
        if (rc) return rc;
      }
      CK(cudaEventRecord(g->ev_unpacked[r], ctx->stream));
    }
  }
  g->first = false;
  return BF_OK;
}

}  // namespace

extern "C" {

int bf_group_update_ghosts(bf_group* g) {
  if (!g) return BF_EINVAL;
  int rc = group_ghosts(g);
  if (rc) return rc;
  for (bf_ctx* ctx : g->ctxs) {
    cudaSetDevice(ctx->device);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return BF_ECUDA;
  }
  return BF_OK;
}

int bf_group_step(bf_group* g, int step_index, double* sumsq_out, int* failed_rank) {
  if (!g) return BF_EINVAL;
  *failed_rank = -1;
  const int n = (int)g->ctxs.size();
  const int nst = g->ctxs[0]->sch.rk_stages;
  for (bf_ctx* ctx : g->ctxs) {
    cudaSetDevice(ctx->device);
    int rc = reset_error(ctx);
    if (rc) {
      *failed_rank = ctx->rank;
      return rc;
    }
  }
  for (int k = 0; k < nst; ++k) {
    int rc = group_ghosts(g);
    if (rc) return rc;
    for (bf_ctx* ctx : g->ctxs) {
      cudaSetDevice(ctx->device);
      rc = launch_stage_kernel(ctx, k, stage_flags(ctx, step_index, k, nst), rk_alpha(nst, k));
      if (rc) {
        *failed_rank = ctx->rank;
        return rc;
      }
    }
  }
  double tot[5] = {0, 0, 0, 0, 0};
  for (int r = 0; r < n; ++r) {
    bf_ctx* ctx = g->ctxs[r];
    cudaSetDevice(ctx->device);
    double s[5];
    unsigned long long key;
    int rc = collect(ctx, s, &key);
    if (rc) {
      *failed_rank = r;
      return rc;
    }
    if (key != NO_ERROR) {
      decode_error(ctx, key);
      *failed_rank = r;
      return BF_ENONPHYSICAL;
    }
    for (int v = 0; v < 5; ++v) tot[v] = (r == 0) ? s[v] : tot[v] + s[v];
  }
  for (int v = 0; v < 5; ++v) sumsq_out[v] = tot[v];
  return BF_OK;
}

int bf_set_stream(bf_ctx* ctx, void* cuda_stream) {
  if (!ctx) return BF_EINVAL;
  ctx->stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : ctx->own_stream;
  return BF_OK;
}

int bf_set_profiling(bf_ctx* ctx, int on) {
  if (!ctx) return BF_EINVAL;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  drain_profile(ctx);
  ctx->profiling = on != 0;
  for (int k = 0; k < 4; ++k) {
    ctx->prof_launches[k] = 0;
    ctx->prof_ms[k] = 0.0;
  }
  ctx->prof_kernels = 0;
  return BF_OK;
}

int bf_kernel_stats(bf_ctx* ctx, int kernel_class, long long* launches, double* total_ms) {
  if (!ctx || kernel_class < 0 || kernel_class > 4) return BF_EINVAL;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  drain_profile(ctx);
  if (kernel_class == 4) {   // every kernel launched inside a timed scope
    *launches = ctx->prof_kernels;
    *total_ms = ctx->prof_ms[0] + ctx->prof_ms[1] + ctx->prof_ms[2] + ctx->prof_ms[3];
    return BF_OK;
  }
  *launches = ctx->prof_launches[kernel_class];
  *total_ms = ctx->prof_ms[kernel_class];
  return BF_OK;
}

void bf_release_cache(int device) {
  release_arena_cache(device);
  int n = 0, cur = -1;
  cudaGetDeviceCount(&n);
  cudaGetDevice(&cur);
  for (int d = 0; d < n; ++d) {
    if (device >= 0 && d != device) continue;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  }
  if (cur >= 0) cudaSetDevice(cur);
}

int bf_transfer_counters(const bf_ctx* ctx, long long out[6]) {
  if (!ctx || !out) return BF_EINVAL;
  for (int q = 0; q < 6; ++q) out[q] = ctx->xc[q];
  return BF_OK;
}

long long bf_cache_bytes(int device) {
  ArenaCache& c = arena_cache();
  std::lock_guard<std::mutex> g(c.m);
  long long n = 0;
  for (const auto& e : c.free)
    if (device < 0 || e.dev == device) n += (long long)e.bytes;
  return n;
}

long long bf_transfer_bytes(const bf_ctx* ctx, int direction) {
  if (!ctx) return -1;
  return direction == 0 ? ctx->bytes_h2d : ctx->bytes_d2h;
}

int bf_probe_remote_order(int n, const int* peer_rank, const int* tag, const int* block,
                          int* order_out) {
  if (n < 0 || (n > 0 && (!peer_rank || !tag || !block || !order_out))) return BF_EINVAL;
  std::vector<int> idx(n);
  for (int q = 0; q < n; ++q) idx[q] = q;
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
    return remote_before(peer_rank[a], tag[a], block[a], peer_rank[b], tag[b], block[b]);
  });
  for (int q = 0; q < n; ++q) order_out[q] = idx[q];
  return BF_OK;
}

int bf_probe_unpack_map(const int own_dims[3], int ghost_depth, int ndim, int face,
                        const int box[6], const int axis_map[6], int peer_face, long long* out,
                        long long out_len) {
  const int ghost[3] = {ghost_depth, ghost_depth, ndim == 3 ? ghost_depth : 0};
  int send[6], recv[6];
  halo_boxes(face, box, own_dims, ghost, send, recv);
  int ext[3];
  for (int a = 0; a < 3; ++a) ext[a] = recv[2 * a + 1] - recv[2 * a];
  int perm[3];
  bool flip[3];
  unpack_axes(face, axis_map, peer_face, perm, flip);
  int P[3];
  for (int a = 0; a < 3; ++a) P[perm[a]] = ext[a];
  const long long Pst[3] = {1, P[0], (long long)P[0] * P[1]};
  long long origin = 0, stride[3];
  for (int a = 0; a < 3; ++a) {
    const long long s = Pst[perm[a]];
    if (flip[a]) {
      origin += (long long)(ext[a] - 1) * s;
      stride[a] = -s;
    } else {
      stride[a] = s;
    }
  }
  const long long total = (long long)ext[0] * ext[1] * ext[2];
  if (out_len < total) return BF_EINVAL;
  long long m = 0;
  for (int o2 = 0; o2 < ext[2]; ++o2)
    for (int o1 = 0; o1 < ext[1]; ++o1)
      for (int o0 = 0; o0 < ext[0]; ++o0)
        out[m++] = origin + o0 * stride[0] + o1 * stride[1] + o2 * stride[2];
  return BF_OK;
}

}  // extern "C"
