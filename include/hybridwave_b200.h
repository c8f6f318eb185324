/*
 * hybridwave_b200 — C ABI of the sm_100a DG acoustic right-hand side and
 * time update (drop-in for the hot path of the reference Python package
 * `hybridwave`, which has no native layer of its own: the Python
 * `Discretization.compute_rhs` / `timeint` entry points are what these
 * symbols replace; see INTEGRATION.md for the ctypes binding).
 *
 * Conventions
 *   - every pointer is a device pointer owned by the caller; the library
 *     never allocates device memory;
 *   - per-type state buffers are element-major (K, 4, Np) with fields
 *     (p, u1, u2, u3), Np and node/mode order exactly the reference's
 *     (hybridwave/dg.py:10-13, basis.py:151-155, 289-292, 348-352, 423-429);
 *   - type slots: 0 hex, 1 wedge, 2 pyramid, 3 tet (hybridwave/refelem.py:35);
 *   - return value 0 = success; nonzero = error, message via hw_last_error()
 *     (the Python layer raises ValueError, matching the reference's
 *     exceptions-only error model).
 */
#ifndef HYBRIDWAVE_B200_H
#define HYBRIDWAVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { HW_HEX = 0, HW_WEDGE = 1, HW_PYRAMID = 2, HW_TET = 3, HW_NTYPES = 4 };
enum { HW_F64 = 0, HW_F32 = 1 };
enum { HW_FORM_STRONG = 0, HW_FORM_SKEW = 1 };
enum { HW_GL = 0, HW_SEM = 1 };

/* nbr_code bit layout (one int32 per element face) */
#define HW_NBR_TYPE(c) ((c) & 3)
#define HW_NBR_FACE(c) (((c) >> 2) & 7)
#define HW_NBR_PERM(c) (((c) >> 5) & 15)
#define HW_NBR_BOUNDARY 0x200

/* One element type present in the mesh.  Geometry record per element
 * (scalar type = dtype); dense types carry per face FS = 6 words (n_x, n_y,
 * n_z, Jacobian scale, avg(rho c), 1/avg(rho c)):
 *   hex      72: 8 vertices (x, y, z); per face (avg, 1/avg); affine flag;
 *                if affine: G[3][3], J, per face (n_x, n_y, n_z, Js), 1/J
 *   wedge    40: G[3][3] (G[c][x] = d r_c / d x_x), 1/sqrt(J), 5 faces x FS
 *                (scale = Js/sqrt(J)); non-affine wedges in the mesh: op[8] =
 *                per-element cubature geometry, op[9] = cubature operators
 *                (layout: struct Naw, csrc/hw_kernels.cuh), scalar kernel
 *   pyramid  40: G[3][3], 5 faces x FS (scale = Js/J; non-affine: Js), non-affine
 *                flag (then op[8] = (K, Np, 10) G, J per node, op[9] =
 *                (K, NFQ, 4) base-face normal, Js per point)
 *   tet      33: G[3][3], 4 faces x FS (scale = Js/J)
 * mat: per element (kappa, 1/rho, rho*c, 0).
 * op/iop: constant operators and index tables, layouts documented in
 *   paper_1507_02557_b200/device.py (_pack_ops, _mma_ops, _pack_iops):
 *   iop hex {0 face table, 1 node->face point, 2 face gather index},
 *   tet {0 face nodes, 1 gather index}, wedge/pyramid {1 gather index}. */
typedef struct {
  int64_t K;
  const void* geo;
  const void* mat;
  const int32_t* nbr_elem;   /* (K, nfaces) neighbour element index        */
  const int32_t* nbr_code;   /* (K, nfaces) packed type/face/perm/boundary */
  const void* op[10];
  const int32_t* iop[4];
  int32_t form;              /* HW_FORM_STRONG or HW_FORM_SKEW            */
  int32_t pad_;
} hw_type_t;

typedef struct {
  int32_t N;
  int32_t dtype;             /* HW_F64 / HW_F32                           */
  int32_t formulation;       /* HW_GL / HW_SEM                            */
  int32_t device;            /* CUDA ordinal the buffers live on: made     *
                              * current for each call (-1: leave as is)   */
  double penalty_scale;      /* hybridwave/dg.py:341-342                  */
  const int32_t* perm_tri;   /* (6, (N+1)(N+2)/2) face-point permutations */
  const int32_t* perm_quad;  /* (8, (N+1)^2)                              */
  /* Face-trace buffers (K, 4, Nfp) of the publishing types (wedge, pyramid,
   * and hex under GL; NULL for the others): tr_in holds the traces of the
   * input state of a stage, tr_out receives those of its output state
   * (LSRK / AB epilogue; may be NULL).  hw_rhs fills tr_in itself; before
   * the first hw_lsrk_stage / hw_ab_step call hw_traces. */
  void* tr_in[HW_NTYPES];
  void* tr_out[HW_NTYPES];
  hw_type_t t[HW_NTYPES];
  /* Optional extra RHS term per type, state layout (K, 4, Np) (NULL:
   * none): hw_rhs / hw_lsrk_stage / hw_ab_step add it to dU/dtau in their
   * epilogue, so the published traces of the new state include it.  Filled
   * by hw_forcing (assign = 1: the pressure forcing) and
   * hw_wedge_face_correction (accumulating). */
  const void* frc[HW_NTYPES];
} hw_mesh_t;

/* per-type buffers, NULL for absent types */
typedef struct {
  void* p[HW_NTYPES];
} hw_fields_t;

/* optional per-type element subsets (multi-rate: active levels only);
 * n[t] < 0 means "all elements of type t" */
typedef struct {
  const int32_t* idx[HW_NTYPES];
  int64_t n[HW_NTYPES];
} hw_subset_t;

/* dU/dtau = diag(kappa, 1/rho) M^-1 (A U) — replaces
 * Discretization.compute_rhs (hybridwave/dg.py:492-506, forcing = None). */
int hw_rhs(const hw_mesh_t* mesh, const hw_fields_t* q, hw_fields_t* rhs,
           const hw_subset_t* subset, void* stream);

/* Face traces of q for the publishing types into tr (same layout as
 * mesh->tr_in); the state's traces at the device face points. */
int hw_traces(const hw_mesh_t* mesh, const hw_fields_t* q, hw_fields_t* tr,
              const hw_subset_t* subset, void* stream);

/* One low-storage RK stage (Carpenter-Kennedy (4,5), 2N storage):
 *   res = a*res + dt*rhs(q_in);  q_out = q_in + b*res.
 * q_in and q_out must be distinct (neighbours read q_in). */
int hw_lsrk_stage(const hw_mesh_t* mesh, const hw_fields_t* q_in,
                  hw_fields_t* q_out, hw_fields_t* res, double a, double b,
                  double dt, const hw_subset_t* subset, void* stream);

/* One Adams-Bashforth step with n_hist (1..3) slopes — replaces
 * ab3_step(single_rate_run) (hybridwave/timeint.py:41-72):
 *   h0 = rhs(q_in);  q_out = q_in + dt*(c0*h0 + c1*h1 + c2*h2). */
int hw_ab_step(const hw_mesh_t* mesh, const hw_fields_t* q_in,
               hw_fields_t* q_out, hw_fields_t* h0, const hw_fields_t* h1,
               const hw_fields_t* h2, int n_hist, double c0, double c1,
               double c2, double dt, const hw_subset_t* subset, void* stream);

/* Multi-rate AB3 support (hybridwave/timeint.py:111-173):
 * out = q + dt_lev * (c0*h0 + c1*h1 + c2*h2) on the listed elements of
 * every type (the dense-output "effective state" of non-stepping levels and
 * the per-level state update). */
int hw_axpy3(const hw_mesh_t* mesh, const hw_fields_t* q, hw_fields_t* out,
             const hw_fields_t* h0, const hw_fields_t* h1,
             const hw_fields_t* h2, int n_hist, double c0, double c1,
             double c2, double dt, const hw_subset_t* subset, void* stream);

/* history shift on the listed elements: h2 <- h1, h1 <- h0, h0 <- rhs */
int hw_hist_push(const hw_mesh_t* mesh, hw_fields_t* h0, hw_fields_t* h1,
                 hw_fields_t* h2, const hw_fields_t* rhs,
                 const hw_subset_t* subset, void* stream);

/* Pack partition-interface state for the halo exchange: for each listed
 * element, copy its (4, Np) state into the contiguous send buffer. */
int hw_halo_pack(const hw_mesh_t* mesh, int elem_type, const void* q,
                 const int32_t* idx, int64_t n, void* sendbuf, void* stream);

/* Forcing residual of the pressure equation, integrated on the device
 * (replaces Discretization._forcing_residual + its mass inverse and kappa,
 * hybridwave/dg.py:497-515, 479-490).  f: (K, nq) fp64 values of the forcing
 * at the type's cubature points (evaluated by the caller, on the device or
 * copied in); B: (Np, nq) = [invM_ref] V^T diag(w); scale: (K, nq) = J
 * (sqrt(J) for wedges) at the cubature points; nodefac: (K, Np) per-node
 * mass inverse (1/(w3 J) hex, 1/J tet and pyramid, 1 wedge).  Adds alpha*F
 * to the p field of out1 and beta*F to that of out2 (NULL: none): the RHS
 * (alpha 1), or an LSRK stage's residual (h) and new state (b h), or an AB
 * step's new slope (1) and new state (dt c0).  assign = 1: out1 = alpha*F
 * (p field; out2 unused) — the forcing buffer of hw_mesh_t.frc. */
int hw_forcing(const hw_mesh_t* mesh, int elem_type, const double* f,
               const double* B, const double* scale, const double* nodefac,
               int nq, double alpha, void* out1, double beta, void* out2,
               int assign, void* stream);

/* Tet and pyramid faces across a triangle of a non-affine (LSC-DG) wedge
 * (elem_type HW_TET or HW_PYRAMID): adds to the extra-RHS buffer `out`
 * (state layout, all four fields; installed as mesh->frc) the difference
 * between the reference's face-cubature surface integral
 * (hybridwave/dg.py:326-354 at the stored 6(N+1)^2 points, wedge trace
 * q/sqrt(J)) and the kernel's nodal lift of the unscaled wedge trace.  One
 * row per (element, face): idata [elem, face, nb_off[nfn]] (offsets of the
 * wedge's published triangle trace at my face nodes in
 * mesh->tr_in[HW_WEDGE], field 0), fdata [avg(rho c), 1/avg, n(3), Js,
 * s-1 at the nq points, 1/J per node]; L (nfaces, nq, nfn)
 * nodal-to-cubature interpolants, P (nfaces, Np, nq) = [invM_ref] Vf_f^T
 * diag(w) (tets: with invM_ref; pyramids: orthonormal basis, without)
 * (layout: paper_1507_02557_b200/device.py wedge_face_corrections). */
int hw_wedge_face_correction(const hw_mesh_t* mesh, int elem_type, int n_pairs,
                             const int32_t* idata, const double* fdata,
                             const double* L, const double* P, int nq, int nfn,
                             void* out, void* stream);

/* Face-level halo exchange of partitioned runs (no reference counterpart:
 * the reference has no distributed path).  A
 * partition-boundary element's neighbour across the cut is a ghost whose
 * only data the kernels read is the shared face: its face nodes (tet, SEM
 * hex state) or its published face traces (wedge, pyramid, GL hex).
 * gather: buf[c*n + i] = src[off[i] + c*stride];  scatter: dst[off[i] +
 * c*stride] = buf[c*n + i]  (c = 0..3 fields; off = flat element-row
 * offsets of field 0, stride = Np for states, Nfp for trace buffers). */
int hw_halo_gather(const hw_mesh_t* mesh, const void* src, int64_t stride,
                   const int64_t* off, int64_t n, void* buf, void* stream);
int hw_halo_scatter(const hw_mesh_t* mesh, const void* buf, int64_t stride,
                    const int64_t* off, int64_t n, void* dst, void* stream);

/* Discrete energy U^T M U with material weights (p^2 / kappa + rho |u|^2)
 * per element type (discrete_energy, hybridwave/dg.py:655-674).  out is a
 * DEVICE pointer to HW_NTYPES doubles: zeroed on `stream`, then one sum
 * per type slot (asynchronous, graph-capturable). */
int hw_energy(const hw_mesh_t* mesh, const hw_fields_t* q, double* out,
              void* stream);

/* One-time per-mesh setup on the mesh's device (synchronous; call once
 * after filling hw_mesh_t, before the first launch and outside any CUDA
 * graph capture): uploads the order/formulation constant tables the
 * kernels read from constant memory (hex node -> face-point map). */
int hw_prepare(const hw_mesh_t* mesh);

const char* hw_last_error(void);
int hw_version(void);
/* kernel launches this library has issued so far (all devices, all
 * threads; captured launches count once, at capture, not per graph replay).
 * Instrumentation for the benchmark's gpu_launches; no reference
 * counterpart. */
long long hw_launch_count(void);
/* the N values compiled into this library (bit N set) */
int hw_supported_orders(void);

#ifdef __cplusplus
}
#endif
#endif
