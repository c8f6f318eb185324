// Shared device-side definitions of the sm_100a DG acoustic kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/hybridwave_b200.h"

namespace hw {

constexpr int NT = 256;  // threads per block of the scalar dense and trace kernels

template <int N>
struct Dims {
  static constexpr int N1 = N + 1;
  static constexpr int NFQ = N1 * N1;                      // quad face points
  static constexpr int NFN = (N + 1) * (N + 2) / 2;        // tri face nodes
  static constexpr int NP_HEX = N1 * N1 * N1;
  static constexpr int NP_TET = (N + 1) * (N + 2) * (N + 3) / 6;
  static constexpr int NP_WEDGE = N1 * N1 * (N + 2) / 2;
  static constexpr int NP_PYR = (N + 1) * (N + 2) * (2 * N + 3) / 6;
  static constexpr int NQ_WEDGE = N1 * N1 * N1;
  static constexpr int NFP_HEX = 6 * NFQ;
  static constexpr int NFP_TET = 4 * NFN;
  static constexpr int NFP_WEDGE = 2 * NFN + 3 * NFQ;
  static constexpr int NFP_PYR = NFQ + 4 * NFN;
};

// geometry record words per element.  Dense types: G[3][3] (+ 1/sqrt(J)
// for wedges) then per face FS words (n_x, n_y, n_z, Jacobian scale,
// avg(rho c), 1/avg(rho c)).  Hex: 8 vertices, per face (avg, 1/avg), an
// affine flag, then for affine hexes G[3][3], J and per face (n, Js).
constexpr int FS = 6;
// pyramid: word 39 = non-affine flag (per-node geometry in op[8], base-face
// points in op[9]; scalar kernel)
constexpr int PY_NAFF = 9 + 5 * FS;
constexpr int GEO_HEX = 72, GEO_WEDGE = 10 + 5 * FS, GEO_PYR = 9 + 5 * FS + 1,
              GEO_TET = 9 + 4 * FS;
constexpr int HX_Z = 24, HX_AFF = 36, HX_G = 37, HX_J = 46, HX_F = 47, HX_IJ = 71;
constexpr int NF_HEX = 6, NF_WEDGE = 5, NF_PYR = 5, NF_TET = 4;

// epilogue of the fused RHS kernels
enum { MODE_RHS = 0, MODE_LSRK = 1, MODE_AB = 2 };

struct Epi {
  int mode;
  int nhist;
  double a, b, dt, c0, c1, c2;
  void* out[HW_NTYPES];        // rhs (MODE_RHS) / new slope h0 (MODE_AB)
  void* res[HW_NTYPES];        // LSRK residual (in/out)
  void* qout[HW_NTYPES];       // advanced state
  const void* h1[HW_NTYPES];
  const void* h2[HW_NTYPES];
  const void* frc[HW_NTYPES];  // extra RHS term (state layout: forcing, face corrections)
};

// extra RHS term at the flat state index `base` (0 without one)
template <typename S>
__device__ __forceinline__ S frc_at(const Epi& E, int t, size_t base) {
  return E.frc[t] ? ((const S*)E.frc[t])[base] : S(0);
}

template <int N>
__device__ __forceinline__ int face_offset(int t, int f) {
  using D = Dims<N>;
  switch (t) {
    case HW_HEX: return f * D::NFQ;
    case HW_TET: return f * D::NFN;
    case HW_WEDGE: return f < 2 ? f * D::NFN : 2 * D::NFN + (f - 2) * D::NFQ;
    default: return f == 0 ? 0 : D::NFQ + (f - 1) * D::NFN;  // pyramid
  }
}

template <int N>
__host__ __device__ constexpr int n_face_points(int t) {
  return t == HW_HEX ? Dims<N>::NFP_HEX
       : t == HW_TET ? Dims<N>::NFP_TET
       : t == HW_WEDGE ? Dims<N>::NFP_WEDGE : Dims<N>::NFP_PYR;
}

template <int N>
__host__ __device__ constexpr int n_dofs(int t) {
  return t == HW_HEX ? Dims<N>::NP_HEX
       : t == HW_TET ? Dims<N>::NP_TET
       : t == HW_WEDGE ? Dims<N>::NP_WEDGE : Dims<N>::NP_PYR;
}

template <typename R>
__device__ __forceinline__ R ldg(const R* p) { return __ldg(p); }
__device__ __forceinline__ double2 ldg2(const double* p) {   // 16-byte aligned pair
  return __ldg(reinterpret_cast<const double2*>(p));
}

// Upwind flux of the acoustic system at one face point, own side (-) and
// neighbour side (+), with my outward normal n (hybridwave/dg.py:337-350).
template <typename R>
__device__ __forceinline__ void upwind_flux(R pm, const R um[3], R pp, const R up[3],
                                            const R n[3], R tau_p, R tau_u, bool skew,
                                            R& flux_p, R& flux_un) {
  R dp = pp - pm;
  R unm = n[0] * um[0] + n[1] * um[1] + n[2] * um[2];
  R unp = n[0] * up[0] + n[1] * up[1] + n[2] * up[2];
  R dun = unp - unm;
  flux_p = skew ? (R(0.5) * tau_p * dp - R(0.5) * (unp + unm))
                : R(0.5) * (tau_p * dp - dun);
  flux_un = R(0.5) * (tau_u * dun - dp);
}

// penalties from avg(rho c) of the two sides (hybridwave/dg.py:61-69,
// 341-342); avg is precomputed per face on the host
template <typename R>
__device__ __forceinline__ void penalties(R avg, R inv_avg, R scale, R& tp, R& tu) {
  tp = scale * inv_avg;
  tu = scale * avg;
}

// Neighbour-side trace at my face point jj: the neighbour element's state
// evaluated at its own face point p = perm[jj] (coincident with mine).
// Reads the neighbour's coefficients straight from the input state (L2
// resident for mesh-ordered elements); there is no trace buffer.
template <int N, typename R>
__device__ __forceinline__ void neighbour_trace(const hw_mesh_t& M, const hw_fields_t& Q,
                                                int code, int k2, int jj, bool tri,
                                                R tr[4]) {
  using D = Dims<N>;
  const int t2 = HW_NBR_TYPE(code), f2 = HW_NBR_FACE(code), pc = HW_NBR_PERM(code);
  const int p = tri ? __ldg(M.perm_tri + pc * D::NFN + jj)
                    : __ldg(M.perm_quad + pc * D::NFQ + jj);
  if (t2 == HW_TET) {
    const R* q2 = (const R*)Q.p[HW_TET] + (size_t)k2 * 4 * D::NP_TET;
    const int node = __ldg(M.t[HW_TET].iop[0] + f2 * D::NFN + p);
#pragma unroll
    for (int c = 0; c < 4; ++c) tr[c] = ldg(q2 + c * D::NP_TET + node);
  } else if (t2 == HW_HEX) {
    const R* q2 = (const R*)Q.p[HW_HEX] + (size_t)k2 * 4 * D::NP_HEX;
    const int* tab = M.t[HW_HEX].iop[0] + 3 * (f2 * D::NFQ + p);
    const int base = __ldg(tab), stride = __ldg(tab + 1), end = __ldg(tab + 2);
    if (M.formulation == HW_SEM) {
      const int node = base + (end ? N : 0) * stride;
#pragma unroll
      for (int c = 0; c < 4; ++c) tr[c] = ldg(q2 + c * D::NP_HEX + node);
    } else {
      const R* ve = (const R*)M.t[HW_HEX].op[1] + end * D::N1;
#pragma unroll
      for (int c = 0; c < 4; ++c) tr[c] = R(0);
#pragma unroll
      for (int l = 0; l < D::N1; ++l) {
        const R w = ldg(ve + l);
#pragma unroll
        for (int c = 0; c < 4; ++c) tr[c] += w * ldg(q2 + c * D::NP_HEX + base + l * stride);
      }
    }
  } else {
    // dense trace operators (wedge, pyramid): E^T stored (Np, Nfp)
    const int np = (t2 == HW_WEDGE) ? D::NP_WEDGE : D::NP_PYR;
    const int nfp = (t2 == HW_WEDGE) ? D::NFP_WEDGE : D::NFP_PYR;
    const R* q2 = (const R*)Q.p[t2] + (size_t)k2 * 4 * np;
    const R* ET = (const R*)M.t[t2].op[5] + face_offset<N>(t2, f2) + p;
#pragma unroll
    for (int c = 0; c < 4; ++c) tr[c] = R(0);
    for (int m = 0; m < np; ++m) {
      const R e = ldg(ET + (size_t)m * nfp);
#pragma unroll
      for (int c = 0; c < 4; ++c) tr[c] += e * ldg(q2 + c * np + m);
    }
    if (t2 == HW_WEDGE) {
      const R s = ldg((const R*)M.t[HW_WEDGE].geo + (size_t)k2 * GEO_WEDGE + 9);
#pragma unroll
      for (int c = 0; c < 4; ++c) tr[c] *= s;
    }
  }
}

// Epilogue: value v = dU/dtau at (type t, flat index idx) with q_in value qv.
template <typename R>
__device__ __forceinline__ void epilogue(const Epi& E, int t, size_t idx, R v, R qv) {
  if (E.mode == MODE_RHS) {
    ((R*)E.out[t])[idx] = v;
  } else if (E.mode == MODE_LSRK) {
    R* res = (R*)E.res[t];
    const R r = R(E.a) * res[idx] + R(E.dt) * v;
    res[idx] = r;
    ((R*)E.qout[t])[idx] = qv + R(E.b) * r;
  } else {
    ((R*)E.out[t])[idx] = v;
    R acc = R(E.c0) * v;
    if (E.nhist > 1) acc += R(E.c1) * ((const R*)E.h1[t])[idx];
    if (E.nhist > 2) acc += R(E.c2) * ((const R*)E.h2[t])[idx];
    ((R*)E.qout[t])[idx] = qv + R(E.dt) * acc;
  }
}

// ------------------------------------------------------------------ TMA bulk copies
// 1-D bulk copies (cp.async.bulk, SASS UBLKCP) between global memory and
// shared memory, completed through an mbarrier (loads) or a bulk group
// (stores).  The TMA engine moves the bytes: no LSU instructions and no L1
// data-pipe wavefronts per element row, which is the resource the stage
// kernels are bound by.  Sizes and both addresses must be multiples of 16 B.

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

// make the initialised barrier visible to the async proxy (TMA)
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_store(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n"); }

// the issuing thread waits until its bulk stores have READ their shared
// memory (the CTA's shared memory must outlive them)
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

// generic-proxy shared-memory writes -> visible to a following bulk store
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

}  // namespace hw
